import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)
L = capi.lib()
L.rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
def run():
    assert L.rl_dgemm(None, 1, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n) == 0, capi.last_error()
for _ in range(2): run()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
K = 5
e0.record()
for _ in range(K): run()
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / K
print(f"dgemm n={n}: {ms:.3f} ms, {2*n**3/ms/1e9:.2f} TF/s ({2*n**3/ms/1e9/35.46*100:.1f}% of cuBLAS 35.46)")
ref = a @ b
print("max err", (c - ref).abs().max().item())
