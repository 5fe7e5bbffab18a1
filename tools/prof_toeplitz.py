"""One config-5-shaped Toeplitz sketch (for ncu): 32768 x 16384 -> 256."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_5802_b200 import capi
L = capi.lib()
L.rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
m, k, l = int(os.environ.get("M", 32768)), 16384, 256
g = torch.Generator(device="cuda"); g.manual_seed(5)
a = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g)
c = torch.randn(k, dtype=torch.float64, device="cuda", generator=g)
o = torch.empty(m, l, dtype=torch.float64, device="cuda")
for _ in range(2):
    assert L.rl_toeplitz_right_multiply(None, 1, m, k, a.data_ptr(), k, c.data_ptr(), l, o.data_ptr()) == 0
torch.cuda.synchronize()
print("ok")
