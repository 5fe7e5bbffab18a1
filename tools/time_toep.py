"""Device timing of the config-5 Toeplitz sketch Y = A T (32768 x 16384 -> 256,
overlap-save kernel) with a float64 torch check of a few rows — dev tool."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
if os.environ.get('RANDLA_VARIANT_LIB'):
    capi.LIB_PATH = os.environ['RANDLA_VARIANT_LIB']
    capi._lib = None
L = capi.lib()
L.rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
m, k, l = 32768, 16384, 256
g = torch.Generator(device="cuda").manual_seed(5)
a = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g)
c = torch.randn(k, dtype=torch.float64, device="cuda", generator=g)
o = torch.empty(m, l, dtype=torch.float64, device="cuda")
run = lambda: L.rl_toeplitz_right_multiply(None, 1, m, k, a.data_ptr(), k, c.data_ptr(), l, o.data_ptr())
for _ in range(3): assert run() == 0
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): run()
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 10
# T[t, j] = c[(t - j) mod k] (the leading k x l block of the circulant)
idx = (torch.arange(k, device="cuda")[:, None] - torch.arange(l, device="cuda")[None, :]) % k
T = c[idx]
rows = torch.arange(0, m, 997, device="cuda")
ref = a[rows] @ T
err = float((o[rows] - ref).norm() / ref.norm())
print(f"toeplitz sketch {m}x{k}->{l}: {ms:.3f} ms, {m*k*8/ms/1e6:.0f} GB/s, rel err vs torch {err:.2e}")
