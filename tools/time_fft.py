import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
if os.environ.get('RANDLA_VARIANT_LIB'):  # dev A/B: a variant library from tools/build_variant.sh
    capi.LIB_PATH = os.environ['RANDLA_VARIANT_LIB']
    capi._lib = None
L = capi.lib()
L.rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
def timeit(f, k=5):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): f()
    e1.record(); e1.synchronize(); return e0.elapsed_time(e1) / k
# config 3: 8192 x 8192 circulant
n = 8192
g = torch.Generator(device="cuda"); g.manual_seed(5)
a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g); c = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
o = torch.empty_like(a)
ms = timeit(lambda: L.rl_circulant_right_multiply(None, 1, n, n, a.data_ptr(), c.data_ptr(), o.data_ptr()))
print("checksum", float(o.abs().sum()), float(o[17, :5].sum()))
print(f"circulant 8192x8192: {ms:.3f} ms, {2*8*n*n/ms/1e6:.1f} GB/s ({2*8*n*n/ms/1e6/6534.5*100:.1f}% HBM)")
del a, o
m, k, l = 32768, 16384, 256
a = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g); c = torch.randn(k, dtype=torch.float64, device="cuda", generator=g)
o = torch.empty(m, l, dtype=torch.float64, device="cuda")
ms = timeit(lambda: L.rl_toeplitz_right_multiply(None, 1, m, k, a.data_ptr(), k, c.data_ptr(), l, o.data_ptr()), 3)
byt = 8*m*k + 8*m*l
print("checksum", float(o.abs().sum()), float(o[17, :5].sum()))
print(f"toeplitz 32768x16384 -> 256: {ms:.3f} ms, {byt/ms/1e6:.1f} GB/s ({byt/ms/1e6/6534.5*100:.1f}% HBM)")
