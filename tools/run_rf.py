"""One range-finder call (config-4 shape by default) for launch profiling."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
if os.environ.get('RANDLA_VARIANT_LIB'):  # dev A/B: a variant library from tools/build_variant.sh
    capi.LIB_PATH = os.environ['RANDLA_VARIANT_LIB']
    capi._lib = None
m = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
r = int(sys.argv[3]) if len(sys.argv) > 3 else 64
kind = capi.RL_MULT_GAUSSIAN if (len(sys.argv) <= 4 or sys.argv[4] == "g") else capi.RL_MULT_GAUSSIAN_CIRCULANT
L = capi.lib()
L.rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
g = torch.Generator(device="cuda").manual_seed(0)
u = torch.linalg.qr(torch.randn(m, r, dtype=torch.float64, device="cuda", generator=g))[0]
v = torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g))[0]
s = torch.logspace(0, -2, r, dtype=torch.float64, device="cuda")
a = (u * s) @ v.T + 1e-10 * torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
q = a.new_empty(m, r)
mlt = capi.rl_multiplier(); mlt.kind = kind; mlt.seed = 41
info = capi.rl_lowrank_info()
for _ in range(2):
    rc = L.rl_range_find_residual(None, capi.RL_DEVICE, m, n, a.data_ptr(), r, ctypes.byref(mlt), 0, q.data_ptr(), ctypes.byref(info))
    if not os.environ.get('RANDLA_VARIANT_LIB'):
        assert rc == 0, capi.last_error()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
L.rl_range_find_residual(None, capi.RL_DEVICE, m, n, a.data_ptr(), r, ctypes.byref(mlt), 0, q.data_ptr(), ctypes.byref(info))
e1.record(); e1.synchronize()
print(f"range_find {m}x{n} r={r}: {e0.elapsed_time(e1):.2f} ms, its {info.power_iterations}, fro {info.residual_frobenius:.3e} spec {info.residual_spectral:.3e}")
