import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
if os.environ.get('RANDLA_VARIANT_LIB'):  # dev A/B: a variant library from tools/build_variant.sh
    capi.LIB_PATH = os.environ['RANDLA_VARIANT_LIB']
    capi._lib = None
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
torch.manual_seed(0)
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
a.diagonal().add_(2.0 * n ** 0.5)
lu = torch.empty_like(a)
info = capi.rl_solve_info()
L = capi.lib()
L.rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
reps = int(os.environ.get("GENP_REPS", "1"))
rc = L.rl_genp_factor(None, 1, n, a.data_ptr(), lu.data_ptr(), ctypes.byref(info))
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    rc = L.rl_genp_factor(None, 1, n, a.data_ptr(), lu.data_ptr(), ctypes.byref(info))
e1.record(); e1.synchronize()
print(f"genp_factor n={n}: {e0.elapsed_time(e1) / reps:.3f} ms/call (incl. verdict), checksum {float(lu.abs().sum()):.17g}")
print("rc", rc, capi.last_error(), "minpiv", info.min_abs_pivot)
