import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
a.diagonal().add_(2.0 * n ** 0.5)
lu = torch.empty_like(a)
info = capi.rl_solve_info()
L = capi.lib()
L.rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
rc = L.rl_genp_factor(None, 1, n, a.data_ptr(), lu.data_ptr(), ctypes.byref(info))
print("rc", rc, capi.last_error(), "minpiv", info.min_abs_pivot)
