import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
if os.environ.get("RANDLA_VARIANT_LIB"):
    capi.LIB_PATH = os.environ["RANDLA_VARIANT_LIB"]
    capi._lib = None
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
lu = torch.randn(n, n, dtype=torch.float64, device="cuda") / n
lu.diagonal().add_(1.0)
b = torch.randn(n, dtype=torch.float64, device="cuda"); x = torch.empty_like(b)
L = capi.lib()
L.rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
def run(): assert L.rl_lu_solve(None, 1, n, lu.data_ptr(), b.data_ptr(), x.data_ptr()) == 0
run(); torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); e1.synchronize()
print(f"lu_solve n={n}: {e0.elapsed_time(e1):.3f} ms")
Lm = torch.tril(lu, -1) + torch.eye(n, dtype=lu.dtype, device="cuda"); U = torch.triu(lu)
ref = torch.linalg.solve_triangular(U, torch.linalg.solve_triangular(Lm, b[:, None], upper=False, unitriangular=True), upper=True)[:, 0]
print("rel err", ((x - ref).norm() / ref.norm()).item())
