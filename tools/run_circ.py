import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
L = capi.lib()
L.rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); c = torch.randn(n, dtype=torch.float64, device="cuda")
o = torch.empty_like(a)
for _ in range(2): assert L.rl_circulant_right_multiply(None, 1, n, n, a.data_ptr(), c.data_ptr(), o.data_ptr()) == 0
torch.cuda.synchronize(); print("ok")
