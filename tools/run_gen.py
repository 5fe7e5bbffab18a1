import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
L = capi.lib()
n = 8192
g = torch.empty(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    assert L.rl_gen_gaussian_device(None, n, n, 2, g.data_ptr(), n, None) == 0
torch.cuda.synchronize(); print("ok")
