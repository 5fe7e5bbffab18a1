"""Quick device timing of the batched 32x32 kernel (config 2) — dev tool."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time
import numpy as np
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
if os.environ.get('RANDLA_VARIANT_LIB'):  # dev A/B: a variant library from tools/build_variant.sh
    capi.LIB_PATH = os.environ['RANDLA_VARIANT_LIB']
    capi._lib = None

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
t0 = time.time()
seeds = np.array([[rl.derive_seed(7 + i, k) for k in (1, 2, 3)] for i in range(n)], dtype=np.uint64)
a = rl.gen_gaussian_batch(n, 32, 32, seeds[:, 0])
b = rl.gen_gaussian_batch(n, 32, 1, seeds[:, 1]).reshape(n, 32)
g = rl.gen_gaussian_batch(n, 32, 32, seeds[:, 2])
print("gen s", time.time() - t0)
da, dg, db = (torch.from_numpy(t).cuda() for t in (a, g, b))
lu = torch.empty_like(da); x = torch.empty_like(db)
r = torch.empty(n, dtype=torch.float64, device="cuda"); gr = torch.empty_like(r)
st = torch.empty(n, dtype=torch.int32, device="cuda")
L = capi.lib()
s = torch.cuda.current_stream()
L.rl_context_set_stream(None, ctypes.c_void_p(s.cuda_stream))
def run():
    rc = L.rl_batched_genp_solve_32(None, 1, n, da.data_ptr(), dg.data_ptr(), db.data_ptr(), lu.data_ptr(),
                                    x.data_ptr(), r.data_ptr(), gr.data_ptr(), st.data_ptr(), None)
    assert rc == 0, capi.last_error()
for _ in range(3): run()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
K = int(os.environ.get("TB_K", "20"))
e0.record()
for _ in range(K): run()
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / K
byts = n * 25104
print(f"batched32: {ms:.4f} ms/batch, {n/ms*1e3:.3e} solves/s, {byts/ms/1e6:.1f} GB/s ({byts/ms/1e6/6534.5*100:.1f}% of 6534.5)")
print("checksum x", float(x.abs().sum()), "lu", float(lu.abs().sum()))
print("zero pivots", int((st != 0).sum()), "max resid", float(r.max()), "median", float(r.median()))
