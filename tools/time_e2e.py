"""Break down the end-to-end (host buffers) dense solve: device generator,
pinned H2D bandwidth, full e2e call."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
if os.environ.get('RANDLA_VARIANT_LIB'):  # dev A/B: a variant library from tools/build_variant.sh
    capi.LIB_PATH = os.environ['RANDLA_VARIANT_LIB']
    capi._lib = None
L = capi.lib()
n = 8192
g = torch.empty(n, n, dtype=torch.float64, device="cuda")
hard = ctypes.c_int64(0)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    assert L.rl_gen_gaussian_device(None, n, n, 2, g.data_ptr(), n, ctypes.byref(hard)) == 0
    torch.cuda.synchronize(); print(f"gen_gaussian_device 8192^2: {(time.perf_counter()-t0)*1e3:.2f} ms, hard {hard.value} ({hard.value/(n*n/2)*100:.2f}% of pairs)")
h = torch.empty(n, n, dtype=torch.float64).pin_memory()
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g.copy_(h, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"pinned H2D 512 MiB: {dt*1e3:.2f} ms = {n*n*8/dt/1e9:.1f} GB/s")
t0 = time.perf_counter(); hv = np.empty((n, n)); L.rl_gen_gaussian(n, n, 2, hv.ctypes.data); print(f"host gen: {(time.perf_counter()-t0)*1e3:.1f} ms, threads {os.cpu_count()}")
hA = torch.from_numpy(np.random.default_rng(1).standard_normal((n, n))).pin_memory()
hb = torch.from_numpy(np.random.default_rng(2).standard_normal(n)).pin_memory()
hx = torch.empty(n, dtype=torch.float64).pin_memory()
m2 = capi.rl_multiplier(); m2.kind = capi.RL_MULT_GAUSSIAN; m2.seed = 2
info = capi.rl_solve_info()
for i in range(3):
    t0 = time.perf_counter()
    rc = L.rl_preprocessed_genp_solve(None, capi.RL_HOST, n, hA.data_ptr(), hb.data_ptr(), None, ctypes.byref(m2), 0, hx.data_ptr(), None, 0, ctypes.byref(info))
    dt = time.perf_counter() - t0
    print(f"e2e: {dt*1e3:.2f} ms rc={rc} stages {[round(x,2) for x in info.stage_ms]}")
