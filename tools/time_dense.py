import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi
if os.environ.get('RANDLA_VARIANT_LIB'):
    capi.LIB_PATH = os.environ['RANDLA_VARIANT_LIB']
    capi._lib = None
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
t0 = time.time()
a = torch.from_numpy(rl.gen_gaussian(n, n, 1)).cuda()
g = torch.from_numpy(rl.gen_gaussian(n, n, 2)).cuda()
b = torch.from_numpy(rl.gen_gaussian_vector(n, 3)).cuda()
print("gen+upload s", time.time() - t0)
x = torch.empty_like(b)
L = capi.lib()
L.rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
m = capi.rl_multiplier(); m.kind = 1; m.dense = g.data_ptr()
info = capi.rl_solve_info()
def run():
    rc = L.rl_preprocessed_genp_solve(None, 1, n, a.data_ptr(), b.data_ptr(), None, ctypes.byref(m), 0, x.data_ptr(), None, 0, ctypes.byref(info))
    assert rc == 0, capi.last_error()
run(); torch.cuda.synchronize()
for rep in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.time(); e0.record(); run(); e1.record(); e1.synchronize(); w = time.time() - w0
    ms = e0.elapsed_time(e1)
    F = (2*n**3 - n**2) + sum(mm*(1+2*mm) for mm in range(n)) + 2*n**2 + (2*n**2 - n)
    print(f"preprocess_solve n={n}: {ms:.2f} ms (wall {w*1e3:.2f}), {F/ms/1e9:.2f} TF/s ({F/ms/1e9/35.46*100:.1f}% of 35.46); resid {info.residual_history[0]:.3e} growth {info.growth:.3e} minpiv {info.min_abs_pivot:.3e}")
# component timing
P = torch.empty_like(a)
def t(f, k=3):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): f()
    e1.record(); e1.synchronize(); return e0.elapsed_time(e1)/k
gm = t(lambda: L.rl_dgemm(None, 1, n, n, n, a.data_ptr(), n, g.data_ptr(), n, P.data_ptr(), n))
print(f"  dgemm {gm:.2f} ms ({2*n**3/gm/1e9:.2f} TF/s)")
lu = torch.empty_like(a); inf2 = capi.rl_solve_info()
def fac():
    P2 = P.clone()
    assert L.rl_genp_factor(None, 1, n, P2.data_ptr(), lu.data_ptr(), ctypes.byref(inf2)) == 0, capi.last_error()
fm = t(fac, 2)
print(f"  genp_factor (incl. 2 copies + stats) {fm:.2f} ms ({2*n**3/3/fm/1e9:.2f} TF/s)")
sm = t(lambda: L.rl_lu_solve(None, 1, n, lu.data_ptr(), b.data_ptr(), x.data_ptr()))
print(f"  lu_solve {sm:.3f} ms")
