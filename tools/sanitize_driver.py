"""Small-shape driver for compute-sanitizer (racecheck / memcheck / synccheck):
one call of each kernel family whose shared-memory protocol could race --
the TMA + mbarrier DGEMM ring, the fused GENP panel kernels (lu_panel64 with
its two-steps-per-barrier diagonal block and the L11^-1 CTA), the clustered
power_pass_kernel (st.async exchange), the r2c FFT rows (incl. parent 16384)
and the 2-CTA DSMEM split FFT, the batched 32x32 kernel, the device Gaussian
generator, block elimination -- each checked against a host result so a
sanitizer-clean run is also a correct one.

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1406_5802_b200 as rl  # noqa: E402
from paper_1406_5802_b200 import capi  # noqa: E402

L = capi.lib()
rng = np.random.default_rng(0)


def check(name, ok):
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        sys.exit(1)


# DGEMM (TMA ring, big / small / tiny configurations and the accumulate path)
for m, n, k in [(300, 260, 200), (128, 64, 512), (70, 40, 33)]:
    a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
    check(f"dgemm {m}x{n}x{k}", np.abs(rl.matmul(a, b) - a @ b).max() <= 1e-12 * np.abs(a @ b).max())

# blocked GENP: 128-column super-panels + lookahead (n >= 256), 64-wide (n = 192), ragged tail
for n in (640, 192, 300):
    a = rng.standard_normal((n, n)) + n * np.eye(n)
    f = rl.genp_factor(a)
    check(f"genp n={n}", np.abs(f.lower @ f.upper - a).max() <= 1e-10 * np.abs(a).max())

# preprocessed solve (device generator, product, GENP, verdict, chain solve)
n = 512
a = rl.gen_gaussian(n, n, 1)
b = rl.gen_gaussian_vector(n, 3)
out = rl.preprocess_solve(a, b, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 2), 1)
check("preprocess_solve n=512", out.residual_history[-1] < 1e-10)

# range finder + residual: clustered power_pass_kernel (one-pass power step)
m, n, l = 2048, 1024, 32
u, _ = np.linalg.qr(rng.standard_normal((m, l)))
v, _ = np.linalg.qr(rng.standard_normal((n, l)))
a = (u * np.logspace(0, -3, l)) @ v.T + 1e-6 * rng.standard_normal((m, n))
res = rl.range_find(a, l, 0, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 5))
s1 = np.linalg.norm(a - res.q @ (res.q.T @ a), 2)
check("range_find + power_pass", abs(res.info["residual_spectral"] / s1 - 1) < 1e-3)

# FFT rows: r2c at 8192 and parent 16384 (aligned), and the 2-CTA split kernel (unaligned A)
for k in (8192, 16384):
    a = rl.gen_gaussian(6, k, 7)
    c = rl.gen_gaussian_vector(k, 8)
    y = rl.matmul_by_toeplitz_block(a, c, 256)
    dense = np.array([[c[(i - j) % k] for j in range(256)] for i in range(k)])
    check(f"toeplitz rows k={k}", np.abs(y - a @ dense).max() <= 1e-10 * np.abs(y).max())
k = 16384
buf = torch.from_numpy(rl.gen_gaussian(1, 4 * k + 1, 9).reshape(-1)).cuda()
da = buf[1:1 + 4 * k]  # 8-byte offset: not 16-byte aligned -> the split (2-CTA DSMEM) path
dc = torch.from_numpy(rl.gen_gaussian_vector(k, 10)).cuda()
dy = torch.empty(4, 128, dtype=torch.float64, device="cuda")
rc = L.rl_toeplitz_right_multiply(None, capi.RL_DEVICE, 4, k, da.data_ptr(), k, dc.data_ptr(), 128, dy.data_ptr())
c = dc.cpu().numpy()
dense = np.array([[c[(i - j) % k] for j in range(128)] for i in range(k)])
ref = da.cpu().numpy().reshape(4, k) @ dense
check("toeplitz split kernel (unaligned)", rc == 0 and np.abs(dy.cpu().numpy() - ref).max() <= 1e-10 * np.abs(ref).max())

# batched 32x32
import oracle  # noqa: E402  (test infrastructure: the checker)
r = oracle.C.batched_config2(64, base=7)
bo = rl.batched_preprocess_solve_32(r["a"], r["g"], r["b"])
check("batched 32x32", np.abs(bo.x - r["x"]).max() <= 1e-8 * np.abs(r["x"]).max())

# device Gaussian generator (two halves, host-finished attempts)
g = torch.empty(300, 257, dtype=torch.float64, device="cuda")
hard = ctypes.c_int64(0)
L.rl_gen_gaussian_device(None, 300, 257, 11, g.data_ptr(), 257, ctypes.byref(hard))
check("device generator", np.array_equal(g.cpu().numpy(), rl.gen_gaussian(300, 257, 11)))

# block elimination (GEPP leaves, Jacobi singular values, Schur tiles)
a = rl.gen_gaussian(96, 96, 12)
f = rl.block_ge_factor(a, [32, 32, 32])
x = rl.block_solve(f, rl.gen_gaussian_vector(96, 13))
check("block_ge", np.abs(a @ x - rl.gen_gaussian_vector(96, 13)).max() <= 1e-9)
torch.cuda.synchronize()
print("sanitize driver done")
