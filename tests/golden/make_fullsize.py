"""Full-size oracle fixtures at the BASELINE.json sizes, made by the REFERENCE
ITSELF (oracle/_ref: the reference's own headers compiled read-only from
/root/reference by oracle/Makefile) on the inputs of tools/config_inputs.py.

Runs in the dev container only, once (about half an hour on 8 cores: the
reference's genp_factor and FFT loops are single-threaded). Writes
tests/golden/fullsize_{headline,cfg3,cfg4,cfg5}.npz. The GPU tests
(tests/test_fullsize_gpu.py) rebuild the same inputs on the GPU box, assert
their SHA-256 against the fixture, and compare the device results with what
is stored here.

What is stored (compact: the n x n factors themselves are 512 MiB each):
  - x, the residual history, the ZeroPivot verdict, the growth
    rho = max|U| / max|product| and the pivots diag(U) (all of them);
  - whole rows of the packed L\\U at fixed indices (block boundaries, ends);
  - L W and U W for a seeded Gaussian W (n x 8): ||(dL) W||_F / ||L W||_F
    estimates the relative Frobenius error of the whole factor
    (E||dL w||^2 = ||dL||_F^2 for Gaussian w);
  - low rank: Q W_l and rows of Q, the rank verdict, ||R||_F, and ||R||_2 by
    the reference's own spectral_norm_estimate (norms.hpp:35-78) on the
    explicit residual R = A - Q (Q^T A) (lowrank.hpp:35-37,99-102), plus the
    exact sigma_max(R) by LAPACK SVD where that is affordable (config 4).

Usage: python tests/golden/make_fullsize.py [headline cfg3 cfg4 cfg5]
       python tests/golden/make_fullsize.py floor [headline cfg3]   (adds the rounding floors)
       python tests/golden/make_fullsize.py floor_alg [headline cfg3]   (adds the algorithm floors)
       python tests/golden/make_fullsize.py floor_inv [headline cfg3]   (... with the inverse-based U12)
       python tests/golden/make_fullsize.py floor_lowrank [cfg4 cfg5]   (the range finder's floors)
"""
import ctypes
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import config_inputs  # noqa: E402
import oracle  # noqa: E402

R = oracle.REF
assert R is not None, "oracle/_ref not built: run `make -C oracle` with /root/reference present"
HERE = os.path.dirname(os.path.abspath(__file__))
WORK = os.environ.get("RANDLA_FULLSIZE_WORK", "/tmp/randla_fullsize_inputs")
ROWS = np.array([0, 1, 2, 63, 64, 127, 128, 129, 255, 256, 1000, 2047, 2048, 4095, 4096, 6000, 8190, 8191])
W_SEED = 99
W_COLS = 8


def blas_threads(k):
    """the oracle's GEMM hook pins the shared OpenBLAS to one thread; the
    LAPACK-only extras (SVD) may use more"""
    lib = ctypes.CDLL(oracle.openblas_path())
    lib.scipy_openblas_set_num_threads64_(ctypes.c_int(k))


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def lu_digest(lu, n):
    """rows of the packed factors and the L W, U W sketches"""
    w = R.gen_gaussian(n, W_COLS, W_SEED)
    low = np.tril(lu, -1)
    low[np.diag_indices(n)] = 1.0
    lw = low @ w
    del low
    uw = np.triu(lu) @ w
    rows = ROWS[ROWS < n]
    return dict(lu_rows_idx=rows, lu_rows=lu[rows].copy(), lw=lw, uw=uw, w_seed=np.array([W_SEED]),
                pivots=np.diag(lu).copy(), max_abs_u=np.array([np.abs(np.triu(lu)).max()]))


def positive_qr_q(y):
    """qr.hpp:22-47 restated for real input (the reference's Householder QR is
    Eigen's, absent here): LAPACK Householder Q, column j times sign(r_jj), and
    the rank check |r_jj| <= tol_rank(m, n) * spectral_norm_estimate(y)."""
    m, l = y.shape
    q, r = np.linalg.qr(y)
    d = np.diag(r).copy()
    scale = R.spectral_norm_estimate(y)
    tol = 1e-13 * max(m, l) * scale  # tol_rank (types.hpp:41-42)
    bad = np.nonzero(np.abs(d) <= tol)[0]
    q *= np.where(d < 0, -1.0, 1.0)
    return q, (int(bad[0]) + 1 if len(bad) else 0), scale, np.abs(d)


def headline():
    n = 8192
    a = R.gen_gaussian(n, n, 1)
    g = R.gen_gaussian(n, n, 2)
    b = R.gen_gaussian(n, 1, 3).reshape(n)
    log("headline: inputs")
    p = R.matmul(a, g)
    log("headline: product")
    est = R.spectral_norm_estimate(p)
    log("headline: estimate", est)
    lu, zs = R.genp_factor(p)
    log("headline: genp_factor, zero step", zs)
    out = lu_digest(lu, n)
    out["max_abs_product"] = np.array([np.abs(p).max()])
    out["growth"] = out["max_abs_u"] / out["max_abs_product"]
    # the reference's own composite (preprocess.hpp:156-180), refine 0 and 1
    for refine in (0, 1):
        r = R.preprocess_solve(a, b, post_kind=1, seed=2, refine=refine)
        assert r["status"] == 0
        out[f"x_refine{refine}"] = r["x"]
        out[f"history_refine{refine}"] = r["history"]
        log("headline: preprocess_solve refine", refine, r["history"])
    out["zero_step"] = np.array([zs])
    out["estimate"] = np.array([est])
    out["sha_a"] = np.array([config_inputs.sha(a)])
    del lu
    blas_threads(8)
    out["kappa_a"] = np.array([_kappa(a)])
    out["kappa_product"] = np.array([_kappa(p)])
    log("headline: kappa", out["kappa_a"], out["kappa_product"])
    np.savez(os.path.join(HERE, "fullsize_headline.npz"), **out)


def _kappa(a):
    s = np.linalg.svd(a, compute_uv=False)
    return s[0] / s[-1]


def cfg3():
    rec = config_inputs.build("cfg3", WORK)
    inp = config_inputs.load("cfg3", WORK, mmap=False)
    a, c, b = inp["A"], inp["c"], inp["b"]
    n = a.shape[0]
    log("cfg3: inputs", rec["sha256"])
    p, st = R.matmul_by_circulant(a, c)  # circulant.hpp:171-185
    assert st == 0
    log("cfg3: product")
    est = R.spectral_norm_estimate(p)
    lu, zs = R.genp_factor(p)
    log("cfg3: genp_factor, zero step", zs)
    out = lu_digest(lu, n)
    out["max_abs_product"] = np.array([np.abs(p).max()])
    out["growth"] = out["max_abs_u"] / out["max_abs_product"]
    # chain solve x = C (LU)^-1 b (preprocess.hpp:170-172, apply_vec = circulant_apply)
    y = R.lu_solve(lu, b)
    x, st = R.circulant_apply(c, y)
    assert st == 0
    out["x_refine0"] = x
    out["history_refine0"] = np.array([np.linalg.norm(b - a @ x) / np.linalg.norm(b)])
    out["zero_step"] = np.array([zs])
    out["estimate"] = np.array([est])
    for k, v in rec["sha256"].items():
        out[f"sha_{k}"] = np.array([v])
    out["kappa_a"] = np.array([1e4])  # by construction (sigma 1 .. 1e-4)
    blas_threads(8)
    out["kappa_product"] = np.array([_kappa(p)])
    log("cfg3: kappa(product)", out["kappa_product"])
    np.savez(os.path.join(HERE, "fullsize_cfg3.npz"), **out)


def _threaded_rows(fn, m, chunks=8):
    """run fn(r0, r1) over row blocks on threads (ctypes releases the GIL; the
    rows are independent, so the result is the single-call result bit for bit)"""
    step = (m + chunks - 1) // chunks
    ts = [threading.Thread(target=fn, args=(r0, min(m, r0 + step))) for r0 in range(0, m, step)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


def lowrank(cfg):
    rec = config_inputs.build(cfg, WORK)
    inp = config_inputs.load(cfg, WORK, mmap=False)
    a = inp["A"]
    m, n = a.shape
    prm = config_inputs.CONFIGS[cfg]
    l = prm["r"]
    log(cfg, "inputs", rec["sha256"])
    if cfg == "cfg4":
        h = R.gen_gaussian(n, l, prm["h_seed"])  # materialize({Gaussian, seed}) (multipliers.hpp:191-192)
        y = R.matmul(a, h)
    else:
        c = inp["c"]
        y = np.empty((m, l))

        def part(r0, r1):
            y[r0:r1], st = R.matmul_by_toeplitz_block(a[r0:r1], c, l)  # circulant.hpp:187-203
            assert st == 0

        _threaded_rows(part, m)
    log(cfg, "sketch")
    q, bad, y_est, rdiag = positive_qr_q(y)
    log(cfg, "qr, rank verdict", bad)
    bmat = R.matmul(np.ascontiguousarray(q.T), a)  # Q^H A (lowrank.hpp:35-37)
    res = a - R.matmul(q, bmat)
    del bmat
    fro = np.linalg.norm(res)
    log(cfg, "||R||_F", fro)
    spec_est = R.spectral_norm_estimate(res)
    log(cfg, "||R||_2 estimate", spec_est)
    wl = R.gen_gaussian(l, W_COLS, W_SEED)
    out = dict(qw=q @ wl, q_rows=q[:64].copy(), w_seed=np.array([W_SEED]), rank_deficient=np.array([bad]),
               sketch_estimate=np.array([y_est]), r_diag=rdiag, residual_frobenius=np.array([fro]),
               residual_spectral_estimate=np.array([spec_est]), sketch_rows=y[:64].copy(),
               sketch_fro=np.array([np.linalg.norm(y)]))
    for k, v in rec["sha256"].items():
        out[f"sha_{k}"] = np.array([v])
    if cfg == "cfg4":
        blas_threads(8)
        out["residual_spectral_svd"] = np.array([np.linalg.svd(res, compute_uv=False)[0]])
        log(cfg, "sigma_max(R)", out["residual_spectral_svd"])
    np.savez(os.path.join(HERE, f"fullsize_{cfg}.npz"), **out)


def rounding_floor(name):
    """The reference's own forward-error floor on this input: genp_factor (and
    the chain solve) of the SAME product computed in another, equally valid
    summation order -- the headline's A G as eight K-slab products summed
    slab by slab, config 3's A C as A times the dense
    circulant instead of the FFT -- compared with the fixture in the same
    digests. That is exactly what separates any two correct implementations
    (the device's DMMA GEMM / r2c FFT included). GENP's L, U and pivots follow
    the leading principal minors (growth ~1e4-1e5 here), not kappa(A), so this
    floor -- not 1e-10 kappa(A) -- is what they can agree to; the GPU tests
    hold the device to a small multiple of it."""
    fx = dict(np.load(os.path.join(HERE, f"fullsize_{name}.npz")))
    n = 8192
    blas_threads(8)
    if name == "headline":
        a = R.gen_gaussian(n, n, 1)
        g = R.gen_gaussian(n, n, 2)
        b = R.gen_gaussian(n, 1, 3).reshape(n)
        # the same product summed in another association: eight K-slabs of
        # 1024, each a BLAS product, accumulated slab by slab (OpenBLAS's own
        # blocking is thread-count independent, so a plain a @ g would repeat
        # the fixture's bits)
        p = np.zeros((n, n))
        for k0 in range(0, n, 1024):
            p += a[:, k0:k0 + 1024] @ g[k0:k0 + 1024, :]
    else:
        config_inputs.build("cfg3", WORK)
        inp = config_inputs.load("cfg3", WORK, mmap=False)
        a, c, b = inp["A"], inp["c"], inp["b"]
        idx = (np.arange(n)[:, None] - np.arange(n)[None, :]) % n
        p = a @ c[idx]  # A times the dense circulant (circulant.hpp:31-38), not the FFT
        del idx
    blas_threads(1)
    lu, zs = R.genp_factor(p)
    assert zs == 0
    d = lu_digest(lu, n)
    y = R.lu_solve(lu, b)
    if name == "headline":
        x = g @ y
    else:
        x, st = R.circulant_apply(c, y)
    rel = lambda u, v: float(np.linalg.norm(u - v) / np.linalg.norm(v))  # noqa: E731
    floor = {"x": rel(x, fx["x_refine0"]), "pivots": rel(d["pivots"], fx["pivots"]),
             "lu_rows": rel(d["lu_rows"], fx["lu_rows"]), "L_sketch": rel(d["lw"], fx["lw"]),
             "U_sketch": rel(d["uw"], fx["uw"]),
             "growth": float(abs(d["max_abs_u"][0] / np.abs(p).max() - fx["growth"][0]) / fx["growth"][0])}
    log(name, "rounding floor", floor)
    for k, v in floor.items():
        fx[f"floor_{k}"] = np.array([v])
    np.savez(os.path.join(HERE, f"fullsize_{name}.npz"), **fx)


def lowrank_floor(cfg):
    """The range finder's own rounding floor: the sketch formed in another,
    equally valid order -- config 4's A H as eight K-slab products, config 5's
    Toeplitz product as A times the dense Toeplitz block instead of the FFT --
    then the same restated QR and residual; the relative change of ||R||_F,
    of the power-iteration ||R||_2 and of Q against the fixture."""
    fx = dict(np.load(os.path.join(HERE, f"fullsize_{cfg}.npz")))
    config_inputs.build(cfg, WORK)
    inp = config_inputs.load(cfg, WORK, mmap=False)
    a = inp["A"]
    m, n = a.shape
    prm = config_inputs.CONFIGS[cfg]
    l = prm["r"]
    blas_threads(8)
    if cfg == "cfg4":
        h = R.gen_gaussian(n, l, prm["h_seed"])
        y = np.zeros((m, l))
        for k0 in range(0, n, 1024):
            y += a[:, k0:k0 + 1024] @ h[k0:k0 + 1024]
    else:
        c = inp["c"]
        idx = (np.arange(n)[:, None] - np.arange(l)[None, :]) % n
        y = a @ c[idx]  # the dense Toeplitz block (circulant.hpp:143-169)
    blas_threads(1)
    q, bad, _, _ = positive_qr_q(y)
    assert bad == 0
    res = a - R.matmul(q, R.matmul(np.ascontiguousarray(q.T), a))
    fro = np.linalg.norm(res)
    est = R.spectral_norm_estimate(res)
    wl = R.gen_gaussian(l, W_COLS, W_SEED)
    floor = {"fro": abs(fro / fx["residual_frobenius"][0] - 1),
             "spec": abs(est / fx["residual_spectral_estimate"][0] - 1),
             "q": float(np.linalg.norm(q @ wl - fx["qw"]) / np.linalg.norm(fx["qw"]))}
    log(cfg, "lowrank floor", floor)
    for k, v in floor.items():
        fx[f"floor_{k}"] = np.array([v])
    np.savez(os.path.join(HERE, f"fullsize_{cfg}.npz"), **fx)


def blocked_genp(p, nb=128, explicit_inverse=False):
    """GENP (no pivoting) of p as a right-looking blocked factorisation with
    BLAS updates: unblocked 128-column panels, U12 = L11^-1 A12, A22 -= L21 U12
    -- the algorithm class of the device's, in LAPACK / OpenBLAS arithmetic.
    explicit_inverse: U12 = (L11^-1) A12 with the inverse formed first, as the
    device does (MAGMA-style TRSM by inverted diagonal blocks)"""
    import scipy.linalg as sl
    a = p.copy()
    n = a.shape[0]
    for k in range(0, n, nb):
        e = min(k + nb, n)
        for j in range(k, e):
            a[j + 1:, j] /= a[j, j]
            if j + 1 < e:
                a[j + 1:, j + 1:e] -= np.outer(a[j + 1:, j], a[j, j + 1:e])
        if e < n:
            if explicit_inverse:
                linv = sl.solve_triangular(a[k:e, k:e], np.eye(e - k), lower=True, unit_diagonal=True)
                a[k:e, e:] = linv @ a[k:e, e:]
            else:
                a[k:e, e:] = sl.solve_triangular(a[k:e, k:e], a[k:e, e:], lower=True, unit_diagonal=True)
            a[e:, e:] -= a[e:, k:e] @ a[k:e, e:]
    return a


def algorithm_floor(name, explicit_inverse=False):
    """The reference's GENP against a blocked right-looking GENP with BLAS
    updates (blocked_genp) on the SAME product bits: the disagreement of two
    correct elimination orders, the other half of what separates the device
    (blocked, K = 128 DMMA updates, FMA) from the reference's scalar loop."""
    fx = dict(np.load(os.path.join(HERE, f"fullsize_{name}.npz")))
    n = 8192
    blas_threads(8)
    if name == "headline":
        a = R.gen_gaussian(n, n, 1)
        g = R.gen_gaussian(n, n, 2)
        b = R.gen_gaussian(n, 1, 3).reshape(n)
        p = a @ g  # bit-identical to the reference's product (OpenBLAS blocking is thread-count independent)
    else:
        config_inputs.build("cfg3", WORK)
        inp = config_inputs.load("cfg3", WORK, mmap=False)
        a, c, b = inp["A"], inp["c"], inp["b"]
        blas_threads(1)
        p, st = R.matmul_by_circulant(a, c)
        blas_threads(8)
    lu = blocked_genp(p, explicit_inverse=explicit_inverse)
    d = lu_digest(lu, n)
    import scipy.linalg as sl
    y = sl.solve_triangular(np.triu(lu), sl.solve_triangular(lu, b, lower=True, unit_diagonal=True), lower=False)
    if name == "headline":
        x = g @ y
    else:
        blas_threads(1)
        x, st = R.circulant_apply(c, y)
    rel = lambda u, v: float(np.linalg.norm(u - v) / np.linalg.norm(v))  # noqa: E731
    floor = {"x": rel(x, fx["x_refine0"]), "pivots": rel(d["pivots"], fx["pivots"]),
             "lu_rows": rel(d["lu_rows"], fx["lu_rows"]), "L_sketch": rel(d["lw"], fx["lw"]),
             "U_sketch": rel(d["uw"], fx["uw"]),
             "growth": float(abs(d["max_abs_u"][0] / np.abs(p).max() - fx["growth"][0]) / fx["growth"][0])}
    tag = "floor_inv" if explicit_inverse else "floor_alg"
    log(name, tag, floor)
    for k, v in floor.items():
        fx[f"{tag}_{k}"] = np.array([v])
    np.savez(os.path.join(HERE, f"fullsize_{name}.npz"), **fx)


if __name__ == "__main__":
    if sys.argv[1:2] == ["floor_lowrank"]:
        for w in sys.argv[2:] or ["cfg4", "cfg5"]:
            lowrank_floor(w)
        sys.exit(0)
    if sys.argv[1:2] in (["floor_alg"], ["floor_inv"]):
        for w in sys.argv[2:] or ["headline", "cfg3"]:
            algorithm_floor(w, explicit_inverse=sys.argv[1] == "floor_inv")
        sys.exit(0)
    if sys.argv[1:2] == ["floor"]:
        for w in sys.argv[2:] or ["headline", "cfg3"]:
            rounding_floor(w)
        sys.exit(0)
    which = sys.argv[1:] or ["headline", "cfg3", "cfg4", "cfg5"]
    for w in which:
        t = time.time()
        {"headline": headline, "cfg3": cfg3, "cfg4": lambda: lowrank("cfg4"), "cfg5": lambda: lowrank("cfg5")}[w]()
        log(w, "done in", round(time.time() - t), "s")
