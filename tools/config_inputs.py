"""INPUT CONSTRUCTION ONLY (untimed) — the BASELINE.json config 3-5 matrices,
built on the host deterministically so that the committed oracle fixtures
(tests/golden/make_fullsize.py), the full-size GPU parity tests and bench.py all
see the SAME bytes.

Recipe (BASELINE.json configs; the reference's gen_lownumrank pattern,
testbed/inputs.hpp:67-83: column-scaled orthonormal factor times the other
factor's transpose):
  Q(.)   = the canonical thin QR factor with positive diagonal R
           (qr.hpp:33-45): Householder QR (LAPACK dgeqrf/dorgqr through numpy),
           column j multiplied by sign(r_jj)
  config 3: U = Q(gen_gaussian(8192,8192,11)), V = Q(gen_gaussian(8192,8192,12)),
            sigma_j = 10^(-4j/8191), A = (U diag sigma) V^T,
            c = gen_gaussian_vector(8192,13), b = gen_gaussian_vector(8192,14)
  config 4: U_r = Q(gen_gaussian(8192,64,42)), V_r = Q(gen_gaussian(8192,64,43)),
            sigma_j = 10^(-2j/63), A = (U_r diag sigma) V_r^T + 1e-10 gen_gaussian(8192,8192,44),
            H = gen_gaussian(8192,64,41) (drawn inside range_find)
  config 5: U_r = Q(gen_gaussian(32768,256,51)), V_r = Q(gen_gaussian(16384,256,52)),
            sigma_j = 10^(-3j/255), A = (U_r diag sigma) V_r^T + 1e-12 gen_gaussian(32768,16384,53),
            H = ToeplitzBlock(RealCirculant(gen_gaussian_vector(16384,21)), 16384, 256)
Seeds BASELINE.json leaves open are recorded in BASELINE.md §3 / DESIGN.md §7.

Determinism: gen_gaussian is the bit-exact host generator (librandla_b200's
rl_gen_gaussian, identical to the reference's RngStream). The BLAS/LAPACK
steps run in a child process with OPENBLAS_CORETYPE and OPENBLAS_NUM_THREADS
pinned (OpenBLAS results depend on the kernel family and thread split, not on
the machine otherwise), sigma uses the C library's pow (no SIMD math), and the
remaining steps are single IEEE operations. The builder prints the SHA-256 of
every array; fixtures record them, and tests assert them before comparing.

Usage: python tools/config_inputs.py {cfg3,cfg4,cfg5} OUTDIR
       (writes OUTDIR/<cfg>_<name>.npy and OUTDIR/<cfg>.json with the digests)
In-process callers use build(cfg, outdir) / load(cfg, outdir).
"""
import hashlib
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PIN_ENV = {"OPENBLAS_CORETYPE": "Haswell", "OPENBLAS_NUM_THREADS": "8", "OMP_NUM_THREADS": "8"}

CONFIGS = {
    "cfg3": dict(m=8192, n=8192, r=8192, su=11, sv=12, sigma_hi_exp=4.0, se=None, noise=0.0, c_seed=13, b_seed=14),
    "cfg4": dict(m=8192, n=8192, r=64, su=42, sv=43, sigma_hi_exp=2.0, se=44, noise=1e-10, h_seed=41),
    "cfg5": dict(m=32768, n=16384, r=256, su=51, sv=52, sigma_hi_exp=3.0, se=53, noise=1e-12, h_seed=21),
}


def sha(a):
    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sigma(r, hi_exp):
    """sigma_j = 10^(-hi_exp j/(r-1)), j < r, by the C library's pow."""
    return [math.pow(10.0, -hi_exp * j / (r - 1)) for j in range(r)]


def _positive_q(g):
    """qr.hpp:33-45 for real input: Householder Q, column j times sign(r_jj)."""
    import numpy as np
    q, r = np.linalg.qr(g)
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    q *= d
    return q


def _gen(m, n, seed):
    sys.path.insert(0, ROOT)
    import paper_1406_5802_b200 as rl
    return rl.gen_gaussian(m, n, seed)


def _factor_child(m, r, seed, out):
    """child process: Q(gen_gaussian(m, r, seed)) -> out (.npy)"""
    import numpy as np
    np.save(out, _positive_q(_gen(m, r, seed)))


def _build_here(cfg, outdir):
    import numpy as np
    p = CONFIGS[cfg]
    m, n, r = p["m"], p["n"], p["r"]
    os.makedirs(outdir, exist_ok=True)
    fu, fv = os.path.join(outdir, f"{cfg}_U.npy"), os.path.join(outdir, f"{cfg}_V.npy")
    # the two orthonormal factors in two pinned child processes at once
    procs = [subprocess.Popen([sys.executable, __file__, "--factor", str(mm), str(r), str(s), f],
                              env={**os.environ, **PIN_ENV})
             for mm, s, f in ((m, p["su"], fu), (n, p["sv"], fv))]
    for pr in procs:
        if pr.wait() != 0:
            raise RuntimeError(f"{cfg}: factor child failed")
    u = np.load(fu)
    v = np.load(fv)
    os.remove(fu)
    os.remove(fv)
    u *= np.asarray(sigma(r, p["sigma_hi_exp"]))  # U diag(sigma): column scaling (inputs.hpp:75-77)
    a = u @ v.T  # matmul(scaled, t.transpose()) (inputs.hpp:78)
    del u, v
    if p["se"] is not None:
        e = _gen(m, n, p["se"])
        e *= p["noise"]
        a += e
        del e
    digests = {"A": sha(a)}
    np.save(os.path.join(outdir, f"{cfg}_A.npy"), a)
    if cfg == "cfg3":
        c = _gen(n, 1, p["c_seed"]).reshape(n)
        b = _gen(n, 1, p["b_seed"]).reshape(n)
        np.save(os.path.join(outdir, f"{cfg}_c.npy"), c)
        np.save(os.path.join(outdir, f"{cfg}_b.npy"), b)
        digests["c"], digests["b"] = sha(c), sha(b)
    if cfg == "cfg5":
        c = _gen(n, 1, p["h_seed"]).reshape(n)
        np.save(os.path.join(outdir, f"{cfg}_c.npy"), c)
        digests["c"] = sha(c)
    with open(os.path.join(outdir, f"{cfg}.json"), "w") as f:
        json.dump({"config": cfg, "params": p, "sha256": digests, "pin": PIN_ENV}, f, indent=1)
    return digests


def build(cfg, outdir):
    """Build config `cfg` into outdir in a pinned child process (numpy's
    OpenBLAS reads OPENBLAS_CORETYPE at load, and the oracle's GEMM hook sets
    the shared OpenBLAS to one thread). Returns the digest record."""
    subprocess.run([sys.executable, __file__, cfg, outdir], check=True, env={**os.environ, **PIN_ENV})
    with open(os.path.join(outdir, f"{cfg}.json")) as f:
        return json.load(f)


def load(cfg, outdir, mmap=True):
    import numpy as np
    out = {}
    for name in ("A", "b", "c"):
        f = os.path.join(outdir, f"{cfg}_{name}.npy")
        if os.path.exists(f):
            out[name] = np.load(f, mmap_mode="r" if mmap else None)
    with open(os.path.join(outdir, f"{cfg}.json")) as f:
        out["record"] = json.load(f)
    return out


if __name__ == "__main__":
    if sys.argv[1] == "--factor":
        _factor_child(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
    else:
        for k, v in PIN_ENV.items():
            if os.environ.get(k) != v:
                raise SystemExit(f"{k} must be {v}: run through build() (pinned environment)")
        # stderr: the caller (bench.py) owns stdout for its one JSON line
        print(json.dumps(_build_here(sys.argv[1], sys.argv[2])), file=sys.stderr)
