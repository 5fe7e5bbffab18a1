"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU oracle.

`C`   : liboracle.so, the plain-C restatement (oracle.c), always present after
        `make -C oracle` (built by __graft_entry__.build()).
`REF` : oracle/_ref/librandla_ref.so, the reference's own headers compiled
        with our Eigen shim; None when it was not built (it needs
        /root/reference at build time, and then travels to the GPU box as a
        built file).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module. The product package never does.
"""
import ctypes
import glob
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i32p = ctypes.POINTER(ctypes.c_int)
i64 = ctypes.c_int64
u64 = ctypes.c_uint64


def openblas_path():
    """numpy's bundled scipy-openblas (ILP64); the oracle's GEMM hook."""
    try:
        libs = os.path.join(os.path.dirname(np.__file__), "..", "numpy.libs")
        cands = sorted(glob.glob(os.path.join(libs, "libscipy_openblas64_*.so")))
        return os.path.abspath(cands[0]) if cands else ""
    except Exception:
        return ""


os.environ.setdefault("RANDLA_ORACLE_OPENBLAS", openblas_path())


def build():
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path):
    if not os.path.exists(path):
        return None
    return ctypes.CDLL(path)


def ptr(a):
    if a is None:
        return None
    if a.dtype == np.float64:
        return a.ctypes.data_as(_dp)
    if a.dtype == np.int64:
        return a.ctypes.data_as(_i64p)
    if a.dtype == np.uint64:
        return a.ctypes.data_as(_u64p)
    raise TypeError(a.dtype)


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


class _C:
    def __init__(self, lib):
        self.lib = lib
        s = lambda n, r, a: _sig(lib, n, r, a)
        s("or_singular_values", None, [i64, i64, _dp, _dp])
        self.hash_label = s("or_hash_label", u64, [ctypes.c_char_p])
        self.derive_seed = s("or_derive_seed", u64, [u64, u64, u64])
        self._gen = s("or_gen_gaussian", None, [i64, i64, u64, _dp])
        self._genc = s("or_gen_real_circulant_column", None, [i64, u64, _dp])
        self._matmul = s("or_matmul", None, [i64, i64, i64, _dp, _dp, _dp])
        self.uses_blas = s("or_matmul_uses_blas", ctypes.c_int, [])
        self._normest = s("or_spectral_norm_estimate", ctypes.c_double, [i64, i64, _dp])
        self._genp = s("or_genp_factor", ctypes.c_int, [i64, _dp, _dp, _i64p, _dp])
        self._solve = s("or_lu_solve", None, [i64, _dp, _dp, _dp])
        self._gsteps = s("or_genp_steps", None, [i64, _dp, i64, i64])
        self._fft = s("or_fft", ctypes.c_int, [i64, _dp])
        self._ifft = s("or_inverse_fft", ctypes.c_int, [i64, _dp])
        self._capply = s("or_circulant_apply", ctypes.c_int, [i64, _dp, _dp, _dp])
        self._mcirc = s("or_matmul_by_circulant", ctypes.c_int, [i64, i64, _dp, _dp, _dp])
        self._mtoep = s("or_matmul_by_toeplitz_block", ctypes.c_int, [i64, i64, _dp, i64, _dp, i64, _dp])
        self._pre = s("or_preprocess_solve", ctypes.c_int,
                      [i64, _dp, _dp, ctypes.c_int, _dp, i64, _dp, _dp, _i32p, _i64p, _dp, _dp])
        self._batch = s("or_batched_config2", None,
                        [i64, u64, i64, i64, ctypes.c_int, _dp, _dp, _dp, _dp, _dp, _i64p, _dp, _dp])
        self._qr = s("or_qr", ctypes.c_int, [i64, i64, _dp, _dp, _dp, _i64p])

    def gen_gaussian(self, m, n, seed):
        out = np.empty((m, n))
        self._gen(m, n, seed, ptr(out))
        return out

    def gen_gaussian_vector(self, n, seed):
        return self.gen_gaussian(n, 1, seed).reshape(n)

    def gen_real_circulant_column(self, n, seed):
        out = np.empty(n)
        self._genc(n, seed, ptr(out))
        return out

    def matmul(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty((a.shape[0], b.shape[1]))
        self._matmul(a.shape[0], a.shape[1], b.shape[1], ptr(a), ptr(b), ptr(out))
        return out

    def spectral_norm_estimate(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        return self._normest(a.shape[0], a.shape[1], ptr(a))

    def genp_factor(self, a):
        """-> (packed LU, zero_step (0 = ok), tol)"""
        a = np.ascontiguousarray(a, dtype=np.float64)
        lu = np.empty_like(a)
        zs = np.zeros(1, np.int64)
        tol = np.zeros(1)
        self._genp(a.shape[0], ptr(a), ptr(lu), ptr(zs), ptr(tol))
        return lu, int(zs[0]), float(tol[0])

    def lu_solve(self, lu, b):
        lu = np.ascontiguousarray(lu, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        self._solve(lu.shape[0], ptr(lu), ptr(b), ptr(x))
        return x

    def genp_steps(self, lu, j0, j1):
        """elimination steps j0..j1-1 of genp_factor, in place (lu C-contiguous)"""
        assert lu.flags.c_contiguous and lu.dtype == np.float64
        self._gsteps(lu.shape[0], ptr(lu), j0, j1)

    def fft(self, z, inverse=False):
        w = np.ascontiguousarray(np.asarray(z, dtype=np.complex128)).copy()
        v = w.view(np.float64)
        (self._ifft if inverse else self._fft)(w.shape[0], ptr(v))
        return w

    def circulant_apply(self, c, x):
        c = np.ascontiguousarray(c, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        st = self._capply(c.shape[0], ptr(c), ptr(x), ptr(y))
        return y, st

    def matmul_by_circulant(self, a, c):
        a = np.ascontiguousarray(a, dtype=np.float64)
        c = np.ascontiguousarray(c, dtype=np.float64)
        out = np.empty_like(a)
        st = self._mcirc(a.shape[0], a.shape[1], ptr(a), ptr(c), ptr(out))
        return out, st

    def matmul_by_toeplitz_block(self, a, c, l):
        a = np.ascontiguousarray(a, dtype=np.float64)
        c = np.ascontiguousarray(c, dtype=np.float64)
        out = np.empty((a.shape[0], l))
        st = self._mtoep(a.shape[0], a.shape[1], ptr(a), c.shape[0], ptr(c), l, ptr(out))
        return out, st

    def preprocess_solve(self, a, b, post_kind=0, post=None, refine=0, want_lu=False):
        """post_kind 0 none / 1 dense (post = G) / 2 circulant (post = c).
        -> dict(x, history, diverged, status, zero_step, lu, product)"""
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        n = a.shape[0]
        post = None if post is None else np.ascontiguousarray(post, dtype=np.float64)
        x = np.empty(n)
        hist = np.empty(refine + 1)
        div = ctypes.c_int(0)
        zs = np.zeros(1, np.int64)
        lu = np.empty((n, n)) if want_lu else None
        prod = np.empty((n, n)) if want_lu else None
        st = self._pre(n, ptr(a), ptr(b), post_kind, ptr(post), refine, ptr(x), ptr(hist), ctypes.byref(div),
                       ptr(zs), ptr(lu), ptr(prod))
        return dict(x=x, history=hist, diverged=bool(div.value), status=st, zero_step=int(zs[0]), lu=lu,
                    product=prod)

    def batched_config2(self, count, base=7, i0=0, threads=1, dim=32, want_inputs=True, want_lu=False):
        d = dim
        a = np.empty((count, d, d)) if want_inputs else None
        g = np.empty((count, d, d)) if want_inputs else None
        b = np.empty((count, d)) if want_inputs else None
        x = np.empty((count, d))
        res = np.empty(count)
        st = np.empty(count, np.int64)
        gr = np.empty(count)
        lu = np.empty((count, d, d)) if want_lu else None
        self._batch(d, base, i0, count, threads, ptr(a), ptr(g), ptr(b), ptr(x), ptr(res), ptr(st), ptr(gr),
                    ptr(lu))
        return dict(a=a, g=g, b=b, x=x, resid=res, status=st, growth=gr, lu=lu)

    def qr(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        m, l = a.shape
        q = np.empty((m, l))
        r = np.empty((l, l))
        bad = np.zeros(1, np.int64)
        st = self._qr(m, l, ptr(a), ptr(q), ptr(r), ptr(bad))
        return q, r, st, int(bad[0])


class _Ref:
    def __init__(self, lib):
        self.lib = lib
        s = lambda n, r, a: _sig(lib, n, r, a)
        self.hash_label = s("ref_hash_label", u64, [ctypes.c_char_p])
        self.derive_seed = s("ref_derive_seed", u64, [u64, u64, u64])
        self._golden = s("ref_golden_draws", None, [ctypes.c_char_p, u64, i64, _dp, _dp])
        self._gen = s("ref_gen_gaussian", None, [i64, i64, u64, _dp])
        self._genc = s("ref_gen_real_circulant_column", None, [i64, u64, _dp])
        self._genf = s("ref_gen_finite_set_uniform", None, [i64, i64, u64, u64, _dp])
        self._genk = s("ref_gen_circ_skew_product", None, [i64, u64, _dp])
        self._matmul = s("ref_matmul", ctypes.c_int, [i64, i64, i64, _dp, _dp, _dp])
        self._normest = s("ref_spectral_norm_estimate", ctypes.c_double, [i64, i64, _dp])
        self._genp = s("ref_genp_factor", ctypes.c_int, [i64, _dp, _dp, _i64p])
        self._solve = s("ref_lu_solve", None, [i64, _dp, _dp, _dp])
        self._schur = s("ref_schur_complement", ctypes.c_int, [i64, _dp, i64, _dp])
        self._fft = s("ref_fft", ctypes.c_int, [i64, _dp, ctypes.c_int])
        self._capply = s("ref_circulant_apply", ctypes.c_int, [i64, _dp, _dp, _dp])
        self._mcirc = s("ref_matmul_by_circulant", ctypes.c_int, [i64, i64, _dp, _dp, _dp])
        self._mtoep = s("ref_matmul_by_toeplitz_block", ctypes.c_int, [i64, i64, _dp, i64, _dp, i64, _dp])
        self._pre = s("ref_preprocess_solve", ctypes.c_int,
                      [i64, _dp, _dp, ctypes.c_int, u64, i64, _dp, _dp, _i32p, _i64p])
        self._pre2 = s("ref_preprocess_solve_spec", ctypes.c_int,
                       [i64, _dp, _dp, ctypes.c_int, ctypes.c_int, u64, ctypes.c_int, ctypes.c_int, u64, u64, i64,
                        _dp, _dp, _i32p, _i64p])
        self._sketch = s("ref_range_sketch", ctypes.c_int,
                         [i64, i64, _dp, i64, ctypes.c_int, ctypes.c_int, u64, u64, i64, _dp])
        self._mat = s("ref_materialize", ctypes.c_int, [ctypes.c_int, ctypes.c_int, u64, u64, i64, i64, _dp])
        self._batch = s("ref_batched_config2", i64, [i64, u64, i64, i64, _dp, _dp])
        self._trials = s("ref_parallel_dense_trials", i64, [i64, i64, _dp, _dp, _u64p, _dp])
        self._gepp = s("ref_gepp_factor", ctypes.c_int, [i64, _dp, _dp, _i64p])
        self._gepp_solve = s("ref_gepp_solve", ctypes.c_int, [i64, _dp, _dp, _dp, ctypes.c_int])
        self._block_ge = s("ref_block_ge", ctypes.c_int, [i64, _dp, i64, _i64p, _dp, _dp, _dp, _dp, _dp, _i64p])
        # the complex field (interleaved buffers)
        self._zgenp = s("ref_zgenp_factor", ctypes.c_int, [i64, _dp, _dp, _i64p])
        self._zpre = s("ref_zpreprocess_solve_spec", ctypes.c_int,
                       [i64, _dp, _dp, ctypes.c_int, ctypes.c_int, u64, ctypes.c_int, ctypes.c_int, u64, u64, i64,
                        _dp, _dp, _i32p, _i64p])
        self._zmat = s("ref_zmaterialize", ctypes.c_int, [ctypes.c_int, ctypes.c_int, u64, u64, i64, i64, _dp])
        self._zsketch = s("ref_zrange_sketch", ctypes.c_int,
                          [i64, i64, _dp, i64, ctypes.c_int, ctypes.c_int, u64, u64, i64, _dp])
        self._ucirc = s("ref_gen_unitary_circulant", None, [i64, u64, _dp])
        self._srftc = s("ref_srft_columns", None, [i64, i64, u64, _i64p])
        self._srftm = s("ref_srft_matrix", ctypes.c_int, [i64, i64, u64, ctypes.c_int, _dp])
        self._znormest = s("ref_zspectral_norm_estimate", ctypes.c_double, [i64, i64, _dp])
        self._dft = s("ref_dft_dense", ctypes.c_int, [i64, _dp])
        self._gder = s("ref_gaussian_derived", None, [u64, u64, i64, _dp])

    # status codes of the ref_* entry points (ref_capi.cpp)
    DIM, ZERO_PIVOT, SINGULAR_BLOCK, SINGULAR = 1, 2, 3, 6

    def gepp_factor(self, a):
        """gepp_factor (lu.hpp:62-98): (packed L\\U, perm, status)."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        n = a.shape[0]
        packed = np.empty_like(a)
        perm = np.empty(n, np.int64)
        st = self._gepp(n, ptr(a), ptr(packed), ptr(perm))
        return packed, perm, st

    def gepp_solve(self, a, b, transpose=False):
        """lu_solve / lu_solve_transpose (lu.hpp:100-147) with gepp_factor(a)."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        st = self._gepp_solve(a.shape[0], ptr(a), ptr(b), ptr(x), 1 if transpose else 0)
        if st != 0:
            raise RuntimeError(f"ref_gepp_solve failed ({st})")
        return x

    def block_ge(self, a, split, b):
        """block_ge_factor(a, split) (block_ge.hpp:168-181): dict with pivots,
        reassembled, x = block_solve(b), last_leaf (the deepest Schur leaf's
        block_matrix), status and position."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        n = a.shape[0]
        sp = np.ascontiguousarray(split, dtype=np.int64)
        k = int(sp[-1]) if len(sp) else 0
        out = {"pivots": np.empty(n), "reassembled": np.empty((n, n)), "x": np.empty(n),
               "last_leaf": np.empty((max(k, 1), max(k, 1)))}
        pos = np.zeros(1, np.int64)
        st = self._block_ge(n, ptr(a), len(sp), ptr(sp) if len(sp) else None, ptr(b), ptr(out["pivots"]),
                            ptr(out["reassembled"]), ptr(out["x"]), ptr(out["last_leaf"]), ptr(pos))
        out["status"], out["position"] = st, int(pos[0])
        return out

    def golden_draws(self, label, seed, trials):
        d = np.empty(trials)
        st = np.empty(4)
        self._golden(label.encode(), seed, trials, ptr(d), ptr(st))
        return d, st

    def gen_gaussian(self, m, n, seed):
        out = np.empty((m, n))
        self._gen(m, n, seed, ptr(out))
        return out

    def gen_real_circulant_column(self, n, seed):
        out = np.empty(n)
        self._genc(n, seed, ptr(out))
        return out

    def gen_finite_set_uniform(self, m, n, seed, card):
        out = np.empty((m, n))
        self._genf(m, n, seed, card, ptr(out))
        return out

    def gen_circ_skew_product(self, n, seed):
        out = np.empty((n, n))
        self._genk(n, seed, ptr(out))
        return out

    def matmul(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty((a.shape[0], b.shape[1]))
        self._matmul(a.shape[0], a.shape[1], b.shape[1], ptr(a), ptr(b), ptr(out))
        return out

    def spectral_norm_estimate(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        return self._normest(a.shape[0], a.shape[1], ptr(a))

    def genp_factor(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        lu = np.empty_like(a)
        zs = np.zeros(1, np.int64)
        st = self._genp(a.shape[0], ptr(a), ptr(lu), ptr(zs))
        return lu, int(zs[0]) if st == 2 else 0

    def schur_complement(self, a, k):
        """block_ge.hpp:202-218: E - D B^-1 C of the leading k x k block (GEPP)."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        n = a.shape[0]
        out = np.empty((n - k, n - k))
        st = self._schur(n, ptr(a), k, ptr(out))
        if st != 0:
            raise RuntimeError(f"ref_schur_complement failed ({st})")
        return out

    def lu_solve(self, lu, b):
        lu = np.ascontiguousarray(lu, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        self._solve(lu.shape[0], ptr(lu), ptr(b), ptr(x))
        return x

    def fft(self, z, inverse=False):
        w = np.ascontiguousarray(np.asarray(z, dtype=np.complex128)).copy()
        self._fft(w.shape[0], ptr(w.view(np.float64)), 1 if inverse else 0)
        return w

    def circulant_apply(self, c, x):
        c = np.ascontiguousarray(c, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        st = self._capply(c.shape[0], ptr(c), ptr(x), ptr(y))
        return y, st

    def matmul_by_circulant(self, a, c):
        a = np.ascontiguousarray(a, dtype=np.float64)
        c = np.ascontiguousarray(c, dtype=np.float64)
        out = np.empty_like(a)
        st = self._mcirc(a.shape[0], a.shape[1], ptr(a), ptr(c), ptr(out))
        return out, st

    def matmul_by_toeplitz_block(self, a, c, l):
        a = np.ascontiguousarray(a, dtype=np.float64)
        c = np.ascontiguousarray(c, dtype=np.float64)
        out = np.empty((a.shape[0], l))
        st = self._mtoep(a.shape[0], a.shape[1], ptr(a), c.shape[0], ptr(c), l, ptr(out))
        return out, st

    def preprocess_solve(self, a, b, post_kind=0, seed=0, refine=0):
        """post_kind 0 none / 1 Gaussian(seed) / 2 reference RealCirculant(seed)"""
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        n = a.shape[0]
        x = np.empty(n)
        hist = np.empty(refine + 1)
        div = ctypes.c_int(0)
        zs = np.zeros(1, np.int64)
        st = self._pre(n, ptr(a), ptr(b), post_kind, seed, refine, ptr(x), ptr(hist), ctypes.byref(div), ptr(zs))
        return dict(x=x, history=hist, diverged=bool(div.value), status=st, zero_step=int(zs[0]))

    def preprocess_solve_spec(self, a, b, pre=(0, 0, 0), post=(0, 0, 0), refine=0, card=65536):
        """preprocess_solve with MultiplierSpecs given as (kind, variant, seed),
        kinds = the reference's MultiplierKind ordinals"""
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        n = a.shape[0]
        x = np.empty(n)
        hist = np.empty(refine + 1)
        div = ctypes.c_int(0)
        zs = np.zeros(1, np.int64)
        st = self._pre2(n, ptr(a), ptr(b), pre[0], pre[1], pre[2], post[0], post[1], post[2], card, refine, ptr(x),
                        ptr(hist), ctypes.byref(div), ptr(zs))
        return dict(x=x, history=hist, diverged=bool(div.value), status=st, zero_step=int(zs[0]))

    def range_sketch(self, a, l, kind, seed, variant=0, power_steps=0, card=65536):
        """range_find's sketch (lowrank.hpp:51-81) -> (Y, status)"""
        a = np.ascontiguousarray(a, dtype=np.float64)
        m, n = a.shape
        y = np.empty((m, l))
        st = self._sketch(m, n, ptr(a), l, kind, variant, seed, card, power_steps, ptr(y))
        return y, st

    def materialize(self, kind, rows, cols, seed, variant=0, card=65536):
        out = np.empty((rows, cols))
        st = self._mat(kind, variant, seed, card, rows, cols, ptr(out))
        return out, st

    # ---- complex field (numpy complex128 in and out) ----
    @staticmethod
    def _z(a):
        return np.ascontiguousarray(a, dtype=np.complex128)

    def zgenp_factor(self, a):
        a = self._z(a)
        n = a.shape[0]
        lu = np.empty((n, n), np.complex128)
        zs = np.zeros(1, np.int64)
        st = self._zgenp(n, ptr(a.view(np.float64)), ptr(lu.view(np.float64)), ptr(zs))
        return lu, st, int(zs[0])

    def zpreprocess_solve_spec(self, a, b, pre=(0, 0, 0), post=(0, 0, 0), refine=0, card=65536):
        a, b = self._z(a), self._z(b)
        n = a.shape[0]
        x = np.empty(n, np.complex128)
        hist = np.empty(refine + 1)
        div = ctypes.c_int(0)
        zs = np.zeros(1, np.int64)
        st = self._zpre(n, ptr(a.view(np.float64)), ptr(b.view(np.float64)), pre[0], pre[1], pre[2], post[0],
                        post[1], post[2], card, refine, ptr(x.view(np.float64)), ptr(hist), ctypes.byref(div), ptr(zs))
        return dict(x=x, history=hist, diverged=bool(div.value), status=st, zero_step=int(zs[0]))

    def zmaterialize(self, kind, rows, cols, seed, variant=0, card=65536):
        out = np.empty((rows, cols), np.complex128)
        st = self._zmat(kind, variant, seed, card, rows, cols, ptr(out.view(np.float64)))
        return out, st

    def zrange_sketch(self, a, l, kind, seed, variant=0, power_steps=0, card=65536):
        a = self._z(a)
        m, n = a.shape
        y = np.empty((m, l), np.complex128)
        st = self._zsketch(m, n, ptr(a.view(np.float64)), l, kind, variant, seed, card, power_steps,
                           ptr(y.view(np.float64)))
        return y, st

    def gen_unitary_circulant(self, n, seed):
        out = np.empty(n, np.complex128)
        self._ucirc(n, seed, ptr(out.view(np.float64)))
        return out

    def srft_columns(self, n, l, seed):
        out = np.empty(l, np.int64)
        self._srftc(n, l, seed, ptr(out))
        return out

    def srft_matrix(self, n, l, seed, variant=0):
        out = np.empty((n, l), np.complex128)
        st = self._srftm(n, l, seed, variant, ptr(out.view(np.float64)))
        return out, st

    def zspectral_norm_estimate(self, a):
        a = self._z(a)
        return float(self._znormest(a.shape[0], a.shape[1], ptr(a.view(np.float64))))

    def gaussian_derived(self, seed, key, count):
        out = np.empty(count)
        self._gder(seed, key, count, ptr(out))
        return out

    def dft_dense(self, n):
        out = np.empty((n, n), np.complex128)
        st = self._dft(n, ptr(out.view(np.float64)))
        assert st == 0
        return out

    def batched_config2(self, count, base=7, i0=0, dim=32):
        x = np.empty((count, dim))
        res = np.empty(count)
        nf = self._batch(dim, base, i0, count, ptr(x), ptr(res))
        return dict(x=x, resid=res, failures=int(nf))

    def parallel_dense_trials(self, a_all, b_all, seeds):
        a_all = np.ascontiguousarray(a_all, dtype=np.float64)
        b_all = np.ascontiguousarray(b_all, dtype=np.float64)
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        t, n, _ = a_all.shape
        res = np.empty(t)
        nf = self._trials(n, t, ptr(a_all), ptr(b_all), ptr(seeds), ptr(res))
        return res, int(nf)


_clib = _load(os.path.join(HERE, "liboracle.so"))
C = _C(_clib) if _clib is not None else None
_rlib = _load(os.path.join(HERE, "_ref", "librandla_ref.so"))
REF = _Ref(_rlib) if _rlib is not None else None
