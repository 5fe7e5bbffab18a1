"""Reference-shaped host API over the C ABI.

Mirrors the `randla` header API for the hot path (namespace randla,
/root/reference/proj/include/randla/*.hpp, double instantiation): the same
function names, argument meaning and error behaviour (typed exceptions
carrying the 1-based step / position). Arrays are numpy (host, the drop-in
form: every call stages through the device) or torch CUDA tensors (device
pointers, no host round trip); results come back in the same form.

The computation always runs in librandla_b200.so on the GPU; there is no CPU
path in this module.
"""
import ctypes
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import capi


# ---- error contract (types.hpp:44-78) ------------------------------------
class RandlaError(RuntimeError):
    pass


class DimensionError(ValueError):
    """randla::DimensionError (std::invalid_argument), types.hpp:44-46"""


class SingularMatrixError(RandlaError):
    """types.hpp:48-50"""


class RankDeficiencyError(RandlaError):
    """types.hpp:52-54"""

    def __init__(self, msg, column=0):
        super().__init__(msg)
        self.column = column


class ZeroPivotError(RandlaError):
    """GENP met a pivot below tolerance at `step` (1-based), types.hpp:56-62"""

    def __init__(self, step):
        super().__init__(f"zero pivot at elimination step {step}")
        self.step = step


class SingularPivotBlockError(RandlaError):
    """types.hpp:64-68"""

    def __init__(self, position):
        super().__init__(f"numerically singular pivot block at position {position}")
        self.position = position


class LogicError(RuntimeError):
    """std::logic_error — real circulant product with non-negligible imaginary
    part (circulant.hpp:63-64)"""


class DeviceError(RuntimeError):
    pass


def _raise(status, info_step=0, what=""):
    if status == capi.RL_OK:
        return
    msg = capi.last_error() or what
    if status == capi.RL_ERR_DIMENSION:
        raise DimensionError(msg)
    if status == capi.RL_ERR_ZERO_PIVOT:
        raise ZeroPivotError(info_step)
    if status == capi.RL_ERR_SINGULAR_PIVOT_BLOCK:
        raise SingularPivotBlockError(info_step)
    if status == capi.RL_ERR_RANK_DEFICIENCY:
        raise RankDeficiencyError(msg, info_step)
    if status == capi.RL_ERR_SINGULAR_MATRIX:
        raise SingularMatrixError(msg)
    if status == capi.RL_ERR_LOGIC:
        raise LogicError(msg)
    raise DeviceError(f"librandla_b200 status {status}: {msg}")


# ---- multipliers (multipliers.hpp:20-56) ------------------------------------
class MultiplierKind(enum.IntEnum):
    """randla::MultiplierKind (multipliers.hpp:20-29), the same ordinals; the
    reference's CamelCase names are aliases. In this real pipeline the complex
    families raise DimensionError exactly where the reference's real
    instantiation does. GAUSSIAN_CIRCULANT is an extension outside the
    reference's range: RealCirculant(gen_gaussian_vector(n, seed)), the
    N(0,1)-column circulant of BASELINE configs 3 and 5."""
    NONE = capi.RL_MULT_NONE
    GAUSSIAN = capi.RL_MULT_GAUSSIAN
    REAL_CIRCULANT = capi.RL_MULT_REAL_CIRCULANT          # uniform[-1,1] first column
    UNITARY_CIRCULANT = capi.RL_MULT_UNITARY_CIRCULANT
    TOEPLITZ_BLOCK = capi.RL_MULT_TOEPLITZ_BLOCK
    SRFT = capi.RL_MULT_SRFT
    FINITE_SET_UNIFORM = capi.RL_MULT_FINITE_SET_UNIFORM
    CIRC_SKEW_PRODUCT = capi.RL_MULT_CIRC_SKEW_PRODUCT
    GAUSSIAN_CIRCULANT = capi.RL_MULT_GAUSSIAN_CIRCULANT  # extension: N(0,1) first column
    # the reference's spellings
    None_ = capi.RL_MULT_NONE
    Gaussian = capi.RL_MULT_GAUSSIAN
    RealCirculant = capi.RL_MULT_REAL_CIRCULANT
    UnitaryCirculant = capi.RL_MULT_UNITARY_CIRCULANT
    ToeplitzBlock = capi.RL_MULT_TOEPLITZ_BLOCK
    Srft = capi.RL_MULT_SRFT
    FiniteSetUniform = capi.RL_MULT_FINITE_SET_UNIFORM
    CircSkewProduct = capi.RL_MULT_CIRC_SKEW_PRODUCT


class ToeplitzVariant(enum.IntEnum):
    """randla::ToeplitzVariant (multipliers.hpp:31)"""
    REAL = capi.RL_TOEPLITZ_REAL
    UNITARY = capi.RL_TOEPLITZ_UNITARY
    Real = capi.RL_TOEPLITZ_REAL
    Unitary = capi.RL_TOEPLITZ_UNITARY


@dataclass
class MultiplierSpec:
    """randla::MultiplierSpec (multipliers.hpp:33-40): the same fields
    (rows / cols 0 = taken from the call, as SideMultiplier::make and
    range_find set them), plus two B200 extras: an explicit `dense` multiplier
    or circulant first `column` instead of the seeded draw."""
    kind: MultiplierKind = MultiplierKind.NONE
    seed: int = 0
    rows: int = 0
    cols: int = 0
    set_cardinality: int = 65536
    variant: ToeplitzVariant = ToeplitzVariant.REAL
    dense: Optional[object] = None
    column: Optional[object] = None


def multiplier_is_complex(spec):
    """multipliers.hpp:42-52"""
    return spec.kind in (MultiplierKind.UNITARY_CIRCULANT, MultiplierKind.SRFT) or (
        spec.kind == MultiplierKind.TOEPLITZ_BLOCK and spec.variant == ToeplitzVariant.UNITARY)


def derive_seed(seed, k1, k2=0):
    """multipliers.hpp:54-56"""
    return int(capi.lib().rl_derive_seed(seed, k1, k2))


def hash_label(label):
    """rng.hpp:87-95"""
    return int(capi.lib().rl_hash_label(label.encode()))


def gen_gaussian(m, n, seed):
    """multipliers.hpp:58-65 — bit-identical to the reference generator."""
    out = np.empty((m, n))
    _raise(capi.lib().rl_gen_gaussian(m, n, seed, out.ctypes.data))
    return out


def gen_gaussian_vector(n, seed):
    """testbed/inputs.hpp:85-90"""
    return gen_gaussian(n, 1, seed).reshape(n)


def gen_gaussian_batch(count, m, n, seeds):
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = np.empty((count, m, n))
    _raise(capi.lib().rl_gen_gaussian_batch(count, m, n, seeds.ctypes.data, out.ctypes.data))
    return out


def gen_real_circulant_column(n, seed):
    """multipliers.hpp:67-73 (first column of gen_real_circulant)"""
    out = np.empty(n)
    _raise(capi.lib().rl_gen_real_circulant_column(n, seed, out.ctypes.data))
    return out


def gen_real_circulant(n, seed):
    """gen_real_circulant (multipliers.hpp:67-73): first column uniform on [-1, 1]"""
    return RealCirculant(gen_real_circulant_column(n, seed))


def gen_real_toeplitz_block(n, l, seed):
    """gen_real_toeplitz_block (multipliers.hpp:84-86)"""
    return ToeplitzBlock(gen_real_circulant(n, seed), n, l)


def gen_finite_set_uniform(m, n, seed, cardinality):
    """gen_finite_set_uniform (multipliers.hpp:142-154), bit-identical."""
    if cardinality < 2:
        raise DimensionError("gen_finite_set_uniform: cardinality must be >= 2")
    out = np.empty((m, n))
    _raise(capi.lib().rl_gen_finite_set_uniform(m, n, seed, cardinality, out.ctypes.data))
    return out


def materialize(spec, device=False):
    """materialize<double>(spec) (multipliers.hpp:174-218): the dense sample
    of a real family (spec.rows x spec.cols), generated by the reference's
    generators; circulant and skew-product expansions run on the GPU."""
    if spec.rows <= 0 or spec.cols <= 0:
        raise DimensionError("materialize: spec.rows and spec.cols must be set")
    if multiplier_is_complex(spec):
        raise DimensionError("complex multiplier family requested in a real pipeline")
    out = _empty_like_kind(device, (spec.rows, spec.cols))
    m, keep = _multiplier(spec, device)
    _sync_stream_for(device)
    _raise(capi.lib().rl_materialize(_ctx(), _mem(device), ctypes.byref(m), spec.rows, spec.cols, capi.addr(out)))
    del keep
    return out


# ---- array plumbing ----------------------------------------------------------
def _is_device(*arrays):
    dev = None
    for a in arrays:
        if a is None:
            continue
        d = not isinstance(a, np.ndarray)
        if dev is None:
            dev = d
        elif dev != d:
            raise DimensionError("mixing host (numpy) and device (torch) arrays in one call")
    return bool(dev)


def _host(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _dev(a):
    import torch
    if a.dtype != torch.float64 or not a.is_cuda:
        raise DimensionError("device arrays must be float64 CUDA tensors")
    return a.contiguous()


def _empty_like_kind(device, shape, ref=None):
    if device:
        import torch
        return torch.empty(shape, dtype=torch.float64, device=ref.device if ref is not None else "cuda")
    return np.empty(shape)


def _ctx():
    return None  # per-thread default context


def _mem(device):
    return capi.RL_DEVICE if device else capi.RL_HOST


def _sync_stream_for(device):
    """Device calls run on the context stream; make torch's current stream the
    context stream so ordering with surrounding torch work is preserved."""
    if device:
        import torch
        capi.lib().rl_context_set_stream(None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))


# ---- batched small GENP (BASELINE config 2) ----------------------------------
@dataclass
class BatchedSolve:
    lu: object
    x: object
    residual: object
    growth: object
    status: object
    summary: dict


def batched_preprocess_solve_32(a, g, b, want_lu=True, want_summary=True):
    """Many independent preprocess_solve(A_i, b_i, none, {Gaussian, G_i}, 0)
    (preprocess.hpp:156-180) on 32x32 systems. a, g: (batch, 32, 32); b: (batch, 32).
    Per-system ZeroPivot verdicts are returned in `status` (1-based step, 0 = ok)
    instead of raising, as the reference's trial engine counts them
    (testbed/experiment.hpp:36-40)."""
    device = _is_device(a, g, b)
    if a.shape[-2:] != (32, 32) or g.shape != a.shape or b.shape != a.shape[:-1]:
        raise DimensionError("batched_preprocess_solve_32: shapes must be (B,32,32), (B,32,32), (B,32)")
    batch = a.shape[0]
    if device:
        import torch
        a, g, b = _dev(a), _dev(g), _dev(b)
        lu = torch.empty_like(a) if want_lu else None
        x = torch.empty_like(b)
        r = torch.empty(batch, dtype=torch.float64, device=a.device)
        gr = torch.empty_like(r)
        st = torch.empty(batch, dtype=torch.int32, device=a.device)
    else:
        a, g, b = _host(a), _host(g), _host(b)
        lu = np.empty_like(a) if want_lu else None
        x = np.empty_like(b)
        r = np.empty(batch)
        gr = np.empty(batch)
        st = np.empty(batch, np.int32)
    _sync_stream_for(device)
    summ = capi.rl_batch_summary()
    rc = capi.lib().rl_batched_genp_solve_32(_ctx(), _mem(device), batch, capi.addr(a), capi.addr(g), capi.addr(b),
                                             capi.addr(lu), capi.addr(x), capi.addr(r), capi.addr(gr),
                                             capi.addr(st), ctypes.byref(summ) if want_summary else None)
    _raise(rc)
    s = {k: getattr(summ, k) for k, _ in summ._fields_} if want_summary else {}
    return BatchedSolve(lu, x, r, gr, st, s)


# ---- dense products ------------------------------------------------------------
def matmul(a, b):
    """matmul (matrix.hpp:115-121): C = A B, FP64 DMMA on the GPU."""
    if _any_complex(a, b):
        return _zmatmul(a, b)
    device = _is_device(a, b)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise DimensionError("matmul: inner dimensions differ")
    m, k = a.shape
    n = b.shape[1]
    if device:
        a, b = _dev(a), _dev(b)
        c = _empty_like_kind(True, (m, n), a)
    else:
        a, b = _host(a), _host(b)
        c = np.empty((m, n))
    _sync_stream_for(device)
    _raise(capi.lib().rl_dgemm(_ctx(), _mem(device), m, n, k, capi.addr(a), k, capi.addr(b), n, capi.addr(c), n))
    return c


def svd_values(a):
    """svd_values (svd.hpp:76-88): the min(m, n) singular values, non-increasing,
    by the device's one-sided Jacobi (small matrices: one CTA)."""
    if _any_complex(a):
        return _zsvd_values(a)
    device = _is_device(a)
    a = _dev(a) if device else _host(a)
    m, n = a.shape
    out = np.empty(min(m, n))
    if device:
        a = a.cpu().numpy()
    _raise(capi.lib().rl_singular_values(_ctx(), capi.RL_HOST, m, n, capi.addr(_host(a)), capi.addr(out)))
    return out


def spectral_norm(a):
    """spectral_norm (norms.hpp:11-14) = svd_values(a)[0]"""
    return float(svd_values(a)[0])


def spectral_norm_estimate(a):
    """spectral_norm_estimate (norms.hpp:35-78), evaluated on the GPU in the
    reference's summation order (bit-identical for a given matrix)."""
    device = _is_device(a)
    a = _dev(a) if device else _host(a)
    m, n = a.shape
    out = ctypes.c_double(0.0)
    _sync_stream_for(device)
    _raise(capi.lib().rl_spectral_norm_estimate(_ctx(), _mem(device), m, n, capi.addr(a), ctypes.byref(out)))
    return out.value


# ---- GENP (lu.hpp) ---------------------------------------------------------------
@dataclass
class LuFactors:
    """LuFactors (lu.hpp:17-28) held packed: strict lower = L (unit diagonal),
    upper incl. diagonal = U; perm is always None (no pivoting)."""
    packed: object
    perm: object = None
    info: dict = field(default_factory=dict)

    @property
    def lower(self):
        p = self.packed
        if isinstance(p, np.ndarray):
            return np.tril(p, -1) + np.eye(p.shape[0])
        import torch
        return torch.tril(p, -1) + torch.eye(p.shape[0], dtype=p.dtype, device=p.device)

    @property
    def upper(self):
        p = self.packed
        if isinstance(p, np.ndarray):
            return np.triu(p)
        import torch
        return torch.triu(p)

    def pivots(self):
        p = self.packed
        return np.diag(p).copy() if isinstance(p, np.ndarray) else p.diagonal().clone()


def genp_factor(a):
    """genp_factor (lu.hpp:40-58): unpivoted elimination; raises
    ZeroPivotError(step) exactly when the reference does."""
    device = _is_device(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionError("genp_factor: square input required")
    n = a.shape[0]
    a = _dev(a) if device else _host(a)
    lu = _empty_like_kind(device, (n, n), a)
    info = capi.rl_solve_info()
    _sync_stream_for(device)
    rc = capi.lib().rl_genp_factor(_ctx(), _mem(device), n, capi.addr(a), capi.addr(lu), ctypes.byref(info))
    _raise(rc, info.zero_pivot_step)
    return LuFactors(lu, None, info.as_dict())


def lu_solve(f, b):
    """lu_solve (lu.hpp:100-123) on packed factors (GENP, or GEPP when f.perm
    is set)."""
    if isinstance(f, LuFactors) and f.perm is not None:
        return _gepp_solve(f, b, False)
    lu = f.packed if isinstance(f, LuFactors) else f
    device = _is_device(lu, b)
    n = lu.shape[0]
    if b.shape[0] != n:
        raise DimensionError("lu_solve: length mismatch")
    lu = _dev(lu) if device else _host(lu)
    b = _dev(b) if device else _host(b)
    x = _empty_like_kind(device, (n,), b)
    _sync_stream_for(device)
    _raise(capi.lib().rl_lu_solve(_ctx(), _mem(device), n, capi.addr(lu), capi.addr(b), capi.addr(x)))
    return x


# ---- block elimination (block_ge.hpp) ----------------------------------------------
def _index_like(device, n, ref=None):
    if device:
        import torch
        return torch.empty(n, dtype=torch.int64, device=ref.device if ref is not None else "cuda")
    return np.empty(n, dtype=np.int64)


def gepp_factor(a):
    """gepp_factor (lu.hpp:62-98): partial pivoting (first maximal |u_ij|),
    bit-identical to the reference; raises SingularMatrixError when the best
    pivot is <= tol_pivot(n) * spectral_norm_estimate(a)."""
    device = _is_device(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionError("gepp_factor: square input required")
    n = a.shape[0]
    a = _dev(a) if device else _host(a)
    lu = _empty_like_kind(device, (n, n), a)
    perm = _index_like(device, n, a)
    step = ctypes.c_int64(0)
    _sync_stream_for(device)
    _raise(capi.lib().rl_gepp_factor(_ctx(), _mem(device), n, capi.addr(a), capi.addr(lu), capi.addr(perm),
                                     ctypes.byref(step)), step.value)
    return LuFactors(lu, perm)


def _gepp_solve(f, b, transpose):
    lu, perm = f.packed, f.perm
    device = _is_device(lu, b)
    n = lu.shape[0]
    if perm is None:  # GENP factors: identity permutation
        perm = _index_like(device, n, lu)
        if device:
            import torch
            torch.arange(n, out=perm)
        else:
            perm[:] = np.arange(n)
    if b.shape[0] != n:
        raise DimensionError("lu_solve: length mismatch")
    nrhs = 1 if b.ndim == 1 else b.shape[1]
    lu = _dev(lu) if device else _host(lu)
    b = _dev(b) if device else _host(b)
    x = _empty_like_kind(device, tuple(b.shape), b)
    _sync_stream_for(device)
    _raise(capi.lib().rl_gepp_solve(_ctx(), _mem(device), n, nrhs, capi.addr(lu), capi.addr(perm), capi.addr(b),
                                    capi.addr(x), 1 if transpose else 0))
    return x


def lu_solve_transpose(f, c):
    """lu_solve_transpose (lu.hpp:127-147): solves A^T x = c from A's factors
    (GEPP or GENP); c may hold several right-hand sides as columns."""
    return _gepp_solve(f, c, True)


def balanced_split(n):
    """balanced_split (block_ge.hpp:184-194): halve until scalar blocks."""
    out, remaining = [], n
    while remaining > 1:
        half = remaining // 2
        out.append(half)
        remaining -= half
    out.append(remaining)
    return out


@dataclass
class BlockNode:
    """BlockNode (block_ge.hpp:18-35): an internal node eliminates the first
    pivot_size rows/columns; leaves hold their block and its GEPP factors."""
    dim: int
    offset: int
    pivot_size: int = 0
    block_matrix: object = None
    block_lu: object = None
    db_inv: object = None
    b_inv_c: object = None
    pivot_child: object = None
    schur_child: object = None

    def leaf(self):
        return self.pivot_size == 0


def _copy(x):
    return x.copy() if isinstance(x, np.ndarray) else x.clone()


class BlockFactorization:
    """BlockFactorization (block_ge.hpp:37-83) over the flat device factors of
    rl_block_ge_factor: the tree's blocks are copies of their regions."""

    def __init__(self, factors, perm, leaf_blocks, split):
        self.factors, self.perm, self.split = factors, perm, list(split)
        n = factors.shape[0]
        offs, o = [], 0
        for i, k in enumerate(self.split):
            offs.append((o, n - o if i + 1 == len(self.split) else k))
            o += offs[-1][1]

        def leaf(o, k):
            f = factors[o:o + k, o:o + k]
            return BlockNode(k, o, 0, _copy(leaf_blocks[o:o + k, o:o + k]), LuFactors(_copy(f), _copy(perm[o:o + k])))

        node = None
        for o, k in reversed(offs):
            if node is None:
                node = leaf(o, k)
                continue
            node = BlockNode(n - o, o, k, None, None, _copy(factors[o + k:, o:o + k]), _copy(factors[o:o + k, o + k:]),
                             leaf(o, k), node)
        self.root = node

    def pivots(self):
        """Elimination pivots in order: the leaves' U diagonals (block_ge.hpp:43-48)."""
        f = self.factors
        return np.diag(f).copy() if isinstance(f, np.ndarray) else f.diagonal().clone()

    def reassemble(self):
        """reassemble (block_ge.hpp:50-80): rebuild the input from the tree."""
        def rec(node):
            if node.leaf():
                lu = matmul(node.block_lu.lower, node.block_lu.upper)
                out = _copy(lu)
                out[node.block_lu.perm] = lu  # A(perm[i], :) = (L U)(i, :)
                return out
            b, sc = rec(node.pivot_child), rec(node.schur_child)
            c = matmul(b, node.b_inv_c)
            d = matmul(node.db_inv, b)
            k = node.pivot_size
            out = _copy(node.db_inv.new_zeros((node.dim, node.dim)) if not isinstance(b, np.ndarray)
                        else np.zeros((node.dim, node.dim)))
            out[:k, :k] = b
            out[:k, k:] = c
            out[k:, :k] = d
            out[k:, k:] = sc + matmul(node.db_inv, c)
            return out
        return rec(self.root)


def block_ge_factor(a, split):
    """block_ge_factor (block_ge.hpp:168-181): recursive block elimination
    along `split` (pivot block sizes in elimination order), the reference's
    arithmetic order throughout (leaf GEPP, strips by lu_solve /
    lu_solve_transpose, natural-order Schur complements). Raises
    DimensionError on a bad split, SingularPivotBlockError(offset + 1) when a
    pivot block's smallest singular value is <= tol_pivot(n) *
    spectral_norm_estimate(a), SingularMatrixError from a leaf's GEPP."""
    device = _is_device(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionError("block_ge_factor: square input required")
    n = a.shape[0]
    split = [int(k) for k in split]
    if not split or sum(split) != n:
        raise DimensionError("block_ge_factor: split must sum to the dimension")
    if any(k == 0 for k in split):
        raise DimensionError("block_ge_factor: zero block size")
    a = _dev(a) if device else _host(a)
    factors = _empty_like_kind(device, (n, n), a)
    leaves = _empty_like_kind(device, (n, n), a)
    perm = _index_like(device, n, a)
    sp = (ctypes.c_int64 * len(split))(*split)
    pos = ctypes.c_int64(0)
    _sync_stream_for(device)
    _raise(capi.lib().rl_block_ge_factor(_ctx(), _mem(device), n, capi.addr(a), len(split), sp, capi.addr(factors),
                                         capi.addr(perm), capi.addr(leaves), ctypes.byref(pos)), pos.value)
    return BlockFactorization(factors, perm, leaves, split)


def block_solve(f, b):
    """block_solve (block_ge.hpp:198-201) on a block_ge_factor result."""
    n = f.factors.shape[0]
    if b.shape[0] != n:
        raise DimensionError("block_solve: length mismatch")
    device = _is_device(f.factors, b)
    b = _dev(b) if device else _host(b)
    x = _empty_like_kind(device, (n,), b)
    sp = (ctypes.c_int64 * len(f.split))(*f.split)
    _sync_stream_for(device)
    _raise(capi.lib().rl_block_solve(_ctx(), _mem(device), n, len(f.split), sp, capi.addr(f.factors),
                                     capi.addr(f.perm), capi.addr(b), capi.addr(x)))
    return x


def schur_complement(a, k):
    """schur_complement (block_ge.hpp:202-218): E - D (B^-1 C) for the leading
    k x k block B, B factored by gepp_factor (raises SingularMatrixError on a
    singular leading block); the product D X on the FP64 tensor path."""
    n = a.shape[0]
    if a.ndim != 2 or a.shape[1] != n:
        raise DimensionError("schur_complement: square input required")
    if k <= 0 or k >= n:
        raise DimensionError("schur_complement: need 0 < k < n")
    device = _is_device(a)
    a = _dev(a) if device else _host(a)
    b_lu = gepp_factor(_copy(a[:k, :k]) if device else np.ascontiguousarray(a[:k, :k]))
    c = a[:k, k:].contiguous() if device else np.ascontiguousarray(a[:k, k:])
    x = _gepp_solve(b_lu, c, False)
    d = a[k:, :k].contiguous() if device else np.ascontiguousarray(a[k:, :k])
    return a[k:, k:] - matmul(d, x)


# ---- preprocessed solve (preprocess.hpp) -------------------------------------------
@dataclass
class SolveOutcome:
    """SolveOutcome (preprocess.hpp:9-14) plus the device diagnostics."""
    x: object
    residual_history: List[float]
    diverged: bool
    info: dict
    lu: object = None


def _multiplier(spec, device):
    m = capi.rl_multiplier()
    if spec is None:
        m.kind = capi.RL_MULT_NONE
        return m, []
    m.kind = int(spec.kind)
    m.variant = int(getattr(spec, "variant", 0))
    m.set_cardinality = int(getattr(spec, "set_cardinality", 65536))
    m.seed = int(spec.seed) & 0xFFFFFFFFFFFFFFFF
    keep = []
    if spec.dense is not None:
        d = _dev(spec.dense) if device else _host(spec.dense)
        keep.append(d)
        m.dense = capi.addr(d)
    if spec.column is not None:
        c = _dev(spec.column) if device else _host(spec.column)
        keep.append(c)
        m.column = capi.addr(c)
    return m, keep


def _check_side(spec, n):
    """SideMultiplier::make's shape rule (preprocess.hpp:29-32)"""
    if spec is None:
        return
    rows = spec.rows or n
    cols = spec.cols or n
    if rows != n or cols != n:
        raise DimensionError("solve preprocessing takes square n-by-n multipliers")


def preprocess_solve(a, b, pre_spec=None, post_spec=None, refine_steps=0, want_lu=False, want_norm_a=False):
    """preprocess_solve(a, b, pre, post, refine) (preprocess.hpp:156-180):
    product F (A H) (dense sides by the DMMA GEMM, circulant sides through the
    FFT kernel), GENP, x = H (LU)^-1 (F b), refinement steps. Raises
    ZeroPivotError like the reference; retry with preprocess_solve_with_retry."""
    if _any_complex(a, b):
        return _zpreprocess_solve(a, b, pre_spec, post_spec, refine_steps, want_lu)
    device = _is_device(a, b)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionError("preprocess_solve: square input required")
    n = a.shape[0]
    if b.shape[0] != n:
        raise DimensionError("preprocess_solve: length mismatch")
    _check_side(pre_spec, n)
    _check_side(post_spec, n)
    if refine_steps < 0:
        raise DimensionError("preprocess_solve: negative refine_steps")
    a = _dev(a) if device else _host(a)
    b = _dev(b) if device else _host(b)
    x = _empty_like_kind(device, (n,), b)
    lu = _empty_like_kind(device, (n, n), a) if want_lu else None
    m, keep = _multiplier(post_spec, device)
    fm, fkeep = _multiplier(pre_spec, device)
    info = capi.rl_solve_info()
    hist = (ctypes.c_double * (refine_steps + 1))()  # SolveOutcome::residual_history has refine + 1 entries
    info.history = ctypes.cast(hist, ctypes.POINTER(ctypes.c_double))
    info.history_capacity = refine_steps + 1
    _sync_stream_for(device)
    rc = capi.lib().rl_preprocessed_genp_solve(_ctx(), _mem(device), n, capi.addr(a), capi.addr(b), ctypes.byref(fm),
                                               ctypes.byref(m), refine_steps, capi.addr(x), capi.addr(lu),
                                               1 if want_norm_a else 0, ctypes.byref(info))
    del keep, fkeep
    _raise(rc, info.zero_pivot_step)
    d = info.as_dict()
    return SolveOutcome(x, d["residual_history"], bool(info.diverged), d, lu)


def preprocess_solve_with_retry(a, b, pre_spec, post_spec, refine_steps=0, max_retries=3):
    """preprocess.hpp:182-196: on ZeroPivot reseed with
    derive_seed(seed, 0x52455452, attempt + 1)."""
    import copy
    pre = copy.copy(pre_spec) if pre_spec is not None else MultiplierSpec()
    post = copy.copy(post_spec) if post_spec is not None else MultiplierSpec()
    for attempt in range(max_retries + 1):
        try:
            return preprocess_solve(a, b, pre, post, refine_steps)
        except ZeroPivotError:
            if attempt >= max_retries:
                raise
            pre.seed = derive_seed(pre.seed, 0x52455452, attempt + 1)
            post.seed = derive_seed(post.seed, 0x52455452, attempt + 1)


# ---- FFT and structured multipliers (fft.hpp, circulant.hpp) ---------------------
def _fft(v, inverse):
    device = _is_device(v)
    if device:
        import torch
        if not v.is_complex():
            v = v.to(torch.complex128)
        z = v.to(torch.complex128).contiguous().clone()
        n = z.shape[-1]
        count = z.numel() // n if n else 0
        zr = torch.view_as_real(z)
    else:
        z = np.array(v, dtype=np.complex128, copy=True, order="C")
        n = z.shape[-1] if z.ndim else 0
        count = z.size // n if n else 0
        zr = z.view(np.float64)
    if n == 0:
        raise DimensionError("inverse_fft: empty input" if inverse else "fft: empty input")
    _sync_stream_for(device)
    _raise(capi.lib().rl_fft(_ctx(), _mem(device), count, n, capi.addr(zr), 1 if inverse else 0))
    return z


def fft(v):
    """fft (fft.hpp:76-86): Omega v with omega = exp(+2 pi i / n), the
    reference's sign; a batch of vectors along the last axis. Real input is
    promoted to complex (fft.hpp:86)."""
    return _fft(v, False)


def inverse_fft(v):
    """inverse_fft (fft.hpp:88-98): Omega^-1 v = Omega^H v / n."""
    return _fft(v, True)


class CirculantMatrix:
    """CirculantMatrix<double> / RealCirculant (circulant.hpp:17-50): held by
    its first column, entry (i, j) = c[(i - j) mod n]; the spectrum fft(c) is
    computed on the GPU at construction, as the reference does eagerly."""

    def __init__(self, first_column):
        c = first_column
        if (isinstance(c, np.ndarray) and c.size == 0) or len(c) == 0:
            raise DimensionError("circulant: empty first column")
        self._c = c if not isinstance(c, (list, tuple)) else np.asarray(c, dtype=np.float64)
        self._spectrum = None

    def size(self):
        return int(self._c.shape[0])

    def first_column(self):
        return self._c

    def spectrum(self):
        if self._spectrum is None:
            self._spectrum = fft(self._c)
        return self._spectrum

    def entry(self, i, j):
        n = self.size()
        return self._c[(i + n - j) % n]

    def dense(self):
        n = self.size()
        if _any_complex(self._c):  # entry (i, j) = c[(i - j) mod n] (circulant.hpp:27-36): a gather
            idx = (np.arange(n)[:, None] - np.arange(n)[None, :]) % n
            if isinstance(self._c, np.ndarray):
                return self._c[idx]
            import torch
            return self._c[torch.from_numpy(idx).to(self._c.device)]
        spec = MultiplierSpec(MultiplierKind.REAL_CIRCULANT, 0, n, n, column=self._c)
        return materialize(spec, device=_is_device(self._c))

    def transposed(self):
        """circulant.hpp:40-45: first column c[(n - i) mod n]"""
        n = self.size()
        idx = (n - np.arange(n)) % n
        if isinstance(self._c, np.ndarray):
            return CirculantMatrix(self._c[idx].copy())
        import torch
        return CirculantMatrix(self._c[torch.from_numpy(idx).to(self._c.device)].contiguous())


RealCirculant = CirculantMatrix


class ToeplitzBlock:
    """ToeplitzBlock<double> (circulant.hpp:143-169): the leading rows x cols
    block of a parent circulant, entry (i, j) = c[(i - j) mod n]."""

    def __init__(self, parent, rows, cols):
        n = parent.size()
        if rows > n or cols > n or rows < 1 or cols < 1:
            raise DimensionError("toeplitz block exceeds parent dimensions")
        self.parent, self._rows, self._cols = parent, rows, cols

    def rows(self):
        return self._rows

    def cols(self):
        return self._cols

    def entry(self, i, j):
        return self.parent.entry(i, j)

    def dense(self):
        n = self.parent.size()
        spec = MultiplierSpec(MultiplierKind.TOEPLITZ_BLOCK, 0, self._rows, self._cols, column=self.parent.first_column())
        if self._rows != n:  # the block of a larger parent: expand the parent's leading block
            full = self.parent.dense()
            return full[: self._rows, : self._cols].copy() if isinstance(full, np.ndarray) else \
                full[: self._rows, : self._cols].contiguous()
        return materialize(spec, device=_is_device(self.parent.first_column()))


def _column_of(c):
    return c.first_column() if isinstance(c, CirculantMatrix) else c


def circulant_apply(c, x):
    """circulant_apply(RealCirculant, x) (circulant.hpp:91-96): C x by FFT on the GPU."""
    c = _column_of(c)
    if _any_complex(c, x):
        return _zcirculant_apply(c, x)
    device = _is_device(c, x)
    n = c.shape[0]
    if x.shape[0] != n:
        raise DimensionError("circulant_apply: length mismatch")
    c = _dev(c) if device else _host(c)
    x = _dev(x) if device else _host(x)
    y = _empty_like_kind(device, (n,), x)
    _sync_stream_for(device)
    _raise(capi.lib().rl_circulant_apply(_ctx(), _mem(device), n, capi.addr(c), capi.addr(x), capi.addr(y)))
    return y


def matmul_by_circulant(a, c):
    """matmul_by_circulant(A, C) (circulant.hpp:171-185): A (m x n) times the
    real circulant C (a RealCirculant or its first column), by FFT on the GPU."""
    c = _column_of(c)
    if _any_complex(a, c):
        if c.shape[0] != a.shape[1]:
            raise DimensionError("matmul_by_circulant: shape mismatch")
        return _zcirc_right(a, c, c.shape[0])
    device = _is_device(a, c)
    m, n = a.shape
    if c.shape[0] != n:
        raise DimensionError("matmul_by_circulant: shape mismatch")
    a = _dev(a) if device else _host(a)
    c = _dev(c) if device else _host(c)
    out = _empty_like_kind(device, (m, n), a)
    _sync_stream_for(device)
    _raise(capi.lib().rl_circulant_right_multiply(_ctx(), _mem(device), m, n, capi.addr(a), capi.addr(c),
                                                  capi.addr(out)))
    return out


def matmul_by_toeplitz_block(a, c, cols=None):
    """matmul_by_toeplitz_block(A, T) (circulant.hpp:187-203): A (m x k) times
    the Toeplitz block T (a ToeplitzBlock, or a parent first column c and the
    block's column count), by FFT on the GPU."""
    if isinstance(c, ToeplitzBlock):
        if a.shape[1] != c.rows():
            raise DimensionError("matmul_by_toeplitz_block: shape mismatch")
        c, cols = c.parent.first_column(), c.cols()
    if _any_complex(a, c):
        if a.shape[1] > c.shape[0] or cols > c.shape[0] or cols < 1:
            raise DimensionError("toeplitz block exceeds parent dimensions")
        return _zcirc_right(a, c, cols)
    device = _is_device(a, c)
    m, k = a.shape
    np_ = c.shape[0]
    if k > np_ or cols > np_ or cols < 1:
        raise DimensionError("toeplitz block exceeds parent dimensions")
    a = _dev(a) if device else _host(a)
    c = _dev(c) if device else _host(c)
    out = _empty_like_kind(device, (m, cols), a)
    _sync_stream_for(device)
    _raise(capi.lib().rl_toeplitz_right_multiply(_ctx(), _mem(device), m, k, capi.addr(a), np_, capi.addr(c), cols,
                                                 capi.addr(out)))
    return out


# ---- low-rank (qr.hpp, lowrank.hpp) ---------------------------------------------
def qr(y):
    """Thin QR with positive diagonal (qr.hpp:21-47) by CholeskyQR2 on the GPU;
    raises RankDeficiencyError(column) per qr.hpp:33-38."""
    device = _is_device(y)
    m, l = y.shape
    y = _dev(y) if device else _host(y)
    q = _empty_like_kind(device, (m, l), y)
    r = _empty_like_kind(device, (l, l), y)
    bad = ctypes.c_int64(0)
    _sync_stream_for(device)
    rc = capi.lib().rl_cholqr2(_ctx(), _mem(device), m, l, capi.addr(y), capi.addr(q), capi.addr(r), ctypes.byref(bad))
    _raise(rc, bad.value)
    return q, r


def orthonormal_basis(y):
    """qr.hpp:51-54"""
    return qr(y)[0]


@dataclass
class LowRankResult:
    """LowRankResult (lowrank.hpp:21-43) plus the residual norms evaluated on the
    device against the same A."""
    q: object
    rank: int
    oversample: int
    power_steps: int
    info: dict

    def sketch_width(self):
        return self.q.shape[1]


def range_find(a, r, p, spec, power_steps=0, with_residual=True):
    """range_find (lowrank.hpp:62-83): Y = A H (Toeplitz blocks through the FFT
    kernel, every other real family materialized and multiplied by the DMMA
    GEMM), power_steps alternating products Y <- A (A^T Y) (lowrank.hpp:51-57),
    Q = orthonormal_basis(Y). With with_residual (one call, A resident once)
    the result also carries ||A - Q Q^T A||_F and _2 of this A in `info`."""
    if _any_complex(a):
        return _zrange_find(a, r, p, spec, power_steps)
    device = _is_device(a)
    m, n = a.shape
    l = r + p
    if r < 1 or l > min(m, n):
        raise DimensionError("range_find: rank plus oversampling exceeds matrix size")
    if power_steps < 0:
        raise DimensionError("range_find: negative power_steps")
    a = _dev(a) if device else _host(a)
    q = _empty_like_kind(device, (m, l), a)
    mlt, keep = _multiplier(spec, device)
    info = capi.rl_lowrank_info()
    _sync_stream_for(device)
    fn = capi.lib().rl_range_find_residual if with_residual else capi.lib().rl_range_find
    rc = fn(_ctx(), _mem(device), m, n, capi.addr(a), l, ctypes.byref(mlt), power_steps, capi.addr(q),
            ctypes.byref(info))
    del keep
    _raise(rc, info.rank_deficient_column)
    d = {k: getattr(info, k) for k, _ in info._fields_ if k != "reserved"}
    if not with_residual:
        d = {"rank_deficient_column": d["rank_deficient_column"]}
    return LowRankResult(q, r, p, power_steps, d)


def basis_residual(result, truth_left):
    """basis_residual (lowrank.hpp:88-93): ||Q (Q^H S_r) - S_r||_2 for the
    leading left singular basis S_r, products and norm on the GPU."""
    q = result.q
    if _any_complex(q, truth_left):
        qh = np.ascontiguousarray(np.asarray(q).conj().T) if isinstance(q, np.ndarray) else q.conj().T.contiguous()
        d = matmul(q, matmul(qh, truth_left)) - truth_left
        return spectral_norm(d)
    y = matmul(np.ascontiguousarray(np.asarray(q).T) if isinstance(q, np.ndarray) else q.T.contiguous(), truth_left)
    d = matmul(q, y) - truth_left
    return spectral_norm(d)


def residual_norms(a, result):
    """||A - Q (Q^T A)||_F and ||.||_2 (power iteration, norms.hpp:52-77 on
    the implicit operator) of `a` against result.q, on the GPU."""
    q = result.q
    if _any_complex(a, q):
        return _zresidual_norms(a, q)
    device = _is_device(a, q)
    m, n = a.shape
    l = q.shape[1]
    if q.shape[0] != m:
        raise DimensionError("approximation_residual: shape mismatch")
    a = _dev(a) if device else _host(a)
    q = _dev(q) if device else _host(q)
    info = capi.rl_lowrank_info()
    _sync_stream_for(device)
    _raise(capi.lib().rl_approximation_residual(_ctx(), _mem(device), m, n, capi.addr(a), l, capi.addr(q),
                                                ctypes.byref(info)))
    return {"residual_frobenius": info.residual_frobenius, "residual_spectral": info.residual_spectral,
            "power_iterations": info.power_iterations}


def approximation_residual(a, result):
    """approximation_residual(a, result) (lowrank.hpp:99-102):
    ||A - Q (Q^H A)||_2 of the given A, evaluated on the GPU."""
    return residual_norms(a, result)["residual_spectral"]


# ---- the complex field (Matrix<Complex>) -------------------
# Complex arrays are numpy complex128 (host) or torch complex128 CUDA tensors
# (device); the library computes on the GPU (complex.cu).
Complex = complex


class SketchVariant(enum.IntEnum):
    """SketchVariant (lowrank.hpp:199)"""
    SRFT = 0
    CIRCULANT_PERMUTATION = 1
    Srft = 0
    CirculantPermutation = 1


def _any_complex(*arrays):
    for a in arrays:
        if a is None:
            continue
        if isinstance(a, np.ndarray):
            if np.iscomplexobj(a):
                return True
        elif hasattr(a, "is_complex"):
            if a.is_complex():
                return True
        elif isinstance(a, (list, tuple)) and any(isinstance(v, complex) for v in a):
            return True
    return False


def _zhost(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _zdev(a):
    import torch
    if not a.is_cuda:
        raise DimensionError("device arrays must be CUDA tensors")
    return a.to(torch.complex128).contiguous()


def _zempty(device, shape, ref=None):
    if device:
        import torch
        return torch.empty(shape, dtype=torch.complex128, device=ref.device if ref is not None else "cuda")
    return np.empty(shape, np.complex128)


def _zprep(device, *arrays):
    return [None if a is None else (_zdev(a) if device else _zhost(a)) for a in arrays]


def to_complex(a):
    """to_complex (matrix.hpp): the same entries with zero imaginary parts."""
    if isinstance(a, np.ndarray):
        return a.astype(np.complex128)
    import torch
    return a.to(torch.complex128)


def unit_roots(n):
    """polar(1, 2 pi k / n), k < n, rounded as the reference (glibc via std::polar)."""
    out = np.empty(n, np.complex128)
    _raise(capi.lib().rl_unit_roots(n, out.ctypes.data))
    return out


def dft_dense(n):
    """dft_dense (fft.hpp:21-30): Omega = (root[(i j) mod n]), bit-identical."""
    if n < 1:
        raise DimensionError("dft_dense: n must be positive")
    root = unit_roots(n)
    i = np.arange(n, dtype=np.int64)
    return root[np.outer(i, i) % n]


def gen_dft_input(n):
    """gen_dft_input (testbed/inputs.hpp:49-55): the transform matrix itself."""
    if n < 64 or n & (n - 1):
        raise DimensionError("gen_dft_input: need a power of two >= 64")
    return dft_dense(n)


def gen_unitary_circulant(n, seed):
    """gen_unitary_circulant (multipliers.hpp:75-82): spectrum on the unit
    circle from the reference's stream, first column inverse_fft(u) on the GPU."""
    out = np.empty(n, np.complex128)
    _raise(capi.lib().rl_gen_unitary_circulant(_ctx(), capi.RL_HOST, n, seed, out.ctypes.data))
    return CirculantMatrix(out)


def gen_unitary_toeplitz_block(n, l, seed):
    """gen_unitary_toeplitz_block (multipliers.hpp:88-90)"""
    return ToeplitzBlock(gen_unitary_circulant(n, seed), n, l)


def srft_columns(n, l, seed):
    """srft_columns (multipliers.hpp:132-138): the sorted sampled column indices."""
    out = np.empty(l, np.int64)
    _raise(capi.lib().rl_srft_columns(n, l, seed, out.ctypes.data))
    return out


def materialize_complex(spec, device=False):
    """materialize<Complex>(spec) (multipliers.hpp:174-218): every family, the
    complex ones (unitary circulant / Toeplitz, SRFT) included, on the GPU."""
    if spec.rows <= 0 or spec.cols <= 0:
        raise DimensionError("materialize: spec.rows and spec.cols must be set")
    out = _zempty(device, (spec.rows, spec.cols))
    m, keep = _multiplier(spec, device)
    _sync_stream_for(device)
    _raise(capi.lib().rl_zmaterialize(_ctx(), _mem(device), ctypes.byref(m), spec.rows, spec.cols, capi.addr(out)))
    del keep
    return out


def gen_srft(n, l, seed):
    """gen_srft (multipliers.hpp:123-130): sqrt(n/l) D Omega R, bit-identical."""
    if l < 1 or l > n:
        raise DimensionError("gen_srft: need 1 <= l <= n")
    return materialize_complex(MultiplierSpec(MultiplierKind.SRFT, seed, n, l))


def _zmatmul(a, b):
    device = _is_device(a, b)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise DimensionError("matmul: inner dimensions differ")
    a, b = _zprep(device, a, b)
    m, k = a.shape
    n = b.shape[1]
    c = _zempty(device, (m, n), a)
    _sync_stream_for(device)
    _raise(capi.lib().rl_zgemm(_ctx(), _mem(device), m, n, k, capi.addr(a), capi.addr(b), capi.addr(c)))
    return c


def _zsvd_values(a):
    device = _is_device(a)
    (a,) = _zprep(device, a)
    m, n = a.shape
    out = np.empty(min(m, n))
    _sync_stream_for(device)
    _raise(capi.lib().rl_zsingular_values(_ctx(), _mem(device), m, n, capi.addr(a),
                                          capi.addr(out) if not device else capi.addr(_out_dev(out))))
    return out if not device else _out_dev.last.cpu().numpy()


def _out_dev(out):
    import torch
    _out_dev.last = torch.empty(out.shape, dtype=torch.float64, device="cuda")
    return _out_dev.last


def _zcirculant_apply(c, x):
    device = _is_device(c, x)
    n = c.shape[0]
    if x.shape[0] != n:
        raise DimensionError("circulant_apply: length mismatch")
    c, x = _zprep(device, c, x)
    y = _zempty(device, (n,), x)
    _sync_stream_for(device)
    _raise(capi.lib().rl_zcirculant_apply(_ctx(), _mem(device), n, capi.addr(c), capi.addr(x), capi.addr(y)))
    return y


def _zcirc_right(a, c, cols):
    device = _is_device(a, c)
    m, k = a.shape
    np_ = c.shape[0]
    a, c = _zprep(device, a, c)
    out = _zempty(device, (m, cols), a)
    _sync_stream_for(device)
    _raise(capi.lib().rl_zcirculant_right_multiply(_ctx(), _mem(device), m, k, capi.addr(a), np_, capi.addr(c), cols,
                                                   capi.addr(out)))
    return out


def _zpreprocess_solve(a, b, pre_spec, post_spec, refine_steps, want_lu):
    """preprocess_solve<Complex> (preprocess.hpp:156-180) on the GPU."""
    device = _is_device(a, b)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionError("preprocess_solve: square input required")
    n = a.shape[0]
    if b.shape[0] != n:
        raise DimensionError("preprocess_solve: length mismatch")
    _check_side(pre_spec, n)
    _check_side(post_spec, n)
    if refine_steps < 0:
        raise DimensionError("preprocess_solve: negative refine_steps")
    a, b = _zprep(device, a, b)
    x = _zempty(device, (n,), b)
    lu = _zempty(device, (n, n), a) if want_lu else None
    m, keep = _multiplier(post_spec, device)
    fm, fkeep = _multiplier(pre_spec, device)
    info = capi.rl_solve_info()
    hist = (ctypes.c_double * (refine_steps + 1))()
    info.history = ctypes.cast(hist, ctypes.POINTER(ctypes.c_double))
    info.history_capacity = refine_steps + 1
    _sync_stream_for(device)
    rc = capi.lib().rl_zpreprocessed_genp_solve(_ctx(), _mem(device), n, capi.addr(a), capi.addr(b),
                                                ctypes.byref(fm), ctypes.byref(m), refine_steps, capi.addr(x),
                                                capi.addr(lu), ctypes.byref(info))
    del keep, fkeep
    _raise(rc, info.zero_pivot_step)
    d = info.as_dict()
    return SolveOutcome(x, d["residual_history"], bool(info.diverged), d, lu)


def _zrange_find(a, r, p, spec, power_steps):
    """range_find<Complex> (lowrank.hpp:62-83) with the residual of this A."""
    device = _is_device(a)
    m, n = a.shape
    l = r + p
    if r < 1 or l > min(m, n):
        raise DimensionError("range_find: rank plus oversampling exceeds matrix size")
    if power_steps < 0:
        raise DimensionError("range_find: negative power_steps")
    (a,) = _zprep(device, a)
    q = _zempty(device, (m, l), a)
    mlt, keep = _multiplier(spec, device)
    info = capi.rl_lowrank_info()
    _sync_stream_for(device)
    rc = capi.lib().rl_zrange_find_residual(_ctx(), _mem(device), m, n, capi.addr(a), l, ctypes.byref(mlt),
                                            power_steps, capi.addr(q), ctypes.byref(info))
    del keep
    _raise(rc, info.rank_deficient_column)
    d = {k: getattr(info, k) for k, _ in info._fields_ if k != "reserved"}
    return LowRankResult(q, r, p, power_steps, d)


def _zresidual_norms(a, q):
    device = _is_device(a, q)
    m, n = a.shape
    l = q.shape[1]
    if q.shape[0] != m:
        raise DimensionError("approximation_residual: shape mismatch")
    a, q = _zprep(device, a, q)
    info = capi.rl_lowrank_info()
    _sync_stream_for(device)
    _raise(capi.lib().rl_zapproximation_residual(_ctx(), _mem(device), m, n, capi.addr(a), l, capi.addr(q),
                                                 ctypes.byref(info)))
    return {"residual_frobenius": info.residual_frobenius, "residual_spectral": info.residual_spectral,
            "power_iterations": info.power_iterations}


@dataclass
class SrftCheckResult:
    """SrftCheckResult (lowrank.hpp:200-205)"""
    residual: float
    bound: float
    sketch_width: int
    clamped: bool


def srft_sketch_check(a, r, seed, variant=SketchVariant.SRFT, known_sigma_r1=None):
    """srft_sketch_check (lowrank.hpp:216-261): the sampled-transform sketch at
    its prescribed width (clamped to n), basis, ||(I - P_Y) A|| and the bound
    sqrt(1 + 7 n / l) sigma_{r+1}, on the GPU."""
    device = _is_device(a)
    a = _dev(a) if device else _host(a)
    m, n = a.shape
    if r < 1 or r > n:
        raise DimensionError("srft_sketch_check: rank out of range")
    out = capi.rl_srft_check()
    _sync_stream_for(device)
    sigma = -1.0 if known_sigma_r1 is None else float(known_sigma_r1)
    _raise(capi.lib().rl_srft_sketch_check(_ctx(), _mem(device), m, n, capi.addr(a), r, seed, int(variant), sigma,
                                           ctypes.byref(out)))
    return SrftCheckResult(out.residual, out.bound, int(out.sketch_width), bool(out.clamped))


def posterior_estimate(a, result, r_probes, seed):
    """posterior_estimate (lowrank.hpp:177-196): 10 sqrt(2/pi) max_j
    ||(A - Q Q^H A) g_j|| over r_probes Gaussian probes g_j drawn from
    RngStream(seed).derived(j + 1); the products on the GPU."""
    if r_probes < 1:
        raise DimensionError("posterior_estimate: need at least one probe")
    n = a.shape[1]
    g = np.empty((r_probes, n))
    for j in range(r_probes):
        _raise(capi.lib().rl_gen_gaussian_derived(seed, j + 1, n, g[j].ctypes.data))
    cplx = _any_complex(a, result.q)
    gt = np.ascontiguousarray(g.T).astype(np.complex128 if cplx else np.float64)
    q = result.q
    ag = matmul(a, gt if isinstance(a, np.ndarray) else _to_device_like(gt, a))
    qh = (np.ascontiguousarray(np.asarray(q).conj().T) if isinstance(q, np.ndarray) else q.conj().T.contiguous())
    proj = matmul(q, matmul(qh, ag))
    d = ag - proj
    d = d if isinstance(d, np.ndarray) else d.cpu().numpy()
    worst = float(np.sqrt((np.abs(d) ** 2).sum(axis=0)).max())
    return 10.0 * math.sqrt(2.0 / math.pi) * worst


def _to_device_like(x, ref):
    import torch
    return torch.from_numpy(x).to(ref.device)
