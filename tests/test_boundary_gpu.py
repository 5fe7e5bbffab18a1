"""GPU parity of the drop-in boundary beyond the headline path, against the
REFERENCE ITSELF (oracle/_ref, the reference's own headers):

  fft / inverse_fft                fft.hpp:76-98 (radix, Stockham and dense lengths)
  RealCirculant, circulant_apply   circulant.hpp:17-98
  materialize(spec), every real family   multipliers.hpp:174-218
  preprocess_solve with left and right multipliers of every real family,
  long refinement histories        preprocess.hpp:27-180
  range_find with every real sketch family and power steps   lowrank.hpp:51-81
  approximation_residual(a, result) evaluated on the A it is given   lowrank.hpp:99-102
  the complex families raise DimensionError, as the reference's real pipeline
"""
import ctypes

import numpy as np
import pytest

import paper_1406_5802_b200 as rl
from paper_1406_5802_b200 import capi

pytestmark = pytest.mark.gpu
K = rl.MultiplierKind


def crand(n, seed):
    g = rl.gen_gaussian(n, 2, seed)
    return g[:, 0] + 1j * g[:, 1]


@pytest.mark.parametrize("n", [1, 2, 6, 8, 12, 100, 1024, 8192, 16384, 65536])
def test_fft_and_inverse_vs_reference(cuda, orc, n):
    v = crand(n, 100 + n)
    f = rl.fft(v)
    ref = orc.REF.fft(v)
    bar = 1e-12 * n * np.linalg.norm(v)  # the reference's own FFT bar (tests/test_transforms.cpp:67-74)
    assert np.abs(f - ref).max() <= bar, (n, np.abs(f - ref).max())
    back = rl.inverse_fft(f)
    assert np.abs(back - v).max() <= bar
    assert np.abs(back - orc.REF.fft(ref, inverse=True)).max() <= bar
    if n <= 1024:  # batches along the last axis, and device tensors
        import torch
        vb = np.stack([v, 2 * v, crand(n, 7)])
        fb = rl.fft(torch.from_numpy(vb).cuda()).cpu().numpy()
        for i in range(3):
            assert np.abs(fb[i] - orc.REF.fft(vb[i])).max() <= bar * 3


def test_fft_kats(cuda):
    """tests/test_transforms.cpp:57-65: e1 -> all ones; (1, 1) -> (2, 0)"""
    e1 = np.zeros(8, complex)
    e1[0] = 1
    assert np.abs(rl.fft(e1) - 1).max() <= 1e-14
    two = rl.fft(np.array([1, 1], complex))
    assert abs(two[0] - 2) <= 1e-14 and abs(two[1]) <= 1e-14


@pytest.mark.parametrize("n", [2, 5, 6, 64, 1000, 8192])
def test_circulant_type_and_apply_vs_reference(cuda, orc, n):
    c = rl.gen_real_circulant(n, 40 + n)
    col = c.first_column()
    assert np.array_equal(col, orc.REF.gen_real_circulant_column(n, 40 + n))
    spec = c.spectrum()
    assert np.abs(spec - orc.REF.fft(col)).max() <= 1e-12 * n * np.linalg.norm(col)
    x = rl.gen_gaussian_vector(n, 3)
    y = rl.circulant_apply(c, x)
    yr, st = orc.REF.circulant_apply(col, x)
    assert st == 0
    assert np.linalg.norm(y - yr) <= 1e-12 * np.linalg.norm(yr)
    if n <= 1000:
        assert np.array_equal(c.dense(), orc.REF.materialize(int(K.REAL_CIRCULANT), n, n, 40 + n)[0])
        ct = c.transposed().first_column()
        assert np.array_equal(ct, col[(n - np.arange(n)) % n])


MATERIALIZE_CASES = [
    (K.GAUSSIAN, 0, 33, 17, "exact"),
    (K.FINITE_SET_UNIFORM, 0, 40, 9, "exact"),
    (K.REAL_CIRCULANT, 0, 24, 24, "exact"),
    (K.TOEPLITZ_BLOCK, 0, 30, 7, "exact"),
    (K.CIRC_SKEW_PRODUCT, 0, 48, 48, "gemm"),
    (K.NONE, 0, 9, 9, "exact"),
]


@pytest.mark.parametrize("kind,variant,rows,cols,how", MATERIALIZE_CASES, ids=lambda v: str(v))
def test_materialize_every_real_family_vs_reference(cuda, orc, kind, variant, rows, cols, how):
    spec = rl.MultiplierSpec(kind, 77, rows, cols, variant=rl.ToeplitzVariant(variant))
    got = rl.materialize(spec)
    ref, st = orc.REF.materialize(int(kind), rows, cols, 77, variant)
    assert st == 0
    if how == "exact":
        assert np.array_equal(got, ref)
    else:  # a product of two expansions: the GEMM bar (tests/test_field_core.cpp:52-58)
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max() * rows


@pytest.mark.parametrize("kind,variant", [(K.UNITARY_CIRCULANT, 0), (K.SRFT, 0), (K.TOEPLITZ_BLOCK, 1)])
def test_complex_families_raise_dimension_error(cuda, orc, kind, variant):
    """multipliers.hpp:178-180, preprocess.hpp:53: the real pipeline throws DimensionError"""
    a = rl.gen_gaussian(16, 16, 1)
    b = rl.gen_gaussian_vector(16, 2)
    spec = rl.MultiplierSpec(kind, 5, variant=rl.ToeplitzVariant(variant))
    for pre, post in ((None, spec), (spec, None)):
        with pytest.raises(rl.DimensionError, match="complex multiplier family"):
            rl.preprocess_solve(a, b, pre, post, 0)
        assert orc.REF.preprocess_solve_spec(a, b, pre=(int(kind), variant, 5) if pre else (0, 0, 0),
                                             post=(int(kind), variant, 5) if post else (0, 0, 0))["status"] == 1
    with pytest.raises(rl.DimensionError):
        rl.range_find(rl.gen_gaussian(32, 16, 3), 4, 0, spec)


SOLVE_CASES = [  # (pre (kind, variant, seed), post (kind, variant, seed))
    ((K.NONE, 0, 0), (K.GAUSSIAN, 0, 11)),
    ((K.GAUSSIAN, 0, 12), (K.NONE, 0, 0)),
    ((K.GAUSSIAN, 0, 13), (K.GAUSSIAN, 0, 14)),
    ((K.REAL_CIRCULANT, 0, 15), (K.GAUSSIAN, 0, 16)),
    ((K.TOEPLITZ_BLOCK, 0, 17), (K.NONE, 0, 0)),
    ((K.NONE, 0, 0), (K.TOEPLITZ_BLOCK, 0, 18)),
    ((K.NONE, 0, 0), (K.FINITE_SET_UNIFORM, 0, 19)),
    ((K.NONE, 0, 0), (K.CIRC_SKEW_PRODUCT, 0, 20)),
    ((K.FINITE_SET_UNIFORM, 0, 21), (K.REAL_CIRCULANT, 0, 22)),
]


@pytest.mark.parametrize("n", [64, 256])
@pytest.mark.parametrize("pre,post", SOLVE_CASES, ids=lambda v: f"{v[0].name}")
def test_preprocess_solve_two_sided_vs_reference(cuda, orc, n, pre, post):
    a = rl.gen_gaussian(n, n, 1000 + n)
    b = rl.gen_gaussian_vector(n, 3)
    ref = orc.REF.preprocess_solve_spec(a, b, pre=tuple(map(int, pre)), post=tuple(map(int, post)), refine=1)
    mk = lambda s: rl.MultiplierSpec(s[0], s[2], variant=rl.ToeplitzVariant(s[1]))  # noqa: E731
    if ref["status"] == 2:
        with pytest.raises(rl.ZeroPivotError) as e:
            rl.preprocess_solve(a, b, mk(pre), mk(post), 1)
        assert e.value.step == ref["zero_step"]
        return
    assert ref["status"] == 0
    out = rl.preprocess_solve(a, b, mk(pre), mk(post), 1)
    kappa = np.linalg.cond(a)
    assert np.linalg.norm(out.x - ref["x"]) <= 1e-10 * kappa * np.linalg.norm(ref["x"])
    assert len(out.residual_history) == 2
    assert out.residual_history[1] <= max(10 * ref["history"][1], 1e-14)


def test_long_refinement_history_vs_reference(cuda, orc):
    """refine_steps > 7: the whole refine + 1 history (preprocess.hpp:124-140)"""
    n = 128
    a = rl.gen_gaussian(n, n, 5)
    b = rl.gen_gaussian_vector(n, 6)
    ref = orc.REF.preprocess_solve_spec(a, b, post=(int(K.GAUSSIAN), 0, 7), refine=11)
    out = rl.preprocess_solve(a, b, None, rl.MultiplierSpec(K.GAUSSIAN, 7), 11)
    h = [v for v in ref["history"] if not np.isnan(v)]
    assert len(out.residual_history) == len(h)
    assert out.diverged == ref["diverged"]
    assert out.residual_history[0] <= 10 * h[0]
    # through the raw ABI without a history buffer: refused, never truncated
    info = capi.rl_solve_info()
    m = capi.rl_multiplier(kind=int(K.GAUSSIAN), seed=7)
    x = np.empty(n)
    rc = capi.lib().rl_preprocessed_genp_solve(None, capi.RL_HOST, n, a.ctypes.data, b.ctypes.data, None,
                                               ctypes.byref(m), 8, x.ctypes.data, None, 0, ctypes.byref(info))
    assert rc == capi.RL_ERR_INVALID_ARGUMENT


SKETCH_CASES = [
    (K.GAUSSIAN, 0, 0),
    (K.GAUSSIAN, 0, 2),
    (K.TOEPLITZ_BLOCK, 0, 0),
    (K.TOEPLITZ_BLOCK, 0, 1),
    (K.GAUSSIAN_CIRCULANT, 0, 0),
    (K.FINITE_SET_UNIFORM, 0, 0),
]


@pytest.mark.parametrize("kind,variant,power", SKETCH_CASES, ids=lambda v: str(v))
def test_range_find_families_and_power_steps_vs_reference(cuda, orc, kind, variant, power):
    m, n, l = 300, 256, 12
    u = orc.C.gen_gaussian(m, l, 1)
    v = orc.C.gen_gaussian(n, l, 2)
    # power steps raise the spectrum to the power 2s+1 (lowrank.hpp:51-57): keep
    # the sketch numerically full rank for both QRs
    a = (u * np.logspace(0, -1 if power else -3, l)) @ v.T + 1e-9 * orc.C.gen_gaussian(m, n, 3)
    spec = rl.MultiplierSpec(kind, 31, variant=rl.ToeplitzVariant(variant))
    res = rl.range_find(a, l, 0, spec, power)
    if kind == K.GAUSSIAN_CIRCULANT:  # the extension: the Toeplitz block of the Gaussian-column parent
        y, st = orc.REF.matmul_by_toeplitz_block(a, orc.C.gen_gaussian(n, 1, 31).reshape(n), l)
    else:
        y, st = orc.REF.range_sketch(a, l, int(kind), 31, variant, power)
    assert st == 0
    qo, _, qst, _ = orc.C.qr(y)  # the restated Householder QR with qr.hpp:33-45's phases
    assert qst == 0
    kap = np.linalg.cond(y)
    assert np.abs(res.q - qo).max() <= 1e-13 * kap * np.sqrt(m), np.abs(res.q - qo).max()
    # the residual of the A it is handed (lowrank.hpp:99-102), not a cached one:
    # ||A - Q Q^T A||_2 for the returned Q, and the reference's Q gives the same
    # value to the Q agreement above
    q = res.q
    r_mine = np.linalg.norm(a - q @ (q.T @ a), 2)
    assert abs(rl.approximation_residual(a, res) - r_mine) <= 1e-6 * r_mine + 1e-14
    r2 = np.linalg.norm(2 * a - q @ (q.T @ (2 * a)), 2)
    assert abs(rl.approximation_residual(2 * a, res) - r2) <= 1e-6 * r2 + 1e-14
    r_ref = np.linalg.norm(a - qo @ (qo.T @ a), 2)
    assert abs(r_mine - r_ref) <= 2 * np.abs(res.q - qo).max() * np.sqrt(m * l) * np.linalg.norm(a, 2) + 1e-14


def test_context_follows_current_device(cuda):
    """the per-thread default context is the one for cudaGetDevice()"""
    assert capi.lib().rl_context_device(None) == cuda.cuda.current_device()
