"""GPU parity: CholeskyQR2 orthonormal basis (qr.hpp:21-54) and the range
finder + residual (lowrank.hpp:62-102) vs the oracle, including the
reference's own low-rank test cases (tests/test_lowrank.cpp:20-52)."""
import numpy as np
import pytest

import paper_1406_5802_b200 as rl

pytestmark = pytest.mark.gpu


def _lownumrank(n, r, seed, tail=1e-10):
    """testbed/inputs.hpp:67-83 pattern: Q(Gaussian) diag(1/j, tail) Q(Gaussian)^T"""
    rng = np.random.default_rng(seed)
    s, _ = np.linalg.qr(rng.standard_normal((n, n)))
    t, _ = np.linalg.qr(rng.standard_normal((n, n)))
    sig = np.array([1.0 / (j + 1) if j < r else tail for j in range(n)])
    return (s * sig) @ t.T, sig


def test_qr_matches_oracle_householder(cuda, orc):
    for m, l in [(64, 8), (200, 30), (1000, 64), (4096, 256), (37, 37)]:
        y = orc.C.gen_gaussian(m, l, m + l)
        q, r = rl.qr(y)
        qo, ro, st, _ = orc.C.qr(y)
        assert st == 0
        kap = np.linalg.cond(y)
        assert np.abs(q - qo).max() <= 1e-13 * kap * np.sqrt(m), np.abs(q - qo).max()
        assert np.abs(r - ro).max() <= 1e-12 * kap * np.abs(ro).max()
        assert np.linalg.norm(q.T @ q - np.eye(l)) <= 1e-10 * max(m, l)  # tol_orth (types.hpp:39)
        assert (np.diag(r) > 0).all()


def test_qr_kat_and_rank_deficiency(cuda, orc):
    """tests/test_field_core.cpp:80-86: QR of (3,4)^T; duplicated column ->
    RankDeficiencyError at that column (qr.hpp:37-38)."""
    q, r = rl.qr(np.array([[3.0], [4.0]]))
    np.testing.assert_allclose(q[:, 0], [0.6, 0.8], atol=1e-15)
    assert abs(r[0, 0] - 5.0) < 1e-14
    y = orc.C.gen_gaussian(300, 20, 3)
    y[:, 11] = y[:, 4]
    _, _, st, bad = orc.C.qr(y)
    assert st == 4
    with pytest.raises(rl.RankDeficiencyError) as e:
        rl.qr(y)
    assert e.value.column == bad == 12


def test_range_finder_exact_low_rank(cuda, orc):
    """tests/test_lowrank.cpp:20-29"""
    n, r = 24, 5
    a, sig = _lownumrank(n, r, 11, tail=0.0)
    res = rl.range_find(a, r, 0, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 12))
    assert res.sketch_width() == r
    assert rl.approximation_residual(a, res) <= 1e-10 * np.linalg.norm(a, 2)
    assert np.linalg.norm(res.q.T @ res.q - np.eye(r)) <= 1e-10 * n


def test_axis_aligned_residual(cuda):
    """tests/test_lowrank.cpp:31-39: residual == the dropped singular value"""
    a = np.diag([1.0, 1e-10])
    h = np.array([[1.0], [0.0]])
    res = rl.range_find(a, 1, 0, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 0, dense=h))
    assert abs(rl.approximation_residual(a, res) - 1e-10) <= 1e-12 * 1e-10
    assert abs(res.info["residual_frobenius"] - 1e-10) <= 1e-12 * 1e-10


def test_mean_residual_known_rank_ensemble(cuda):
    """tests/test_lowrank.cpp:41-52 analogue (20 trials, n=64, r=8)"""
    tot = 0.0
    for t in range(20):
        a, _ = _lownumrank(64, 8, 1000 + t)
        res = rl.range_find(a, 8, 0, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, rl.derive_seed(22, t)))
        tot += rl.approximation_residual(a, res)
    assert tot / 20 <= 1e-6


@pytest.mark.parametrize("kind", ["gaussian", "toeplitz"])
def test_range_find_residual_vs_oracle(cuda, orc, kind):
    """Y, Q and the residual norms against the reference on the same inputs:
    the sketch by the reference's own code, Q by the restated Householder QR
    with qr.hpp:33-45's phases, ||R||_F of the explicit residual, and ||R||_2
    by the reference's own spectral_norm_estimate (norms.hpp:35-78) run on the
    explicit residual -- the device runs the same power iteration (start
    vector, stopping rule) on the implicit operator. Bars: the north star's
    1e-9 relative for both norms (measured agreement ~1e-12 .. 1e-10, see
    DESIGN.md §2)."""
    m = n = 1024
    r = 32
    u = orc.C.gen_gaussian(m, r, 61)
    v = orc.C.gen_gaussian(n, r, 62)
    u, _ = np.linalg.qr(u)
    v, _ = np.linalg.qr(v)
    a = (u * np.logspace(0, -2, r)) @ v.T + 1e-10 * orc.C.gen_gaussian(m, n, 63)
    if kind == "gaussian":
        spec = rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 77)
        y_ref, st = orc.REF.range_sketch(a, r, int(rl.MultiplierKind.GAUSSIAN), 77)
    else:
        spec = rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN_CIRCULANT, 21)
        y_ref, st = orc.REF.matmul_by_toeplitz_block(a, orc.C.gen_gaussian_vector(n, 21), r)
    assert st == 0
    res = rl.range_find(a, r, 0, spec)
    q_ref, _, st, _ = orc.C.qr(y_ref)
    assert st == 0
    kap = np.linalg.cond(y_ref)
    assert np.abs(res.q - q_ref).max() <= 1e-13 * kap * np.sqrt(m)
    resid_ref = a - q_ref @ (q_ref.T @ a)
    fro_ref = np.linalg.norm(resid_ref)
    est_ref = orc.REF.spectral_norm_estimate(resid_ref)
    e_fro = abs(res.info["residual_frobenius"] / fro_ref - 1)
    e_spec = abs(res.info["residual_spectral"] / est_ref - 1)
    print(kind, "fro", e_fro, "spec vs reference estimate", e_spec, "its", res.info["power_iterations"])
    assert e_fro <= 1e-9
    assert e_spec <= 1e-9


@pytest.mark.parametrize("m,n,r", [(1000, 998, 17), (2050, 4100, 40), (3001, 640, 64), (513, 9000, 8)])
def test_power_iteration_one_pass_shapes(cuda, m, n, r):
    """||A - Q Q^T A||_2 by the one-pass power step (a cluster of CTAs per row
    range, rows not a multiple of the exchange size, columns ragged against the
    cluster's column split): a lower bound of sigma_1 that converges to it."""
    rng = np.random.default_rng(m + n + r)
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    a = (u * np.logspace(0, -3, r)) @ v.T + 1e-6 * rng.standard_normal((m, n))
    res = rl.range_find(a, r, 0, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 5))
    resid = a - res.q @ (res.q.T @ a)
    s1 = np.linalg.norm(resid, 2)
    est = res.info["residual_spectral"]
    assert est <= s1 * (1 + 1e-12)
    assert abs(est / s1 - 1) <= 1e-3, (est, s1, res.info["power_iterations"])
    assert abs(res.info["residual_frobenius"] / np.linalg.norm(resid) - 1) <= 1e-6
