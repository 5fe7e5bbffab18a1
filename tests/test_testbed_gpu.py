"""GPU: the trial engine's inputs and presets (testbed/inputs.hpp:18-49,
testbed/presets.hpp:90-119, 219-243) on the device path."""
import numpy as np
import pytest

from paper_1406_5802_b200 import randla as rl
from paper_1406_5802_b200 import testbed

pytestmark = pytest.mark.gpu


def _hard_block_oracle(orc, n, seed):
    """inputs.hpp:18-49 with the oracle's Householder QR and GEMM."""
    k = n // 2
    u = orc.C.qr(orc.C.gen_gaussian(k, k, orc.C.derive_seed(seed, 1, 0)))[0]
    v = orc.C.qr(orc.C.gen_gaussian(k, k, orc.C.derive_seed(seed, 2, 0)))[0]
    u[:, k - 4:] = 0.0
    a_k = orc.C.matmul(u, np.ascontiguousarray(v.T))

    def toeplitz(s):
        d = orc.C.gen_gaussian_vector(2 * k - 1, s)
        i = np.arange(k)
        t = d[(i[:, None] + (k - 1)) - i[None, :]]
        return t / orc.C.spectral_norm_estimate(t)

    out = np.empty((n, n))
    out[:k, :k] = a_k
    out[:k, k:] = toeplitz(orc.C.derive_seed(seed, 3, 0))
    out[k:, :k] = toeplitz(orc.C.derive_seed(seed, 4, 0))
    out[k:, k:] = toeplitz(orc.C.derive_seed(seed, 5, 0))
    return out


@pytest.mark.parametrize("n", [8, 64, 256])
def test_gen_hard_block_vs_oracle(cuda, orc, n):
    a = testbed.gen_hard_block(n, 77)
    ref = _hard_block_oracle(orc, n, 77)
    assert np.abs(a - ref).max() <= 1e-12
    k = n // 2
    s = np.linalg.svd(a[:k, :k], compute_uv=False)
    assert np.all(s[-4:] < 1e-13) and np.all(np.abs(s[:-4] - 1) < 1e-12)  # exactly four zero singular values


def test_table3_and_table4_presets_pass_reference_checks(cuda, orc):
    for name in ("table3", "table4"):
        reports, checks = testbed.run_preset(name, 2024, 8, dims=[64, 128])
        assert all(c.passed for c in checks), (name, [(c.description, c.passed) for c in checks])
        assert all(r.failures == 0 for r in reports)
    # one trial against the oracle on identical inputs: refinement brings both
    # to working accuracy, the first residuals agree in magnitude
    rep, _ = testbed.run_preset("table3", 2024, 1, dims=[64])
    ts = rl.derive_seed(2024, rl.hash_label("table3/n=64"), 0)
    a = testbed.gen_hard_block(64, rl.derive_seed(ts, 1))
    b = rl.gen_gaussian_vector(64, rl.derive_seed(ts, 2))
    g = orc.C.gen_gaussian(64, 64, rl.derive_seed(ts, 3))
    ref = orc.C.preprocess_solve(a, b, 1, g, refine=1)
    dev = rep[0].column("residual_iter0").values[0], rep[0].column("residual_iter1").values[0]
    assert 0.1 < dev[0] / ref["history"][0] < 10 and dev[1] < 1e-12 and ref["history"][1] < 1e-12


def test_gepp_baseline_and_lowrank_presets_pass_reference_checks(cuda):
    """table2 (GEPP baseline), table6 / table7 (Gaussian sketch), table8 /
    table10 (real Toeplitz sketch), table13 with the reference's checks
    (presets.hpp:201-406), trials running concurrently on the worker pool"""
    for name, trials in (("table2", 8), ("table6", 100), ("table7", 100), ("table8", 100), ("table10", 100),
                         ("table13", 8)):
        reports, checks = testbed.run_preset(name, 7, trials, dims=[64])
        assert all(c.passed for c in checks), (name, [(c.description, c.passed) for c in checks])
        assert all(r.failures == 0 for r in reports), name
        assert reports[0].trials == trials


def test_concurrent_trials_equal_sequential(cuda):
    """order- and concurrency-independent reports (experiment.hpp:13-17)"""
    w = testbed.WORKERS
    try:
        testbed.WORKERS = 1
        seq, _ = testbed.run_preset("table7", 3, 12, dims=[64])
        testbed.WORKERS = 6
        par, _ = testbed.run_preset("table7", 3, 12, dims=[64])
    finally:
        testbed.WORKERS = w
    assert seq[0].column("rn2").values == par[0].column("rn2").values


def test_lowrank_bounds_vs_reference_formula(cuda, orc):
    """error_bounds_from_parts (lowrank.hpp:132-170) against numpy on the same parts"""
    inst = testbed.gen_lownumrank(64, 8, 5)
    h = rl.gen_gaussian(64, 8, 6)
    rep = testbed.error_bounds_from_parts(inst.right, inst.singulars, h, 8)
    gsv = np.linalg.svd(inst.right.T @ h, compute_uv=False)
    dp = np.sqrt(2) * np.linalg.norm(h) / gsv[-1] * inst.singulars[8] / inst.singulars[7]
    assert rep.delta_plus == pytest.approx(dp, rel=1e-10)
    assert rep.delta_plus_prime == pytest.approx(inst.singulars[8] + 2 * dp * inst.singulars[0], rel=1e-10)
    # the instance: sigma_j = 1/(j+1) up to r, 1e-10 beyond, between orthonormal factors
    s = np.linalg.svd(inst.a, compute_uv=False)
    assert np.allclose(s[:8], 1.0 / np.arange(1, 9), rtol=1e-12) and np.allclose(s[8:], 1e-10, rtol=1e-4)


def test_complex_presets_pass_reference_checks(cuda):
    """the complex-field presets (presets.hpp:244-342, 408-457): table5 (unitary
    circulant multipliers on to_complex of the hard-block inputs), table5a (the
    DFT matrix with a Gaussian rescue), table9 / table11 (unitary Toeplitz
    sketch), table14 (SRFT / circulant-permutation sketch checks), and table12
    (the a-posteriori estimator), with the reference's checks"""
    for name, trials, dims in (("table5", 8, [64]), ("table5a", 16, [256]), ("table9", 100, [64]),
                               ("table11", 100, [64]), ("table12", 100, [64]), ("table14", 8, [64])):
        reports, checks = testbed.run_preset(name, 11, trials, dims=dims)
        assert checks and all(c.passed for c in checks), (name, [(c.description, c.passed) for c in checks])
        assert all(r.failures == 0 for r in reports), name


def test_posterior_probes_match_reference_stream(orc):
    """posterior_estimate's probes: RngStream(seed).derived(j + 1).next_gaussian (lowrank.hpp:183-186)"""
    if orc.REF is None:
        pytest.skip("oracle/_ref not built")
    g = np.empty(33)
    rl.capi.lib().rl_gen_gaussian_derived(12345, 3, 33, g.ctypes.data)
    np.testing.assert_array_equal(g, orc.REF.gaussian_derived(12345, 3, 33))
