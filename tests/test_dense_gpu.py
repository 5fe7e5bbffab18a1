"""GPU parity: dense preprocessed GENP (BASELINE config 1 and the headline
path) through the C ABI vs the CPU oracle on identical seeded inputs.

Tolerances (BASELINE north_star): LU and x within relative Frobenius error
1e-10 * kappa of the factored product (for LU: of its worst leading minor,
the quantity GENP's sensitivity follows); verdicts identical; growth to
rounding."""
import numpy as np
import pytest

import paper_1406_5802_b200 as rl

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_genp_kats(cuda):
    """tests/test_elimination.cpp:29-50"""
    f = rl.genp_factor(np.eye(3))
    np.testing.assert_array_equal(f.lower, np.eye(3))
    np.testing.assert_array_equal(f.upper, np.eye(3))
    assert f.perm is None
    with pytest.raises(rl.ZeroPivotError) as e:
        rl.genp_factor(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert e.value.step == 1
    f = rl.genp_factor(np.array([[2.0, 1.0], [4.0, 5.0]]))
    assert f.lower[1, 0] == 2.0 and f.upper[0, 0] == 2.0 and f.upper[0, 1] == 1.0 and f.upper[1, 1] == 3.0
    assert f.lower[0, 1] == 0.0


def test_genp_bit_identical_under_contention(cuda):
    """The blocked factorisation's streams (lookahead chain, in-place U12
    GEMMs, the second-half panel's T handoff, the forward-substitution stream)
    must not race: repeated factorisations and solves of the same matrix,
    each while other kernels load the SMs from another stream, are
    bit-identical. (A 64-row tile configuration of the in-place U12 once let a
    late-scheduled second tile row read rows the first had already
    overwritten, only under contention.)"""
    torch = cuda
    n = 2048  # every super-panel's U12 is a small product here
    a = rl.gen_gaussian(n, n, 11)
    g = rl.gen_gaussian(n, n, 12)
    b = rl.gen_gaussian_vector(n, 13)
    da, dg, db = (torch.from_numpy(v).cuda() for v in (a, g, b))
    hog = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
    side = torch.cuda.Stream()
    outs = []
    for rep in range(6):
        with torch.cuda.stream(side):
            for _ in range(rep % 3):
                hog = (hog @ hog) * (1.0 / 4096)
        out = rl.preprocess_solve(da, db, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 0, dense=dg), 0,
                                  want_lu=True)
        torch.cuda.synchronize()
        outs.append((out.x.cpu().numpy().copy(), out.lu.cpu().numpy().copy()))
    for x, lu in outs[1:]:
        assert np.array_equal(x, outs[0][0])
        assert np.array_equal(lu, outs[0][1])


@pytest.mark.parametrize("n", [1, 2, 3, 5, 64, 65, 127, 128, 129, 200, 511, 1024])
def test_genp_factor_vs_oracle(cuda, orc, n):
    a = orc.C.gen_gaussian(n, n, 100 + n)
    g = orc.C.gen_gaussian(n, n, 200 + n)
    p = orc.C.matmul(a, g)  # preprocessed product keeps the leading minors healthy
    lu_ref, zs, _ = orc.C.genp_factor(p)
    assert zs == 0
    f = rl.genp_factor(p)
    kmin = max(np.linalg.cond(p[:k, :k]) for k in range(1, n + 1, max(1, n // 32)))
    assert _rel(f.packed, lu_ref) <= 1e-10 * kmin
    b = orc.C.gen_gaussian_vector(n, 7)
    x = rl.lu_solve(f, b)
    xr = orc.C.lu_solve(lu_ref, b)
    assert _rel(x, xr) <= 1e-10 * np.linalg.cond(p)


def test_spectral_norm_estimate_bit_exact(cuda, orc):
    """exact-order device power iteration == the reference's, bit for bit"""
    rng = np.random.default_rng(11)
    for shape in [(1, 1), (7, 3), (64, 64), (300, 200), (1024, 1024)]:
        a = rng.standard_normal(shape)
        assert rl.spectral_norm_estimate(a) == orc.C.spectral_norm_estimate(a)
    assert rl.spectral_norm_estimate(np.zeros((4, 4))) == 0.0


@pytest.mark.parametrize("refine", [0, 1])
def test_config1_parity(cuda, orc, golden, refine):
    """BASELINE config 1: n=1024, A seed 1, G seed 2, b seed 3."""
    n = 1024
    a = rl.gen_gaussian(n, n, 1)
    b = rl.gen_gaussian_vector(n, 3)
    out = rl.preprocess_solve(a, b, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 2), refine, want_lu=True,
                              want_norm_a=True)
    ref = orc.C.preprocess_solve(a, b, 1, orc.C.gen_gaussian(n, n, 2), refine=refine, want_lu=True)
    kap = np.linalg.cond(ref["product"])
    assert _rel(out.x, ref["x"]) <= 1e-10 * kap
    assert _rel(out.x, golden[f"cfg1_x_refine{refine}"]) <= 1e-10 * kap
    assert len(out.residual_history) == refine + 1 and not out.diverged
    # growth: max|U| / max|AG| within rounding of the reference's
    assert abs(out.info["growth"] / golden["cfg1_growth"][0] - 1) <= 1e-10 * kap
    assert out.info["zero_pivot_step"] == 0 and out.info["norm_estimate_evaluated"] == 0
    # pivots, reference ordering
    np.testing.assert_allclose(np.diag(out.lu), golden["cfg1_pivots"], rtol=1e-10 * kap)
    # residual level matches the reference's ||Ax-b||/||b||
    assert out.residual_history[0] < 10 * golden[f"cfg1_hist_refine{refine}"][0] + 1e-15
    if refine:
        assert out.residual_history[1] < 1e-3 * out.residual_history[0]
    assert 0 < out.info["residual_rel_a"] < 1e-6


def test_identity_solve_exact(cuda, orc):
    """tests/test_elimination.cpp:244-253: preprocessed solve exact on I"""
    b = orc.C.gen_gaussian_vector(8, 60)
    out = rl.preprocess_solve(np.eye(8), b, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 61), 0)
    assert len(out.residual_history) == 1 and out.residual_history[0] <= 1e-13
    np.testing.assert_allclose(out.x, b, rtol=1e-12, atol=1e-12)


def test_zero_pivot_verdicts_match_oracle(cuda, orc):
    """ZeroPivot propagates with the reference's 1-based step, including the
    ambiguous band that needs the exact estimate."""
    n = 96
    cases = []
    a = np.eye(n)
    a[0, 0] = 0.0
    cases.append(a)                       # step 1
    a = np.eye(n)
    a[70, 70] = 0.0
    cases.append(a)                       # step 71 (second base panel)
    for piv in (5e-11, 9.6e-12, 5e-12):   # tol_pivot(96) * est(=1) = 9.6e-12; ||I||_F bound = 9.4e-11
        a = np.eye(n)
        a[40, 40] = piv
        cases.append(a)
    for a in cases:
        _, zs, _ = orc.C.genp_factor(a)
        if zs:
            with pytest.raises(rl.ZeroPivotError) as e:
                rl.genp_factor(a)
            assert e.value.step == zs
            with pytest.raises(rl.ZeroPivotError) as e:
                rl.preprocess_solve(a, np.ones(n), None, None, 0)
            assert e.value.step == zs
        else:
            f = rl.genp_factor(a)
            assert f.info["norm_estimate_evaluated"] == 1


def test_retry_wrapper(cuda, orc):
    """preprocess.hpp:182-196: identity multipliers keep failing; a Gaussian
    multiplier rescues the anti-identity immediately."""
    n = 64
    a = np.eye(n)[::-1].copy()
    b = orc.C.gen_gaussian_vector(n, 991)
    with pytest.raises(rl.ZeroPivotError):
        rl.preprocess_solve_with_retry(a, b, None, None, 0, 2)
    out = rl.preprocess_solve_with_retry(a, b, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 992), 0, 3)
    assert out.residual_history[0] <= 1e-3


def test_device_pointer_path_matches_host(cuda, orc):
    torch = cuda
    n = 512
    a = rl.gen_gaussian(n, n, 21)
    b = rl.gen_gaussian_vector(n, 22)
    g = rl.gen_gaussian(n, n, 23)
    h = rl.preprocess_solve(a, b, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 23), 0)
    d = rl.preprocess_solve(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), None,
                            rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 0, dense=torch.from_numpy(g).cuda()), 0)
    np.testing.assert_array_equal(h.x, d.x.cpu().numpy())


@pytest.mark.parametrize("n,family", [(64, "uniform"), (256, "uniform"), (1024, "gaussian"), (300, "uniform")])
def test_circulant_preprocessed_solve_vs_oracle(cuda, orc, n, family):
    """preprocess_solve with a circulant post-multiplier (preprocess.hpp:36-49,
    :65-73, :91): product by FFT (power-of-two n) or dense expansion (n=300),
    GENP, x = C y by FFT, one refinement step."""
    if family == "uniform":
        spec = rl.MultiplierSpec(rl.MultiplierKind.REAL_CIRCULANT, 13)
        c = orc.C.gen_real_circulant_column(n, 13)
    else:  # BASELINE config 3 recipe: Haar U, V, log-spaced sigma (kappa = 1e4), Gaussian column
        spec = rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN_CIRCULANT, 13)
        c = orc.C.gen_gaussian_vector(n, 13)
    if family == "gaussian":
        u, _ = np.linalg.qr(orc.C.gen_gaussian(n, n, 11))
        v, _ = np.linalg.qr(orc.C.gen_gaussian(n, n, 12))
        a = (u * np.logspace(0, -4, n)) @ v.T
    else:
        a = orc.C.gen_gaussian(n, n, 5)
    b = orc.C.gen_gaussian_vector(n, 14)
    out = rl.preprocess_solve(a, b, None, spec, 1, want_lu=True)
    ref = orc.C.preprocess_solve(a, b, 2, c, refine=1, want_lu=True)
    assert ref["status"] == 0
    kap = np.linalg.cond(ref["product"])
    assert _rel(out.x, ref["x"]) <= 1e-10 * kap
    assert len(out.residual_history) == 2
    assert out.residual_history[1] <= max(10 * ref["history"][1], 1e-14)
    if family == "uniform" and n == 256:
        # the reference's own family through the reference's own headers
        if orc.REF is not None:
            r2 = orc.REF.preprocess_solve(a, b, 2, 13, refine=1)
            assert _rel(out.x, r2["x"]) <= 1e-10 * kap


def test_config3_full_size_device(cuda, orc):
    """BASELINE config 3 at n=8192 (A = U diag(sigma) V^T, kappa = 1e4, Haar U/V
    from QR of N(0,1) matrices, seeds 11/12; Gaussian circulant seed 13, b seed 14):
    device run checked through size-independent properties and a sampled
    product row against the oracle."""
    torch = cuda
    n = 8192
    gu = torch.from_numpy(rl.gen_gaussian(n, n, 11)).cuda()
    u, _ = torch.linalg.qr(gu)
    del gu
    gv = torch.from_numpy(rl.gen_gaussian(n, n, 12)).cuda()
    v, _ = torch.linalg.qr(gv)
    del gv
    sig = torch.logspace(0, -4, n, dtype=torch.float64, device="cuda")
    a = (u * sig) @ v.T
    del u, v
    b = torch.from_numpy(rl.gen_gaussian_vector(n, 14)).cuda()
    out = rl.preprocess_solve(a, b, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN_CIRCULANT, 13), 1)
    torch.cuda.synchronize()
    assert out.info["zero_pivot_step"] == 0
    assert out.residual_history[1] < 1e-12, out.residual_history
    r = (a @ out.x - b).norm().item() / b.norm().item()
    assert abs(r - out.residual_history[1]) <= 0.5 * out.residual_history[1] + 1e-16
    # product rows against the oracle's FFT product
    c = orc.C.gen_gaussian_vector(n, 13)
    rows = [0, 4097, 8191]
    ref, st = orc.C.matmul_by_circulant(a[rows].cpu().numpy(), c)
    got = rl.matmul_by_circulant(a[rows].contiguous(), torch.from_numpy(c).cuda()).cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max()


@pytest.mark.parametrize("n,ks", [(1024, (256, 512, 768)), (700, (256, 512))])
def test_schur_blocks_vs_reference_block_ge(cuda, orc, n, ks):
    """SURVEY §8(a) a27 / config 3's block size 256: the trailing factors of the
    device's blocked GENP give the Schur complement of every leading k x k block,
    which is elimination-path independent; it must match the reference's own
    schur_complement (block_ge.hpp:202-218, GEPP on the pivot block), the
    quantity block_ge_factor's Schur children hold (tests/test_elimination.cpp:
    141-153, tests/acceptance.cpp:246-259)."""
    if orc.REF is None:
        pytest.skip("reference build (oracle/_ref) not present")
    a = orc.C.gen_gaussian(n, n, 1)
    g = orc.C.gen_gaussian(n, n, 2)
    p = orc.C.matmul(a, g)
    f = rl.genp_factor(p)
    for k in ks:
        s_dev = f.lower[k:, k:] @ f.upper[k:, k:]
        s_ref = orc.REF.schur_complement(p, k)
        kb = np.linalg.cond(p[:k, :k])
        assert _rel(s_dev, s_ref) <= 1e-10 * kb, (k, _rel(s_dev, s_ref), kb)


def test_headline_full_size_properties(cuda):
    """The headline workload at full size (n = 8192, config-1 recipe) through the
    C ABI: the host-buffer call with the multiplier drawn from its seed (device
    generator) returns the same bits as the device-resident call with the
    host-generated G; the pivot verdict needs no exact estimate; the solution's
    residual ||Ax - b|| / (||A||_F ||x||) and the growth factor agree with
    torch fp64 recomputations from the returned factors."""
    torch = cuda
    n = 8192
    a = rl.gen_gaussian(n, n, 1)
    b = rl.gen_gaussian_vector(n, 3)
    g = rl.gen_gaussian(n, n, 2)
    host = rl.preprocess_solve(a, b, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 2), 0)
    da, db, dg = (torch.from_numpy(t).cuda() for t in (a, b, g))
    dev = rl.preprocess_solve(da, db, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 0, dense=dg), 0, want_lu=True)
    torch.cuda.synchronize()
    x = dev.x
    np.testing.assert_array_equal(host.x, x.cpu().numpy())
    assert dev.info["zero_pivot_step"] == 0 and dev.info["norm_estimate_evaluated"] == 0
    # GENP's backward error follows its growth (~2e5 here): ||Ax-b|| / (||A||_F ||x||)
    # ~ 1e-9, within the n * growth * eps bound; one refinement step (the
    # paper's recipe, preprocess.hpp:115-143) recovers working accuracy
    r = torch.linalg.vector_norm(da @ x - db) / (torch.linalg.matrix_norm(da) * torch.linalg.vector_norm(x))
    assert r.item() < n * dev.info["growth"] * 2.2e-16, r.item()
    ref1 = rl.preprocess_solve(da, db, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 0, dense=dg), 1)
    assert ref1.residual_history[1] < 1e-3 * ref1.residual_history[0], ref1.residual_history
    p = da @ dg
    umax = torch.triu(dev.lu).abs().max()
    growth = (umax / p.abs().max()).item()
    assert abs(growth / dev.info["growth"] - 1) < 1e-12, (growth, dev.info["growth"])


@pytest.mark.parametrize("n", [1031, 2050])
def test_host_chunked_upload_odd_sizes(cuda, orc, n):
    """Host-buffer calls upload A in row blocks under the product (n >= 1024);
    odd n (padded leading dimension) and uneven blocks must give the same x as
    the device-resident call, and match the oracle within tolerance."""
    torch = cuda
    a = orc.C.gen_gaussian(n, n, 31)
    b = orc.C.gen_gaussian_vector(n, 32)
    g = orc.C.gen_gaussian(n, n, 33)
    h = rl.preprocess_solve(a, b, None, rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 33), 0)
    d = rl.preprocess_solve(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), None,
                            rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 0, dense=torch.from_numpy(g).cuda()), 0)
    np.testing.assert_array_equal(h.x, d.x.cpu().numpy())
    if n <= 1100:
        ref = orc.C.preprocess_solve(a, b, 1, g, refine=0, want_lu=True)
        assert _rel(h.x, ref["x"]) <= 1e-10 * np.linalg.cond(ref["product"])
