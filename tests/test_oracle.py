"""CPU: pin the plain-C oracle restatement (oracle/oracle.c) to the
reference — its golden vectors, KATs and outputs of the reference's own
headers (oracle/_ref, fixtures in tests/golden/golden.npz)."""
import numpy as np
import pytest


def test_golden_rng_csv(orc, golden):
    """tests/test_testbed.cpp:187-204: run_experiment(label unit/golden,
    seed 12345, 3 trials) of RngStream(ts).next_double()."""
    C = orc.C
    key = C.hash_label(b"unit/golden")
    assert key == int(golden["hash_label_unit_golden"][0])
    draws = []
    for t in range(3):
        ts = C.derive_seed(12345, key, t)
        draws.append(C.gen_real_circulant_column(1, ts)[0] * 0.5 + 0.5)  # next_symmetric = 2u-1
    np.testing.assert_array_equal(np.array(draws), golden["golden_draws"])
    # summarize (stats.hpp:19-34): sequential sum, population std; the
    # reference test's expected CSV fields, printed %.17g
    ssum = 0.0
    for v in draws:
        ssum += v
    mean = ssum / 3
    var = 0.0
    for v in draws:
        var += (v - mean) * (v - mean)
    std = (var / 3) ** 0.5
    fields = ["%.17g" % x for x in (mean, max(draws), min(draws), std)]
    assert fields == ["0.27212314401380694", "0.58099988541126291", "0.063155289723205499", "0.22290071872626696"]
    np.testing.assert_array_equal(golden["golden_stats"], [mean, max(draws), min(draws), std])


def test_rng_streams_match_reference(orc, golden):
    C = orc.C
    np.testing.assert_array_equal(C.gen_gaussian(7, 5, 42), golden["gauss_7x5_seed42"])
    np.testing.assert_array_equal(C.gen_gaussian_vector(1001, 3), golden["gauss_vec_1001_seed3"])
    np.testing.assert_array_equal(C.gen_real_circulant_column(64, 13), golden["circ_col_64_seed13"])
    for s, k1, k2, want in golden["derive_seed_cases"]:
        assert C.derive_seed(int(s), int(k1), int(k2)) == int(want)


def test_genp_kats(orc, golden):
    """tests/test_elimination.cpp:29-50"""
    C = orc.C
    lu, zs, _ = C.genp_factor(np.eye(3))
    assert zs == 0 and np.array_equal(lu, np.eye(3))
    lu, zs, _ = C.genp_factor(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert zs == 1 == int(golden["kat_genp_swap_step"][0])
    lu, zs, _ = C.genp_factor(np.array([[2.0, 1.0], [4.0, 5.0]]))
    assert zs == 0
    assert lu[1, 0] == 2.0 and lu[0, 0] == 2.0 and lu[0, 1] == 1.0 and lu[1, 1] == 3.0
    np.testing.assert_array_equal(lu, golden["kat_genp_2x2_lu"])


def test_fft_kats(orc, golden):
    """tests/test_transforms.cpp:57-65 (FFT of e1 is all ones) plus the
    reference's own outputs (radix-2 and dense fallback)."""
    C = orc.C
    e1 = np.zeros(16, complex)
    e1[0] = 1
    np.testing.assert_array_equal(C.fft(e1), np.ones(16, complex))
    np.testing.assert_array_equal(C.fft(golden["fft_in_64"]), golden["fft_out_64"])
    np.testing.assert_array_equal(C.fft(golden["fft_in_64"], inverse=True), golden["ifft_out_64"])
    np.testing.assert_array_equal(C.fft(golden["fft_in_64"][:12]), golden["fft_out_12"])
    # omega = exp(+2 pi i / n): compare with numpy's (sign -1) DFT conjugated
    z = golden["fft_in_64"]
    np.testing.assert_allclose(C.fft(z), np.conj(np.fft.fft(np.conj(z))), rtol=0, atol=1e-12)


def test_circulant_kats(orc, golden):
    """two-point circulant (1,2)*(3,4) = (11,10) (tests/test_transforms.cpp:93-98),
    dense-expansion agreement, reference outputs."""
    C = orc.C
    y, st = C.circulant_apply(np.array([1.0, 2.0]), np.array([3.0, 4.0]))
    assert st == 0 and np.allclose(y, [11.0, 10.0], rtol=0, atol=1e-14)
    a, c = golden["circ_a_16x64"], golden["circ_c_64"]
    out, st = C.matmul_by_circulant(a, c)
    assert st == 0
    np.testing.assert_array_equal(out, golden["circ_ac_16x64"])
    n = c.shape[0]
    dense = np.array([[c[(i - j) % n] for j in range(n)] for i in range(n)])
    np.testing.assert_allclose(out, a @ dense, rtol=0, atol=1e-11 * np.abs(a @ dense).max())
    out, st = C.matmul_by_toeplitz_block(a[:, :48], c, 20)
    assert st == 0
    np.testing.assert_array_equal(out, golden["toep_ac_16x48_l20"])
    np.testing.assert_allclose(out, a[:, :48] @ dense[:48, :20], rtol=0, atol=1e-11 * np.abs(out).max())


def test_config1_against_reference(orc, golden):
    """BASELINE config 1 through the restatement vs the reference's own
    preprocess_solve (same GEMM hook, so bitwise when the hook matches)."""
    C = orc.C
    n = 1024
    A = C.gen_gaussian(n, n, 1)
    b = C.gen_gaussian_vector(n, 3)
    G = C.gen_gaussian(n, n, 2)
    for refine in (0, 1):
        p = C.preprocess_solve(A, b, 1, G, refine=refine, want_lu=True)
        assert p["status"] == 0
        if C.uses_blas() == int(golden["cfg1_gemm"][0]):
            np.testing.assert_array_equal(p["x"], golden[f"cfg1_x_refine{refine}"])
            np.testing.assert_array_equal(p["history"], golden[f"cfg1_hist_refine{refine}"])
        else:
            np.testing.assert_allclose(p["x"], golden[f"cfg1_x_refine{refine}"], rtol=1e-6)
    assert golden["cfg1_hist_refine0"][0] < 1e-5
    assert golden["cfg1_hist_refine1"][1] < 1e-3 * golden["cfg1_hist_refine1"][0]  # refinement gain


def test_config2_against_reference(orc, golden):
    C = orc.C
    r = C.batched_config2(256, base=7, threads=4)
    assert (r["status"] == 0).all()
    np.testing.assert_array_equal(r["x"], golden["cfg2_x_256"])
    np.testing.assert_array_equal(r["resid"], golden["cfg2_resid_256"])


@pytest.mark.skipif(__import__("oracle").REF is None, reason="oracle/_ref not built (needs /root/reference)")
def test_restatement_bitwise_vs_reference_headers(orc):
    """Random shapes: restatement == reference headers, bit for bit."""
    C, R = orc.C, orc.REF
    rng = np.random.default_rng(0)
    for n in (1, 2, 5, 17, 64):
        a = rng.standard_normal((n, n))
        assert C.spectral_norm_estimate(a) == R.spectral_norm_estimate(a)
        l1, z1, _ = C.genp_factor(a)
        l2, z2 = R.genp_factor(a)
        assert z1 == z2 and np.array_equal(l1, l2)
        b = rng.standard_normal(n)
        assert np.array_equal(C.lu_solve(l1, b), R.lu_solve(l1, b))
        c = rng.standard_normal(n)
        o1, s1 = C.matmul_by_circulant(a, c)
        o2, s2 = R.matmul_by_circulant(a, c)
        assert s1 == s2 and np.array_equal(o1, o2)
        p1 = C.preprocess_solve(a, b, 1, C.gen_gaussian(n, n, 9), refine=2)
        p2 = R.preprocess_solve(a, b, 1, 9, refine=2)
        assert p1["status"] == p2["status"]
        if p1["status"] == 0:
            assert np.array_equal(p1["x"], p2["x"]) and np.array_equal(p1["history"], p2["history"])
    # zero-pivot verdicts agree (hard block of zeros)
    a = np.eye(6)
    a[2, 2] = 0.0
    assert C.genp_factor(a)[1] == R.genp_factor(a)[1] == 3
    # reference uniform circulant family through preprocess_solve
    a = rng.standard_normal((32, 32))
    b = rng.standard_normal(32)
    p1 = C.preprocess_solve(a, b, 2, C.gen_real_circulant_column(32, 77), refine=1)
    p2 = R.preprocess_solve(a, b, 2, 77, refine=1)
    assert np.array_equal(p1["x"], p2["x"])


def test_qr_restatement_properties(orc):
    """qr.hpp:21-47 invariants: orthonormal Q, positive diagonal, A = QR,
    rank verdict (tests/test_field_core.cpp:73-108, KAT (3,4)^T)."""
    C = orc.C
    q, r, st, _ = C.qr(np.array([[3.0], [4.0]]))
    assert st == 0 and np.allclose(q[:, 0], [0.6, 0.8], atol=1e-15) and abs(r[0, 0] - 5.0) < 1e-14
    a = np.random.default_rng(1).standard_normal((200, 30))
    q, r, st, _ = C.qr(a)
    assert st == 0
    assert np.abs(q.T @ q - np.eye(30)).max() < 1e-13
    assert (np.diag(r) > 0).all() and np.allclose(np.triu(r), r)
    assert np.abs(q @ r - a).max() < 1e-12
    a[:, 7] = a[:, 3]
    q, r, st, bad = C.qr(a)
    assert st == 4 and bad == 8
