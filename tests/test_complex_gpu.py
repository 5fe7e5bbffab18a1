"""GPU parity for the complex field: the unitary
circulant, unitary Toeplitz block and SRFT families (multipliers.hpp:75-138),
and the complex pipelines they run in — preprocess_solve<Complex>
(preprocess.hpp:156-180), range_find<Complex> (lowrank.hpp:62-102) and
srft_sketch_check (lowrank.hpp:216-261) — against the reference's own headers
(oracle/_ref: REF.z*). The reference's QR is Eigen's Householder, absent
here: its unique positive-diagonal Q is restated with numpy's LAPACK QR and
the phase normalisation of qr.hpp:33-45."""
import numpy as np
import pytest

import paper_1406_5802_b200 as rl
from paper_1406_5802_b200.randla import MultiplierKind as K, MultiplierSpec as Spec, ToeplitzVariant as V

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref(orc):
    if orc.REF is None:
        pytest.skip("oracle/_ref not built")
    return orc.REF


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def canonical_q(y):
    """the reference's qr (qr.hpp:21-47): Householder Q with R's diagonal
    rotated real positive"""
    q, r = np.linalg.qr(y)
    d = np.diag(r)
    return q * (d / np.abs(d))[None, :]


# ---- multipliers -----------------------------------------------------------------
def test_srft_and_real_families_bit_identical(cuda, ref):
    for n, l, seed in [(64, 64, 3), (64, 16, 9), (100, 37, 11), (256, 256, 5)]:
        dev = rl.materialize_complex(Spec(K.SRFT, seed, n, l))
        exp, st = ref.zmaterialize(int(K.SRFT), n, l, seed)
        assert st == 0
        np.testing.assert_array_equal(dev, exp)
        np.testing.assert_array_equal(rl.srft_columns(n, l, seed), ref.srft_columns(n, l, seed))
    for kind, card in [(K.GAUSSIAN, 65536), (K.FINITE_SET_UNIFORM, 7)]:
        dev = rl.materialize_complex(Spec(kind, 21, 50, 20, set_cardinality=card))
        exp, st = ref.zmaterialize(int(kind), 50, 20, 21, card=card)
        np.testing.assert_array_equal(dev, exp)


def test_unitary_circulant_and_toeplitz(cuda, ref):
    for n, seed in [(64, 1), (128, 7), (96, 3), (1024, 2)]:
        c = rl.gen_unitary_circulant(n, seed).first_column()
        cr = ref.gen_unitary_circulant(n, seed)
        # the same spectrum bits, inverse-transformed by two FFT implementations
        assert np.abs(c - cr).max() <= 1e-15 * 4 * np.log2(n)
        dense = rl.materialize_complex(Spec(K.UNITARY_CIRCULANT, seed, n, n))
        exp, st = ref.zmaterialize(int(K.UNITARY_CIRCULANT), n, n, seed)
        assert st == 0 and rel(dense, exp) <= 1e-14
        assert np.linalg.norm(dense.conj().T @ dense - np.eye(n)) <= 1e-12  # unitary
        t = rl.materialize_complex(Spec(K.TOEPLITZ_BLOCK, seed, n, n // 4, variant=V.UNITARY))
        exp, st = ref.zmaterialize(int(K.TOEPLITZ_BLOCK), n, n // 4, seed, variant=1)
        assert st == 0 and rel(t, exp) <= 1e-14
    # the real pipeline still refuses the complex families (multipliers.hpp:176-179)
    with pytest.raises(rl.DimensionError):
        rl.materialize(Spec(K.SRFT, 1, 8, 8))


def test_complex_products(cuda, ref):
    rng = np.random.default_rng(5)
    a, b = crandn(rng, 70, 45), crandn(rng, 45, 33)
    assert rel(rl.matmul(a, b), a @ b) <= 1e-14
    # matmul_by_circulant / _toeplitz_block / circulant_apply over C (circulant.hpp:81-203)
    c = rl.gen_unitary_circulant(64, 4)
    cd = c.dense()
    a = crandn(rng, 20, 64)
    assert rel(rl.matmul_by_circulant(a, c), a @ cd) <= 1e-13
    t = rl.ToeplitzBlock(c, 64, 10)
    assert rel(rl.matmul_by_toeplitz_block(a, t), a @ cd[:, :10]) <= 1e-13
    x = crandn(rng, 64)
    assert rel(rl.circulant_apply(c, x), cd @ x) <= 1e-13
    # a real circulant against complex data (circulant.hpp:96-98)
    rc = rl.gen_real_circulant(64, 8)
    assert rel(rl.matmul_by_circulant(a, rc), a @ rc.dense()) <= 1e-13
    # complex singular values (svd.hpp:76-88)
    m = crandn(rng, 30, 20)
    np.testing.assert_allclose(rl.svd_values(m), np.linalg.svd(m, compute_uv=False), rtol=1e-12)


# ---- complex GENP and preprocess_solve ---------------------------------------------
@pytest.mark.parametrize("n", [64, 100, 200, 257])
def test_complex_genp_vs_reference(cuda, ref, n):
    rng = np.random.default_rng(n)
    a = crandn(rng, n, n) + 2 * np.sqrt(n) * np.eye(n)
    out = rl.preprocess_solve(a, crandn(rng, n), None, None, 0, want_lu=True)
    lu_ref, st, _ = ref.zgenp_factor(a)
    assert st == 0
    kappa = np.linalg.cond(a)
    assert rel(out.lu, lu_ref) <= 1e-10 * kappa
    assert rel(np.diag(out.lu), np.diag(lu_ref)) <= 1e-10 * kappa


POSTS = [(K.GAUSSIAN, 0), (K.REAL_CIRCULANT, 0), (K.UNITARY_CIRCULANT, 0), (K.TOEPLITZ_BLOCK, 0),
         (K.TOEPLITZ_BLOCK, 1), (K.SRFT, 0), (K.FINITE_SET_UNIFORM, 0), (K.CIRC_SKEW_PRODUCT, 0)]


@pytest.mark.parametrize("kind,variant", POSTS)
def test_complex_preprocess_solve_vs_reference(cuda, ref, kind, variant):
    rng = np.random.default_rng(int(kind) * 10 + variant)
    n = 96
    a = crandn(rng, n, n)
    b = crandn(rng, n)
    seed = 1234 + int(kind)
    out = rl.preprocess_solve(a, b, None, Spec(kind, seed, variant=variant), 1)
    exp = ref.zpreprocess_solve_spec(a, b, post=(int(kind), variant, seed), refine=1)
    assert exp["status"] == 0
    kappa = np.linalg.cond(a)
    assert rel(out.x, exp["x"]) <= 1e-10 * kappa, (rel(out.x, exp["x"]), kappa)
    h, he = np.asarray(out.residual_history), exp["history"]
    assert len(h) == 2 and not out.diverged
    assert 0.1 * he[0] <= h[0] <= 10 * he[0], (h, he)
    assert h[1] <= 1e-13 and he[1] <= 1e-13


def test_complex_two_sided_and_device_arrays(cuda, ref):
    torch = cuda
    rng = np.random.default_rng(3)
    n = 80
    a, b = crandn(rng, n, n), crandn(rng, n)
    pre, post = Spec(K.UNITARY_CIRCULANT, 5), Spec(K.SRFT, 6)
    out = rl.preprocess_solve(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), pre, post, 0)
    exp = ref.zpreprocess_solve_spec(a, b, pre=(int(K.UNITARY_CIRCULANT), 0, 5), post=(int(K.SRFT), 0, 6))
    assert exp["status"] == 0
    assert rel(out.x.cpu().numpy(), exp["x"]) <= 1e-10 * np.linalg.cond(a)


def test_dft_input_table5a(cuda, ref):
    """gen_dft_input (testbed/inputs.hpp:49-55) with a Gaussian rescue
    (presets.hpp:254-279): the transform matrix is bit-identical, the solve
    agrees with the reference"""
    for n in (64, 128, 256):
        d = rl.gen_dft_input(n)
        np.testing.assert_array_equal(d, ref.dft_dense(n))
        b = rl.to_complex(rl.gen_gaussian_vector(n, 2))
        out = rl.preprocess_solve(d, b, None, Spec(K.GAUSSIAN, 3), 1)
        exp = ref.zpreprocess_solve_spec(d, b, post=(int(K.GAUSSIAN), 0, 3), refine=1)
        assert exp["status"] == 0
        assert rel(out.x, exp["x"]) <= 1e-10 * np.linalg.cond(d)
        assert out.residual_history[0] <= 1e-4  # the preset's check (presets.hpp:280-282)


def test_complex_zero_pivot_verdict(cuda, ref):
    rng = np.random.default_rng(9)
    n = 70
    a = crandn(rng, n, n)
    a[:3, :3] = np.outer(a[:3, 0], [1, 2j, -1])  # leading 3x3 block of rank one: step 2
    b = crandn(rng, n)
    exp = ref.zpreprocess_solve_spec(a, b)
    assert exp["status"] == ref.ZERO_PIVOT
    with pytest.raises(rl.ZeroPivotError) as e:
        rl.preprocess_solve(a, b, None, None, 0)
    assert e.value.step == exp["zero_step"] == 2


# ---- complex range finder ----------------------------------------------------------
def lownumrank_c(n, r, seed):
    rng = np.random.default_rng(seed)
    s, _ = np.linalg.qr(crandn(rng, n, n))
    t, _ = np.linalg.qr(crandn(rng, n, n))
    sig = np.array([1.0 / (j + 1) if j < r else 1e-10 for j in range(n)])
    return (s * sig) @ t.conj().T


@pytest.mark.parametrize("kind,variant,ps", [(K.TOEPLITZ_BLOCK, 1, 0), (K.TOEPLITZ_BLOCK, 0, 0), (K.SRFT, 0, 0),
                                             (K.GAUSSIAN, 0, 1), (K.UNITARY_CIRCULANT, 0, 0)])
def test_complex_range_find_vs_reference(cuda, ref, kind, variant, ps):
    n, r = 128, 8
    a = lownumrank_c(n, r, int(kind) + 10 * variant)
    l = n if kind == K.UNITARY_CIRCULANT else r
    res = rl.range_find(a, l, 0, Spec(kind, 77, variant=variant), ps)
    y, st = ref.zrange_sketch(a, l, int(kind), 77, variant=variant, power_steps=ps)
    assert st == 0
    q_ref = canonical_q(y)
    kap = np.linalg.cond(y)
    assert rel(res.q, q_ref) <= 1e-13 * kap * np.sqrt(n), (rel(res.q, q_ref), kap)
    assert np.linalg.norm(res.q.conj().T @ res.q - np.eye(l)) <= 1e-10 * n
    # positive real R diagonal (qr.hpp:40-45), where R_jj stands above rounding
    rd = np.diag(res.q.conj().T @ y)
    big = np.abs(rd) > 1e-6 * np.abs(rd).max()
    assert (np.abs(np.angle(rd[big])) < 1e-8).all()
    r_ref = a - q_ref @ (q_ref.conj().T @ a)
    fro = np.linalg.norm(r_ref)
    spec = np.linalg.norm(r_ref, 2)
    assert abs(res.info["residual_frobenius"] - fro) <= 1e-6 * fro + 1e-14
    assert abs(res.info["residual_spectral"] - spec) <= 1e-6 * spec + 1e-14
    # approximation_residual(a, result) on the given A (lowrank.hpp:99-102)
    again = rl.residual_norms(a, res)
    assert again["residual_frobenius"] == pytest.approx(res.info["residual_frobenius"], rel=1e-10)


def test_complex_range_find_rank_deficiency(cuda):
    rng = np.random.default_rng(4)
    a = crandn(rng, 64, 3) @ crandn(rng, 3, 64)  # rank 3
    with pytest.raises(rl.RankDeficiencyError):
        rl.range_find(a, 6, 0, Spec(K.GAUSSIAN, 2), 0)


# ---- srft_sketch_check ---------------------------------------------------------------
@pytest.mark.parametrize("variant", [rl.SketchVariant.SRFT, rl.SketchVariant.CIRCULANT_PERMUTATION])
def test_srft_sketch_check(cuda, ref, variant):
    from paper_1406_5802_b200 import testbed
    for n in (64, 128):
        inst = testbed.gen_lownumrank(n, 8, rl.derive_seed(5, 1))
        seed = rl.derive_seed(5, 2)
        res = rl.srft_sketch_check(inst.a, 8, seed, variant, inst.singulars[8])
        assert res.clamped and res.sketch_width == n  # the prescribed width exceeds n at these sizes
        s, st = ref.srft_matrix(n, n, seed, int(variant))
        assert st == 0
        mine = rl.materialize_complex(Spec(K.SRFT, seed, n, n)) if variant == rl.SketchVariant.SRFT else None
        if mine is not None:
            np.testing.assert_array_equal(mine, s)
        ac = inst.a.astype(np.complex128)
        q = canonical_q(ac @ s)
        resid = np.linalg.norm(ac - q @ (q.conj().T @ ac), 2)
        bound = np.sqrt(1.0 + 7.0 * n / n) * inst.singulars[8]
        assert res.bound == pytest.approx(bound, rel=1e-15)
        # a square unitary-up-to-scaling sketch: the residual is rounding level
        assert res.residual <= 1e-12 and resid <= 1e-12
        assert (res.residual <= res.bound) == (resid <= bound)
    # without the known sigma: svd_values(a)[r]
    res2 = rl.srft_sketch_check(inst.a, 8, seed, variant)
    assert res2.bound == pytest.approx(res.bound, rel=1e-8)
