"""Oracle pins for block elimination (block_ge.hpp) — CPU only.

oracle.REF runs the reference's own block_ge_factor / gepp_factor /
lu_solve_transpose (compiled from /root/reference by oracle/Makefile); its
svd_values goes to our singular-values stand-in for Eigen's JacobiSVD
(oracle.c one-sided Jacobi). These tests re-run the reference's own
assertions for the path (tests/test_elimination.cpp:85-176, 330-349) on it,
so that the GPU parity tests can compare against it bit for bit."""
import numpy as np
import pytest

import oracle

REF = oracle.REF
pytestmark = pytest.mark.skipif(REF is None, reason="oracle/_ref not built")


def _rand(n, seed):
    return np.random.default_rng(seed).standard_normal((n, n))


def test_singular_values_standin():
    for m, n, seed in ((8, 8, 1), (13, 7, 2), (5, 9, 3), (64, 64, 4)):
        a = np.random.default_rng(seed).standard_normal((m, n))
        out = np.empty(min(m, n))
        oracle.C.lib.or_singular_values(m, n, oracle.ptr(a), oracle.ptr(out))
        ref = np.linalg.svd(a, compute_uv=False)
        np.testing.assert_allclose(out, ref, rtol=1e-13, atol=1e-15 * ref[0])


def test_gepp_solve_transpose():
    """tests/test_elimination.cpp:79-88: lu_solve_transpose residual"""
    a = _rand(9, 31)
    c = np.random.default_rng(32).standard_normal(9)
    x = REF.gepp_solve(a, c, transpose=True)
    assert np.linalg.norm(a.T @ x - c) / np.linalg.norm(c) <= 1e-11
    packed, perm, st = REF.gepp_factor(a)
    assert st == 0 and sorted(perm.tolist()) == list(range(9))
    lower = np.tril(packed, -1) + np.eye(9)
    np.testing.assert_allclose((lower @ np.triu(packed))[np.argsort(perm)], a, atol=1e-13)


def test_degenerate_blocking_is_genp_bitwise():
    """tests/test_elimination.cpp:91-97"""
    a = _rand(8, 41)
    lu, _ = REF.genp_factor(a)
    o = REF.block_ge(a, [1] * 8, np.ones(8))
    assert o["status"] == 0
    np.testing.assert_array_equal(o["pivots"], np.diag(lu))


def test_single_block_and_schur_oracle():
    """tests/test_elimination.cpp:99-119"""
    a = _rand(6, 42)
    b = np.random.default_rng(43).standard_normal(6)
    o = REF.block_ge(a, [6], b)
    assert np.linalg.norm(o["reassembled"] - a) <= 1e-12 * np.linalg.norm(a)
    assert np.linalg.norm(a @ o["x"] - b) / np.linalg.norm(b) <= 1e-12
    a = _rand(8, 44)
    o = REF.block_ge(a, [4, 4], np.ones(8))
    s = a[4:, 4:] - a[4:, :4] @ np.linalg.inv(a[:4, :4]) @ a[:4, 4:]
    assert np.linalg.norm(o["last_leaf"] - s) <= 1e-11 * np.linalg.norm(s)


def test_reassembly_and_path_independence():
    """tests/test_elimination.cpp:121-153"""
    a = _rand(10, 45)
    for split in ([2, 3, 5], [5, 5], [5, 2, 1, 1, 1]):
        o = REF.block_ge(a, split, np.ones(10))
        assert np.linalg.norm(o["reassembled"] - a) <= 1e-9 * 10 * np.linalg.norm(a, 2)
    for seed in range(20):
        a = _rand(8, 100 + seed) + 8 * np.eye(8)
        s1 = REF.block_ge(a, [4, 4], np.ones(8))["last_leaf"]
        s2 = REF.block_ge(a, [2, 2, 4], np.ones(8))["last_leaf"]
        assert np.linalg.norm(s1 - s2) <= 1e-11
        assert np.linalg.norm(s1 - REF.schur_complement(a, 4)) <= 1e-11


def test_bad_splits_and_singular_pivot_block():
    """tests/test_elimination.cpp:333-349"""
    a = _rand(6, 75)
    assert REF.block_ge(a, [3, 2], np.ones(6))["status"] == REF.DIM
    assert REF.block_ge(a, [], np.ones(6))["status"] == REF.DIM
    s = np.diag([0.0, 1.0, 1.0, 1.0])
    o = REF.block_ge(s, [2, 2], np.ones(4))
    assert o["status"] == REF.SINGULAR_BLOCK and o["position"] == 1
