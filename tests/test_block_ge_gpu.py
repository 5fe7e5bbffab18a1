"""GPU parity: block elimination (block_ge.hpp) and GEPP (lu.hpp:62-147)
through the C ABI vs the reference's own code (oracle.REF, compiled from
/root/reference). The device kernels keep the reference's arithmetic order
(no FMA, natural-order Schur sums), so the bar is bit-identity: GEPP factors
and permutation, lu_solve / lu_solve_transpose, block_ge pivots, the stored
Schur leaf and block_solve's x. reassemble() goes through the DMMA GEMM and
is checked to the reference test's tolerance."""
import numpy as np
import pytest

import oracle
import paper_1406_5802_b200 as rl

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(oracle.REF is None, reason="oracle/_ref not built")]
REF = oracle.REF


def _rand(n, seed):
    return np.random.default_rng(seed).standard_normal((n, n))


@pytest.mark.parametrize("n,seed", [(1, 1), (2, 2), (9, 31), (64, 5), (257, 6)])
def test_gepp_factor_bitwise(cuda, n, seed):
    a = _rand(n, seed)
    packed, perm, st = REF.gepp_factor(a)
    assert st == 0
    f = rl.gepp_factor(a)
    np.testing.assert_array_equal(f.packed, packed)
    np.testing.assert_array_equal(f.perm, perm)
    b = np.random.default_rng(seed + 1).standard_normal(n)
    np.testing.assert_array_equal(rl.lu_solve(f, b), REF.gepp_solve(a, b))
    np.testing.assert_array_equal(rl.lu_solve_transpose(f, b), REF.gepp_solve(a, b, transpose=True))
    # device-resident path gives the same bits
    import torch
    fd = rl.gepp_factor(torch.from_numpy(a).cuda())
    np.testing.assert_array_equal(fd.packed.cpu().numpy(), packed)
    np.testing.assert_array_equal(fd.perm.cpu().numpy(), perm)


def test_gepp_singular(cuda):
    """lu.hpp:81-83: SingularMatrixError at the first step whose best pivot
    is <= tol"""
    a = np.zeros((3, 3))
    a[1, 1] = a[2, 2] = 1.0
    with pytest.raises(rl.SingularMatrixError):
        rl.gepp_factor(a)
    assert REF.gepp_factor(a)[2] == REF.SINGULAR


SPLITS = [
    (8, [1] * 8), (6, [6]), (8, [4, 4]), (8, [2, 2, 4]), (10, [2, 3, 5]), (10, [5, 5]), (10, None),
    (100, [32, 32, 36]), (200, [64, 1, 63, 72]), (300, None),
]


@pytest.mark.parametrize("n,split", SPLITS)
def test_block_ge_bitwise(cuda, n, split):
    split = split or rl.balanced_split(n)
    a = _rand(n, 1000 + n + len(split))
    b = np.random.default_rng(n).standard_normal(n)
    ref = REF.block_ge(a, split, b)
    assert ref["status"] == 0
    f = rl.block_ge_factor(a, split)
    np.testing.assert_array_equal(f.pivots(), ref["pivots"])
    node = f.root
    while not node.leaf():
        node = node.schur_child
    np.testing.assert_array_equal(node.block_matrix, ref["last_leaf"])
    np.testing.assert_array_equal(rl.block_solve(f, b), ref["x"])
    # reassemble (tests/test_elimination.cpp:121-129 bar)
    r = f.reassemble()
    assert np.linalg.norm(r - a) <= 1e-9 * n * np.linalg.norm(a, 2)


def test_block_ge_device_resident(cuda):
    import torch
    n, split = 96, [40, 24, 32]
    a = _rand(n, 77)
    b = np.random.default_rng(78).standard_normal(n)
    ref = REF.block_ge(a, split, b)
    f = rl.block_ge_factor(torch.from_numpy(a).cuda(), split)
    np.testing.assert_array_equal(f.pivots().cpu().numpy(), ref["pivots"])
    np.testing.assert_array_equal(rl.block_solve(f, torch.from_numpy(b).cuda()).cpu().numpy(), ref["x"])
    assert float((f.reassemble().cpu() - torch.from_numpy(a)).norm()) <= 1e-9 * n * np.linalg.norm(a, 2)


def test_block_ge_degenerate_equals_genp(cuda):
    """tests/test_elimination.cpp:91-97 on the device: split of ones gives
    the reference genp_factor's pivots bit for bit"""
    a = _rand(8, 41)
    lu, _ = REF.genp_factor(a)
    np.testing.assert_array_equal(rl.block_ge_factor(a, [1] * 8).pivots(), np.diag(lu))


def test_block_ge_errors(cuda):
    """tests/test_elimination.cpp:333-349"""
    a = _rand(6, 75)
    with pytest.raises(rl.DimensionError):
        rl.block_ge_factor(a, [3, 2])
    with pytest.raises(rl.DimensionError):
        rl.block_ge_factor(a, [])
    with pytest.raises(rl.DimensionError):
        rl.block_ge_factor(a, [6, 0])
    s = np.diag([0.0, 1.0, 1.0, 1.0])
    with pytest.raises(rl.SingularPivotBlockError) as e:
        rl.block_ge_factor(s, [2, 2])
    assert e.value.position == 1
    # a singular block deeper in the split: position = its offset + 1
    m = np.eye(6)
    m[3, 3] = m[4, 4] = 0.0
    ref = REF.block_ge(m, [3, 2, 1], np.ones(6))
    with pytest.raises(rl.SingularPivotBlockError) as e:
        rl.block_ge_factor(m, [3, 2, 1])
    assert ref["status"] == REF.SINGULAR_BLOCK and e.value.position == ref["position"] == 4


def test_schur_complement(cuda):
    """block_ge.hpp:202-218 vs the reference (GEMM summation order differs:
    the reference's own 1e-11 bar, tests/test_elimination.cpp:141-153)"""
    for seed in range(5):
        a = _rand(12, 200 + seed) + 12 * np.eye(12)
        s = rl.schur_complement(a, 5)
        assert np.linalg.norm(s - REF.schur_complement(a, 5)) <= 1e-11 * np.linalg.norm(s)
    with pytest.raises(rl.SingularMatrixError):
        rl.schur_complement(np.diag([0.0, 1.0, 1.0]), 1)
