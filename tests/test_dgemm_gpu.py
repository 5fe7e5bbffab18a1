"""GPU parity: FP64 DMMA GEMM (matmul, matrix.hpp:115-121) against the
oracle's GEMM, at the reference's own GEMM tolerance (1e-13 relative,
tests/test_field_core.cpp:52-58), odd and ragged shapes included."""
import numpy as np
import pytest

import paper_1406_5802_b200 as rl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (3, 5, 7), (128, 16, 128), (129, 17, 130), (200, 1000, 64),
                                   (1024, 1024, 1024), (777, 333, 555), (64, 4096, 8), (2, 2, 2)])
def test_matmul_vs_oracle(cuda, orc, m, k, n):
    rng = np.random.default_rng(m * 1000 + k * 10 + n)
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((k, n))
    c = rl.matmul(a, b)
    ref = orc.C.matmul(a, b)
    err = np.abs(c - ref).max() / max(np.abs(ref).max(), 1e-300)
    assert err <= 1e-13 * max(1.0, np.sqrt(k)), err


def test_matmul_kat_and_device(cuda):
    torch = cuda
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[5.0, 6.0], [7.0, 8.0]])
    np.testing.assert_array_equal(rl.matmul(a, b), [[19.0, 22.0], [43.0, 50.0]])
    da = torch.randn(300, 200, dtype=torch.float64, device="cuda")
    db = torch.randn(200, 100, dtype=torch.float64, device="cuda")
    dc = rl.matmul(da, db)
    torch.cuda.synchronize()
    assert (dc - da @ db).abs().max().item() < 1e-12


def test_matmul_dimension_error(cuda):
    with pytest.raises(rl.DimensionError):
        rl.matmul(np.zeros((3, 4)), np.zeros((5, 2)))


@pytest.mark.parametrize("n", [4096, 6000])
def test_many_wave_genp_updates_exact_and_deterministic(cuda, n):
    """The multi-wave trailing-update GEMMs of blocked GENP (C -= A B with
    K = 64 / 128, thousands of tiles, two CTAs per SM, stage ring refilled as
    the MMA warps release stages): L U reproduces A to rounding and two calls
    return identical bits. (A missing generic->async proxy fence before the
    refill once corrupted a few fragments per call at this size.)"""
    torch = cuda
    import ctypes
    from paper_1406_5802_b200 import capi
    L = capi.lib()
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    lu1, lu2 = torch.empty_like(a), torch.empty_like(a)
    info = capi.rl_solve_info()
    assert L.rl_genp_factor(None, capi.RL_DEVICE, n, a.data_ptr(), lu1.data_ptr(), ctypes.byref(info)) == 0
    assert L.rl_genp_factor(None, capi.RL_DEVICE, n, a.data_ptr(), lu2.data_ptr(), ctypes.byref(info)) == 0
    torch.cuda.synchronize()
    assert torch.equal(lu1, lu2)
    lo = torch.tril(lu1, -1) + torch.eye(n, dtype=torch.float64, device="cuda")
    rel = (torch.linalg.matrix_norm(lo @ torch.triu(lu1) - a) / torch.linalg.matrix_norm(a)).item()
    assert rel <= 1e-13 * n * info.growth, (rel, info.growth)
