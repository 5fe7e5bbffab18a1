"""GPU parity: circulant / Toeplitz right products by FFT
(circulant.hpp:171-203) vs the oracle (the reference's own radix-2 FFT path),
at the reference's FFT tolerance (tests/test_transforms.cpp: 1e-11; acceptance
criterion 14: fast circulant vs dense <= 1e-10)."""
import numpy as np
import pytest

import paper_1406_5802_b200 as rl

pytestmark = pytest.mark.gpu


def _err(x, ref):
    return np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-300)


def test_two_point_kat(cuda):
    """(1,2) circulant times (3,4) = (11,10) (tests/test_transforms.cpp:93-98);
    as a row: a C with a = (3,4): (3*1 + 4*2, 3*2 + 4*1) = (11, 10)."""
    out = rl.matmul_by_circulant(np.array([[3.0, 4.0]]), np.array([1.0, 2.0]))
    np.testing.assert_allclose(out, [[11.0, 10.0]], rtol=0, atol=1e-14)


@pytest.mark.parametrize("m,n", [(1, 2), (3, 4), (5, 8), (7, 16), (4, 32), (9, 64), (33, 256), (16, 1024),
                                 (6, 4096), (7, 8192), (3, 12), (5, 1000)])
def test_circulant_vs_oracle(cuda, orc, m, n):
    a = orc.C.gen_gaussian(m, n, 300 + n)
    c = orc.C.gen_gaussian_vector(n, 13)
    ref, st = orc.C.matmul_by_circulant(a, c)
    assert st == 0
    out = rl.matmul_by_circulant(a, c)
    assert _err(out, ref) <= 1e-11, _err(out, ref)


@pytest.mark.parametrize("m,k,np_,l", [(3, 48, 64, 20), (8, 1000, 1024, 256), (5, 8192, 8192, 64),
                                       (4, 16384, 16384, 256), (7, 12000, 16384, 256), (3, 10, 12, 5),
                                       (2, 8192, 8192, 77), (2, 8192, 8192, 512), (2, 8192, 8192, 513),
                                       (2, 16384, 16384, 1)])
def test_toeplitz_vs_oracle(cuda, orc, m, k, np_, l):
    a = orc.C.gen_gaussian(m, k, 17 + k)
    c = orc.C.gen_gaussian_vector(np_, 21)
    ref, st = orc.C.matmul_by_toeplitz_block(a, c, l)
    assert st == 0
    out = rl.matmul_by_toeplitz_block(a, c, l)
    assert _err(out, ref) <= 1e-11, _err(out, ref)


def test_circulant_vs_dense_product(cuda, orc):
    """acceptance criterion 14 analogue: fast circulant == dense expansion"""
    n = 512
    c = orc.C.gen_real_circulant_column(n, 13)  # the reference's own uniform family
    dense = np.array([[c[(i - j) % n] for j in range(n)] for i in range(n)])
    a = orc.C.gen_gaussian(40, n, 5)
    out = rl.matmul_by_circulant(a, c)
    assert _err(out, a @ dense) <= 1e-10


def test_device_path_and_full_size_property(cuda, orc):
    """config-3 shape (8192 x 8192) on the device: linearity against the
    oracle on a row sample."""
    torch = cuda
    n = 8192
    a = torch.from_numpy(orc.C.gen_gaussian(n, n, 11)).cuda()
    c = orc.C.gen_gaussian_vector(n, 13)
    out = rl.matmul_by_circulant(a, torch.from_numpy(c).cuda())
    torch.cuda.synchronize()
    rows = [0, 1, 4095, 8190, 8191]
    sample = a[rows].cpu().numpy()
    ref, _ = orc.C.matmul_by_circulant(sample, c)
    assert _err(out[rows].cpu().numpy(), ref) <= 1e-11
    # linearity: (a0 + 2 a1) C == a0 C + 2 a1 C
    comb = rl.matmul_by_circulant((a[0:1] + 2 * a[1:2]).contiguous(), torch.from_numpy(c).cuda())
    assert (comb[0] - (out[0] + 2 * out[1])).abs().max().item() <= 1e-11 * out[0:2].abs().max().item()
