"""CPU: the C-ABI library loads, exports every symbol include/randla_capi.h
declares, and its host-side exact multiplier generator is bit-identical to
the oracle (and hence the reference). No compute kernels run here."""
import ctypes

import numpy as np
import pytest

from paper_1406_5802_b200 import capi
import paper_1406_5802_b200 as rl


def test_library_exports_every_header_symbol():
    syms = capi.header_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(capi.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(capi.SIGNATURES), set(syms) ^ set(capi.SIGNATURES)
    assert capi.lib().rl_abi_version() == 2


def test_product_library_is_native_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_derive_seed_and_hash_label(orc, golden):
    for s, k1, k2, want in golden["derive_seed_cases"]:
        assert rl.derive_seed(int(s), int(k1), int(k2)) == int(want)
    assert rl.hash_label("unit/golden") == int(golden["hash_label_unit_golden"][0])


@pytest.mark.parametrize("m,n,seed", [(7, 5, 42), (1, 1, 0), (1001, 1, 3), (300, 301, 2), (2048, 1024, 11)])
def test_gen_gaussian_bit_exact(orc, m, n, seed):
    """large shapes go through the parallel two-pass generator"""
    np.testing.assert_array_equal(rl.gen_gaussian(m, n, seed), orc.C.gen_gaussian(m, n, seed))


def test_gen_gaussian_parallel_thread_counts(orc):
    want = orc.C.gen_gaussian(1500, 700, 99)
    for t in (1, 3, 8):
        capi.lib().rl_set_host_threads(t)
        np.testing.assert_array_equal(rl.gen_gaussian(1500, 700, 99), want)
    capi.lib().rl_set_host_threads(0)


def test_gen_gaussian_batch_config2_seeds(orc):
    seeds = np.array([rl.derive_seed(7 + i, 1) for i in range(300)], dtype=np.uint64)
    got = rl.gen_gaussian_batch(300, 32, 32, seeds)
    r = orc.C.batched_config2(300, base=7, threads=2)
    np.testing.assert_array_equal(got, r["a"])


def test_real_circulant_column(golden):
    np.testing.assert_array_equal(rl.gen_real_circulant_column(64, 13), golden["circ_col_64_seed13"])


def test_dimension_errors_without_device():
    with pytest.raises(rl.DimensionError):
        rl.gen_gaussian(0, 3, 1)


def test_compute_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a device")
    a = np.zeros((4, 32, 32))
    b = np.zeros((4, 32))
    with pytest.raises(rl.DeviceError):
        rl.batched_preprocess_solve_32(a, a, b)


@pytest.mark.parametrize("card", [2, 3, 1000, 65536, 2 ** 63 + 5])
def test_finite_set_uniform_bit_exact_vs_reference(orc, card):
    """gen_finite_set_uniform (multipliers.hpp:142-154) incl. next_below
    rejections (rng.hpp:46-53; card = 2^63 + 5 rejects about half the draws)"""
    import paper_1406_5802_b200 as rl
    if orc.REF is None:
        pytest.skip("oracle/_ref not built")
    for seed in (0, 7, 2 ** 64 - 1):
        got = rl.gen_finite_set_uniform(37, 29, seed, card)
        ref = orc.REF.gen_finite_set_uniform(37, 29, seed, card)
        assert np.array_equal(got, ref)
    big = rl.gen_finite_set_uniform(1024, 600, 5, card)  # the parallel two-pass path
    assert np.array_equal(big, orc.REF.gen_finite_set_uniform(1024, 600, 5, card))
