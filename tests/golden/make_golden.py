"""Regenerate the committed golden fixtures from the REFERENCE ITSELF.

Runs in the dev container only (needs oracle/_ref/librandla_ref.so, i.e. the
reference's own headers compiled by oracle/Makefile; /root/reference does not
exist on the GPU box). Writes tests/golden/golden.npz. The fixtures pin the
plain-C oracle restatement (tests/test_oracle.py) and the CUDA path
(tests/test_*_gpu.py) to the reference's outputs.

Usage: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

R = oracle.REF
assert R is not None, "oracle/_ref not built: run `make -C oracle` with /root/reference present"
out = {}

# tests/test_testbed.cpp:187-204 golden run: label unit/golden, seed 12345, 3 trials
d, st = R.golden_draws("unit/golden", 12345, 3)
out["golden_draws"] = d
out["golden_stats"] = st  # mean, max, min, std

# RNG streams: gen_gaussian, derive_seed, hash_label, real circulant column
out["gauss_7x5_seed42"] = R.gen_gaussian(7, 5, 42)
out["gauss_vec_1001_seed3"] = R.gen_gaussian(1001, 1, 3).reshape(-1)
out["circ_col_64_seed13"] = R.gen_real_circulant_column(64, 13)
out["derive_seed_cases"] = np.array([[s, k1, k2, R.derive_seed(s, k1, k2)]
                                     for s, k1, k2 in [(7, 1, 0), (7, 2, 0), (7, 3, 0), (62, 5, 0),
                                                       (992, 0x52455452, 1), (2**64 - 1, 3, 9)]], dtype=np.uint64)
out["hash_label_unit_golden"] = np.array([R.hash_label(b"unit/golden")], dtype=np.uint64)

# config 1 (n=1024, A seed 1, G seed 2, b seed 3), refine 0 and 1
n = 1024
A = R.gen_gaussian(n, n, 1)
b = R.gen_gaussian(n, 1, 3).reshape(-1)
for refine in (0, 1):
    p = R.preprocess_solve(A, b, 1, 2, refine=refine)
    out[f"cfg1_x_refine{refine}"] = p["x"]
    out[f"cfg1_hist_refine{refine}"] = p["history"]
G = R.gen_gaussian(n, n, 2)
AG = R.matmul(A, G)
lu, zs = R.genp_factor(AG)
assert zs == 0
out["cfg1_pivots"] = np.diag(lu).copy()
out["cfg1_growth"] = np.array([np.abs(np.triu(lu)).max() / np.abs(AG).max()])
out["cfg1_normest_AG"] = np.array([R.spectral_norm_estimate(AG)])
out["cfg1_normest_A"] = np.array([R.spectral_norm_estimate(A)])
out["cfg1_gemm"] = np.array([oracle.C.uses_blas()])

# config 2: first 256 systems with the SURVEY §8(d) seed mapping (base 7)
c2 = R.batched_config2(256, base=7)
out["cfg2_x_256"] = c2["x"]
out["cfg2_resid_256"] = c2["resid"]

# GENP KATs (tests/test_elimination.cpp:29-50) and small transforms
out["kat_genp_2x2_lu"] = R.genp_factor(np.array([[2.0, 1.0], [4.0, 5.0]]))[0]
out["kat_genp_swap_step"] = np.array([R.genp_factor(np.array([[0.0, 1.0], [1.0, 0.0]]))[1]])
z = R.gen_gaussian(64, 2, 5)
zc = z[:, 0] + 1j * z[:, 1]
out["fft_in_64"] = zc
out["fft_out_64"] = R.fft(zc)
out["ifft_out_64"] = R.fft(zc, inverse=True)
z12 = zc[:12]
out["fft_out_12"] = R.fft(z12)  # non-power-of-two dense fallback (fft.hpp:78-82)
a = R.gen_gaussian(16, 64, 6)
c = R.gen_gaussian(64, 1, 13).reshape(-1)
out["circ_a_16x64"] = a
out["circ_c_64"] = c
out["circ_ac_16x64"] = R.matmul_by_circulant(a, c)[0]
out["toep_ac_16x48_l20"] = R.matmul_by_toeplitz_block(a[:, :48], c, 20)[0]

np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz"), **out)
print("wrote", len(out), "arrays")
