/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the preprocessed-GENP /
 * low-rank hot path. Plain-C restatement of the reference algorithms in
 * /root/reference/proj/include/randla/ headers (each function cites the
 * file:line it follows). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product library
 * (paper_1406_5802_b200/csrc) never links or calls it.
 *
 * Pinned against: the reference's golden RNG CSV
 * (tests/test_testbed.cpp:187-204), the GENP KATs
 * (tests/test_elimination.cpp:29-50), the FFT/circulant KATs
 * (tests/test_transforms.cpp), and bitwise/tolerance comparison with the
 * reference's own headers compiled into oracle/_ref (see oracle/Makefile).
 *
 * Storage: row-major double, as Matrix<T> (matrix.hpp:13-25). Complex values
 * are interleaved (re, im) pairs, as std::complex<double>.
 */
#ifndef RANDLA_ORACLE_H
#define RANDLA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference exception types (types.hpp:44-78) */
enum {
    OR_OK = 0,
    OR_DIMENSION_ERROR = 1,
    OR_ZERO_PIVOT = 2,
    OR_LOGIC_ERROR = 5, /* circulant imaginary dust, circulant.hpp:63-64 */
    OR_RANK_DEFICIENCY = 4,
};

typedef struct {
    uint64_t state;
    int has_spare;
    double spare;
} or_rng;

void or_rng_init(or_rng* r, uint64_t seed);
void or_rng_derived(const or_rng* r, uint64_t key, or_rng* out);
uint64_t or_rng_next_u64(or_rng* r);
double or_rng_next_double(or_rng* r);
double or_rng_next_symmetric(or_rng* r);
double or_rng_next_gaussian(or_rng* r);
uint64_t or_hash_label(const char* s);
uint64_t or_derive_seed(uint64_t seed, uint64_t k1, uint64_t k2);

void or_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double* out);
void or_gen_gaussian_vector(int64_t n, uint64_t seed, double* out);
void or_gen_real_circulant_column(int64_t n, uint64_t seed, double* out);

/* row-major C = A(m x k) B(k x n) (OpenBLAS single-thread when found, else loop) */
void or_matmul(int64_t m, int64_t k, int64_t n, const double* a, const double* b, double* c);
int or_matmul_uses_blas(void);
void or_matvec(int64_t m, int64_t n, const double* a, const double* x, double* y);
double or_norm2(int64_t n, const double* v);
double or_frobenius_norm(int64_t m, int64_t n, const double* a);
double or_max_abs(int64_t m, int64_t n, const double* a);
double or_spectral_norm_estimate(int64_t m, int64_t n, const double* a);

/* packed LU: strict lower = L (unit diag implicit), upper incl. diag = U.
 * Returns OR_OK or OR_ZERO_PIVOT with *zero_step = 1-based step. */
int or_genp_factor(int64_t n, const double* a, double* lu, int64_t* zero_step, double* tol_out);
void or_genp_steps(int64_t n, double* lu, int64_t j0, int64_t j1);
void or_lu_solve(int64_t n, const double* lu, const double* b, double* x);
double or_relative_residual(int64_t n, const double* a, const double* x, const double* b);

/* complex interleaved FFT, omega = exp(+2 pi i / n) (fft.hpp:75-98) */
int or_fft(int64_t n, double* z);
int or_inverse_fft(int64_t n, double* z);
/* C x for a real circulant with first column c (circulant.hpp:85-91) */
int or_circulant_apply(int64_t n, const double* c, const double* x, double* y);
/* A (m x n) * C(c) (circulant.hpp:171-185) */
int or_matmul_by_circulant(int64_t m, int64_t n, const double* a, const double* c, double* out);
/* A (m x k) * leading k x l block of C(c), c of parent length np (circulant.hpp:187-203) */
int or_matmul_by_toeplitz_block(int64_t m, int64_t k, const double* a, int64_t np, const double* c,
                                int64_t l, double* out);

/* post multiplier kinds for or_preprocess_solve */
enum { OR_POST_NONE = 0, OR_POST_DENSE = 1, OR_POST_CIRCULANT = 2 };

/* preprocess_solve(a, b, none, post, refine) (preprocess.hpp:156-180).
 * post_kind DENSE: post = n x n dense multiplier; CIRCULANT: post = first
 * column c of length n. history receives refine+1 entries. The factors of the
 * product are written to lu_out when non-null. */
int or_preprocess_solve(int64_t n, const double* a, const double* b, int post_kind, const double* post,
                        int64_t refine, double* x, double* history, int* diverged, int64_t* zero_step,
                        double* lu_out, double* product_out);

/* BASELINE config 2 driver: for i in [i0, i0+count): ts = base + i,
 * A_i = gen_gaussian(32,32,derive_seed(ts,1)), b_i = gen_gaussian_vector(32,
 * derive_seed(ts,2)), G_i = gen_gaussian(32,32,derive_seed(ts,3)); solve with
 * preprocess_solve(A_i, b_i, none, {Gaussian, derive_seed(ts,3)}, 0) on
 * `threads` threads (strided like parallel_for_index, parallel.hpp:14-35).
 * Any output pointer may be null. */
void or_batched_config2(int64_t dim, uint64_t base, int64_t i0, int64_t count, int threads, double* a_out,
                        double* g_out, double* b_out, double* x_out, double* resid_out, int64_t* status_out,
                        double* growth_out, double* lu_out);

/* Householder thin QR with positive diagonal and rank check (qr.hpp:21-47).
 * q: m x l, r: l x l. Returns OR_OK or OR_RANK_DEFICIENCY (*bad_col 1-based). */
int or_qr(int64_t m, int64_t l, const double* a, double* q, double* r, int64_t* bad_col);
/* singular values (non-increasing) of a row-major m x n matrix by one-sided
 * (Hestenes) Jacobi: the stand-in for Eigen's JacobiSVD/BDCSVD values
 * (svd.hpp:76-88), a third-party dependency absent here */
void or_singular_values(int64_t m, int64_t n, const double* a, double* out);

#ifdef __cplusplus
}
#endif

#endif
