/*
 * randla_capi.h — the drop-in boundary of the B200-native preprocessed-GENP /
 * randomized low-rank hot path (arXiv 1406.5802 reference `randla`).
 *
 * A plain C ABI: extern "C", plain pointers, int64 sizes, no C++ or torch
 * types. Each entry point replaces one function template of the reference's
 * header API (namespace randla, /root/reference/proj/include/randla/*.hpp,
 * `double` instantiation); the replaced interface is cited per entry.
 * The C++ header include/randla_b200/randla.hpp re-creates the reference
 * signatures (Matrix<double>, LuFactors, SolveOutcome, typed exceptions) on
 * top of this ABI, and INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Conventions
 *  - Matrices are row-major double, exactly as randla::Matrix
 *    (matrix.hpp:13-25). Packed LU: strictly-lower part = L (unit diagonal
 *    implied), upper part incl. diagonal = U; the reference's LuFactors
 *    (lu.hpp:17-28) is this buffer unpacked.
 *  - Every compute entry takes an rl_mem flag. RL_HOST: all array arguments
 *    are host pointers (pageable or pinned); the call stages them through the
 *    context's device workspace and returns when the outputs are back on the
 *    host. RL_DEVICE: all array arguments are device pointers; the call
 *    enqueues work on the context's stream and returns without a host
 *    synchronisation unless a verdict must be read back (noted per call).
 *  - Errors: the return code maps 1:1 onto the reference's exception types
 *    (types.hpp:44-78); the 1-based step / position / column of a
 *    ZeroPivotError / SingularPivotBlockError / RankDeficiencyError is
 *    returned through the call's info struct. rl_last_error() gives the
 *    message (thread-local).
 *  - Contexts: one rl_context owns a device, a CUDA stream and a grow-only
 *    device workspace. A context must not be used by two threads at once;
 *    passing ctx = NULL selects a per-thread default context, so concurrent
 *    callers (the reference's parallel_for_index workers,
 *    parallel.hpp:24-30) are safe without locking.
 *  - There is no CPU fallback: with no CUDA device every compute entry
 *    returns RL_ERR_NO_DEVICE.
 */
#ifndef RANDLA_CAPI_H
#define RANDLA_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define RL_API __attribute__((visibility("default")))
#else
#define RL_API
#endif

#define RL_ABI_VERSION 1

typedef enum rl_status {
    RL_OK = 0,
    RL_ERR_DIMENSION = 1,             /* randla::DimensionError            types.hpp:44-46 */
    RL_ERR_ZERO_PIVOT = 2,            /* randla::ZeroPivotError{step}      types.hpp:56-62 */
    RL_ERR_SINGULAR_PIVOT_BLOCK = 3,  /* randla::SingularPivotBlockError   types.hpp:64-68 */
    RL_ERR_RANK_DEFICIENCY = 4,       /* randla::RankDeficiencyError       types.hpp:52-54 */
    RL_ERR_LOGIC = 5,                 /* std::logic_error (imaginary dust) circulant.hpp:63-64 */
    RL_ERR_SINGULAR_MATRIX = 6,       /* randla::SingularMatrixError       types.hpp:48-50 */
    RL_ERR_CUDA = 10,
    RL_ERR_NO_DEVICE = 11,
    RL_ERR_OUT_OF_MEMORY = 12,
    RL_ERR_INVALID_ARGUMENT = 13,
    RL_ERR_UNSUPPORTED = 14
} rl_status;

typedef enum rl_mem { RL_HOST = 0, RL_DEVICE = 1 } rl_mem;

/* Multiplier families on the path (multipliers.hpp:20-40). GAUSSIAN_CIRCULANT
 * is RealCirculant(gen_gaussian_vector(n, seed)) — the "Gaussian circulant"
 * of BASELINE configs 3 and 5 (SURVEY §0 finding 2); REAL_CIRCULANT is the
 * reference's own uniform[-1,1] family gen_real_circulant (multipliers.hpp:67-73). */
typedef enum rl_multiplier_kind {
    RL_MULT_NONE = 0,
    RL_MULT_GAUSSIAN = 1,
    RL_MULT_REAL_CIRCULANT = 2,
    RL_MULT_GAUSSIAN_CIRCULANT = 3
} rl_multiplier_kind;

/* A multiplier: drawn from `seed` by the reference's generator
 * (MultiplierSpec, multipliers.hpp:33-40), or supplied explicitly: `dense`
 * (n x n, row-major) for GAUSSIAN, `column` (first column, length n) for the
 * circulant kinds. Explicit buffers live in the call's rl_mem space. */
typedef struct rl_multiplier {
    int32_t kind; /* rl_multiplier_kind */
    uint64_t seed;
    const double* dense;
    const double* column;
} rl_multiplier;

/* Outcome of one preprocessed solve / factorization. */
typedef struct rl_solve_info {
    int64_t zero_pivot_step;     /* 1-based ZeroPivotError step, 0 = none */
    double residual_history[8];  /* ||Ax-b||/||b|| after the solve and each refinement step
                                    (SolveOutcome::residual_history, preprocess.hpp:9-13) */
    int32_t history_len;
    int32_t diverged;            /* SolveOutcome::diverged (preprocess.hpp:129-141) */
    double residual_rel_a;       /* ||Ax-b|| / (||A||_est ||x||), BASELINE config 1 form;
                                    ||A||_est = spectral_norm_estimate(A) when requested, else 0 */
    double growth;               /* max|U| / max|AG|  (SURVEY App. A definition) */
    double min_abs_pivot;        /* min_j |u_jj| */
    double max_abs_product;      /* max|AG| */
    double max_abs_u;            /* max|U| */
    double norm_floor;           /* largest row/column norm of AG (norms.hpp:38-50) */
    double norm_frobenius;       /* ||AG||_F, upper bound of the estimate */
    double norm_estimate;        /* spectral_norm_estimate(AG) when evaluated, else 0 */
    int32_t norm_estimate_evaluated; /* 1 when the verdict needed the power iteration */
    int32_t reserved;
    double pivot_tolerance;      /* tol_pivot(n) * norm used for the verdict (upper bound when lazy) */
    double stage_ms[4];          /* device time (CUDA events on the context stream): product A*H,
                                    factor + verdict, chain solve + refinement, whole call */
} rl_solve_info;

/* Per-batch summary of rl_batched_genp_solve_32. */
typedef struct rl_batch_summary {
    int64_t zero_pivots;         /* systems whose verdict was ZeroPivot */
    int64_t norm_estimates;      /* systems that needed the power iteration */
    double max_growth;
    double max_residual;
    double mean_residual;
} rl_batch_summary;

typedef struct rl_context rl_context;

/* ---- context / runtime ---------------------------------------------- */
RL_API int rl_abi_version(void);
RL_API const char* rl_last_error(void);
RL_API rl_status rl_context_create(int device, rl_context** out);
RL_API rl_status rl_context_destroy(rl_context* ctx);
/* enqueue on an external cudaStream_t (e.g. torch.cuda.current_stream()); NULL selects the
 * legacy default stream. A new context uses its own non-blocking stream. */
RL_API rl_status rl_context_set_stream(rl_context* ctx, void* cuda_stream);
RL_API void* rl_context_get_stream(rl_context* ctx);
RL_API rl_status rl_synchronize(rl_context* ctx);
/* number of kernels this library has launched in this process */
RL_API int64_t rl_kernel_launches(void);
/* number of host threads used by the exact multiplier generator (0 = all cores) */
RL_API void rl_set_host_threads(int threads);

/* ---- seeded multipliers (host, bit-exact to the reference) ----------- */
/* derive_seed (multipliers.hpp:54-56) */
RL_API uint64_t rl_derive_seed(uint64_t seed, uint64_t k1, uint64_t k2);
/* hash_label (rng.hpp:87-95) */
RL_API uint64_t rl_hash_label(const char* label);
/* gen_gaussian(m, n, seed) (multipliers.hpp:58-65); gen_gaussian_vector = n x 1
 * (testbed/inputs.hpp:85-90). Host buffer. Parallel, bit-identical. */
RL_API rl_status rl_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double* out);
/* `count` independent gen_gaussian(m, n, seeds[i]) into out[i*m*n ...] */
RL_API rl_status rl_gen_gaussian_batch(int64_t count, int64_t m, int64_t n, const uint64_t* seeds, double* out);
/* gen_gaussian(m, n, seed) generated on the device into `out` (device, leading
 * dimension ld >= n), bit-identical to rl_gen_gaussian: the polar method runs on
 * the GPU; the ~6% of log(s) evaluations too close to a rounding boundary to
 * match glibc by construction are finished on the host with glibc. Synchronises
 * the context stream. hard_cases (nullable) = attempts finished on the host. */
RL_API rl_status rl_gen_gaussian_device(rl_context* ctx, int64_t m, int64_t n, uint64_t seed, double* out, int64_t ld,
                                        int64_t* hard_cases);
/* gen_real_circulant first column (multipliers.hpp:67-73) */
RL_API rl_status rl_gen_real_circulant_column(int64_t n, uint64_t seed, double* out);

/* ---- dense products ---------------------------------------------------- */
/* C = A B (m x k times k x n, row-major, leading dimensions in elements);
 * replaces matmul (matrix.hpp:115-121). FP64 DMMA tiles. */
RL_API rl_status rl_dgemm(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, int64_t k, const double* a,
                          int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc);
/* spectral_norm_estimate (norms.hpp:35-78) */
RL_API rl_status rl_spectral_norm_estimate(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                           double* out);

/* ---- GENP -------------------------------------------------------------- */
/* genp_factor (lu.hpp:40-58): packed LU of a (n x n); RL_ERR_ZERO_PIVOT with
 * info->zero_pivot_step on a pivot <= tol_pivot(n) * spectral_norm_estimate(a).
 * The verdict is read back to the host (synchronises the stream). */
RL_API rl_status rl_genp_factor(rl_context* ctx, rl_mem mem, int64_t n, const double* a, double* lu,
                                rl_solve_info* info);
/* lu_solve (lu.hpp:100-123) on packed factors */
RL_API rl_status rl_lu_solve(rl_context* ctx, rl_mem mem, int64_t n, const double* lu, const double* b, double* x);

/* ---- block elimination (block_ge.hpp), the reference's arithmetic order -- */
/* gepp_factor (lu.hpp:62-98): packed L\U with partial pivoting (first maximal
 * |u_ij|), perm[i] = original row at position i; RL_ERR_SINGULAR_MATRIX with
 * *singular_step (1-based) when the best pivot <= tol_pivot(n) *
 * spectral_norm_estimate(a). Bit-identical to the reference. */
RL_API rl_status rl_gepp_factor(rl_context* ctx, rl_mem mem, int64_t n, const double* a, double* lu, int64_t* perm,
                                int64_t* singular_step);
/* lu_solve (lu.hpp:100-123) or, transpose != 0, lu_solve_transpose
 * (lu.hpp:127-147) with GEPP factors, for nrhs right-hand sides: the columns
 * of the n x nrhs row-major b; x likewise (x must not alias b) */
RL_API rl_status rl_gepp_solve(rl_context* ctx, rl_mem mem, int64_t n, int64_t nrhs, const double* lu,
                               const int64_t* perm, const double* b, double* x, int32_t transpose);
/* block_ge_factor(a, split) (block_ge.hpp:168-181): split = pivot block sizes
 * in elimination order (sum n). The right-spine factorisation is returned
 * flat: level at offset o with block size k holds its leaf's packed GEPP
 * factors in factors[o:o+k, o:o+k], B^-1 C in factors[o:o+k, o+k:n], D B^-1 in
 * factors[o+k:n, o:o+k], the leaf's local permutation in perm[o:o+k].
 * leaf_blocks (nullable, n x n): each leaf's block matrix (the Schur complement
 * it factors) on its diagonal block. RL_ERR_DIMENSION on a bad split;
 * RL_ERR_SINGULAR_PIVOT_BLOCK with *position = offset + 1 when
 * svd_values(B).back() <= tol_pivot(n) * spectral_norm_estimate(a);
 * RL_ERR_SINGULAR_MATRIX from a leaf's GEPP. */
RL_API rl_status rl_block_ge_factor(rl_context* ctx, rl_mem mem, int64_t n, const double* a, int64_t nsplit,
                                   const int64_t* split, double* factors, int64_t* perm, double* leaf_blocks,
                                   int64_t* position);
/* block_solve (block_ge.hpp:198-201) on rl_block_ge_factor's output */
RL_API rl_status rl_block_solve(rl_context* ctx, rl_mem mem, int64_t n, int64_t nsplit, const int64_t* split,
                               const double* factors, const int64_t* perm, const double* b, double* x);

/* preprocess_solve(a, b, none, post, refine_steps) (preprocess.hpp:156-180):
 * product = A*H (dense GEMM or circulant FFT), GENP, chain solve
 * x = H (LU)^-1 b, refinement. lu_out (n x n, nullable) receives the packed
 * factors of the product. want_norm_a != 0 also evaluates
 * spectral_norm_estimate(A) for info->residual_rel_a. */
RL_API rl_status rl_preprocessed_genp_solve(rl_context* ctx, rl_mem mem, int64_t n, const double* a,
                                            const double* b, const rl_multiplier* post, int64_t refine_steps,
                                            double* x, double* lu_out, int32_t want_norm_a, rl_solve_info* info);

/* BASELINE config 2: `batch` independent 32x32 systems, each
 * preprocess_solve(A_i, b_i, none, {Gaussian, G_i}, 0). a, g: batch x 32 x 32;
 * b, x: batch x 32; lu: batch x 32 x 32 (nullable); resid: ||A_i x_i - b_i||/||b_i||;
 * growth: max|U_i|/max|A_i G_i|; status: 0 or the 1-based ZeroPivot step
 * (x, resid, growth are NaN for such systems). One warp per system. */
RL_API rl_status rl_batched_genp_solve_32(rl_context* ctx, rl_mem mem, int64_t batch, const double* a,
                                          const double* g, const double* b, double* lu, double* x, double* resid,
                                          double* growth, int32_t* status, rl_batch_summary* summary);

/* ---- structured multipliers (FFT) -------------------------------------- */
/* matmul_by_circulant(A, C(c)) (circulant.hpp:171-185): A m x n, c length n */
RL_API rl_status rl_circulant_right_multiply(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                             const double* c, double* out);
/* matmul_by_toeplitz_block(A, ToeplitzBlock(C(c), k, l)) (circulant.hpp:187-203):
 * A m x k, c parent column length np >= k, out m x l */
RL_API rl_status rl_toeplitz_right_multiply(rl_context* ctx, rl_mem mem, int64_t m, int64_t k, const double* a,
                                            int64_t np, const double* c, int64_t l, double* out);

/* ---- low-rank ----------------------------------------------------------- */
/* orthonormal_basis (qr.hpp:51-54) by CholeskyQR2: q (m x l) with positive
 * diag R; RL_ERR_RANK_DEFICIENCY (info column) per qr.hpp:33-38. r nullable. */
RL_API rl_status rl_cholqr2(rl_context* ctx, rl_mem mem, int64_t m, int64_t l, const double* y, double* q,
                            double* r, int64_t* bad_column);
/* range_find + approximation residual (lowrank.hpp:62-83, :99-102):
 * Y = A H (H: n x l Gaussian(seed) or Toeplitz block of a Gaussian circulant
 * of parent length n), Q = orthonormal_basis(Y), residual R = A - Q (Q^T A).
 * Outputs: q (m x l, nullable), frobenius = ||R||_F, spectral = ||R||_2 by
 * the restated power iteration (norms.hpp:52-77). */
typedef struct rl_lowrank_info {
    double residual_frobenius;
    double residual_spectral;
    int64_t rank_deficient_column; /* 0 = none */
    int32_t power_iterations;
    int32_t reserved;
} rl_lowrank_info;
RL_API rl_status rl_range_find_residual(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                        int64_t l, const rl_multiplier* h, double* q, rl_lowrank_info* info);

#ifdef __cplusplus
}
#endif

#endif /* RANDLA_CAPI_H */
