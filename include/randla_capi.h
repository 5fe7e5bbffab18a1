/*
 * randla_capi.h — the drop-in boundary of the B200-native preprocessed-GENP /
 * randomized low-rank hot path (arXiv 1406.5802 reference `randla`).
 *
 * A plain C ABI: extern "C", plain pointers, int64 sizes, no C++ or torch
 * types. Each entry point replaces one function template of the reference's
 * header API (namespace randla, /root/reference/proj/include/randla/<name>.hpp,
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

#define RL_ABI_VERSION 2

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

/* Multiplier families: the ordinals of randla::MultiplierKind
 * (multipliers.hpp:20-29), one for one. In this real (double) pipeline the
 * complex families (UNITARY_CIRCULANT, SRFT, TOEPLITZ_BLOCK with the UNITARY
 * variant) are rejected with RL_ERR_DIMENSION exactly where the reference's
 * real instantiation throws DimensionError("complex multiplier family
 * requested in a real pipeline") (preprocess.hpp:39-53, multipliers.hpp:174-218,
 * lowrank.hpp:71-78).
 * RL_MULT_GAUSSIAN_CIRCULANT is an extension outside the reference's ordinal
 * range: RealCirculant(gen_gaussian_vector(n, seed)), the "circulant with an
 * N(0,1) first column" of BASELINE configs 3 and 5 (the reference's own
 * RealCirculant family draws the column uniform on [-1, 1],
 * multipliers.hpp:67-73); it behaves as RealCirculant / the real ToeplitzBlock
 * everywhere else. */
typedef enum rl_multiplier_kind {
    RL_MULT_NONE = 0,
    RL_MULT_GAUSSIAN = 1,
    RL_MULT_REAL_CIRCULANT = 2,
    RL_MULT_UNITARY_CIRCULANT = 3,
    RL_MULT_TOEPLITZ_BLOCK = 4,
    RL_MULT_SRFT = 5,
    RL_MULT_FINITE_SET_UNIFORM = 6,
    RL_MULT_CIRC_SKEW_PRODUCT = 7,
    RL_MULT_GAUSSIAN_CIRCULANT = 100
} rl_multiplier_kind;

/* randla::ToeplitzVariant (multipliers.hpp:31) */
typedef enum rl_toeplitz_variant { RL_TOEPLITZ_REAL = 0, RL_TOEPLITZ_UNITARY = 1 } rl_toeplitz_variant;

/* A multiplier spec (randla::MultiplierSpec, multipliers.hpp:33-40; rows and
 * cols come from the call: n x n for preprocessing, n x l for sketching).
 * Drawn from `seed` by the reference's generator, or supplied explicitly:
 * `dense` (rows x cols, row-major) for the dense kinds, `column` (first
 * column of the circulant, length n) for the circulant kinds. Explicit buffers
 * live in the call's rl_mem space. set_cardinality 0 means the reference's
 * default 65536. */
typedef struct rl_multiplier {
    int32_t kind;             /* rl_multiplier_kind */
    int32_t variant;          /* rl_toeplitz_variant (TOEPLITZ_BLOCK only) */
    uint64_t seed;
    uint64_t set_cardinality; /* FINITE_SET_UNIFORM only */
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
    /* in: optional caller buffer for the whole residual history (refine_steps + 1 entries;
       residual_history above keeps the first 8). Required when refine_steps > 7. */
    double* history;
    int64_t history_capacity;
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
/* the CUDA device a context (NULL: the calling thread's default context, which
 * is the one for the thread's current device, cudaGetDevice) runs on; -1 when
 * there is no device */
RL_API int rl_context_device(rl_context* ctx);

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
/* gen_finite_set_uniform(m, n, seed, cardinality) (multipliers.hpp:142-154):
 * entries uniform over {-floor(card/2), ..., ceil(card/2) - 1}, next_below
 * rejection sampling (rng.hpp:46-53); RL_ERR_DIMENSION for cardinality < 2 */
RL_API rl_status rl_gen_finite_set_uniform(int64_t m, int64_t n, uint64_t seed, uint64_t cardinality, double* out);
/* materialize(spec) of a real family with rows x cols (multipliers.hpp:174-218)
 * into out (row-major, ld = cols): the dense multiplier the reference would
 * build. Host or device output per `mem`; circulant and skew-product families
 * are expanded on the device. */
RL_API rl_status rl_materialize(rl_context* ctx, rl_mem mem, const rl_multiplier* spec, int64_t rows, int64_t cols,
                                double* out);

/* ---- dense products ---------------------------------------------------- */
/* C = A B (m x k times k x n, row-major, leading dimensions in elements);
 * replaces matmul (matrix.hpp:115-121). FP64 DMMA tiles. */
RL_API rl_status rl_dgemm(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, int64_t k, const double* a,
                          int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc);
/* svd_values (svd.hpp:76-88): the min(m, n) singular values of a (m x n),
 * non-increasing, by one-sided Jacobi on the device (the reference calls
 * Eigen's JacobiSVD / BDCSVD: equal up to rounding). One CTA: meant for the
 * small matrices the reference's checks use, not for the hot path. */
RL_API rl_status rl_singular_values(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a, double* out);
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

/* preprocess_solve(a, b, pre, post, refine_steps) (preprocess.hpp:156-180):
 * product = F (A H) with F = SideMultiplier::make(pre), H = make(post)
 * (preprocess.hpp:27-60: dense kinds by the DMMA GEMM, circulant kinds
 * structured through the FFT kernel), GENP, chain solve x = H (LU)^-1 (F b),
 * refinement. pre / post NULL = None. lu_out (n x n, nullable) receives the
 * packed factors of the product. want_norm_a != 0 also evaluates
 * spectral_norm_estimate(A) for info->residual_rel_a. */
RL_API rl_status rl_preprocessed_genp_solve(rl_context* ctx, rl_mem mem, int64_t n, const double* a,
                                            const double* b, const rl_multiplier* pre, const rl_multiplier* post,
                                            int64_t refine_steps, double* x, double* lu_out, int32_t want_norm_a,
                                            rl_solve_info* info);

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
/* circulant_apply(C(c), x) (circulant.hpp:91-96): y = C x for real c, x, with
 * the reference's imaginary-part check (RL_ERR_LOGIC, circulant.hpp:57-66) */
RL_API rl_status rl_circulant_apply(rl_context* ctx, rl_mem mem, int64_t n, const double* c, const double* x,
                                    double* y);
/* fft / inverse_fft (fft.hpp:76-98) on `count` complex vectors of length n,
 * in place, interleaved (re, im) doubles: forward multiplies by
 * Omega = (omega^{jk}), omega = exp(+2 pi i / n) — the reference's sign —
 * inverse by Omega^-1 = Omega^H / n. Power-of-two lengths run a radix FFT,
 * other lengths the dense O(n^2) transform as the reference does. */
RL_API rl_status rl_fft(rl_context* ctx, rl_mem mem, int64_t count, int64_t n, double* z, int32_t inverse);

/* ---- low-rank ----------------------------------------------------------- */
/* orthonormal_basis (qr.hpp:51-54) by CholeskyQR2: q (m x l) with positive
 * diag R; RL_ERR_RANK_DEFICIENCY (info column) per qr.hpp:33-38. r nullable. */
RL_API rl_status rl_cholqr2(rl_context* ctx, rl_mem mem, int64_t m, int64_t l, const double* y, double* q,
                            double* r, int64_t* bad_column);
/* orthonormal_basis_unchecked (qr.hpp:58-76), real: the basis without the rank verdict */
RL_API rl_status rl_orthonormal_basis_unchecked(rl_context* ctx, rl_mem mem, int64_t m, int64_t l, const double* y,
                                                double* q);
/* Low-rank outcome: the residual R = A - Q (Q^T A) (lowrank.hpp:35-37) in
 * Frobenius and spectral norm (||R||_2 by the restated power iteration of
 * norms.hpp:52-77 on the implicit operator R), the 1-based rank-deficient
 * column of qr (qr.hpp:33-38), 0 = none. */
typedef struct rl_lowrank_info {
    double residual_frobenius;
    double residual_spectral;
    int64_t rank_deficient_column; /* 0 = none */
    int32_t power_iterations;
    int32_t reserved;
} rl_lowrank_info;
/* range_find(a, r, p, spec, power_steps) (lowrank.hpp:62-83) with l = r + p:
 * the sketch Y = A H for H = the spec's n x l multiplier (ToeplitzBlock
 * through the FFT, everything else materialized and multiplied by the DMMA
 * GEMM, as the reference does), power_steps alternating products
 * Y <- A (A^T Y) (lowrank.hpp:51-57), Q = orthonormal_basis(Y) (CholeskyQR2,
 * qr.hpp:51-54) into q (m x l). */
RL_API rl_status rl_range_find(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a, int64_t l,
                               const rl_multiplier* h, int64_t power_steps, double* q, rl_lowrank_info* info);
/* approximation_residual(a, result) (lowrank.hpp:99-102) for a given A (m x n)
 * and basis Q (m x l): residual norms of R = A - Q (Q^T A) into info. */
RL_API rl_status rl_approximation_residual(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                           int64_t l, const double* q, rl_lowrank_info* info);
/* range_find followed by approximation_residual on the same resident A (one
 * call, one upload of A): the BASELINE config 4/5 pipeline. q nullable. */
RL_API rl_status rl_range_find_residual(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                        int64_t l, const rl_multiplier* h, int64_t power_steps, double* q,
                                        rl_lowrank_info* info);

/* ---- the complex field (Matrix<Complex>) -----------
 * Complex arrays are interleaved (re, im) doubles, row-major — the layout of
 * std::complex<double>. Multiplier specs take every MultiplierKind: the
 * complex families (UNITARY_CIRCULANT, TOEPLITZ_BLOCK with RL_TOEPLITZ_UNITARY,
 * SRFT) are drawn from `seed` by the reference's recipes
 * (multipliers.hpp:75-138); explicit `dense` / `column` buffers are real. */

/* preprocess_solve<Complex>(a, b, pre, post, refine_steps) (preprocess.hpp:156-180,
 * SideMultiplier<Complex>::make :27-60): circulant kinds (real or unitary,
 * either Toeplitz variant) stay structured through the FFT, the others are
 * dense (SRFT complex). a, lu_out: n x n; b, x: n (all complex). info as for
 * rl_preprocessed_genp_solve (moduli for growth and pivots; stage_ms unset). */
RL_API rl_status rl_zpreprocessed_genp_solve(rl_context* ctx, rl_mem mem, int64_t n, const double* a,
                                             const double* b, const rl_multiplier* pre, const rl_multiplier* post,
                                             int64_t refine_steps, double* x, double* lu_out, rl_solve_info* info);
/* range_find<Complex>(a, r, p, spec, power_steps) (lowrank.hpp:51-83) with
 * l = r + p, then approximation_residual on the same A (lowrank.hpp:99-102):
 * a m x n complex, q m x l complex (nullable). Q has orthonormal columns and
 * positive real R diagonal (qr.hpp:33-45). */
RL_API rl_status rl_zrange_find_residual(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                         int64_t l, const rl_multiplier* h, int64_t power_steps, double* q,
                                         rl_lowrank_info* info);
/* residual norms of A - Q Q^H A for a given complex A (m x n) and Q (m x l) */
RL_API rl_status rl_zapproximation_residual(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                            int64_t l, const double* q, rl_lowrank_info* info);
/* materialize<Complex>(spec) (multipliers.hpp:174-218): out rows x cols complex */
RL_API rl_status rl_zmaterialize(rl_context* ctx, rl_mem mem, const rl_multiplier* spec, int64_t rows, int64_t cols,
                                 double* out);
/* first column of gen_unitary_circulant(n, seed) (multipliers.hpp:75-82),
 * inverse_fft of the unit spectrum: n complex */
RL_API rl_status rl_gen_unitary_circulant(rl_context* ctx, rl_mem mem, int64_t n, uint64_t seed, double* column);
/* srft_columns(n, l, seed) (multipliers.hpp:132-138): l sorted indices (host) */
RL_API rl_status rl_srft_columns(int64_t n, int64_t l, uint64_t seed, int64_t* out);
/* svd_values of a complex m x n matrix (svd.hpp:76-88), non-increasing */
RL_API rl_status rl_zsingular_values(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a, double* out);
/* srft_sketch_check (lowrank.hpp:200-261) on a real m x n `a` */
typedef struct rl_srft_check {
    double residual;      /* ||(I - P_Y) A|| (spectral_norm_estimate) */
    double bound;         /* sqrt(1 + 7 n / l) sigma_{r+1} */
    int64_t sketch_width; /* l */
    int32_t clamped;      /* the prescribed width reached n and was cut back */
    int32_t reserved;
} rl_srft_check;
/* variant 0 = SketchVariant::Srft, 1 = CirculantPermutation; known_sigma_r1 < 0
 * (or NaN) evaluates svd_values(a)[r] */
RL_API rl_status rl_srft_sketch_check(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a, int64_t r,
                                      uint64_t seed, int32_t variant, double known_sigma_r1, rl_srft_check* out);
/* matmul_by_circulant / matmul_by_toeplitz_block (circulant.hpp:171-203) over
 * the complex field: A (m x k) times the leading k x l block of the np-point
 * circulant with complex first column c (length np), out m x l */
RL_API rl_status rl_zcirculant_right_multiply(rl_context* ctx, rl_mem mem, int64_t m, int64_t k, const double* a,
                                              int64_t np, const double* c, int64_t l, double* out);
/* circulant_apply(C(c), x) (circulant.hpp:81-98), complex c, x, y (length n) */
RL_API rl_status rl_zcirculant_apply(rl_context* ctx, rl_mem mem, int64_t n, const double* c, const double* x,
                                     double* y);
/* genp_factor<Complex> (lu.hpp:40-58): packed L\U (n x n complex), with the
 * reference's ZeroPivot verdict (info->zero_pivot_step) */
RL_API rl_status rl_zgenp_factor(rl_context* ctx, rl_mem mem, int64_t n, const double* a, double* lu,
                                 rl_solve_info* info);
/* lu_solve<Complex> (lu.hpp:100-122) on packed GENP factors: x = U^-1 L^-1 b */
RL_API rl_status rl_zlu_solve(rl_context* ctx, rl_mem mem, int64_t n, const double* lu, const double* b, double* x);
/* orthonormal_basis<Complex> (qr.hpp:51-54; unchecked != 0: orthonormal_basis_unchecked,
 * qr.hpp:58-76): q (m x l) with positive real R diagonal; bad (nullable)
 * receives the 1-based rank-deficient column */
RL_API rl_status rl_zorthonormal_basis(rl_context* ctx, rl_mem mem, int64_t m, int64_t l, const double* y, double* q,
                                       int32_t unchecked, int64_t* bad);
/* matmul<Complex> (matrix.hpp:115-121): c (m x n) = a (m x k) b (k x n) */
RL_API rl_status rl_zgemm(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, int64_t k, const double* a,
                          const double* b, double* c);
/* `count` next_gaussian draws of RngStream(seed).derived(key) (rng.hpp:20-24),
 * the probe vectors of posterior_estimate (lowrank.hpp:177-196) (host) */
RL_API rl_status rl_gen_gaussian_derived(uint64_t seed, uint64_t key, int64_t count, double* out);
/* the unit roots polar(1, 2 pi k / n), k < n (fft.hpp:21-30, multipliers.hpp:98-100),
 * rounded as the reference's host code: n complex (host) */
RL_API rl_status rl_unit_roots(int64_t n, double* out);

#ifdef __cplusplus
}
#endif

#endif /* RANDLA_CAPI_H */
