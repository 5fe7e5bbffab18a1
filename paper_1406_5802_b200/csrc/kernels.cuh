// Internal (C++) interface between the translation units of librandla_b200:
// device-pointer building blocks the C-ABI entry points compose.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <vector>

#include "runtime.cuh"

namespace rl {

// Running statistics a GEMM epilogue can fold over its output tile: sum of
// squares (for ||C||_F) and max |C| (bit pattern of a non-negative double).
struct GemmStats {
    double sumsq;
    unsigned long long maxabs_bits;
};

// C = alpha * A B + (accumulate ? C : 0); row-major device matrices, leading
// dimensions in elements. FP64 DMMA tiles fed by TMA. stats (device, nullable)
// accumulates over the written C.
rl_status gemm(rl_context* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
               int64_t ldb, double* C, int64_t ldc, double alpha, bool accumulate, GemmStats* stats);
// B <- A B in place (B: M x N, ld ldb; A: M x M, M <= 128), e.g. U12 = L11^-1
// A12: a single tile row, so no CTA overwrites rows another still reads
rl_status gemm_inplace_b(rl_context* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, double* BC,
                         int64_t ldb);

// Split-K variant for small M x N with long K (Gram matrices, Q^T A): partial
// products per K-slice into `work` (>= gemm_splitk_work_bytes), then an
// ordered (deterministic) reduction into C.
rl_status gemm_splitk(rl_context* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                      int64_t ldb, double* C, int64_t ldc, double alpha, bool accumulate, int splits, void* work);
size_t gemm_splitk_work_bytes(int64_t M, int64_t N, int splits);

// Statistics of C - A B (||.||_F^2, max|.|) without storing it.
rl_status gemm_residual_stats(rl_context* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                              const double* B, int64_t ldb, const double* C, int64_t ldc, GemmStats* stats);

// In-place blocked GENP of the n x n row-major matrix `a` (ld = lda, even,
// 16-byte aligned) into its packed LU. piv_out / rinv_out (device, n) receive
// u_jj and 1/u_jj. No pivoting, no verdict (the caller decides it).
// fwd_b / fwd_y (device, n, optional): when the super-panel path runs, the
// forward substitution y = L^-1 b (lu.hpp:110-115) follows the panels on a side
// stream, hidden under the factorisation, and *fwd_done is set; the caller then
// needs only lu_solve_upper_device.
rl_status genp_inplace(rl_context* ctx, int64_t n, double* a, int64_t lda, double* piv_out, double* rinv_out,
                       const double* fwd_b = nullptr, double* fwd_y = nullptr, bool* fwd_done = nullptr);

// Triangular solves on packed LU (device): x = U^-1 L^-1 b (x may alias b).
// `rinv` (nullable) = 1/u_jj from genp_inplace; `work` >= lu_solve_work_bytes(n).
rl_status lu_solve_device(rl_context* ctx, int64_t n, const double* lu, int64_t ld, const double* rinv,
                          const double* b, double* x, void* work);
// x = U^-1 y only (the upper half of lu_solve_device; in place allowed)
rl_status lu_solve_upper_device(rl_context* ctx, int64_t n, const double* lu, int64_t ld, const double* rinv,
                                const double* y, double* x, void* work);
size_t lu_solve_work_bytes(int64_t n);

// y = A x (row-major m x n); y = b - A x when `residual` (b given).
rl_status gemv(rl_context* ctx, int64_t m, int64_t n, const double* a, int64_t lda, const double* x, double* y,
               const double* b_for_residual);

// sum of squares of a length-n vector into *out (device scalar)
rl_status sumsq(rl_context* ctx, int64_t n, const double* v, double* out);

// exact-order spectral_norm_estimate (norms.hpp:35-78) on the device; host result
rl_status spectral_norm_estimate_device(rl_context* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                                        double* out);

// out (m x l) = A (m x k) * leading k x l block of the np-point circulant with
// first column c (device); np a power of two <= 16384. spec_ws >= 16*np bytes.
rl_status circulant_rows(rl_context* ctx, int64_t m, int64_t k, const double* a, int64_t lda, int64_t np,
                         const double* c, int64_t l, double* out, int64_t ldo, void* spec_ws);

// batched complex transform of `count` contiguous n-point rows (interleaved
// re/im), in place on the device, the reference's +1 sign forward and 1/n on
// the inverse (fft.hpp:76-98); `work` (>= cfft_work_bytes) unless n is a
// power of two <= 8192
size_t cfft_work_bytes(int64_t count, int64_t n);
rl_status cfft_device(rl_context* ctx, int64_t count, int64_t n, double* z, bool inverse, double* work);

// dense expansion of the leading k x l block of the np-point circulant (device)
rl_status circulant_dense(rl_context* ctx, const double* c, int64_t np, int64_t k, int64_t l, double* h, int64_t ldh);
// whether circulant_rows handles parent length np
bool circulant_fft_ok(int64_t np);

// gen_gaussian(rows, cols, seed) into device memory (ld), bit-identical to the
// reference stream (rng_device.cu). begin() only enqueues work on ctx->stream;
// finish() synchronises it and completes the host-decided attempts.
struct GaussJob {
    rl_context* ctx = nullptr;
    int64_t rows = 0, cols = 0, ld = 0, count = 0, nb = 0, cap = 0;
    uint64_t seed = 0;
    double* out = nullptr;
    char* base = nullptr;
    int64_t *counts = nullptr, *offsets = nullptr, *pair = nullptr;
    unsigned long long* hcount = nullptr;
    uint64_t* attempts = nullptr;
    double* vals = nullptr;
    int64_t h_total = 0, h_hard = 0;  // host copies (pageable; valid after finish's sync)
    int64_t nb1 = 0;                    // gen runs as blocks [0, nb1) then [nb1, nb)
    cudaEvent_t ev1 = nullptr, ev2 = nullptr;  // after each half (with its hard-case count)
    rl_status begin(rl_context* ctx, int64_t rows, int64_t cols, uint64_t seed, double* out, int64_t ld);
    // first_rows_ready (optional) runs once rows [0, k) of the output are final
    // in stream order on ctx->stream (the first half's undecided attempts
    // scattered), while the host still finishes the second half's: work it
    // enqueues on ctx->stream that reads only those rows overlaps that host
    // work. The second half is then scattered on a side stream that
    // ctx->stream waits for.
    rl_status finish(int64_t* hard_cases, const std::function<rl_status(int64_t)>& first_rows_ready = nullptr);
    ~GaussJob();
};
rl_status gen_gaussian_device(rl_context* ctx, int64_t rows, int64_t cols, uint64_t seed, double* out, int64_t ld,
                              int64_t* hard_cases);

// ---- multiplier specs (multipliers.cu) ------------------------------------
// How a real-pipeline spec acts: not at all (identity), as a dense matrix (the
// DMMA GEMM), or as a circulant kept structured (the FFT kernel).
enum class MForm { NONE, DENSE, CIRC };
// SideMultiplier::make (preprocess.hpp:27-60) for an n x n side multiplier:
// RL_ERR_DIMENSION for the complex families (the reference's real pipeline
// throws DimensionError there), RL_ERR_INVALID_ARGUMENT for unknown kinds.
rl_status side_form(const rl_multiplier* m, MForm* out);
// range_find's sketch (lowrank.hpp:62-81) with an n x l multiplier: Toeplitz
// blocks (and the Gaussian-circulant extension) structured, the rest dense
// (materialize: None and RealCirculant need l == n).
rl_status sketch_form(const rl_multiplier* m, int64_t n, int64_t l, MForm* out);
// first column (host, length n) of a structured spec: the explicit column
// (host or device memory per `host`), gen_gaussian_vector(n, seed) for the
// Gaussian-circulant extension, else gen_real_circulant(n, seed)
// (multipliers.hpp:67-73, :84-86).
rl_status multiplier_column(const rl_multiplier* m, int64_t n, bool host, std::vector<double>& col);
// materialize(spec) with spec.rows = rows, spec.cols = cols
// (multipliers.hpp:174-218) into device memory (ld); an explicit `dense`
// buffer is copied (host or device per `host`). Enqueued on ctx->stream
// (the seeded Gaussian synchronises it).
rl_status materialize_device(rl_context* ctx, const rl_multiplier* m, int64_t rows, int64_t cols, bool host,
                             double* out, int64_t ld);
// out (cols x rows, ldo) = in^T (rows x cols, ldi), device
rl_status transpose_device(rl_context* ctx, const double* in, int64_t ldi, int64_t rows, int64_t cols, double* out,
                           int64_t ldo);

// stream-ordered device scratch freed at scope exit
struct StreamBuf {
    double* p = nullptr;
    cudaStream_t s;
    explicit StreamBuf(cudaStream_t st) : s(st) {}
    rl_status alloc(size_t bytes);
    ~StreamBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

// ---- low-rank building blocks (lowrank.cu) --------------------------------
// orthonormal_basis (qr.hpp:51-54) by CholeskyQR2 (shifted CholeskyQR3 on
// breakdown): Q (m x l, ldq) from Y (m x l, ldq), R (l x l, ldr, nullable).
// Options for callers that run it on a real embedding of a complex Y:
// rank_m / rank_l replace (m, l) in tol_rank, reported columns are divided
// by column_group, unchecked skips the verdict (orthonormal_basis_unchecked).
struct CholqrOpts {
    int64_t rank_m = 0, rank_l = 0;
    int64_t column_group = 1;
    bool unchecked = false;
};
rl_status cholqr2_device(rl_context* ctx, int64_t m, int64_t l, const double* y, double* q, int64_t ldq, double* r,
                         int64_t ldr, int64_t* bad_column, const CholqrOpts* opts = nullptr);
// ||A - Q (Q^T A)||_F and ||.||_2 (power iteration) into info (lowrank.hpp:99-102)
rl_status residual_core(rl_context* ctx, int64_t m, int64_t n, const double* A, int64_t ldA, int64_t l,
                        const double* Q, int64_t ldq, rl_lowrank_info* info);

// batched 32x32 kernel (batched32.cu)
rl_status launch_batched_genp32(rl_context* ctx, int64_t batch, const double* a, const double* g, const double* b,
                                double* lu, double* x, double* r, double* growth, int32_t* status, int refine,
                                void* fix_ws);
size_t batched_fix_workspace_bytes(int64_t batch);

}  // namespace rl
