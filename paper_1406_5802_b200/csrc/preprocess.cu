// C-ABI entry points of the dense path:
//   rl_preprocessed_genp_solve  preprocess_solve (preprocess.hpp:156-180)
//   rl_genp_factor              genp_factor      (lu.hpp:40-58)
//   rl_lu_solve                 lu_solve         (lu.hpp:100-123)
//   rl_spectral_norm_estimate   spectral_norm_estimate (norms.hpp:35-78)
//
// The pivot verdict (lu.hpp:44,49: first j with |u_jj| <= tol_pivot(n) *
// spectral_norm_estimate(product)) is decided without the power iteration in
// the common case: floor <= estimate <= ||product||_F (norms.hpp:38-50,77),
// so when every pivot exceeds tol_pivot(n) * ||product||_F the verdict is
// "no ZeroPivot". Only when some pivot falls at or below that bound is the
// estimate evaluated, in the reference's exact summation order, on a
// recomputed product (the GEMM is deterministic, so it is bit-identical).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "device_common.cuh"
#include "kernels.cuh"

extern "C" RL_API rl_status rl_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double* out);
extern "C" RL_API rl_status rl_gen_real_circulant_column(int64_t n, uint64_t seed, double* out);

namespace rl {
namespace {

__global__ void pivot_scan_kernel(const double* __restrict__ piv, int64_t n, double tol, double* __restrict__ out_min,
                                  unsigned long long* __restrict__ out_first) {
    __shared__ double smin[32];
    __shared__ unsigned long long sfirst[32];
    double mn = INFINITY;
    unsigned long long first = ~0ull;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double a = fabs(piv[i]);
        mn = fmin(mn, a);
        if (!(a > tol) && static_cast<unsigned long long>(i) < first) first = static_cast<unsigned long long>(i);
    }
    mn = warp_min(mn);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long f = __shfl_xor_sync(kFull, first, o);
        first = f < first ? f : first;
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        smin[w] = mn;
        sfirst[w] = first;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) {
            mn = fmin(mn, smin[i]);
            first = sfirst[i] < first ? sfirst[i] : first;
        }
        *out_min = mn;
        *out_first = first;
    }
}

// sum of squares and max |.| over a rows x cols matrix (one block per row);
// upper_only restricts row i to columns >= i (max |U| of a packed LU)
__global__ void matrix_stats_kernel(const double* __restrict__ a, int64_t ld, int64_t cols, bool upper_only,
                                    GemmStats* __restrict__ out) {
    const int64_t row = blockIdx.x;
    double s = 0.0, m = 0.0;
    for (int64_t k = (upper_only ? row : 0) + threadIdx.x; k < cols; k += blockDim.x) {
        const double v = a[row * ld + k];
        s = fma(v, v, s);
        m = fmax(m, fabs(v));
    }
    s = warp_sum(s);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) {
        if (!upper_only) atomicAdd(&out->sumsq, s);
        atomicMax(&out->maxabs_bits, static_cast<unsigned long long>(__double_as_longlong(m)));
    }
}

__global__ void axpy_kernel(double* __restrict__ x, const double* __restrict__ d, int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] += d[i];
}

struct Scalars {
    GemmStats prod;   // ||product||_F^2, max|product|
    GemmStats upper;  // max|U|
    double pivmin;
    unsigned long long first;
    double bsq[66];   // sumsq scratch, result at [0]
    double rsq[66];
};

double bits_to_double(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}

unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

// CUDA-event stage timer on the context stream (rl_solve_info::stage_ms)
struct StageTimer {
    cudaStream_t s;
    cudaEvent_t ev[5] = {};
    int n = 0;
    explicit StageTimer(cudaStream_t st) : s(st) {}
    void mark() {
        if (n < 5 && cudaEventCreate(&ev[n]) == cudaSuccess) cudaEventRecord(ev[n++], s);
    }
    void fill(double* out) {  // out[0..2] consecutive stages, out[3] total
        if (n == 0) return;
        cudaEventSynchronize(ev[n - 1]);
        for (int i = 0; i + 1 < n && i < 3; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            out[i] = ms;
        }
        float tot = 0.f;
        cudaEventElapsedTime(&tot, ev[0], ev[n - 1]);
        out[3] = tot;
    }
    ~StageTimer() {
        for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
    }
};

enum PostKind { POST_NONE, POST_DENSE, POST_CIRC };

struct Dense {
    int64_t n = 0, ld = 0;
    PostKind post = POST_NONE;
    double* c = nullptr;   // circulant first column (device)
    double* ct = nullptr;  // transposed circulant's first column c[(n-i) mod n]
    void* spec = nullptr;  // FFT spectrum workspace (16 n bytes)
    // left multiplier F of F (A H) (preprocess.hpp:164): dense n x n, or a
    // circulant kept structured (its transpose's first column fct, spectrum
    // workspace fspec); fr = F r for the chain solver
    PostKind pre = POST_NONE;
    double* F = nullptr;
    double* fct = nullptr;
    void* fspec = nullptr;
    double* fr = nullptr;
    double *A = nullptr, *G = nullptr, *P = nullptr;
    double *b = nullptr, *x = nullptr, *r = nullptr, *y = nullptr, *d = nullptr, *piv = nullptr, *rinv = nullptr;
    void* solve_work = nullptr;
    // y = L^-1 b already formed under the factorisation (genp_inplace's side stream)
    bool fwd_done = false;
    Scalars* sc = nullptr;
    // host-mode pipelining: A arrives in a_chunks row blocks of a_chunk_rows,
    // block c resident once a_ready[c] has fired (0 chunks: A fully resident)
    int a_chunks = 0;
    int64_t a_chunk_rows = 0;
    cudaEvent_t* a_ready = nullptr;
    // A G split at K = k_split (a multiple of the GEMM's k-tile): columns
    // [0, k_split) of A times rows [0, k_split) of G first, then the rest
    // accumulated. A DMMA tile accumulates its k-steps in order in FP64 and C
    // round-trips exactly, so the sum is the unsplit product bit for bit. Used
    // when a seeded G is generated on the device: its first rows are final
    // while the host still finishes the rest (GaussJob::finish).
    int64_t k_split = 0;
    int part1_blocks = 0;  // row blocks whose first K-part is already enqueued
};

// P = A G (or A), blocked GENP in place, growth, verdict (lu.hpp:44-49).
// product P = A H by the multiplier's own method (deterministic: the rare
// exact-verdict path recomputes it bit for bit)
rl_status form_product(rl_context* ctx, Dense& D, double* P, GemmStats* stats) {
    const int64_t n = D.n;
    cudaStream_t s = ctx->stream;
    // with a left multiplier, A H lands in scratch T (or is A itself) and
    // F T is written to P; the verdict statistics belong to the final product
    StreamBuf tbuf(s);
    double* T = P;
    const bool left = D.pre != POST_NONE;
    if (left) {
        if (D.post == POST_NONE) {
            T = D.A;
        } else {
            rl_status st = tbuf.alloc(sizeof(double) * n * D.ld);
            if (st != RL_OK) return st;
            T = tbuf.p;
        }
    }
    GemmStats* ah_stats = left ? nullptr : stats;
    // row blocks of A (all of A when it is already resident); every block's
    // product rows are computed exactly as in one call (per-tile K order)
    const int chunks = D.a_chunks > 0 ? D.a_chunks : 1;
    const int64_t rows = D.a_chunks > 0 ? D.a_chunk_rows : n;
    for (int c = 0; c < chunks; ++c) {
        const int64_t r0 = c * rows, rc = std::min(rows, n - r0);
        if (rc <= 0) break;
        if (D.a_chunks > 0) RL_CUDA(cudaStreamWaitEvent(s, D.a_ready[c], 0));
        const double* Ac = D.A + r0 * D.ld;
        double* Tc = T + r0 * D.ld;
        rl_status st = RL_OK;
        if (D.post == POST_DENSE && D.k_split > 0) {
            const int64_t k1 = D.k_split;
            if (!(c < D.part1_blocks && Tc == D.P + r0 * D.ld))
                st = gemm(ctx, rc, n, k1, Ac, D.ld, D.G, D.ld, Tc, D.ld, 1.0, false, nullptr);
            if (st == RL_OK)
                st = gemm(ctx, rc, n, n - k1, Ac + k1, D.ld, D.G + k1 * D.ld, D.ld, Tc, D.ld, 1.0, true, ah_stats);
        } else if (D.post == POST_DENSE) {
            st = gemm(ctx, rc, n, n, Ac, D.ld, D.G, D.ld, Tc, D.ld, 1.0, false, ah_stats);
        } else if (D.post == POST_CIRC) {
            // matmul_by_circulant (circulant.hpp:171-185), SideMultiplier::right_multiply (preprocess.hpp:65-73)
            st = circulant_rows(ctx, rc, n, Ac, D.ld, n, D.c, n, Tc, D.ld, D.spec);
        } else if (Tc != Ac) {
            RL_CUDA(cudaMemcpy2DAsync(Tc, D.ld * 8, Ac, D.ld * 8, n * 8, rc, cudaMemcpyDeviceToDevice, s));
        }
        if (st != RL_OK) return st;
    }
    D.a_chunks = 0;  // resident from here on (the exact-verdict recompute reuses A)
    bool stats_done = !left && D.post == POST_DENSE;
    if (D.pre == POST_DENSE) {
        // F (A H) (SideMultiplier::left_multiply, preprocess.hpp:76-86)
        rl_status st = gemm(ctx, n, n, n, D.F, D.ld, T, D.ld, P, D.ld, 1.0, false, stats);
        if (st != RL_OK) return st;
        stats_done = true;
    } else if (D.pre == POST_CIRC) {
        // column j of F T is circulant_apply(F, T e_j) (preprocess.hpp:80-84):
        // F T = (T^T F^T)^T, the rows of T^T through the FFT kernel
        StreamBuf ub(s);
        rl_status st = ub.alloc(sizeof(double) * n * D.ld);
        if (st != RL_OK) return st;
        if ((st = transpose_device(ctx, T, D.ld, n, n, ub.p, D.ld)) != RL_OK) return st;
        if ((st = circulant_rows(ctx, n, n, ub.p, D.ld, n, D.fct, n, P, D.ld, D.fspec)) != RL_OK) return st;
        if ((st = transpose_device(ctx, P, D.ld, n, n, ub.p, D.ld)) != RL_OK) return st;
        RL_CUDA(cudaMemcpyAsync(P, ub.p, sizeof(double) * n * D.ld, cudaMemcpyDeviceToDevice, s));
    }
    if (stats && !stats_done) {
        matrix_stats_kernel<<<static_cast<unsigned>(n), 256, 0, s>>>(P, D.ld, n, false, stats);
        RL_CHECK_LAUNCH("matrix_stats_kernel");
    }
    return RL_OK;
}

// the first K-part of P = A G (columns [0, k_split) of A, rows of G already
// final) for the row blocks [0, blocks) already uploaded; form_product adds
// the rest
rl_status form_product_part1(rl_context* ctx, Dense& D, int blocks) {
    const int64_t n = D.n;
    const int chunks = D.a_chunks > 0 ? std::min(blocks, D.a_chunks) : 1;
    const int64_t rows = D.a_chunks > 0 ? D.a_chunk_rows : n;
    for (int c = 0; c < chunks; ++c) {
        const int64_t r0 = c * rows, rc = std::min(rows, n - r0);
        if (rc <= 0) break;
        if (D.a_chunks > 0) RL_CUDA(cudaStreamWaitEvent(ctx->stream, D.a_ready[c], 0));
        const rl_status st = gemm(ctx, rc, n, D.k_split, D.A + r0 * D.ld, D.ld, D.G, D.ld, D.P + r0 * D.ld, D.ld, 1.0,
                                  false, nullptr);
        if (st != RL_OK) return st;
    }
    D.part1_blocks = chunks;
    return RL_OK;
}

rl_status factor_and_verdict(rl_context* ctx, Dense& D, rl_solve_info* info, StageTimer* tm = nullptr) {
    cudaStream_t s = ctx->stream;
    const int64_t n = D.n;
    RL_CUDA(cudaMemsetAsync(D.sc, 0, sizeof(Scalars), s));
    rl_status st;
    if (tm) tm->mark();
    if ((st = form_product(ctx, D, D.P, &D.sc->prod)) != RL_OK) return st;
    if (tm) tm->mark();
    // with no left multiplier the first chain solve's right-hand side is b, so
    // its forward substitution can follow the panels
    D.fwd_done = false;
    st = genp_inplace(ctx, n, D.P, D.ld, D.piv, D.rinv, D.pre == POST_NONE ? D.b : nullptr, D.y, &D.fwd_done);
    if (st != RL_OK) return st;
    matrix_stats_kernel<<<static_cast<unsigned>(n), 256, 0, s>>>(D.P, D.ld, n, true, &D.sc->upper);
    RL_CHECK_LAUNCH("matrix_stats_kernel(upper)");
    Scalars h;
    RL_CUDA(cudaMemcpyAsync(&h, D.sc, sizeof(GemmStats) * 2, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    const double fro = std::sqrt(h.prod.sumsq);
    const double tol_pivot = 1e-13 * static_cast<double>(n);  // types.hpp:42
    const double tol_hi = tol_pivot * fro * (1.0 + 1e-10);
    pivot_scan_kernel<<<1, 1024, 0, s>>>(D.piv, n, tol_hi, &D.sc->pivmin, &D.sc->first);
    RL_CHECK_LAUNCH("pivot_scan_kernel");
    RL_CUDA(cudaMemcpyAsync(&h.pivmin, &D.sc->pivmin, 16, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    info->min_abs_pivot = h.pivmin;
    info->max_abs_product = bits_to_double(h.prod.maxabs_bits);
    info->max_abs_u = bits_to_double(h.upper.maxabs_bits);
    info->growth = info->max_abs_u / info->max_abs_product;
    info->norm_frobenius = fro;
    info->pivot_tolerance = tol_hi;
    info->norm_estimate = 0.0;
    info->norm_estimate_evaluated = 0;
    info->zero_pivot_step = 0;
    if (h.first == ~0ull) return RL_OK;

    // a pivot at or below tol_pivot * ||P||_F: evaluate the estimate exactly on
    // a recomputed product and apply the reference's test
    double* prod = nullptr;  // stream-ordered: D's pointers live in the context workspace
    RL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&prod), sizeof(double) * n * D.ld, s));
    st = form_product(ctx, D, prod, nullptr);
    double est = 0.0;
    if (st == RL_OK) st = spectral_norm_estimate_device(ctx, n, n, prod, D.ld, &est);
    cudaFreeAsync(prod, s);
    if (st != RL_OK) return st;
    const double tol = tol_pivot * est;
    info->norm_estimate = est;
    info->norm_estimate_evaluated = 1;
    info->pivot_tolerance = tol;
    pivot_scan_kernel<<<1, 1024, 0, s>>>(D.piv, n, tol, &D.sc->pivmin, &D.sc->first);
    RL_CHECK_LAUNCH("pivot_scan_kernel");
    RL_CUDA(cudaMemcpyAsync(&h.first, &D.sc->first, 8, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    if (h.first != ~0ull) {
        info->zero_pivot_step = static_cast<int64_t>(h.first) + 1;
        return set_error(RL_ERR_ZERO_PIVOT, "zero pivot at elimination step %lld",
                         static_cast<long long>(info->zero_pivot_step));
    }
    return RL_OK;
}

// iterative_refine with the chain solver x = G (LU)^-1 r from x0 = 0,
// refine+1 steps (preprocess.hpp:115-143, :170-178)
rl_status chain_solve(rl_context* ctx, Dense& D, int64_t refine, rl_solve_info* info) {
    cudaStream_t s = ctx->stream;
    const int64_t n = D.n;
    rl_status st = sumsq(ctx, n, D.b, D.sc->bsq);
    if (st != RL_OK) return st;
    RL_CUDA(cudaMemsetAsync(D.x, 0, n * 8, s));
    RL_CUDA(cudaMemcpyAsync(D.r, D.b, n * 8, cudaMemcpyDeviceToDevice, s));  // r = b - A*0
    double bsq = 0.0;
    double last = 0.0;
    int streak = 0;
    info->history_len = 0;
    info->diverged = 0;
    const int64_t steps = refine + 1;
    for (int64_t k = 0; k < steps; ++k) {
        // chain solver H (LU)^-1 (F r) (preprocess.hpp:167-169)
        const double* rhs = D.r;
        if (D.pre == POST_DENSE) {
            if ((st = gemv(ctx, n, n, D.F, D.ld, D.r, D.fr, nullptr)) != RL_OK) return st;
            rhs = D.fr;
        } else if (D.pre == POST_CIRC) {  // F r = (r^T F^T)^T
            if ((st = circulant_rows(ctx, 1, n, D.r, n, n, D.fct, n, D.fr, n, D.fspec)) != RL_OK) return st;
            rhs = D.fr;
        }
        if (k == 0 && D.fwd_done)
            st = lu_solve_upper_device(ctx, n, D.P, D.ld, D.rinv, D.y, D.y, D.solve_work);
        else
            st = lu_solve_device(ctx, n, D.P, D.ld, D.rinv, rhs, D.y, D.solve_work);
        if (st != RL_OK) return st;
        if (D.post == POST_DENSE) {  // H y = matvec (preprocess.hpp:88-94)
            st = gemv(ctx, n, n, D.G, D.ld, D.y, D.d, nullptr);
            if (st != RL_OK) return st;
        } else if (D.post == POST_CIRC) {
            // H y = circulant_apply(C, y) (circulant.hpp:85-91): the row y^T times C^T
            st = circulant_rows(ctx, 1, n, D.y, n, n, D.ct, n, D.d, n, D.spec);
            if (st != RL_OK) return st;
        } else {
            RL_CUDA(cudaMemcpyAsync(D.d, D.y, n * 8, cudaMemcpyDeviceToDevice, s));
        }
        axpy_kernel<<<blocks_for(n, 256), 256, 0, s>>>(D.x, D.d, n);
        RL_CHECK_LAUNCH("axpy_kernel");
        st = gemv(ctx, n, n, D.A, D.ld, D.x, D.r, D.b);  // r = b - A x
        if (st != RL_OK) return st;
        st = sumsq(ctx, n, D.r, D.sc->rsq);
        if (st != RL_OK) return st;
        double rsq = 0.0;
        RL_CUDA(cudaMemcpyAsync(&rsq, D.sc->rsq, 8, cudaMemcpyDeviceToHost, s));
        if (k == 0) RL_CUDA(cudaMemcpyAsync(&bsq, D.sc->bsq, 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaStreamSynchronize(s));
        if (k == 0) {
            // history starts at the residual of x0 = 0, which is ||b||/||b|| = 1 (dropped)
            last = 1.0;
        }
        const double rel = std::sqrt(rsq) / std::sqrt(bsq);
        streak = rel > last ? streak + 1 : 0;
        if (info->history_len < 8) info->residual_history[info->history_len] = rel;
        if (info->history && info->history_len < info->history_capacity) info->history[info->history_len] = rel;
        ++info->history_len;
        last = rel;
        if (streak >= 2) {
            info->diverged = 1;
            break;
        }
    }
    return RL_OK;
}

rl_status dense_alloc(rl_context* ctx, Dense& D, int64_t n, bool need_g, bool own_a, bool own_p) {
    D.n = n;
    D.ld = (n + 1) & ~int64_t(1);
    bool ok = with_arena(ctx, [&](Arena& ar) {
        D.sc = ar.take<Scalars>(1);
        D.piv = ar.take<double>(n);
        D.rinv = ar.take<double>(n);
        D.b = ar.take<double>(n);
        D.x = ar.take<double>(n);
        D.r = ar.take<double>(n);
        D.y = ar.take<double>(n);
        D.d = ar.take<double>(n);
        D.fr = ar.take<double>(n);
        D.solve_work = ar.take<char>(lu_solve_work_bytes(n));
        if (own_a) D.A = ar.take<double>(n * D.ld);
        if (need_g) D.G = ar.take<double>(n * D.ld);
        if (own_p) D.P = ar.take<double>(n * D.ld);
    });
    return ok ? RL_OK : RL_ERR_OUT_OF_MEMORY;
}

rl_status copy_in(rl_context* ctx, double* dst, int64_t ld, const double* src, int64_t rows, int64_t cols, bool host) {
    RL_CUDA(cudaMemcpy2DAsync(dst, ld * 8, src, cols * 8, cols * 8, rows,
                              host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx->stream));
    return RL_OK;
}

rl_status copy_out(rl_context* ctx, double* dst, const double* src, int64_t ld, int64_t rows, int64_t cols, bool host) {
    RL_CUDA(cudaMemcpy2DAsync(dst, cols * 8, src, ld * 8, cols * 8, rows,
                              host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->stream));
    return RL_OK;
}

bool aligned_even(const double* p, int64_t ld) {
    return (ld & 1) == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

// zero the outputs; the caller's history buffer (an input) survives
void clear_info(rl_solve_info* info) {
    double* h = info->history;
    const int64_t cap = info->history_capacity;
    std::memset(info, 0, sizeof(*info));
    info->history = h;
    info->history_capacity = cap;
}

}  // namespace
}  // namespace rl

using namespace rl;

extern "C" RL_API rl_status rl_preprocessed_genp_solve(rl_context* ctx, rl_mem mem, int64_t n, const double* a,
                                                       const double* b, const rl_multiplier* pre,
                                                       const rl_multiplier* post, int64_t refine_steps, double* x,
                                                       double* lu_out, int32_t want_norm_a, rl_solve_info* info) {
    rl_solve_info local;
    if (!info) info = &local;
    clear_info(info);
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "preprocess_solve: matrix dimensions must be positive");
    if (!a || !b || !x) return set_error(RL_ERR_INVALID_ARGUMENT, "preprocess_solve: a, b, x are required");
    if (refine_steps < 0) return set_error(RL_ERR_INVALID_ARGUMENT, "preprocess_solve: negative refine_steps");
    // SolveOutcome::residual_history has refine_steps + 1 entries (preprocess.hpp:124-140): beyond the 8
    // inline slots the caller must supply the buffer, never a silently truncated history
    if (refine_steps + 1 > 8 && (!info->history || info->history_capacity < refine_steps + 1))
        return set_error(RL_ERR_INVALID_ARGUMENT,
                         "preprocess_solve: refine_steps = %lld needs rl_solve_info.history with %lld entries",
                         static_cast<long long>(refine_steps), static_cast<long long>(refine_steps + 1));
    // SideMultiplier::make for both sides (preprocess.hpp:27-60, :162-163)
    rl_status st;
    MForm post_form, pre_form;
    if ((st = side_form(post, &post_form)) != RL_OK) return st;
    if ((st = side_form(pre, &pre_form)) != RL_OK) return st;
    const int kind = post ? post->kind : RL_MULT_NONE;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    const bool host = mem == RL_HOST;
    const bool circ = post_form == MForm::CIRC;
    // SideMultiplier::make (preprocess.hpp:27-60): circulants stay structured
    // (FFT products) when the FFT kernel covers n; otherwise their dense
    // expansion goes through the GEMM path
    const bool circ_fft = circ && circulant_fft_ok(n);
    const bool dense = post_form == MForm::DENSE || (circ && !circ_fft);
    const int64_t ld = (n + 1) & ~int64_t(1);
    // device A can be used in place when it is TMA-compatible (even n, aligned)
    const bool own_a = host || !((n & 1) == 0 && aligned_even(a, n));
    const bool g_dev_direct = post_form == MForm::DENSE && !host && post->dense && (n & 1) == 0 &&
                              aligned_even(post->dense, n);
    Dense D;
    D.post = dense ? POST_DENSE : (circ ? POST_CIRC : POST_NONE);
    st = dense_alloc(ctx, D, n, dense && !g_dev_direct, own_a, true);
    if (st != RL_OK) return st;
    cudaStream_t s = ctx->stream;
    // left multiplier F: dense (materialized on the device) or a structured
    // circulant (the dense expansion when the FFT kernel does not cover n)
    StreamBuf fbuf(s);
    if (pre_form != MForm::NONE) {
        const bool fcirc = pre_form == MForm::CIRC && circulant_fft_ok(n);
        D.pre = fcirc ? POST_CIRC : POST_DENSE;
        if ((st = fbuf.alloc(sizeof(double) * (fcirc ? 3 * n + 64 : n * ld))) != RL_OK) return st;
        if (pre_form == MForm::CIRC) {
            std::vector<double> col, colt(static_cast<size_t>(n));
            if ((st = multiplier_column(pre, n, host, col)) != RL_OK) return st;
            for (int64_t i = 0; i < n; ++i) colt[i] = col[(n - i) % n];  // transposed() (circulant.hpp:40-45)
            if (fcirc) {
                D.fct = fbuf.p;
                D.fspec = fbuf.p + n + 32;
                RL_CUDA(cudaMemcpyAsync(D.fct, colt.data(), n * 8, cudaMemcpyHostToDevice, s));
            } else {
                StreamBuf cb(s);
                if ((st = cb.alloc(n * 8)) != RL_OK) return st;
                RL_CUDA(cudaMemcpyAsync(cb.p, col.data(), n * 8, cudaMemcpyHostToDevice, s));
                D.F = fbuf.p;
                if ((st = circulant_dense(ctx, cb.p, n, n, n, D.F, ld)) != RL_OK) return st;
            }
            RL_CUDA(cudaStreamSynchronize(s));  // col / colt are locals
        } else {
            D.F = fbuf.p;
            if ((st = materialize_device(ctx, pre, n, n, host, D.F, ld)) != RL_OK) return st;
        }
    }
    // seeded dense multiplier: generated on the device (exact); its kernels are
    // enqueued first so that they run under the upload of A
    // host A is uploaded in row blocks on the side stream, which waits only for
    // this stream's earlier work (workspace reuse) — not for the generator
    // kernels enqueued next, so block 0 lands under them
#ifndef RL_A_CHUNKS
#define RL_A_CHUNKS 8
#endif
    constexpr int kChunks = RL_A_CHUNKS;  // row blocks of a host A (the first is exposed before the product)
    const bool pipelined_a = own_a && host && n >= 1024 && side_resources(ctx, kChunks) == RL_OK;
    // pageable host A (the C++ drop-in's RealMatrix, a numpy array): copied
    // into the context's grow-only pinned staging by all host cores first
    // (~16 threads beat the driver's single-threaded staging copies several
    // times over), so its row blocks then stream by DMA under the product.
    // Page-locking the caller's buffer per call instead costs more than the
    // copies (cudaHostRegister of 512 MiB: ~50 ms on this pool).
    if (pipelined_a) {
        cudaPointerAttributes pa{};
        const bool pageable = cudaPointerGetAttributes(&pa, a) != cudaSuccess || pa.type == cudaMemoryTypeUnregistered;
        cudaGetLastError();
        double* stage = pageable ? static_cast<double*>(pinned_staging(ctx, sizeof(double) * n * n, 1)) : nullptr;
        if (stage) {
            host_parallel_copy(stage, a, sizeof(double) * n * n);
            a = stage;
        }
    }
    struct SideDrain {  // error exits: the side stream's uploads read the caller's `a` and write the
        cudaStream_t s = nullptr;  // workspace, so they must be done before the call returns
        ~SideDrain() {
            if (s) cudaStreamSynchronize(s);
        }
    } side_drain;
    if (pipelined_a) {
        side_drain.s = ctx->hi_stream;
        cudaEvent_t start = ctx->events[kChunks - 1];
        RL_CUDA(cudaEventRecord(start, s));
        RL_CUDA(cudaStreamWaitEvent(ctx->hi_stream, start, 0));
    }
    // b first: a small copy on the main stream must not queue behind the
    // side stream's row blocks of A on the copy engine
    RL_CUDA(cudaMemcpyAsync(D.b, b, n * 8, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    GaussJob gjob;
    const bool gen_g = kind == RL_MULT_GAUSSIAN && !post->dense;
    if (gen_g && (st = gjob.begin(ctx, n, n, post->seed, D.G, ld)) != RL_OK) return st;
    int a_issued = 0;
    auto upload_a_block = [&](int c) -> rl_status {
        const int64_t r0 = c * D.a_chunk_rows, rc = std::min(D.a_chunk_rows, n - r0);
        if (rc > 0)
            RL_CUDA(cudaMemcpy2DAsync(D.A + r0 * ld, ld * 8, a + r0 * n, n * 8, n * 8, rc, cudaMemcpyHostToDevice,
                                      ctx->hi_stream));
        RL_CUDA(cudaEventRecord(ctx->events[c], ctx->hi_stream));
        return RL_OK;
    };
    if (own_a) {
        // host A: uploaded in row blocks on the side stream; the product of
        // block c starts as soon as block c has landed
        if (pipelined_a) {
            D.a_chunks = kChunks;
            D.a_chunk_rows = (n + kChunks - 1) / kChunks;
            D.a_ready = ctx->events;
            // block 0 now; when the generator still has host-decided values to
            // upload, the other blocks are enqueued after them (same copy
            // engine: those few MB must not queue behind 3/4 of A)
            a_issued = gen_g ? 1 : kChunks;
            for (int c = 0; c < a_issued; ++c)
                if ((st = upload_a_block(c)) != RL_OK) return st;
        } else if ((st = copy_in(ctx, D.A, ld, a, n, n, host)) != RL_OK) {
            return st;
        }
    } else {
        D.A = const_cast<double*>(a);
    }
    struct Col {
        double* p = nullptr;
        cudaStream_t s;
        ~Col() {
            if (p) cudaFreeAsync(p, s);
        }
    } colbuf{nullptr, s};
    if (circ) {
        // first column: explicit, or drawn by the family's generator
        std::vector<double> col;
        if ((st = multiplier_column(post, n, host, col)) != RL_OK) return st;
        std::vector<double> colt(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) colt[i] = col[(n - i) % n];  // circulant.hpp:40-45
        RL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&colbuf.p), sizeof(double) * 2 * n + 16 * n + 256, s));
        D.c = colbuf.p;
        D.ct = colbuf.p + n;
        D.spec = colbuf.p + 2 * n;
        RL_CUDA(cudaMemcpyAsync(D.c, col.data(), n * 8, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaMemcpyAsync(D.ct, colt.data(), n * 8, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaStreamSynchronize(s));
        if (dense && (st = circulant_dense(ctx, D.c, n, n, n, D.G, ld)) != RL_OK) return st;
    } else if (post_form == MForm::DENSE) {
        if (g_dev_direct) {
            D.G = const_cast<double*>(post->dense);
        } else if (post->dense) {
            if ((st = copy_in(ctx, D.G, ld, post->dense, n, n, host)) != RL_OK) return st;
        } else if (gen_g) {
            // materialize(spec) = gen_gaussian(n, n, seed) (multipliers.hpp:191-192).
            // Once G's first rows are final, the first K-part of A G starts
            // under the host's work on the rest of G
            // (for the row blocks of A already issued: the rest of A follows
            // G's last values on the copy engine, as below)
            auto first_rows = [&](int64_t rows1) -> rl_status {
                const int64_t k1 = rows1 / 16 * 16;
                if (k1 < 512 || D.pre != POST_NONE) return RL_OK;
                D.k_split = k1;
                return form_product_part1(ctx, D, D.a_chunks > 0 ? a_issued : 1);
            };
            if ((st = gjob.finish(nullptr, first_rows)) != RL_OK) return st;
        } else if ((st = materialize_device(ctx, post, n, n, host, D.G, ld)) != RL_OK) {
            return st;  // FiniteSetUniform, CircSkewProduct (multipliers.hpp:195-200)
        }
    }
    for (; a_issued > 0 && a_issued < D.a_chunks; ++a_issued)
        if ((st = upload_a_block(a_issued)) != RL_OK) return st;
    StageTimer timer(s);
    st = factor_and_verdict(ctx, D, info, &timer);
    if (st != RL_OK) {
        RL_CUDA(cudaStreamSynchronize(s));
        return st;
    }
    timer.mark();
    st = chain_solve(ctx, D, refine_steps, info);
    if (st != RL_OK) return st;
    timer.mark();
    timer.fill(info->stage_ms);
    RL_CUDA(cudaMemcpyAsync(x, D.x, n * 8, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    if (lu_out && (st = copy_out(ctx, lu_out, D.P, ld, n, n, host)) != RL_OK) return st;
    if (want_norm_a) {
        // BASELINE config-1 residual form ||Ax - b|| / (||A||_est ||x||)
        double na = 0.0;
        st = spectral_norm_estimate_device(ctx, n, n, D.A, ld, &na);
        if (st != RL_OK) return st;
        if ((st = sumsq(ctx, n, D.x, D.sc->bsq)) != RL_OK) return st;  // bsq scratch reused for ||x||^2
        double sq[2];
        RL_CUDA(cudaMemcpyAsync(&sq[0], D.sc->rsq, 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaMemcpyAsync(&sq[1], D.sc->bsq, 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaStreamSynchronize(s));
        info->residual_rel_a = std::sqrt(sq[0]) / (na * std::sqrt(sq[1]));
    }
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}

extern "C" RL_API rl_status rl_genp_factor(rl_context* ctx, rl_mem mem, int64_t n, const double* a, double* lu,
                                           rl_solve_info* info) {
    rl_solve_info local;
    if (!info) info = &local;
    clear_info(info);
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "genp_factor: square input required");
    if (!a || !lu) return set_error(RL_ERR_INVALID_ARGUMENT, "genp_factor: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    const bool host = mem == RL_HOST;
    Dense D;
    st = dense_alloc(ctx, D, n, false, true, true);
    if (st != RL_OK) return st;
    if ((st = copy_in(ctx, D.A, D.ld, a, n, n, host)) != RL_OK) return st;
    st = factor_and_verdict(ctx, D, info);
    if (st != RL_OK && st != RL_ERR_ZERO_PIVOT) return st;
    const rl_status verdict = st;
    if ((st = copy_out(ctx, lu, D.P, D.ld, n, n, host)) != RL_OK) return st;
    RL_CUDA(cudaStreamSynchronize(ctx->stream));
    return verdict;
}

extern "C" RL_API rl_status rl_lu_solve(rl_context* ctx, rl_mem mem, int64_t n, const double* lu, const double* b,
                                        double* x) {
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "lu_solve: length mismatch");
    if (!lu || !b || !x) return set_error(RL_ERR_INVALID_ARGUMENT, "lu_solve: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    const bool host = mem == RL_HOST;
    double *dlu = const_cast<double*>(lu), *db = const_cast<double*>(b), *dx = x;
    void* work = nullptr;
    bool ok = with_arena(ctx, [&](Arena& ar) {
        work = ar.take<char>(lu_solve_work_bytes(n));
        if (host) {
            dlu = ar.take<double>(n * n);
            db = ar.take<double>(n);
            dx = ar.take<double>(n);
        }
    });
    if (!ok) return RL_ERR_OUT_OF_MEMORY;
    cudaStream_t s = ctx->stream;
    if (host) {
        RL_CUDA(cudaMemcpyAsync(dlu, lu, n * n * 8, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaMemcpyAsync(db, b, n * 8, cudaMemcpyHostToDevice, s));
    }
    st = lu_solve_device(ctx, n, dlu, n, nullptr, db, dx, work);
    if (st != RL_OK) return st;
    if (host) {
        RL_CUDA(cudaMemcpyAsync(x, dx, n * 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaStreamSynchronize(s));
    }
    return RL_OK;
}

extern "C" RL_API rl_status rl_spectral_norm_estimate(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                                      double* out) {
    if (m <= 0 || n <= 0) return set_error(RL_ERR_DIMENSION, "spectral_norm_estimate: empty matrix");
    if (!a || !out) return set_error(RL_ERR_INVALID_ARGUMENT, "spectral_norm_estimate: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    double* da = const_cast<double*>(a);
    if (mem == RL_HOST) {
        RL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&da), m * n * 8, ctx->stream));
        RL_CUDA(cudaMemcpyAsync(da, a, m * n * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    st = spectral_norm_estimate_device(ctx, m, n, da, n, out);
    if (mem == RL_HOST) cudaFreeAsync(da, ctx->stream);
    RL_CUDA(cudaStreamSynchronize(ctx->stream));
    return st;
}
