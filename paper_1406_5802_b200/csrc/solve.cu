// Triangular solves, matrix-vector products, reductions and the exact-order
// spectral-norm estimate for the dense path.
//
//  lu_solve_device  lu_solve (lu.hpp:100-123) on packed LU: one kernel per
//                   triangle, 64-row blocks claimed in order through an atomic
//                   ticket; block B folds in the finished blocks C < B as their
//                   flags appear (GEMV from HBM, coalesced) and then solves its
//                   64x64 diagonal block with a warp column sweep. No grid-wide
//                   barrier and no co-residency assumption.
//  gemv             matvec (matrix.hpp:146-156) / residual b - A x
//                   (preprocess.hpp:122-126), one warp per row.
//  spectral_norm_estimate_device
//                   norms.hpp:35-78 in the reference's summation order with
//                   separately rounded products and sums (no FMA), so the
//                   estimate of a given matrix is bit-identical to the
//                   reference's.
#include <algorithm>
#include <cmath>
#include <vector>

#include "device_common.cuh"
#include "kernels.cuh"

namespace rl {
namespace {

constexpr int TB = 64;

__device__ __forceinline__ double div_by(double a, double b, double r) {
    const double q0 = a * r;
    return fma(r, fma(-b, q0, a), q0);
}

__device__ __forceinline__ void wait_flag(const int* flag) {
    while (atomicAdd(const_cast<int*>(flag), 0) == 0) __nanosleep(64);
}

// kUpper = false: y = L^-1 b (unit lower); true: x = U^-1 y (upper, diagonal)
// Block B (64 rows, claimed in dependency order through the ticket) keeps the
// next dependency tile of L/U in registers while it waits for the current
// one's flag, so the HBM read of the tile is off the critical path; the
// diagonal block, its reciprocal pivots and the finished x blocks go through
// shared memory.
template <bool kUpper>
__global__ void __launch_bounds__(256)
trsv_kernel(const double* __restrict__ lu, int64_t ld, int64_t n, const double* __restrict__ rinv,
            const double* rhs, double* out, int* __restrict__ flags, int* __restrict__ ticket) {
    __shared__ int s_blk;
    __shared__ double sdiag[TB][TB + 1];
    __shared__ double sri[TB];
    __shared__ double sx[TB];
    __shared__ double sacc[TB];
    const int tid = threadIdx.x;
    const int64_t nblk = (n + TB - 1) / TB;
    if (tid == 0) s_blk = atomicAdd(ticket, 1);
    __syncthreads();
    const int64_t order = s_blk;
    if (order >= nblk) return;
    const int64_t B = kUpper ? nblk - 1 - order : order;
    const int64_t r0 = B * TB;
    const int nr = static_cast<int>(min(static_cast<int64_t>(TB), n - r0));

    // diagonal block (identity-padded past nr) and 1/u_jj while the dependencies finish
    for (int idx = tid; idx < TB * TB; idx += 256) {
        const int i = idx / TB, k = idx % TB;
        sdiag[i][k] = (i < nr && k < nr) ? lu[(r0 + i) * ld + r0 + k] : (i == k ? 1.0 : 0.0);
    }
    if (kUpper && tid < TB) sri[tid] = tid < nr ? (rinv ? __ldcg(rinv + r0 + tid) : 1.0 / lu[(r0 + tid) * ld + r0 + tid]) : 1.0;
    // off-diagonal contributions: thread (row, q) takes columns q, q+4, ... of each tile
    const int row = tid >> 2, q = tid & 3;
    const bool live = row < nr;
    double acc = 0.0;
    const int64_t ndep = kUpper ? nblk - 1 - B : B;
    double cur[TB / 4], nxt[TB / 4];
    auto load_tile = [&](int64_t t, double (&v)[TB / 4]) {
        const int64_t C = kUpper ? nblk - 1 - t : t;
        const int64_t c0 = C * TB;
        const int nc = static_cast<int>(min(static_cast<int64_t>(TB), n - c0));
        const double* lrow = lu + (r0 + row) * ld + c0;
#pragma unroll
        for (int j = 0; j < TB / 4; ++j) {
            const int k = q + 4 * j;
            v[j] = (live && k < nc) ? __ldcs(lrow + k) : 0.0;
        }
    };
    if (ndep > 0) load_tile(0, cur);
    for (int64_t t = 0; t < ndep; ++t) {
        const int64_t C = kUpper ? nblk - 1 - t : t;
        if (t + 1 < ndep) load_tile(t + 1, nxt);
        if (tid == 0) {
            wait_flag(&flags[C]);
            __threadfence();
        }
        __syncthreads();
        const int64_t c0 = C * TB;
        const int nc = static_cast<int>(min(static_cast<int64_t>(TB), n - c0));
        if (tid < TB) sx[tid] = tid < nc ? __ldcg(out + c0 + tid) : 0.0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < TB / 4; ++j) acc = fma(cur[j], sx[q + 4 * j], acc);
        __syncthreads();  // sx is rewritten by the next dependency
#pragma unroll
        for (int j = 0; j < TB / 4; ++j) cur[j] = nxt[j];
    }
    acc += __shfl_xor_sync(kFull, acc, 1);
    acc += __shfl_xor_sync(kFull, acc, 2);
    if (q == 0) sacc[row] = live ? __ldcg(rhs + r0 + row) - acc : 0.0;
    __syncthreads();

    // diagonal block: column sweep on warp 0, two rows per lane, fully unrolled
    if (tid < 32) {
        const int lane = tid;
        double v0 = sacc[lane];
        double v1 = sacc[lane + 32];
        if (!kUpper) {
#pragma unroll
            for (int k = 0; k < TB; ++k) {
                const double yk = __shfl_sync(kFull, k < 32 ? v0 : v1, k & 31);
                if (lane > k) v0 = fma(-sdiag[lane][k], yk, v0);
                if (lane + 32 > k) v1 = fma(-sdiag[lane + 32][k], yk, v1);
            }
        } else {
#pragma unroll
            for (int k = TB - 1; k >= 0; --k) {
                const double d = sdiag[k][k];
                const double ri = sri[k];
                if (lane == k) v0 = div_by(v0, d, ri);
                if (lane + 32 == k) v1 = div_by(v1, d, ri);
                const double xk = __shfl_sync(kFull, k < 32 ? v0 : v1, k & 31);
                if (lane < k) v0 = fma(-sdiag[lane][k], xk, v0);
                if (lane + 32 < k) v1 = fma(-sdiag[lane + 32][k], xk, v1);
            }
        }
        if (lane < nr) out[r0 + lane] = v0;
        if (lane + 32 < nr) out[r0 + lane + 32] = v1;
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(&flags[B], 1);
    }
}

// y[row] = (b ? b[row] : 0) - / + A[row,:] x ; one warp per row
__global__ void __launch_bounds__(256)
gemv_kernel(const double* __restrict__ a, int64_t lda, int64_t m, int64_t n, const double* __restrict__ x,
            double* __restrict__ y, const double* __restrict__ b) {
    const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= m) return;
    const double* ar = a + row * lda;
    double acc = 0.0;
    if ((lda & 1) == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        const double2* a2 = reinterpret_cast<const double2*>(ar);
        const double2* x2 = reinterpret_cast<const double2*>(x);
        const int64_t n2 = n / 2;
        // four independent accumulators: four 16-byte loads in flight per lane
        double c1 = 0.0, c2 = 0.0, c3 = 0.0;
        int64_t k = lane;
        for (; k + 96 < n2; k += 128) {
            const double2 a0 = __ldcs(a2 + k), a1 = __ldcs(a2 + k + 32), a2v = __ldcs(a2 + k + 64),
                          a3 = __ldcs(a2 + k + 96);
            const double2 x0 = x2[k], x1 = x2[k + 32], x2v = x2[k + 64], x3 = x2[k + 96];
            acc = fma(a0.x, x0.x, fma(a0.y, x0.y, acc));
            c1 = fma(a1.x, x1.x, fma(a1.y, x1.y, c1));
            c2 = fma(a2v.x, x2v.x, fma(a2v.y, x2v.y, c2));
            c3 = fma(a3.x, x3.x, fma(a3.y, x3.y, c3));
        }
        for (; k < n2; k += 32) {
            const double2 av = __ldcs(a2 + k), xv = x2[k];
            acc = fma(av.x, xv.x, fma(av.y, xv.y, acc));
        }
        acc = (acc + c1) + (c2 + c3);
        if ((n & 1) && lane == 0) acc = fma(ar[n - 1], x[n - 1], acc);
    } else {
        for (int64_t k = lane; k < n; k += 32) acc = fma(ar[k], x[k], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) y[row] = b ? b[row] - acc : acc;
}

// deterministic sum of squares: per-block partials, then one block
__global__ void sumsq_partial_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ part) {
    __shared__ double sm[32];
    double s = 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        s = fma(v[i], v[i], s);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
        s = warp_sum(s);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
    }
}

__global__ void sum_final_kernel(const double* __restrict__ part, int np, double* __restrict__ out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += 32) s += part[i];
    s = warp_sum(s);
    if (threadIdx.x == 0) *out = s;
}

// ---- exact-order power iteration pieces (norms.hpp:35-78) -------------------
// column sums of squares (i ascending) and row sums (j ascending), max into out
__global__ void normest_floor_kernel(const double* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                                     double* __restrict__ colsq, double* __restrict__ rowsq) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n) {
        double s = 0.0;
        for (int64_t i = 0; i < m; ++i) s = __dadd_rn(s, __dmul_rn(a[i * lda + t], a[i * lda + t]));
        colsq[t] = s;
    }
    if (t < m) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s = __dadd_rn(s, __dmul_rn(a[t * lda + j], a[t * lda + j]));
        rowsq[t] = s;
    }
}

// ax_i = sum_j a_ij x_j  (j ascending)
__global__ void normest_ax_kernel(const double* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                                  const double* __restrict__ x, double* __restrict__ ax) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) s = __dadd_rn(s, __dmul_rn(a[i * lda + j], x[j]));
    ax[i] = s;
}

// y_j = sum_i a_ij ax_i  (i ascending)
__global__ void normest_aty_kernel(const double* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                                   const double* __restrict__ ax, double* __restrict__ y) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s = __dadd_rn(s, __dmul_rn(a[i * lda + j], ax[i]));
    y[j] = s;
}

// sequential norm2 (matrix.hpp:172-177) of v into *out; one thread
__global__ void seq_norm2_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s = __dadd_rn(s, __dmul_rn(v[i], v[i]));
    *out = sqrt(s);
}

// x = (1/ny) * y
__global__ void scale_kernel(const double* __restrict__ y, int64_t n, const double* __restrict__ ny, double* __restrict__ x) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) x[j] = __dmul_rn(1.0 / *ny, y[j]);
}

__global__ void normest_init_kernel(double* __restrict__ x, int64_t n) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) x[j] = 1.0 + static_cast<double>(j) / (static_cast<double>(n) + 1.0);
}

__global__ void max_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, v[i]);
    m = warp_max(m);
    __shared__ double sm[32];
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) m = fmax(m, sm[i]);
        *out = m;
    }
}

unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

size_t lu_solve_work_bytes(int64_t n) { return align_up(sizeof(int) * 2 * ((n + TB - 1) / TB + 2)); }

rl_status lu_solve_device(rl_context* ctx, int64_t n, const double* lu, int64_t ld, const double* rinv, const double* b,
                          double* x, void* work) {
    if (n <= 0) return RL_OK;
    const int64_t nblk = (n + TB - 1) / TB;
    int* flags = static_cast<int*>(work);
    int* ticket = flags + nblk;
    int* flags2 = ticket + 1;
    int* ticket2 = flags2 + nblk;
    RL_CUDA(cudaMemsetAsync(work, 0, sizeof(int) * 2 * (nblk + 1), ctx->stream));
    const unsigned grid = static_cast<unsigned>(nblk);
    trsv_kernel<false><<<grid, 256, 0, ctx->stream>>>(lu, ld, n, rinv, b, x, flags, ticket);
    RL_CHECK_LAUNCH("trsv_kernel<lower>");
    trsv_kernel<true><<<grid, 256, 0, ctx->stream>>>(lu, ld, n, rinv, x, x, flags2, ticket2);
    RL_CHECK_LAUNCH("trsv_kernel<upper>");
    return RL_OK;
}

rl_status lu_solve_upper_device(rl_context* ctx, int64_t n, const double* lu, int64_t ld, const double* rinv,
                                const double* y, double* x, void* work) {
    if (n <= 0) return RL_OK;
    const int64_t nblk = (n + TB - 1) / TB;
    int* flags2 = static_cast<int*>(work);
    int* ticket2 = flags2 + nblk;
    RL_CUDA(cudaMemsetAsync(work, 0, sizeof(int) * (nblk + 1), ctx->stream));
    trsv_kernel<true><<<static_cast<unsigned>(nblk), 256, 0, ctx->stream>>>(lu, ld, n, rinv, y, x, flags2, ticket2);
    RL_CHECK_LAUNCH("trsv_kernel<upper>");
    return RL_OK;
}

rl_status gemv(rl_context* ctx, int64_t m, int64_t n, const double* a, int64_t lda, const double* x, double* y,
               const double* b) {
    if (m <= 0) return RL_OK;
    gemv_kernel<<<blocks_for(m, 8), 256, 0, ctx->stream>>>(a, lda, m, n, x, y, b);
    RL_CHECK_LAUNCH("gemv_kernel");
    return RL_OK;
}

rl_status sumsq(rl_context* ctx, int64_t n, const double* v, double* out) {
    // out[0] = result; out[1..64] scratch partials
    const int np = static_cast<int>(std::min<int64_t>(64, std::max<int64_t>(1, (n + 1023) / 1024)));
    sumsq_partial_kernel<<<np, 256, 0, ctx->stream>>>(v, n, out + 1);
    RL_CHECK_LAUNCH("sumsq_partial_kernel");
    sum_final_kernel<<<1, 32, 0, ctx->stream>>>(out + 1, np, out);
    RL_CHECK_LAUNCH("sum_final_kernel");
    return RL_OK;
}

rl_status spectral_norm_estimate_device(rl_context* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                                        double* out) {
    // stream-ordered scratch (callers may hold pointers into the context workspace)
    cudaStream_t s = ctx->stream;
    double* buf = nullptr;
    RL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), sizeof(double) * (3 * n + 2 * m + 8), s));
    struct Free {
        double* p;
        cudaStream_t s;
        ~Free() { cudaFreeAsync(p, s); }
    } guard{buf, s};
    double *colsq = buf, *x = buf + n, *y = buf + 2 * n, *rowsq = buf + 3 * n, *ax = buf + 3 * n + m,
           *sc = buf + 3 * n + 2 * m;
    const int64_t mn = std::max(m, n);
    normest_floor_kernel<<<blocks_for(mn, 128), 128, 0, s>>>(a, lda, m, n, colsq, rowsq);
    RL_CHECK_LAUNCH("normest_floor_kernel");
    max_kernel<<<1, 1024, 0, s>>>(colsq, n, sc);
    max_kernel<<<1, 1024, 0, s>>>(rowsq, m, sc + 1);
    RL_CHECK_LAUNCH("max_kernel");
    double h[2];
    RL_CUDA(cudaMemcpyAsync(h, sc, 16, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    const double floor_norm = std::sqrt(std::max(h[0], h[1]));
    if (floor_norm == 0.0) {
        *out = 0.0;
        return RL_OK;
    }
    normest_init_kernel<<<blocks_for(n, 256), 256, 0, s>>>(x, n);
    seq_norm2_kernel<<<1, 1, 0, s>>>(x, n, sc + 2);
    scale_kernel<<<blocks_for(n, 256), 256, 0, s>>>(x, n, sc + 2, x);
    RL_CHECK_LAUNCH("normest init");
    double est = 0.0;
    for (int it = 0; it < 200; ++it) {
        normest_ax_kernel<<<blocks_for(m, 128), 128, 0, s>>>(a, lda, m, n, x, ax);
        seq_norm2_kernel<<<1, 1, 0, s>>>(ax, m, sc);
        normest_aty_kernel<<<blocks_for(n, 128), 128, 0, s>>>(a, lda, m, n, ax, y);
        seq_norm2_kernel<<<1, 1, 0, s>>>(y, n, sc + 1);
        scale_kernel<<<blocks_for(n, 256), 256, 0, s>>>(y, n, sc + 1, x);
        RL_CHECK_LAUNCH("normest iteration");
        RL_CUDA(cudaMemcpyAsync(h, sc, 16, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaStreamSynchronize(s));
        const double nax = h[0], ny = h[1];
        if (nax == 0.0 || ny == 0.0) break;
        if (std::fabs(nax - est) <= 1e-9 * nax) {
            est = nax;
            break;
        }
        est = nax;
    }
    *out = std::max(est, floor_norm);
    return RL_OK;
}

}  // namespace rl
