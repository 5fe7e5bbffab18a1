// Recursive block Gaussian elimination (block_ge.hpp:88-219) on the device,
// with the reference's own arithmetic order so that its results are
// bit-identical to the reference's:
//   rl_gepp_factor    gepp_factor (lu.hpp:62-98): partial pivoting, first
//                     maximal |u_ij|, u_ik - l u_jk without FMA
//   rl_block_ge_factor block_ge_factor (block_ge.hpp:168-181) for a split
//                     (pivot block sizes in elimination order): per level the
//                     leaf check svd_values(B).back() <= tol
//                     (block_ge.hpp:97-99), the leaf's GEPP, B^-1 C by
//                     lu_solve, D B^-1 by lu_solve_transpose, and
//                     S = E - (D B^-1) C accumulated in natural order
//                     (block_ge.hpp:126-134)
//   rl_block_solve    block_solve (block_ge.hpp:141-163, 198-201)
//
// The factorisation of a split is a right spine (each pivot child is a leaf),
// so it is stored flat in one n x n buffer: level l at offset o with pivot
// block size k holds the leaf's packed GEPP factors in [o, o+k)^2, B^-1 C in
// rows [o, o+k) right of it and D B^-1 in columns [o, o+k) below it; perm
// holds each leaf's local row permutation at [o, o+k).
//
// Singular values for the leaf check come from a one-sided (Hestenes) Jacobi
// sweep on the device; the reference calls Eigen's JacobiSVD/BDCSVD
// (svd.hpp:76-88), a third-party library absent here. Both return the
// singular values to high relative accuracy; only the comparison with tol
// uses them.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "device_common.cuh"
#include "kernels.cuh"

namespace rl {
namespace {

constexpr int GT = 1024;  // gepp threads (one CTA)

// gepp_factor (lu.hpp:62-98) in place on a (n x n, ld), packed L\U, local
// row permutation perm[i] = original row of position i. *bad = first 1-based
// step whose best |u_ij| <= tol (0 = none).
__global__ void __launch_bounds__(GT) gepp_kernel(double* __restrict__ a, int64_t ld, int n,
                                                   int64_t* __restrict__ perm, double tol, int64_t* __restrict__ bad) {
    __shared__ double smag[GT / 32];
    __shared__ int sidx[GT / 32];
    __shared__ int s_best;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < n; i += GT) perm[i] = i;
    if (tid == 0) *bad = 0;
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        // first maximal |u_ij|, i >= j (lu.hpp:72-80: strict > keeps the first)
        double bm = -1.0;
        int bi = n;
        for (int i = j + tid; i < n; i += GT) {
            const double m = fabs(a[i * ld + j]);
            if (m > bm) {
                bm = m;
                bi = i;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double om = __shfl_xor_sync(kFull, bm, o);
            const int oi = __shfl_xor_sync(kFull, bi, o);
            if (om > bm || (om == bm && oi < bi)) {
                bm = om;
                bi = oi;
            }
        }
        if (lane == 0) {
            smag[warp] = bm;
            sidx[warp] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            double m = smag[0];
            int i0 = sidx[0];
            for (int w = 1; w < GT / 32; ++w)
                if (smag[w] > m || (smag[w] == m && sidx[w] < i0)) {
                    m = smag[w];
                    i0 = sidx[w];
                }
            s_best = (m <= tol) ? -1 : i0;  // lu.hpp:81-83
            if (m <= tol) *bad = j + 1;
        }
        __syncthreads();
        const int best = s_best;
        if (best < 0) return;
        if (best != j) {  // swap whole packed rows (U part and L part), lu.hpp:84-88
            for (int k = tid; k < n; k += GT) {
                const double t = a[j * ld + k];
                a[j * ld + k] = a[best * ld + k];
                a[best * ld + k] = t;
            }
            if (tid == 0) {
                const int64_t t = perm[j];
                perm[j] = perm[best];
                perm[best] = t;
            }
        }
        __syncthreads();
        const double piv = a[j * ld + j];
        for (int i = j + 1 + tid; i < n; i += GT) a[i * ld + j] = __ddiv_rn(a[i * ld + j], piv);  // lu.hpp:91
        __syncthreads();
        const int w = n - j - 1;
        for (int64_t e = tid; e < static_cast<int64_t>(w) * w; e += GT) {
            const int i = j + 1 + static_cast<int>(e / w), k = j + 1 + static_cast<int>(e % w);
            a[i * ld + k] = __dsub_rn(a[i * ld + k], __dmul_rn(a[i * ld + j], a[j * ld + k]));  // lu.hpp:94
        }
        __syncthreads();
    }
}

// lu_solve (lu.hpp:100-123) / lu_solve_transpose (lu.hpp:127-147) with GEPP
// factors, one right-hand side per thread, the reference's loop order.
// Right-hand side r, element t: in[r * rs + t * es]; same strides out.
__global__ void gepp_solve_kernel(const double* __restrict__ lu, int64_t ld, int n, const int64_t* __restrict__ perm,
                                  const double* __restrict__ in, int64_t in_rs, int64_t in_es, double* __restrict__ out,
                                  int64_t out_rs, int64_t out_es, int64_t nrhs, int transpose, double* __restrict__ work) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= nrhs) return;
    double* y = work + r * n;  // per-rhs scratch (global; L1-resident)
    const double* b = in + r * in_rs;
    double* x = out + r * out_rs;
    if (!transpose) {
        for (int i = 0; i < n; ++i) y[i] = b[perm[i] * in_es];
        for (int i = 0; i < n; ++i) {  // forward, unit L
            double acc = y[i];
            for (int k = 0; k < i; ++k) acc = __dsub_rn(acc, __dmul_rn(lu[i * ld + k], y[k]));
            y[i] = acc;
        }
        for (int i = n - 1; i >= 0; --i) {  // backward, U
            double acc = y[i];
            for (int k = i + 1; k < n; ++k) acc = __dsub_rn(acc, __dmul_rn(lu[i * ld + k], y[k]));
            y[i] = __ddiv_rn(acc, lu[i * ld + i]);
        }
        for (int i = 0; i < n; ++i) x[i * out_es] = y[i];
    } else {
        for (int i = 0; i < n; ++i) {  // U^T w = c
            double acc = b[i * in_es];
            for (int k = 0; k < i; ++k) acc = __dsub_rn(acc, __dmul_rn(lu[k * ld + i], y[k]));
            y[i] = __ddiv_rn(acc, lu[i * ld + i]);
        }
        for (int ii = n - 1; ii >= 0; --ii) {  // L^T z = w
            double acc = y[ii];
            for (int k = ii + 1; k < n; ++k) acc = __dsub_rn(acc, __dmul_rn(lu[k * ld + ii], y[k]));
            y[ii] = acc;
        }
        for (int i = 0; i < n; ++i) x[perm[i] * out_es] = y[i];  // undo P
    }
}

// S = E - X C in place of E (rows x cols), X rows x k, C k x cols, each entry
// accumulated t = 0..k-1 in order without FMA (block_ge.hpp:128-134):
// 32x32 output tiles, 32-deep shared-memory slabs of X and C.
constexpr int ST = 32;
__global__ void __launch_bounds__(ST * 8) schur_natural_kernel(double* __restrict__ e, int64_t lde,
                                                               const double* __restrict__ x, int64_t ldx,
                                                               const double* __restrict__ c, int64_t ldc, int64_t rows,
                                                               int64_t cols, int64_t k) {
    __shared__ double sx[ST][ST + 1];
    __shared__ double sc[ST][ST + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8: each thread 4 rows
    const int64_t i0 = static_cast<int64_t>(blockIdx.y) * ST, j0 = static_cast<int64_t>(blockIdx.x) * ST;
    double acc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t i = i0 + ty + 8 * q, j = j0 + tx;
        acc[q] = (i < rows && j < cols) ? e[i * lde + j] : 0.0;
    }
    for (int64_t t0 = 0; t0 < k; t0 += ST) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = ty + 8 * q;
            const int64_t xi = i0 + r, xt = t0 + tx, ct = t0 + r, cj = j0 + tx;
            sx[r][tx] = (xi < rows && xt < k) ? x[xi * ldx + xt] : 0.0;
            sc[r][tx] = (ct < k && cj < cols) ? c[ct * ldc + cj] : 0.0;
        }
        __syncthreads();
        const int tn = static_cast<int>(std::min<int64_t>(ST, k - t0));
        for (int t = 0; t < tn; ++t) {
            const double cv = sc[t][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = __dsub_rn(acc[q], __dmul_rn(sx[ty + 8 * q][t], cv));
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t i = i0 + ty + 8 * q, j = j0 + tx;
        if (i < rows && j < cols) e[i * lde + j] = acc[q];
    }
}

// y[i] -= sum_t M(i, t) v[t] in order (acc -= a * b, block_ge.hpp:147-151 and
// :156-159), one row per thread
__global__ void row_update_kernel(double* __restrict__ y, const double* __restrict__ m, int64_t ldm,
                                  const double* __restrict__ v, int64_t rows, int64_t k) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double acc = y[i];
    for (int64_t t = 0; t < k; ++t) acc = __dsub_rn(acc, __dmul_rn(m[i * ldm + t], v[t]));
    y[i] = acc;
}

// Singular values of a (m x n, ld, m >= n) by one-sided Jacobi on its
// columns, one CTA: the columns are copied transposed into w (n rows of
// length m), n/2 disjoint pairs per round (round-robin order), one warp per
// pair; sweeps until no pair is rotated. sv (n) receives the column norms
// (unsorted).
constexpr int JT = 512;
__global__ void __launch_bounds__(JT) jacobi_sv_kernel(const double* __restrict__ a, int64_t ld, int m, int n,
                                                        double* __restrict__ w, int* __restrict__ order,
                                                        double* __restrict__ sv) {
    __shared__ int s_rot;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int np = n + (n & 1);  // with a dummy column when n is odd
    for (int64_t e = tid; e < static_cast<int64_t>(m) * n; e += JT) {
        const int i = static_cast<int>(e / n), p = static_cast<int>(e % n);
        w[static_cast<int64_t>(p) * m + i] = a[i * ld + p];
    }
    for (int i = tid; i < np; i += JT) order[i] = i;
    __syncthreads();
    int cur = 0;  // order ping-pongs between [0, np) and [np, 2 np)
    for (int sweep = 0; sweep < 60; ++sweep) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int round = 0; round < np - 1; ++round) {
            const int* ord = order + cur * np;
            for (int pr = warp; pr < np / 2; pr += JT / 32) {
                int p = ord[pr], q = ord[np - 1 - pr];
                if (p >= n || q >= n) continue;
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                double* wp = w + static_cast<int64_t>(p) * m;
                double* wq = w + static_cast<int64_t>(q) * m;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = lane; i < m; i += 32) {
                    al = fma(wp[i], wp[i], al);
                    be = fma(wq[i], wq[i], be);
                    ga = fma(wp[i], wq[i], ga);
                }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum(ga);
                if (ga != 0.0 && fabs(ga) > 1e-15 * sqrt(al * be)) {
                    const double zeta = (be - al) / (2.0 * ga);
                    const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
                    for (int i = lane; i < m; i += 32) {
                        const double xp = wp[i], xq = wq[i];
                        wp[i] = cs * xp - sn * xq;
                        wq[i] = sn * xp + cs * xq;
                    }
                    if (lane == 0) s_rot = 1;
                }
            }
            // round-robin: keep position 0, rotate the others by one
            int* nxt = order + (cur ^ 1) * np;
            for (int i = tid; i < np; i += JT) nxt[i] = i == 0 ? ord[0] : (i == 1 ? ord[np - 1] : ord[i - 1]);
            cur ^= 1;
            __syncthreads();
        }
        if (!s_rot) break;
        __syncthreads();
    }
    for (int p = warp; p < n; p += JT / 32) {
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s = fma(w[static_cast<int64_t>(p) * m + i], w[static_cast<int64_t>(p) * m + i], s);
        s = warp_sum(s);
        if (lane == 0) sv[p] = sqrt(s);
    }
}

__global__ void copy_block_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd,
                                  int64_t rows, int64_t cols) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= rows * cols) return;
    const int64_t i = e / cols, j = e % cols;
    dst[i * ldd + j] = src[i * lds + j];
}

__global__ void min_kernel(const double* __restrict__ v, int n, double* __restrict__ out) {
    double m = INFINITY;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmin(m, v[i]);
    m = warp_min(m);
    __shared__ double s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmin(m, s[w]);
        *out = fmin(m, s[0]);
    }
}

struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

template <typename T>
rl_status dev_alloc(DevBuf& b, cudaStream_t s, size_t count, T** out) {
    b.s = s;
    RL_CUDA(cudaMallocAsync(&b.p, std::max<size_t>(count, 1) * sizeof(T), s));
    *out = static_cast<T*>(b.p);
    return RL_OK;
}

inline unsigned nblocks(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

// GEPP of the k x k block at `blk` (ld) in place; tol = tol_pivot(k) *
// spectral_norm_estimate(block) (lu.hpp:66). *bad_step: 1-based failing step.
rl_status gepp_inplace(rl_context* ctx, int64_t k, double* blk, int64_t ld, int64_t* perm_dev, int64_t* bad_step) {
    double est = 0.0;
    rl_status st = spectral_norm_estimate_device(ctx, k, k, blk, ld, &est);
    if (st != RL_OK) return st;
    const double tol = 1e-13 * static_cast<double>(k) * est;
    int64_t* dbad = nullptr;
    DevBuf bb;
    if ((st = dev_alloc(bb, ctx->stream, 1, &dbad)) != RL_OK) return st;
    gepp_kernel<<<1, GT, 0, ctx->stream>>>(blk, ld, static_cast<int>(k), perm_dev, tol, dbad);
    RL_CHECK_LAUNCH("gepp_kernel");
    RL_CUDA(cudaMemcpyAsync(bad_step, dbad, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    RL_CUDA(cudaStreamSynchronize(ctx->stream));
    return *bad_step ? set_error(RL_ERR_SINGULAR_MATRIX, "gepp_factor: matrix is singular to working precision at step %lld",
                                 static_cast<long long>(*bad_step))
                     : RL_OK;
}

// smallest singular value of the k x k block (device), host result
rl_status min_singular_value(rl_context* ctx, int64_t k, const double* blk, int64_t ld, double* out) {
    rl_status st;
    double *w = nullptr, *sv = nullptr, *mn = nullptr;
    int* order = nullptr;
    DevBuf bw, bs, bo, bm;
    if ((st = dev_alloc(bw, ctx->stream, static_cast<size_t>(k * k), &w)) != RL_OK) return st;
    if ((st = dev_alloc(bs, ctx->stream, static_cast<size_t>(k), &sv)) != RL_OK) return st;
    if ((st = dev_alloc(bo, ctx->stream, static_cast<size_t>(2 * (k + 1)), &order)) != RL_OK) return st;
    if ((st = dev_alloc(bm, ctx->stream, 1, &mn)) != RL_OK) return st;
    jacobi_sv_kernel<<<1, JT, 0, ctx->stream>>>(blk, ld, static_cast<int>(k), static_cast<int>(k), w, order, sv);
    RL_CHECK_LAUNCH("jacobi_sv_kernel");
    min_kernel<<<1, 256, 0, ctx->stream>>>(sv, static_cast<int>(k), mn);
    RL_CHECK_LAUNCH("min_kernel");
    RL_CUDA(cudaMemcpyAsync(out, mn, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    RL_CUDA(cudaStreamSynchronize(ctx->stream));
    return RL_OK;
}

rl_status gepp_solve(rl_context* ctx, const double* lu, int64_t ld, int64_t n, const int64_t* perm, const double* in,
                     int64_t in_rs, int64_t in_es, double* out, int64_t out_rs, int64_t out_es, int64_t nrhs,
                     bool transpose) {
    if (nrhs <= 0) return RL_OK;
    double* work = nullptr;
    DevBuf bw;
    rl_status st;
    if ((st = dev_alloc(bw, ctx->stream, static_cast<size_t>(nrhs * n), &work)) != RL_OK) return st;
    gepp_solve_kernel<<<nblocks(nrhs, 64), 64, 0, ctx->stream>>>(lu, ld, static_cast<int>(n), perm, in, in_rs, in_es,
                                                                out, out_rs, out_es, nrhs, transpose ? 1 : 0, work);
    RL_CHECK_LAUNCH("gepp_solve_kernel");
    return RL_OK;
}

}  // namespace rl

using namespace rl;

namespace {
rl_status check_split(int64_t n, int64_t nsplit, const int64_t* split) {
    if (nsplit <= 0 || !split) return set_error(RL_ERR_DIMENSION, "block_ge_factor: split must sum to the dimension");
    int64_t s = 0;
    for (int64_t i = 0; i < nsplit; ++i) {
        if (split[i] <= 0) return set_error(RL_ERR_DIMENSION, "block_ge_factor: zero block size");
        s += split[i];
    }
    if (s != n) return set_error(RL_ERR_DIMENSION, "block_ge_factor: split must sum to the dimension");
    return RL_OK;
}
}  // namespace

extern "C" RL_API rl_status rl_gepp_factor(rl_context* ctx, rl_mem mem, int64_t n, const double* a, double* lu,
                                           int64_t* perm, int64_t* singular_step) {
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "gepp_factor: square input required");
    if (!a || !lu || !perm) return set_error(RL_ERR_INVALID_ARGUMENT, "gepp_factor: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    double* dlu = lu;
    int64_t* dperm = perm;
    DevBuf b1, b2;
    if (mem == RL_HOST) {
        if ((st = dev_alloc(b1, s, static_cast<size_t>(n * n), &dlu)) != RL_OK) return st;
        if ((st = dev_alloc(b2, s, static_cast<size_t>(n), &dperm)) != RL_OK) return st;
        RL_CUDA(cudaMemcpyAsync(dlu, a, n * n * 8, cudaMemcpyHostToDevice, s));
    } else if (lu != a) {
        RL_CUDA(cudaMemcpyAsync(dlu, a, n * n * 8, cudaMemcpyDeviceToDevice, s));
    }
    int64_t bad = 0;
    st = gepp_inplace(ctx, n, dlu, n, dperm, &bad);
    if (singular_step) *singular_step = bad;
    if (st != RL_OK) return st;
    if (mem == RL_HOST) {
        RL_CUDA(cudaMemcpyAsync(lu, dlu, n * n * 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaMemcpyAsync(perm, dperm, n * 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaStreamSynchronize(s));
    }
    return RL_OK;
}

extern "C" RL_API rl_status rl_gepp_solve(rl_context* ctx, rl_mem mem, int64_t n, int64_t nrhs, const double* lu,
                                          const int64_t* perm, const double* b, double* x, int32_t transpose) {
    if (n <= 0 || nrhs < 0) return set_error(RL_ERR_DIMENSION, "lu_solve: length mismatch");
    if (nrhs == 0) return RL_OK;
    if (!lu || !perm || !b || !x) return set_error(RL_ERR_INVALID_ARGUMENT, "lu_solve: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const double *dlu = lu, *db = b;
    const int64_t* dperm = perm;
    double* dx = x;
    DevBuf b1, b2, b3, b4;
    if (mem == RL_HOST) {
        double *t1, *t3, *t4;
        int64_t* t2;
        if ((st = dev_alloc(b1, s, static_cast<size_t>(n * n), &t1)) != RL_OK) return st;
        if ((st = dev_alloc(b2, s, static_cast<size_t>(n), &t2)) != RL_OK) return st;
        if ((st = dev_alloc(b3, s, static_cast<size_t>(n * nrhs), &t3)) != RL_OK) return st;
        if ((st = dev_alloc(b4, s, static_cast<size_t>(n * nrhs), &t4)) != RL_OK) return st;
        RL_CUDA(cudaMemcpyAsync(t1, lu, n * n * 8, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaMemcpyAsync(t2, perm, n * 8, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaMemcpyAsync(t3, b, n * nrhs * 8, cudaMemcpyHostToDevice, s));
        dlu = t1;
        dperm = t2;
        db = t3;
        dx = t4;
    }
    // right-hand side r is column r of the n x nrhs row-major b (and x)
    if ((st = gepp_solve(ctx, dlu, n, n, dperm, db, 1, nrhs, dx, 1, nrhs, nrhs, transpose != 0)) != RL_OK) return st;
    if (mem == RL_HOST) {
        RL_CUDA(cudaMemcpyAsync(x, dx, n * nrhs * 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaStreamSynchronize(s));
    }
    return RL_OK;
}

extern "C" RL_API rl_status rl_block_ge_factor(rl_context* ctx, rl_mem mem, int64_t n, const double* a, int64_t nsplit,
                                               const int64_t* split, double* factors, int64_t* perm,
                                               double* leaf_blocks, int64_t* position) {
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "block_ge_factor: square input required");
    rl_status st = check_split(n, nsplit, split);
    if (st != RL_OK) return st;
    if (!a || !factors || !perm) return set_error(RL_ERR_INVALID_ARGUMENT, "block_ge_factor: null pointer");
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    if (position) *position = 0;
    cudaStream_t s = ctx->stream;
    // work: the current Schur complement in place of a copy of a; f: factors
    double *work = nullptr, *f = factors, *leaves = leaf_blocks;
    int64_t* dperm = perm;
    DevBuf bw, bf, bp, bl;
    if ((st = dev_alloc(bw, s, static_cast<size_t>(n * n), &work)) != RL_OK) return st;
    if (mem == RL_HOST) {
        if ((st = dev_alloc(bf, s, static_cast<size_t>(n * n), &f)) != RL_OK) return st;
        if ((st = dev_alloc(bp, s, static_cast<size_t>(n), &dperm)) != RL_OK) return st;
        if (leaf_blocks && (st = dev_alloc(bl, s, static_cast<size_t>(n * n), &leaves)) != RL_OK) return st;
    }
    RL_CUDA(cudaMemcpyAsync(work, a, n * n * 8, mem == RL_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    RL_CUDA(cudaMemsetAsync(f, 0, n * n * 8, s));
    if (leaves) RL_CUDA(cudaMemsetAsync(leaves, 0, n * n * 8, s));
    // singular_tol = tol_pivot(n) * spectral_norm_estimate(a) (block_ge.hpp:176)
    double est = 0.0;
    if ((st = spectral_norm_estimate_device(ctx, n, n, work, n, &est)) != RL_OK) return st;
    const double tol = 1e-13 * static_cast<double>(n) * est;
    int64_t o = 0;
    for (int64_t lvl = 0; lvl < nsplit; ++lvl) {
        const bool last = lvl + 1 == nsplit;
        const int64_t k = last ? n - o : split[lvl], rest = n - o - k;
        double* B = work + o * n + o;
        if (leaves) {
            copy_block_kernel<<<nblocks(k * k, 256), 256, 0, s>>>(B, n, leaves + o * n + o, n, k, k);
            RL_CHECK_LAUNCH("copy_block_kernel");
        }
        // leaf: svd_values(B).back() <= tol -> SingularPivotBlockError(offset + 1)
        double smin = 0.0;
        if ((st = min_singular_value(ctx, k, B, n, &smin)) != RL_OK) return st;
        if (smin <= tol) {
            if (position) *position = o + 1;
            return set_error(RL_ERR_SINGULAR_PIVOT_BLOCK, "block_ge_factor: singular pivot block at %lld",
                             static_cast<long long>(o + 1));
        }
        // the leaf's GEPP factors, in the diagonal block of f
        double* FB = f + o * n + o;
        copy_block_kernel<<<nblocks(k * k, 256), 256, 0, s>>>(B, n, FB, n, k, k);
        RL_CHECK_LAUNCH("copy_block_kernel");
        int64_t bad = 0;
        if ((st = gepp_inplace(ctx, k, FB, n, dperm + o, &bad)) != RL_OK) {
            if (position) *position = o + bad;
            return st;
        }
        if (rest > 0) {
            const double* C = work + o * n + o + k;  // k x rest
            const double* D = work + (o + k) * n + o;  // rest x k
            // B^-1 C column by column (block_ge.hpp:116-120) -> f rows [o, o+k), right
            if ((st = gepp_solve(ctx, FB, n, k, dperm + o, C, 1, n, f + o * n + o + k, 1, n, rest, false)) != RL_OK)
                return st;
            // D B^-1 row by row (block_ge.hpp:121-125) -> f columns [o, o+k), below
            if ((st = gepp_solve(ctx, FB, n, k, dperm + o, D, n, 1, f + (o + k) * n + o, n, 1, rest, true)) != RL_OK)
                return st;
            // S = E - (D B^-1) C in place of E (block_ge.hpp:126-134)
            const dim3 grid(nblocks(rest, ST), nblocks(rest, ST));
            schur_natural_kernel<<<grid, dim3(ST, 8), 0, s>>>(work + (o + k) * n + o + k, n, f + (o + k) * n + o, n, C, n,
                                                              rest, rest, k);
            RL_CHECK_LAUNCH("schur_natural_kernel");
        }
        o += k;
    }
    if (mem == RL_HOST) {
        RL_CUDA(cudaMemcpyAsync(factors, f, n * n * 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaMemcpyAsync(perm, dperm, n * 8, cudaMemcpyDeviceToHost, s));
        if (leaf_blocks) RL_CUDA(cudaMemcpyAsync(leaf_blocks, leaves, n * n * 8, cudaMemcpyDeviceToHost, s));
    }
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}

extern "C" RL_API rl_status rl_block_solve(rl_context* ctx, rl_mem mem, int64_t n, int64_t nsplit, const int64_t* split,
                                           const double* factors, const int64_t* perm, const double* b, double* x) {
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "block_solve: length mismatch");
    rl_status st = check_split(n, nsplit, split);
    if (st != RL_OK) return st;
    if (!factors || !perm || !b || !x) return set_error(RL_ERR_INVALID_ARGUMENT, "block_solve: null pointer");
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const double* f = factors;
    const int64_t* dperm = perm;
    double *v = nullptr, *t = nullptr, *xs = x;
    DevBuf bf, bp, bv, bt, bx;
    if (mem == RL_HOST) {
        double* tf;
        int64_t* tp;
        if ((st = dev_alloc(bf, s, static_cast<size_t>(n * n), &tf)) != RL_OK) return st;
        if ((st = dev_alloc(bp, s, static_cast<size_t>(n), &tp)) != RL_OK) return st;
        if ((st = dev_alloc(bx, s, static_cast<size_t>(n), &xs)) != RL_OK) return st;
        RL_CUDA(cudaMemcpyAsync(tf, factors, n * n * 8, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaMemcpyAsync(tp, perm, n * 8, cudaMemcpyHostToDevice, s));
        f = tf;
        dperm = tp;
    }
    if ((st = dev_alloc(bv, s, static_cast<size_t>(n), &v)) != RL_OK) return st;
    if ((st = dev_alloc(bt, s, static_cast<size_t>(n), &t)) != RL_OK) return st;
    RL_CUDA(cudaMemcpyAsync(v, b, n * 8, mem == RL_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    // block_solve_node on the right spine: going down, u2 -= (D B^-1) v1 at
    // each level (v then holds v1 | u2 in place); at the leaf lu_solve; going
    // up, w1 = lu_solve(B, v1) and x1 = w1 - (B^-1 C) w2.
    std::vector<int64_t> off, ks;
    int64_t o = 0;
    for (int64_t lvl = 0; lvl < nsplit; ++lvl) {
        const int64_t k = lvl + 1 == nsplit ? n - o : split[lvl];
        off.push_back(o);
        ks.push_back(k);
        o += k;
    }
    const int64_t L = static_cast<int64_t>(off.size());
    for (int64_t lvl = 0; lvl + 1 < L; ++lvl) {
        const int64_t oo = off[lvl], k = ks[lvl], rest = n - oo - k;
        row_update_kernel<<<nblocks(rest, 128), 128, 0, s>>>(v + oo + k, f + (oo + k) * n + oo, n, v + oo, rest, k);
        RL_CHECK_LAUNCH("row_update_kernel");
    }
    for (int64_t lvl = L - 1; lvl >= 0; --lvl) {
        const int64_t oo = off[lvl], k = ks[lvl], rest = n - oo - k;
        // w1 = lu_solve(B, v1) -> t[oo, oo+k)
        if ((st = gepp_solve(ctx, f + oo * n + oo, n, k, dperm + oo, v + oo, 0, 1, t + oo, 0, 1, 1, false)) != RL_OK)
            return st;
        if (rest > 0) {
            // x1 = w1 - (B^-1 C) w2, w2 = t[oo+k, n) (already final)
            row_update_kernel<<<nblocks(k, 128), 128, 0, s>>>(t + oo, f + oo * n + oo + k, n, t + oo + k, k, rest);
            RL_CHECK_LAUNCH("row_update_kernel");
        }
    }
    RL_CUDA(cudaMemcpyAsync(xs, t, n * 8, cudaMemcpyDeviceToDevice, s));
    if (mem == RL_HOST) RL_CUDA(cudaMemcpyAsync(x, xs, n * 8, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}

// svd_values (svd.hpp:76-88): the min(m, n) singular values, non-increasing,
// by the one-sided Jacobi kernel (on a^T when m < n: same values)
extern "C" RL_API rl_status rl_singular_values(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                               double* out) {
    if (m <= 0 || n <= 0) return set_error(RL_ERR_DIMENSION, "svd_values: empty matrix");
    if (!a || !out) return set_error(RL_ERR_INVALID_ARGUMENT, "svd_values: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    const int64_t r = std::min(m, n), c = std::max(m, n);  // operate on the tall orientation (c x r)
    double *da = nullptr, *w = nullptr, *sv = nullptr, *tall = nullptr;
    int* order = nullptr;
    DevBuf ba, bw, bs, bo, bt;
    if ((st = dev_alloc(ba, s, static_cast<size_t>(m * n), &da)) != RL_OK) return st;
    if ((st = dev_alloc(bt, s, static_cast<size_t>(m * n), &tall)) != RL_OK) return st;
    if ((st = dev_alloc(bw, s, static_cast<size_t>(m * n), &w)) != RL_OK) return st;
    if ((st = dev_alloc(bs, s, static_cast<size_t>(r), &sv)) != RL_OK) return st;
    if ((st = dev_alloc(bo, s, static_cast<size_t>(2 * (r + 1)), &order)) != RL_OK) return st;
    RL_CUDA(cudaMemcpyAsync(da, a, m * n * 8, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    const double* src = da;
    if (m < n) {
        if ((st = transpose_device(ctx, da, n, m, n, tall, m)) != RL_OK) return st;
        src = tall;
    }
    jacobi_sv_kernel<<<1, JT, 0, s>>>(src, r, static_cast<int>(c), static_cast<int>(r), w, order, sv);
    RL_CHECK_LAUNCH("jacobi_sv_kernel");
    std::vector<double> h(static_cast<size_t>(r));
    RL_CUDA(cudaMemcpyAsync(h.data(), sv, r * 8, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    std::sort(h.begin(), h.end(), [](double x, double y) { return x > y; });
    if (host) {
        std::memcpy(out, h.data(), r * 8);
    } else {
        RL_CUDA(cudaMemcpyAsync(out, h.data(), r * 8, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaStreamSynchronize(s));
    }
    return RL_OK;
}
