// The complex field (randla's Matrix<Complex> instantiations) on sm_100a:
// the unitary circulant, unitary Toeplitz block and
// SRFT families, and the complex pipelines they run in:
//
//   rl_zpreprocessed_genp_solve  preprocess_solve<Complex> (preprocess.hpp:156-180)
//                                with SideMultiplier<Complex>::make (:27-60)
//   rl_zrange_find_residual      range_find<Complex> (lowrank.hpp:62-83) and
//   rl_zapproximation_residual   approximation_residual (:99-102)
//   rl_srft_sketch_check         srft_sketch_check (lowrank.hpp:216-261)
//   rl_zmaterialize              materialize<Complex> (multipliers.hpp:174-218)
//   rl_gen_unitary_circulant     gen_unitary_circulant (multipliers.hpp:75-82)
//   rl_zsingular_values          svd_values<Complex> (svd.hpp:76-88)
//
// Layouts. Complex data at the boundary is interleaved (re, im) doubles, the
// std::complex<double> layout. Complex products run on the FP64 DMMA GEMM
// through real block forms with no redundant flops:
//   C = A B      as [Ar | Ai] (m x 2k) * [[Br, Bi], [-Bi, Br]] (2k x 2n) = [Cr | Ci]
//   C = A B_real as [Ar ; Ai] (2m x k) * B (k x n)                     = [Cr ; Ci]
//   C = A_real B as A (m x k) * [Br | Bi] (k x 2n)                     = [Cr | Ci]
// GENP keeps the product in a "panel-planar" layout W (n x 2n real): column
// block b (64 complex columns, or the ragged rest) stores its real parts then
// its imaginary parts, so a panel's [L21r | L21i] is one contiguous K = 128
// operand and the trailing update A22 -= L21 U12 is ONE real GEMM
// (M = rest, N = 2 rest, K = 128) against [[U12r, U12i], [-U12i, U12r]] laid
// out in W's column order. The diagonal block (complex GENP in shared
// memory), L21 (row substitution) and U12 (column substitution) are complex
// kernels.
// The low-rank path runs the real CholeskyQR2 / residual machinery on the
// real embedding E(M) = [[Mr, -Mi], [Mi, Mr]]: with the sketch's columns
// ordered (y_1, i y_1, y_2, i y_2, ...), real Gram-Schmidt of E(Y) reproduces
// complex Gram-Schmidt of Y (every other column is the complex basis vector
// with positive real R diagonal, the normalisation of qr.hpp:33-45), and
// E(A) - Q_E Q_E^T E(A) = E(A - Q Q^H A), whose singular values are those of
// the complex residual, each twice.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "device_common.cuh"
#include "kernels.cuh"

extern "C" RL_API rl_status rl_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double* out);
extern "C" RL_API rl_status rl_gen_real_circulant_column(int64_t n, uint64_t seed, double* out);
extern "C" RL_API rl_status rl_singular_values(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                               double* out);

namespace rl {
void host_unit_spectrum(uint64_t seed, int64_t n, double* u2);
void host_srft_columns(uint64_t seed, int64_t n, int64_t l, int64_t* cols);
void host_srft_parts(uint64_t seed, int64_t n, int64_t l, double* d2, double* root2, int64_t* cols);

namespace {

constexpr int ZB = 64;   // complex panel width
constexpr int ZPT = 128; // threads per panel CTA
constexpr int ZQ = 4;    // threads per row / column in the substitutions
constexpr int ZLD = ZB + 1;
constexpr size_t kZPanelSmem = sizeof(double2) * ZB * ZLD + sizeof(double2) * ZB;

unsigned nblk(int64_t n, int t) { return static_cast<unsigned>(std::max<int64_t>(1, (n + t - 1) / t)); }
int64_t even(int64_t x) { return (x + 1) & ~int64_t(1); }

// ---- complex arithmetic ---------------------------------------------------
__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a - b c
__device__ __forceinline__ double2 zfms(double2 a, double2 b, double2 c) {
    return make_double2(fma(-b.x, c.x, fma(b.y, c.y, a.x)), fma(-b.x, c.y, fma(-b.y, c.x, a.y)));
}
// 1 / p, scaled against overflow (p = 0 gives inf / nan, which the verdict flags)
__device__ __forceinline__ double2 zrcp(double2 p) {
    const double s = fmax(fabs(p.x), fabs(p.y));
    const double a = p.x / s, b = p.y / s;
    const double d = s * fma(a, a, b * b);
    return make_double2(a / d, -b / d);
}
__device__ __forceinline__ double zabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ double2 shfl2(double2 v, int src, unsigned mask = kFull) {
    return make_double2(__shfl_sync(mask, v.x, src), __shfl_sync(mask, v.y, src));
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(kFull, v.x, o);
        v.y += __shfl_xor_sync(kFull, v.y, o);
    }
    return v;
}

// W column of complex column j, part 0 (re) / 1 (im)
__host__ __device__ __forceinline__ int64_t wcol(int64_t j, int64_t n, int part) {
    const int64_t b = j / ZB, t = j - b * ZB;
    const int64_t w = n - b * ZB < ZB ? n - b * ZB : ZB;
    return 2 * ZB * b + part * w + t;
}

// ---- layout kernels (grid-stride over the m x n complex entries) -----------
enum class Pack { ROWPLANAR, STACKED, EMBED_B, W };
__global__ void pack_kernel(const double2* __restrict__ z, int64_t ldz, int64_t m, int64_t n, double* __restrict__ r,
                            int64_t ldr, Pack mode, int conj) {
    const int64_t total = m * n;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / n, j = idx - i * n;
        double2 v = z[i * ldz + j];
        if (conj) v.y = -v.y;
        switch (mode) {
            case Pack::ROWPLANAR:  // [Re | Im] (m x 2n)
                r[i * ldr + j] = v.x;
                r[i * ldr + n + j] = v.y;
                break;
            case Pack::STACKED:  // [Re ; Im] (2m x n)
                r[i * ldr + j] = v.x;
                r[(m + i) * ldr + j] = v.y;
                break;
            case Pack::EMBED_B:  // [[Re, Im], [-Im, Re]] (2m x 2n)
                r[i * ldr + j] = v.x;
                r[i * ldr + n + j] = v.y;
                r[(m + i) * ldr + j] = -v.y;
                r[(m + i) * ldr + n + j] = v.x;
                break;
            case Pack::W:  // panel-planar (square n x n)
                r[i * ldr + wcol(j, n, 0)] = v.x;
                r[i * ldr + wcol(j, n, 1)] = v.y;
                break;
        }
    }
}
__global__ void unpack_kernel(const double* __restrict__ r, int64_t ldr, int64_t m, int64_t n, double2* __restrict__ z,
                              int64_t ldz, Pack mode) {
    const int64_t total = m * n;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / n, j = idx - i * n;
        double2 v;
        if (mode == Pack::ROWPLANAR) {
            v = make_double2(r[i * ldr + j], r[i * ldr + n + j]);
        } else if (mode == Pack::STACKED) {
            v = make_double2(r[i * ldr + j], r[(m + i) * ldr + j]);
        } else {
            v = make_double2(r[i * ldr + wcol(j, n, 0)], r[i * ldr + wcol(j, n, 1)]);
        }
        z[i * ldz + j] = v;
    }
}
// real (m x n) -> complex with zero imaginary parts (to_complex, matrix.hpp)
__global__ void lift_kernel(const double* __restrict__ r, int64_t ldr, int64_t m, int64_t n, double2* __restrict__ z,
                            int64_t ldz) {
    const int64_t total = m * n;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / n, j = idx - i * n;
        z[i * ldz + j] = make_double2(r[i * ldr + j], 0.0);
    }
}
// out (n x m) = op(in) (m x n): plain or conjugate transpose
__global__ void ztranspose_kernel(const double2* __restrict__ in, int64_t ldi, int64_t m, int64_t n,
                                  double2* __restrict__ out, int64_t ldo, int conj) {
    __shared__ double2 t[32][33];
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < m && c < n) {
            double2 v = in[r * ldi + c];
            if (conj) v.y = -v.y;
            t[i][threadIdx.x] = v;
        }
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < m && c < n) out[c * ldo + r] = t[threadIdx.x][i];
    }
}

unsigned grid_for(int64_t total) { return static_cast<unsigned>(std::min<int64_t>(nblk(total, 256), 148 * 16)); }

rl_status pack(rl_context* ctx, const double2* z, int64_t ldz, int64_t m, int64_t n, double* r, int64_t ldr, Pack mode,
               bool conj = false) {
    pack_kernel<<<grid_for(m * n), 256, 0, ctx->stream>>>(z, ldz, m, n, r, ldr, mode, conj ? 1 : 0);
    RL_CHECK_LAUNCH("pack_kernel");
    return RL_OK;
}
rl_status unpack(rl_context* ctx, const double* r, int64_t ldr, int64_t m, int64_t n, double2* z, int64_t ldz,
                 Pack mode) {
    unpack_kernel<<<grid_for(m * n), 256, 0, ctx->stream>>>(r, ldr, m, n, z, ldz, mode);
    RL_CHECK_LAUNCH("unpack_kernel");
    return RL_OK;
}
rl_status lift(rl_context* ctx, const double* r, int64_t ldr, int64_t m, int64_t n, double2* z, int64_t ldz) {
    lift_kernel<<<grid_for(m * n), 256, 0, ctx->stream>>>(r, ldr, m, n, z, ldz);
    RL_CHECK_LAUNCH("lift_kernel");
    return RL_OK;
}
rl_status ztranspose(rl_context* ctx, const double2* in, int64_t ldi, int64_t m, int64_t n, double2* out, int64_t ldo,
                     bool conj) {
    ztranspose_kernel<<<dim3(nblk(n, 32), nblk(m, 32)), dim3(32, 8), 0, ctx->stream>>>(in, ldi, m, n, out, ldo,
                                                                                      conj ? 1 : 0);
    RL_CHECK_LAUNCH("ztranspose_kernel");
    return RL_OK;
}

// ---- complex products on the DMMA GEMM --------------------------------------
// C (m x n) = A (m x k) B (k x n), all complex
rl_status zgemm_cc(rl_context* ctx, int64_t m, int64_t n, int64_t k, const double2* A, int64_t lda, const double2* B,
                   int64_t ldb, double2* C, int64_t ldc) {
    cudaStream_t s = ctx->stream;
    StreamBuf ba(s), bb(s), bc(s);
    rl_status st;
    const int64_t la = 2 * k, lb = 2 * n;
    if ((st = ba.alloc(8 * m * la)) != RL_OK || (st = bb.alloc(8 * 2 * k * lb)) != RL_OK ||
        (st = bc.alloc(8 * m * lb)) != RL_OK)
        return st;
    if ((st = pack(ctx, A, lda, m, k, ba.p, la, Pack::ROWPLANAR)) != RL_OK) return st;
    if ((st = pack(ctx, B, ldb, k, n, bb.p, lb, Pack::EMBED_B)) != RL_OK) return st;
    if ((st = gemm(ctx, m, 2 * n, 2 * k, ba.p, la, bb.p, lb, bc.p, lb, 1.0, false, nullptr)) != RL_OK) return st;
    return unpack(ctx, bc.p, lb, m, n, C, ldc, Pack::ROWPLANAR);
}
// C (m x n) = A (m x k, complex) B (k x n, real, ldb even, 16-byte aligned)
rl_status zgemm_cr(rl_context* ctx, int64_t m, int64_t n, int64_t k, const double2* A, int64_t lda, const double* B,
                   int64_t ldb, double2* C, int64_t ldc) {
    cudaStream_t s = ctx->stream;
    StreamBuf ba(s), bc(s);
    rl_status st;
    const int64_t la = even(k), lc = even(n);
    if ((st = ba.alloc(8 * 2 * m * la)) != RL_OK || (st = bc.alloc(8 * 2 * m * lc)) != RL_OK) return st;
    if ((st = pack(ctx, A, lda, m, k, ba.p, la, Pack::STACKED)) != RL_OK) return st;
    if ((st = gemm(ctx, 2 * m, n, k, ba.p, la, B, ldb, bc.p, lc, 1.0, false, nullptr)) != RL_OK) return st;
    return unpack(ctx, bc.p, lc, m, n, C, ldc, Pack::STACKED);
}
// C (m x n) = A (m x k, real, lda even, aligned) B (k x n, complex)
rl_status zgemm_rc(rl_context* ctx, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double2* B,
                   int64_t ldb, double2* C, int64_t ldc) {
    cudaStream_t s = ctx->stream;
    StreamBuf bb(s), bc(s);
    rl_status st;
    const int64_t lb = 2 * n;
    if ((st = bb.alloc(8 * k * lb)) != RL_OK || (st = bc.alloc(8 * m * lb)) != RL_OK) return st;
    if ((st = pack(ctx, B, ldb, k, n, bb.p, lb, Pack::ROWPLANAR)) != RL_OK) return st;
    if ((st = gemm(ctx, m, 2 * n, k, A, lda, bb.p, lb, bc.p, lb, 1.0, false, nullptr)) != RL_OK) return st;
    return unpack(ctx, bc.p, lb, m, n, C, ldc, Pack::ROWPLANAR);
}

// ---- complex GENP on the panel-planar layout ---------------------------------
// load / store the w x w complex diagonal block of panel kb into sd
__device__ __forceinline__ void load_diag(const double* __restrict__ W, int64_t ldw, int64_t c0, int64_t base, int w,
                                          double2 (*sd)[ZLD], int tid) {
    for (int idx = tid; idx < w * w; idx += ZPT) {
        const int i = idx / w, j = idx - i * w;
        const double* row = W + (c0 + i) * ldw + base;
        sd[i][j] = make_double2(row[j], row[w + j]);
    }
}

// Every CTA factors the w x w diagonal block (genp_factor, lu.hpp:47-56,
// l = u_ij / piv as u_ij * (1 / piv)) in shared memory; CTA 0 stores it and
// the pivots; row CTAs then form their rows of L21 = A21 U11^-1 (x U11 = a,
// ZQ threads per row, the owner of column j scales, the group shares x_j).
__global__ void __launch_bounds__(ZPT)
zpanel_kernel(double* __restrict__ W, int64_t ldw, int64_t n, int64_t c0, int w, int row_ctas,
              double2* __restrict__ piv, double2* __restrict__ rinv) {
    extern __shared__ __align__(16) unsigned char zsm[];
    double2 (*sd)[ZLD] = reinterpret_cast<double2 (*)[ZLD]>(zsm);
    double2* sr = reinterpret_cast<double2*>(zsm + sizeof(double2) * ZB * ZLD);
    const int tid = threadIdx.x;
    const int64_t base = 2 * c0;  // W column of the panel block (c0 is a multiple of ZB)
    load_diag(W, ldw, c0, base, w, sd, tid);
    __syncthreads();
    for (int j = 0; j < w; ++j) {
        const double2 rp = zrcp(sd[j][j]);
        if (tid == 0) sr[j] = rp;
        for (int i = j + 1 + tid; i < w; i += ZPT) sd[i][j] = zmul(sd[i][j], rp);
        __syncthreads();
        const int cnt = w - j - 1;
        for (int idx = tid; idx < cnt * cnt; idx += ZPT) {
            const int i = j + 1 + idx / cnt, k = j + 1 + idx % cnt;
            sd[i][k] = zfms(sd[i][k], sd[i][j], sd[j][k]);
        }
        __syncthreads();
    }
    const int b = blockIdx.x;
    if (b == 0) {
        for (int idx = tid; idx < w * w; idx += ZPT) {
            const int i = idx / w, j = idx - i * w;
            double* row = W + (c0 + i) * ldw + base;
            row[j] = sd[i][j].x;
            row[w + j] = sd[i][j].y;
        }
        for (int j = tid; j < w; j += ZPT) {
            piv[c0 + j] = sd[j][j];
            rinv[c0 + j] = sr[j];
        }
    }
    if (b >= row_ctas) return;
    constexpr int RPC = ZPT / ZQ, NS = ZB / ZQ;
    const int q = tid % ZQ, lane = tid & 31;
    const int64_t r = c0 + w + static_cast<int64_t>(b) * RPC + tid / ZQ;
    if (r >= n) return;  // whole groups leave together
    const unsigned gm = ((1u << ZQ) - 1u) << (lane & ~(ZQ - 1));
    double* rowp = W + r * ldw + base;
    double2 x[NS];
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) {
        const int t = q + ZQ * s2;
        x[s2] = t < w ? make_double2(rowp[t], rowp[w + t]) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < ZB; ++j) {
        if (j < w) {
            const int s = j / ZQ, owner = j % ZQ;
            if (q == owner) x[s] = zmul(x[s], sr[j]);  // l_rj (lu.hpp:51)
            const double2 xj = shfl2(x[s], (lane & ~(ZQ - 1)) | owner, gm);
            if (q > owner) x[s] = zfms(x[s], xj, sd[j][q + ZQ * s]);
#pragma unroll
            for (int s2 = s + 1; s2 < NS; ++s2)
                if (q + ZQ * s2 < w) x[s2] = zfms(x[s2], xj, sd[j][q + ZQ * s2]);
        }
    }
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) {
        const int t = q + ZQ * s2;
        if (t < w) {
            rowp[t] = x[s2].x;
            rowp[w + t] = x[s2].y;
        }
    }
}

// U12 = L11^-1 A12 for the trailing columns (forward substitution down each
// column, ZQ threads per column), stored in W and in the GEMM operand
// B = [[U12r, U12i], [-U12i, U12r]] (2w x 2 rest) in W's column order
__global__ void __launch_bounds__(ZPT)
zu12_kernel(double* __restrict__ W, int64_t ldw, int64_t n, int64_t c0, int w, double* __restrict__ B, int64_t ldb) {
    extern __shared__ __align__(16) unsigned char zsm[];
    double2 (*sd)[ZLD] = reinterpret_cast<double2 (*)[ZLD]>(zsm);
    const int tid = threadIdx.x;
    const int64_t base = 2 * c0;
    load_diag(W, ldw, c0, base, w, sd, tid);
    __syncthreads();
    constexpr int CPC = ZPT / ZQ, NS = ZB / ZQ;
    const int q = tid % ZQ, lane = tid & 31;
    const int64_t c = c0 + w + static_cast<int64_t>(blockIdx.x) * CPC + tid / ZQ;
    if (c >= n) return;
    const unsigned gm = ((1u << ZQ) - 1u) << (lane & ~(ZQ - 1));
    const int64_t cre = wcol(c, n, 0), cim = wcol(c, n, 1);
    double2 x[NS];
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) {
        const int t = q + ZQ * s2;
        x[s2] = t < w ? make_double2(W[(c0 + t) * ldw + cre], W[(c0 + t) * ldw + cim]) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < ZB - 1; ++k) {
        if (k < w) {
            const int s = k / ZQ, owner = k % ZQ;
            const double2 xk = shfl2(x[s], (lane & ~(ZQ - 1)) | owner, gm);
            if (q > owner) x[s] = zfms(x[s], sd[q + ZQ * s][k], xk);
#pragma unroll
            for (int s2 = s + 1; s2 < NS; ++s2)
                if (q + ZQ * s2 < w) x[s2] = zfms(x[s2], sd[q + ZQ * s2][k], xk);
        }
    }
    const int64_t off = 2 * (c0 + w);  // W column where the trailing blocks start
    const int64_t bre = cre - off, bim = cim - off;
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) {
        const int t = q + ZQ * s2;
        if (t < w) {
            W[(c0 + t) * ldw + cre] = x[s2].x;
            W[(c0 + t) * ldw + cim] = x[s2].y;
            B[t * ldb + bre] = x[s2].x;
            B[t * ldb + bim] = x[s2].y;
            B[(w + t) * ldb + bre] = -x[s2].y;
            B[(w + t) * ldb + bim] = x[s2].x;
        }
    }
}

rl_status zgenp_configure() {
    static PerDeviceOnce once;
    return once_per_device(once, []() -> rl_status {
        RL_CUDA(cudaFuncSetAttribute(zpanel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kZPanelSmem)));
        RL_CUDA(cudaFuncSetAttribute(zu12_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kZPanelSmem)));
        return RL_OK;
    });
}

// right-looking blocked complex GENP of W (n x 2n panel-planar, ldw even) in
// place; piv / rinv (n complex) receive u_jj and 1 / u_jj. No verdict.
rl_status zgenp_inplace(rl_context* ctx, int64_t n, double* W, int64_t ldw, double2* piv, double2* rinv) {
    cudaStream_t s = ctx->stream;
    rl_status st;
    if ((st = zgenp_configure()) != RL_OK) return st;
    StreamBuf bb(s);
    if (n > ZB && (st = bb.alloc(8 * 2 * ZB * 2 * (n - ZB))) != RL_OK) return st;
    for (int64_t c0 = 0; c0 < n; c0 += ZB) {
        const int w = static_cast<int>(std::min<int64_t>(ZB, n - c0));
        const int64_t rest = n - c0 - w;
        const int row_ctas = static_cast<int>((rest + ZPT / ZQ - 1) / (ZPT / ZQ));
        zpanel_kernel<<<std::max(1, row_ctas), ZPT, kZPanelSmem, s>>>(W, ldw, n, c0, w, row_ctas, piv, rinv);
        RL_CHECK_LAUNCH("zpanel_kernel");
        if (rest <= 0) break;
        const int64_t ldb = 2 * rest;
        zu12_kernel<<<nblk(rest, ZPT / ZQ), ZPT, kZPanelSmem, s>>>(W, ldw, n, c0, w, bb.p, ldb);
        RL_CHECK_LAUNCH("zu12_kernel");
        // A22 -= L21 U12: [L21r | L21i] (rest x 2w) * B (2w x 2 rest), one real GEMM
        double* a21 = W + (c0 + w) * ldw + 2 * c0;
        double* a22 = W + (c0 + w) * ldw + 2 * (c0 + w);
        if ((st = gemm(ctx, rest, 2 * rest, 2 * w, a21, ldw, bb.p, ldb, a22, ldw, -1.0, true, nullptr)) != RL_OK)
            return st;
    }
    return RL_OK;
}

// ---- lu_solve (lu.hpp:100-122) on W, one CTA ---------------------------------
// forward (unit L) then backward (U, times 1/u_jj) in 32-row blocks: warp 0
// solves the diagonal block from shared memory, every warp folds the block
// into the remaining rows (one row per warp, a coalesced dot per row)
constexpr int TS = 1024;
__device__ __forceinline__ double2 wz(const double* __restrict__ W, int64_t ldw, int64_t n, int64_t i, int64_t j) {
    const double* row = W + i * ldw;
    return make_double2(row[wcol(j, n, 0)], row[wcol(j, n, 1)]);
}
__global__ void __launch_bounds__(TS)
zlu_solve_kernel(const double* __restrict__ W, int64_t ldw, int64_t n, const double2* __restrict__ rinv,
                 double2* __restrict__ y) {
    __shared__ double2 blk[32];
    __shared__ double2 dg[32][33];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // forward
    for (int64_t r0 = 0; r0 < n; r0 += 32) {
        const int nb = static_cast<int>(std::min<int64_t>(32, n - r0));
        for (int idx = tid; idx < nb * nb; idx += TS) {
            const int i = idx / nb, k = idx - i * nb;
            dg[i][k] = wz(W, ldw, n, r0 + i, r0 + k);
        }
        __syncthreads();
        if (warp == 0) {
            double2 v = lane < nb ? y[r0 + lane] : make_double2(0.0, 0.0);
            for (int k = 0; k < nb - 1; ++k) {
                const double2 vk = shfl2(v, k);
                if (lane > k && lane < nb) v = zfms(v, dg[lane][k], vk);
            }
            if (lane < nb) {
                blk[lane] = v;
                y[r0 + lane] = v;
            }
        }
        __syncthreads();
        for (int64_t i = r0 + nb + warp; i < n; i += TS / 32) {
            double2 acc = lane < nb ? zmul(wz(W, ldw, n, i, r0 + lane), blk[lane]) : make_double2(0.0, 0.0);
            acc = warp_sum2(acc);
            if (lane == 0) y[i] = make_double2(y[i].x - acc.x, y[i].y - acc.y);
        }
        __syncthreads();
    }
    // backward
    for (int64_t r0 = ((n - 1) / 32) * 32; r0 >= 0; r0 -= 32) {
        const int nb = static_cast<int>(std::min<int64_t>(32, n - r0));
        for (int idx = tid; idx < nb * nb; idx += TS) {
            const int i = idx / nb, k = idx - i * nb;
            dg[i][k] = wz(W, ldw, n, r0 + i, r0 + k);
        }
        __syncthreads();
        if (warp == 0) {
            double2 v = lane < nb ? y[r0 + lane] : make_double2(0.0, 0.0);
            for (int k = nb - 1; k >= 0; --k) {
                if (lane == k) v = zmul(v, rinv[r0 + k]);  // y_k / u_kk (lu.hpp:120)
                const double2 vk = shfl2(v, k);
                if (lane < k) v = zfms(v, dg[lane][k], vk);
            }
            if (lane < nb) {
                blk[lane] = v;
                y[r0 + lane] = v;
            }
        }
        __syncthreads();
        for (int64_t i = warp; i < r0; i += TS / 32) {
            double2 acc = lane < nb ? zmul(wz(W, ldw, n, i, r0 + lane), blk[lane]) : make_double2(0.0, 0.0);
            acc = warp_sum2(acc);
            if (lane == 0) y[i] = make_double2(y[i].x - acc.x, y[i].y - acc.y);
        }
        __syncthreads();
    }
}

__global__ void diag_rcp_kernel(const double2* __restrict__ lu, int64_t n, double2* __restrict__ rinv) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) rinv[j] = zrcp(lu[j * n + j]);
}

// ---- matvec / residual --------------------------------------------------------
// y = M v (M m x n complex, or real when mr != nullptr); y = b - M v when b given
__global__ void zgemv_kernel(const double2* __restrict__ M, const double* __restrict__ mr, int64_t ldm, int64_t m,
                             int64_t n, const double2* __restrict__ v, const double2* __restrict__ b,
                             double2* __restrict__ y) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
    if (i >= m) return;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t j = lane; j < n; j += 32) {
        const double2 mij = mr ? make_double2(mr[i * ldm + j], 0.0) : M[i * ldm + j];
        acc = make_double2(fma(mij.x, v[j].x, fma(-mij.y, v[j].y, acc.x)), fma(mij.x, v[j].y, fma(mij.y, v[j].x, acc.y)));
    }
    acc = warp_sum2(acc);
    if (lane == 0) y[i] = b ? make_double2(b[i].x - acc.x, b[i].y - acc.y) : acc;
}
rl_status zgemv(rl_context* ctx, int64_t m, int64_t n, const double2* M, const double* mr, int64_t ldm,
                const double2* v, const double2* b, double2* y) {
    zgemv_kernel<<<nblk(m, 8), 256, 0, ctx->stream>>>(M, mr, ldm, m, n, v, b, y);
    RL_CHECK_LAUNCH("zgemv_kernel");
    return RL_OK;
}
__global__ void zaxpy_kernel(double2* __restrict__ x, const double2* __restrict__ d, int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = make_double2(x[i].x + d[i].x, x[i].y + d[i].y);
}

// ---- circulants through the FFT (circulant.hpp:67-98, :171-203) -------------
// T (m x np) = rows of Z zero-padded to np
__global__ void pad_rows_kernel(const double2* __restrict__ z, int64_t ldz, int64_t m, int64_t k, int64_t np,
                                double2* __restrict__ t) {
    const int64_t total = m * np;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / np, j = idx - i * np;
        t[idx] = j < k ? z[i * ldz + j] : make_double2(0.0, 0.0);
    }
}
// y *= u per row (spectral_apply, circulant.hpp:67-73)
__global__ void spectral_scale_kernel(double2* __restrict__ t, int64_t m, int64_t np, const double2* __restrict__ u) {
    const int64_t total = m * np;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 a = t[idx], b = u[idx % np];
        t[idx] = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
    }
}
__global__ void take_cols_kernel(const double2* __restrict__ t, int64_t m, int64_t np, int64_t l,
                                 double2* __restrict__ out, int64_t ldo) {
    const int64_t total = m * l;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / l, j = idx - i * l;
        out[i * ldo + j] = t[i * np + j];
    }
}
// first column of the transposed circulant: c~[i] = c[(-i) mod n] (circulant.hpp:39-45)
__global__ void reverse_col_kernel(const double2* __restrict__ c, int64_t n, double2* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = c[(n - i) % n];
}
// dense expansion, entry (i, j) = c[(i - j) mod np] (circulant.hpp:27-36), rows x cols
__global__ void zcirc_dense_kernel(const double2* __restrict__ c, int64_t np, int64_t rows, int64_t cols,
                                   double2* __restrict__ out, int64_t ldo, const int64_t* __restrict__ colmap) {
    const int64_t total = rows * cols;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / cols, j0 = idx - i * cols;
        const int64_t j = colmap ? colmap[j0] : j0;
        out[i * ldo + j0] = c[((i - j) % np + np) % np];
    }
}
// gen_srft entries d_i * root[(i col_j) mod n] (multipliers.hpp:102-106), the
// complex product rounded as on the host (no FMA)
__global__ void srft_dense_kernel(const double2* __restrict__ d, const double2* __restrict__ root,
                                  const int64_t* __restrict__ cols, int64_t n, int64_t l, double2* __restrict__ out,
                                  int64_t ldo) {
    const int64_t total = n * l;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / l, j = idx - i * l;
        const double2 a = d[i], b = root[(i * cols[j]) % n];
        out[i * ldo + j] = make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
    }
}

// A structured circulant: its first column c (np complex) and the spectra
// fft(c) (circulant_apply) and fft(c~) (row products through C^T), device
struct ZCirc {
    int64_t np = 0;
    double2 *col = nullptr, *spec = nullptr, *spec_t = nullptr;
    StreamBuf buf;
    explicit ZCirc(cudaStream_t s) : buf(s) {}
};

rl_status spectrum_of(rl_context* ctx, const double2* c, int64_t np, double2* out) {
    RL_CUDA(cudaMemcpyAsync(out, c, np * 16, cudaMemcpyDeviceToDevice, ctx->stream));
    StreamBuf w(ctx->stream);
    rl_status st;
    const size_t wb = cfft_work_bytes(1, np);
    if (wb && (st = w.alloc(wb)) != RL_OK) return st;
    return cfft_device(ctx, 1, np, reinterpret_cast<double*>(out), false, w.p);
}

// fill zc from a complex first column already on the device at zc.col
rl_status zcirc_finish(rl_context* ctx, ZCirc& zc) {
    rl_status st;
    if ((st = spectrum_of(ctx, zc.col, zc.np, zc.spec)) != RL_OK) return st;
    StreamBuf rev(ctx->stream);
    if ((st = rev.alloc(zc.np * 16)) != RL_OK) return st;
    double2* r = reinterpret_cast<double2*>(rev.p);
    reverse_col_kernel<<<nblk(zc.np, 256), 256, 0, ctx->stream>>>(zc.col, zc.np, r);
    RL_CHECK_LAUNCH("reverse_col_kernel");
    return spectrum_of(ctx, r, zc.np, zc.spec_t);
}

// out (m x l) = rows of Z (m x k) padded to np, times the circulant whose
// spectrum is `u` (C^T for matmul_by_circulant / _toeplitz_block, C itself
// for circulant_apply), first l entries (circulant.hpp:171-203)
rl_status zcirc_rows(rl_context* ctx, int64_t m, int64_t k, const double2* Z, int64_t ldz, int64_t np,
                     const double2* u, int64_t l, double2* out, int64_t ldo) {
    cudaStream_t s = ctx->stream;
    StreamBuf bt(s), bw(s);
    rl_status st;
    if ((st = bt.alloc(16 * m * np)) != RL_OK) return st;
    const size_t wb = cfft_work_bytes(m, np);
    if (wb && (st = bw.alloc(wb)) != RL_OK) return st;
    double2* t = reinterpret_cast<double2*>(bt.p);
    pad_rows_kernel<<<grid_for(m * np), 256, 0, s>>>(Z, ldz, m, k, np, t);
    RL_CHECK_LAUNCH("pad_rows_kernel");
    if ((st = cfft_device(ctx, m, np, bt.p, false, bw.p)) != RL_OK) return st;
    spectral_scale_kernel<<<grid_for(m * np), 256, 0, s>>>(t, m, np, u);
    RL_CHECK_LAUNCH("spectral_scale_kernel");
    if ((st = cfft_device(ctx, m, np, bt.p, true, bw.p)) != RL_OK) return st;
    take_cols_kernel<<<grid_for(m * l), 256, 0, s>>>(t, m, np, l, out, ldo);
    RL_CHECK_LAUNCH("take_cols_kernel");
    return RL_OK;
}

// ---- complex multiplier specs ---------------------------------------------------
bool known_kind(int k) { return (k >= RL_MULT_NONE && k <= RL_MULT_CIRC_SKEW_PRODUCT) || k == RL_MULT_GAUSSIAN_CIRCULANT; }

// the column of a circulant-backed spec (np entries, complex, device):
// UnitaryCirculant / Unitary Toeplitz: inverse_fft(u) of the unit spectrum
// (multipliers.hpp:77-82); the real families: their real column lifted
rl_status zcirc_from_spec(rl_context* ctx, const rl_multiplier* m, int64_t np, bool host, ZCirc& zc) {
    cudaStream_t s = ctx->stream;
    rl_status st;
    zc.np = np;
    if ((st = zc.buf.alloc(16 * 3 * np)) != RL_OK) return st;
    zc.col = reinterpret_cast<double2*>(zc.buf.p);
    zc.spec = zc.col + np;
    zc.spec_t = zc.spec + np;
    const bool unitary = m->kind == RL_MULT_UNITARY_CIRCULANT ||
                         (m->kind == RL_MULT_TOEPLITZ_BLOCK && m->variant == RL_TOEPLITZ_UNITARY);
    std::vector<double> h(static_cast<size_t>(2 * np), 0.0);
    if (unitary) {
        host_unit_spectrum(m->seed, np, h.data());
        RL_CUDA(cudaMemcpyAsync(zc.col, h.data(), np * 16, cudaMemcpyHostToDevice, s));
        StreamBuf w(s);
        const size_t wb = cfft_work_bytes(1, np);
        if (wb && (st = w.alloc(wb)) != RL_OK) return st;
        if ((st = cfft_device(ctx, 1, np, reinterpret_cast<double*>(zc.col), true, w.p)) != RL_OK) return st;
    } else {
        std::vector<double> col;
        if ((st = multiplier_column(m, np, host, col)) != RL_OK) return st;
        for (int64_t i = 0; i < np; ++i) h[2 * i] = col[i];
        RL_CUDA(cudaMemcpyAsync(zc.col, h.data(), np * 16, cudaMemcpyHostToDevice, s));
    }
    if ((st = zcirc_finish(ctx, zc)) != RL_OK) return st;
    RL_CUDA(cudaStreamSynchronize(s));  // h is a local
    return RL_OK;
}

// materialize<Complex>(spec) with rows x cols into out (device, ldo complex)
rl_status zmaterialize_device(rl_context* ctx, const rl_multiplier* m, int64_t rows, int64_t cols, bool host,
                              double2* out, int64_t ldo) {
    cudaStream_t s = ctx->stream;
    rl_status st;
    if (!known_kind(m->kind)) return set_error(RL_ERR_INVALID_ARGUMENT, "unknown multiplier kind %d", m->kind);
    const bool unitary = m->kind == RL_MULT_UNITARY_CIRCULANT ||
                         (m->kind == RL_MULT_TOEPLITZ_BLOCK && m->variant == RL_TOEPLITZ_UNITARY);
    if (m->kind == RL_MULT_SRFT) {  // gen_srft(rows, cols, seed) (multipliers.hpp:123-130)
        if (cols < 1 || cols > rows) return set_error(RL_ERR_DIMENSION, "gen_srft: need 1 <= l <= n");
        std::vector<double> d(static_cast<size_t>(2 * rows)), root(static_cast<size_t>(2 * rows));
        std::vector<int64_t> idx(static_cast<size_t>(cols));
        host_srft_parts(m->seed, rows, cols, d.data(), root.data(), idx.data());
        StreamBuf b(s);
        if ((st = b.alloc(16 * 2 * rows + 8 * cols)) != RL_OK) return st;
        double2* dd = reinterpret_cast<double2*>(b.p);
        double2* dr = dd + rows;
        int64_t* dc = reinterpret_cast<int64_t*>(dr + rows);
        RL_CUDA(cudaMemcpyAsync(dd, d.data(), rows * 16, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaMemcpyAsync(dr, root.data(), rows * 16, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaMemcpyAsync(dc, idx.data(), cols * 8, cudaMemcpyHostToDevice, s));
        srft_dense_kernel<<<grid_for(rows * cols), 256, 0, s>>>(dd, dr, dc, rows, cols, out, ldo);
        RL_CHECK_LAUNCH("srft_dense_kernel");
        RL_CUDA(cudaStreamSynchronize(s));
        return RL_OK;
    }
    if (unitary) {
        if (m->kind == RL_MULT_UNITARY_CIRCULANT && rows != cols)
            return set_error(RL_ERR_DIMENSION, "circulant multiplier must be square");
        if (cols > rows) return set_error(RL_ERR_DIMENSION, "toeplitz block exceeds parent dimensions");
        ZCirc zc(s);
        if ((st = zcirc_from_spec(ctx, m, rows, host, zc)) != RL_OK) return st;
        zcirc_dense_kernel<<<grid_for(rows * cols), 256, 0, s>>>(zc.col, rows, rows, cols, out, ldo, nullptr);
        RL_CHECK_LAUNCH("zcirc_dense_kernel");
        RL_CUDA(cudaStreamSynchronize(s));
        return RL_OK;
    }
    // the real families, lifted (multipliers.hpp:180-186)
    StreamBuf b(s);
    const int64_t ld = even(cols);
    if ((st = b.alloc(8 * rows * ld)) != RL_OK) return st;
    if ((st = materialize_device(ctx, m, rows, cols, host, b.p, ld)) != RL_OK) return st;
    return lift(ctx, b.p, ld, rows, cols, out, ldo);
}

// SideMultiplier<Complex>::make (preprocess.hpp:27-60) for an n x n side
enum class ZForm { NONE, DENSE_REAL, DENSE_COMPLEX, CIRC };
struct ZSide {
    ZForm form = ZForm::NONE;
    double* dr = nullptr;   // n x ld real (DENSE_REAL)
    double2* dc = nullptr;  // n x n complex (DENSE_COMPLEX)
    int64_t ld = 0;
    ZCirc circ;
    StreamBuf buf;
    explicit ZSide(cudaStream_t s) : circ(s), buf(s) {}
};
rl_status zside_make(rl_context* ctx, const rl_multiplier* m, int64_t n, bool host, ZSide& side) {
    side.form = ZForm::NONE;
    if (!m || m->kind == RL_MULT_NONE) return RL_OK;
    if (!known_kind(m->kind)) return set_error(RL_ERR_INVALID_ARGUMENT, "unknown multiplier kind %d", m->kind);
    if (m->kind == RL_MULT_TOEPLITZ_BLOCK && m->variant != RL_TOEPLITZ_REAL && m->variant != RL_TOEPLITZ_UNITARY)
        return set_error(RL_ERR_INVALID_ARGUMENT, "unknown Toeplitz variant %d", m->variant);
    rl_status st;
    switch (m->kind) {
        case RL_MULT_REAL_CIRCULANT:
        case RL_MULT_UNITARY_CIRCULANT:
        case RL_MULT_TOEPLITZ_BLOCK:  // both variants keep the n x n parent circulant (preprocess.hpp:40-52)
        case RL_MULT_GAUSSIAN_CIRCULANT:
            side.form = ZForm::CIRC;
            return zcirc_from_spec(ctx, m, n, host, side.circ);
        case RL_MULT_SRFT:
            side.form = ZForm::DENSE_COMPLEX;
            side.ld = n;
            if ((st = side.buf.alloc(16 * n * n)) != RL_OK) return st;
            side.dc = reinterpret_cast<double2*>(side.buf.p);
            return zmaterialize_device(ctx, m, n, n, host, side.dc, n);
        default:  // Gaussian, finite set, circulant x skew-circulant: real, lifted
            side.form = ZForm::DENSE_REAL;
            side.ld = even(n);
            if ((st = side.buf.alloc(8 * n * side.ld)) != RL_OK) return st;
            side.dr = side.buf.p;
            return materialize_device(ctx, m, n, n, host, side.dr, side.ld);
    }
}
// A H (right_multiply, preprocess.hpp:63-73) into out (n x n complex)
rl_status zside_right(rl_context* ctx, const ZSide& h, int64_t n, const double2* a, double2* out) {
    switch (h.form) {
        case ZForm::NONE:
            RL_CUDA(cudaMemcpyAsync(out, a, 16 * n * n, cudaMemcpyDeviceToDevice, ctx->stream));
            return RL_OK;
        case ZForm::DENSE_REAL: return zgemm_cr(ctx, n, n, n, a, n, h.dr, h.ld, out, n);
        case ZForm::DENSE_COMPLEX: return zgemm_cc(ctx, n, n, n, a, n, h.dc, h.ld, out, n);
        case ZForm::CIRC: return zcirc_rows(ctx, n, n, a, n, n, h.circ.spec_t, n, out, n);
    }
    return RL_OK;
}
// F A (left_multiply, preprocess.hpp:75-86): column by column for the circulant
rl_status zside_left(rl_context* ctx, const ZSide& f, int64_t n, const double2* a, double2* out) {
    switch (f.form) {
        case ZForm::NONE:
            RL_CUDA(cudaMemcpyAsync(out, a, 16 * n * n, cudaMemcpyDeviceToDevice, ctx->stream));
            return RL_OK;
        case ZForm::DENSE_REAL: return zgemm_rc(ctx, n, n, n, f.dr, f.ld, a, n, out, n);
        case ZForm::DENSE_COMPLEX: return zgemm_cc(ctx, n, n, n, f.dc, f.ld, a, n, out, n);
        case ZForm::CIRC: {
            StreamBuf bt(ctx->stream), bu(ctx->stream);
            rl_status st;
            if ((st = bt.alloc(16 * n * n)) != RL_OK || (st = bu.alloc(16 * n * n)) != RL_OK) return st;
            double2* t = reinterpret_cast<double2*>(bt.p);
            double2* u = reinterpret_cast<double2*>(bu.p);
            if ((st = ztranspose(ctx, a, n, n, n, t, n, false)) != RL_OK) return st;  // columns as rows
            if ((st = zcirc_rows(ctx, n, n, t, n, n, f.circ.spec, n, u, n)) != RL_OK) return st;
            return ztranspose(ctx, u, n, n, n, out, n, false);
        }
    }
    return RL_OK;
}
// H v (apply_vec, preprocess.hpp:88-94)
rl_status zside_apply(rl_context* ctx, const ZSide& h, int64_t n, const double2* v, double2* out) {
    switch (h.form) {
        case ZForm::NONE:
            RL_CUDA(cudaMemcpyAsync(out, v, 16 * n, cudaMemcpyDeviceToDevice, ctx->stream));
            return RL_OK;
        case ZForm::DENSE_REAL: return zgemv(ctx, n, n, nullptr, h.dr, h.ld, v, nullptr, out);
        case ZForm::DENSE_COMPLEX: return zgemv(ctx, n, n, h.dc, nullptr, h.ld, v, nullptr, out);
        case ZForm::CIRC: return zcirc_rows(ctx, 1, n, v, n, n, h.circ.spec, n, out, n);
    }
    return RL_OK;
}

// ---- statistics of the product and the factors --------------------------------
struct ZStats {
    double sumsq;
    unsigned long long maxp, maxu, minpiv;  // bit patterns of non-negative doubles
    unsigned long long first;               // first pivot index at or below the tolerance
};
__global__ void zstats_kernel(const double* __restrict__ W, int64_t ldw, int64_t n, bool upper, ZStats* st) {
    double sq = 0.0, mx = 0.0;
    const int64_t total = n * n;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / n, j = idx - i * n;
        if (upper && j < i) continue;
        const double a2 = zabs2(make_double2(W[i * ldw + wcol(j, n, 0)], W[i * ldw + wcol(j, n, 1)]));
        sq += a2;
        mx = fmax(mx, a2);
    }
    sq = warp_sum(sq);
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) {
        if (!upper) atomicAdd(&st->sumsq, sq);
        atomicMax(upper ? &st->maxu : &st->maxp, static_cast<unsigned long long>(__double_as_longlong(sqrt(mx))));
    }
}
__global__ void zpivots_kernel(const double2* __restrict__ piv, int64_t n, double tol, ZStats* st) {
    double mn = INFINITY;
    unsigned long long first = ~0ull;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double a = sqrt(zabs2(piv[j]));  // detail::abs_of (lu.hpp:31-34)
        mn = fmin(mn, a);
        if (!(a > tol) && static_cast<unsigned long long>(j) < first) first = static_cast<unsigned long long>(j);
    }
    mn = warp_min(mn);
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long f = __shfl_xor_sync(kFull, first, o);
        first = f < first ? f : first;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&st->minpiv, static_cast<unsigned long long>(__double_as_longlong(mn)));
        atomicMin(&st->first, first);
    }
}
double bits(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}

// E(M) = [[Mr, -Mi], [Mi, Mr]] (2m x 2n) with rows and columns stacked
__global__ void embed_kernel(const double2* __restrict__ z, int64_t ldz, int64_t m, int64_t n, double* __restrict__ e,
                             int64_t lde) {
    const int64_t total = m * n;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / n, j = idx - i * n;
        const double2 v = z[i * ldz + j];
        e[i * lde + j] = v.x;
        e[i * lde + n + j] = -v.y;
        e[(m + i) * lde + j] = v.y;
        e[(m + i) * lde + n + j] = v.x;
    }
}
rl_status embed(rl_context* ctx, const double2* z, int64_t ldz, int64_t m, int64_t n, double* e, int64_t lde) {
    embed_kernel<<<grid_for(m * n), 256, 0, ctx->stream>>>(z, ldz, m, n, e, lde);
    RL_CHECK_LAUNCH("embed_kernel");
    return RL_OK;
}
// Y_E (2m x 2l) from Y (m x l): column 2j = [Re y_j ; Im y_j], column 2j+1 =
// [-Im y_j ; Re y_j] (i y_j), so real Gram-Schmidt runs (y_1, i y_1, y_2, ...)
__global__ void embed_cols_kernel(const double2* __restrict__ y, int64_t ldy, int64_t m, int64_t l,
                                  double* __restrict__ e, int64_t lde) {
    const int64_t total = m * l;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / l, j = idx - i * l;
        const double2 v = y[i * ldy + j];
        e[i * lde + 2 * j] = v.x;
        e[(m + i) * lde + 2 * j] = v.y;
        e[i * lde + 2 * j + 1] = -v.y;
        e[(m + i) * lde + 2 * j + 1] = v.x;
    }
}
__global__ void extract_cols_kernel(const double* __restrict__ e, int64_t lde, int64_t m, int64_t l,
                                    double2* __restrict__ q, int64_t ldq) {
    const int64_t total = m * l;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / l, j = idx - i * l;
        q[i * ldq + j] = make_double2(e[i * lde + 2 * j], e[(m + i) * lde + 2 * j]);
    }
}

// svd_values of a contiguous device matrix (rl_singular_values, block_ge.cu) into a host vector
rl_status svd_values_dev(rl_context* ctx, int64_t m, int64_t n, const double* a, std::vector<double>& out) {
    const int64_t k = std::min(m, n);
    StreamBuf b(ctx->stream);
    rl_status st;
    if ((st = b.alloc(8 * k)) != RL_OK) return st;
    if ((st = rl_singular_values(ctx, RL_DEVICE, m, n, a, b.p)) != RL_OK) return st;
    out.resize(static_cast<size_t>(k));
    RL_CUDA(cudaMemcpyAsync(out.data(), b.p, 8 * k, cudaMemcpyDeviceToHost, ctx->stream));
    RL_CUDA(cudaStreamSynchronize(ctx->stream));
    return RL_OK;
}

void clear_info(rl_solve_info* info) {
    double* h = info->history;
    const int64_t cap = info->history_capacity;
    std::memset(info, 0, sizeof(*info));
    info->history = h;
    info->history_capacity = cap;
}

}  // namespace

// ---- the complex solve -----------------------------------------------------------
rl_status zsolve(rl_context* ctx, bool host, int64_t n, const double* a, const double* b,
                 const rl_multiplier* pre, const rl_multiplier* post, int64_t refine, double* x_out, double* lu_out,
                 rl_solve_info* info) {
    cudaStream_t s = ctx->stream;
    rl_status st;
    const int64_t ldw = 2 * n;
    StreamBuf bA(s), bP(s), bW(s), bv(s), bsc(s);
    if ((st = bA.alloc(16 * n * n)) != RL_OK || (st = bP.alloc(16 * n * n)) != RL_OK ||
        (st = bW.alloc(8 * n * ldw)) != RL_OK || (st = bv.alloc(16 * 9 * n)) != RL_OK ||
        (st = bsc.alloc(sizeof(ZStats) + 64)) != RL_OK)
        return st;
    double2* A = reinterpret_cast<double2*>(bA.p);
    double2* P = reinterpret_cast<double2*>(bP.p);
    double* W = bW.p;
    double2* vb = reinterpret_cast<double2*>(bv.p);
    double2 *piv = vb, *rinv = vb + n, *bb = vb + 2 * n, *x = vb + 3 * n, *r = vb + 4 * n, *fr = vb + 5 * n,
            *y = vb + 6 * n, *d = vb + 7 * n;
    ZStats* zs = reinterpret_cast<ZStats*>(bsc.p);
    double* scal = reinterpret_cast<double*>(zs + 1);
    const cudaMemcpyKind kin = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    RL_CUDA(cudaMemcpyAsync(A, a, 16 * n * n, kin, s));
    if (b) RL_CUDA(cudaMemcpyAsync(bb, b, 16 * n, kin, s));

    ZSide F(s), H(s);
    if ((st = zside_make(ctx, pre, n, host, F)) != RL_OK) return st;
    if ((st = zside_make(ctx, post, n, host, H)) != RL_OK) return st;
    // product = F (A H) (preprocess.hpp:166)
    if (F.form == ZForm::NONE) {
        if ((st = zside_right(ctx, H, n, A, P)) != RL_OK) return st;
    } else {
        StreamBuf bt(s);
        if ((st = bt.alloc(16 * n * n)) != RL_OK) return st;
        double2* t = reinterpret_cast<double2*>(bt.p);
        if ((st = zside_right(ctx, H, n, A, t)) != RL_OK) return st;
        if ((st = zside_left(ctx, F, n, t, P)) != RL_OK) return st;
    }
    if ((st = pack(ctx, P, n, n, n, W, ldw, Pack::W)) != RL_OK) return st;

    // GENP + verdict (lu.hpp:40-58): pivots at or below tol_pivot(n) * ||P||_F
    // need the estimate; floor <= estimate <= ||P||_F
    ZStats init{0.0, 0ull, 0ull, 0x7ff0000000000000ull, ~0ull};
    RL_CUDA(cudaMemcpyAsync(zs, &init, sizeof(init), cudaMemcpyHostToDevice, s));
    zstats_kernel<<<grid_for(n * n), 256, 0, s>>>(W, ldw, n, false, zs);
    RL_CHECK_LAUNCH("zstats_kernel");
    if ((st = zgenp_inplace(ctx, n, W, ldw, piv, rinv)) != RL_OK) return st;
    zstats_kernel<<<grid_for(n * n), 256, 0, s>>>(W, ldw, n, true, zs);
    RL_CHECK_LAUNCH("zstats_kernel(upper)");
    ZStats hs;
    RL_CUDA(cudaMemcpyAsync(&hs, zs, sizeof(hs), cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    const double fro = std::sqrt(hs.sumsq);
    const double tol_pivot = 1e-13 * static_cast<double>(n);  // types.hpp:42
    const double tol_hi = tol_pivot * fro * (1.0 + 1e-10);
    zpivots_kernel<<<nblk(n, 256), 256, 0, s>>>(piv, n, tol_hi, zs);
    RL_CHECK_LAUNCH("zpivots_kernel");
    RL_CUDA(cudaMemcpyAsync(&hs, zs, sizeof(hs), cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    info->min_abs_pivot = bits(hs.minpiv);
    info->max_abs_product = bits(hs.maxp);
    info->max_abs_u = bits(hs.maxu);
    info->growth = info->max_abs_u / info->max_abs_product;
    info->norm_frobenius = fro;
    info->pivot_tolerance = tol_hi;
    if (hs.first != ~0ull) {
        // the exact test: spectral_norm_estimate of the product (norms.hpp:35-78),
        // evaluated on its real embedding (same singular values, same floor)
        StreamBuf be(s);
        if ((st = be.alloc(8 * 4 * n * n)) != RL_OK) return st;
        if ((st = embed(ctx, P, n, n, n, be.p, 2 * n)) != RL_OK) return st;
        double est = 0.0;
        if ((st = spectral_norm_estimate_device(ctx, 2 * n, 2 * n, be.p, 2 * n, &est)) != RL_OK) return st;
        const double tol = tol_pivot * est;
        info->norm_estimate = est;
        info->norm_estimate_evaluated = 1;
        info->pivot_tolerance = tol;
        hs.first = ~0ull;
        RL_CUDA(cudaMemcpyAsync(&zs->first, &hs.first, 8, cudaMemcpyHostToDevice, s));
        zpivots_kernel<<<nblk(n, 256), 256, 0, s>>>(piv, n, tol, zs);
        RL_CHECK_LAUNCH("zpivots_kernel");
        RL_CUDA(cudaMemcpyAsync(&hs.first, &zs->first, 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaStreamSynchronize(s));
        if (hs.first != ~0ull) {
            info->zero_pivot_step = static_cast<int64_t>(hs.first) + 1;
            return set_error(RL_ERR_ZERO_PIVOT, "zero pivot at elimination step %lld",
                             static_cast<long long>(info->zero_pivot_step));
        }
    }
    if (lu_out) {
        double2* lu = P;  // the product is no longer needed
        if ((st = unpack(ctx, W, ldw, n, n, lu, n, Pack::W)) != RL_OK) return st;
        RL_CUDA(cudaMemcpyAsync(lu_out, lu, 16 * n * n, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    }
    if (!b) {  // genp_factor only
        RL_CUDA(cudaStreamSynchronize(s));
        return RL_OK;
    }

    // iterative_refine with the chain solver H (LU)^-1 (F r) from x0 = 0,
    // refine + 1 steps (preprocess.hpp:115-143, :167-178)
    RL_CUDA(cudaMemsetAsync(x, 0, 16 * n, s));
    RL_CUDA(cudaMemcpyAsync(r, bb, 16 * n, cudaMemcpyDeviceToDevice, s));
    if ((st = sumsq(ctx, 2 * n, reinterpret_cast<const double*>(bb), scal)) != RL_OK) return st;
    double bsq = 0.0, last = 1.0;
    int streak = 0;
    for (int64_t k = 0; k <= refine; ++k) {
        if ((st = zside_apply(ctx, F, n, r, fr)) != RL_OK) return st;
        RL_CUDA(cudaMemcpyAsync(y, fr, 16 * n, cudaMemcpyDeviceToDevice, s));
        zlu_solve_kernel<<<1, TS, 0, s>>>(W, ldw, n, rinv, y);
        RL_CHECK_LAUNCH("zlu_solve_kernel");
        if ((st = zside_apply(ctx, H, n, y, d)) != RL_OK) return st;
        zaxpy_kernel<<<nblk(n, 256), 256, 0, s>>>(x, d, n);
        RL_CHECK_LAUNCH("zaxpy_kernel");
        if ((st = zgemv(ctx, n, n, A, nullptr, n, x, bb, r)) != RL_OK) return st;  // r = b - A x
        if ((st = sumsq(ctx, 2 * n, reinterpret_cast<const double*>(r), scal + 1)) != RL_OK) return st;
        double rsq = 0.0;
        RL_CUDA(cudaMemcpyAsync(&rsq, scal + 1, 8, cudaMemcpyDeviceToHost, s));
        if (k == 0) RL_CUDA(cudaMemcpyAsync(&bsq, scal, 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaStreamSynchronize(s));
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
    RL_CUDA(cudaMemcpyAsync(x_out, x, 16 * n, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}

// ---- the complex range finder ---------------------------------------------------
// Y (m x l) = A S for the spec's n x l multiplier (lowrank.hpp:62-81)
rl_status zsketch(rl_context* ctx, bool host, int64_t m, int64_t n, const double2* A, int64_t l,
                  const rl_multiplier* h, double2* Y) {
    cudaStream_t s = ctx->stream;
    rl_status st;
    if (!known_kind(h->kind)) return set_error(RL_ERR_INVALID_ARGUMENT, "unknown multiplier kind %d", h->kind);
    if (h->kind == RL_MULT_TOEPLITZ_BLOCK || h->kind == RL_MULT_GAUSSIAN_CIRCULANT) {
        // matmul_by_toeplitz_block: rows through the parent n-point circulant's transpose
        ZCirc zc(s);
        if ((st = zcirc_from_spec(ctx, h, n, host, zc)) != RL_OK) return st;
        return zcirc_rows(ctx, m, n, A, n, n, zc.spec_t, l, Y, l);
    }
    if (h->kind == RL_MULT_NONE) {
        if (n != l) return set_error(RL_ERR_DIMENSION, "identity multiplier must be square");
        RL_CUDA(cudaMemcpyAsync(Y, A, 16 * m * n, cudaMemcpyDeviceToDevice, s));
        return RL_OK;
    }
    const bool complex_dense = h->kind == RL_MULT_SRFT || h->kind == RL_MULT_UNITARY_CIRCULANT;
    if (complex_dense) {
        StreamBuf bs(s);
        if ((st = bs.alloc(16 * n * l)) != RL_OK) return st;
        double2* S = reinterpret_cast<double2*>(bs.p);
        if ((st = zmaterialize_device(ctx, h, n, l, host, S, l)) != RL_OK) return st;
        return zgemm_cc(ctx, m, l, n, A, n, S, l, Y, l);
    }
    StreamBuf bs(s);
    const int64_t ld = even(l);
    if ((st = bs.alloc(8 * n * ld)) != RL_OK) return st;
    if ((st = materialize_device(ctx, h, n, l, host, bs.p, ld)) != RL_OK) return st;
    return zgemm_cr(ctx, m, l, n, A, n, bs.p, ld, Y, l);
}

// Q (m x l complex, device) = orthonormal_basis(Y) through the embedding;
// QE (2m x 2l, ld 2l) keeps the real basis for the residual
rl_status zbasis(rl_context* ctx, int64_t m, int64_t l, const double2* Y, double* QE, double2* Q, bool unchecked,
                 int64_t* bad) {
    StreamBuf be(ctx->stream);
    rl_status st;
    if ((st = be.alloc(8 * 4 * m * l)) != RL_OK) return st;
    embed_cols_kernel<<<grid_for(m * l), 256, 0, ctx->stream>>>(Y, l, m, l, be.p, 2 * l);
    RL_CHECK_LAUNCH("embed_cols_kernel");
    CholqrOpts opts;
    opts.rank_m = m;
    opts.rank_l = l;
    opts.column_group = 2;
    opts.unchecked = unchecked;
    if ((st = cholqr2_device(ctx, 2 * m, 2 * l, be.p, QE, 2 * l, nullptr, 0, bad, &opts)) != RL_OK) return st;
    // In floating point the basis keeps the pairing (column 2j + 1 = i times
    // column 2j) only to O(u kappa(Y)); the even columns are the complex
    // basis. Re-embed them and orthonormalise once more: the input is now
    // orthonormal to O(u kappa), so this pass moves it by that much and
    // restores the pairing to rounding level.
    StreamBuf bq(ctx->stream);
    if ((st = bq.alloc(16 * m * l)) != RL_OK) return st;
    double2* Qc = reinterpret_cast<double2*>(bq.p);
    extract_cols_kernel<<<grid_for(m * l), 256, 0, ctx->stream>>>(QE, 2 * l, m, l, Qc, l);
    RL_CHECK_LAUNCH("extract_cols_kernel");
    embed_cols_kernel<<<grid_for(m * l), 256, 0, ctx->stream>>>(Qc, l, m, l, be.p, 2 * l);
    RL_CHECK_LAUNCH("embed_cols_kernel");
    opts.unchecked = true;
    int64_t bad2 = 0;
    if ((st = cholqr2_device(ctx, 2 * m, 2 * l, be.p, QE, 2 * l, nullptr, 0, &bad2, &opts)) != RL_OK) return st;
    if (Q) {
        extract_cols_kernel<<<grid_for(m * l), 256, 0, ctx->stream>>>(QE, 2 * l, m, l, Q, l);
        RL_CHECK_LAUNCH("extract_cols_kernel");
    }
    return RL_OK;
}

// residual norms of A - Q Q^H A from E(A) and the real basis: ||E(R)||_F =
// sqrt(2) ||R||_F, ||E(R)||_2 = ||R||_2
rl_status zresidual(rl_context* ctx, int64_t m, int64_t n, const double* EA, int64_t l, const double* QE,
                    rl_lowrank_info* info) {
    rl_status st = residual_core(ctx, 2 * m, 2 * n, EA, 2 * n, 2 * l, QE, 2 * l, info);
    if (st != RL_OK) return st;
    info->residual_frobenius /= std::sqrt(2.0);
    return RL_OK;
}

}  // namespace rl

using namespace rl;

namespace {
rl_status staged(rl_context* ctx, bool host, const double* src, int64_t count, StreamBuf& buf, const double2** out) {
    rl_status st;
    if (!host) {
        *out = reinterpret_cast<const double2*>(src);
        return RL_OK;
    }
    if ((st = buf.alloc(16 * count)) != RL_OK) return st;
    RL_CUDA(cudaMemcpyAsync(buf.p, src, 16 * count, cudaMemcpyHostToDevice, ctx->stream));
    *out = reinterpret_cast<const double2*>(buf.p);
    return RL_OK;
}
}  // namespace

extern "C" RL_API rl_status rl_zpreprocessed_genp_solve(rl_context* ctx, rl_mem mem, int64_t n, const double* a,
                                                        const double* b, const rl_multiplier* pre,
                                                        const rl_multiplier* post, int64_t refine_steps, double* x,
                                                        double* lu_out, rl_solve_info* info) {
    rl_solve_info local;
    if (!info) info = &local;
    clear_info(info);
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "preprocess_solve: matrix dimensions must be positive");
    if (!a || !b || !x) return set_error(RL_ERR_INVALID_ARGUMENT, "preprocess_solve: a, b, x are required");
    if (refine_steps < 0) return set_error(RL_ERR_INVALID_ARGUMENT, "preprocess_solve: negative refine_steps");
    if (refine_steps > 7 && (!info->history || info->history_capacity < refine_steps + 1))
        return set_error(RL_ERR_INVALID_ARGUMENT,
                         "preprocess_solve: refine_steps > 7 needs info->history with refine_steps + 1 entries");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    st = zsolve(ctx, mem == RL_HOST, n, a, b, pre, post, refine_steps, x, lu_out, info);
    if (st != RL_OK) cudaStreamSynchronize(ctx->stream);
    return st;
}

namespace {
rl_status zrange_entry(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a, int64_t l,
                       const rl_multiplier* h, int64_t power_steps, double* q_out, rl_lowrank_info* info) {
    rl_lowrank_info local;
    if (!info) info = &local;
    std::memset(info, 0, sizeof(*info));
    if (m <= 0 || n <= 0 || l < 1 || l > std::min(m, n))
        return set_error(RL_ERR_DIMENSION, "range_find: rank plus oversampling exceeds matrix size");
    if (!a || !h) return set_error(RL_ERR_INVALID_ARGUMENT, "range_find: null pointer");
    if (power_steps < 0) return set_error(RL_ERR_INVALID_ARGUMENT, "range_find: negative power_steps");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    StreamBuf ba(s), by(s), bea(s), bqe(s), bq(s);
    const double2* A = nullptr;
    if ((st = staged(ctx, host, a, m * n, ba, &A)) != RL_OK) return st;
    if ((st = by.alloc(16 * m * l)) != RL_OK || (st = bqe.alloc(8 * 4 * m * l)) != RL_OK ||
        (st = bq.alloc(16 * m * l)) != RL_OK)
        return st;
    double2* Y = reinterpret_cast<double2*>(by.p);
    if ((st = zsketch(ctx, host, m, n, A, l, h, Y)) != RL_OK) return st;
    if (power_steps > 0) {
        // sketch = A (A^H sketch) (lowrank.hpp:51-57)
        StreamBuf bah(s), bz(s);
        if ((st = bah.alloc(16 * n * m)) != RL_OK || (st = bz.alloc(16 * n * l)) != RL_OK) return st;
        double2* AH = reinterpret_cast<double2*>(bah.p);
        double2* Z = reinterpret_cast<double2*>(bz.p);
        if ((st = ztranspose(ctx, A, n, m, n, AH, m, true)) != RL_OK) return st;
        for (int64_t k = 0; k < power_steps; ++k) {
            if ((st = zgemm_cc(ctx, n, l, m, AH, m, Y, l, Z, l)) != RL_OK) return st;
            if ((st = zgemm_cc(ctx, m, l, n, A, n, Z, l, Y, l)) != RL_OK) return st;
        }
    }
    double2* Q = reinterpret_cast<double2*>(bq.p);
    if ((st = zbasis(ctx, m, l, Y, bqe.p, Q, false, &info->rank_deficient_column)) != RL_OK) {
        cudaStreamSynchronize(s);
        return st;
    }
    if ((st = bea.alloc(8 * 4 * m * n)) != RL_OK) return st;
    if ((st = embed(ctx, A, n, m, n, bea.p, 2 * n)) != RL_OK) return st;
    if ((st = zresidual(ctx, m, n, bea.p, l, bqe.p, info)) != RL_OK) return st;
    if (q_out) RL_CUDA(cudaMemcpyAsync(q_out, Q, 16 * m * l, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}
}  // namespace

extern "C" RL_API rl_status rl_zrange_find_residual(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                                    int64_t l, const rl_multiplier* h, int64_t power_steps,
                                                    double* q, rl_lowrank_info* info) {
    return zrange_entry(ctx, mem, m, n, a, l, h, power_steps, q, info);
}

extern "C" RL_API rl_status rl_zapproximation_residual(rl_context* ctx, rl_mem mem, int64_t m, int64_t n,
                                                       const double* a, int64_t l, const double* q,
                                                       rl_lowrank_info* info) {
    rl_lowrank_info local;
    if (!info) info = &local;
    std::memset(info, 0, sizeof(*info));
    if (m <= 0 || n <= 0 || l < 1 || l > m) return set_error(RL_ERR_DIMENSION, "approximation_residual: bad shapes");
    if (!a || !q) return set_error(RL_ERR_INVALID_ARGUMENT, "approximation_residual: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    StreamBuf ba(s), bq(s), bea(s), bqe(s);
    const double2 *A = nullptr, *Q = nullptr;
    if ((st = staged(ctx, host, a, m * n, ba, &A)) != RL_OK) return st;
    if ((st = staged(ctx, host, q, m * l, bq, &Q)) != RL_OK) return st;
    if ((st = bea.alloc(8 * 4 * m * n)) != RL_OK || (st = bqe.alloc(8 * 4 * m * l)) != RL_OK) return st;
    if ((st = embed(ctx, A, n, m, n, bea.p, 2 * n)) != RL_OK) return st;
    embed_cols_kernel<<<grid_for(m * l), 256, 0, s>>>(Q, l, m, l, bqe.p, 2 * l);
    RL_CHECK_LAUNCH("embed_cols_kernel");
    st = zresidual(ctx, m, n, bea.p, l, bqe.p, info);
    RL_CUDA(cudaStreamSynchronize(s));
    return st;
}

extern "C" RL_API rl_status rl_zmaterialize(rl_context* ctx, rl_mem mem, const rl_multiplier* spec, int64_t rows,
                                            int64_t cols, double* out) {
    if (!spec || !out) return set_error(RL_ERR_INVALID_ARGUMENT, "materialize: null pointer");
    if (rows <= 0 || cols <= 0) return set_error(RL_ERR_DIMENSION, "materialize: empty shape");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    const bool host = mem == RL_HOST;
    StreamBuf tmp(ctx->stream);
    double2* d = reinterpret_cast<double2*>(out);
    if (host) {
        if ((st = tmp.alloc(16 * rows * cols)) != RL_OK) return st;
        d = reinterpret_cast<double2*>(tmp.p);
    }
    if ((st = zmaterialize_device(ctx, spec, rows, cols, host, d, cols)) != RL_OK) return st;
    if (host) RL_CUDA(cudaMemcpyAsync(out, d, 16 * rows * cols, cudaMemcpyDeviceToHost, ctx->stream));
    RL_CUDA(cudaStreamSynchronize(ctx->stream));
    return RL_OK;
}

extern "C" RL_API rl_status rl_gen_unitary_circulant(rl_context* ctx, rl_mem mem, int64_t n, uint64_t seed,
                                                     double* column) {
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "circulant: empty first column");
    if (!column) return set_error(RL_ERR_INVALID_ARGUMENT, "gen_unitary_circulant: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    rl_multiplier m{};
    m.kind = RL_MULT_UNITARY_CIRCULANT;
    m.seed = seed;
    ZCirc zc(ctx->stream);
    if ((st = zcirc_from_spec(ctx, &m, n, mem == RL_HOST, zc)) != RL_OK) return st;
    RL_CUDA(cudaMemcpyAsync(column, zc.col, 16 * n, mem == RL_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                            ctx->stream));
    RL_CUDA(cudaStreamSynchronize(ctx->stream));
    return RL_OK;
}

// genp_factor<Complex> (lu.hpp:40-58): packed L\U of a complex n x n matrix
extern "C" RL_API rl_status rl_zgenp_factor(rl_context* ctx, rl_mem mem, int64_t n, const double* a, double* lu,
                                            rl_solve_info* info) {
    rl_solve_info local;
    if (!info) info = &local;
    clear_info(info);
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "genp_factor: square input required");
    if (!a || !lu) return set_error(RL_ERR_INVALID_ARGUMENT, "genp_factor: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    st = zsolve(ctx, mem == RL_HOST, n, a, nullptr, nullptr, nullptr, 0, nullptr, lu, info);
    if (st != RL_OK) cudaStreamSynchronize(ctx->stream);
    return st;
}

// lu_solve<Complex> (lu.hpp:100-122) on packed GENP factors
extern "C" RL_API rl_status rl_zlu_solve(rl_context* ctx, rl_mem mem, int64_t n, const double* lu, const double* b,
                                         double* x) {
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "lu_solve: length mismatch");
    if (!lu || !b || !x) return set_error(RL_ERR_INVALID_ARGUMENT, "lu_solve: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    StreamBuf bl(s), bw(s), bv(s);
    const double2* L = nullptr;
    if ((st = staged(ctx, host, lu, n * n, bl, &L)) != RL_OK) return st;
    if ((st = bw.alloc(8 * n * 2 * n)) != RL_OK || (st = bv.alloc(16 * 2 * n)) != RL_OK) return st;
    double2* rinv = reinterpret_cast<double2*>(bv.p);
    double2* y = rinv + n;
    if ((st = pack(ctx, L, n, n, n, bw.p, 2 * n, Pack::W)) != RL_OK) return st;
    diag_rcp_kernel<<<nblk(n, 256), 256, 0, s>>>(L, n, rinv);
    RL_CHECK_LAUNCH("diag_rcp_kernel");
    RL_CUDA(cudaMemcpyAsync(y, b, 16 * n, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    zlu_solve_kernel<<<1, TS, 0, s>>>(bw.p, 2 * n, n, rinv, y);
    RL_CHECK_LAUNCH("zlu_solve_kernel");
    RL_CUDA(cudaMemcpyAsync(x, y, 16 * n, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}

// orthonormal_basis / orthonormal_basis_unchecked<Complex> (qr.hpp:51-76):
// q (m x l) with positive real R diagonal; bad (nullable) the 1-based
// rank-deficient column (qr.hpp:33-38)
extern "C" RL_API rl_status rl_zorthonormal_basis(rl_context* ctx, rl_mem mem, int64_t m, int64_t l, const double* y,
                                                  double* q, int32_t unchecked, int64_t* bad) {
    int64_t local = 0;
    if (!bad) bad = &local;
    *bad = 0;
    if (m <= 0 || l <= 0 || m < l) return set_error(RL_ERR_DIMENSION, "qr: expected rows >= cols");
    if (!y || !q) return set_error(RL_ERR_INVALID_ARGUMENT, "qr: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    StreamBuf by(s), bqe(s), bq(s);
    const double2* Y = nullptr;
    if ((st = staged(ctx, host, y, m * l, by, &Y)) != RL_OK) return st;
    if ((st = bqe.alloc(8 * 4 * m * l)) != RL_OK || (st = bq.alloc(16 * m * l)) != RL_OK) return st;
    double2* Q = reinterpret_cast<double2*>(bq.p);
    if ((st = zbasis(ctx, m, l, Y, bqe.p, Q, unchecked != 0, bad)) != RL_OK) {
        cudaStreamSynchronize(s);
        return st;
    }
    RL_CUDA(cudaMemcpyAsync(q, Q, 16 * m * l, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}

// matmul_by_circulant / matmul_by_toeplitz_block (circulant.hpp:171-203)
// over the complex field: A (m x k) times the leading k x l block of the
// np-point circulant with complex first column c
extern "C" RL_API rl_status rl_zcirculant_right_multiply(rl_context* ctx, rl_mem mem, int64_t m, int64_t k,
                                                         const double* a, int64_t np, const double* c, int64_t l,
                                                         double* out) {
    if (m <= 0 || k <= 0 || np <= 0 || l <= 0 || k > np || l > np)
        return set_error(RL_ERR_DIMENSION, "matmul_by_toeplitz_block: shape mismatch");
    if (!a || !c || !out) return set_error(RL_ERR_INVALID_ARGUMENT, "matmul_by_circulant: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    StreamBuf ba(s), bo(s);
    const double2* A = nullptr;
    if ((st = staged(ctx, host, a, m * k, ba, &A)) != RL_OK) return st;
    ZCirc zc(s);
    zc.np = np;
    if ((st = zc.buf.alloc(16 * 3 * np)) != RL_OK) return st;
    zc.col = reinterpret_cast<double2*>(zc.buf.p);
    zc.spec = zc.col + np;
    zc.spec_t = zc.spec + np;
    RL_CUDA(cudaMemcpyAsync(zc.col, c, 16 * np, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    if ((st = zcirc_finish(ctx, zc)) != RL_OK) return st;
    double2* o = reinterpret_cast<double2*>(out);
    if (host) {
        if ((st = bo.alloc(16 * m * l)) != RL_OK) return st;
        o = reinterpret_cast<double2*>(bo.p);
    }
    if ((st = zcirc_rows(ctx, m, k, A, k, np, zc.spec_t, l, o, l)) != RL_OK) return st;
    if (host) RL_CUDA(cudaMemcpyAsync(out, o, 16 * m * l, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}

// circulant_apply(C, x) (circulant.hpp:81-98) over the complex field: y = C x
extern "C" RL_API rl_status rl_zcirculant_apply(rl_context* ctx, rl_mem mem, int64_t n, const double* c,
                                                const double* x, double* y) {
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "circulant_apply: length mismatch");
    if (!c || !x || !y) return set_error(RL_ERR_INVALID_ARGUMENT, "circulant_apply: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    StreamBuf bx(s), by(s);
    const double2* X = nullptr;
    if ((st = staged(ctx, host, x, n, bx, &X)) != RL_OK) return st;
    ZCirc zc(s);
    zc.np = n;
    if ((st = zc.buf.alloc(16 * 3 * n)) != RL_OK) return st;
    zc.col = reinterpret_cast<double2*>(zc.buf.p);
    zc.spec = zc.col + n;
    zc.spec_t = zc.spec + n;
    RL_CUDA(cudaMemcpyAsync(zc.col, c, 16 * n, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    if ((st = zcirc_finish(ctx, zc)) != RL_OK) return st;
    double2* o = reinterpret_cast<double2*>(y);
    if (host) {
        if ((st = by.alloc(16 * n)) != RL_OK) return st;
        o = reinterpret_cast<double2*>(by.p);
    }
    if ((st = zcirc_rows(ctx, 1, n, X, n, n, zc.spec, n, o, n)) != RL_OK) return st;
    if (host) RL_CUDA(cudaMemcpyAsync(y, o, 16 * n, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}

// matmul<Complex> (matrix.hpp:115-121): C (m x n) = A (m x k) B (k x n)
extern "C" RL_API rl_status rl_zgemm(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, int64_t k, const double* a,
                                     const double* b, double* c) {
    if (m <= 0 || n <= 0 || k <= 0) return set_error(RL_ERR_DIMENSION, "matmul: empty operand");
    if (!a || !b || !c) return set_error(RL_ERR_INVALID_ARGUMENT, "matmul: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    StreamBuf ba(s), bb(s), bc(s);
    const double2 *A = nullptr, *B = nullptr;
    if ((st = staged(ctx, host, a, m * k, ba, &A)) != RL_OK) return st;
    if ((st = staged(ctx, host, b, k * n, bb, &B)) != RL_OK) return st;
    double2* C = reinterpret_cast<double2*>(c);
    if (host) {
        if ((st = bc.alloc(16 * m * n)) != RL_OK) return st;
        C = reinterpret_cast<double2*>(bc.p);
    }
    if ((st = zgemm_cc(ctx, m, n, k, A, k, B, n, C, n)) != RL_OK) return st;
    if (host) RL_CUDA(cudaMemcpyAsync(c, C, 16 * m * n, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}

extern "C" RL_API rl_status rl_srft_columns(int64_t n, int64_t l, uint64_t seed, int64_t* out) {
    if (l < 1 || l > n) return set_error(RL_ERR_DIMENSION, "gen_srft: need 1 <= l <= n");
    if (!out) return set_error(RL_ERR_INVALID_ARGUMENT, "srft_columns: null pointer");
    host_srft_columns(seed, n, l, out);
    return RL_OK;
}

extern "C" RL_API rl_status rl_zsingular_values(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                                double* out) {
    if (m <= 0 || n <= 0) return set_error(RL_ERR_DIMENSION, "svd_values: empty matrix");
    if (!a || !out) return set_error(RL_ERR_INVALID_ARGUMENT, "svd_values: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    const bool host = mem == RL_HOST;
    StreamBuf ba(ctx->stream), be(ctx->stream);
    const double2* A = nullptr;
    if ((st = staged(ctx, host, a, m * n, ba, &A)) != RL_OK) return st;
    if ((st = be.alloc(8 * 4 * m * n)) != RL_OK) return st;
    if ((st = embed(ctx, A, n, m, n, be.p, 2 * n)) != RL_OK) return st;
    // the singular values of E(A) are those of A, each twice (sorted non-increasing)
    const int64_t r = std::min(m, n);
    std::vector<double> sv;
    if ((st = svd_values_dev(ctx, 2 * m, 2 * n, be.p, sv)) != RL_OK) return st;
    std::vector<double> h(static_cast<size_t>(r));
    for (int64_t k = 0; k < r; ++k) h[k] = sv[2 * k];
    if (host) {
        std::memcpy(out, h.data(), 8 * r);
    } else {
        RL_CUDA(cudaMemcpyAsync(out, h.data(), 8 * r, cudaMemcpyHostToDevice, ctx->stream));
        RL_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return RL_OK;
}

extern "C" RL_API rl_status rl_srft_sketch_check(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, const double* a,
                                                 int64_t r, uint64_t seed, int32_t variant, double known_sigma_r1,
                                                 rl_srft_check* out) {
    if (!a || !out) return set_error(RL_ERR_INVALID_ARGUMENT, "srft_sketch_check: null pointer");
    if (r < 1 || r > n) return set_error(RL_ERR_DIMENSION, "srft_sketch_check: rank out of range");
    if (variant != 0 && variant != 1) return set_error(RL_ERR_INVALID_ARGUMENT, "srft_sketch_check: unknown variant");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    std::memset(out, 0, sizeof(*out));
    // the prescribed width, clamped to n (lowrank.hpp:222-231)
    const double nd = static_cast<double>(n), rd = static_cast<double>(r);
    const double base = std::sqrt(rd) + std::sqrt(8.0 * std::log(rd * nd) * nd);
    const double prescribed = 4.0 * base * base * std::log(rd);
    int64_t l = prescribed > 0.0 ? static_cast<int64_t>(std::ceil(prescribed)) : 0;
    l = std::max(l, r);
    if (l >= n) {
        l = n;
        out->clamped = 1;
    }
    out->sketch_width = l;
    if (l > m) return set_error(RL_ERR_DIMENSION, "qr: expected rows >= cols");
    // S (n x l): gen_srft, or the same columns of the unitary circulant drawn
    // from the same phases (lowrank.hpp:235-246)
    StreamBuf bs(s), ba(s), bea(s), by(s), bqe(s), bsv(s);
    rl_status e;
    if ((e = bs.alloc(16 * n * l)) != RL_OK) return e;
    double2* S = reinterpret_cast<double2*>(bs.p);
    rl_multiplier spec{};
    spec.seed = seed;
    if (variant == 0) {
        spec.kind = RL_MULT_SRFT;
        if ((e = zmaterialize_device(ctx, &spec, n, l, host, S, l)) != RL_OK) return e;
    } else {
        spec.kind = RL_MULT_UNITARY_CIRCULANT;
        ZCirc zc(s);
        if ((e = zcirc_from_spec(ctx, &spec, n, host, zc)) != RL_OK) return e;
        std::vector<int64_t> cols(static_cast<size_t>(l));
        host_srft_columns(seed, n, l, cols.data());
        StreamBuf bc(s);
        if ((e = bc.alloc(8 * l)) != RL_OK) return e;
        int64_t* dc = reinterpret_cast<int64_t*>(bc.p);
        RL_CUDA(cudaMemcpyAsync(dc, cols.data(), 8 * l, cudaMemcpyHostToDevice, s));
        zcirc_dense_kernel<<<grid_for(n * l), 256, 0, s>>>(zc.col, n, n, l, S, l, dc);
        RL_CHECK_LAUNCH("zcirc_dense_kernel");
        RL_CUDA(cudaStreamSynchronize(s));
    }
    // Y = to_complex(a) S, Q = orthonormal_basis_unchecked(Y), residual of ac
    const int64_t lda = even(n);
    if ((e = ba.alloc(8 * m * lda)) != RL_OK) return e;
    RL_CUDA(cudaMemcpy2DAsync(ba.p, lda * 8, a, n * 8, n * 8, m, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                              s));
    if ((e = by.alloc(16 * m * l)) != RL_OK || (e = bqe.alloc(8 * 4 * m * l)) != RL_OK) return e;
    double2* Y = reinterpret_cast<double2*>(by.p);
    if ((e = zgemm_rc(ctx, m, l, n, ba.p, lda, S, l, Y, l)) != RL_OK) return e;
    int64_t bad = 0;
    if ((e = zbasis(ctx, m, l, Y, bqe.p, nullptr, true, &bad)) != RL_OK) return e;
    // E(to_complex(a)) = [[a, 0], [0, a]]
    StreamBuf bz(s);
    if ((e = bz.alloc(16 * m * n)) != RL_OK || (e = bea.alloc(8 * 4 * m * n)) != RL_OK) return e;
    double2* AC = reinterpret_cast<double2*>(bz.p);
    if ((e = lift(ctx, ba.p, lda, m, n, AC, n)) != RL_OK) return e;
    if ((e = embed(ctx, AC, n, m, n, bea.p, 2 * n)) != RL_OK) return e;
    rl_lowrank_info li{};
    if ((e = zresidual(ctx, m, n, bea.p, l, bqe.p, &li)) != RL_OK) return e;
    out->residual = li.residual_spectral;  // spectral_norm_estimate(resid)
    double sigma = known_sigma_r1;
    if (!(sigma >= 0.0)) {  // svd_values(a)[r] (lowrank.hpp:252-257)
        StreamBuf bc(s);
        const double* ac = ba.p;
        if (lda != n) {
            if ((e = bc.alloc(8 * m * n)) != RL_OK) return e;
            RL_CUDA(cudaMemcpy2DAsync(bc.p, n * 8, ba.p, lda * 8, n * 8, m, cudaMemcpyDeviceToDevice, s));
            ac = bc.p;
        }
        std::vector<double> sv;
        if ((e = svd_values_dev(ctx, m, n, ac, sv)) != RL_OK) return e;
        sigma = r < static_cast<int64_t>(sv.size()) ? sv[r] : 0.0;
    }
    out->bound = std::sqrt(1.0 + 7.0 * nd / static_cast<double>(l)) * sigma;
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}
