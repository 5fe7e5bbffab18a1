// Blocked GENP of a dense n x n matrix, in place (packed LU), for sm_100a.
//
// Mathematically genp_factor (lu.hpp:40-58): natural pivot order, no row
// exchanges. Any recursive block factorization with unpivoted leaves "turns
// into GENP up to the order", so the L and U here are the
// reference's up to rounding. Structure (right-looking, see genp_inplace):
//
//   n >= 256:  128-column super-panels (genp_super128) with a one-super-panel
//              lookahead on a high-priority stream; each super-panel is two
//              fused 64-column panel launches (lu_panel64_kernel: diagonal
//              block in registers, L21 rows, and the 128x128 L11^-1 built by an
//              extra CTA), U12 = L11^-1 A12 as one K = 128 DMMA GEMM, and the
//              trailing update A22 -= L21 U12 as one K = 128 DMMA GEMM
//              (kernels.cuh);
//   n <  256:  64-column panels with the same kernels (lookahead at n >= 192);
//   the ragged last block (< 64 columns): panel_diag_kernel + panel_rows_kernel_dyn.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "device_common.cuh"
#include "kernels.cuh"

namespace rl {
namespace {

constexpr int kBase = 64;  // panel width

// ---- w x w diagonal block (w <= 64): GENP in shared memory --------------
__global__ void __launch_bounds__(256)
panel_diag_kernel(double* __restrict__ a, int64_t lda, int w, double* __restrict__ piv_out,
                  double* __restrict__ rinv_out) {
    __shared__ double s[kBase][kBase + 1];
    const int tid = threadIdx.x;
    for (int idx = tid; idx < w * w; idx += 256) s[idx / w][idx % w] = a[(idx / w) * lda + idx % w];
    __syncthreads();
    const int tx = tid & 15, ty = tid >> 4;
    for (int j = 0; j < w; ++j) {
        const double piv = s[j][j];
        if (tid > j && tid < w) s[tid][j] = s[tid][j] / piv;  // multiplier (lu.hpp:51)
        __syncthreads();
        for (int i = j + 1 + ty; i < w; i += 16) {
            const double l = s[i][j];
            for (int k = j + 1 + tx; k < w; k += 16) s[i][k] = fma(-l, s[j][k], s[i][k]);
        }
        __syncthreads();
    }
    for (int idx = tid; idx < w * w; idx += 256) a[(idx / w) * lda + idx % w] = s[idx / w][idx % w];
    if (tid < w) {
        piv_out[tid] = s[tid][tid];
        rinv_out[tid] = 1.0 / s[tid][tid];
    }
}

// 1/x: MUFU seed + two Newton steps (no division subroutine on the critical path)
__device__ __forceinline__ double rcp64(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// a / b correctly rounded from r = 1/b (one residual correction)
__device__ __forceinline__ double div_by(double a, double b, double r) {
    const double q0 = a * r;
    return fma(r, fma(-b, q0, a), q0);
}

// ragged last block (w < 64): rows below the w x w diagonal block,
// L21 = A21 U11^-1, x U11 = a -> x_j = (a_j - sum_{i<j} x_i u_ij) / u_jj, one row per thread
__global__ void __launch_bounds__(128)
panel_rows_kernel_dyn(double* __restrict__ rows, int64_t lda, int64_t nrows, int w, const double* __restrict__ u11,
                      const double* __restrict__ piv, const double* __restrict__ rinv) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * 128 + threadIdx.x;
    if (r >= nrows) return;
    double* x = rows + r * lda;
    for (int j = 0; j < w; ++j) {
        double acc = x[j];
        for (int i = 0; i < j; ++i) acc = fma(-x[i], u11[i * lda + j], acc);
        x[j] = div_by(acc, piv[j], rinv[j]);
    }
}

// ---- fused right-looking step for a 64-column panel at c0 ------------------
// Every CTA factors the 64x64 diagonal block redundantly in shared memory
// (factor64_blocked: blocked by 16, warp-synchronous diagonal blocks, DMMA
// Schur updates), then does its share of the panel: row CTAs form
// L21 = A21 U11^-1 (x U11 = a, column sweep per row, Q threads per row),
// column CTAs (small matrices only) form U12 = L11^-1 A12 (column sweep per
// column, one column per thread, coalesced). CTA 0 writes the factored
// diagonal block and the pivots. The trailing update A22 -= L21 U12 is a DMMA
// GEMM.
constexpr int PT = 128;  // threads per CTA
#ifndef RL_PANEL_Q4_ROWS
#define RL_PANEL_Q4_ROWS 2048
#endif
constexpr int64_t kPanelQ4Rows = RL_PANEL_Q4_ROWS;


// X = L^-1 for the unit-lower part of a factored 64x64 block (strictly lower
// entries of sd, implicit unit diagonal) by recursive doubling: the eight 8x8
// diagonal blocks by forward substitution (one thread per column), then pairs
// merge, inv([[A, 0], [B, C]]) = [[A^-1, 0], [-C^-1 (B A^-1), C^-1]], at 8, 16
// and 32, each product on DMMA 8x8x4 tiles (one warp per tile).
constexpr int LDX = 66, LDT = 34;
constexpr int kInvFusedSmem = 2 * kBase * LDX * 8;  // X and Y (Y also the 32 x LDT merge scratch)
__device__ __forceinline__ void inv_unit_lower64(const double (*sd)[kBase + 1], double* __restrict__ X,
                                                 double* __restrict__ T, int tid) {
    for (int idx = tid; idx < kBase * LDX; idx += PT) X[idx] = 0.0;
    __syncthreads();
    if (tid < kBase) {
        const int o = 8 * (tid >> 3), j = tid & 7;
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = i == j ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < 7; ++k)
#pragma unroll
            for (int i = k + 1; i < 8; ++i) x[i] = fma(-sd[o + i][o + k], x[k], x[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) X[(o + i) * LDX + o + j] = x[i];
    }
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
#pragma unroll 1
    for (int h = 8; h < kBase; h *= 2) {
        const int tn = h / 8, tiles = (kBase / (2 * h)) * tn * tn;
        // T = B A^-1 (B: rows [o+h, o+2h), cols [o, o+h) of L)
        for (int t = warp; t < tiles; t += PT / 32) {
            const int p = t / (tn * tn), ti = (t / tn) % tn, tj = t % tn, o = 2 * h * p;
            double c0 = 0.0, c1 = 0.0;
            for (int k = 0; k < h; k += 4)
                dmma_884(c0, c1, sd[o + h + 8 * ti + fr][o + k + fc], X[(o + k + fc) * LDX + o + 8 * tj + fr]);
            double* tr = T + (p * h + 8 * ti + fr) * LDT + 8 * tj + 2 * fc;
            tr[0] = c0;
            tr[1] = c1;
        }
        __syncthreads();
        // X_off = -C^-1 T
        for (int t = warp; t < tiles; t += PT / 32) {
            const int p = t / (tn * tn), ti = (t / tn) % tn, tj = t % tn, o = 2 * h * p;
            double c0 = 0.0, c1 = 0.0;
            for (int k = 0; k < h; k += 4)
                dmma_884(c0, c1, X[(o + h + 8 * ti + fr) * LDX + o + h + k + fc], T[(p * h + k + fc) * LDT + 8 * tj + fr]);
            double* xr = X + (o + h + 8 * ti + fr) * LDX + o + 8 * tj + 2 * fc;
            xr[0] = -c0;
            xr[1] = -c1;
        }
        __syncthreads();
    }
}

// GENP of the 64x64 block in sd in place (lu.hpp:47-56 up to rounding),
// blocked by 16: per 16-column step, warp 0 factors the 16x16 diagonal block
// alone (two lanes per row, pivot rows through shared memory, warp barriers
// only), then every thread forms L21 rows (x U_D = a) or U12 columns
// (L_D y = a) by substitution, then the trailing block takes -L21 U12 on DMMA.
// 21.7k cycles per panel launch against 28.7k for the all-threads,
// two-steps-per-barrier elimination it replaced (clock64, RL_PANEL_PHASES);
// factorisation 16.86 -> 16.70 ms.
__device__ __forceinline__ void factor64_blocked(double (*sd)[kBase + 1], double (*pbuf)[2 * kBase], int tid) {
    const int warp = tid >> 5, lane = tid & 31;
    double* rinv16 = pbuf[0] + 64;  // reciprocals of the current block's pivots
#pragma unroll 1
    for (int kb = 0; kb < 4; ++kb) {
        const int J = 16 * kb, m = kBase - J - 16;
        if (warp == 0) {
            const int r = lane >> 1, h = lane & 1;
            double x[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = sd[J + r][J + 8 * h + c];
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                double* pv = pbuf[1] + 16 * (t & 1);
                if (r == t) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) pv[8 * h + c] = x[c];
                }
                __syncwarp();
                const double piv = pv[t];
                double ph[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) ph[c] = pv[8 * h + c];
                const double inv = rcp64(piv);
                if (lane == 0) rinv16[t] = inv;
                const double a_rt = __shfl_sync(kFull, x[t & 7], 2 * r + (t >> 3));
                const bool below = r > t;
                const double l = below ? div_by(a_rt, piv, inv) : 0.0;
                if (below && h == (t >> 3)) x[t & 7] = l;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (8 * h + c > t) x[c] = fma(-l, ph[c], x[c]);
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) sd[J + r][J + 8 * h + c] = x[c];
        }
        __syncthreads();
        if (m == 0) break;
        if (tid < m) {
            // L21 row i: x U_D = a, x_j = (a_j - sum_{q<j} x_q u_qj) / u_jj
            const int i = J + 16 + tid;
            double x[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) x[c] = sd[i][J + c];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
#pragma unroll
                for (int q = 0; q < j; ++q) x[j] = fma(-x[q], sd[J + q][J + j], x[j]);
                x[j] = div_by(x[j], sd[J + j][J + j], rinv16[j]);
            }
#pragma unroll
            for (int c = 0; c < 16; ++c) sd[i][J + c] = x[c];
        } else if (tid >= 64 && tid < 64 + m) {
            // U12 column c: L_D y = a (unit lower)
            const int c = J + 16 + tid - 64;
            double y[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) y[q] = sd[J + q][c];
#pragma unroll
            for (int i = 1; i < 16; ++i)
#pragma unroll
                for (int q = 0; q < i; ++q) y[i] = fma(-sd[J + i][J + q], y[q], y[i]);
#pragma unroll
            for (int q = 0; q < 16; ++q) sd[J + q][c] = y[q];
        }
        __syncthreads();
        {
            // A22 -= L21 U12 (K = 16) on DMMA, one 8x8 tile per warp at a time
            const int tn = m / 8, fr = lane >> 2, fc = lane & 3;
            for (int t = warp; t < tn * tn; t += PT / 32) {
                const int r0 = J + 16 + 8 * (t / tn), c0 = J + 16 + 8 * (t % tn);
                double v0 = sd[r0 + fr][c0 + 2 * fc], v1 = sd[r0 + fr][c0 + 2 * fc + 1];
#pragma unroll
                for (int k = 0; k < 16; k += 4) dmma_884(v0, v1, -sd[r0 + fr][J + k + fc], sd[J + k + fc][c0 + fr]);
                sd[r0 + fr][c0 + 2 * fc] = v0;
                sd[r0 + fr][c0 + 2 * fc + 1] = v1;
            }
        }
        __syncthreads();
    }
}

#ifdef RL_PANEL_PHASES
__device__ unsigned long long g_panel_phase[6];
#endif
// 8x8 tiles (ti0 + {0,1}, 0..7) of S = M N for 64x64 operands in shared
// memory (M row-major with stride ldm, N with stride ldn), one warp
__device__ __forceinline__ void mm64_rows2(const double* M, int ldm, const double* N, int ldn, int ti0, int lane,
                                           double (&acc)[2][8][2]) {
    const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
    for (int k = 0; k < kBase; k += 4) {
        double bf[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) bf[j] = N[(k + fc) * ldn + 8 * j + fr];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double af = M[(8 * (ti0 + i) + fr) * ldm + k + fc];
#pragma unroll
            for (int j = 0; j < 8; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af, bf[j]);
        }
    }
}

// inv128 != nullptr: one extra CTA (the last) builds this 64-column
// sub-panel's share of the super-panel's 128x128 unit-lower inverse (ld 128)
// from its factored copy, concurrently with the L21 rows, with kInvFusedSmem of
// dynamic shared memory:
//   half 0: [La^-1, 0] in rows 0..63
//   half 1: [-Lb^-1 (L_ba La^-1), Lb^-1] in rows 64..127 (L_ba: rows c0.., the
//           previous sub-panel's L21 columns; La^-1 from the half-0 launch)
// so U12 of the super-panel is one K = 128 GEMM.
template <int Q>
__global__ void __launch_bounds__(PT)
lu_panel64_kernel(double* __restrict__ a, int64_t lda, int64_t n, int64_t c0, int row_ctas,
                  double* __restrict__ piv_out, double* __restrict__ rinv_out, double* __restrict__ inv128, int half,
                  unsigned* __restrict__ tflag) {
    __shared__ double sd[kBase][kBase + 1];
    __shared__ __align__(16) double pbuf[2][2 * kBase];
    __shared__ double sp[kBase], sr[kBase];
    const int tid = threadIdx.x;
#ifdef RL_PANEL_PHASES
    const long long t0 = clock64();
#endif
    double* d = a + c0 * lda + c0;
    griddep_wait();  // programmatic launch on the lookahead chain: the update feeding this panel is done
    griddep_launch_dependents();
    if (inv128 && half == 1 && blockIdx.x == gridDim.x - 2) {
        // T = L_ba La^-1 needs nothing of this panel's factorisation: this CTA
        // forms it while the others factor, parks it in the (zero) top-right
        // block of the 128x128 inverse and raises tflag for the inverse CTA
        extern __shared__ double inv_smem[];
        double* Y = inv_smem;
        const double* lba = a + c0 * lda + (c0 - kBase);
        for (int idx = tid; idx < kBase * kBase; idx += PT) {
            const int i = idx >> 6, k = idx & 63;
            sd[i][k] = lba[i * lda + k];
            Y[i * LDX + k] = inv128[i * 128 + k];
        }
        __syncthreads();
        const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
        double acc[2][8][2];
        mm64_rows2(&sd[0][0], kBase + 1, Y, LDX, 2 * warp, lane, acc);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                double* o = inv128 + (8 * (2 * warp + i) + fr) * 128 + kBase + 8 * j + 2 * fc;
                o[0] = acc[i][j][0];
                o[1] = acc[i][j][1];
            }
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicExch(tflag, static_cast<unsigned>(c0 + 1));
        return;
    }
    for (int idx = tid; idx < kBase * kBase; idx += PT) sd[idx >> 6][idx & 63] = d[(idx >> 6) * lda + (idx & 63)];
    for (int idx = tid; idx < 4 * kBase; idx += PT) (&pbuf[0][0])[idx] = 0.0;
    __syncthreads();
#ifdef RL_PANEL_PHASES
    const long long t1 = clock64();
#endif
    factor64_blocked(sd, pbuf, tid);
    if (tid < kBase) {
        sp[tid] = sd[tid][tid];
        sr[tid] = 1.0 / sd[tid][tid];
    }
    __syncthreads();
    const int b = blockIdx.x;
#ifdef RL_PANEL_PHASES
    const long long t2 = clock64();
    if (tid == 0 && b == 0) {
        atomicExch(&g_panel_phase[0], static_cast<unsigned long long>(t1 - t0));
        atomicExch(&g_panel_phase[1], static_cast<unsigned long long>(t2 - t1));
        atomicExch(&g_panel_phase[3], 1ull);
    }
#endif
    if (inv128 && b == static_cast<int>(gridDim.x) - 1) {
        extern __shared__ double inv_smem[];
        double* X = inv_smem;
        double* Y = inv_smem + kBase * LDX;
        inv_unit_lower64(sd, X, Y, tid);  // X = L^-1 of this block (Y as scratch)
        double* dst = inv128 + half * (kBase * 128 + kBase);
        for (int idx = tid; idx < kBase * kBase; idx += PT) dst[(idx >> 6) * 128 + (idx & 63)] = X[(idx >> 6) * LDX + (idx & 63)];
        if (half == 0) {
            for (int idx = tid; idx < kBase * kBase; idx += PT) inv128[(idx >> 6) * 128 + kBase + (idx & 63)] = 0.0;
#ifdef RL_PANEL_PHASES
            if (tid == 0) atomicExch(&g_panel_phase[4], static_cast<unsigned long long>(clock64() - t2));
#endif
            return;
        }
        // off-diagonal block -Lb^-1 T, T = L_ba La^-1 from the CTA before this
        // one (all CTAs of a panel launch are co-resident: row_ctas + 2 <= 66)
        if (tid == 0)
            while (*reinterpret_cast<volatile unsigned*>(tflag) != static_cast<unsigned>(c0 + 1)) __nanosleep(64);
        __syncthreads();
        __threadfence();
        for (int idx = tid; idx < kBase * kBase; idx += PT) {
            const int i = idx >> 6, k = idx & 63;
            sd[i][k] = __ldcg(inv128 + i * 128 + kBase + k);
        }
        __syncthreads();
        for (int idx = tid; idx < kBase * kBase; idx += PT) inv128[(idx >> 6) * 128 + kBase + (idx & 63)] = 0.0;
        const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
        double acc[2][8][2];
        mm64_rows2(X, LDX, &sd[0][0], kBase + 1, 2 * warp, lane, acc);  // Lb^-1 T
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                double* o = inv128 + (kBase + 8 * (2 * warp + i) + fr) * 128 + 8 * j + 2 * fc;
                o[0] = -acc[i][j][0];
                o[1] = -acc[i][j][1];
            }
#ifdef RL_PANEL_PHASES
        if (tid == 0) atomicExch(&g_panel_phase[5], static_cast<unsigned long long>(clock64() - t2));
#endif
        return;
    }
    if (b == 0) {
        for (int idx = tid; idx < kBase * kBase; idx += PT) d[(idx >> 6) * lda + (idx & 63)] = sd[idx >> 6][idx & 63];
        if (tid < kBase) {
            piv_out[c0 + tid] = sp[tid];
            rinv_out[c0 + tid] = sr[tid];
        }
    }
    const int64_t rest = n - c0 - kBase;
    if (b < row_ctas) {
        // Q threads per row (lanes q = 0..Q-1 of a group), thread q holding
        // columns q, q + Q, ...: the owner of column j divides, the group
        // shares the quotient by a shuffle, each thread updates its columns.
        // Same operations per element in the same order as Q = 1.
        constexpr int RPC = PT / Q, NS = kBase / Q;
        const int q = tid % Q, lane = tid & 31;
        const int64_t r = c0 + kBase + static_cast<int64_t>(b) * RPC + tid / Q;
        if (r >= n) return;  // whole groups leave together
        const unsigned gm = Q == 1 ? 1u << lane : ((1u << Q) - 1u) << (lane & ~(Q - 1));
        double* rowp = a + r * lda + c0;
        double x[NS];
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) x[s2] = rowp[q + Q * s2];
#pragma unroll
        for (int j = 0; j < kBase; ++j) {
            const int s = j / Q, owner = j % Q;
            if (q == owner) x[s] = div_by(x[s], sp[j], sr[j]);
            const double xj = Q == 1 ? x[s] : __shfl_sync(gm, x[s], (lane & ~(Q - 1)) | owner);
            if (q > owner) x[s] = fma(-xj, sd[j][q + Q * s], x[s]);
#pragma unroll
            for (int s2 = s + 1; s2 < NS; ++s2) x[s2] = fma(-xj, sd[j][q + Q * s2], x[s2]);
        }
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) rowp[q + Q * s2] = x[s2];
#ifdef RL_PANEL_PHASES
        if (tid == 0 && b == 0) atomicExch(&g_panel_phase[2], static_cast<unsigned long long>(clock64() - t2));
#endif
    } else {
        const int64_t c = c0 + kBase + static_cast<int64_t>(b - row_ctas) * PT + tid;
        if (c - c0 - kBase >= rest) return;
        double* col = a + c0 * lda + c;
        double x[kBase];
#pragma unroll
        for (int i = 0; i < kBase; ++i) x[i] = col[i * lda];
#pragma unroll
        for (int k = 0; k < kBase - 1; ++k)
#pragma unroll
            for (int i = k + 1; i < kBase; ++i) x[i] = fma(-sd[i][k], x[k], x[i]);
#pragma unroll
        for (int i = 0; i < kBase; ++i) col[i * lda] = x[i];
    }
}

// Forward substitution (lu.hpp:110-115) by column blocks, right-looking,
// following the factorisation: once the panel of columns [c0, c0 + w) is
// factored, y_k = L_kk^-1 y_k (every CTA solves the w x w unit-lower diagonal
// block with a warp sweep; CTA 0 stores it to ys, never back into the
// working vector y that the other CTAs read it from), then each row below
// takes y_i -= L[i, c0:c0+w] y_k (one thread per row, its 64 loads in flight).
constexpr int FWD_ROWS = 256;  // rows below the block per CTA (one per thread)
__global__ void __launch_bounds__(256) fwd_panel_kernel(const double* __restrict__ a, int64_t lda, int64_t n,
                                                        int64_t c0, int w, double* __restrict__ y,
                                                        double* __restrict__ ys) {
    __shared__ double sl[kBase][kBase + 1];
    __shared__ double sy[kBase];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const double* d = a + c0 * lda + c0;
    for (int idx = tid; idx < kBase * kBase; idx += 256) {
        const int i = idx >> 6, k = idx & 63;
        sl[i][k] = (i < w && k < i) ? d[i * lda + k] : 0.0;
    }
    if (tid < kBase) sy[tid] = tid < w ? y[c0 + tid] : 0.0;
    __syncthreads();
    if (warp == 0) {
        double v0 = sy[lane], v1 = sy[lane + 32];
#pragma unroll
        for (int k = 0; k < kBase; ++k) {  // zero multipliers past w leave the values unchanged
            const double yk = __shfl_sync(kFull, k < 32 ? v0 : v1, k & 31);
            if (lane > k) v0 = fma(-sl[lane][k], yk, v0);
            if (lane + 32 > k) v1 = fma(-sl[lane + 32][k], yk, v1);
        }
        sy[lane] = v0;
        sy[lane + 32] = v1;
    }
    __syncthreads();
    if (blockIdx.x == 0 && tid < w) ys[c0 + tid] = sy[tid];
    // rows below: one thread per row, every load of the row in flight at once
    const int64_t r = c0 + w + static_cast<int64_t>(blockIdx.x) * FWD_ROWS + tid;
    if (tid < FWD_ROWS && r < n) {
        const double* lr = a + r * lda + c0;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (w == kBase) {
#pragma unroll
            for (int j = 0; j < kBase; j += 2) {
                const double2 v = __ldcg(reinterpret_cast<const double2*>(lr + j));
                acc[j & 3] = fma(v.x, sy[j], acc[j & 3]);
                acc[(j + 1) & 3] = fma(v.y, sy[j + 1], acc[(j + 1) & 3]);
            }
        } else {
            for (int j = 0; j < w; ++j) acc[j & 3] = fma(lr[j], sy[j], acc[j & 3]);
        }
        y[r] -= (acc[0] + acc[1]) + (acc[2] + acc[3]);
    }
}

// ---- U12 = L11^-1 A12 for the trailing columns of a 64-row panel ---------
// (the column half of the fused step, split out so it can run after the
// trailing update of the previous step while the next panel factors on the
// lookahead stream); L11 comes from the already factored diagonal block.
__global__ void __launch_bounds__(PT)
lu_u12_kernel(double* __restrict__ a, int64_t lda, int64_t c0, int64_t col_begin, int64_t ncols) {
    __shared__ double sl[kBase][kBase + 1];
    const int tid = threadIdx.x;
    const double* d = a + c0 * lda + c0;
    for (int idx = tid; idx < kBase * kBase; idx += PT) sl[idx >> 6][idx & 63] = d[(idx >> 6) * lda + (idx & 63)];
    __syncthreads();
    const int64_t cidx = static_cast<int64_t>(blockIdx.x) * PT + tid;
    if (cidx >= ncols) return;
    double* col = a + c0 * lda + col_begin + cidx;
    double x[kBase];
#pragma unroll
    for (int i = 0; i < kBase; ++i) x[i] = col[i * lda];
#pragma unroll
    for (int k = 0; k < kBase - 1; ++k)
#pragma unroll
        for (int i = k + 1; i < kBase; ++i) x[i] = fma(-sl[i][k], x[k], x[i]);
#pragma unroll
    for (int i = 0; i < kBase; ++i) col[i * lda] = x[i];
}

struct Ctx {
    rl_context* ctx;
    double* a;
    int64_t n, lda;
    double* piv;
    double* rinv;
};

// the ragged last block (w < 64 columns): diagonal block in one CTA, then L21
rl_status panel(const Ctx& g, int64_t c0, int64_t w) {
    const int64_t m = g.n - c0;
    double* d = g.a + c0 * g.lda + c0;
    panel_diag_kernel<<<1, 256, 0, g.ctx->stream>>>(d, g.lda, static_cast<int>(w), g.piv + c0, g.rinv + c0);
    RL_CHECK_LAUNCH("panel_diag_kernel");
    const int64_t rows = m - w;
    if (rows > 0) {
        const unsigned blocks = static_cast<unsigned>((rows + 127) / 128);
        double* r = g.a + (c0 + w) * g.lda + c0;
        panel_rows_kernel_dyn<<<blocks, 128, 0, g.ctx->stream>>>(r, g.lda, rows, static_cast<int>(w), d, g.piv + c0,
                                                                 g.rinv + c0);
        RL_CHECK_LAUNCH("panel_rows_kernel_dyn");
    }
    return RL_OK;
}

}  // namespace

// Right-looking GENP in 128-column super-panels, each factored as two
// 64-column sub-panels, so that the bulk trailing update is one K = 128 GEMM
// per super-panel (half the C read/write traffic per flop of K = 64), with a
// one-super-panel lookahead on two streams:
//   hi: U12 of the next super-panel's 128 columns -> GEMM_a1 (its first 64
//       columns) -> factor_super(s+1)
//   lo: GEMM_a2 (its other 64 columns) -> U12(s) for every later column ->
//       GEMM_b(s), the lookahead's next columns first
// factor_super(c0): panel_L(c0); U12 of the first half onto the second half's
// 64 columns; their K = 64 update; panel_L(c0 + 64).
// U12(s) = L11^-1 A12 is one K = 128 GEMM with the super-panel's 128x128
// unit-lower inverse, assembled by the two panel launches' extra CTAs. The
// chain on hi is latency-bound late in the factorisation; its kernels are
// launched with programmatic stream serialization (griddepcontrol) so each
// starts while its predecessor drains.
#ifdef RL_GENP_TRACE
// developer timeline of the lookahead schedule (never in the product build):
// one-thread kernels stamp %globaltimer into a managed buffer
__global__ void stamp_kernel(unsigned long long* slot) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *slot = t;
}
struct GenpTrace {
    unsigned long long* buf = nullptr;
    std::vector<int> tags;
    GenpTrace() { cudaMallocManaged(&buf, 8 * 4096); }
    void mark(int tag, cudaStream_t s) {
        if (tags.size() >= 4096) return;
        stamp_kernel<<<1, 1, 0, s>>>(buf + tags.size());
        tags.push_back(tag);
    }
    ~GenpTrace() {
        cudaDeviceSynchronize();
#ifdef RL_PANEL_PHASES
        unsigned long long ph[6];
        cudaMemcpyFromSymbol(ph, g_panel_phase, sizeof(ph));
        std::fprintf(stderr, "P load %.0f factor %.0f rows %.0f inv0 %.0f inv1 %.0f cycles (last launch)\n",
                     double(ph[0]), double(ph[1]), double(ph[2]), double(ph[4]), double(ph[5]));
#endif
        for (size_t i = 0; i < tags.size(); ++i)
            std::fprintf(stderr, "T %d %.1f\n", tags[i], (buf[i] - buf[0]) * 1e-3);
        cudaFree(buf);
    }
};
#define TRACE(tag, s) trace.mark(tag, s)
#else
#define TRACE(tag, s) \
    do {              \
    } while (0)
#endif
static rl_status genp_super128(rl_context* ctx, int64_t n, double* a, int64_t lda, double* piv_out,
                               double* rinv_out, const double* fwd_b, double* fwd_y) {
    constexpr int64_t W = 2 * kBase;
    const int64_t S = n / W;  // full super-panels
    Ctx g{ctx, a, n, lda, piv_out, rinv_out};
    rl_status st;
    constexpr int kRing = 8, kFsRing = 8;
    if ((st = side_resources(ctx, kRing + 2 + kFsRing)) != RL_OK) return st;
    cudaStream_t lo = ctx->stream, hi = ctx->hi_stream, fs = ctx->fs_stream;
    cudaEvent_t* ev = ctx->events;
    int e = 0, f = 0;
    auto next_event = [&]() { return ev[2 + (e++ % kRing)]; };
    auto at = [&](int64_t r, int64_t c) { return a + r * lda + c; };
    double* fwd_work = nullptr;  // the working right-hand side (fs-stream-ordered scratch)
    // the forward substitution of columns [c0, c0 + w) on fs, once their panel
    // (enqueued on sm) is done
    auto fwd_after = [&](cudaStream_t sm, int64_t c0, int64_t w) -> rl_status {
        if (!fwd_y) return RL_OK;
        cudaEvent_t ef = ev[2 + kRing + (f++ % (kFsRing - 1))];  // the last one is fwd_guard's
        RL_CUDA(cudaEventRecord(ef, sm));
        RL_CUDA(cudaStreamWaitEvent(fs, ef, 0));
        const int64_t below = n - c0 - w;
        const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, (below + FWD_ROWS - 1) / FWD_ROWS));
        fwd_panel_kernel<<<grid, 256, 0, fs>>>(a, lda, n, c0, static_cast<int>(w), fwd_work, fwd_y);
        RL_CHECK_LAUNCH("fwd_panel_kernel");
        return RL_OK;
    };
    // GEMM C -= A B on stream sm (ctx->stream is what gemm() launches on)
    // programmatic dependent launch for kernels on the lookahead chain (hi),
    // except right after a cross-stream event wait (only kernel-to-kernel edges
    // of one stream are relaxed)
    bool hi_waited = true;
    auto hi_wait = [&](cudaEvent_t e) -> rl_status {
        RL_CUDA(cudaStreamWaitEvent(hi, e, 0));
        hi_waited = true;
        return RL_OK;
    };
    auto use_pdl = [&](cudaStream_t sm) {
#ifdef RL_NO_PDL
        return false;
#endif
        if (sm != hi) return false;
        const bool ok = !hi_waited;
        hi_waited = false;
        return ok;
    };
    auto update = [&](cudaStream_t sm, int64_t M, int64_t N, int64_t Kd, const double* A, const double* B,
                      double* C) -> rl_status {
        if (M <= 0 || N <= 0) return RL_OK;
        cudaStream_t keep = ctx->stream;
        ctx->stream = sm;
        ctx->pdl = use_pdl(sm);
        const rl_status r = gemm(ctx, M, N, Kd, A, lda, B, lda, C, lda, -1.0, true, nullptr);
        ctx->pdl = false;
        ctx->stream = keep;
        return r;
    };
    static PerDeviceOnce inv_configured_once;
    {
        const rl_status cst = once_per_device(inv_configured_once, [&]() -> rl_status {
            RL_CUDA(cudaFuncSetAttribute(lu_panel64_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kInvFusedSmem));
            RL_CUDA(cudaFuncSetAttribute(lu_panel64_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kInvFusedSmem));
            RL_CUDA(cudaFuncSetAttribute(lu_panel64_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kInvFusedSmem));
            return RL_OK;
        });
        if (cst != RL_OK) return cst;
    }
    // per super-panel 128x128 unit-lower L11^-1 (128 KiB each, ld 128; the
    // ragged tail's 64-column step uses the top-left block of one more),
    // stream-ordered scratch
    double* inv = nullptr;
    RL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&inv), sizeof(double) * W * W * (S + 1) + 256, lo));
    // the T-ready flag of the second-half panel launches (values c0 + 1, never reused)
    unsigned* tflag = reinterpret_cast<unsigned*>(inv + W * W * (S + 1));
    RL_CUDA(cudaMemsetAsync(tflag, 0, 256, lo));
    struct Free {
        double* p;
        cudaStream_t s;
        ~Free() { cudaFreeAsync(p, s); }
    } inv_guard{inv, lo};
    auto inv_of = [&](int64_t c0) { return inv + (c0 / W) * W * W; };  // super-panel containing column c0
    // panel: factor the diagonal block and L21 = A21 U11^-1 by substitution;
    // the extra CTA fills this half of the super-panel's L11^-1
    auto panel_l = [&](cudaStream_t sm, int64_t c0) -> rl_status {
        // late panels sit on the exposed lookahead chain with idle SMs: more
        // threads per row shorten the L21 substitution (RL_PANEL_Q4_ROWS)
        const int64_t rest = n - c0 - kBase;
        const int q = rest <= kPanelQ4Rows ? 4 : (rest <= 2 * kPanelQ4Rows ? 2 : 1);
        const int rpc = PT / q;
        const int blocks = static_cast<int>(std::max<int64_t>(1, (rest + rpc - 1) / rpc));
        const int half = static_cast<int>((c0 / kBase) & 1);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(blocks + 1 + half));
        cfg.blockDim = dim3(PT);
        cfg.dynamicSmemBytes = kInvFusedSmem;
        cfg.stream = sm;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = use_pdl(sm) ? 1 : 0;
        double* inv_c = inv_of(c0);
        if (q == 4)
            cudaLaunchKernelEx(&cfg, lu_panel64_kernel<4>, a, lda, n, c0, blocks, piv_out, rinv_out, inv_c, half, tflag);
        else if (q == 2)
            cudaLaunchKernelEx(&cfg, lu_panel64_kernel<2>, a, lda, n, c0, blocks, piv_out, rinv_out, inv_c, half, tflag);
        else
            cudaLaunchKernelEx(&cfg, lu_panel64_kernel<1>, a, lda, n, c0, blocks, piv_out, rinv_out, inv_c, half, tflag);
        RL_CHECK_LAUNCH("lu_panel64_kernel");
        return fwd_after(sm, c0, kBase);
    };
    // U12 = L11^-1 A12 in place for rows [r0, r0 + rows), rows = 64 (the
    // top-left block) or 128 (the whole super-panel inverse): gemm_inplace_b
    // keeps one CTA tile row, so each output column block reads all of its
    // own input before any store (a 64-row tile configuration here once let a
    // late-scheduled second tile row read rows the first had overwritten)
    auto u12 = [&](cudaStream_t sm, int64_t r0, int64_t rows, int64_t cb, int64_t ncols) -> rl_status {
        if (ncols <= 0) return RL_OK;
        cudaStream_t keep = ctx->stream;
        ctx->stream = sm;
        ctx->pdl = use_pdl(sm);
        const rl_status r = gemm_inplace_b(ctx, rows, ncols, rows, inv_of(r0), W, at(r0, cb), lda);
        ctx->pdl = false;
        ctx->stream = keep;
        return r;
    };
#ifdef RL_GENP_TRACE
    GenpTrace trace;
#endif
    // second_ready: the event after which the second half's 64 columns are
    // fully updated (GEMM_a2 on the other stream), or nullptr
    auto factor_super = [&](cudaStream_t sm, int64_t c0, cudaEvent_t second_ready) -> rl_status {
        rl_status r;
        if ((r = panel_l(sm, c0)) != RL_OK) return r;
        TRACE(6, sm);
        if (second_ready) {
            if (sm == hi) {
                if ((r = hi_wait(second_ready)) != RL_OK) return r;
            } else {
                RL_CUDA(cudaStreamWaitEvent(sm, second_ready, 0));
            }
        }
        if ((r = u12(sm, c0, kBase, c0 + kBase, kBase)) != RL_OK) return r;
        TRACE(7, sm);
        if ((r = update(sm, n - c0 - kBase, kBase, kBase, at(c0 + kBase, c0), at(c0, c0 + kBase),
                        at(c0 + kBase, c0 + kBase))) != RL_OK)
            return r;
        TRACE(8, sm);
        return panel_l(sm, c0 + kBase);
    };
    TRACE(0, lo);
    RL_CUDA(cudaEventRecord(ev[0], lo));  // prior work on the caller's stream
    if (fwd_y) {
        RL_CUDA(cudaStreamWaitEvent(fs, ev[0], 0));
        RL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&fwd_work), sizeof(double) * n, fs));
        RL_CUDA(cudaMemcpyAsync(fwd_work, fwd_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, fs));
    }
    // on every exit (errors included) the caller's stream orders after the
    // forward-substitution stream, which writes fwd_y, and its scratch is freed
    struct FsJoin {
        double* p;
        cudaStream_t fs, lo;
        cudaEvent_t ev;
        ~FsJoin() {
            if (!p) return;
            cudaEventRecord(ev, fs);
            cudaStreamWaitEvent(lo, ev, 0);
            cudaFreeAsync(p, fs);
        }
    } fwd_guard{fwd_work, fs, lo, ev[2 + kRing + kFsRing - 1]};
    if ((st = hi_wait(ev[0])) != RL_OK) return st;
    if ((st = factor_super(hi, 0, nullptr)) != RL_OK) return st;
    cudaEvent_t el = next_event();
    RL_CUDA(cudaEventRecord(el, hi));
    // Per super-panel s (c0 = s W), the lookahead chain on hi is
    //   U12 of the next super-panel's own 128 columns -> GEMM_a1 (its first 64
    //   columns) -> panel_L -> [GEMM_a2 from lo] -> small U12 -> update -> panel_L
    // while lo runs GEMM_a2 (the next super-panel's other 64 columns), U12 of
    // every later column and GEMM_b. hi's U12 waits only for lo's GEMM_b(s-1)
    // (which last touched those columns), not for lo's U12 of all the rest.
    cudaEvent_t eb = nullptr;  // lo: GEMM_b(s-1) done
    for (int64_t sp = 0; sp < S; ++sp) {
        const int64_t c0 = sp * W, rest = n - c0 - W;
        if (rest <= 0) break;
        const bool next_full = sp + 1 < S;
        RL_CUDA(cudaStreamWaitEvent(lo, el, 0));  // factor_super(s): L21, U11, L11^-1
        TRACE(1, lo);
        if (next_full) {
            // hi: U12 of columns [c0 + W, c0 + 2W), GEMM_a1
            if (eb && (st = hi_wait(eb)) != RL_OK) return st;
            if ((st = u12(hi, c0, W, c0 + W, W)) != RL_OK) return st;
            cudaEvent_t eua = next_event();
            RL_CUDA(cudaEventRecord(eua, hi));
            TRACE(2, hi);
            if ((st = update(hi, rest, kBase, W, at(c0 + W, c0), at(c0, c0 + W), at(c0 + W, c0 + W))) != RL_OK)
                return st;
            TRACE(3, hi);
            // lo: GEMM_a2 (the next super-panel's second 64 columns)
            RL_CUDA(cudaStreamWaitEvent(lo, eua, 0));
            if ((st = update(lo, rest, kBase, W, at(c0 + W, c0), at(c0, c0 + W + kBase), at(c0 + W, c0 + W + kBase))) !=
                RL_OK)
                return st;
            cudaEvent_t ea2 = next_event();
            RL_CUDA(cudaEventRecord(ea2, lo));
            // hi: factor_super(s+1), its second half after GEMM_a2
            if ((st = factor_super(hi, c0 + W, ea2)) != RL_OK) return st;
            TRACE(4, hi);
            el = next_event();
            RL_CUDA(cudaEventRecord(el, hi));
        }
        // lo: U12 and GEMM_b(s) on the remaining columns (all of them before the tail)
        const int64_t cb = next_full ? c0 + 2 * W : c0 + W;
        if ((st = u12(lo, c0, W, cb, n - cb)) != RL_OK) return st;
        // the columns the lookahead needs next (super-panel s+2) first, so the
        // chain on hi waits only for them; then the rest. (Pairing two
        // super-panels' bulk updates into one K = 2W GEMM, bit-identical, was
        // measured slower: 17.0 against 16.9 ms.)
        const int64_t first = next_full ? std::min<int64_t>(W, n - cb) : n - cb;
        if ((st = update(lo, rest, first, W, at(c0 + W, c0), at(c0, cb), at(c0 + W, cb))) != RL_OK) return st;
        eb = next_event();
        RL_CUDA(cudaEventRecord(eb, lo));
        if (n - cb > first &&
            (st = update(lo, rest, n - cb - first, W, at(c0 + W, c0), at(c0, cb + first), at(c0 + W, cb + first))) !=
                RL_OK)
            return st;
        TRACE(5, lo);
    }
    RL_CUDA(cudaEventRecord(ev[1], hi));
    RL_CUDA(cudaStreamWaitEvent(lo, ev[1], 0));
    // tail (< 128 columns, fully updated): one 64-column step, then the ragged rest
    int64_t c0 = S * W;
    if (n - c0 >= kBase) {
        if ((st = panel_l(lo, c0)) != RL_OK) return st;
        const int64_t rest = n - c0 - kBase;
        if ((st = u12(lo, c0, kBase, c0 + kBase, rest)) != RL_OK) return st;
        if ((st = update(lo, rest, rest, kBase, at(c0 + kBase, c0), at(c0, c0 + kBase), at(c0 + kBase, c0 + kBase))) !=
            RL_OK)
            return st;
        c0 += kBase;
    }
    if (c0 < n) {
        if ((st = panel(g, c0, n - c0)) != RL_OK) return st;
        if ((st = fwd_after(lo, c0, n - c0)) != RL_OK) return st;
    }
    return RL_OK;  // fwd_guard: the caller's stream sees y
}

rl_status genp_inplace(rl_context* ctx, int64_t n, double* a, int64_t lda, double* piv_out, double* rinv_out,
                       const double* fwd_b, double* fwd_y, bool* fwd_done) {
    if (fwd_done) *fwd_done = false;
    if (n <= 0) return RL_OK;
    Ctx g{ctx, a, n, lda, piv_out, rinv_out};
    const int64_t K = n / kBase;  // full 64-column panels
    rl_status st;
    if (K >= 4) {
        const bool fwd = fwd_b && fwd_y && fwd_done;
        st = genp_super128(ctx, n, a, lda, piv_out, rinv_out, fwd ? fwd_b : nullptr, fwd ? fwd_y : nullptr);
        if (st == RL_OK && fwd) *fwd_done = true;
        return st;
    }
    if (K >= 3) {
        // right-looking GENP with a one-panel lookahead on two streams:
        //   hi: GEMM_a(k) (next panel's 64 columns) -> panel_L(k+1)
        //   lo: U12(k) -> GEMM_b(k) (all later columns)
        // so the latency-bound panel factorisation of step k+1 runs under the
        // bulk trailing update of step k.
        constexpr int kRing = 8;
        if ((st = side_resources(ctx, kRing + 2)) != RL_OK) return st;
        cudaStream_t lo = ctx->stream, hi = ctx->hi_stream;
        cudaEvent_t* ev = ctx->events;
        int e = 0;
        auto next_event = [&]() { return ev[2 + (e++ % kRing)]; };
        RL_CUDA(cudaEventRecord(ev[0], lo));  // prior work on the caller's stream
        RL_CUDA(cudaStreamWaitEvent(hi, ev[0], 0));
        auto panel_l = [&](int64_t c0) -> rl_status {
            const int64_t rest = n - c0 - kBase;
            const int blocks = static_cast<int>(std::max<int64_t>(1, (rest + PT - 1) / PT));
            lu_panel64_kernel<1><<<blocks, PT, 0, hi>>>(a, lda, n, c0, blocks, piv_out, rinv_out, nullptr, 0, nullptr);
            RL_CHECK_LAUNCH("lu_panel64_kernel");
            return RL_OK;
        };
        if ((st = panel_l(0)) != RL_OK) return st;
        cudaEvent_t el = next_event();
        RL_CUDA(cudaEventRecord(el, hi));
        for (int64_t k = 0; k < K; ++k) {
            const int64_t c0 = k * kBase, rest = n - c0 - kBase;
            if (rest <= 0) break;
            // lo: U12(k) for all trailing columns
            RL_CUDA(cudaStreamWaitEvent(lo, el, 0));
            lu_u12_kernel<<<static_cast<unsigned>((rest + PT - 1) / PT), PT, 0, lo>>>(a, lda, c0, c0 + kBase, rest);
            RL_CHECK_LAUNCH("lu_u12_kernel");
            cudaEvent_t eu = next_event();
            RL_CUDA(cudaEventRecord(eu, lo));
            const int64_t wa = std::min<int64_t>(kBase, rest);  // next panel's columns
            const bool next_full = (k + 1 < K);
            // hi: GEMM_a(k) -> panel_L(k+1)
            RL_CUDA(cudaStreamWaitEvent(hi, eu, 0));
            if (next_full) {
                cudaStream_t keep = ctx->stream;
                ctx->stream = hi;
                st = gemm(ctx, rest, wa, kBase, a + (c0 + kBase) * lda + c0, lda, a + c0 * lda + c0 + kBase, lda,
                          a + (c0 + kBase) * lda + c0 + kBase, lda, -1.0, true, nullptr);
                ctx->stream = keep;
                if (st != RL_OK) return st;
                if ((st = panel_l(c0 + kBase)) != RL_OK) return st;
                el = next_event();
                RL_CUDA(cudaEventRecord(el, hi));
            }
            // lo: GEMM_b(k) on the remaining columns (or all of them when the
            // ragged tail follows)
            const int64_t cb = next_full ? c0 + 2 * kBase : c0 + kBase;
            const int64_t nb = n - cb;
            if (nb > 0) {
                st = gemm(ctx, rest, nb, kBase, a + (c0 + kBase) * lda + c0, lda, a + c0 * lda + cb, lda,
                          a + (c0 + kBase) * lda + cb, lda, -1.0, true, nullptr);
                if (st != RL_OK) return st;
            }
        }
        RL_CUDA(cudaEventRecord(ev[1], hi));
        RL_CUDA(cudaStreamWaitEvent(lo, ev[1], 0));
        const int64_t c0 = K * kBase;
        if (c0 < n) return panel(g, c0, n - c0);  // ragged last block (< 64 columns)
        return RL_OK;
    }
    // small matrices: fused steps on one stream
    int64_t c0 = 0;
    for (; c0 + kBase <= n; c0 += kBase) {
        const int64_t rest = n - c0 - kBase;
        const int blocks = static_cast<int>((rest + PT - 1) / PT);
        lu_panel64_kernel<1><<<std::max(1, 2 * blocks), PT, 0, ctx->stream>>>(a, lda, n, c0, blocks, piv_out, rinv_out,
                                                                        nullptr, 0, nullptr);
        RL_CHECK_LAUNCH("lu_panel64_kernel");
        if (rest > 0) {
            st = gemm(ctx, rest, rest, kBase, a + (c0 + kBase) * lda + c0, lda, a + c0 * lda + c0 + kBase, lda,
                      a + (c0 + kBase) * lda + c0 + kBase, lda, -1.0, true, nullptr);
            if (st != RL_OK) return st;
        }
    }
    if (c0 < n) return panel(g, c0, n - c0);  // ragged last block (< 64 columns)
    return RL_OK;
}

}  // namespace rl
