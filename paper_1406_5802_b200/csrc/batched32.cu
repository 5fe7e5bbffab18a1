// Batched small GENP — BASELINE config 2: many independent 32x32 systems,
// each preprocess_solve(A_i, b_i, none, {Gaussian, G_i}, refine)
// (preprocess.hpp:156-180) on one warp, register-resident.
//
// Per system (one warp):
//   1. A_i, G_i -> shared memory (coalesced 16-byte streaming loads).
//   2. P = A_i G_i with FP64 tensor-core MMA (mma.sync m8n8k4, 128 DMMA).
//   3. P row-per-lane in registers; exact-order row/column norms
//      (norms.hpp:38-50 floor) and ||P||_F bound the pivot tolerance.
//   4. GENP (lu.hpp:47-56): 31 unrolled elimination steps; the pivot row is
//      broadcast through a 256-byte shared row buffer, every lane divides its
//      own multiplier. All pivots are seen by every lane (warp-uniform).
//   5. Verdict: tol = tol_pivot(32) * spectral_norm_estimate(P) (lu.hpp:44).
//      floor <= estimate <= ||P||_F, so the power iteration runs only when a
//      pivot lies in the band (tol_pivot*floor, tol_pivot*||P||_F]; it then
//      runs in the reference's exact summation order (no FMA), so the verdict
//      is the reference's.
//   6. Solves (lu.hpp:110-122) with shuffle broadcasts, x = G y, residual
//      ||b - A x|| / ||b|| (lu.hpp:155-161 / preprocess.hpp:122-128),
//      growth max|U| / max|P|, packed LU written back coalesced.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "device_common.cuh"
#include "runtime.cuh"

namespace rl {
namespace {

constexpr int D = 32;
constexpr int LD = 36;  // padded shared row stride (doubles): conflict-free DMMA fragments
constexpr int WARPS = 4;
constexpr int MAT = D * LD;
constexpr double kTolPivot32 = 1e-13 * 32.0;  // tol_pivot(32), types.hpp:42

struct __align__(16) WarpSmem {
    double A[MAT];
    double G[MAT];
    double P[MAT];
    double vec[D];
    double piv[D];
    double scratch[D];
};
constexpr size_t kSmemBytes = sizeof(WarpSmem) * WARPS;

__device__ __forceinline__ void load_matrix(double* s, const double* g, int lane) {
    const double2* g2 = reinterpret_cast<const double2*>(g);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int p = lane + 32 * q;
        const double2 v = ld_stream(g2 + p);
        *reinterpret_cast<double2*>(s + (p >> 4) * LD + 2 * (p & 15)) = v;
    }
}

__device__ __forceinline__ void store_matrix(double* g, const double* s, int lane) {
    double2* g2 = reinterpret_cast<double2*>(g);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int p = lane + 32 * q;
        st_stream(g2 + p, *reinterpret_cast<const double2*>(s + (p >> 4) * LD + 2 * (p & 15)));
    }
}

// spectral_norm_estimate (norms.hpp:52-77) of the 32x32 matrix in s.P, in the
// reference's summation order with separately rounded multiplies and adds, so
// the estimate is bit-identical to the reference's for the same matrix.
__device__ double exact_power_iteration(WarpSmem& s, int lane) {
    double* x = s.vec;
    if (lane == 0) {
        for (int j = 0; j < D; ++j) x[j] = 1.0 + static_cast<double>(j) / (static_cast<double>(D) + 1.0);
        double nx = 0.0;
        for (int j = 0; j < D; ++j) nx = __dadd_rn(nx, __dmul_rn(x[j], x[j]));
        nx = sqrt(nx);
        const double inv = 1.0 / nx;
        for (int j = 0; j < D; ++j) x[j] = __dmul_rn(inv, x[j]);
    }
    __syncwarp();
    double est = 0.0;
    for (int it = 0; it < 200; ++it) {
        double axi = 0.0;  // (A x)_lane, j ascending (matrix.hpp:149-154)
        for (int j = 0; j < D; ++j) axi = __dadd_rn(axi, __dmul_rn(s.P[lane * LD + j], x[j]));
        s.scratch[lane] = axi;
        __syncwarp();
        double nax = 0.0;
        for (int i = 0; i < D; ++i) nax = __dadd_rn(nax, __dmul_rn(s.scratch[i], s.scratch[i]));
        nax = sqrt(nax);
        if (nax == 0.0) break;
        double yj = 0.0;  // (A^T A x)_lane, i ascending (norms.hpp:60-63)
        for (int i = 0; i < D; ++i) yj = __dadd_rn(yj, __dmul_rn(s.P[i * LD + lane], s.scratch[i]));
        __syncwarp();
        x[lane] = yj;
        __syncwarp();
        double ny = 0.0;
        for (int j = 0; j < D; ++j) ny = __dadd_rn(ny, __dmul_rn(x[j], x[j]));
        ny = sqrt(ny);
        if (ny == 0.0) break;
        const double inv = 1.0 / ny;
        __syncwarp();
        x[lane] = __dmul_rn(inv, yj);
        __syncwarp();
        if (fabs(nax - est) <= 1e-9 * nax) {
            est = nax;
            break;
        }
        est = nax;
    }
    __syncwarp();
    return est;
}

__global__ void __launch_bounds__(WARPS * 32, 2)
batched_genp32_kernel(const double* __restrict__ gA, const double* __restrict__ gG, const double* __restrict__ gB,
                      double* __restrict__ gLU, double* __restrict__ gX, double* __restrict__ gR,
                      double* __restrict__ gGrowth, int32_t* __restrict__ gStatus, int64_t batch, int refine) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& s = reinterpret_cast<WarpSmem*>(smem_raw)[warp];

    for (int64_t sys = static_cast<int64_t>(blockIdx.x) * WARPS + warp; sys < batch;
         sys += static_cast<int64_t>(gridDim.x) * WARPS) {
        const size_t mo = static_cast<size_t>(sys) * D * D;
        load_matrix(s.A, gA + mo, lane);
        load_matrix(s.G, gG + mo, lane);
        const double bl = gB[sys * D + lane];
        __syncwarp();

        // ---- P = A G on the FP64 tensor path (4x4 tiles of 8x8, k = 4 per MMA)
        {
            double c[4][4][2];
#pragma unroll
            for (int ti = 0; ti < 4; ++ti)
#pragma unroll
                for (int tj = 0; tj < 4; ++tj) c[ti][tj][0] = c[ti][tj][1] = 0.0;
            const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                double af[4], bf[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    af[t] = s.A[(8 * t + fr) * LD + 4 * kk + fc];
                    bf[t] = s.G[(4 * kk + fc) * LD + 8 * t + fr];
                }
#pragma unroll
                for (int ti = 0; ti < 4; ++ti)
#pragma unroll
                    for (int tj = 0; tj < 4; ++tj) dmma_884(c[ti][tj][0], c[ti][tj][1], af[ti], bf[tj]);
            }
#pragma unroll
            for (int ti = 0; ti < 4; ++ti)
#pragma unroll
                for (int tj = 0; tj < 4; ++tj)
                    *reinterpret_cast<double2*>(&s.P[(8 * ti + fr) * LD + 8 * tj + 2 * fc]) =
                        make_double2(c[ti][tj][0], c[ti][tj][1]);
        }
        __syncwarp();

        // ---- row `lane` of P into registers; norms in the reference's order
        double p[D];
#pragma unroll
        for (int m = 0; m < D / 2; ++m) {
            const double2 v = *reinterpret_cast<const double2*>(&s.P[lane * LD + 2 * m]);
            p[2 * m] = v.x;
            p[2 * m + 1] = v.y;
        }
        double rowsq = 0.0, colsq = 0.0, amax = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            rowsq = __dadd_rn(rowsq, __dmul_rn(p[k], p[k]));
            amax = fmax(amax, fabs(p[k]));
        }
#pragma unroll 8
        for (int i = 0; i < D; ++i) {
            const double v = s.P[i * LD + lane];
            colsq = __dadd_rn(colsq, __dmul_rn(v, v));
        }
        const double floor_norm = sqrt(warp_max(fmax(rowsq, colsq)));
        const double fro = sqrt(warp_sum(rowsq));
        const double max_p = warp_max(amax);
        const double tol_lo = kTolPivot32 * floor_norm;
        const double tol_hi = kTolPivot32 * fro * (1.0 + 1e-10);

        // ---- GENP, natural pivot order, no exchanges (lu.hpp:47-56)
        int first_hi = 0;
        double piv_first_hi = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if (lane == j) {
#pragma unroll
                for (int m = j / 2; m < D / 2; ++m)
                    *reinterpret_cast<double2*>(&s.vec[2 * m]) = make_double2(p[2 * m], p[2 * m + 1]);
            }
            __syncwarp();
            double r[D];
#pragma unroll
            for (int m = j / 2; m < D / 2; ++m) {
                const double2 v = *reinterpret_cast<const double2*>(&s.vec[2 * m]);
                r[2 * m] = v.x;
                r[2 * m + 1] = v.y;
            }
            const double piv = r[j];
            if (lane == 0) s.piv[j] = piv;
            if (first_hi == 0 && fabs(piv) <= tol_hi) {
                first_hi = j + 1;
                piv_first_hi = piv;
            }
            if (lane > j) {
                const double l = p[j] / piv;
                p[j] = l;
#pragma unroll
                for (int k = j + 1; k < D; ++k) p[k] = fma(-l, r[k], p[k]);
            }
            __syncwarp();
        }

        // ---- verdict (lu.hpp:44,49)
        int zero_step = 0;
        if (first_hi != 0) {
            if (fabs(piv_first_hi) <= tol_lo) {
                zero_step = first_hi;
            } else {
                const double est = fmax(exact_power_iteration(s, lane), floor_norm);
                const double tol = kTolPivot32 * est;
                for (int j = 0; j < D; ++j)
                    if (fabs(s.piv[j]) <= tol) {
                        zero_step = j + 1;
                        break;
                    }
            }
        }

        // ---- growth max|U| / max|P|
        double umax = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k)
            if (k >= lane) umax = fmax(umax, fabs(p[k]));
        umax = warp_max(umax);

        // ---- chain solve x = G (LU)^-1 r, refinement (preprocess.hpp:115-143)
        const double bnorm = sqrt(warp_sum(bl * bl));
        double x = 0.0, rl_ = bl, rel = 0.0;
        for (int step = 0; step <= refine; ++step) {
            double y = rl_;
#pragma unroll
            for (int k = 0; k < D; ++k) {  // forward, unit L
                const double yk = __shfl_sync(kFull, y, k);
                if (lane > k) y = fma(-p[k], yk, y);
            }
#pragma unroll
            for (int k = D - 1; k >= 0; --k) {  // backward, U
                if (lane == k) y = y / p[k];
                const double xk = __shfl_sync(kFull, y, k);
                if (lane < k) y = fma(-p[k], xk, y);
            }
            __syncwarp();
            s.vec[lane] = y;
            __syncwarp();
            double d = 0.0;  // d = G y (matvec, matrix.hpp:146-156)
#pragma unroll
            for (int m = 0; m < D / 2; ++m) {
                const double2 gv = *reinterpret_cast<const double2*>(&s.G[lane * LD + 2 * m]);
                const double2 yv = *reinterpret_cast<const double2*>(&s.vec[2 * m]);
                d = fma(gv.x, yv.x, d);
                d = fma(gv.y, yv.y, d);
            }
            x += d;
            __syncwarp();
            s.vec[lane] = x;
            __syncwarp();
            double ax = 0.0;
#pragma unroll
            for (int m = 0; m < D / 2; ++m) {
                const double2 av = *reinterpret_cast<const double2*>(&s.A[lane * LD + 2 * m]);
                const double2 xv = *reinterpret_cast<const double2*>(&s.vec[2 * m]);
                ax = fma(av.x, xv.x, ax);
                ax = fma(av.y, xv.y, ax);
            }
            rl_ = bl - ax;
            rel = sqrt(warp_sum(rl_ * rl_)) / bnorm;
            __syncwarp();
        }

        // ---- outputs
        const double nan = __longlong_as_double(0x7ff8000000000000ll);
        if (gLU) {
#pragma unroll
            for (int m = 0; m < D / 2; ++m)
                *reinterpret_cast<double2*>(&s.P[lane * LD + 2 * m]) = make_double2(p[2 * m], p[2 * m + 1]);
            __syncwarp();
            store_matrix(gLU + mo, s.P, lane);
        }
        gX[sys * D + lane] = zero_step ? nan : x;
        if (lane == 0) {
            if (gR) gR[sys] = zero_step ? nan : rel;
            if (gGrowth) gGrowth[sys] = zero_step ? nan : umax / max_p;
            if (gStatus) gStatus[sys] = zero_step;
        }
        __syncwarp();
    }
}

struct SummaryAccum {
    double max_growth, max_resid, sum_resid;
    long long zero_pivots, counted;
};

// deterministic single-block reduction of the per-system outputs
__global__ void batch_summary_kernel(const double* __restrict__ r, const double* __restrict__ g,
                                     const int32_t* __restrict__ st, int64_t batch, SummaryAccum* out) {
    __shared__ double sm[3][32];
    __shared__ long long sc[2][32];
    double mg = 0.0, mr = 0.0, sr = 0.0;
    long long zp = 0, cnt = 0;
    for (int64_t i = threadIdx.x; i < batch; i += blockDim.x) {
        if (st[i] != 0) {
            ++zp;
            continue;
        }
        mg = fmax(mg, g[i]);
        mr = fmax(mr, r[i]);
        sr += r[i];
        ++cnt;
    }
    mg = warp_max(mg);
    mr = warp_max(mr);
    sr = warp_sum(sr);
    for (int o = 16; o > 0; o >>= 1) {
        zp += __shfl_xor_sync(kFull, zp, o);
        cnt += __shfl_xor_sync(kFull, cnt, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sm[0][w] = mg;
        sm[1][w] = mr;
        sm[2][w] = sr;
        sc[0][w] = zp;
        sc[1][w] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        SummaryAccum a{0, 0, 0, 0, 0};
        for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) {
            a.max_growth = fmax(a.max_growth, sm[0][i]);
            a.max_resid = fmax(a.max_resid, sm[1][i]);
            a.sum_resid += sm[2][i];
            a.zero_pivots += sc[0][i];
            a.counted += sc[1][i];
        }
        *out = a;
    }
}

}  // namespace

rl_status launch_batched_genp32(rl_context* ctx, int64_t batch, const double* a, const double* g, const double* b,
                                double* lu, double* x, double* r, double* growth, int32_t* status, int refine) {
    static bool configured = false;
    if (!configured) {
        RL_CUDA(cudaFuncSetAttribute(batched_genp32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kSmemBytes)));
        configured = true;
    }
    if (batch == 0) return RL_OK;
    const int64_t ctas_needed = (batch + WARPS - 1) / WARPS;
    const int64_t grid = std::min<int64_t>(ctas_needed, static_cast<int64_t>(ctx->num_sms) * 2);
    batched_genp32_kernel<<<static_cast<unsigned>(grid), WARPS * 32, kSmemBytes, ctx->stream>>>(
        a, g, b, lu, x, r, growth, status, batch, refine);
    RL_CHECK_LAUNCH("batched_genp32_kernel");
    return RL_OK;
}

}  // namespace rl

extern "C" RL_API rl_status rl_batched_genp_solve_32(rl_context* ctx, rl_mem mem, int64_t batch, const double* a,
                                                     const double* g, const double* b, double* lu, double* x,
                                                     double* resid, double* growth, int32_t* status,
                                                     rl_batch_summary* summary) {
    using namespace rl;
    if (batch < 0) return set_error(RL_ERR_DIMENSION, "rl_batched_genp_solve_32: negative batch");
    if (batch > 0 && (!a || !g || !b || !x))
        return set_error(RL_ERR_INVALID_ARGUMENT, "rl_batched_genp_solve_32: a, g, b, x are required");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    if (batch == 0) {
        if (summary) *summary = rl_batch_summary{0, 0, 0.0, 0.0, 0.0};
        return RL_OK;
    }
    const size_t mb = static_cast<size_t>(batch) * 32 * 32, vb = static_cast<size_t>(batch) * 32;
    const double *da = a, *dg = g, *db = b;
    double *dlu = lu, *dx = x, *dr = resid, *dgr = growth;
    int32_t* dst = status;
    SummaryAccum* dsum = nullptr;
    const bool host = mem == RL_HOST;
    const bool need_status = host ? (status != nullptr || summary != nullptr) : (status != nullptr);
    bool ok = with_arena(ctx, [&](Arena& ar) {
        if (host) {
            da = ar.take<double>(mb);
            dg = ar.take<double>(mb);
            db = ar.take<double>(vb);
            dlu = lu ? ar.take<double>(mb) : nullptr;
            dx = ar.take<double>(vb);
            dr = (resid || summary) ? ar.take<double>(batch) : nullptr;
            dgr = (growth || summary) ? ar.take<double>(batch) : nullptr;
            dst = need_status ? ar.take<int32_t>(batch) : nullptr;
        } else if (summary) {
            if (!dr) dr = ar.take<double>(batch);
            if (!dgr) dgr = ar.take<double>(batch);
            if (!dst) dst = ar.take<int32_t>(batch);
        }
        if (summary) dsum = ar.take<SummaryAccum>(1);
    });
    if (!ok) return RL_ERR_OUT_OF_MEMORY;
    cudaStream_t s = ctx->stream;
    if (host) {
        RL_CUDA(cudaMemcpyAsync(const_cast<double*>(da), a, mb * 8, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaMemcpyAsync(const_cast<double*>(dg), g, mb * 8, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaMemcpyAsync(const_cast<double*>(db), b, vb * 8, cudaMemcpyHostToDevice, s));
    }
    st = launch_batched_genp32(ctx, batch, da, dg, db, dlu, dx, dr, dgr, dst, 0);
    if (st != RL_OK) return st;
    SummaryAccum hsum{};
    if (summary) {
        batch_summary_kernel<<<1, 1024, 0, s>>>(dr, dgr, dst, batch, dsum);
        RL_CHECK_LAUNCH("batch_summary_kernel");
        RL_CUDA(cudaMemcpyAsync(&hsum, dsum, sizeof(hsum), cudaMemcpyDeviceToHost, s));
    }
    if (host) {
        if (lu) RL_CUDA(cudaMemcpyAsync(lu, dlu, mb * 8, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaMemcpyAsync(x, dx, vb * 8, cudaMemcpyDeviceToHost, s));
        if (resid) RL_CUDA(cudaMemcpyAsync(resid, dr, batch * 8, cudaMemcpyDeviceToHost, s));
        if (growth) RL_CUDA(cudaMemcpyAsync(growth, dgr, batch * 8, cudaMemcpyDeviceToHost, s));
        if (status) RL_CUDA(cudaMemcpyAsync(status, dst, batch * 4, cudaMemcpyDeviceToHost, s));
    }
    if (host || summary) RL_CUDA(cudaStreamSynchronize(s));
    if (summary) {
        summary->zero_pivots = hsum.zero_pivots;
        summary->norm_estimates = -1;  // not tracked per batch
        summary->max_growth = hsum.max_growth;
        summary->max_residual = hsum.max_resid;
        summary->mean_residual = hsum.counted ? hsum.sum_resid / static_cast<double>(hsum.counted) : 0.0;
    }
    return RL_OK;
}
