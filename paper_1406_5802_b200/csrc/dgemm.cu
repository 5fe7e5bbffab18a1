// FP64 GEMM for sm_100a: C = alpha * A B (+ C), row-major.
//
// Replaces matmul (matrix.hpp:115-121, Eigen) on the hot path: the A*G
// preprocessing product (preprocess.hpp:65-73), the trailing Schur updates of
// blocked GENP, and the low-rank products A*H, Q^T A, Q (Q^T A)
// (lowrank.hpp:35-37, :80).
//
// tcgen05.mma has no f64 kind on sm_100a; the FP64 tensor path is DMMA
// (mma.sync .f64, SASS DMMA.8x8x4), measured at 37.0 TF/s on this B200
// against 36.4 for DFMA and 35.5 for cuBLAS DGEMM (profiles/r01_fp64_peak.txt).
//
// Tiling: 128x64 CTA tiles, k-slabs of 16, 8 warps of 32x32, two CTAs per SM
// (the C prologue / epilogue of one overlaps the other's main loop); a
// 128x128 one-CTA tile for the split-K partial products. Operands arrive by TMA
// (cp.async.bulk.tensor.2d, 128-byte swizzle) into a 4-stage shared-memory
// ring guarded by mbarriers; one thread issues the copies. CTAs are rastered
// in groups of 8 tile-rows so concurrently resident CTAs share A and B panels
// in L2. The epilogue optionally accumulates into C (Schur update) and folds
// ||C||_F^2 / max|C| into device statistics (pivot-tolerance bound, growth).
#include <algorithm>
#include <mutex>

#include "device_common.cuh"
#include "kernels.cuh"
#include "tma.cuh"

namespace rl {
namespace {

constexpr int BK = 16, GROUP_M = 8;

// Tile configurations. Big: 128x128 CTA tile, 8 warps of 64x32, one CTA per
// SM (long-K products such as A*G). Small: 128x64 tile, 8 warps of 32x32,
// two CTAs per SM so one CTA's epilogue (C read-modify-write) overlaps the
// other's MMA main loop — the short-K Schur updates of blocked GENP.
template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int MINB_>
struct Cfg {
    static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
    static constexpr int MI = BM / WM / 8, NJ = BN / WN / 8;  // 8x8 fragments per warp
    static constexpr int A_STAGE = BM * BK * 8, B_STAGE = BK * BN * 8;
    static constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
    static constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 128;
    static constexpr int THREADS = WM * WN * 32;
};
using BigCfg = Cfg<128, 128, 2, 4, 4, 1>;
using SmallCfg = Cfg<128, 64, 4, 2, 4, 2>;
// latency-bound small products (the GENP tail's U12, GEMM_a and panel
// updates): 64x32 tiles, 4 warps of 32x16, four CTAs per SM, so a problem of a
// few 128x64 tiles still spreads over the SMs
using TinyCfg = Cfg<64, 32, 2, 2, 4, 4>;
// one tile row of up to 128 rows, 32-column tiles: for products computed in
// place over their B operand (U12 = L11^-1 A12 overwriting A12), where every
// CTA must read all rows of its column block before any CTA stores into them
#ifndef RL_COLCFG
#define RL_COLCFG 128, 16, 8, 1, 4, 2
#endif
using ColCfg = Cfg<RL_COLCFG>;

// element (r, k) of a 128-byte-swizzled tile with 16 doubles per row
__device__ __forceinline__ int swz128(int r, int k) { return r * 128 + ((((k >> 1) ^ (r & 7))) << 4) + ((k & 1) << 3); }

// kAccum: accumulators start from C (C +- A B); kStats: fold ||.||_F^2 / max|.|
// of the result into *stats; kStore = false: statistics only (e.g. the
// low-rank residual A - Q (Q^T A) is never materialised). Split-K: blockIdx.y
// takes k-tiles [y*ktc, (y+1)*ktc) and writes its partial at C + y*split_stride.
template <class CF, bool kAccum, bool kStats, bool kStore>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB)
dgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, double* __restrict__ C,
             int64_t ldc, int M, int N, int K, double alpha, GemmStats* __restrict__ stats, int ktc,
             int64_t split_stride, int c_ahead) {
    constexpr int BM = CF::BM, BN = CF::BN, STAGES = CF::STAGES, MI = CF::MI, NJ = CF::NJ;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the 128B swizzle, keeping the pointer in the
    // shared window so operand reads compile to LDS (not generic LD)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CF::STAGE_BYTES);
    uint64_t* empty = full + STAGES;  // stage drained by every MMA warp

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp / CF::WN, wn = warp % CF::WN;
    const int fr = lane >> 2, fc = lane & 3;
    const int rbase = wm * (MI * 8), cbase = wn * (NJ * 8);

    // grouped raster over (tiles_m x tiles_n)
    const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
    const int t = blockIdx.x;
    const int group = t / (GROUP_M * tiles_n);
    const int first_m = group * GROUP_M;
    const int gsize = min(tiles_m - first_m, GROUP_M);
    const int tm_ = first_m + (t % (GROUP_M * tiles_n)) % gsize;
    const int tn_ = (t % (GROUP_M * tiles_n)) / gsize;
    const int m0 = tm_ * BM, n0 = tn_ * BN;
    const int KT_all = (K + BK - 1) / BK;
    const int kt0 = ktc > 0 ? static_cast<int>(blockIdx.y) * ktc : 0;
    const int KT = ktc > 0 ? min(ktc, KT_all - kt0) : KT_all;
    C += static_cast<int64_t>(blockIdx.y) * split_stride;

    constexpr int MMA_WARPS = CF::THREADS / 32;
    if (tid == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], MMA_WARPS);
        }
        mbar_fence_init();
    }
    __syncthreads();
    // everything above touches no data of the previous kernel
    griddep_wait();
    griddep_launch_dependents();

    auto issue = [&](int kt) {
        const int s = kt % STAGES;
        unsigned char* st = smem + s * CF::STAGE_BYTES;
        mbar_expect_tx(&full[s], CF::STAGE_BYTES);
        tma_load_2d(st, &tmA, (kt0 + kt) * BK, m0, &full[s]);
#pragma unroll
        for (int j = 0; j < BN / 16; ++j)
            tma_load_2d(st + CF::A_STAGE + j * 2048, &tmB, n0 + 16 * j, (kt0 + kt) * BK, &full[s]);
    };
    if (tid == 0)
        for (int kt = 0; kt < min(STAGES, KT); ++kt) issue(kt);

    // accumulators: 0, or (kAccum) the current C tile, fetched with all loads
    // in flight at once while the first TMA stages land; alpha = -1 is then
    // applied by negating the A fragments (C - A B, the Schur update)
    double acc[MI][NJ][2];
    const bool vec_ok = ((ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (kAccum) {
#pragma unroll
        for (int i = 0; i < MI; ++i) {
            const int row = m0 + rbase + 8 * i + fr;
            if (row >= M) continue;
            const double* crow = C + static_cast<int64_t>(row) * ldc;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int col = n0 + cbase + 8 * j + 2 * fc;
                if (vec_ok && col + 1 < N) {
                    const double2 o = *reinterpret_cast<const double2*>(crow + col);
                    acc[i][j][0] = o.x;
                    acc[i][j][1] = o.y;
                } else {
                    if (col < N) acc[i][j][0] = crow[col];
                    if (col + 1 < N) acc[i][j][1] = crow[col + 1];
                }
            }
        }
    }
    // alpha = -1: flip the sign bit of the A fragments (an integer op, exact)
    const int sign_hi = kAccum && alpha < 0.0 ? static_cast<int>(0x80000000u) : 0;
    // the C tile of the tile one resident wave ahead into L2, so that its
    // up-front C read (above) hits L2 instead of drawing on HBM in a burst
    // with every other tile of its wave
    if (kAccum && c_ahead > 0 && ktc == 0) {
        const int ta = t + c_ahead;
        if (ta < tiles_m * tiles_n && tid < BM) {
            const int ga = ta / (GROUP_M * tiles_n), fa = ga * GROUP_M, sa = min(tiles_m - fa, GROUP_M);
            const int ma = (fa + (ta % (GROUP_M * tiles_n)) % sa) * BM, na = ((ta % (GROUP_M * tiles_n)) / sa) * BN;
            const int row = ma + tid;
            const int cols = min(BN, N - na);
            if (row < M && cols > 0 && vec_ok) {
                const double* p = C + static_cast<int64_t>(row) * ldc + na;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(static_cast<unsigned>(cols * 8) & ~15u));
            }
        }
    }

    for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        mbar_wait(&full[s], (kt / STAGES) & 1);
        const unsigned char* sa = smem + s * CF::STAGE_BYTES;
        const unsigned char* sb = sa + CF::A_STAGE;
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk) {
            const int k = 4 * kk + fc;
            double af[MI], bf[NJ];
#pragma unroll
            for (int i = 0; i < MI; ++i)
                af[i] = __hiloint2double(
                    __double2hiint(*reinterpret_cast<const double*>(sa + swz128(rbase + 8 * i + fr, k))) ^ sign_hi,
                    __double2loint(*reinterpret_cast<const double*>(sa + swz128(rbase + 8 * i + fr, k))));
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int n = cbase + 8 * j + fr;
                bf[j] = *reinterpret_cast<const double*>(sb + (n >> 4) * 2048 + swz128(k, n & 15));
            }
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        // release the stage; thread 0 refills it once every warp has (the
        // other warps run ahead on the stages already landed, no CTA barrier)
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (tid == 0 && kt + STAGES < KT) {
            mbar_wait(&empty[s], (kt / STAGES) & 1);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(kt + STAGES);
        }
        __syncwarp();  // warp 0 reconverges before its next mma.sync (.aligned)
    }

    // ---- epilogue
    double ssq = 0.0, amax = 0.0;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
        const int row = m0 + rbase + 8 * i + fr;
        if (row >= M) continue;
        double* crow = C + static_cast<int64_t>(row) * ldc;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int col = n0 + cbase + 8 * j + 2 * fc;
            const double v0 = kAccum ? acc[i][j][0] : alpha * acc[i][j][0];
            const double v1 = kAccum ? acc[i][j][1] : alpha * acc[i][j][1];
            if (vec_ok && col + 1 < N) {
                if (kStore) *reinterpret_cast<double2*>(crow + col) = make_double2(v0, v1);
                if (kStats) {
                    ssq = fma(v0, v0, fma(v1, v1, ssq));
                    amax = fmax(amax, fmax(fabs(v0), fabs(v1)));
                }
            } else {
                if (col < N) {
                    if (kStore) crow[col] = v0;
                    if (kStats) {
                        ssq = fma(v0, v0, ssq);
                        amax = fmax(amax, fabs(v0));
                    }
                }
                if (col + 1 < N) {
                    if (kStore) crow[col + 1] = v1;
                    if (kStats) {
                        ssq = fma(v1, v1, ssq);
                        amax = fmax(amax, fabs(v1));
                    }
                }
            }
        }
    }
    if (kStats) {
        ssq = warp_sum(ssq);
        amax = warp_max(amax);
        if (lane == 0) {
            atomicAdd(&stats->sumsq, ssq);
            atomicMax(&stats->maxabs_bits, static_cast<unsigned long long>(__double_as_longlong(amax)));
        }
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

template <class CF, bool A, bool S, bool T>
void configure_once() {
    static PerDeviceOnce once;
    once_per_device(once, [] {
        return cudaFuncSetAttribute(dgemm_kernel<CF, A, S, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(CF::SMEM_BYTES)) == cudaSuccess
                   ? RL_OK
                   : RL_ERR_CUDA;  // a failure surfaces at the launch
    });
}

template <class CF, bool A, bool S, bool T>
void launch_cfg(dim3 grid, cudaStream_t st, const CUtensorMap& ta, const CUtensorMap& tb, double* C, int64_t ldc, int m,
                int n, int k, double alpha, GemmStats* stats, int ktc, int64_t split_stride, int c_ahead, bool pdl) {
    configure_once<CF, A, S, T>();
    if (pdl) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(CF::THREADS);
        cfg.dynamicSmemBytes = CF::SMEM_BYTES;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, dgemm_kernel<CF, A, S, T>, ta, tb, C, ldc, m, n, k, alpha, stats, ktc, split_stride,
                           c_ahead);
        return;
    }
    dgemm_kernel<CF, A, S, T><<<grid, CF::THREADS, CF::SMEM_BYTES, st>>>(ta, tb, C, ldc, m, n, k, alpha, stats, ktc,
                                                                       split_stride, c_ahead);
}

// encode the operand maps for configuration CF and launch over all tiles
template <class CF, bool A, bool S, bool T>
rl_status run_cfg(rl_context* ctx, int64_t M, int64_t N, int64_t K, const double* Ap, int64_t lda, const double* Bp,
                  int64_t ldb, double* C, int64_t ldc, double alpha, GemmStats* stats, int splits, int ktc,
                  int64_t split_stride) {
    CUtensorMap ta, tb;
    if (!make_tmap_2d(&ta, Ap, M, K, lda, CF::BM, BK, true) || !make_tmap_2d(&tb, Bp, K, N, ldb, BK, 16, true))
        return set_error(RL_ERR_CUDA, "gemm: cuTensorMapEncodeTiled failed");
    const int64_t tiles = ((M + CF::BM - 1) / CF::BM) * ((N + CF::BN - 1) / CF::BN);
    if (tiles > 0x7fffffff) return set_error(RL_ERR_DIMENSION, "gemm: too many tiles");
    launch_cfg<CF, A, S, T>(dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(splits)), ctx->stream, ta, tb, C,
                            ldc, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), alpha, stats, ktc,
                            split_stride, A ? ctx->num_sms * CF::MINB : 0, ctx->pdl);
    RL_CHECK_LAUNCH("dgemm_kernel");
    return RL_OK;
}

__global__ void reduce_splits_kernel(const double* __restrict__ part, int splits, int64_t slab, int64_t M, int64_t N,
                                     int64_t ldp, double* __restrict__ C, int64_t ldc, bool accumulate, double alpha) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= M * N) return;
    const int64_t i = idx / N, j = idx % N;
    double s = 0.0;
    for (int q = 0; q < splits; ++q) s += part[q * slab + i * ldp + j];
    C[i * ldc + j] = accumulate ? C[i * ldc + j] + alpha * s : alpha * s;
}

}  // namespace

bool make_tmap_2d(CUtensorMap* out, const double* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_rows,
                  uint32_t box_cols, bool swizzle128) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

rl_status gemm(rl_context* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
               int64_t ldb, double* C, int64_t ldc, double alpha, bool accumulate, GemmStats* stats) {
    if (M <= 0 || N <= 0) return RL_OK;
    if (K <= 0) {
        if (!accumulate)
            for (int64_t r = 0; r < M; ++r) RL_CUDA(cudaMemsetAsync(C + r * ldc, 0, N * 8, ctx->stream));
        return RL_OK;
    }
    if ((lda & 1) || (ldb & 1) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
        return set_error(RL_ERR_INVALID_ARGUMENT, "gemm: TMA needs 16-byte aligned operands with even leading dimensions");
    if (accumulate && alpha != 1.0 && alpha != -1.0)
        return set_error(RL_ERR_INVALID_ARGUMENT, "gemm: accumulate supports alpha = +1 or -1");
    if (M > (int64_t(1) << 30) || N > (int64_t(1) << 30) || K > (int64_t(1) << 30))
        return set_error(RL_ERR_DIMENSION, "gemm: dimension too large");
    // the two-CTAs-per-SM 128x64 configuration: one CTA's prologue / epilogue
    // (the C tile) overlaps the other's MMA main loop. Measured on this pool
    // (tools/gemm_update_bench.cu): 35.5 TF/s at 8192^3 against 34.2 for the
    // one-CTA 128x128 tile, and 32.2 against 27.3 for the K = 128 Schur update.
    // Problems that would not fill the SMs with it: 64x32 tiles.
    const bool small = true;
    const int64_t small_tiles = ((M + 127) / 128) * ((N + 63) / 64);
    const bool tiny = small_tiles < ctx->num_sms;
#define RL_GEMM_DISPATCH(AC, ST)                                                                                   \
    return tiny    ? run_cfg<TinyCfg, AC, ST, true>(ctx, M, N, K, A, lda, B, ldb, C, ldc, alpha, stats, 1, 0, 0)  \
           : small ? run_cfg<SmallCfg, AC, ST, true>(ctx, M, N, K, A, lda, B, ldb, C, ldc, alpha, stats, 1, 0, 0) \
                   : run_cfg<BigCfg, AC, ST, true>(ctx, M, N, K, A, lda, B, ldb, C, ldc, alpha, stats, 1, 0, 0)
    if (accumulate) {
        if (stats) RL_GEMM_DISPATCH(true, true);
        RL_GEMM_DISPATCH(true, false);
    }
    if (stats) RL_GEMM_DISPATCH(false, true);
    RL_GEMM_DISPATCH(false, false);
#undef RL_GEMM_DISPATCH
}

rl_status gemm_inplace_b(rl_context* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, double* BC,
                         int64_t ldb) {
    if (M <= 0 || N <= 0) return RL_OK;
    if (M > 128 || K != M)
        return set_error(RL_ERR_INVALID_ARGUMENT, "gemm_inplace_b: one tile row of at most 128 rows (K = M)");
    if ((lda & 1) || (ldb & 1) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(BC) & 15))
        return set_error(RL_ERR_INVALID_ARGUMENT, "gemm_inplace_b: TMA needs 16-byte aligned operands with even leading dimensions");
    const bool tiny = (N + 63) / 64 < ctx->num_sms;  // ColCfg.BM = 128 too
    return tiny ? run_cfg<ColCfg, false, false, true>(ctx, M, N, K, A, lda, BC, ldb, BC, ldb, 1.0, nullptr, 1, 0, 0)
                : run_cfg<SmallCfg, false, false, true>(ctx, M, N, K, A, lda, BC, ldb, BC, ldb, 1.0, nullptr, 1, 0, 0);
}

rl_status gemm_residual_stats(rl_context* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                              const double* B, int64_t ldb, const double* C, int64_t ldc, GemmStats* stats) {
    if (M <= 0 || N <= 0) return RL_OK;
    if ((lda & 1) || (ldb & 1) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
        return set_error(RL_ERR_INVALID_ARGUMENT, "gemm_residual_stats: misaligned operands");
    const bool small = true;  // as gemm(): the two-CTAs-per-SM tile wins at every K measured
    return small ? run_cfg<SmallCfg, true, true, false>(ctx, M, N, K, A, lda, B, ldb, const_cast<double*>(C), ldc, -1.0,
                                                        stats, 1, 0, 0)
                 : run_cfg<BigCfg, true, true, false>(ctx, M, N, K, A, lda, B, ldb, const_cast<double*>(C), ldc, -1.0,
                                                      stats, 1, 0, 0);
}

size_t gemm_splitk_work_bytes(int64_t M, int64_t N, int splits) {
    return static_cast<size_t>(splits) * static_cast<size_t>(M) * static_cast<size_t>((N + 1) & ~int64_t(1)) * 8 + 256;
}

rl_status gemm_splitk(rl_context* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                      int64_t ldb, double* C, int64_t ldc, double alpha, bool accumulate, int splits, void* work) {
    if (M <= 0 || N <= 0) return RL_OK;
    const int KT = static_cast<int>((K + BK - 1) / BK);
    splits = std::max(1, std::min(splits, KT));
    if (splits == 1) return gemm(ctx, M, N, K, A, lda, B, ldb, C, ldc, alpha, accumulate, nullptr);
    if ((lda & 1) || (ldb & 1) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
        return set_error(RL_ERR_INVALID_ARGUMENT, "gemm_splitk: misaligned operands");
    const int ktc = (KT + splits - 1) / splits;
    splits = (KT + ktc - 1) / ktc;
    const int64_t ldp = (N + 1) & ~int64_t(1);
    const int64_t slab = M * ldp;
    double* part = static_cast<double*>(work);
    // skinny products (the range finder's A H with r <= 64 columns, Q^T A with
    // r <= 64 rows): a tile that does not overhang the short side
#ifndef RL_SPLITK_SKINNY
#define RL_SPLITK_SKINNY 1
#endif
    rl_status st;
    if (RL_SPLITK_SKINNY && N <= 64 && M > 64)
        st = run_cfg<SmallCfg, false, false, true>(ctx, M, N, K, A, lda, B, ldb, part, ldp, 1.0, nullptr, splits, ktc,
                                                   slab);
    else if (RL_SPLITK_SKINNY && M <= 64)
        st = run_cfg<TinyCfg, false, false, true>(ctx, M, N, K, A, lda, B, ldb, part, ldp, 1.0, nullptr, splits, ktc,
                                                  slab);
    else
        st = run_cfg<BigCfg, false, false, true>(ctx, M, N, K, A, lda, B, ldb, part, ldp, 1.0, nullptr, splits, ktc,
                                                 slab);
    if (st != RL_OK) return st;
    reduce_splits_kernel<<<static_cast<unsigned>((M * N + 255) / 256), 256, 0, ctx->stream>>>(
        part, splits, slab, M, N, ldp, C, ldc, accumulate, alpha);
    RL_CHECK_LAUNCH("reduce_splits_kernel");
    return RL_OK;
}

}  // namespace rl

// ---- C ABI: rl_dgemm (matmul, matrix.hpp:115-121) ---------------------------
extern "C" RL_API rl_status rl_dgemm(rl_context* ctx, rl_mem mem, int64_t m, int64_t n, int64_t k, const double* a,
                                     int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc) {
    using namespace rl;
    if (m <= 0 || n <= 0 || k <= 0) return set_error(RL_ERR_DIMENSION, "rl_dgemm: matrix dimensions must be positive");
    if (lda < k || ldb < n || ldc < n) return set_error(RL_ERR_DIMENSION, "rl_dgemm: leading dimension too small");
    if (!a || !b || !c) return set_error(RL_ERR_INVALID_ARGUMENT, "rl_dgemm: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    const bool host = mem == RL_HOST;
    const bool repack_a = host || (lda & 1) || (reinterpret_cast<uintptr_t>(a) & 15);
    const bool repack_b = host || (ldb & 1) || (reinterpret_cast<uintptr_t>(b) & 15);
    const int64_t la = (k + 1) & ~int64_t(1), lb = (n + 1) & ~int64_t(1);
    double *da = const_cast<double*>(a), *db = const_cast<double*>(b), *dc = c;
    int64_t lda2 = lda, ldb2 = ldb, ldc2 = ldc;
    bool ok = with_arena(ctx, [&](Arena& ar) {
        if (repack_a) da = ar.take<double>(m * la);
        if (repack_b) db = ar.take<double>(k * lb);
        if (host) dc = ar.take<double>(m * n);
    });
    if (!ok) return RL_ERR_OUT_OF_MEMORY;
    cudaStream_t s = ctx->stream;
    const cudaMemcpyKind ka = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    if (repack_a) {
        RL_CUDA(cudaMemcpy2DAsync(da, la * 8, a, lda * 8, k * 8, m, ka, s));
        lda2 = la;
    }
    if (repack_b) {
        RL_CUDA(cudaMemcpy2DAsync(db, lb * 8, b, ldb * 8, n * 8, k, ka, s));
        ldb2 = lb;
    }
    if (host) ldc2 = n;
    st = gemm(ctx, m, n, k, da, lda2, db, ldb2, dc, ldc2, 1.0, false, nullptr);
    if (st != RL_OK) return st;
    if (host) {
        RL_CUDA(cudaMemcpy2DAsync(c, ldc * 8, dc, n * 8, n * 8, m, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaStreamSynchronize(s));
    }
    return RL_OK;
}
