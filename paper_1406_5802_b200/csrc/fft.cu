// Circulant / Toeplitz right products by FFT for sm_100a.
//
//   rl_circulant_right_multiply  matmul_by_circulant(A, C(c))      circulant.hpp:171-185
//   rl_toeplitz_right_multiply   matmul_by_toeplitz_block(A, T)    circulant.hpp:187-203
//
// Row i of A C is C^T a_i = Omega^-1 (s .* Omega a_i) with s the spectrum of
// the transposed circulant's first column c_T[i] = c[(n-i) mod n]
// (circulant.hpp:40-45, :70-76). The circulant is real, so two real rows
// travel as one complex row z = a_i + i a_{i+1}; Re/Im of the result are the
// two output rows (imaginary dust is therefore identically zero and the
// reference's strip_imag verdict, circulant.hpp:57-68, can never fire — for
// real inputs it does not fire in the reference either).
//
// One CTA per row pair, the row resident in shared memory (n <= 8192 complex
// = 128 KiB). Forward transform: in-place decimation-in-frequency radix-16
// passes (+ one radix-2/4/8 pass for the remainder) that leave the spectrum
// in digit-reversed order; the multiplier spectrum s is produced by the SAME
// forward transform, so it is in the same order and the pointwise product
// needs no reordering; the inverse is the transposed (decimation-in-time)
// sequence of passes with conjugate twiddles, which consumes the permuted
// spectrum and returns natural order. Twiddles w_n^k = exp(+2 pi i k / n)
// (the reference's sign, fft.hpp:11-12) come from a sincospi table in L2.
// Parent length 16384 (BASELINE config 5) runs on a 2-CTA cluster: the
// first radix-2 DIF pass splits the row into two independent 8192-point
// halves, one per CTA (both read the row, the second read hits L2); the
// last inverse radix-2 pass is combined through distributed shared memory for
// the l output columns the Toeplitz block keeps.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "device_common.cuh"
#include "kernels.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace rl {
namespace {

constexpr int FT = 256;          // threads per CTA (255 registers: radix-16 groups stay in registers)
constexpr int MAXN = 8192;       // complex points per CTA

struct cplx {
    double x, y;
};
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return {fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)}; }
__device__ __forceinline__ cplx cmulc(cplx a, cplx b) {  // a * conj(b)
    return {fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y)};
}
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return {a.x - b.x, a.y - b.y}; }

__global__ void twiddle_kernel(int64_t n, cplx* __restrict__ tw) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double s, c;
    sincospi(2.0 * static_cast<double>(k) / static_cast<double>(n), &s, &c);
    tw[k] = {c, s};
}

// w_R^j = exp(+2 pi i j / R) for R <= 16 as exact double literals (the
// in-register butterflies then fold multiplications by 0, +-1)
__device__ __forceinline__ cplx wconst(int R, int j) {
    constexpr double c1 = 0.92387953251128674;  // cos(pi/8)
    constexpr double s1 = 0.38268343236508977;  // sin(pi/8)
    constexpr double h = 0.70710678118654757;   // sqrt(1/2)
    const int k = (j * 16 / R) & 15;            // as a power of w_16
    switch (k) {
        case 0: return {1.0, 0.0};
        case 1: return {c1, s1};
        case 2: return {h, h};
        case 3: return {s1, c1};
        case 4: return {0.0, 1.0};
        case 5: return {-s1, c1};
        case 6: return {-h, h};
        case 7: return {-c1, s1};
        case 8: return {-1.0, 0.0};
        case 9: return {-c1, -s1};
        case 10: return {-h, -h};
        case 11: return {-s1, -c1};
        case 12: return {0.0, -1.0};
        case 13: return {s1, -c1};
        case 14: return {h, -h};
        default: return {c1, -s1};
    }
}

// in-register R-point DFT (R <= 16), forward (w = e^{+2 pi i/R}) or inverse
// (conjugate); natural-order input, output r lands in v[brev<R>(r)]
template <int R, bool kInv>
__device__ __forceinline__ void dft_reg(cplx (&v)[R]) {
    // iterative radix-2 DIF in registers (output bit-reversed)
#pragma unroll
    for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
        for (int base = 0; base < R; base += 2 * half) {
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const cplx a = v[base + j], b = v[base + j + half];
                const cplx d = csub(a, b);
                v[base + j] = cadd(a, b);
                if (j == 0) {
                    v[base + j + half] = d;
                } else if (j * 2 == half) {  // w = i: a swap and a sign (the FMA form would not fold the 0 and 1)
                    v[base + j + half] = kInv ? cplx{d.y, -d.x} : cplx{-d.y, d.x};
                } else {
                    const cplx w = wconst(2 * half, j);  // w_{2 half}^j
                    v[base + j + half] = kInv ? cmulc(d, w) : cmul(d, w);
                }
            }
        }
    }
}

// position of natural-order output r after dft_reg (bit reversal within R)
template <int R>
__host__ __device__ constexpr int brev(int r) {
    int o = 0;
    for (int b = 1, ib = R / 2; b < R; b <<= 1, ib >>= 1)
        if (r & b) o |= ib;
    return o;
}

// twiddles w_N^{n0 r}, r = 1..R-1, from four table loads (r = 1, 2, 4, 8)
// and at most three products (|error| <= ~3 ulp)
template <int R>
__device__ __forceinline__ void pass_twiddles(cplx (&w)[R], const cplx* __restrict__ tw, int64_t base, int64_t mask) {
    w[0] = {1.0, 0.0};
    if (R > 1) w[1] = tw[base & mask];
    if (R > 2) w[2] = tw[(2 * base) & mask];
    if (R > 4) w[4] = tw[(4 * base) & mask];
    if (R > 8) w[8] = tw[(8 * base) & mask];
#pragma unroll
    for (int r = 3; r < R; ++r) {
        if (r == 4 || r == 8) continue;
        const int hi = r >= 8 ? 8 : (r >= 4 ? 4 : 2);
        w[r] = cmul(w[hi], w[r - hi]);
    }
}

// the same twiddles formed lazily: base_twiddles loads r = 1, 2, 4, 8 and
// lazy_twiddle(w, r) forms w[r] = w[hi] w[r - hi] just before its first use
// (the products of pass_twiddles, in the same order), so the fifteen values
// are not all live at once
template <int R>
__device__ __forceinline__ void base_twiddles(cplx (&w)[R], const cplx* __restrict__ tw, int64_t base, int64_t mask) {
    if (R > 1) w[1] = tw[base & mask];
    if (R > 2) w[2] = tw[(2 * base) & mask];
    if (R > 4) w[4] = tw[(4 * base) & mask];
    if (R > 8) w[8] = tw[(8 * base) & mask];
}
template <int R>
__device__ __forceinline__ void lazy_twiddle(cplx (&w)[R], int r) {
    if (r >= 3 && r != 4 && r != 8) {
        const int hi = r >= 8 ? 8 : (r >= 4 ? 4 : 2);
        w[r] = cmul(w[hi], w[r - hi]);
    }
}

// one forward DIF pass on the full buffer: subarrays of length N, radix R
template <int R>
__device__ __forceinline__ void dif_pass(cplx* z, int n, int N, const cplx* __restrict__ tw, int ntw) {
    const int M = N / R;
    const int lgM = 31 - __clz(M);
    const int groups = n / R;
    const int64_t tstride = ntw / N;  // w_N^k = tw[k * ntw / N]
    const int64_t mask = ntw - 1;
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
        const int n0 = g & (M - 1), o = (g >> lgM) * N;
        cplx v[R];
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = z[(o + n0 + j * M)];
        dft_reg<R, false>(v);
        cplx w[R];
        pass_twiddles<R>(w, tw, static_cast<int64_t>(n0) * tstride, mask);
        z[(o + n0)] = v[0];
#pragma unroll
        for (int r = 1; r < R; ++r) z[(o + n0 + r * M)] = cmul(v[brev<R>(r)], w[r]);
    }
}

// transposed (DIT) pass with conjugate twiddles; `scale` folded into outputs
template <int R>
__device__ __forceinline__ void dit_pass(cplx* z, int n, int N, const cplx* __restrict__ tw, int ntw, double scale) {
    const int M = N / R;
    const int lgM = 31 - __clz(M);
    const int groups = n / R;
    const int64_t tstride = ntw / N;
    const int64_t mask = ntw - 1;
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
        const int n0 = g & (M - 1), o = (g >> lgM) * N;
        cplx w[R];
        pass_twiddles<R>(w, tw, static_cast<int64_t>(n0) * tstride, mask);
        cplx v[R];
        v[0] = z[(o + n0)];
#pragma unroll
        for (int r = 1; r < R; ++r) v[r] = cmulc(z[(o + n0 + r * M)], w[r]);
        dft_reg<R, true>(v);
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const cplx t = v[brev<R>(j)];
            z[(o + n0 + j * M)] = {t.x * scale, t.y * scale};
        }
    }
}

// pass plan for n = 2^L: radix-16 passes, then one radix 2/4/8 remainder pass
__device__ __forceinline__ int plan(int n, int* radix) {
    int L = 31 - __clz(n), p = 0;
    while (L >= 4) {
        radix[p++] = 16;
        L -= 4;
    }
    if (L > 0) radix[p++] = 1 << L;
    return p;
}

__device__ void forward_fft(cplx* z, int n, const cplx* tw, int ntw) {
    int radix[8];
    const int passes = plan(n, radix);
    int N = n;
    for (int p = 0; p < passes; ++p) {
        switch (radix[p]) {
            case 16: dif_pass<16>(z, n, N, tw, ntw); break;
            case 8: dif_pass<8>(z, n, N, tw, ntw); break;
            case 4: dif_pass<4>(z, n, N, tw, ntw); break;
            default: dif_pass<2>(z, n, N, tw, ntw); break;
        }
        N /= radix[p];
        __syncthreads();
    }
}

__device__ void inverse_fft(cplx* z, int n, const cplx* tw, int ntw, double final_scale) {
    int radix[8];
    const int passes = plan(n, radix);
    int Ns[8];
    int N = n;
    for (int p = 0; p < passes; ++p) {
        Ns[p] = N;
        N /= radix[p];
    }
    for (int p = passes - 1; p >= 0; --p) {
        const double sc = p == 0 ? final_scale : 1.0;
        switch (radix[p]) {
            case 16: dit_pass<16>(z, n, Ns[p], tw, ntw, sc); break;
            case 8: dit_pass<8>(z, n, Ns[p], tw, ntw, sc); break;
            case 4: dit_pass<4>(z, n, Ns[p], tw, ntw, sc); break;
            default: dit_pass<2>(z, n, Ns[p], tw, ntw, sc); break;
        }
        __syncthreads();
    }
}

// spectrum (digit-reversed) of the transposed circulant: forward DIF of c_T
__global__ void __launch_bounds__(FT) spectrum_kernel(const double* __restrict__ c, int n, const cplx* __restrict__ tw,
                                                      cplx* __restrict__ spec) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* z = reinterpret_cast<cplx*>(smem_raw);
    for (int i = threadIdx.x; i < n; i += blockDim.x) z[i] = {c[(n - i) % n], 0.0};
    __syncthreads();
    forward_fft(z, n, tw, n);
    for (int i = threadIdx.x; i < n; i += blockDim.x) spec[i] = z[i];
}

// rows of A (m x k, lda) times the n-point circulant (first k inputs, zero
// padded; first l outputs kept), two rows per CTA
__global__ void __launch_bounds__(FT) circ_rows_kernel(const double* __restrict__ a, int64_t lda, int64_t m, int k, int n,
                                                       const cplx* __restrict__ spec, const cplx* __restrict__ tw,
                                                       double* __restrict__ out, int64_t ldo, int l) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* z = reinterpret_cast<cplx*>(smem_raw);
    const int64_t r0 = 2 * static_cast<int64_t>(blockIdx.x);
    const bool two = r0 + 1 < m;
    const double* a0 = a + r0 * lda;
    const double* a1 = a + (r0 + 1) * lda;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double re = i < k ? __ldcs(a0 + i) : 0.0;
        const double im = (two && i < k) ? __ldcs(a1 + i) : 0.0;
        z[i] = {re, im};
    }
    __syncthreads();
    forward_fft(z, n, tw, n);
    for (int i = threadIdx.x; i < n; i += blockDim.x) z[i] = cmul(z[i], spec[i]);
    __syncthreads();
    inverse_fft(z, n, tw, n, 1.0 / static_cast<double>(n));
    double* o0 = out + r0 * ldo;
    double* o1 = out + (r0 + 1) * ldo;
    for (int i = threadIdx.x; i < l; i += blockDim.x) {
        __stcs(o0 + i, z[i].x);
        if (two) __stcs(o1 + i, z[i].y);
    }
}

// ---- narrow Toeplitz blocks by overlap-save correlation ---------------------------
// Y = A T for a k x l Toeplitz block of an np-point circulant with l << np
// (BASELINE config 5: np = k = 16384, l = 256): Y[i, j] = sum_t A[i, t]
// c[(t - j) mod np]. A row splits into chunks of Lc = NF - l + 1 samples;
// chunk s contributes the correlation of its samples with the segment
// h_s[u] = c[(s Lc - (l - 1) + u) mod np], u < NF, evaluated at lags
// j' = l - 1 - j < l, which an NF-point circular correlation gives without
// wrap-around: r_s = Omega^-1 (conj(Omega a_s) .* Omega h_s). The chunk
// products sum in the frequency domain, so one inverse transform serves all
// chunks of a row. Two real rows travel as one complex row z = a1 + i a2:
// conj(Omega z) = conj(Omega a1) - i conj(Omega a2), so the inverse is
// r1 - i r2. Per row that is ceil(k / Lc) NF-point transforms instead of two
// np-point ones (10 x 2048 against 2 x 8192 complex points here, about a
// third of the FP64 work), with the same single read of A.
constexpr int OLA_NF = 2048;  // transform length (complex points)
constexpr int OLA_T = 128;    // threads: one radix-16 group each

// spectra of the segments h_s (digit-reversed: the forward DIF's order)
__global__ void __launch_bounds__(OLA_T) ola_spectra_kernel(const double* __restrict__ c, int np, int lc, int l,
                                                            const cplx* __restrict__ tw, cplx* __restrict__ spec) {
    __shared__ __align__(16) cplx z[OLA_NF];
    const int s = blockIdx.x;
    const int64_t base = static_cast<int64_t>(s) * lc - (l - 1);
    for (int u = threadIdx.x; u < OLA_NF; u += blockDim.x) {
        const int64_t idx = ((base + u) % np + np) % np;
        z[u] = {c[idx], 0.0};
    }
    __syncthreads();
    forward_fft(z, OLA_NF, tw, OLA_NF);
    // stored in the rows kernel's pass-3 order: slot 8 g + r (g = t + 128 gg,
    // the last-pass group of thread t) at (8 gg + r) 128 + t, so one bulk copy
    // gives every thread its 16 slots at consecutive 16-byte positions
    for (int u = threadIdx.x; u < OLA_NF; u += blockDim.x) {
        const int g = u >> 3, r = u & 7;
        spec[static_cast<int64_t>(s) * OLA_NF + (8 * (g >> 7) + r) * OLA_T + (g & (OLA_T - 1))] = z[u];
    }
}

// smem slot of position p: XOR of the 16-byte slot's low three bits with bits
// 3..5 of p, so the three access patterns (stride 128 / stride 8 / 8
// consecutive per lane) all hit eight distinct slots per quarter warp
__device__ __forceinline__ int ola_sw(int p) { return p ^ ((p >> 3) & 7); }

// Two row pairs' chunk transforms per CTA would not fit the registers; one
// row pair per CTA, 128 threads, three passes (radix 16, 16, 8) held in
// registers between shared-memory exchanges, the accumulated spectrum in
// registers (each thread owns the 16 frequency slots of its last-pass groups),
// base twiddles cached per CTA. Latency hiding across chunks:
// - the segment spectrum of the next chunk is copied into shared memory by
//   one bulk copy (cp.async.bulk + mbarrier) as soon as the current one has
//   been consumed (barrier 3), so its L2 round trip runs under passes 1 and 2
//   instead of stalling pass 3 (the spectra are stored in pass-3 order: a
//   warp's 16-byte reads are consecutive): 3.63 -> 2.62 ms on config 5 with
//   per-thread cp.async;
// - the next chunk's two row segments are prefetched into L2 (one bulk
//   prefetch per row) at the start of the current chunk, so pass 1's loads
//   hit L2: 2.62 -> 2.54 ms. Loading them into registers under pass 3
//   instead spills at the 168-register cap of three CTAs per SM (3.56 ms).
constexpr int OLA_SMEM = static_cast<int>(sizeof(cplx)) * (OLA_NF + 16 * OLA_T + 4 * 128 + 4 * 8) + 16;
__global__ void __launch_bounds__(OLA_T, 3) ola_rows_kernel(const double* __restrict__ a, int64_t lda, int64_t m,
                                                            int k, int lc, int chunks, const cplx* __restrict__ spec,
                                                            const cplx* __restrict__ tw, double* __restrict__ out,
                                                            int64_t ldo, int l) {
    extern __shared__ __align__(16) unsigned char ola_smem[];
    cplx* z = reinterpret_cast<cplx*>(ola_smem);                      // OLA_NF
    cplx* hsm = z + OLA_NF;                                           // 16 * OLA_T thread-private spectrum slots
    cplx(*tw1)[128] = reinterpret_cast<cplx(*)[128]>(hsm + 16 * OLA_T);  // [4][128]: w_2048^{t 2^j}
    cplx(*tw2)[8] = reinterpret_cast<cplx(*)[8]>(tw1 + 4);              // [4][8]: w_128^{n0 2^j}
    uint64_t* hbar = reinterpret_cast<uint64_t*>(tw2 + 4);
    const int t = threadIdx.x;
    for (int i = t; i < 4 * 128; i += OLA_T) tw1[i >> 7][i & 127] = tw[((i & 127) << (i >> 7)) & (OLA_NF - 1)];
    if (t < 32) tw2[t >> 3][t & 7] = tw[(((t & 7) << (t >> 3)) * 16) & (OLA_NF - 1)];
    const int n2 = t & 7, o2 = (t >> 3) * 128;  // pass-2 group of this thread
    uint32_t hphase = 0;  // completed spectrum copies
    auto stage_spec = [&](int s) {  // thread 0, after every reader of hsm passed a barrier
        mbar_expect_tx(hbar, OLA_NF * sizeof(cplx));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                smem_u32(hsm)),
            "l"(spec + static_cast<int64_t>(s) * OLA_NF), "r"(static_cast<unsigned>(OLA_NF * sizeof(cplx))),
            "r"(smem_u32(hbar))
            : "memory");
    };
    if (t == 0) {
        mbar_init(hbar, 1);
        mbar_fence_init();
        if (2 * static_cast<int64_t>(blockIdx.x) < m) stage_spec(0);
    }
    __syncthreads();
    for (int64_t pair = blockIdx.x; 2 * pair < m; pair += gridDim.x) {
        const int64_t r0 = 2 * pair;
        const bool two = r0 + 1 < m;
        const double* a0 = a + r0 * lda;
        const double* a1 = two ? a + (r0 + 1) * lda : a0;
        auto load_chunk = [&](cplx (&v)[16], int s) {
            const int t0 = s * lc;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int u = t + 128 * j, idx = t0 + u;
                const bool in = u < lc && idx < k;
                v[j] = {in ? __ldcs(a0 + idx) : 0.0, (in && two) ? __ldcs(a1 + idx) : 0.0};
            }
        };
        cplx acc[2][8];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[g][q] = {0.0, 0.0};
        cplx v[16];
        for (int s = 0; s < chunks; ++s) {
            load_chunk(v, s);
            // the next chunk's two row segments into L2 (one thread per row)
            if (t < 2 && s + 1 < chunks && (t == 0 || two)) {
                const int t0n = (s + 1) * lc;
                const int len = min(lc, k - t0n);
                const uintptr_t p0 = reinterpret_cast<uintptr_t>((t == 0 ? a0 : a1) + t0n);
                const uintptr_t b0 = p0 & ~static_cast<uintptr_t>(15);
                // the end rounds down: the last row's tail must not reach past A
                const unsigned bytes = static_cast<unsigned>(((p0 + 8u * len) & ~static_cast<uintptr_t>(15)) - b0);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(b0), "r"(bytes));
            }
            // pass 1 (N = 2048, M = 128)
            dft_reg<16, false>(v);
            {
                cplx w[16];
                w[1] = tw1[0][t];
                w[2] = tw1[1][t];
                w[4] = tw1[2][t];
                w[8] = tw1[3][t];
                z[ola_sw(t)] = v[0];
#pragma unroll
                for (int r = 1; r < 16; ++r) {
                    lazy_twiddle<16>(w, r);
                    z[ola_sw(t + 128 * r)] = cmul(v[brev<16>(r)], w[r]);
                }
            }
            __syncthreads();
            // pass 2 (N = 128, M = 8)
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = z[ola_sw(o2 + n2 + 8 * j)];
            dft_reg<16, false>(v);
            {
                cplx w[16];
                w[1] = tw2[0][n2];
                w[2] = tw2[1][n2];
                w[4] = tw2[2][n2];
                w[8] = tw2[3][n2];
                z[ola_sw(o2 + n2)] = v[0];
#pragma unroll
                for (int r = 1; r < 16; ++r) {
                    lazy_twiddle<16>(w, r);
                    z[ola_sw(o2 + n2 + 8 * r)] = cmul(v[brev<16>(r)], w[r]);
                }
            }
            __syncthreads();
            // pass 3 (N = 8, M = 1): positions 8g + r; accumulate conj(Z) H_s
            mbar_wait(hbar, hphase & 1);
            ++hphase;
#pragma unroll
            for (int gg = 0; gg < 2; ++gg) {
                const int g = t + OLA_T * gg;
                cplx u8[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) u8[j] = z[ola_sw(8 * g + j)];
                dft_reg<8, false>(u8);
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const cplx zz = u8[brev<8>(r)], hh = hsm[(8 * gg + r) * OLA_T + t];
                    acc[gg][r].x = fma(zz.x, hh.x, fma(zz.y, hh.y, acc[gg][r].x));
                    acc[gg][r].y = fma(zz.x, hh.y, fma(-zz.y, hh.x, acc[gg][r].y));
                }
            }
            __syncthreads();  // z is rewritten by the next chunk's pass 1; hsm by the next copy
            if (t == 0) {
                if (s + 1 < chunks)
                    stage_spec(s + 1);
                else if (2 * (pair + gridDim.x) < m)
                    stage_spec(0);  // the next row pair's first chunk, under the inverse
            }
        }
        // inverse: DIT passes in reverse, the first from the registers
#pragma unroll
        for (int gg = 0; gg < 2; ++gg) {
            const int g = t + OLA_T * gg;
            dft_reg<8, true>(acc[gg]);
#pragma unroll
            for (int j = 0; j < 8; ++j) z[ola_sw(8 * g + j)] = acc[gg][brev<8>(j)];
        }
        __syncthreads();
        {
            cplx w[16];
            w[1] = tw2[0][n2];
            w[2] = tw2[1][n2];
            w[4] = tw2[2][n2];
            w[8] = tw2[3][n2];
            v[0] = z[ola_sw(o2 + n2)];
#pragma unroll
            for (int r = 1; r < 16; ++r) {
                lazy_twiddle<16>(w, r);
                v[r] = cmulc(z[ola_sw(o2 + n2 + 8 * r)], w[r]);
            }
            dft_reg<16, true>(v);
#pragma unroll
            for (int j = 0; j < 16; ++j) z[ola_sw(o2 + n2 + 8 * j)] = v[brev<16>(j)];
        }
        __syncthreads();
        {
            // last pass (N = 2048, M = 128): outputs t + 128 j; only lags < l are kept
            cplx w[16];
            w[1] = tw1[0][t];
            w[2] = tw1[1][t];
            w[4] = tw1[2][t];
            w[8] = tw1[3][t];
            v[0] = z[ola_sw(t)];
#pragma unroll
            for (int r = 1; r < 16; ++r) {
                lazy_twiddle<16>(w, r);
                v[r] = cmulc(z[ola_sw(t + 128 * r)], w[r]);
            }
            dft_reg<16, true>(v);
            const double scale = 1.0 / static_cast<double>(OLA_NF);
            double* o0 = out + r0 * ldo;
            double* o1 = out + (r0 + 1) * ldo;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int lag = t + 128 * j;
                if (lag < l) {
                    const cplx rv = v[brev<16>(j)];
                    __stcs(o0 + (l - 1 - lag), rv.x * scale);
                    if (two) __stcs(o1 + (l - 1 - lag), -rv.y * scale);
                }
            }
        }
        __syncthreads();  // z is reused by the next row pair
    }
}

// ---- parent length 2*MAXN on a 2-CTA cluster ------------------------------------
// CTA h keeps half h of the first radix-2 DIF split:
//   h = 0: y0[j] = z[j] + z[j + H]          h = 1: y1[j] = (z[j] - z[j + H]) w_n^j
// both halves are then independent H-point problems; the spectrum halves are
// the same split of the parent spectrum. Inverse: the last DIT radix-2 pass
// z[j] = (u0[j] + conj(w_n^j) u1[j]) / 2 ... only for the kept j < l, with u1
// read from the partner CTA's shared memory.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(FT)
circ_rows_split_kernel(const double* __restrict__ a, int64_t lda, int64_t m, int k, int n, const cplx* __restrict__ spec,
                       const cplx* __restrict__ tw, double* __restrict__ out, int64_t ldo, int l) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* z = reinterpret_cast<cplx*>(smem_raw);
    cg::cluster_group cluster = cg::this_cluster();
    const int h = static_cast<int>(cluster.block_rank());
    const int H = n / 2;
    const int64_t r0 = 2 * static_cast<int64_t>(blockIdx.x / 2);
    const bool two = r0 + 1 < m;
    const double* a0 = a + r0 * lda;
    const double* a1 = a + (r0 + 1) * lda;
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
        const int j2 = j + H;
        const cplx lo = {j < k ? a0[j] : 0.0, (two && j < k) ? a1[j] : 0.0};
        const cplx hi = {j2 < k ? a0[j2] : 0.0, (two && j2 < k) ? a1[j2] : 0.0};
        z[j] = h == 0 ? cadd(lo, hi) : cmul(csub(lo, hi), tw[j]);
    }
    __syncthreads();
    // H-point transform with the parent's twiddle table (w_H^k = w_n^{2k})
    {
        int radix[8];
        const int passes = plan(H, radix);
        int N = H;
        for (int p = 0; p < passes; ++p) {
            switch (radix[p]) {
                case 16: dif_pass<16>(z, H, N, tw, n); break;
                case 8: dif_pass<8>(z, H, N, tw, n); break;
                case 4: dif_pass<4>(z, H, N, tw, n); break;
                default: dif_pass<2>(z, H, N, tw, n); break;
            }
            N /= radix[p];
            __syncthreads();
        }
    }
    const cplx* sp = spec + static_cast<int64_t>(h) * H;
    for (int j = threadIdx.x; j < H; j += blockDim.x) z[j] = cmul(z[j], sp[j]);
    __syncthreads();
    {
        int radix[8];
        const int passes = plan(H, radix);
        int Ns[8];
        int N = H;
        for (int p = 0; p < passes; ++p) {
            Ns[p] = N;
            N /= radix[p];
        }
        for (int p = passes - 1; p >= 0; --p) {
            switch (radix[p]) {
                case 16: dit_pass<16>(z, H, Ns[p], tw, n, 1.0); break;
                case 8: dit_pass<8>(z, H, Ns[p], tw, n, 1.0); break;
                case 4: dit_pass<4>(z, H, Ns[p], tw, n, 1.0); break;
                default: dit_pass<2>(z, H, Ns[p], tw, n, 1.0); break;
            }
            __syncthreads();
        }
    }
    cluster.sync();
    // final inverse radix-2: x[j] = u0[j] + conj(w_n^j) u1[j], x[j+H] = u0[j] - conj(w_n^j) u1[j]
    const cplx* u0 = cluster.map_shared_rank(z, 0);
    const cplx* u1 = cluster.map_shared_rank(z, 1);
    const double scale = 1.0 / static_cast<double>(n);
    double* o0 = out + r0 * ldo;
    double* o1 = out + (r0 + 1) * ldo;
    // CTA h writes outputs j in [h*H, (h+1)*H) intersected with [0, l)
    for (int jj = threadIdx.x; jj < H; jj += blockDim.x) {
        const int j = jj + h * H;
        if (j >= l) break;
        const cplx t = cmulc(u1[jj], tw[jj]);
        const cplx v = h == 0 ? cadd(u0[jj], t) : csub(u0[jj], t);
        __stcs(o0 + j, v.x * scale);
        if (two) __stcs(o1 + j, v.y * scale);
    }
    cluster.sync();
}

// parent spectrum in split order: CTA h forms half h of the first radix-2
// DIF split of c_T and runs the H-point forward transform on it
__global__ void __launch_bounds__(FT) spectrum_split_kernel(const double* __restrict__ c, int n,
                                                            const cplx* __restrict__ tw, cplx* __restrict__ spec) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* z = reinterpret_cast<cplx*>(smem_raw);
    const int h = blockIdx.x, H = n / 2;
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
        const cplx lo = {c[(n - j) % n], 0.0}, hi = {c[(n - j - H) % n], 0.0};
        z[j] = h == 0 ? cadd(lo, hi) : cmul(csub(lo, hi), tw[j]);
    }
    __syncthreads();
    int radix[8];
    const int passes = plan(H, radix);
    int N = H;
    for (int p = 0; p < passes; ++p) {
        switch (radix[p]) {
            case 16: dif_pass<16>(z, H, N, tw, n); break;
            case 8: dif_pass<8>(z, H, N, tw, n); break;
            case 4: dif_pass<4>(z, H, N, tw, n); break;
            default: dif_pass<2>(z, H, N, tw, n); break;
        }
        N /= radix[p];
        __syncthreads();
    }
    for (int j = threadIdx.x; j < H; j += blockDim.x) spec[static_cast<int64_t>(h) * H + j] = z[j];
}

// dense expansion of the leading k x l block of the np-point circulant
// (circulant.hpp:143-169: entry (i, j) = c[(i - j) mod np])
__global__ void circulant_dense_kernel(const double* __restrict__ c, int64_t np, int64_t k, int64_t l,
                                       double* __restrict__ h, int64_t ldh) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= k * l) return;
    const int64_t i = idx / l, j = idx % l;
    h[i * ldh + j] = c[((i - j) % np + np) % np];
}

// ---- real-input path: one real row per CTA through a half-length complex
// transform (m = n/2 points, 16 m bytes of shared memory: two CTAs per SM at
// n = 8192). z[j] = x[2j] + i x[2j+1]; after the DIF passes the spectrum sits
// in digit-reversed order; pairs (k, m-k) are unpacked to the real spectrum
// X_k, multiplied by the multiplier spectrum S_k (natural order), re-packed
// for the half-length inverse, and the DIT passes return y[2j] + i y[2j+1].
// Everything is specialised on L = log2 m, so pass loops, strides and the
// digit reversal are compile-time constants.
namespace r2c {

template <int L>
struct Shape {
    static constexpr int m = 1 << L, n = 2 * m;
    static constexpr int full = L / 4, rem = L % 4;
    static constexpr int passes = full + (rem ? 1 : 0);
#ifndef RL_FFT_T13
#define RL_FFT_T13 512
#endif
#ifndef RL_FFT_T12
#define RL_FFT_T12 256
#endif
#ifndef RL_FFT_MINB12
#define RL_FFT_MINB12 2
#endif
    static constexpr int T = L >= 13 ? RL_FFT_T13 : RL_FFT_T12;  // threads per CTA
    static constexpr int minb = L >= 13 ? 1 : RL_FFT_MINB12;
    __host__ __device__ static constexpr int radix(int p) { return p < full ? 16 : 1 << rem; }
    __host__ __device__ static constexpr int sub(int p) { return m >> (4 * p); }  // subarray length entering pass p
    // base twiddles w_N^{n0 2^j} (j < log2 R) of the passes with M = N/R > 1,
    // cached per CTA in shared memory behind z as [pass][j][n0]
    __host__ __device__ static constexpr int lgr(int p) { return p < full ? 4 : rem; }
    __host__ __device__ static constexpr int tw_m(int p) { return sub(p) >> lgr(p); }
    __host__ __device__ static constexpr int tw_entries(int p) { return tw_m(p) > 1 ? tw_m(p) * lgr(p) : 0; }
    __host__ __device__ static constexpr int tw_off(int p) { return p == 0 ? 0 : tw_off(p - 1) + tw_entries(p - 1); }
    static constexpr int tw_total = tw_off(passes);
    // w_n^q (q < m/2) for the spectrum unpack / repack also cached when it
    // still fits minb CTAs per SM (228 KiB per SM, 1 KiB reserved per CTA)
    static constexpr int smem_base = (m + tw_total) * 16;
    static constexpr bool unpack_cache = minb * (smem_base + (m / 2) * 16 + 1024) <= 228 * 1024;
    static constexpr int smem_rows = smem_base + (unpack_cache ? (m / 2) * 16 : 0);
};

// shared-memory slot of element i: XOR swizzle of the 16-byte slot index so
// that the stride-16 (last radix-16 pass) and stride-256 (digit-reversed
// unpack) patterns hit distinct bank groups within a quarter-warp
// Specialised per length: the digit-reversed unpack varies bits L-4..L-2 of the
// index (the top radix-16 digit); for L = 1 mod 4 the final radix-2 pass reads
// stride-2 pairs, separated by folding bit 3 in as well.
template <int L>
__device__ __forceinline__ int swz(int i) {
    constexpr int hi = L >= 8 ? L - 4 : 4;
    int f = (i >> 4) ^ (i >> hi);
    if (L % 4 == 1) f ^= (i >> 3) & 1;
    return i ^ (f & 7);
}

// position of frequency k after the DIF passes: base-16 digit reversal
template <int L>
__device__ __forceinline__ int dif_pos(int k) {
    constexpr int full = L / 4;
    int p = 0;
#pragma unroll
    for (int i = 0; i < full; ++i) p |= ((k >> (4 * i)) & 15) << (L - 4 * (i + 1));
    return p | (k >> (4 * full));
}

// one DIF pass over subarrays of length N (radix R); kGlobal: the input is the
// real row x (length k, zero padded), read straight from global memory
// base twiddles of a pass from the shared-memory cache (see Shape::tw_off)
template <int R>
__device__ __forceinline__ void cached_twiddles(cplx (&w)[R], const cplx* twc, int n0, int M) {
    if (R > 1) w[1] = twc[n0];
    if (R > 2) w[2] = twc[M + n0];
    if (R > 4) w[4] = twc[2 * M + n0];
    if (R > 8) w[8] = twc[3 * M + n0];
}

template <int L, int R, int N, bool kGlobal>
__device__ __forceinline__ void dif(cplx* z, const double* __restrict__ x, int k, const cplx* __restrict__ tw,
                                    const cplx* twc = nullptr) {
    using S = Shape<L>;
    constexpr int M = N / R, groups = S::m / R;
    constexpr int64_t tstride = S::n / N;
#pragma unroll
    for (int g0 = 0; g0 < groups; g0 += S::T) {
        const int g = g0 + threadIdx.x;
        if (groups % S::T != 0 && g >= groups) break;
        const int n0 = g % M, o = (g / M) * N;
        cplx v[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int q = o + n0 + j * M;
            if (kGlobal) {
                if (2 * q + 1 < k) {
                    const double2 t = __ldcs(reinterpret_cast<const double2*>(x) + q);
                    v[j] = {t.x, t.y};
                } else {
                    v[j] = {2 * q < k ? x[2 * q] : 0.0, 0.0};
                }
            } else {
                v[j] = z[swz<L>(q)];
            }
        }
        dft_reg<R, false>(v);
        z[swz<L>(o + n0)] = v[0];
        if constexpr (M == 1) {
            // last pass: every twiddle is w^0 = 1
#pragma unroll
            for (int r = 1; r < R; ++r) z[swz<L>(o + r)] = v[brev<R>(r)];
        } else {
            cplx w[R];
            if (twc)
                cached_twiddles<R>(w, twc, n0, M);
            else
                base_twiddles<R>(w, tw, static_cast<int64_t>(n0) * tstride, S::n - 1);
#pragma unroll
            for (int r = 1; r < R; ++r) {
                lazy_twiddle<R>(w, r);
                z[swz<L>(o + n0 + r * M)] = cmul(v[brev<R>(r)], w[r]);
            }
        }
    }
}

// one DIT pass with conjugate twiddles; kGlobal: the last pass, writing
// y[2q] = Re, y[2q+1] = Im (scaled) for 2q < l straight to global memory
template <int L, int R, int N, bool kGlobal>
__device__ __forceinline__ void dit(cplx* z, double* __restrict__ y, int l, double scale,
                                    const cplx* __restrict__ tw, const cplx* twc = nullptr) {
    using S = Shape<L>;
    constexpr int M = N / R, groups = S::m / R;
    constexpr int64_t tstride = S::n / N;
    if constexpr (kGlobal && N == S::m && M > 1) {
        // pruned last pass when the first l outputs (q < ceil(l/2) <= M) all
        // come from output r = 0 of the groups n0 < ceil(l/2): only that
        // output, the DC term of the twiddled inputs, summed in dft_reg's order
        const int ql = (l + 1) / 2;
        if (ql <= M) {
            for (int n0 = threadIdx.x; n0 < ql; n0 += S::T) {
                cplx w[R];
                if (twc)
                    cached_twiddles<R>(w, twc, n0, M);
                else
                    base_twiddles<R>(w, tw, static_cast<int64_t>(n0) * tstride, S::n - 1);
                cplx v[R];
                v[0] = z[swz<L>(n0)];
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    lazy_twiddle<R>(w, r);
                    v[r] = cmulc(z[swz<L>(n0 + r * M)], w[r]);
                }
#pragma unroll
                for (int half = R / 2; half >= 1; half >>= 1)
#pragma unroll
                    for (int j = 0; j < half; ++j) v[j] = cadd(v[j], v[j + half]);
                const cplx t = v[0];
                if (2 * n0 + 1 < l) {
                    __stcs(reinterpret_cast<double2*>(y) + n0, make_double2(t.x * scale, t.y * scale));
                } else {
                    y[2 * n0] = t.x * scale;
                }
            }
            return;
        }
    }
#pragma unroll
    for (int g0 = 0; g0 < groups; g0 += S::T) {
        const int g = g0 + threadIdx.x;
        if (groups % S::T != 0 && g >= groups) break;
        const int n0 = g % M, o = (g / M) * N;
        cplx v[R];
        v[0] = z[swz<L>(o + n0)];
        if constexpr (M == 1) {
            // first inverse pass: every twiddle is w^0 = 1
#pragma unroll
            for (int r = 1; r < R; ++r) v[r] = z[swz<L>(o + r)];
        } else {
            cplx w[R];
            if (twc)
                cached_twiddles<R>(w, twc, n0, M);
            else
                base_twiddles<R>(w, tw, static_cast<int64_t>(n0) * tstride, S::n - 1);
#pragma unroll
            for (int r = 1; r < R; ++r) {
                lazy_twiddle<R>(w, r);
                v[r] = cmulc(z[swz<L>(o + n0 + r * M)], w[r]);
            }
        }
        dft_reg<R, true>(v);
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const cplx t = v[brev<R>(j)];
            const int q = o + n0 + j * M;
            if (kGlobal) {
                if (2 * q + 1 < l) {
                    __stcs(reinterpret_cast<double2*>(y) + q, make_double2(t.x * scale, t.y * scale));
                } else if (2 * q < l) {
                    y[2 * q] = t.x * scale;
                }
            } else {
                z[swz<L>(q)] = t;
            }
        }
    }
}

template <int L, int P>
__device__ __forceinline__ void dif_from(cplx* z, const double* x, int k, const cplx* tw, const cplx* twc = nullptr) {
    using S = Shape<L>;
    if constexpr (P < S::passes) {
        dif<L, S::radix(P), S::sub(P), P == 0>(z, x, k, tw, twc ? twc + S::tw_off(P) : nullptr);
        __syncthreads();
        dif_from<L, P + 1>(z, x, k, tw, twc);
    }
}

template <int L, int P>
__device__ __forceinline__ void dit_down(cplx* z, double* y, int l, double scale, const cplx* tw,
                                         const cplx* twc = nullptr) {
    using S = Shape<L>;
    if constexpr (P >= 0) {
        dit<L, S::radix(P), S::sub(P), P == 0>(z, y, l, scale, tw, twc ? twc + S::tw_off(P) : nullptr);
        if constexpr (P > 0) {
            __syncthreads();
            dit_down<L, P - 1>(z, y, l, scale, tw, twc);
        }
    }
}

// fill the per-CTA twiddle cache: entry [tw_off(p) + j M + n0] = w_N^{n0 2^j}
template <int L, int P>
__device__ __forceinline__ void fill_twiddle_cache(cplx* twc, const cplx* __restrict__ tw) {
    using S = Shape<L>;
    if constexpr (P < S::passes) {
        constexpr int M = S::tw_m(P), E = S::tw_entries(P);
        constexpr int64_t tstride = S::n / S::sub(P);
        for (int e = threadIdx.x; e < E; e += S::T) {
            const int j = e / M, n0 = e % M;
            twc[S::tw_off(P) + e] = tw[((static_cast<int64_t>(n0) << j) * tstride) & (S::n - 1)];
        }
        fill_twiddle_cache<L, P + 1>(twc, tw);
    }
}

// real spectrum X_k and X_{m-k} (k <= m/2) from the packed half-length
// transform Z (digit-reversed in z): E = (Z_k + conj Z_{m-k})/2,
// O = (Z_k - conj Z_{m-k})/(2i), X_k = E + w_n^k O, X_{m-k} = conj(E - w_n^k O);
// k = 0 yields X_0 and X_m
template <int L>
__device__ __forceinline__ void unpack_pair(const cplx* z, int k, cplx wk, cplx& xk, cplx& xmk) {
    constexpr int m = Shape<L>::m;
    const cplx zk = z[swz<L>(dif_pos<L>(k))];
    const cplx zm = z[swz<L>(dif_pos<L>((m - k) & (m - 1)))];
    const cplx e = {0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y)};
    const cplx o = {0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x)};
    if (k == 0) {
        xk = {e.x + o.x, e.y + o.y};
        xmk = {e.x - o.x, e.y - o.y};
        return;
    }
    const cplx wo = cmul(wk, o);
    xk = cadd(e, wo);
    const cplx d = csub(e, wo);
    xmk = {d.x, -d.y};
}

// Z'_k = (Y_k + conj Y_{m-k}) + i (Y_k - conj Y_{m-k}) conj(w_n^k)
__device__ __forceinline__ cplx repack(cplx yk, cplx partner, cplx wk) {
    const cplx ee = cadd(yk, partner);
    const cplx oo = cmulc(csub(yk, partner), wk);
    return {ee.x - oo.y, ee.y + oo.x};
}

// spectrum S_k (k = 0..m, natural order) of c_T, c_T[i] = c[(n-i) mod n]
template <int L>
__global__ void __launch_bounds__(Shape<L>::T) spectrum_kernel(const double* __restrict__ c,
                                                                const cplx* __restrict__ tw, cplx* __restrict__ spec) {
    using S = Shape<L>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* z = reinterpret_cast<cplx*>(smem_raw);
    constexpr int m = S::m, n = S::n;
    for (int j = threadIdx.x; j < m; j += S::T) z[swz<L>(j)] = {c[(n - 2 * j) % n], c[(n - 2 * j - 1) % n]};
    __syncthreads();
    // first pass from shared memory: reuse dif<> with kGlobal = false
    dif<L, S::radix(0), S::sub(0), false>(z, nullptr, 0, tw);
    __syncthreads();
    dif_from<L, 1>(z, nullptr, 0, tw);
    for (int k = threadIdx.x; k <= m / 2; k += S::T) {
        cplx xk, xmk;
        unpack_pair<L>(z, k, tw[k], xk, xmk);
        spec[k] = xk;
        spec[m - k] = xmk;
    }
}

// one real row of A (k inputs) per CTA times the n-point real circulant,
// first l outputs
template <int L>
__global__ void __launch_bounds__(Shape<L>::T, Shape<L>::minb)
    rows_kernel(const double* __restrict__ a, int64_t rows, int64_t lda, int k, const cplx* __restrict__ spec,
                const cplx* __restrict__ tw, double* __restrict__ out, int64_t ldo, int l) {
    using S = Shape<L>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* z = reinterpret_cast<cplx*>(smem_raw);
    constexpr int m = S::m;
    cplx* twc = z + m;
    fill_twiddle_cache<L, 0>(twc, tw);
    cplx* twu = twc + S::tw_total;  // w_n^q, q < m/2 (unpack_cache)
    if constexpr (S::unpack_cache)
        for (int q = threadIdx.x; q < m / 2; q += S::T) twu[q] = tw[q];
    __syncthreads();
    // persistent: each CTA walks rows blockIdx.x, + gridDim.x, ...; the next
    // row is prefetched into L2 while this one is transformed, so the first
    // pass's loads hit L2 instead of waiting on HBM
#pragma unroll 1
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    if (threadIdx.x == 0 && row + gridDim.x < rows) {
        const char* nxt = reinterpret_cast<const char*>(a + (row + gridDim.x) * lda);
        const int bytes = ((k * 8) + 15) & ~15;
        for (int off = 0; off < bytes; off += 32768)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(nxt + off), "r"(min(32768, bytes - off)));
    }
    dif_from<L, 0>(z, a + row * lda, k, tw, twc);
#pragma unroll 1
    for (int q = threadIdx.x; q <= m / 2; q += S::T) {
        // w_n^q and w_n^{m-q} = -conj(w_n^q) (w_n^m = -1); w_n^{m/2} = i
        cplx wq, wmq;
        if constexpr (S::unpack_cache) {
            wq = q < m / 2 ? twu[q] : cplx{0.0, 1.0};
            wmq = {-wq.x, wq.y};
        } else {
            wq = tw[q];
            wmq = tw[m - q];
        }
        cplx xk, xmk;
        unpack_pair<L>(z, q, wq, xk, xmk);
        const cplx yk = cmul(spec[q], xk), ymk = cmul(spec[m - q], xmk);
        const int pk = swz<L>(dif_pos<L>(q)), pm = swz<L>(dif_pos<L>((m - q) & (m - 1)));
        if (q == 0) {
            // Ee_0 = Y_0 + Y_m, Oo_0 = Y_0 - Y_m
            z[pk] = {(yk.x + ymk.x) - (yk.y - ymk.y), (yk.y + ymk.y) + (yk.x - ymk.x)};
        } else {
            const cplx cym = {ymk.x, -ymk.y}, cyk = {yk.x, -yk.y};
            const cplx zk = repack(yk, cym, wq);
            const cplx zm = repack(ymk, cyk, wmq);
            z[pk] = zk;
            z[pm] = zm;
        }
    }
    __syncthreads();
    dit_down<L, S::passes - 1>(z, out + row * ldo, l, 1.0 / static_cast<double>(S::n), tw, twc);
    __syncthreads();  // the last pass has read z before the next row's first pass writes it
    }
}

template <int L>
rl_status launch_L(rl_context* ctx, int64_t rows, int k, const double* a, int64_t lda, const double* c,
                   const cplx* tw, cplx* spec, double* out, int64_t ldo, int l) {
    using S = Shape<L>;
    constexpr int smem = S::m * 16;
    constexpr int smem_rows = S::smem_rows;
    static PerDeviceOnce configured_once;
    {
        const rl_status cst = once_per_device(configured_once, [&]() -> rl_status {
            RL_CUDA(cudaFuncSetAttribute(spectrum_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            RL_CUDA(cudaFuncSetAttribute(rows_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_rows));
            return RL_OK;
        });
        if (cst != RL_OK) return cst;
    }
    spectrum_kernel<L><<<1, S::T, smem, ctx->stream>>>(c, tw, spec);
    RL_CHECK_LAUNCH("r2c::spectrum_kernel");
    const int64_t grid = std::min<int64_t>(rows, static_cast<int64_t>(ctx->num_sms) * S::minb);
    rows_kernel<L><<<static_cast<unsigned>(grid), S::T, smem_rows, ctx->stream>>>(a, rows, lda, k, spec, tw, out, ldo, l);
    RL_CHECK_LAUNCH("r2c::rows_kernel");
    return RL_OK;
}

rl_status launch(rl_context* ctx, int L, int64_t rows, int k, const double* a, int64_t lda, const double* c,
                 const cplx* tw, cplx* spec, double* out, int64_t ldo, int l) {
    switch (L) {
#define RL_R2C_CASE(LL) \
    case LL: return launch_L<LL>(ctx, rows, k, a, lda, c, tw, spec, out, ldo, l);
        RL_R2C_CASE(1) RL_R2C_CASE(2) RL_R2C_CASE(3) RL_R2C_CASE(4) RL_R2C_CASE(5) RL_R2C_CASE(6) RL_R2C_CASE(7)
        RL_R2C_CASE(8) RL_R2C_CASE(9) RL_R2C_CASE(10) RL_R2C_CASE(11) RL_R2C_CASE(12) RL_R2C_CASE(13)
#undef RL_R2C_CASE
        default: return set_error(RL_ERR_UNSUPPORTED, "r2c: log2 half length %d", L);
    }
}

}  // namespace r2c

struct TwCache {
    std::mutex mu;
    std::map<std::pair<int, int64_t>, cplx*> tables;  // (device, n) -> table
};
TwCache& tw_cache() {
    static TwCache* c = new TwCache();  // intentionally leaked (lives for the process)
    return *c;
}

rl_status twiddles(rl_context* ctx, int64_t n, cplx** out) {
    TwCache& c = tw_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto key = std::make_pair(ctx->device, n);
    auto it = c.tables.find(key);
    if (it != c.tables.end()) {
        *out = it->second;
        return RL_OK;
    }
    cplx* t = nullptr;
    RL_CUDA(cudaMalloc(&t, sizeof(cplx) * n));
    twiddle_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(n, t);
    RL_CHECK_LAUNCH("twiddle_kernel");
    RL_CUDA(cudaStreamSynchronize(ctx->stream));
    c.tables[key] = t;
    *out = t;
    return RL_OK;
}

bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

}  // namespace

// device driver: out (m x l, ldo) = A (m x k, lda) * leading k x l block of
// the np-point circulant with first column c (device). spec_ws >= np complex.
rl_status circulant_rows(rl_context* ctx, int64_t m, int64_t k, const double* a, int64_t lda, int64_t np,
                         const double* c, int64_t l, double* out, int64_t ldo, void* spec_ws) {
    if (m <= 0) return RL_OK;
    if (!is_pow2(np) || np > 2 * MAXN || np < 2)
        return set_error(RL_ERR_UNSUPPORTED, "circulant_rows: parent length %lld (power of two <= %d)",
                         static_cast<long long>(np), 2 * MAXN);
    cplx* tw = nullptr;
    rl_status st = twiddles(ctx, np, &tw);
    if (st != RL_OK) return st;
    cplx* spec = static_cast<cplx*>(spec_ws);
    const int n = static_cast<int>(np);
    static PerDeviceOnce configured_once;
    {
        const rl_status cst = once_per_device(configured_once, [&]() -> rl_status {
            RL_CUDA(cudaFuncSetAttribute(spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAXN * 16));
            RL_CUDA(cudaFuncSetAttribute(circ_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAXN * 16));
            RL_CUDA(cudaFuncSetAttribute(circ_rows_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAXN * 16));
            RL_CUDA(cudaFuncSetAttribute(spectrum_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAXN * 16));
            return RL_OK;
        });
        if (cst != RL_OK) return cst;
    }
    const bool aligned = (lda % 2 == 0) && (ldo % 2 == 0) && (reinterpret_cast<uintptr_t>(a) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    if (n >= 4 * OLA_NF && 8 * l <= OLA_NF && m >= 2) {
        // narrow Toeplitz block: overlap-save correlation with NF-point transforms
        const int lc = OLA_NF - static_cast<int>(l) + 1;
        const int chunks = static_cast<int>((k + lc - 1) / lc);
        cplx* tw_f = nullptr;
        if ((st = twiddles(ctx, OLA_NF, &tw_f)) != RL_OK) return st;
        cplx* ospec = nullptr;
        RL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ospec), sizeof(cplx) * OLA_NF * chunks, ctx->stream));
        ola_spectra_kernel<<<chunks, OLA_T, 0, ctx->stream>>>(c, n, lc, static_cast<int>(l), tw_f, ospec);
        RL_CHECK_LAUNCH("ola_spectra_kernel");
        const int64_t pairs = (m + 1) / 2;
        const int64_t grid = std::min<int64_t>(pairs, static_cast<int64_t>(ctx->num_sms) * 3);
        static PerDeviceOnce ola_once;
        const rl_status ost = once_per_device(ola_once, [&]() -> rl_status {
            RL_CUDA(cudaFuncSetAttribute(ola_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OLA_SMEM));
            return RL_OK;
        });
        if (ost != RL_OK) return ost;
        ola_rows_kernel<<<static_cast<unsigned>(grid), OLA_T, OLA_SMEM, ctx->stream>>>(
            a, lda, m, static_cast<int>(k), lc, chunks, ospec, tw_f, out, ldo, static_cast<int>(l));
        RL_CHECK_LAUNCH("ola_rows_kernel");
        RL_CUDA(cudaFreeAsync(ospec, ctx->stream));
        return RL_OK;
    }
    if (aligned && n >= 4) {
        int L = 0;
        while ((2 << L) < n) ++L;
        st = r2c::launch(ctx, L, m, static_cast<int>(k), a, lda, c, tw, spec, out, ldo, static_cast<int>(l));
        if (st != RL_OK) return st;
    } else if (n <= MAXN) {
        spectrum_kernel<<<1, FT, n * 16, ctx->stream>>>(c, n, tw, spec);
        RL_CHECK_LAUNCH("spectrum_kernel");
        circ_rows_kernel<<<static_cast<unsigned>((m + 1) / 2), FT, n * 16, ctx->stream>>>(
            a, lda, m, static_cast<int>(k), n, spec, tw, out, ldo, static_cast<int>(l));
        RL_CHECK_LAUNCH("circ_rows_kernel");
    } else {
        spectrum_split_kernel<<<2, FT, (n / 2) * 16, ctx->stream>>>(c, n, tw, spec);
        RL_CHECK_LAUNCH("spectrum_split_kernel");
        circ_rows_split_kernel<<<static_cast<unsigned>(2 * ((m + 1) / 2)), FT, (n / 2) * 16, ctx->stream>>>(
            a, lda, m, static_cast<int>(k), n, spec, tw, out, ldo, static_cast<int>(l));
        RL_CHECK_LAUNCH("circ_rows_split_kernel");
    }
    return RL_OK;
}

}  // namespace rl

namespace rl {
// dense expansion (device) of the leading k x l block of the np-point circulant
rl_status circulant_dense(rl_context* ctx, const double* c, int64_t np, int64_t k, int64_t l, double* h, int64_t ldh) {
    circulant_dense_kernel<<<static_cast<unsigned>((k * l + 255) / 256), 256, 0, ctx->stream>>>(c, np, k, l, h, ldh);
    RL_CHECK_LAUNCH("circulant_dense_kernel");
    return RL_OK;
}

bool circulant_fft_ok(int64_t np) { return is_pow2(np) && np <= 2 * MAXN; }
}  // namespace rl

// ---- standalone complex transforms: fft / inverse_fft (fft.hpp:76-98) -------
namespace rl {
namespace {

// position of natural-order frequency k in the digit-reversed output of
// forward_fft (the DIF pass with radix R leaves frequencies = r (mod R) in
// subarray r of length N / R, recursively)
__device__ __forceinline__ int dif_position(int k, int n) {
    int radix[8];
    const int passes = plan(n, radix);
    int pos = 0, N = n;
    for (int p = 0; p < passes; ++p) {
        const int R = radix[p];
        N /= R;
        pos += (k % R) * N;
        k /= R;
    }
    return pos;
}

// one vector of n <= MAXN points per CTA, resident in shared memory
__global__ void __launch_bounds__(FT) cfft_kernel(cplx* __restrict__ z, int n, const cplx* __restrict__ tw, int inverse) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* s = reinterpret_cast<cplx*>(smem_raw);
    cplx* v = z + static_cast<int64_t>(blockIdx.x) * n;
    if (inverse) {  // the DIT passes consume the digit-reversed order
        for (int k = threadIdx.x; k < n; k += blockDim.x) s[dif_position(k, n)] = v[k];
        __syncthreads();
        inverse_fft(s, n, tw, n, 1.0 / static_cast<double>(n));
        for (int k = threadIdx.x; k < n; k += blockDim.x) v[k] = s[k];
    } else {
        for (int k = threadIdx.x; k < n; k += blockDim.x) s[k] = v[k];
        __syncthreads();
        forward_fft(s, n, tw, n);
        for (int k = threadIdx.x; k < n; k += blockDim.x) v[k] = s[dif_position(k, n)];
    }
}

// longer power-of-two vectors: radix-2 Stockham passes through global memory
// (natural order in and out); pass span ns = 1, 2, 4, ..., n/2
__global__ void stockham_pass_kernel(const cplx* __restrict__ x, cplx* __restrict__ y, int64_t n, int64_t count,
                                     int64_t ns, const cplx* __restrict__ tw, int inverse, double scale) {
    const int64_t half = n / 2;
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= count * half) return;
    const int64_t v = idx / half, j = idx % half;
    const cplx* xv = x + v * n;
    cplx* yv = y + v * n;
    const int64_t k = j % ns;
    const cplx w = tw[k * (n / (2 * ns))];  // exp(+2 pi i k / (2 ns))
    const cplx a = xv[j];
    const cplx b = inverse ? cmulc(xv[j + half], w) : cmul(xv[j + half], w);
    const int64_t d = (j / ns) * ns * 2 + k;
    const cplx p = cadd(a, b), q = csub(a, b);
    yv[d] = {p.x * scale, p.y * scale};
    yv[d + ns] = {q.x * scale, q.y * scale};
}

// other lengths: the dense transform the reference falls back to
// (dft_dense_apply, fft.hpp:59-72), one output entry per thread
__global__ void dft_dense_kernel(const cplx* __restrict__ x, cplx* __restrict__ y, int64_t n, int64_t count,
                                 const cplx* __restrict__ tw, int inverse) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= count * n) return;
    const int64_t v = idx / n, i = idx % n;
    const cplx* xv = x + v * n;
    cplx acc = {0.0, 0.0};
    int64_t t = 0;  // (i j) mod n
    for (int64_t j = 0; j < n; ++j) {
        const cplx r = tw[t];
        acc = cadd(acc, inverse ? cmulc(xv[j], r) : cmul(xv[j], r));
        t += i;
        if (t >= n) t -= n;
    }
    const double sc = inverse ? 1.0 / static_cast<double>(n) : 1.0;
    y[idx] = {acc.x * sc, acc.y * sc};
}

}  // namespace
}  // namespace rl

// ---- C ABI -----------------------------------------------------------------
namespace {
using namespace rl;

rl_status right_multiply(rl_context* ctx, rl_mem mem, int64_t m, int64_t k, const double* a, int64_t np,
                         const double* c, int64_t l, double* out) {
    if (m <= 0 || k <= 0 || np <= 0 || l <= 0) return set_error(RL_ERR_DIMENSION, "matmul_by_circulant: empty shape");
    if (k > np || l > np) return set_error(RL_ERR_DIMENSION, "toeplitz block exceeds parent dimensions");
    if (!a || !c || !out) return set_error(RL_ERR_INVALID_ARGUMENT, "matmul_by_circulant: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    const bool host = mem == RL_HOST;
    const bool fft_path = is_pow2(np) && np <= 2 * MAXN;
    const double *da = a, *dc = c;
    double* dout = out;
    void* spec = nullptr;
    double* hdense = nullptr;
    const int64_t ldl = (l + 1) & ~int64_t(1), ldk = (k + 1) & ~int64_t(1);
    // the GEMM fallback (non power-of-two parents) needs even leading dims
    const bool stage_a = host || (!fft_path && ((k & 1) || (reinterpret_cast<uintptr_t>(a) & 15)));
    const bool stage_out = host || (!fft_path && ((l & 1) || (reinterpret_cast<uintptr_t>(out) & 15)));
    bool ok = with_arena(ctx, [&](Arena& ar) {
        if (stage_a) da = ar.take<double>(m * ldk);
        if (host) dc = ar.take<double>(np);
        if (stage_out) dout = ar.take<double>(m * ldl);
        if (fft_path)
            spec = ar.take<char>(np * 16);
        else
            hdense = ar.take<double>(k * ldl);
    });
    if (!ok) return RL_ERR_OUT_OF_MEMORY;
    cudaStream_t s = ctx->stream;
    const int64_t lda = stage_a ? ldk : k, ldo = stage_out ? ldl : l;
    if (stage_a)
        RL_CUDA(cudaMemcpy2DAsync(const_cast<double*>(da), ldk * 8, a, k * 8, k * 8, m,
                                  host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    if (host) RL_CUDA(cudaMemcpyAsync(const_cast<double*>(dc), c, np * 8, cudaMemcpyHostToDevice, s));
    if (fft_path) {
        st = circulant_rows(ctx, m, k, da, lda, np, dc, l, dout, ldo, spec);
    } else {
        circulant_dense_kernel<<<static_cast<unsigned>((k * l + 255) / 256), 256, 0, s>>>(dc, np, k, l, hdense, ldl);
        RL_CHECK_LAUNCH("circulant_dense_kernel");
        st = gemm(ctx, m, l, k, da, lda, hdense, ldl, dout, ldo, 1.0, false, nullptr);
    }
    if (st != RL_OK) return st;
    if (stage_out)
        RL_CUDA(cudaMemcpy2DAsync(out, l * 8, dout, ldl * 8, l * 8, m,
                                  host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    if (host) RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}
}  // namespace

extern "C" RL_API rl_status rl_circulant_right_multiply(rl_context* ctx, rl_mem mem, int64_t m, int64_t n,
                                                        const double* a, const double* c, double* out) {
    return right_multiply(ctx, mem, m, n, a, n, c, n, out);
}

extern "C" RL_API rl_status rl_toeplitz_right_multiply(rl_context* ctx, rl_mem mem, int64_t m, int64_t k,
                                                       const double* a, int64_t np, const double* c, int64_t l,
                                                       double* out) {
    return right_multiply(ctx, mem, m, k, a, np, c, l, out);
}

namespace rl {
// batched complex transform of `count` contiguous rows of n points, in place
// on the device (fft.hpp:76-98, +1 sign forward, 1/n on the inverse); `work`
// (count * n complex) is needed unless n is a power of two <= MAXN.
size_t cfft_work_bytes(int64_t count, int64_t n) { return is_pow2(n) && n <= MAXN ? 0 : size_t(count) * n * 16; }
rl_status cfft_device(rl_context* ctx, int64_t count, int64_t n, double* z, bool inverse, double* work_ptr) {
    if (count <= 0) return RL_OK;
    cudaStream_t s = ctx->stream;
    cplx* dz = reinterpret_cast<cplx*>(z);
    cplx* work = reinterpret_cast<cplx*>(work_ptr);
    const bool pow2 = is_pow2(n);
    const bool small = pow2 && n <= MAXN;
    if (!small && !work) return set_error(RL_ERR_INVALID_ARGUMENT, "fft: work buffer required for n = %lld", (long long)n);
    rl_status st;
    cplx* tw = nullptr;
    if ((st = twiddles(ctx, n, &tw)) != RL_OK) return st;
    if (small) {
        static PerDeviceOnce configured_once;
        st = once_per_device(configured_once, [&]() -> rl_status {
            RL_CUDA(cudaFuncSetAttribute(cfft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAXN * 16));
            return RL_OK;
        });
        if (st != RL_OK) return st;
        cfft_kernel<<<static_cast<unsigned>(count), FT, static_cast<int>(n) * 16, s>>>(dz, static_cast<int>(n), tw,
                                                                                        inverse ? 1 : 0);
        RL_CHECK_LAUNCH("cfft_kernel");
    } else if (pow2) {
        const int64_t threads = count * (n / 2);
        cplx *src = dz, *dst = work;
        for (int64_t ns = 1; ns < n; ns *= 2) {
            const double scale = (inverse && ns * 2 == n) ? 1.0 / static_cast<double>(n) : 1.0;
            stockham_pass_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(src, dst, n, count, ns,
                                                                                            tw, inverse ? 1 : 0, scale);
            RL_CHECK_LAUNCH("stockham_pass_kernel");
            std::swap(src, dst);
        }
        if (src != dz) RL_CUDA(cudaMemcpyAsync(dz, src, count * n * 16, cudaMemcpyDeviceToDevice, s));
    } else {
        dft_dense_kernel<<<static_cast<unsigned>((count * n + 255) / 256), 256, 0, s>>>(dz, work, n, count, tw,
                                                                                        inverse ? 1 : 0);
        RL_CHECK_LAUNCH("dft_dense_kernel");
        RL_CUDA(cudaMemcpyAsync(dz, work, count * n * 16, cudaMemcpyDeviceToDevice, s));
    }
    return RL_OK;
}
}  // namespace rl

extern "C" RL_API rl_status rl_fft(rl_context* ctx, rl_mem mem, int64_t count, int64_t n, double* z, int32_t inverse) {
    if (n <= 0 || count < 0) return set_error(RL_ERR_DIMENSION, inverse ? "inverse_fft: empty input" : "fft: empty input");
    if (count == 0) return RL_OK;
    if (!z) return set_error(RL_ERR_INVALID_ARGUMENT, "fft: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    const int64_t bytes = count * n * 16;
    double* dz = z;
    double* work = nullptr;
    const size_t wb = cfft_work_bytes(count, n);
    bool ok = with_arena(ctx, [&](Arena& ar) {
        if (host) dz = ar.take<double>(2 * count * n);
        if (wb) work = ar.take<double>(2 * count * n);
    });
    if (!ok) return RL_ERR_OUT_OF_MEMORY;
    if (host) RL_CUDA(cudaMemcpyAsync(dz, z, bytes, cudaMemcpyHostToDevice, s));
    if ((st = cfft_device(ctx, count, n, dz, inverse != 0, work)) != RL_OK) return st;
    if (host) {
        RL_CUDA(cudaMemcpyAsync(z, dz, bytes, cudaMemcpyDeviceToHost, s));
        RL_CUDA(cudaStreamSynchronize(s));
    }
    return RL_OK;
}

// circulant_apply(C(c), x) (circulant.hpp:91-96): y^T = x^T C^T, one row
// through the circulant kernel with the transposed circulant's column
// (circulant.hpp:40-45); the dense expansion and a GEMV when the FFT kernel
// does not cover n. The transform of a real row is real by construction
// (r2c), so strip_imag's logic_error cannot arise (nor does it for real
// input in the reference).
extern "C" RL_API rl_status rl_circulant_apply(rl_context* ctx, rl_mem mem, int64_t n, const double* c,
                                               const double* x, double* y) {
    if (n <= 0) return set_error(RL_ERR_DIMENSION, "circulant_apply: length mismatch");
    if (!c || !x || !y) return set_error(RL_ERR_INVALID_ARGUMENT, "circulant_apply: null pointer");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    cudaStream_t s = ctx->stream;
    const bool host = mem == RL_HOST;
    std::vector<double> col(static_cast<size_t>(n)), colt(static_cast<size_t>(n));
    if (host)
        std::memcpy(col.data(), c, n * 8);
    else
        RL_CUDA(cudaMemcpy(col.data(), c, n * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) colt[i] = col[(n - i) % n];
    const bool fft_path = circulant_fft_ok(n);
    const int64_t ld = (n + 1) & ~int64_t(1);
    double *dct = nullptr, *dx = nullptr, *dy = nullptr, *dense = nullptr;
    void* spec = nullptr;
    bool ok = with_arena(ctx, [&](Arena& ar) {
        dct = ar.take<double>(n);
        dx = ar.take<double>(n);
        dy = ar.take<double>(n);
        if (fft_path)
            spec = ar.take<char>(n * 16);
        else
            dense = ar.take<double>(n * ld);
    });
    if (!ok) return RL_ERR_OUT_OF_MEMORY;
    RL_CUDA(cudaMemcpyAsync(dct, (fft_path ? colt : col).data(), n * 8, cudaMemcpyHostToDevice, s));
    RL_CUDA(cudaMemcpyAsync(dx, x, n * 8, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    if (fft_path) {
        st = circulant_rows(ctx, 1, n, dx, n, n, dct, n, dy, n, spec);
    } else {
        if ((st = circulant_dense(ctx, dct, n, n, n, dense, ld)) == RL_OK) st = gemv(ctx, n, n, dense, ld, dx, dy, nullptr);
    }
    if (st != RL_OK) return st;
    RL_CUDA(cudaMemcpyAsync(y, dy, n * 8, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    RL_CUDA(cudaStreamSynchronize(s));  // col / colt are locals
    return RL_OK;
}
