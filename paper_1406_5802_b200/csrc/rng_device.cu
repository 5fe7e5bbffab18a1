// Exact seeded Gaussian multipliers generated on the device.
//
// Same stream as rng_host.cpp / the reference (rng.hpp:16-85, multipliers.hpp:
// 58-65): polar attempt a uses draws 2a+1, 2a+2 of the splitmix64 stream,
// u = 2 d - 1, s = u*u + v*v (two roundings), accepted when 0 < s < 1, and the
// pair (u f, v f) with f = sqrt(-2 log(s) / s) fills outputs 2i, 2i+1 for the
// i-th accepted attempt. Everything except log(s) is integer work or a single
// correctly rounded IEEE operation, so the device reproduces it bit for bit
// (explicit __dmul_rn / __dadd_rn / __ddiv_rn / __dsqrt_rn: no contraction).
//
// log(s): the reference calls glibc's log, which is not correctly rounded but
// is documented to stay within 0.52 ulp of the exact value. The device
// evaluates log(s) in double-double (~2^-100 relative), rounds it, and
// measures the distance of the exact value from the rounded one: when it is
// below kSafe = 0.47 of the smaller neighbouring gap, every result within
// 0.53 ulp of the exact value is that same double, so glibc (documented bound
// 0.519 ulp; worst seen over 3.1e7 polar samples against a binary128 log:
// 0.5184) returns it too. The remaining attempts (6 %) are listed and finished on the host
// with glibc itself (rng_host.cpp: host_polar_pairs), then scattered back.
// The tests compare whole 8192 x 8192 matrices bit for bit against the host
// generator.
//
// Parallel layout: pass 1 counts accepted attempts per 4096-attempt block,
// one block scan gives every block its output offset, pass 2 regenerates
// each block (warp scans place each thread's pairs).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "device_common.cuh"
#include "kernels.cuh"

namespace rl {
// host side of the hard cases (rng_host.cpp, glibc log)
void host_polar_pairs(uint64_t seed, const uint64_t* attempts, int64_t count, double* out2);
uint64_t host_stream_state(uint64_t seed);
}  // namespace rl

namespace rl {
namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr int GT = 256;           // threads per block
constexpr int PER_THREAD = 16;    // attempts per thread
constexpr int PER_BLOCK = GT * PER_THREAD;
constexpr double kSafe = 0.47;

__device__ __forceinline__ uint64_t finalize(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double symmetric_at(uint64_t state0, uint64_t t) {
    const double d = __dmul_rn(static_cast<double>(finalize(state0 + t * kGamma) >> 11), 0x1.0p-53);
    return __dsub_rn(__dmul_rn(2.0, d), 1.0);
}

__device__ __forceinline__ bool attempt(uint64_t state0, uint64_t a, double& u, double& v, double& s) {
    u = symmetric_at(state0, 2 * a + 1);
    v = symmetric_at(state0, 2 * a + 2);
    s = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
    return !(s >= 1.0 || s == 0.0);
}

// ---- double-double arithmetic ------------------------------------------------
struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    const dd t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo = __fma_rn(a.hi, b.lo, __fma_rn(a.lo, b.hi, p.lo));
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo = __fma_rn(a.lo, b, p.lo);
    return quick_two_sum(p.hi, p.lo);
}
// a / b with a exact double, b double-double
__device__ __forceinline__ dd dd_div(double a, dd b) {
    const double q1 = __ddiv_rn(a, b.hi);
    // r = a - q1 * b
    dd p = dd_mul_d(b, q1);
    dd r = dd_add({a, 0.0}, {-p.hi, -p.lo});
    const double q2 = __ddiv_rn(r.hi, b.hi);
    p = dd_mul_d(b, q2);
    r = dd_add(r, {-p.hi, -p.lo});
    const double q3 = __ddiv_rn(r.hi, b.hi);
    dd q = quick_two_sum(q1, q2);
    return dd_add(q, {q3, 0.0});
}

// log(s) for s in (0, 1) in double-double: s = 2^k m, m in [sqrt(1/2), sqrt(2)),
// log m = 2 atanh(z), z = (m - 1) / (m + 1), |z| <= 0.1716
__device__ __forceinline__ dd log_dd(double s) {
    int k;
    double m = frexp(s, &k);  // m in [0.5, 1)
    if (m < 0.70710678118654752) {
        m = __dmul_rn(m, 2.0);
        --k;
    }
    const double num = __dsub_rn(m, 1.0);  // exact (Sterbenz)
    const dd den = two_sum(m, 1.0);        // exact
    const dd z = dd_div(num, den);
    const dd z2 = dd_mul(z, z);
    // atanh(z)/z = 1 + z2/3 + z2^2 T(z2), T(x) = sum_{j>=2} x^(j-2) / (2j+1);
    // the tail is below 2^-10 relative, so T in double is ample
    const double x = z2.hi;
    double t = 1.0 / 45.0;  // j = 22
#pragma unroll
    for (int j = 21; j >= 2; --j) t = __fma_rn(t, x, 1.0 / (2.0 * j + 1.0));
    const dd third = {0x1.5555555555555p-2, 0x1.5555555555555p-56};
    dd ser = dd_add({1.0, 0.0}, dd_mul(z2, third));
    ser = dd_add(ser, {__dmul_rn(__dmul_rn(x, x), t), 0.0});
    dd lm = dd_mul(z, ser);
    lm = {__dmul_rn(lm.hi, 2.0), __dmul_rn(lm.lo, 2.0)};
    if (k == 0) return lm;
    const dd ln2 = {0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
    return dd_add(dd_mul_d(ln2, static_cast<double>(k)), lm);
}

// glibc-equal log(s), or false when the exact value is too close to a
// rounding boundary to decide
__device__ __forceinline__ bool log_decided(double s, double& out) {
    const dd t = log_dd(s);
    const dd r = quick_two_sum(t.hi, t.lo);  // r.hi = round(t), r.lo = t - r.hi
    const double mag = fabs(r.hi);
    const double below = __dsub_rn(mag, __longlong_as_double(__double_as_longlong(mag) - 1));
    out = r.hi;
    return fabs(r.lo) < kSafe * below;
}

struct Pos {
    int64_t rows, cols, ld;
};
__device__ __forceinline__ int64_t where(const Pos& p, int64_t k) {
    if (p.ld == p.cols) return k;
    const int64_t i = k / p.cols;
    return i * p.ld + (k - i * p.cols);
}

__global__ void __launch_bounds__(GT) count_kernel(uint64_t state0, int64_t* __restrict__ counts) {
    const uint64_t a0 = (static_cast<uint64_t>(blockIdx.x) * GT + threadIdx.x) * PER_THREAD;
    int c = 0;
#pragma unroll 4
    for (int j = 0; j < PER_THREAD; ++j) {
        double u, v, s;
        c += attempt(state0, a0 + j, u, v, s) ? 1 : 0;
    }
    __shared__ int red[GT / 32];
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < GT / 32; ++w) t += red[w];
        counts[blockIdx.x] = t;
    }
}

// exclusive scan of counts[0..nb) into offsets[0..nb], offsets[nb] = total (one block)
__global__ void __launch_bounds__(1024) scan_kernel(const int64_t* __restrict__ counts, int64_t nb,
                                                    int64_t* __restrict__ offsets) {
    __shared__ int64_t part[1024];
    const int64_t per = (nb + 1023) / 1024;
    const int64_t lo = threadIdx.x * per, hi = min(nb, lo + per);
    int64_t sum = 0;
    for (int64_t i = lo; i < hi; ++i) sum += counts[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const int64_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    int64_t run = part[threadIdx.x] - sum;
    for (int64_t i = lo; i < hi; ++i) {
        offsets[i] = run;
        run += counts[i];
    }
    if (threadIdx.x == 1023) offsets[nb] = part[1023];
}

struct Hard {
    unsigned long long* count;
    uint64_t* attempt;   // attempt index
    int64_t* pair;       // output pair index
    int64_t cap;
};

__global__ void __launch_bounds__(GT) gen_kernel(uint64_t state0, const int64_t* __restrict__ offsets,
                                                 int64_t count, double* __restrict__ out, Pos pos, Hard hard,
                                                 int64_t block0) {
    const int64_t bx = block0 + blockIdx.x;
    const uint64_t a0 = (static_cast<uint64_t>(bx) * GT + threadIdx.x) * PER_THREAD;
    const int64_t pairs = (count + 1) / 2;
    const int64_t boff = offsets[bx];
    if (boff >= pairs) return;
    unsigned mask = 0;
#pragma unroll 4
    for (int j = 0; j < PER_THREAD; ++j) {
        double u, v, s;
        if (attempt(state0, a0 + j, u, v, s)) mask |= 1u << j;
    }
    // block-exclusive prefix of the per-thread accepted counts
    const int c = __popc(mask);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    __shared__ int wsum[GT / 32];
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int before = 0;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    int64_t idx = boff + before + incl - c;
    while (mask) {
        const int j = __ffs(mask) - 1;
        mask &= mask - 1;
        if (idx >= pairs) break;
        double u, v, s;
        attempt(state0, a0 + j, u, v, s);
        double lg;
        if (log_decided(s, lg)) {
            const double f = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, lg), s));
            out[where(pos, 2 * idx)] = __dmul_rn(u, f);
            if (2 * idx + 1 < count) out[where(pos, 2 * idx + 1)] = __dmul_rn(v, f);
        } else {
            const unsigned long long slot = atomicAdd(hard.count, 1ull);
            if (static_cast<int64_t>(slot) < hard.cap) {
                hard.attempt[slot] = a0 + j;
                hard.pair[slot] = idx;
            }
        }
        ++idx;
    }
}

__global__ void scatter_kernel(const int64_t* __restrict__ pair, const double* __restrict__ vals, int64_t n,
                               int64_t count, double* __restrict__ out, Pos pos) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = pair[i];
    out[where(pos, 2 * p)] = vals[2 * i];
    if (2 * p + 1 < count) out[where(pos, 2 * p + 1)] = vals[2 * i + 1];
}

}  // namespace

// Phase 1 (asynchronous): count, scan and generate on the context stream.
rl_status GaussJob::begin(rl_context* c, int64_t r, int64_t cl, uint64_t sd, double* o, int64_t l) {
    ctx = c;
    rows = r;
    cols = cl;
    seed = sd;
    out = o;
    ld = l;
    count = rows * cols;
    if (count <= 0) return RL_OK;
    const int64_t pairs = (count + 1) / 2;
    const uint64_t state0 = host_stream_state(seed);
    // attempts: expected pairs / (pi/4) plus 8 standard deviations plus one block
    const double need = static_cast<double>(pairs) / 0.78539816339744831 + 8.0 * std::sqrt(static_cast<double>(pairs)) +
                        PER_BLOCK;
    nb = static_cast<int64_t>(need / PER_BLOCK) + 1;
    cap = pairs / 12 + 4096;  // hard cases are 6% of the pairs; overflow falls back to the host
    cudaStream_t s = ctx->stream;
    const size_t bytes = align_up(8 * nb) + align_up(8 * (nb + 1)) + 256 + align_up(8 * cap) * 2 + align_up(16 * cap);
    RL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&base), bytes, s));
    size_t off = 0;
    auto take = [&](size_t b) {
        char* p = base + off;
        off += align_up(b);
        return p;
    };
    counts = reinterpret_cast<int64_t*>(take(8 * nb));
    offsets = reinterpret_cast<int64_t*>(take(8 * (nb + 1)));
    hcount = reinterpret_cast<unsigned long long*>(take(256));
    attempts = reinterpret_cast<uint64_t*>(take(8 * cap));
    pair = reinterpret_cast<int64_t*>(take(8 * cap));
    vals = reinterpret_cast<double*>(take(16 * cap));
    RL_CUDA(cudaMemsetAsync(hcount, 0, 8, s));
    count_kernel<<<static_cast<unsigned>(nb), GT, 0, s>>>(state0, counts);
    RL_CHECK_LAUNCH("count_kernel");
    scan_kernel<<<1, 1024, 0, s>>>(counts, nb, offsets);
    RL_CHECK_LAUNCH("scan_kernel");
    // pinned readback slots: the copies stay asynchronous. The generator runs
    // in two halves so the host can finish the first half's undecided
    // attempts while the second half generates.
    RL_CUDA(cudaMemcpyAsync(ctx->host_scalars + 0, offsets + nb, 8, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaMemcpyAsync(ctx->host_scalars + 3, offsets + nb / 2, 8, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaEventCreateWithFlags(&ev1, cudaEventDisableTiming));
    RL_CUDA(cudaEventCreateWithFlags(&ev2, cudaEventDisableTiming));
    nb1 = nb / 2;
    if (nb1 > 0) {
        gen_kernel<<<static_cast<unsigned>(nb1), GT, 0, s>>>(state0, offsets, count, out, Pos{rows, cols, ld},
                                                             Hard{hcount, attempts, pair, cap}, 0);
        RL_CHECK_LAUNCH("gen_kernel");
    }
    RL_CUDA(cudaMemcpyAsync(ctx->host_scalars + 2, hcount, 8, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaEventRecord(ev1, s));
    gen_kernel<<<static_cast<unsigned>(nb - nb1), GT, 0, s>>>(state0, offsets, count, out, Pos{rows, cols, ld},
                                                              Hard{hcount, attempts, pair, cap}, nb1);
    RL_CHECK_LAUNCH("gen_kernel");
    RL_CUDA(cudaMemcpyAsync(ctx->host_scalars + 1, hcount, 8, cudaMemcpyDeviceToHost, s));
    RL_CUDA(cudaEventRecord(ev2, s));
    return RL_OK;
}

// Phase 2: wait for the counts, finish the undecided attempts with glibc on
// the host and scatter them (synchronises the context stream).
rl_status GaussJob::finish(int64_t* hard_cases, const std::function<rl_status(int64_t)>& first_rows_ready) {
    if (count <= 0) return RL_OK;
    cudaStream_t s = ctx->stream;
    const int64_t pairs = (count + 1) / 2;
    // pinned staging for every possible hard case: attempt indices in, (u f, v f) out
    char* stage = static_cast<char*>(pinned_staging(ctx, 24 * static_cast<size_t>(cap)));
    uint64_t* att = stage ? reinterpret_cast<uint64_t*>(stage) : nullptr;
    double* hv = stage ? reinterpret_cast<double*>(stage + 8 * cap) : nullptr;
    // finish [lo, hi) of the hard list: attempts down (side stream `ds` when the
    // main stream is still generating), host logs, values up and scattered on
    // the main stream; in pipelined chunks
    cudaStream_t ds = nullptr;
    struct DsGuard {  // on every exit (errors included) the side stream's copies out of `attempts`
        cudaStream_t* p;  // finish before ~GaussJob frees it on the main stream
        ~DsGuard() {
            if (*p) {
                cudaStreamSynchronize(*p);
                cudaStreamDestroy(*p);
            }
        }
    } ds_guard{&ds};
    auto resolve = [&](int64_t lo, int64_t hi, cudaStream_t down, cudaStream_t up) -> rl_status {
        const int64_t nh = hi - lo;
        if (nh <= 0) return RL_OK;
        constexpr int kMaxChunks = 4;
        const int nchunks = nh >= 4 * 65536 ? kMaxChunks : 1;
        const int64_t cs = (nh + nchunks - 1) / nchunks;
        cudaEvent_t ev[kMaxChunks];
        for (int c = 0; c < nchunks; ++c) RL_CUDA(cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming));
        struct Ev {
            cudaEvent_t* e;
            int n;
            ~Ev() {
                for (int c = 0; c < n; ++c) cudaEventDestroy(e[c]);
            }
        } ev_guard{ev, nchunks};
        for (int c = 0; c < nchunks; ++c) {
            const int64_t o = lo + c * cs, k = std::min(cs, hi - o);
            RL_CUDA(cudaMemcpyAsync(att + o, attempts + o, 8 * k, cudaMemcpyDeviceToHost, down));
            RL_CUDA(cudaEventRecord(ev[c], down));
        }
        for (int c = 0; c < nchunks; ++c) {
            const int64_t o = lo + c * cs, k = std::min(cs, hi - o);
            RL_CUDA(cudaEventSynchronize(ev[c]));
            host_polar_pairs(seed, att + o, k, hv + 2 * o);
            RL_CUDA(cudaMemcpyAsync(vals + 2 * o, hv + 2 * o, 16 * k, cudaMemcpyHostToDevice, up));
            scatter_kernel<<<static_cast<unsigned>((k + 255) / 256), 256, 0, up>>>(pair + o, vals + 2 * o, k, count,
                                                                                   out, Pos{rows, cols, ld});
            RL_CHECK_LAUNCH("scatter_kernel");
        }
        return RL_OK;
    };
    rl_status st;
    int64_t done = 0;
    // first half, under the second half's generation
    RL_CUDA(cudaEventSynchronize(ev1));
    h_total = ctx->host_scalars[0];
    const int64_t n1 = ctx->host_scalars[2];
    if (stage && h_total >= pairs && n1 <= cap && n1 > 0) {
        RL_CUDA(cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking));
        RL_CUDA(cudaStreamWaitEvent(ds, ev1, 0));
        if ((st = resolve(0, n1, ds, s)) != RL_OK) return st;
        done = n1;
    }
    // rows [0, rows1) hold only first-half values, final in stream order now
    bool overlapped = false;
    if (first_rows_ready && stage && h_total >= pairs && n1 <= cap) {
        const int64_t half_vals = 2 * static_cast<int64_t>(ctx->host_scalars[3]);
        const int64_t rows1 = std::min<int64_t>(rows, half_vals / cols);
        if (rows1 > 0) {
            if ((st = first_rows_ready(rows1)) != RL_OK) return st;
            overlapped = true;
        }
    }
    RL_CUDA(cudaEventSynchronize(ev2));
    h_hard = static_cast<int64_t>(ctx->host_scalars[1]);
    if (!stage || h_total < pairs || h_hard > cap) {
        // astronomically unlikely: too few accepted attempts, or too many hard
        // cases for the list; generate on the host and upload (after, and so
        // over, anything already scattered)
        std::vector<double> hg(static_cast<size_t>(count));
        rl_gen_gaussian(rows, cols, seed, hg.data());
        RL_CUDA(cudaMemcpy2DAsync(out, ld * 8, hg.data(), cols * 8, cols * 8, rows, cudaMemcpyHostToDevice, s));
        RL_CUDA(cudaStreamSynchronize(s));
        if (hard_cases) *hard_cases = -1;
        return RL_OK;
    }
    if (hard_cases) *hard_cases = h_hard;
    // the second half's attempts also come down on the side stream: on the
    // main stream they would queue behind the first half's uploads, which
    // share the H2D engine with the caller's own uploads
    if (overlapped && !ds) RL_CUDA(cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking));
    if (overlapped) {
        // the main stream's GEMM fills every SM: the second half's scatter
        // must be scheduled ahead of its remaining CTAs, or it (and the host,
        // which waits for its copies) waits for the whole GEMM
        int lo_p = 0, hi_p = 0;
        cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p);
        cudaStream_t hs = nullptr;
        RL_CUDA(cudaStreamCreateWithPriority(&hs, cudaStreamNonBlocking, hi_p));
        RL_CUDA(cudaStreamWaitEvent(hs, ev2, 0));
        cudaStreamSynchronize(ds);  // ds only ever held the first half's attempt downloads
        cudaStreamDestroy(ds);
        ds = hs;
    }
    if (ds) RL_CUDA(cudaStreamWaitEvent(ds, ev2, 0));
    // the second half's values go up and scatter on the side stream when the
    // main stream already runs work queued by first_rows_ready (only the
    // rows >= rows1 they touch are not read by it), else on the main stream
    cudaStream_t up = overlapped ? ds : s;
    if ((st = resolve(done, h_hard, ds ? ds : s, up)) != RL_OK) return st;
    if (overlapped) {
        cudaEvent_t e_done;
        RL_CUDA(cudaEventCreateWithFlags(&e_done, cudaEventDisableTiming));
        RL_CUDA(cudaEventRecord(e_done, ds));
        RL_CUDA(cudaStreamWaitEvent(s, e_done, 0));
        // the staging buffer is reused by the next call: its copies must be done
        const cudaError_t e = cudaEventSynchronize(e_done);
        cudaEventDestroy(e_done);
        RL_CUDA(e);
        return RL_OK;
    }
    // the staging buffer is reused by the next call: the copies must be done
    RL_CUDA(cudaStreamSynchronize(s));
    return RL_OK;
}

GaussJob::~GaussJob() {
    if (base) cudaFreeAsync(base, ctx->stream);
    if (ev1) cudaEventDestroy(ev1);
    if (ev2) cudaEventDestroy(ev2);
}

rl_status gen_gaussian_device(rl_context* ctx, int64_t rows, int64_t cols, uint64_t seed, double* out, int64_t ld,
                              int64_t* hard_cases) {
    GaussJob job;
    rl_status st = job.begin(ctx, rows, cols, seed, out, ld);
    if (st != RL_OK) return st;
    return job.finish(hard_cases);
}

}  // namespace rl

extern "C" RL_API rl_status rl_gen_gaussian_device(rl_context* ctx, int64_t m, int64_t n, uint64_t seed, double* out,
                                                   int64_t ld, int64_t* hard_cases) {
    if (m <= 0 || n <= 0 || !out) return rl::set_error(RL_ERR_DIMENSION, "gen_gaussian_device: empty shape");
    if (ld < n) return rl::set_error(RL_ERR_DIMENSION, "gen_gaussian_device: ld < n");
    rl_status st;
    ctx = rl::resolve(ctx, &st);
    if (!ctx) return st;
    return rl::gen_gaussian_device(ctx, m, n, seed, out, ld, hard_cases);
}
