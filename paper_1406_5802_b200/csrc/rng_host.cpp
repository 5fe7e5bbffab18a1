// Exact seeded multiplier generation on the host, parallel across cores.
//
// The reference draws every multiplier from one sequential RngStream
// (rng.hpp:16-85): splitmix64 counter steps, Marsaglia polar Gaussians
// (rng.hpp:56-71), entry (i, j) of gen_gaussian = draw i*n + j
// (multipliers.hpp:58-65). Device generation cannot be bit-exact because
// glibc's log is not correctly rounded (SURVEY §0 finding 6), so the
// multipliers are generated here, bit-identical to the reference, and
// uploaded.
//
// Parallelisation without changing a single bit: draw t of a stream is
// finalize(state0 + t * gamma), so polar attempt a (draws 2a+1, 2a+2) can be
// evaluated at any index. Pass 1 counts accepted attempts per chunk (integer
// ops and one exact compare, no log); a prefix sum gives every chunk its
// output offset; pass 2 generates the chunks independently.
//
// Compiled with -ffp-contract=off and no -march flags: u*u + v*v and the
// polar factor round exactly as in the reference's x86-64 build.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <mutex>
#include <condition_variable>
#include <functional>
#include <new>
#include <pthread.h>
#include <complex>
#include <vector>

#include "../../include/randla_capi.h"

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

inline uint64_t finalize(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// rng.hpp:74-80
inline uint64_t mix_key(uint64_t state, uint64_t key) {
    state ^= key + kGamma + (state << 6) + (state >> 2);
    return finalize(state + kGamma);
}

inline uint64_t stream_state(uint64_t seed) { return mix_key(kGamma, seed); }  // rng.hpp:18

// rng.hpp:40-43: uniform on [-1, 1] from draw number t (1-based) of the stream
inline double symmetric_at(uint64_t state0, uint64_t t) {
    const double d = static_cast<double>(finalize(state0 + t * kGamma) >> 11) * 0x1.0p-53;
    return 2.0 * d - 1.0;
}

// polar attempt a: accepted when 0 < s < 1 (rng.hpp:61-66)
inline bool attempt(uint64_t state0, uint64_t a, double& u, double& v, double& s) {
    u = symmetric_at(state0, 2 * a + 1);
    v = symmetric_at(state0, 2 * a + 2);
    s = u * u + v * v;
    return !(s >= 1.0 || s == 0.0);
}

int g_threads = 0;

int thread_count() {
    int t = g_threads > 0 ? g_threads : static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, t);
}

// Persistent worker pool: parallel_for hands out indices to workers that
// stay alive between calls (spawning threads per call costs ~0.3 ms, a
// noticeable share of the device generator's host-decided tail). Every pool
// thread joins every call; the caller drains too.
// The pool is per process: a forked child (pthread_atfork handler below)
// starts a fresh one instead of waiting on the parent's threads, which do not
// exist in the child; the parent's pool object is abandoned there, never
// joined. A caller that finds the pool busy with another caller's call runs
// its own indices itself instead of queueing behind it.
class Pool;
std::atomic<Pool*> g_pool{nullptr};
std::mutex g_pool_mu;

class Pool {
  public:
    static Pool& get() {
        static const bool registered = [] {
            pthread_atfork(nullptr, nullptr, [] {
                new (&g_pool_mu) std::mutex();  // the child has one thread: nothing can hold it
                g_pool.store(nullptr);
            });
            return true;
        }();
        (void)registered;
        Pool* p = g_pool.load();
        if (p) return *p;
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (!g_pool.load()) g_pool.store(new Pool());  // never destroyed: workers die with the process
        return *g_pool.load();
    }
    void run(int helpers, int64_t count, const std::function<void(int64_t)>& fn) {
        std::unique_lock<std::mutex> call(call_mu_, std::try_to_lock);  // one parallel_for at a time
        if (!call.owns_lock()) {
            for (int64_t i = 0; i < count; ++i) fn(i);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            while (static_cast<int>(threads_.size()) < helpers) threads_.emplace_back([this] { loop(); });
            fn_ = &fn;
            count_ = count;
            next_.store(0);
            pending_ = static_cast<int>(threads_.size());
            ++gen_;
        }
        cv_.notify_all();
        drain();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

  private:
    void drain() {
        for (int64_t i = next_.fetch_add(1); i < count_; i = next_.fetch_add(1)) (*fn_)(i);
    }
    void loop() {
        uint64_t seen = 0;
        {
            std::lock_guard<std::mutex> lk(mu_);
            seen = gen_ - 1;  // created for the call in progress: join it
        }
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            drain();
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }

    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> threads_;
    const std::function<void(int64_t)>* fn_ = nullptr;
    int64_t count_ = 0;
    std::atomic<int64_t> next_{0};
    int pending_ = 0;
    uint64_t gen_ = 1;
    bool stop_ = false;  // never set: the pool lives as long as the process
};

template <typename F>
void parallel_for(int64_t count, F&& fn) {
    const int workers = static_cast<int>(std::min<int64_t>(thread_count(), count));
    if (workers <= 1) {
        for (int64_t i = 0; i < count; ++i) fn(i);
        return;
    }
    const std::function<void(int64_t)> f = [&](int64_t i) { fn(i); };
    Pool::get().run(workers - 1, count, f);
}

// Sequential generator (small matrices): exactly RngStream::next_gaussian,
// from a stream state (stream_state(seed), or a derived stream's)
void gaussian_from_state(uint64_t s0, int64_t count, double* out) {
    uint64_t a = 0;
    int64_t k = 0;
    while (k < count) {
        double u, v, s;
        if (!attempt(s0, a++, u, v, s)) continue;
        const double f = std::sqrt(-2.0 * std::log(s) / s);
        out[k++] = u * f;
        if (k < count) out[k++] = v * f;
    }
}

void gaussian_sequential(uint64_t seed, int64_t count, double* out) { gaussian_from_state(stream_state(seed), count, out); }

constexpr int64_t kChunk = 1 << 16;  // polar attempts per chunk

void gaussian_parallel(uint64_t seed, int64_t count, double* out) {
    const int64_t pairs_needed = (count + 1) / 2;
    if (count <= 4 * kChunk || thread_count() == 1) {
        gaussian_sequential(seed, count, out);
        return;
    }
    const uint64_t s0 = stream_state(seed);
    std::vector<int64_t> accepted;
    int64_t have = 0;
    while (have < pairs_needed) {
        // enough chunks for the remaining pairs at acceptance pi/4, plus slack
        const int64_t base = static_cast<int64_t>(accepted.size());
        const int64_t more = static_cast<int64_t>((pairs_needed - have) / (kChunk * 0.78539816)) + 2;
        accepted.resize(base + more);
        parallel_for(more, [&](int64_t i) {
            const uint64_t a0 = static_cast<uint64_t>(base + i) * kChunk;
            int64_t c = 0;
            for (int64_t j = 0; j < kChunk; ++j) {
                double u, v, s;
                c += attempt(s0, a0 + j, u, v, s) ? 1 : 0;
            }
            accepted[base + i] = c;
        });
        have = 0;
        for (int64_t c : accepted) have += c;
    }
    std::vector<int64_t> offset(accepted.size() + 1, 0);
    for (size_t i = 0; i < accepted.size(); ++i) offset[i + 1] = offset[i] + accepted[i];
    int64_t chunks = 0;
    while (offset[chunks] < pairs_needed) ++chunks;
    parallel_for(chunks, [&](int64_t i) {
        const uint64_t a0 = static_cast<uint64_t>(i) * kChunk;
        int64_t k = 2 * offset[i];
        for (int64_t j = 0; j < kChunk && k < count; ++j) {
            double u, v, s;
            if (!attempt(s0, a0 + j, u, v, s)) continue;
            const double f = std::sqrt(-2.0 * std::log(s) / s);
            out[k++] = u * f;
            if (k < count) out[k++] = v * f;
        }
    });
}

}  // namespace

namespace rl {
uint64_t host_stream_state(uint64_t seed) { return stream_state(seed); }

// ---- complex families' host draws (multipliers.hpp:75-138), sequential on
// one stream and rounded exactly as the reference (glibc cos/sin through
// std::polar, no FMA contraction) ------------------------------------------
namespace {
constexpr double kTwoPi = 2.0 * 3.141592653589793;  // 2.0 * std::numbers::pi
struct SeqStream {  // RngStream::next_u64 / next_double / next_below (rng.hpp:30-53)
    uint64_t s0, t = 0;
    explicit SeqStream(uint64_t seed) : s0(stream_state(seed)) {}
    uint64_t next_u64() { return finalize(s0 + (++t) * kGamma); }
    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    uint64_t next_below(uint64_t bound) {
        const uint64_t limit = bound * ((~uint64_t{0}) / bound);
        uint64_t v;
        do {
            v = next_u64();
        } while (v >= limit);
        return v % bound;
    }
};
// sample_without_replacement (multipliers.hpp:112-121)
void sample_columns(SeqStream& rng, int64_t n, int64_t l, int64_t* out) {
    std::vector<int64_t> pool(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) pool[i] = i;
    for (int64_t i = 0; i < l; ++i) {
        const int64_t j = i + static_cast<int64_t>(rng.next_below(static_cast<uint64_t>(n - i)));
        std::swap(pool[i], pool[j]);
    }
    std::sort(pool.begin(), pool.begin() + l);
    std::copy(pool.begin(), pool.begin() + l, out);
}
}  // namespace

// spectrum of gen_unitary_circulant (multipliers.hpp:77-82): u_j =
// polar(1, 2 pi phi_j), phi_j = next_double draws 1..n; u2 interleaved
void host_unit_spectrum(uint64_t seed, int64_t n, double* u2) {
    SeqStream rng(seed);
    for (int64_t j = 0; j < n; ++j) {
        const std::complex<double> u = std::polar(1.0, kTwoPi * rng.next_double());
        u2[2 * j] = u.real();
        u2[2 * j + 1] = u.imag();
    }
}

// srft_columns (multipliers.hpp:132-138)
void host_srft_columns(uint64_t seed, int64_t n, int64_t l, int64_t* cols) {
    SeqStream rng(seed);
    for (int64_t i = 0; i < n; ++i) rng.next_double();
    sample_columns(rng, n, l, cols);
}

// the parts of gen_srft(n, l, seed) (multipliers.hpp:94-130): d_i = sqrt(n/l)
// polar(1, 2 pi phi_i), root_k = polar(1, 2 pi k / n), the sampled columns;
// entry (i, j) = d_i * root[(i cols_j) mod n]
void host_srft_parts(uint64_t seed, int64_t n, int64_t l, double* d2, double* root2, int64_t* cols) {
    SeqStream rng(seed);
    std::vector<double> phases(static_cast<size_t>(n));
    for (double& p : phases) p = rng.next_double();
    sample_columns(rng, n, l, cols);
    const double scale = std::sqrt(static_cast<double>(n) / static_cast<double>(l));
    for (int64_t i = 0; i < n; ++i) {
        const std::complex<double> d = scale * std::polar(1.0, kTwoPi * phases[i]);
        d2[2 * i] = d.real();
        d2[2 * i + 1] = d.imag();
        const std::complex<double> r = std::polar(1.0, kTwoPi * static_cast<double>(i) / static_cast<double>(n));
        root2[2 * i] = r.real();
        root2[2 * i + 1] = r.imag();
    }
}

void host_parallel_copy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kPiece = size_t(4) << 20;
    const int64_t pieces = static_cast<int64_t>((bytes + kPiece - 1) / kPiece);
    parallel_for(pieces, [&](int64_t i) {
        const size_t off = static_cast<size_t>(i) * kPiece;
        std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, std::min(kPiece, bytes - off));
    });
}

// finish listed polar attempts with glibc's log (rng_device.cu hard cases):
// out2[2i], out2[2i+1] = u f, v f of attempt attempts[i]
void host_polar_pairs(uint64_t seed, const uint64_t* attempts, int64_t count, double* out2) {
    const uint64_t s0 = stream_state(seed);
    constexpr int64_t kGroup = 4096;
    parallel_for((count + kGroup - 1) / kGroup, [&](int64_t g) {
        const int64_t hi = std::min(count, (g + 1) * kGroup);
        for (int64_t i = g * kGroup; i < hi; ++i) {
            double u, v, s;
            attempt(s0, attempts[i], u, v, s);
            const double f = std::sqrt(-2.0 * std::log(s) / s);
            out2[2 * i] = u * f;
            out2[2 * i + 1] = v * f;
        }
    });
}
}  // namespace rl

extern "C" {

RL_API void rl_set_host_threads(int threads) { g_threads = threads; }

// multipliers.hpp:54-56: RngStream(seed).derived(k1, k2).next_u64()
RL_API uint64_t rl_derive_seed(uint64_t seed, uint64_t k1, uint64_t k2) {
    const uint64_t st = mix_key(mix_key(stream_state(seed), k1), k2);
    return finalize(st + kGamma);
}

// rng.hpp:87-95
RL_API uint64_t rl_hash_label(const char* s) {
    uint64_t h = 1469598103934665603ull;
    for (; *s; ++s) {
        h ^= static_cast<uint64_t>(static_cast<unsigned char>(*s));
        h *= 1099511628211ull;
    }
    return h;
}

// `count` next_gaussian draws of RngStream(seed).derived(key) (rng.hpp:20-24),
// the probe vectors of posterior_estimate (lowrank.hpp:177-196)
RL_API rl_status rl_gen_gaussian_derived(uint64_t seed, uint64_t key, int64_t count, double* out) {
    if (count <= 0 || !out) return RL_ERR_DIMENSION;
    gaussian_from_state(mix_key(stream_state(seed), key), count, out);
    return RL_OK;
}

// polar(1, 2 pi k / n) for k < n (fft.hpp:21-30, multipliers.hpp:98-100)
RL_API rl_status rl_unit_roots(int64_t n, double* out) {
    if (n <= 0 || !out) return RL_ERR_DIMENSION;
    for (int64_t k = 0; k < n; ++k) {
        const std::complex<double> r = std::polar(1.0, 2.0 * 3.141592653589793 * static_cast<double>(k) /
                                                           static_cast<double>(n));
        out[2 * k] = r.real();
        out[2 * k + 1] = r.imag();
    }
    return RL_OK;
}

RL_API rl_status rl_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double* out) {
    if (m <= 0 || n <= 0 || !out) return RL_ERR_DIMENSION;
    gaussian_parallel(seed, m * n, out);
    return RL_OK;
}

RL_API rl_status rl_gen_gaussian_batch(int64_t count, int64_t m, int64_t n, const uint64_t* seeds, double* out) {
    if (count < 0 || m <= 0 || n <= 0 || (count > 0 && (!out || !seeds))) return RL_ERR_DIMENSION;
    const int64_t per = m * n;
    constexpr int64_t kGroup = 256;
    parallel_for((count + kGroup - 1) / kGroup, [&](int64_t g) {
        const int64_t hi = std::min(count, (g + 1) * kGroup);
        for (int64_t i = g * kGroup; i < hi; ++i) gaussian_sequential(seeds[i], per, out + i * per);
    });
    return RL_OK;
}

// multipliers.hpp:67-73: next_symmetric draws 1..n
RL_API rl_status rl_gen_real_circulant_column(int64_t n, uint64_t seed, double* out) {
    if (n <= 0 || !out) return RL_ERR_DIMENSION;
    const uint64_t s0 = stream_state(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = symmetric_at(s0, static_cast<uint64_t>(i) + 1);
    return RL_OK;
}

// gen_finite_set_uniform (multipliers.hpp:142-154): entry (i, j) is the
// (i n + j)-th next_below(card) of one stream, minus floor(card / 2).
// next_below rejects draws >= card * floor((2^64 - 1) / card) (rng.hpp:46-53),
// so the draw -> entry map is data-dependent; as for the Gaussians, pass 1
// counts the accepted draws per chunk, a prefix sum places every chunk, and
// pass 2 fills the chunks independently (bit-identical to the sequence).
RL_API rl_status rl_gen_finite_set_uniform(int64_t m, int64_t n, uint64_t seed, uint64_t card, double* out) {
    if (m <= 0 || n <= 0 || !out || card < 2) return RL_ERR_DIMENSION;
    const uint64_t s0 = stream_state(seed);
    const uint64_t limit = card * (~uint64_t{0} / card);
    const int64_t offset = static_cast<int64_t>(card / 2);
    const int64_t count = m * n;
    constexpr int64_t kDraws = 1 << 16;
    auto draw = [&](uint64_t t) { return finalize(s0 + t * kGamma); };  // draw t (1-based) of the stream
    std::vector<int64_t> accepted;
    int64_t have = 0;
    while (have < count) {
        const int64_t base = static_cast<int64_t>(accepted.size());
        const int64_t more = (count - have) / kDraws + 2;
        accepted.resize(base + more);
        parallel_for(more, [&](int64_t i) {
            const uint64_t t0 = static_cast<uint64_t>(base + i) * kDraws + 1;
            int64_t c = 0;
            for (int64_t j = 0; j < kDraws; ++j) c += draw(t0 + j) < limit ? 1 : 0;
            accepted[base + i] = c;
        });
        have = 0;
        for (int64_t c : accepted) have += c;
    }
    std::vector<int64_t> start(accepted.size() + 1, 0);
    for (size_t i = 0; i < accepted.size(); ++i) start[i + 1] = start[i] + accepted[i];
    int64_t chunks = 0;
    while (start[chunks] < count) ++chunks;
    parallel_for(chunks, [&](int64_t i) {
        const uint64_t t0 = static_cast<uint64_t>(i) * kDraws + 1;
        int64_t k = start[i];
        for (int64_t j = 0; j < kDraws && k < count; ++j) {
            const uint64_t v = draw(t0 + j);
            if (v >= limit) continue;
            out[k++] = static_cast<double>(static_cast<int64_t>(v % card) - offset);
        }
    });
    return RL_OK;
}

}  // extern "C"
