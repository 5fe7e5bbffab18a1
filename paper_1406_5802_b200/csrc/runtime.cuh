// Runtime plumbing shared by every entry point of librandla_b200.so:
// contexts (device + stream + grow-only device workspace), thread-local error
// messages, the kernel-launch counter and host<->device staging helpers.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <mutex>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/randla_capi.h"

struct rl_context {
    int device = 0;
    int num_sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    void* ws = nullptr;  // device workspace
    size_t ws_bytes = 0;
    void* flags = nullptr;  // small zero-initialised device scratch for verdicts / counters
    size_t flags_bytes = 0;
    // lookahead stream (high priority) and an event pool for intra-call
    // dependencies between it and `stream` (created on first use)
    cudaStream_t hi_stream = nullptr;
    // forward-substitution stream: y = L^-1 b follows the GENP panels (genp.cu)
    cudaStream_t fs_stream = nullptr;
    cudaEvent_t* events = nullptr;
    int num_events = 0;
    // grow-only pinned host staging: slot 0 the exact generator's hard cases,
    // slot 1 a pageable host A on its way to the device
    void* pinned[2] = {nullptr, nullptr};
    size_t pinned_bytes[2] = {0, 0};
    // 4 KiB pinned host scalars for asynchronous device->host readbacks
    int64_t* host_scalars = nullptr;
    // set around launches on a latency-bound chain of small kernels (the GENP
    // lookahead): gemm() then launches with programmatic stream serialization
    bool pdl = false;
};

namespace rl {

extern std::atomic<int64_t> g_launches;

rl_status set_error(rl_status st, const char* fmt, ...);
rl_status cuda_error(cudaError_t e, const char* what);

// Resolve ctx (NULL -> per-thread default context). Returns nullptr and sets
// the error when no device is present.
rl_context* resolve(rl_context* ctx, rl_status* st);

// Grow-only device workspace; returns nullptr on OOM (error already set).
void* workspace(rl_context* ctx, size_t bytes);

// Grow-only pinned host buffer `slot` (0 or 1) owned by the context (nullptr on failure).
void* pinned_staging(rl_context* ctx, size_t bytes, int slot = 0);

// memcpy on the host worker pool (all cores; serial when the pool is busy)
void host_parallel_copy(void* dst, const void* src, size_t bytes);

// High-priority side stream and at least `count` reusable timing-free events.
rl_status side_resources(rl_context* ctx, int count);

inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Check for an asynchronous launch error right after a launch.
#define RL_CHECK_LAUNCH(what)                                   \
    do {                                                        \
        ::rl::count_launch();                                   \
        cudaError_t e_ = cudaGetLastError();                    \
        if (e_ != cudaSuccess) return ::rl::cuda_error(e_, what); \
    } while (0)

#define RL_CUDA(call)                                            \
    do {                                                         \
        cudaError_t e_ = (call);                                 \
        if (e_ != cudaSuccess) return ::rl::cuda_error(e_, #call); \
    } while (0)

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// One-time per-device setup (kernel attributes such as the dynamic shared
// memory limit are per device): runs f() the first time for the current
// device, under a lock so that no caller launches before it has finished.
struct PerDeviceOnce {
    std::mutex mu;
    uint64_t done = 0;
};
template <typename F>
rl_status once_per_device(PerDeviceOnce& o, F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    std::lock_guard<std::mutex> lk(o.mu);
    if (o.done & bit) return RL_OK;
    const rl_status st = f();
    if (st == RL_OK) o.done |= bit;
    return st;
}

// Bump allocator over the context workspace for one call.
struct Arena {
    char* base = nullptr;
    size_t used = 0, cap = 0;
    template <typename T>
    T* take(size_t count) {
        size_t off = align_up(used);
        used = off + count * sizeof(T);
        return reinterpret_cast<T*>(base + off);
    }
};

// Two-phase arena sizing: pass 1 with base == nullptr measures, pass 2 carves.
template <typename F>
bool with_arena(rl_context* ctx, F&& carve) {
    Arena probe;
    carve(probe);
    void* p = workspace(ctx, probe.used + 256);
    if (!p) return false;
    Arena real;
    real.base = static_cast<char*>(p);
    real.cap = probe.used + 256;
    carve(real);
    return true;
}

}  // namespace rl
