// Context management, errors and launch accounting for the C ABI
// (include/randla_capi.h).
#include <cstring>
#include <unistd.h>
#include <mutex>
#include <vector>

#include "runtime.cuh"

namespace rl {

std::atomic<int64_t> g_launches{0};

static thread_local std::string t_error;

rl_status set_error(rl_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    t_error = buf;
    return st;
}

rl_status cuda_error(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) return set_error(RL_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
        return set_error(RL_ERR_NO_DEVICE, "%s: %s", what, cudaGetErrorString(e));
    return set_error(RL_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

static rl_status init_context(rl_context* c, int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return set_error(RL_ERR_NO_DEVICE, "no CUDA device available (librandla_b200 has no CPU fallback)");
    if (device < 0 || device >= count) return set_error(RL_ERR_INVALID_ARGUMENT, "device %d out of range", device);
    RL_CUDA(cudaSetDevice(device));
    c->device = device;
    RL_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    RL_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    c->flags_bytes = 4096;
    RL_CUDA(cudaMalloc(&c->flags, c->flags_bytes));
    RL_CUDA(cudaMemset(c->flags, 0, c->flags_bytes));
    RL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->host_scalars), 4096, cudaHostAllocDefault));
    // call-scoped scratch comes from cudaMallocAsync: keep up to 2 GiB of the
    // pool mapped between calls instead of returning it at every synchronisation
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = uint64_t(2) << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    return RL_OK;
}

static void destroy_context(rl_context* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->ws) cudaFree(c->ws);
    if (c->flags) cudaFree(c->flags);
    for (void* p : c->pinned)
        if (p) cudaFreeHost(p);
    if (c->host_scalars) cudaFreeHost(c->host_scalars);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    if (c->hi_stream) cudaStreamDestroy(c->hi_stream);
    if (c->fs_stream) cudaStreamDestroy(c->fs_stream);
    for (int i = 0; i < c->num_events; ++i) cudaEventDestroy(c->events[i]);
    delete[] c->events;
    delete c;
}

// Per-thread default contexts, one per (thread, device): a NULL context
// resolves to the calling thread's context for its CURRENT device
// (cudaGetDevice), so one process per GPU (torch.cuda.set_device(local_rank))
// and threads that switch devices both land on the right GPU. They come from a
// process-wide pool keyed by device: a thread that exits hands its contexts
// back (no CUDA calls at thread exit), so callers that spawn fresh worker
// threads per call (parallel_for_index, parallel.hpp:14-35) reuse streams and
// workspaces instead of leaking them.
static constexpr int kMaxDevices = 64;
static std::mutex g_pool_mu;
static std::vector<rl_context*>* g_pool = new std::vector<rl_context*>[kMaxDevices];  // intentionally leaked
static pid_t g_pool_pid = getpid();

struct ThreadDefault {
    rl_context* ctx[kMaxDevices] = {};
    pid_t pid = getpid();
    ~ThreadDefault() {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (pid != getpid() || g_pool_pid != pid) return;  // forked child: the parent's contexts are not ours
        for (int d = 0; d < kMaxDevices; ++d)
            if (ctx[d]) g_pool[d].push_back(ctx[d]);
    }
};
static thread_local ThreadDefault t_default;

rl_context* resolve(rl_context* ctx, rl_status* st) {
    *st = RL_OK;
    if (ctx) {
        cudaSetDevice(ctx->device);
        return ctx;
    }
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *st = set_error(RL_ERR_NO_DEVICE, "no CUDA device available (librandla_b200 has no CPU fallback)");
        return nullptr;
    }
    if (dev < 0 || dev >= kMaxDevices) {
        *st = set_error(RL_ERR_INVALID_ARGUMENT, "device %d beyond the supported %d", dev, kMaxDevices);
        return nullptr;
    }
    if (t_default.pid != getpid()) {  // a forked child inherits the parent's thread-local pointers: drop them
        for (int d = 0; d < kMaxDevices; ++d) t_default.ctx[d] = nullptr;
        t_default.pid = getpid();
    }
    rl_context*& mine = t_default.ctx[dev];
    if (!mine) {
        {
            std::lock_guard<std::mutex> lk(g_pool_mu);
            if (g_pool_pid != getpid()) {  // contexts pooled by the parent process are unusable here
                for (int d = 0; d < kMaxDevices; ++d) g_pool[d].clear();
                g_pool_pid = getpid();
            }
            if (!g_pool[dev].empty()) {
                mine = g_pool[dev].back();
                g_pool[dev].pop_back();
            }
        }
        if (!mine) {
            rl_context* c = new rl_context();
            rl_status s = init_context(c, dev);
            if (s != RL_OK) {
                delete c;
                *st = s;
                return nullptr;
            }
            mine = c;
        }
    }
    return mine;
}

rl_status side_resources(rl_context* ctx, int count) {
    if (!ctx->hi_stream) {
        int lo = 0, hi = 0;
        RL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        RL_CUDA(cudaStreamCreateWithPriority(&ctx->hi_stream, cudaStreamNonBlocking, hi));
        RL_CUDA(cudaStreamCreateWithPriority(&ctx->fs_stream, cudaStreamNonBlocking, hi));
    }
    if (ctx->num_events < count) {
        cudaEvent_t* ev = new cudaEvent_t[count];
        for (int i = 0; i < ctx->num_events; ++i) ev[i] = ctx->events[i];
        for (int i = ctx->num_events; i < count; ++i) RL_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        delete[] ctx->events;
        ctx->events = ev;
        ctx->num_events = count;
    }
    return RL_OK;
}

void* pinned_staging(rl_context* ctx, size_t bytes, int slot) {
    if (bytes <= ctx->pinned_bytes[slot]) return ctx->pinned[slot];
    cudaStreamSynchronize(ctx->stream);
    if (ctx->hi_stream) cudaStreamSynchronize(ctx->hi_stream);
    if (ctx->fs_stream) cudaStreamSynchronize(ctx->fs_stream);
    if (ctx->pinned[slot]) cudaFreeHost(ctx->pinned[slot]);
    ctx->pinned[slot] = nullptr;
    ctx->pinned_bytes[slot] = 0;
    const size_t want = align_up(bytes, size_t(1) << 20);
    if (cudaHostAlloc(&ctx->pinned[slot], want, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        ctx->pinned[slot] = nullptr;
        return nullptr;
    }
    ctx->pinned_bytes[slot] = want;
    return ctx->pinned[slot];
}

void* workspace(rl_context* ctx, size_t bytes) {
    if (bytes <= ctx->ws_bytes) return ctx->ws;
    cudaStreamSynchronize(ctx->stream);
    if (ctx->ws) cudaFree(ctx->ws);
    ctx->ws = nullptr;
    ctx->ws_bytes = 0;
    size_t want = align_up(bytes, size_t(1) << 20);
    cudaError_t e = cudaMalloc(&ctx->ws, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        ctx->ws = nullptr;
        cuda_error(e, "workspace allocation");
        return nullptr;
    }
    ctx->ws_bytes = want;
    return ctx->ws;
}

}  // namespace rl

extern "C" {

RL_API int rl_abi_version(void) { return RL_ABI_VERSION; }

RL_API const char* rl_last_error(void) { return rl::t_error.c_str(); }

RL_API rl_status rl_context_create(int device, rl_context** out) {
    if (!out) return rl::set_error(RL_ERR_INVALID_ARGUMENT, "rl_context_create: null out");
    rl_context* c = new rl_context();
    rl_status st = rl::init_context(c, device);
    if (st != RL_OK) {
        delete c;
        *out = nullptr;
        return st;
    }
    *out = c;
    return RL_OK;
}

RL_API rl_status rl_context_destroy(rl_context* ctx) {
    rl::destroy_context(ctx);
    return RL_OK;
}

RL_API rl_status rl_context_set_stream(rl_context* ctx, void* s) {
    rl_status st;
    ctx = rl::resolve(ctx, &st);
    if (!ctx) return st;
    ctx->stream = static_cast<cudaStream_t>(s);  // NULL = the legacy default stream
    return RL_OK;
}

RL_API void* rl_context_get_stream(rl_context* ctx) {
    rl_status st;
    ctx = rl::resolve(ctx, &st);
    return ctx ? static_cast<void*>(ctx->stream) : nullptr;
}

RL_API rl_status rl_synchronize(rl_context* ctx) {
    rl_status st;
    ctx = rl::resolve(ctx, &st);
    if (!ctx) return st;
    RL_CUDA(cudaStreamSynchronize(ctx->stream));
    return RL_OK;
}

RL_API int64_t rl_kernel_launches(void) { return rl::g_launches.load(); }

RL_API int rl_context_device(rl_context* ctx) {
    rl_status st;
    ctx = rl::resolve(ctx, &st);
    return ctx ? ctx->device : -1;
}

}  // extern "C"
