// Entry points declared in include/randla_capi.h whose kernels are not in
// this build yet: they fail loudly with RL_ERR_UNSUPPORTED (never a CPU
// fallback). Each moves to its own translation unit when implemented.
#include "runtime.cuh"

#define RL_PENDING(name)                                                          \
    return rl::set_error(RL_ERR_UNSUPPORTED, "%s: not implemented in this build", name)

extern "C" {

RL_API rl_status rl_cholqr2(rl_context*, rl_mem, int64_t, int64_t, const double*, double*, double*, int64_t*) {
    RL_PENDING("rl_cholqr2");
}

RL_API rl_status rl_range_find_residual(rl_context*, rl_mem, int64_t, int64_t, const double*, int64_t,
                                        const rl_multiplier*, double*, rl_lowrank_info*) {
    RL_PENDING("rl_range_find_residual");
}

}  // extern "C"
