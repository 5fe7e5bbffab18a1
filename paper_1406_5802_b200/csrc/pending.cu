// Entry points declared in include/randla_capi.h whose kernels are not in
// this build yet: they fail loudly with RL_ERR_UNSUPPORTED (never a CPU
// fallback). Each moves to its own translation unit when implemented.
#include "runtime.cuh"

#define RL_PENDING(name)                                                          \
    return rl::set_error(RL_ERR_UNSUPPORTED, "%s: not implemented in this build", name)

extern "C" {

}  // extern "C"
