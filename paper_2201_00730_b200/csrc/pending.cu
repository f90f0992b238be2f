// pending.cu -- entry points declared in include/uot_b200.h whose kernels are
// being brought up; they fail loudly (never a CPU fallback).
#include "../../include/uot_b200.h"
#include "common.cuh"

#define UOT_PENDING(name)                                         \
  do {                                                            \
    uot::set_error("%s: not implemented in this build", name);   \
    return uot::UOT_INVALID;                                      \
  } while (0)

extern "C" {
int uot_mot1d_workspace_size(int32_t, int32_t, int32_t, size_t*) {
  UOT_PENDING("uot_mot1d_workspace_size");
}
int uot_mot1d_batched(int32_t, int32_t, int32_t, const double*, const double*, const double*,
                      double*, int32_t*, double*, int32_t*, int32_t*, void*, size_t, void*) {
  UOT_PENDING("uot_mot1d_batched");
}
int uot_bary_workspace_size(const uot_bary_desc*, size_t*) { UOT_PENDING("uot_bary_workspace_size"); }
int uot_bary_run(const uot_bary_desc*, void*, size_t, void*) { UOT_PENDING("uot_bary_run"); }
}
