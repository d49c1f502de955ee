// Entry points whose implementation lands in engine.cu / partition.cu.
#include "capi_util.cuh"

extern "C" {
#define FSX_PENDING(sig)                                         \
  sig {                                                          \
    fsx::capi_set_error("fsx: not implemented in this build");   \
    return FSX_ERR_CONFIG;                                       \
  }
FSX_PENDING(int fsx_cost_estimate(fsx_ctx*, const uint64_t*, const uint64_t*, int, double, double, double, double*, void*))
FSX_PENDING(int fsx_fbs_partition(fsx_ctx*, const uint64_t*, const int32_t*, const int32_t*, uint64_t, int, int32_t*, uint64_t*, void*))
FSX_PENDING(int fsx_vbs_partition(fsx_ctx*, const uint64_t*, const int32_t*, const int32_t*, uint64_t, int, double, const int32_t*, int32_t*, int32_t*, uint64_t*, void*))
FSX_PENDING(int fsx_autotune_update(int, int32_t*, double*, double*, int, double, double, const double*))
FSX_PENDING(int fsx_a2a_ce(fsx_engine*, const void*, const uint64_t*, const uint64_t*, void*, uint64_t, uint64_t*, void*))
}
