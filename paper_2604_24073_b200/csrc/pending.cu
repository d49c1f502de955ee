// Entry points whose implementation lands in engine.cu / partition.cu.
#include "capi_util.cuh"

extern "C" {
#define FSX_PENDING(sig)                                         \
  sig {                                                          \
    fsx::capi_set_error("fsx: not implemented in this build");   \
    return FSX_ERR_CONFIG;                                       \
  }
FSX_PENDING(int fsx_engine_create(fsx_ctx*, fsx_table*, const fsx_engine_config*, fsx_engine**))
FSX_PENDING(int fsx_engine_destroy(fsx_engine*))
FSX_PENDING(int fsx_engine_connect_local(fsx_engine*, int, fsx_engine*))
FSX_PENDING(int fsx_engine_export(fsx_engine*, void*, uint64_t*))
FSX_PENDING(int fsx_engine_connect_ipc(fsx_engine*, int, const void*, uint64_t))
FSX_PENDING(int fsx_nccl_unique_id(void*))
FSX_PENDING(int fsx_engine_connect_nccl(fsx_engine*, const void*))
FSX_PENDING(int fsx_engine_forward(fsx_engine*, const uint64_t*, uint64_t, const uint64_t*, uint64_t, void*, void*))
FSX_PENDING(int fsx_engine_backward(fsx_engine*, const void*, void*))
FSX_PENDING(int fsx_engine_finalize(fsx_engine*, void*))
FSX_PENDING(int fsx_engine_stats(fsx_engine*, int, uint64_t*))
FSX_PENDING(int fsx_engine_exposed_ms(fsx_engine*, double*))
FSX_PENDING(int fsx_cost_estimate(fsx_ctx*, const uint64_t*, const uint64_t*, int, double, double, double, double*, void*))
FSX_PENDING(int fsx_fbs_partition(fsx_ctx*, const uint64_t*, const int32_t*, const int32_t*, uint64_t, int, int32_t*, uint64_t*, void*))
FSX_PENDING(int fsx_vbs_partition(fsx_ctx*, const uint64_t*, const int32_t*, const int32_t*, uint64_t, int, double, const int32_t*, int32_t*, int32_t*, uint64_t*, void*))
FSX_PENDING(int fsx_autotune_update(int, int32_t*, double*, double*, int, double, double, const double*))
FSX_PENDING(int fsx_a2a_ce(fsx_engine*, const void*, const uint64_t*, const uint64_t*, void*, uint64_t, uint64_t*, void*))
uint64_t fsx_engine_slot_bytes(const fsx_engine*) { return 0; }
}
