// C-ABI plumbing: every extern "C" entry point runs inside FSX_API_BEGIN /
// FSX_API_END, which turns fsx::Error (and any std::exception) into a status
// code plus a thread-local message for fsx_last_error().
#pragma once

#include <string>

#include "common.cuh"

#define FSX_STR_(x) #x
#define FSX_STR(x) FSX_STR_(x)

namespace fsx {
void capi_set_error(const std::string& msg);
const char* capi_last_error();
// max over n u64 keys into *d_max (pre-zeroed)
void capi_launch_max_u64(Ctx* ctx, const uint64_t* d_keys, uint64_t n, uint64_t* d_max,
                         cudaStream_t s);
}  // namespace fsx

#define FSX_API_BEGIN try {
#define FSX_API_END                                        \
  }                                                        \
  catch (const ::fsx::Error& e) {                          \
    ::fsx::capi_set_error(e.what());                       \
    return e.code;                                         \
  }                                                        \
  catch (const std::bad_alloc&) {                          \
    ::fsx::capi_set_error("fsx: host allocation failed");  \
    return FSX_ERR_NOMEM;                                  \
  }                                                        \
  catch (const std::exception& e) {                        \
    ::fsx::capi_set_error(e.what());                       \
    return FSX_ERR_CUDA;                                   \
  }                                                        \
  return FSX_OK;

#define FSX_CHECK_RC(expr)                                         \
  do {                                                             \
    int rc_ = (expr);                                              \
    if (rc_ != FSX_OK) throw ::fsx::Error(rc_, capi_last_error()); \
  } while (0)
