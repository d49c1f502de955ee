// Shared infrastructure for libfsx: error classes, the per-rank context, the
// device error word, launch accounting and small device helpers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "fsx.h"

namespace fsx {

// Host-side exception carrying an fsx.h status class; the C ABI catches it
// and returns the code, keeping the message for fsx_last_error().
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "cuda: %s failed at %s:%d: %s", what, file, line,
                  cudaGetErrorString(e));
    throw Error(e == cudaErrorMemoryAllocation ? FSX_ERR_NOMEM : FSX_ERR_CUDA, buf);
  }
}
inline void cu_check(CUresult e, const char* what, const char* file, int line) {
  if (e != CUDA_SUCCESS) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "cuda driver: %s failed at %s:%d: CUresult %d", what, file, line,
                  static_cast<int>(e));
    throw Error(FSX_ERR_CUDA, buf);
  }
}

// Driver entry points used by the copy-engine transport, resolved through the
// runtime (cudaGetDriverEntryPoint) so libfsx.so has no link-time dependency
// on libcuda and loads on machines without a driver (build/CPU checks).
namespace drv {
using WriteValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32 write_value32();
WaitValue32 wait_value32();
}  // namespace drv
#define FSX_CUDA(x) ::fsx::cuda_check((x), #x, __FILE__, __LINE__)
#define FSX_CU(x) ::fsx::cu_check((x), #x, __FILE__, __LINE__)

// ---- device error word ------------------------------------------------------
// Kernels that detect a condition the reference throws on record it here
// (first writer wins); the host turns it into the same exception class and
// message at the next sync point.
enum DevErrKind : int {
  kErrNone = 0,
  kErrRowRange = 1,     // a = id, b = total_rows        -> domain_error
  kErrNotOwned = 2,     // a = id, b = shard             -> domain_error
  kErrNonFinite = 3,    // a = id                        -> domain_error
  kErrRecvNotOwned = 4, // a = id                        -> ProtocolError
  kErrMissingRow = 5,   // a = id                        -> ProtocolError
  kErrCapacity = 6,     // a = needed, b = capacity      -> CollectiveError
  kErrMissingCoRow = 7, // a = id                        -> ProtocolError
  kErrMaskOverlap = 8,  //                               -> ProtocolError
  kErrSegIndex = 9,     // a = index, b = segments       -> out_of_range
};

struct DevErr {
  int kind;
  int pad;
  unsigned long long a, b;
};

__device__ __forceinline__ void report(DevErr* e, int kind, unsigned long long a,
                                       unsigned long long b) {
  if (atomicCAS(&e->kind, 0, kind) == 0) {
    e->a = a;
    e->b = b;
  }
}

std::string describe(const DevErr& e, int* code);

// ---- per-rank context ----------------------------------------------------------
struct Ctx {
  int device = 0;
  int rank = 0;
  int world = 1;
  DevErr* d_err = nullptr;   // device error word
  DevErr* h_err = nullptr;   // pinned host mirror
  std::atomic<uint64_t> launches{0};
  int num_sms = 148;
  // grid caps (CTAs per SM) of the row movers and update kernels. The
  // compute-stream kernels must leave register room on every SM for the
  // side lanes' latency-bound kernels (dedup / collision of the next
  // iteration), or those wait for a whole merge / update to drain.
  // Overridable for tuning: FSX_COPY_PER_SM, FSX_SINGLE_PER_SM, FSX_FLAT_PER_SM.
  unsigned copy_per_sm = 3, single_per_sm = 8, flat_per_sm = 16, warp_per_sm = 3;
  bool sgd_warp = true;  // FSX_SGD_WARP=0: the thread-per-vector k_sgd_flat + k_sgd_combine
  // the bulk-copy staged persistent update (sgd_stream.cuh); FSX_SGD_STREAM=0:
  // k_sgd_single + k_sgd_warp. stream_per_sm caps its CTAs (4 warps) per SM.
  bool sgd_stream = true;
  unsigned stream_per_sm = 8;
  unsigned stream_variant = 0;
  // k_sgd_stream's own span per launch (fsx_ctx_kernel_span): device ring
  static constexpr uint64_t kSpanSlots = 4096;
  unsigned long long* d_span = nullptr;
  uint64_t span_next = 0;
  bool span_on = false;  // FSX_STREAM_VARIANT (tuning): ring depth / CTAs per SM
  unsigned warp_variant = 0;  // FSX_WARP_VARIANT (tuning): k_sgd_warp unroll / min CTAs per SM
  bool pdl = true;       // programmatic dependent launches (FSX_PDL=0: plain launches)
  bool onesweep = true;  // decoupled look-back radix passes (FSX_ONESWEEP=0: 3 launches per pass)

  void check_error(cudaStream_t s);  // D2H the word, sync `s`, throw if set
};

// RAII device switch for host threads that drive several contexts.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Launch helper: counts launches and checks the launch error.
// Every kernel is a programmatic dependent launch (PDL) when ctx->pdl: the
// next kernel on a stream is scheduled while the previous one drains, and
// waits for its completion (and memory) at its first statement — the
// FSX_PDL_ENTER() that opens every __global__ function. Each kernel then
// releases its own dependent as soon as all of its CTAs are resident, so a
// chain of short latency-bound kernels (the side lanes' sort / scan / flag
// kernels) overlaps launch latency with the predecessor's tail.
#define FSX_PDL_ENTER()                                  \
  do {                                                   \
    asm volatile("griddepcontrol.wait;" ::: "memory");   \
    asm volatile("griddepcontrol.launch_dependents;" ::); \
  } while (0)

#define FSX_LAUNCH(ctx_, kern_, grid_, block_, smem_, strm_, ...)                       \
  do {                                                                                \
    if ((ctx_)->pdl) {                                                                 \
      cudaLaunchConfig_t cfg_{};                                                      \
      cfg_.gridDim = dim3(grid_);                                                      \
      cfg_.blockDim = dim3(block_);                                                    \
      cfg_.dynamicSmemBytes = (smem_);                                                 \
      cfg_.stream = (strm_);                                                         \
      cudaLaunchAttribute at_[1];                                                     \
      at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                 \
      at_[0].val.programmaticStreamSerializationAllowed = 1;                          \
      cfg_.attrs = at_;                                                               \
      cfg_.numAttrs = 1;                                                              \
      FSX_CUDA(cudaLaunchKernelEx(&cfg_, kern_, __VA_ARGS__));                       \
    } else {                                                                          \
      kern_<<<(grid_), (block_), (smem_), (strm_)>>>(__VA_ARGS__);                     \
      FSX_CUDA(cudaGetLastError());                                                   \
    }                                                                                 \
    (ctx_)->launches.fetch_add(1, std::memory_order_relaxed);                          \
  } while (0)

// ---- device buffers ----------------------------------------------------------
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) FSX_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

inline unsigned ceil_div(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// grid for a grid-stride kernel: enough CTAs to fill every SM `per_sm` times,
// never more than the work needs
inline unsigned grid_for(const Ctx* c, uint64_t items, unsigned per_cta, unsigned per_sm = 8) {
  uint64_t need = (items + per_cta - 1) / per_cta;
  uint64_t cap = static_cast<uint64_t>(c->num_sms) * per_sm;
  if (need < 1) need = 1;
  return static_cast<unsigned>(need < cap ? need : cap);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace fsx
