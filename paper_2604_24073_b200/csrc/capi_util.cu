#include "capi_util.cuh"

namespace fsx {

namespace {
thread_local std::string g_last_error;

__global__ void k_max_u64(const uint64_t* __restrict__ k, uint64_t n, unsigned long long* out) { FSX_PDL_ENTER();
  unsigned long long m = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    m = k[i] > m ? k[i] : m;
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
    m = y > m ? y : m;
  }
  if ((threadIdx.x & 31u) == 0) atomicMax(out, m);
}
}  // namespace

void capi_set_error(const std::string& msg) { g_last_error = msg; }

namespace drv {
namespace {
void* entry(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  FSX_CUDA(cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess)
    raise(FSX_ERR_CUDA, std::string("cuda driver entry point not found: ") + name);
  return fn;
}
}  // namespace
WriteValue32 write_value32() {
  static WriteValue32 f = reinterpret_cast<WriteValue32>(entry("cuStreamWriteValue32"));
  return f;
}
WaitValue32 wait_value32() {
  static WaitValue32 f = reinterpret_cast<WaitValue32>(entry("cuStreamWaitValue32"));
  return f;
}
}  // namespace drv
const char* capi_last_error() { return g_last_error.c_str(); }

void capi_launch_max_u64(Ctx* ctx, const uint64_t* d_keys, uint64_t n, uint64_t* d_max,
                         cudaStream_t s) {
  FSX_LAUNCH(ctx, k_max_u64, grid_for(ctx, n, 256 * 8, 4), 256, 0, s, d_keys, n,
             reinterpret_cast<unsigned long long*>(d_max));
}

}  // namespace fsx
