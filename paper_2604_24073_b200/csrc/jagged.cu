// Jagged reshuffle kernels: the segment movers behind the
// reference's indexed_permute / keyed_transpose (include/freescale/jagged.hpp:
// 89-111, 227-248). ranged_dispatch / ranged_combine (:120-199) are contiguous
// slices and concatenations of the same layout and need no kernel of their own
// (the Python mirror does them with device copies).
//
// Layout: values = one contiguous array of `elem_bytes`-sized elements,
// offsets = u64 [n + 1] exclusive prefix of the lengths (offsets[n] = total).
#include <mutex>
#include <unordered_map>
#include <vector>

#include "capi_util.cuh"
#include "common.cuh"
#include "table.cuh"

namespace fsx {
namespace {

constexpr int kJagThreads = 256;
constexpr int kJagTile = 2048;  // segments per scan tile

// out_len[j] = len(perm[j]); bad indices flagged (first writer wins) and
// counted as empty so the scan stays defined
__global__ void k_perm_lengths(const uint64_t* __restrict__ offs, uint64_t n_segs,
                               const uint64_t* __restrict__ perm, uint64_t n_perm,
                               uint64_t* __restrict__ out_len, DevErr* err) { FSX_PDL_ENTER();
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n_perm;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = perm[j];
    if (k >= n_segs) {
      report(err, kErrSegIndex, k, n_segs);
      out_len[j] = 0;
    } else {
      out_len[j] = offs[k + 1] - offs[k];
    }
  }
}

// exclusive scan of u64 lengths, three launches: tile sums, scan of the tile
// sums (one CTA), tile-local scan + carry
__global__ void __launch_bounds__(kJagThreads) k_tile_sums(const uint64_t* __restrict__ len, uint64_t n,
                                                           uint64_t* __restrict__ sums) { FSX_PDL_ENTER();
  __shared__ uint64_t ws[kJagThreads / 32];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kJagTile;
  uint64_t s = 0;
  for (int i = threadIdx.x; i < kJagTile; i += kJagThreads)
    if (base + i < n) s += len[base + i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < kJagThreads / 32; ++w) t += ws[w];
    sums[blockIdx.x] = t;
  }
}

__global__ void k_scan_sums(uint64_t* sums, uint64_t tiles, uint64_t* total) { FSX_PDL_ENTER();
  // one warp: sequential carry over 32-wide chunks
  const unsigned lane = threadIdx.x & 31u;
  uint64_t carry = 0;
  for (uint64_t t0 = 0; t0 < tiles; t0 += 32) {
    const uint64_t t = t0 + lane;
    const uint64_t v = t < tiles ? sums[t] : 0;
    uint64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= static_cast<unsigned>(o)) x += y;
    }
    if (t < tiles) sums[t] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) *total = carry;
}

__global__ void __launch_bounds__(kJagThreads) k_tile_scan(const uint64_t* __restrict__ len, uint64_t n,
                                                           const uint64_t* __restrict__ sums,
                                                           const uint64_t* __restrict__ total,
                                                           uint64_t* __restrict__ offs) { FSX_PDL_ENTER();
  // each thread owns kJagTile / kJagThreads consecutive segments
  constexpr int kPer = kJagTile / kJagThreads;
  __shared__ uint64_t ws[kJagThreads / 32];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kJagTile + threadIdx.x * kPer;
  uint64_t v[kPer], own = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    v[i] = base + i < n ? len[base + i] : 0;
    own += v[i];
  }
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint64_t x = own;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= static_cast<unsigned>(o)) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  uint64_t run = sums[blockIdx.x] + x - own;
  for (unsigned w = 0; w < warp; ++w) run += ws[w];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    if (base + i < n) offs[base + i] = run;
    run += v[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) offs[n] = *total;
}

}  // namespace

// shared with workload.cu (record decode)
void exclusive_offsets(Ctx* ctx, const uint64_t* len, uint64_t n, uint64_t* offs, DevBuf<uint64_t>& scratch,
                       cudaStream_t s) {
  const uint64_t tiles = ceil_div(n > 0 ? n : 1, kJagTile);
  scratch.ensure(tiles + 1);
  FSX_LAUNCH(ctx, k_tile_sums, static_cast<unsigned>(tiles), kJagThreads, 0, s, len, n, scratch.p);
  FSX_LAUNCH(ctx, k_scan_sums, 1, 32, 0, s, scratch.p, tiles, scratch.p + tiles);
  FSX_LAUNCH(ctx, k_tile_scan, static_cast<unsigned>(tiles), kJagThreads, 0, s, len, n, scratch.p,
             scratch.p + tiles, offs);
}

namespace {

// segment mover: warp per output segment, `U`-byte units (16/8/4/1),
// coalesced over the segment; long segments stream, short ones finish fast
template <class U>
__global__ void __launch_bounds__(kJagThreads) k_perm_values(const char* __restrict__ in,
                                                             const uint64_t* __restrict__ offs, uint64_t n_segs,
                                                             const uint64_t* __restrict__ perm,
                                                             const uint64_t* __restrict__ out_offs, uint64_t n_perm,
                                                             uint32_t elem_bytes, char* __restrict__ out) { FSX_PDL_ENTER();
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t upe = elem_bytes / sizeof(U);  // units per element
  for (uint64_t j = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; j < n_perm; j += warps) {
    const uint64_t k = perm[j];
    if (k >= n_segs) continue;
    const uint64_t b = offs[k], e = offs[k + 1];
    const U* src = reinterpret_cast<const U*>(in) + b * upe;
    U* dst = reinterpret_cast<U*>(out) + out_offs[j] * upe;
    const uint64_t units = (e - b) * upe;
    for (uint64_t t = lane; t < units; t += 32) dst[t] = src[t];
  }
}

// keyed_transpose permutation (jagged.hpp:232-241): target position of (f, s)
__global__ void k_transpose_perm(uint64_t keys, uint64_t samples, int feature_major, uint64_t* __restrict__ perm) { FSX_PDL_ENTER();
  const uint64_t n = keys * samples;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (feature_major) {  // target (s, f) <- source f * S + s
      const uint64_t s = i / keys, f = i - s * keys;
      perm[i] = f * samples + s;
    } else {  // target (f, s) <- source s * F + f
      const uint64_t f = i / samples, s = i - f * samples;
      perm[i] = s * keys + f;
    }
  }
}

}  // namespace
}  // namespace fsx

using namespace fsx;

namespace {
cudaStream_t JS(void* s) { return static_cast<cudaStream_t>(s); }

// offsets-scan scratch per (context, device), reused across calls: a local
// buffer meant a cudaMalloc / cudaFree pair per call, and cudaFree
// synchronises the whole device (stalling the engine's lanes mid-training,
// balancer stage 3). The lock covers a call's use of it (every call ends
// with a stream sync before its scratch is free again).
struct JagScratch {
  std::mutex m;
  DevBuf<uint64_t> buf;
};
JagScratch& jag_scratch(const Ctx* ctx) {
  static std::mutex m;
  static auto* bufs = new std::unordered_map<uint64_t, JagScratch>();
  std::lock_guard<std::mutex> g(m);
  return (*bufs)[reinterpret_cast<uintptr_t>(ctx) ^ (static_cast<uint64_t>(ctx->device) << 56)];
}
}  // namespace

extern "C" {

int fsx_jagged_offsets(fsx_ctx* ctx, const uint64_t* d_lengths, uint64_t n, uint64_t* d_offsets,
                       uint64_t* h_total, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  cudaStream_t s = JS(stream);
  JagScratch& js = jag_scratch(ctx);
  std::lock_guard<std::mutex> lk(js.m);
  exclusive_offsets(ctx, d_lengths, n, d_offsets, js.buf, s);
  uint64_t tot = 0;
  FSX_CUDA(cudaMemcpyAsync(&tot, d_offsets + n, 8, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  if (h_total) *h_total = tot;
  FSX_API_END
}

int fsx_jagged_permute(fsx_ctx* ctx, const void* d_values, uint32_t elem_bytes, const uint64_t* d_offsets,
                       uint64_t n_segs, const uint64_t* d_perm, uint64_t n_perm, void* d_out_values,
                       uint64_t out_capacity, uint64_t* d_out_lengths, uint64_t* d_out_offsets,
                       uint64_t* h_out_total, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  cudaStream_t s = JS(stream);
  if (elem_bytes == 0) raise(FSX_ERR_INVALID_ARGUMENT, "jagged: element size must be positive");
  if (n_perm) {
    FSX_LAUNCH(ctx, k_perm_lengths, grid_for(ctx, n_perm, 256, 8), 256, 0, s, d_offsets, n_segs, d_perm, n_perm,
               d_out_lengths, ctx->d_err);
  }
  ctx->check_error(s);  // out-of-range index: the reference throws before moving anything
  JagScratch& js = jag_scratch(ctx);
  std::lock_guard<std::mutex> lk(js.m);
  exclusive_offsets(ctx, d_out_lengths, n_perm, d_out_offsets, js.buf, s);
  uint64_t tot = 0;
  FSX_CUDA(cudaMemcpyAsync(&tot, d_out_offsets + n_perm, 8, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  if (h_out_total) *h_out_total = tot;
  if (!d_out_values) return FSX_OK;  // sizing call
  if (tot > out_capacity)
    raise(FSX_ERR_INVALID_ARGUMENT, "jagged: output capacity " + std::to_string(out_capacity) +
                                        " below the permuted total " + std::to_string(tot));
  if (n_perm && tot) {
    const unsigned grid = grid_for(ctx, n_perm * 32, kJagThreads, 8);
    const uintptr_t al = reinterpret_cast<uintptr_t>(d_values) | reinterpret_cast<uintptr_t>(d_out_values);
    if (elem_bytes % 16 == 0 && al % 16 == 0)
      FSX_LAUNCH(ctx, k_perm_values<uint4>, grid, kJagThreads, 0, s, static_cast<const char*>(d_values), d_offsets,
                 n_segs, d_perm, d_out_offsets, n_perm, elem_bytes, static_cast<char*>(d_out_values));
    else if (elem_bytes % 8 == 0 && al % 8 == 0)
      FSX_LAUNCH(ctx, k_perm_values<uint64_t>, grid, kJagThreads, 0, s, static_cast<const char*>(d_values),
                 d_offsets, n_segs, d_perm, d_out_offsets, n_perm, elem_bytes, static_cast<char*>(d_out_values));
    else if (elem_bytes % 4 == 0 && al % 4 == 0)
      FSX_LAUNCH(ctx, k_perm_values<uint32_t>, grid, kJagThreads, 0, s, static_cast<const char*>(d_values),
                 d_offsets, n_segs, d_perm, d_out_offsets, n_perm, elem_bytes, static_cast<char*>(d_out_values));
    else
      FSX_LAUNCH(ctx, k_perm_values<uint8_t>, grid, kJagThreads, 0, s, static_cast<const char*>(d_values),
                 d_offsets, n_segs, d_perm, d_out_offsets, n_perm, elem_bytes, static_cast<char*>(d_out_values));
  }
  FSX_API_END
}

int fsx_keyed_transpose_perm(fsx_ctx* ctx, uint64_t num_keys, uint64_t num_samples, int feature_major,
                             uint64_t* d_perm, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  const uint64_t n = num_keys * num_samples;
  if (n)
    FSX_LAUNCH(ctx, k_transpose_perm, grid_for(ctx, n, 256, 8), 256, 0, JS(stream), num_keys, num_samples,
               feature_major ? 1 : 0, d_perm);
  FSX_API_END
}

}  // extern "C"
