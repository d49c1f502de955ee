// Sequence load balancer on the GPU (K12-K14): per-rank cost
// estimate (sim.hpp:24-35), FBS snake partition (partition.cpp:157-176) and
// the exact min-max VBS DP (partition.cpp:56-92, 178-209), bit-exact with the
// reference: integer keys for the sort, f64 with explicit round-to-nearest
// intrinsics (no FMA contraction) for every floating-point value.
#include <cmath>
#include <cstring>
#include <vector>

#include <memory>
#include <mutex>
#include <unordered_map>

#include "capi_util.cuh"
#include "table.cuh"

namespace fsx {
namespace {

// ---- K12: cost model --------------------------------------------------------------
// One CTA per group: exact u64 sums of L and L^2. The reference accumulates
// L^2 in f64 in sample order; that sum is exact (hence order-free and equal to
// the integer sum) while every L < 2^26 and the total stays below 2^53 — the
// CTA checks both and otherwise its thread 0 redoes the f64 sum sequentially.
__global__ void k_cost(const uint64_t* __restrict__ lens, const uint64_t* __restrict__ offsets,
                       double c0, double c1, double c2, double* __restrict__ out) { FSX_PDL_ENTER();
  __shared__ unsigned long long s_tok, s_sq, s_big;
  const uint64_t lo = offsets[blockIdx.x], hi = offsets[blockIdx.x + 1];
  if (threadIdx.x == 0) { s_tok = 0; s_sq = 0; s_big = 0; }
  __syncthreads();
  unsigned long long tok = 0, sq = 0, big = 0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint64_t l = lens[i];
    tok += l;
    big |= (l >> 26) != 0;
    sq += (l >> 26) ? 0 : l * l;
  }
  atomicAdd(&s_tok, tok);
  atomicAdd(&s_sq, sq);
  atomicOr(&s_big, big);
  __syncthreads();
  if (threadIdx.x == 0) {
    double sqd;
    if (s_big || s_sq >= (1ull << 53)) {
      sqd = 0.0;
      for (uint64_t i = lo; i < hi; ++i) {
        const double l = static_cast<double>(lens[i]);
        sqd = __dadd_rn(sqd, __dmul_rn(l, l));
      }
    } else {
      sqd = static_cast<double>(s_sq);
    }
    // c0 + c1 * tokens + c2 * sq, left to right (sim.hpp:21-23)
    out[blockIdx.x] = __dadd_rn(__dadd_rn(c0, __dmul_rn(c1, static_cast<double>(s_tok))), __dmul_rn(c2, sqd));
  }
}

// ---- K13: sorted_indices (partition.cpp:14-24) -----------------------------------
// key = (maxlen - len) << (bo + bl) | origin << bl | local: ascending key ==
// descending length, then origin, then local index.
__global__ void k_partition_keys(const uint64_t* __restrict__ lens, const int32_t* __restrict__ origin,
                                 const int32_t* __restrict__ local, uint64_t m, uint64_t maxlen, int bo,
                                 int bl, uint64_t* __restrict__ keys) { FSX_PDL_ENTER();
  for (uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; g < m;
       g += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    keys[g] = ((maxlen - lens[g]) << (bo + bl)) | (static_cast<uint64_t>(origin[g]) << bl) |
              static_cast<uint64_t>(local[g]);
}

// snake deal (partition.cpp:169-174): sorted position k -> rank
__global__ void k_fbs_assign(const uint32_t* __restrict__ sorted, uint64_t m, int n,
                             int32_t* __restrict__ assignment, uint64_t* __restrict__ order) { FSX_PDL_ENTER();
  const uint64_t per = m / static_cast<uint64_t>(n);
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < m;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t pass = k / n, pos = k % n;
    const uint64_t rank = (pass % 2 == 0) ? pos : static_cast<uint64_t>(n) - 1 - pos;
    const uint32_t g = sorted[k];
    order[rank * per + pass] = g;
    assignment[g] = static_cast<int32_t>(rank);
  }
}

// ---- K14: VBS weights, prefix and the min-max DP ---------------------------------
// w[k] = pow(len[sorted[k]], alpha) for alpha in {1, 2} is exact in f64 for
// L < 2^26 (std::pow returns the exact product then); prefix sums are exact
// integers below 2^53. Both are checked; otherwise the host supplies weights.
__global__ void k_vbs_weights(const uint64_t* __restrict__ lens, const uint32_t* __restrict__ sorted,
                              uint64_t m, int alpha2, uint64_t* __restrict__ wint) { FSX_PDL_ENTER();
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < m;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t l = lens[sorted[k]];
    wint[k] = alpha2 ? l * l : l;
  }
}

// sequential f64 prefix (prefix[i+1] = prefix[i] + w[i], partition.cpp:58-59)
// for weights that are not exact integers: one thread, reference order
__global__ void k_prefix_seq(const double* __restrict__ w, uint64_t m, double* __restrict__ prefix) { FSX_PDL_ENTER();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    prefix[0] = 0.0;
    for (uint64_t i = 0; i < m; ++i) {
      s = __dadd_rn(s, w[i]);
      prefix[i + 1] = s;
    }
  }
}

// u64 inclusive scan: one CTA of 1024 threads, contiguous chunks (m <= ~1M)
__global__ void __launch_bounds__(1024) k_prefix_u64(const uint64_t* __restrict__ w, uint64_t m,
                                                     double* __restrict__ prefix) { FSX_PDL_ENTER();
  __shared__ unsigned long long part[1024];
  const uint64_t per = (m + blockDim.x - 1) / blockDim.x;
  const uint64_t lo = threadIdx.x * per, hi = lo + per < m ? lo + per : m;
  unsigned long long s = 0;
  for (uint64_t i = lo; i < hi; ++i) s += w[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (unsigned t = 0; t < blockDim.x; ++t) {
      const unsigned long long x = part[t];
      part[t] = run;
      run += x;
    }
  }
  __syncthreads();
  unsigned long long run = part[threadIdx.x];
  if (threadIdx.x == 0) prefix[0] = 0.0;
  for (uint64_t i = lo; i < hi; ++i) {
    run += w[i];
    prefix[i + 1] = static_cast<double>(run);
  }
}

__global__ void k_fill_inf(double* __restrict__ dp, uint64_t n) { FSX_PDL_ENTER();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dp[i] = __longlong_as_double(0x7ff0000000000000ll);
}

// dp layer k=1: dp[1][j] = prefix[j]
__global__ void k_dp_first(const double* __restrict__ prefix, uint64_t m, double* __restrict__ dp1) { FSX_PDL_ENTER();
  for (uint64_t j = 1 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j <= m;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dp1[j] = prefix[j];
}

// One thread per j: the reference's downward scan with its exact tie-break —
// strict `<` keeps the largest x attaining the minimum, and the scan stops
// once the trailing segment alone reaches the best cost (partition.cpp:66-81).
__global__ void k_dp_layer(const double* __restrict__ prefix, const double* __restrict__ prev,
                           uint64_t m, int k, double* __restrict__ cur, uint32_t* __restrict__ cut) { FSX_PDL_ENTER();
  for (uint64_t j = static_cast<uint64_t>(k) + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       j <= m; j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double best = __longlong_as_double(0x7ff0000000000000ll);
    uint64_t best_x = j - 1;
    const double pj = prefix[j];
    for (uint64_t x = j - 1; x + 1 >= static_cast<uint64_t>(k); --x) {
      const double seg = __dsub_rn(pj, prefix[x]);
      if (seg >= best) break;
      const double pv = prev[x];
      const double cost = pv < seg ? seg : pv;  // std::max(pv, seg)
      if (cost < best) {
        best = cost;
        best_x = x;
      }
      if (x == 0) break;
    }
    cur[j] = best;
    cut[j] = static_cast<uint32_t>(best_x);
  }
}

// backtrack (partition.cpp:84-90): sizes of the n segments
__global__ void k_dp_backtrack(const uint32_t* __restrict__ cut, uint64_t m, int n, int32_t* __restrict__ sizes) { FSX_PDL_ENTER();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    uint64_t j = m;
    for (int k = n; k >= 1; --k) {
      const uint64_t x = k == 1 ? 0 : cut[static_cast<uint64_t>(k) * (m + 1) + j];
      sizes[k - 1] = static_cast<int32_t>(j - x);
      j = x;
    }
  }
}

// contiguous segments of the sorted order: sorted position k -> rank
__global__ void k_vbs_assign(const uint32_t* __restrict__ sorted, uint64_t m, const int32_t* __restrict__ sizes,
                             int n, int32_t* __restrict__ assignment, uint64_t* __restrict__ order) { FSX_PDL_ENTER();
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < m;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t start = 0;
    int r = 0;
    while (r < n - 1 && k >= start + static_cast<uint64_t>(sizes[r])) {
      start += static_cast<uint64_t>(sizes[r]);
      ++r;
    }
    order[k] = sorted[k];
    assignment[sorted[k]] = r;
  }
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

template <class T>
void h2d(DevBuf<T>& d, const T* h, uint64_t n, cudaStream_t s) {
  d.ensure(n ? n : 1);
  if (n) FSX_CUDA(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

// Device scratch of the partitioners per (context, device), grown on demand
// and kept across calls: the balancer partitions every iteration, and a
// cudaMalloc / cudaFree pair per buffer per call (cudaFree synchronises the
// device) cost more than the sort itself at config 2's 65,536 samples. The
// lock covers one call's use (each call ends with a stream sync).
struct PartScratch {
  std::mutex m;
  DevBuf<uint64_t> lens, k0, k1, o, w;
  DevBuf<int32_t> origin, local, a, sizes;
  DevBuf<uint32_t> v0, v1, perm, cut;
  DevBuf<double> prefix, dw, dp;
  RadixScratch radix;
};
PartScratch& part_scratch(const Ctx* ctx) {
  static std::mutex m;
  static auto* bufs = new std::unordered_map<uint64_t, std::unique_ptr<PartScratch>>();
  std::lock_guard<std::mutex> g(m);
  auto& p = (*bufs)[reinterpret_cast<uintptr_t>(ctx) ^ (static_cast<uint64_t>(ctx->device) << 56)];
  if (!p) p = std::make_unique<PartScratch>();
  return *p;
}

// sorted_indices on the device: returns the permutation (sorted position -> g)
void sorted_indices(Ctx* ctx, const uint64_t* h_lens, const int32_t* h_origin, const int32_t* h_local,
                    uint64_t m, cudaStream_t s, PartScratch& ps) {
  DevBuf<uint64_t>& d_lens = ps.lens;
  DevBuf<uint32_t>& perm_out = ps.perm;
  uint64_t maxlen = 0;
  int32_t maxo = 0, maxl = 0;
  for (uint64_t g = 0; g < m; ++g) {
    maxlen = h_lens[g] > maxlen ? h_lens[g] : maxlen;
    if (h_origin[g] < 0 || h_local[g] < 0)
      raise(FSX_ERR_INVALID_ARGUMENT, "partition: negative origin rank or local index");
    maxo = h_origin[g] > maxo ? h_origin[g] : maxo;
    maxl = h_local[g] > maxl ? h_local[g] : maxl;
  }
  const int bo = bits_for(static_cast<uint64_t>(maxo)), bl = bits_for(static_cast<uint64_t>(maxl));
  const int blen = bits_for(maxlen);
  if (blen + bo + bl > 64) raise(FSX_ERR_CONFIG, "partition: sort key wider than 64 bits");
  h2d(d_lens, h_lens, m, s);
  DevBuf<int32_t>& d_o = ps.origin;
  DevBuf<int32_t>& d_l = ps.local;
  h2d(d_o, h_origin, m, s);
  h2d(d_l, h_local, m, s);
  ps.k0.ensure(m); ps.k1.ensure(m); ps.v0.ensure(m); ps.v1.ensure(m);
  FSX_LAUNCH(ctx, k_partition_keys, grid_for(ctx, m, 256, 8), 256, 0, s, d_lens.p, d_o.p, d_l.p, m,
             maxlen, bo, bl, ps.k0.p);
  uint64_t* ko;
  uint32_t* vo;
  radix_sort_pairs<uint64_t>(ctx, ps.k0.p, ps.v0.p, ps.k1.p, ps.v1.p, m, nullptr, blen + bo + bl, ps.radix, s, &ko,
                             &vo);
  perm_out.ensure(m);
  FSX_CUDA(cudaMemcpyAsync(perm_out.p, vo, m * 4, cudaMemcpyDeviceToDevice, s));
}

}  // namespace
}  // namespace fsx

using namespace fsx;

extern "C" {

int fsx_cost_estimate(fsx_ctx* ctx, const uint64_t* d_lens, const uint64_t* h_offsets, int num_groups,
                      double c0, double c1, double c2, double* h_out, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  if (num_groups <= 0) return FSX_OK;
  cudaStream_t s = S(stream);
  DevBuf<uint64_t> off;
  h2d(off, h_offsets, static_cast<uint64_t>(num_groups) + 1, s);
  DevBuf<double> out(num_groups);
  FSX_LAUNCH(ctx, k_cost, num_groups, 256, 0, s, d_lens, off.p, c0, c1, c2, out.p);
  FSX_CUDA(cudaMemcpyAsync(h_out, out.p, sizeof(double) * num_groups, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  FSX_API_END
}

int fsx_fbs_partition(fsx_ctx* ctx, const uint64_t* h_lens, const int32_t* h_origin, const int32_t* h_local,
                      uint64_t m, int num_ranks, int32_t* h_assignment, uint64_t* h_order, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  if (num_ranks < 1) raise(FSX_ERR_INVALID_ARGUMENT, "fbs: num_ranks must be >= 1");
  if (m % static_cast<uint64_t>(num_ranks) != 0)
    raise(FSX_ERR_INVALID_ARGUMENT, "fbs: " + std::to_string(m) + " samples not divisible by " +
                                        std::to_string(num_ranks) + " ranks");
  if (m == 0) return FSX_OK;
  cudaStream_t s = S(stream);
  PartScratch& ps = part_scratch(ctx);
  std::lock_guard<std::mutex> lk(ps.m);
  sorted_indices(ctx, h_lens, h_origin, h_local, m, s, ps);
  DevBuf<uint32_t>& perm = ps.perm;
  DevBuf<int32_t>& a = ps.a;
  DevBuf<uint64_t>& o = ps.o;
  a.ensure(m);
  o.ensure(m);
  FSX_LAUNCH(ctx, k_fbs_assign, grid_for(ctx, m, 256, 8), 256, 0, s, perm.p, m, num_ranks, a.p, o.p);
  FSX_CUDA(cudaMemcpyAsync(h_assignment, a.p, m * 4, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaMemcpyAsync(h_order, o.p, m * 8, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  ctx->check_error(s);
  FSX_API_END
}

int fsx_vbs_partition(fsx_ctx* ctx, const uint64_t* h_lens, const int32_t* h_origin, const int32_t* h_local,
                      uint64_t m, int num_ranks, double alpha, const int32_t* h_tuned_sizes,
                      int32_t* h_sizes_out, int32_t* h_assignment, uint64_t* h_order, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  if (!(alpha > 0)) raise(FSX_ERR_INVALID_ARGUMENT, "vbs: alpha must be > 0");
  if (m == 0) raise(FSX_ERR_INVALID_ARGUMENT, "vbs: no samples");
  if (static_cast<uint64_t>(num_ranks) > m)
    raise(FSX_ERR_INVALID_ARGUMENT, "vbs: " + std::to_string(num_ranks) + " ranks but only " +
                                        std::to_string(m) + " samples (cannot give every rank one)");
  if (m >= (1ull << 32)) raise(FSX_ERR_CONFIG, "vbs: too many samples");
  cudaStream_t s = S(stream);
  const int n = num_ranks;
  PartScratch& ps = part_scratch(ctx);
  std::lock_guard<std::mutex> lk(ps.m);
  sorted_indices(ctx, h_lens, h_origin, h_local, m, s, ps);
  DevBuf<uint64_t>& d_lens = ps.lens;
  DevBuf<uint32_t>& perm = ps.perm;
  std::vector<int32_t> sizes(n);
  bool tuned = false;
  if (h_tuned_sizes) {
    uint64_t tot = 0;
    bool pos = true;
    for (int r = 0; r < n; ++r) {
      tot += static_cast<uint64_t>(h_tuned_sizes[r] > 0 ? h_tuned_sizes[r] : 0);
      pos &= h_tuned_sizes[r] >= 0;
    }
    tuned = pos && tot == m;  // partition.cpp:189-195
  }
  DevBuf<int32_t>& d_sizes = ps.sizes;
  d_sizes.ensure(n);
  if (tuned) {
    std::memcpy(sizes.data(), h_tuned_sizes, sizeof(int32_t) * n);
    FSX_CUDA(cudaMemcpyAsync(d_sizes.p, sizes.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
  } else {
    DevBuf<double>& prefix = ps.prefix;
    prefix.ensure(m + 1);
    uint64_t maxlen = 0;
    for (uint64_t g = 0; g < m; ++g) maxlen = h_lens[g] > maxlen ? h_lens[g] : maxlen;
    const bool a1 = alpha == 1.0, a2 = alpha == 2.0;
    const bool exact_int = (a1 || a2) && maxlen < (1ull << 26) &&
                           static_cast<double>(maxlen) * static_cast<double>(a2 ? maxlen : 1) *
                                   static_cast<double>(m) < 9.0e15;
    if (exact_int) {
      DevBuf<uint64_t>& w = ps.w;
      w.ensure(m);
      FSX_LAUNCH(ctx, k_vbs_weights, grid_for(ctx, m, 256, 8), 256, 0, s, d_lens.p, perm.p, m, a2 ? 1 : 0, w.p);
      FSX_LAUNCH(ctx, k_prefix_u64, 1, 1024, 0, s, w.p, m, prefix.p);
    } else {
      // weights by the host's std::pow in sorted order (partition.cpp:197-200)
      std::vector<uint32_t> hp(m);
      FSX_CUDA(cudaMemcpyAsync(hp.data(), perm.p, m * 4, cudaMemcpyDeviceToHost, s));
      FSX_CUDA(cudaStreamSynchronize(s));
      std::vector<double> w(m);
      for (uint64_t k = 0; k < m; ++k) w[k] = std::pow(static_cast<double>(h_lens[hp[k]]), alpha);
      DevBuf<double>& dw = ps.dw;
      dw.ensure(m);
      FSX_CUDA(cudaMemcpyAsync(dw.p, w.data(), m * 8, cudaMemcpyHostToDevice, s));
      FSX_LAUNCH(ctx, k_prefix_seq, 1, 32, 0, s, dw.p, m, prefix.p);
      FSX_CUDA(cudaStreamSynchronize(s));
    }
    // dp [n+1][m+1], cut [n+1][m+1]
    const uint64_t cols = m + 1;
    DevBuf<double>& dp = ps.dp;
    DevBuf<uint32_t>& cut = ps.cut;
    dp.ensure(static_cast<uint64_t>(n + 1) * cols);
    cut.ensure(static_cast<uint64_t>(n + 1) * cols);
    FSX_LAUNCH(ctx, k_fill_inf, grid_for(ctx, (n + 1) * cols, 256, 8), 256, 0, s, dp.p, (n + 1) * cols);
    FSX_LAUNCH(ctx, k_dp_first, grid_for(ctx, m, 256, 8), 256, 0, s, prefix.p, m, dp.p + cols);
    for (int k = 2; k <= n; ++k)
      FSX_LAUNCH(ctx, k_dp_layer, grid_for(ctx, m, 128, 16), 128, 0, s, prefix.p, dp.p + (k - 1) * cols, m, k,
                 dp.p + k * cols, cut.p + k * cols);
    FSX_LAUNCH(ctx, k_dp_backtrack, 1, 32, 0, s, cut.p, m, n, d_sizes.p);
    FSX_CUDA(cudaMemcpyAsync(sizes.data(), d_sizes.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    FSX_CUDA(cudaStreamSynchronize(s));
  }
  DevBuf<int32_t>& a = ps.a;
  DevBuf<uint64_t>& o = ps.o;
  a.ensure(m);
  o.ensure(m);
  FSX_LAUNCH(ctx, k_vbs_assign, grid_for(ctx, m, 256, 8), 256, 0, s, perm.p, m, d_sizes.p, n, a.p, o.p);
  FSX_CUDA(cudaMemcpyAsync(h_assignment, a.p, m * 4, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaMemcpyAsync(h_order, o.p, m * 8, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  if (h_sizes_out) std::memcpy(h_sizes_out, sizes.data(), sizeof(int32_t) * n);
  ctx->check_error(s);
  FSX_API_END
}

// autotune_update (partition.cpp:211-269): n <= a few dozen, host f64; this
// TU is compiled with -ffp-contract=off semantics for host code (the f64
// expressions below must not contract into FMA to match the reference).
int fsx_autotune_update(int n, int32_t* sizes, double* ema_local, double* ema_global, int step,
                        double delta, double decay, const double* t) {
  FSX_API_BEGIN
  if (n < 1) raise(FSX_ERR_INVALID_ARGUMENT, "autotune: expected at least one rank");
  double mean = 0;
  for (int r = 0; r < n; ++r) {
    if (t[r] <= 0) raise(FSX_ERR_INVALID_ARGUMENT, "autotune: execution times must be > 0");
    mean += t[r];
  }
  mean /= static_cast<double>(n);
  const bool first = *ema_global == 0.0;
  volatile double dm = decay, om = 1 - decay;  // keep the products separate (no contraction)
  if (first) {
    *ema_global = mean;
  } else {
    const double a = dm * *ema_global;
    const double b = om * mean;
    *ema_global = a + b;
  }
  for (int r = 0; r < n; ++r) {
    if (first) {
      ema_local[r] = t[r];
    } else {
      const double a = dm * ema_local[r];
      const double b = om * t[r];
      ema_local[r] = a + b;
    }
  }
  int total = 0;
  for (int r = 0; r < n; ++r) total += sizes[r];
  std::vector<int32_t> desired(sizes, sizes + n);
  const double hi_t = (1 + delta) * *ema_global, lo_t = (1 - delta) * *ema_global;
  for (int r = 0; r < n; ++r) {
    if (ema_local[r] > hi_t) desired[r] = desired[r] - step > 1 ? desired[r] - step : 1;
    else if (ema_local[r] < lo_t) desired[r] += step;
  }
  int diff = -total;
  for (int r = 0; r < n; ++r) diff += desired[r];
  while (diff > 0) {
    int donor = 0;
    for (int r = 1; r < n; ++r)
      if (desired[r] > desired[donor] || (desired[r] == desired[donor] && ema_local[r] > ema_local[donor])) donor = r;
    if (desired[donor] <= 1) break;
    --desired[donor];
    --diff;
  }
  while (diff < 0) {
    int recv = 0;
    for (int r = 1; r < n; ++r)
      if (desired[r] < desired[recv] || (desired[r] == desired[recv] && ema_local[r] < ema_local[recv])) recv = r;
    ++desired[recv];
    ++diff;
  }
  std::memcpy(sizes, desired.data(), sizeof(int32_t) * n);
  FSX_API_END
}

}  // extern "C"
