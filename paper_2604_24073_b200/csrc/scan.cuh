// Multi-counter stream compaction / exclusive scan.
//
// Most hot-path bookkeeping is "for every item, emit it at its rank among the
// items of the same category": unique-after-sort, owner compaction, per-source
// pack lists, co/ex gradient splits. One primitive covers them all: an Op gives
// each item a small vector of NC counts; the primitive computes, for every
// item, the exclusive prefix of those vectors over the item order and calls
// Op::emit with it (and the grand totals). Two launches, no host round trip,
// no spin waits:
//   1. k_tile_reduce : per-tile sums            (one CTA per 2048-item tile)
//   2. k_tile_emit   : every CTA sums the tile sums before it (its prefix) and
//                      all of them (the grand totals, CTA 0 also stores them)
//                      from L2, then re-counts, block-scans (warp shuffles),
//                      and emits
// Item counts may live on the device (d_n); grids are sized by capacity and
// tiles beyond *d_n exit early, so chains of these never need a host sync.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace fsx {

constexpr int kScanThreads = 256;
#ifndef FSX_SCAN_IPT
#define FSX_SCAN_IPT 8
#endif
constexpr int kScanIPT = FSX_SCAN_IPT;  // items per thread unless the Op says otherwise
constexpr int kScanTile = kScanThreads * kScanIPT;

// Items per thread of an Op's scan: Op::kIPT when it declares one. Ops whose
// live count is small next to the GPU (a few tens of thousands of rows) use
// fewer items per thread so their tiles spread over every SM: these scans are
// latency-bound chains of dependent loads, not bandwidth-bound.
template <class Op, class = void>
struct ScanIPT {
  static constexpr int v = kScanIPT;
};
template <class Op>
struct ScanIPT<Op, std::void_t<decltype(Op::kIPT)>> {
  static constexpr int v = Op::kIPT;
};

__device__ __forceinline__ uint64_t scan_n(uint64_t n_cap, const uint64_t* d_n) {
  if (d_n == nullptr) return n_cap;
  uint64_t n = *d_n;
  return n < n_cap ? n : n_cap;
}

// Block-wide exclusive scan of NC counters held by each thread; returns the
// exclusive prefix in `v` and the block total in `total`.
template <int NC>
__device__ __forceinline__ void block_exclusive_scan(uint32_t (&v)[NC], uint32_t (&total)[NC]) {
  __shared__ uint32_t warp_tot[kScanThreads / 32][NC];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t incl[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t x = v[c];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= static_cast<unsigned>(o)) x += y;
    }
    incl[c] = x;
  }
  if (lane == 31) {
#pragma unroll
    for (int c = 0; c < NC; ++c) warp_tot[warp][c] = incl[c];
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
      uint32_t t = warp_tot[w][c];
      if (w < static_cast<int>(warp)) before += t;
      all += t;
    }
    v[c] = before + incl[c] - v[c];
    total[c] = all;
  }
  __syncthreads();
}

template <class Op>
static __global__ void __launch_bounds__(kScanThreads) k_tile_reduce(Op op, uint64_t n_cap,
                                                              const uint64_t* d_n,
                                                              uint32_t* tile_sums) { FSX_PDL_ENTER();
  constexpr int NC = Op::NC;
  constexpr int IPT = ScanIPT<Op>::v;
  const uint64_t n = scan_n(n_cap, d_n);
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * (kScanThreads * IPT);
  uint32_t acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0;
  if (base < n) {
    const uint64_t first = base + static_cast<uint64_t>(threadIdx.x) * IPT;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      const uint64_t i = first + q;
      if (i < n) {
        uint32_t cnt[NC];
        op.count(i, cnt);
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] += cnt[c];
      }
    }
  }
  uint32_t total[NC];
  block_exclusive_scan<NC>(acc, total);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) tile_sums[static_cast<uint64_t>(blockIdx.x) * NC + c] = total[c];
  }
}

// One CTA of 1024 threads: exclusive scan over `tiles` rows of NC counters
// (in place, all counters in one block pass), grand totals to `totals`.
template <int NC>
static __global__ void __launch_bounds__(1024) k_scan_tiles(uint32_t* tile_sums, unsigned tiles,
                                                            uint64_t* totals) { FSX_PDL_ENTER();
  __shared__ uint32_t wt[32][NC];
  const unsigned per = (tiles + blockDim.x - 1) / blockDim.x;
  const unsigned lo = threadIdx.x * per;
  const unsigned hi = min(tiles, lo + per);
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t s[NC], incl[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) s[c] = 0;
  for (unsigned t = lo; t < hi; ++t)
#pragma unroll
    for (int c = 0; c < NC; ++c) s[c] += tile_sums[static_cast<uint64_t>(t) * NC + c];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t x = s[c];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= static_cast<unsigned>(o)) x += y;
    }
    incl[c] = x;
    if (lane == 31) wt[warp][c] = x;
  }
  __syncthreads();
  const unsigned nw = blockDim.x >> 5;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t before = 0, all = 0;
    for (unsigned w = 0; w < nw; ++w) {
      const uint32_t t = wt[w][c];
      before += w < warp ? t : 0u;
      all += t;
    }
    uint32_t run = before + incl[c] - s[c];
    if (totals && threadIdx.x == 0) totals[c] = all;
    for (unsigned t = lo; t < hi; ++t) {
      const uint32_t x = tile_sums[static_cast<uint64_t>(t) * NC + c];
      tile_sums[static_cast<uint64_t>(t) * NC + c] = run;
      run += x;
    }
  }
}

template <class Op>
static __global__ void __launch_bounds__(kScanThreads) k_tile_emit(Op op, uint64_t n_cap,
                                                                   const uint64_t* d_n,
                                                                   const uint32_t* tile_sums,
                                                                   unsigned tiles,
                                                                   uint64_t* d_totals) { FSX_PDL_ENTER();
  constexpr int NC = Op::NC;
  constexpr int IPT = ScanIPT<Op>::v;
  __shared__ uint32_t s_pre[NC], s_tot[NC];
  const uint64_t n = scan_n(n_cap, d_n);
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * (kScanThreads * IPT);
  if (base >= n && blockIdx.x != 0) return;  // whole CTA exits together
  // prefix of this tile and grand totals, straight from the tile sums (L2)
  {
    uint32_t pre[NC], all[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) pre[c] = all[c] = 0;
    for (unsigned t = threadIdx.x; t < tiles; t += blockDim.x)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const uint32_t x = tile_sums[static_cast<uint64_t>(t) * NC + c];
        all[c] += x;
        pre[c] += t < blockIdx.x ? x : 0u;
      }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        pre[c] += __shfl_xor_sync(0xffffffffu, pre[c], o);
        all[c] += __shfl_xor_sync(0xffffffffu, all[c], o);
      }
    }
    __shared__ uint32_t w_pre[kScanThreads / 32][NC], w_all[kScanThreads / 32][NC];
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < NC; ++c) { w_pre[warp][c] = pre[c]; w_all[warp][c] = all[c]; }
    __syncthreads();
    if (threadIdx.x < NC) {
      uint32_t p = 0, a = 0;
      for (int w = 0; w < kScanThreads / 32; ++w) { p += w_pre[w][threadIdx.x]; a += w_all[w][threadIdx.x]; }
      s_pre[threadIdx.x] = p;
      s_tot[threadIdx.x] = a;
      if (blockIdx.x == 0 && d_totals) d_totals[threadIdx.x] = a;
    }
    __syncthreads();
  }
  if (base >= n) return;  // CTA 0 of an empty input: totals stored, nothing to emit
  const uint64_t first = base + static_cast<uint64_t>(threadIdx.x) * IPT;
  uint32_t run[NC], tot[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) { run[c] = 0; tot[c] = s_tot[c]; }
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const uint64_t i = first + q;
    if (i < n) {
      uint32_t cnt[NC];
      op.count(i, cnt);
#pragma unroll
      for (int c = 0; c < NC; ++c) run[c] += cnt[c];
    }
  }
  uint32_t total[NC];
  block_exclusive_scan<NC>(run, total);
#pragma unroll
  for (int c = 0; c < NC; ++c) run[c] += s_pre[c];
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const uint64_t i = first + q;
    if (i < n) {
      uint32_t cnt[NC];
      op.count(i, cnt);
      op.emit(i, run, cnt, tot);
#pragma unroll
      for (int c = 0; c < NC; ++c) run[c] += cnt[c];
    }
  }
}

// Scratch for one scan of up to `n_cap` items with NC counters.
struct ScanScratch {
  DevBuf<uint32_t> tiles;
  void ensure(uint64_t n_cap, int nc, int tile = kScanTile) {
    tiles.ensure(static_cast<size_t>(ceil_div(n_cap > 0 ? n_cap : 1, tile)) * nc);
  }
};

// Run the three phases on `stream`. d_totals (nullable, device, NC u64) gets
// the grand totals. n_cap bounds the grid; d_n (nullable) is the live count.
template <class Op>
void run_scan(Ctx* ctx, const Op& op, uint64_t n_cap, const uint64_t* d_n, ScanScratch& s,
              uint64_t* d_totals, cudaStream_t stream) {
  constexpr int NC = Op::NC;
  if (n_cap == 0) {
    if (d_totals) FSX_CUDA(cudaMemsetAsync(d_totals, 0, sizeof(uint64_t) * NC, stream));
    return;
  }
  constexpr int kTile = kScanThreads * ScanIPT<Op>::v;
  s.ensure(n_cap, NC, kTile);
  const unsigned tiles = ceil_div(n_cap, kTile);
  FSX_LAUNCH(ctx, k_tile_reduce<Op>, tiles, kScanThreads, 0, stream, op, n_cap, d_n, s.tiles.p);
  FSX_LAUNCH(ctx, k_tile_emit<Op>, tiles, kScanThreads, 0, stream, op, n_cap, d_n, s.tiles.p, tiles,
             d_totals);
}

}  // namespace fsx
