// Stable LSD radix sort of (key, u32 payload) pairs, up-to-9-bit digits
// (passes = ceil(nbits / 9); 27-bit row keys sort in 3 passes).
//
// Per digit pass, three launches:
//   k_radix_hist    per-2048-key tile digit histogram; equal digits inside a
//                   warp are aggregated with __match_any_sync so Zipf-hot keys
//                   cost one shared atomic per warp, not one per key
//   k_radix_rows    exclusive scan of each digit's row of tile counts (one
//                   warp per digit) and the digit totals
//   k_radix_scatter stable rank inside the tile: each warp walks its
//                   contiguous 256-key chunk in 32-key rounds; match_any gives
//                   the equal-digit peers, popc(peers & lanemask_lt) the rank
//                   among them, a per-warp shared counter the running offset;
//                   a per-digit prefix over warps then orders the warps.
// Stability (index order is preserved inside every digit bucket) is what makes
// the owner's per-row gradient order equal the reference's (source, position)
// order (embedding.cpp:159-166).
// Only the significant bits are sorted: callers pass nbits (e.g. 27 for the
// local row index of an 80M-row shard), giving ceil(nbits/8) passes.
#pragma once

#include "scan.cuh"

namespace fsx {

constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixWarpItems = 128;  // per warp per tile (1024-key tiles: >= 1 CTA per SM at 150K keys)
constexpr int kRadixTile = kRadixWarps * kRadixWarpItems;
constexpr int kRadixRounds = kRadixWarpItems / 32;
constexpr int kRadixMaxBits = 9;
constexpr int kRadixBins = 1 << kRadixMaxBits;  // 512
constexpr int kBinsPerThread = kRadixBins / kRadixThreads;

template <class K>
__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const K* __restrict__ keys,
                                                              uint64_t n_cap, const uint64_t* d_n,
                                                              int shift, unsigned mask, uint32_t* counts,
                                                              unsigned tiles) { FSX_PDL_ENTER();
  __shared__ uint32_t hist[kRadixBins];
  const uint64_t n = scan_n(n_cap, d_n);
  for (int b = 0; b < kBinsPerThread; ++b) hist[threadIdx.x + b * kRadixThreads] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kRadixTile + warp * kRadixWarpItems;
#pragma unroll 4
  for (int r = 0; r < kRadixRounds; ++r) {
    const uint64_t i = base + r * 32 + lane;
    const unsigned d = i < n ? static_cast<unsigned>((keys[i] >> shift) & mask) : 0xffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (d <= mask && (peers & lanemask_lt()) == 0) atomicAdd(&hist[d], __popc(peers));
  }
  __syncthreads();
  for (int b = 0; b < kBinsPerThread; ++b) {
    const unsigned d = threadIdx.x + b * kRadixThreads;
    if (d <= mask) counts[static_cast<uint64_t>(d) * tiles + blockIdx.x] = hist[d];
  }
}

// one warp per digit: exclusive scan of counts[d][0..tiles) in place, total[d]
static __global__ void __launch_bounds__(256) k_radix_rows(uint32_t* __restrict__ counts,
                                                           unsigned tiles, unsigned bins,
                                                           uint32_t* __restrict__ total) { FSX_PDL_ENTER();
  const unsigned lane = threadIdx.x & 31u;
  const unsigned d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (d >= bins) return;
  uint32_t* row = counts + static_cast<uint64_t>(d) * tiles;
  uint32_t carry = 0;
  for (unsigned t0 = 0; t0 < tiles; t0 += 32) {
    const unsigned t = t0 + lane;
    const uint32_t v = t < tiles ? row[t] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= static_cast<unsigned>(o)) x += y;
    }
    if (t < tiles) row[t] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) total[d] = carry;
}

template <class K>
__global__ void __launch_bounds__(kRadixThreads) k_radix_scatter(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
    uint32_t* __restrict__ vout, uint64_t n_cap, const uint64_t* d_n, int shift, unsigned mask,
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ digit_total, unsigned tiles) { FSX_PDL_ENTER();
  __shared__ uint32_t wcount[kRadixWarps][kRadixBins];
  __shared__ uint32_t tile_off[kRadixBins];
  __shared__ uint32_t wsum[kRadixWarps];
  const uint64_t n = scan_n(n_cap, d_n);
  const uint64_t tile_base = static_cast<uint64_t>(blockIdx.x) * kRadixTile;
  if (tile_base >= n) return;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const unsigned bins = mask + 1;
  for (int w = 0; w < kRadixWarps; ++w)
    for (int b = 0; b < kBinsPerThread; ++b) wcount[w][threadIdx.x + b * kRadixThreads] = 0;
  {
    // digit base = exclusive scan of the digit totals; each thread owns
    // kBinsPerThread consecutive digits
    uint32_t tot[kBinsPerThread], own = 0;
    for (int b = 0; b < kBinsPerThread; ++b) {
      const unsigned d = threadIdx.x * kBinsPerThread + b;
      tot[b] = d < bins ? digit_total[d] : 0u;
      own += tot[b];
    }
    uint32_t x = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= static_cast<unsigned>(o)) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t run = x - own;
    for (unsigned w = 0; w < warp; ++w) run += wsum[w];
    for (int b = 0; b < kBinsPerThread; ++b) {
      const unsigned d = threadIdx.x * kBinsPerThread + b;
      if (d < bins) tile_off[d] = run + offsets[static_cast<uint64_t>(d) * tiles + blockIdx.x];
      run += tot[b];
    }
  }
  __syncthreads();
  const uint64_t base = tile_base + warp * kRadixWarpItems;
  K k[kRadixRounds];
  uint32_t v[kRadixRounds], rk[kRadixRounds];
  unsigned dg[kRadixRounds];
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const uint64_t i = base + r * 32 + lane;
    const bool valid = i < n;
    k[r] = valid ? kin[i] : K(0);
    v[r] = valid ? (vin ? vin[i] : static_cast<uint32_t>(i)) : 0u;
    dg[r] = valid ? static_cast<unsigned>((k[r] >> shift) & mask) : 0xffffu;
  }
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const unsigned d = dg[r];
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned before = __popc(peers & lanemask_lt());
    uint32_t run = d <= mask ? wcount[warp][d] : 0u;
    rk[r] = run + before;
    __syncwarp();
    if (d <= mask && before == 0) wcount[warp][d] = run + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int b = 0; b < kBinsPerThread; ++b) {
    const unsigned d = threadIdx.x + b * kRadixThreads;
    uint32_t run = 0;
    for (int w = 0; w < kRadixWarps; ++w) {
      const uint32_t x = wcount[w][d];
      wcount[w][d] = run;
      run += x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const unsigned d = dg[r];
    if (d <= mask) {
      const uint32_t pos = tile_off[d] + wcount[warp][d] + rk[r];
      kout[pos] = k[r];
      vout[pos] = v[r];
    }
  }
}

// ---- onesweep variant (FSX_ONESWEEP, default on) ------------------------------
// One launch computes every pass's global digit histogram (one read of the
// keys); each pass is then ONE launch: CTAs take tiles in order from a
// counter, rank keys inside the tile exactly as k_radix_scatter does, publish
// the tile's per-digit count, and find the count of all earlier tiles by
// decoupled look-back over those published words (aggregate / inclusive
// flags) instead of a separate per-tile histogram + scan. 1 + passes launches
// instead of 3 * passes; same stable order.
constexpr int kOsMaxPasses = 8;
constexpr uint32_t kOsAgg = 1u << 30, kOsIncl = 2u << 30, kOsCount = (1u << 30) - 1u;

template <class K>
__global__ void __launch_bounds__(kRadixThreads) k_os_hist(const K* __restrict__ keys, uint64_t n_cap,
                                                           const uint64_t* d_n, int passes, int dbits,
                                                           uint32_t* __restrict__ hist) { FSX_PDL_ENTER();
  __shared__ uint32_t h[kOsMaxPasses][kRadixBins];
  for (int i = threadIdx.x; i < kOsMaxPasses * kRadixBins; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint64_t n = scan_n(n_cap, d_n);
  const unsigned mask = (1u << dbits) - 1u;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n_round = (n + 31) & ~uint64_t{31};  // whole warps through match_any
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_round; i += stride) {
    const bool valid = i < n;
    const K k = valid ? keys[i] : K(0);
    for (int ps = 0; ps < passes; ++ps) {
      const unsigned d = valid ? static_cast<unsigned>((k >> (ps * dbits)) & mask) : 0xffffu;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      if (valid && (peers & lanemask_lt()) == 0) atomicAdd(&h[ps][d], __popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadixBins; i += blockDim.x) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

template <class K>
__global__ void __launch_bounds__(kRadixThreads) k_os_scatter(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
    uint32_t* __restrict__ vout, uint64_t n_cap, const uint64_t* d_n, int shift, unsigned mask,
    const uint32_t* __restrict__ digit_total, uint32_t* status, uint32_t* tile_ctr) { FSX_PDL_ENTER();
  __shared__ uint32_t wcount[kRadixWarps][kRadixBins];
  __shared__ uint32_t tile_off[kRadixBins];
  __shared__ uint32_t wsum[kRadixWarps];
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int w = 0; w < kRadixWarps; ++w)
    for (int b = 0; b < kBinsPerThread; ++b) wcount[w][threadIdx.x + b * kRadixThreads] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t n = scan_n(n_cap, d_n);
  const uint64_t tile_base = static_cast<uint64_t>(tile) * kRadixTile;
  if (tile_base >= n) return;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const unsigned bins = mask + 1;
  // digit base = exclusive scan of the pass's global digit totals (each
  // thread owns kBinsPerThread consecutive digits)
  {
    uint32_t tot[kBinsPerThread], own = 0;
    for (int b = 0; b < kBinsPerThread; ++b) {
      const unsigned d = threadIdx.x * kBinsPerThread + b;
      tot[b] = d < bins ? digit_total[d] : 0u;
      own += tot[b];
    }
    uint32_t x = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= static_cast<unsigned>(o)) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t run = x - own;
    for (unsigned w = 0; w < warp; ++w) run += wsum[w];
    for (int b = 0; b < kBinsPerThread; ++b) {
      const unsigned d = threadIdx.x * kBinsPerThread + b;
      if (d < bins) tile_off[d] = run;
      run += tot[b];
    }
  }
  const uint64_t base = tile_base + warp * kRadixWarpItems;
  K k[kRadixRounds];
  uint32_t v[kRadixRounds], rk[kRadixRounds];
  unsigned dg[kRadixRounds];
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const uint64_t i = base + r * 32 + lane;
    const bool valid = i < n;
    k[r] = valid ? kin[i] : K(0);
    v[r] = valid ? (vin ? vin[i] : static_cast<uint32_t>(i)) : 0u;
    dg[r] = valid ? static_cast<unsigned>((k[r] >> shift) & mask) : 0xffffu;
  }
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const unsigned d = dg[r];
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned before = __popc(peers & lanemask_lt());
    uint32_t run = d <= mask ? wcount[warp][d] : 0u;
    rk[r] = run + before;
    __syncwarp();
    if (d <= mask && before == 0) wcount[warp][d] = run + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: warps' exclusive offsets, the tile's count, then look-back
  uint32_t* my = status + static_cast<uint64_t>(tile) * kRadixBins;
  for (int b = 0; b < kBinsPerThread; ++b) {
    const unsigned d = threadIdx.x + b * kRadixThreads;
    uint32_t run = 0;
    for (int w = 0; w < kRadixWarps; ++w) {
      const uint32_t x = wcount[w][d];
      wcount[w][d] = run;
      run += x;
    }
    if (d >= bins) continue;
    if (tile == 0) {
      *reinterpret_cast<volatile uint32_t*>(my + d) = kOsIncl | run;
      continue;
    }
    *reinterpret_cast<volatile uint32_t*>(my + d) = kOsAgg | run;
    // look-back, 8 predecessors' words loaded at once (independent loads:
    // one round trip per 8 tiles instead of one per tile), consumed in order
    // until an inclusive prefix; an unpublished word is re-read
    uint32_t acc = 0;
    for (int64_t t = static_cast<int64_t>(tile) - 1; t >= 0;) {
      constexpr int kLook = 8;
      uint32_t st[kLook];
#pragma unroll
      for (int j = 0; j < kLook; ++j)
        st[j] = t - j >= 0 ? *reinterpret_cast<volatile const uint32_t*>(status + static_cast<uint64_t>(t - j) * kRadixBins + d)
                           : 0u;
      int j = 0;
      bool incl = false;
      for (; j < kLook && t - j >= 0; ++j) {
        if ((st[j] & ~kOsCount) == 0) break;  // not published yet: spin from here
        acc += st[j] & kOsCount;
        if (st[j] & kOsIncl) {
          incl = true;
          break;
        }
      }
      if (incl) break;
      t -= j;
    }
    *reinterpret_cast<volatile uint32_t*>(my + d) = kOsIncl | (acc + run);
    tile_off[d] += acc;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const unsigned d = dg[r];
    if (d <= mask) {
      const uint32_t pos = tile_off[d] + wcount[warp][d] + rk[r];
      kout[pos] = k[r];
      vout[pos] = v[r];
    }
  }
}

struct RadixScratch {
  DevBuf<uint32_t> counts;
  DevBuf<uint32_t> os;  // onesweep: [passes][tiles][bins] status | [passes][bins] hist | [passes] tile counters
  void ensure_onesweep(uint64_t n_cap, int passes) {
    const uint64_t tiles = ceil_div(n_cap > 0 ? n_cap : 1, kRadixTile);
    os.ensure(static_cast<size_t>(passes) * (tiles + 1) * kRadixBins + 32);
  }
};

// Sorts (keys, vals) by bits [0, nbits) stably. `vals` may be null: payload
// is then the input index. Ping-pongs between (k0,v0) and (k1,v1); returns
// the pair holding the result via out pointers. n_cap sizes the grid, d_n is
// the live count (nullable).
template <class K>
void radix_sort_pairs(Ctx* ctx, K* k0, uint32_t* v0, K* k1, uint32_t* v1, uint64_t n_cap,
                      const uint64_t* d_n, int nbits, RadixScratch& s, cudaStream_t stream,
                      K** k_out, uint32_t** v_out, const uint32_t* v_init = nullptr) {
  if (nbits < 1) nbits = 1;
  const int passes = (nbits + kRadixMaxBits - 1) / kRadixMaxBits;
  const int dbits = (nbits + passes - 1) / passes;
  const unsigned mask = (1u << dbits) - 1u, bins = mask + 1;
  const unsigned tiles = ceil_div(n_cap > 0 ? n_cap : 1, kRadixTile);
  s.counts.ensure(static_cast<size_t>(tiles) * kRadixBins + kRadixBins);
  uint32_t* totals = s.counts.p + static_cast<size_t>(tiles) * kRadixBins;
  K* kin = k0;
  K* kout = k1;
  const uint32_t* vin = v_init;
  uint32_t* vbuf_in = v0;
  uint32_t* vout = v1;
  if (n_cap == 0) {
    *k_out = k0;
    *v_out = v0;
    return;
  }
  if (ctx->onesweep && passes <= kOsMaxPasses) {
    const unsigned tiles_os = tiles;
    s.ensure_onesweep(n_cap, passes);
    uint32_t* status = s.os.p;
    uint32_t* hist = status + static_cast<size_t>(passes) * tiles_os * kRadixBins;
    uint32_t* ctr = hist + static_cast<size_t>(passes) * kRadixBins;
    FSX_CUDA(cudaMemsetAsync(s.os.p, 0,
                             (static_cast<size_t>(passes) * (tiles_os + 1) * kRadixBins + 32) * sizeof(uint32_t),
                             stream));
    FSX_LAUNCH(ctx, k_os_hist<K>, grid_for(ctx, n_cap, kRadixThreads, 2), kRadixThreads, 0, stream, kin, n_cap,
               d_n, passes, dbits, hist);
    for (int p = 0; p < passes; ++p) {
      FSX_LAUNCH(ctx, k_os_scatter<K>, tiles_os, kRadixThreads, 0, stream, kin, vin, kout, vout, n_cap, d_n,
                 dbits * p, mask, hist + static_cast<size_t>(p) * kRadixBins,
                 status + static_cast<size_t>(p) * tiles_os * kRadixBins, ctr + p);
      K* kt = kin;
      kin = kout;
      kout = kt;
      vin = vout;
      uint32_t* vt = vbuf_in;
      vbuf_in = vout;
      vout = vt;
    }
    *k_out = kin;
    *v_out = vbuf_in;
    return;
  }
  for (int p = 0; p < passes; ++p) {
    const int shift = dbits * p;
    FSX_LAUNCH(ctx, k_radix_hist<K>, tiles, kRadixThreads, 0, stream, kin, n_cap, d_n, shift, mask,
               s.counts.p, tiles);
    FSX_LAUNCH(ctx, k_radix_rows, ceil_div(bins, 8), 256, 0, stream, s.counts.p, tiles, bins, totals);
    FSX_LAUNCH(ctx, k_radix_scatter<K>, tiles, kRadixThreads, 0, stream, kin, vin, kout, vout,
               n_cap, d_n, shift, mask, s.counts.p, totals, tiles);
    // next pass reads what this one wrote
    K* kt = kin;
    kin = kout;
    kout = kt;
    vin = vout;
    uint32_t* vt = vbuf_in;
    vbuf_in = vout;
    vout = vt;
  }
  *k_out = kin;
  *v_out = vbuf_in;
}

inline int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b > 0 ? b : 1;
}

}  // namespace fsx
