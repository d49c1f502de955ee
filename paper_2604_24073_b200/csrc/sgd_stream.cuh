// k_sgd_stream: the deterministic segmented SGD of kernels.cuh (same work
// lists, same per-row association, same arithmetic) as ONE persistent kernel
// whose row traffic is staged through shared memory by bulk asynchronous
// copies (cp.async.bulk, the 1-D TMA path: SASS UBLKCP) completing on
// mbarriers.
//
// Why: the update is a gather of gradient rows (one per occurrence, in sorted
// order) plus a read-modify-write of each updated table row. In k_sgd_warp /
// k_sgd_single every row moved through registers, so the bytes a warp could
// keep in flight were bounded by its registers (100 per thread: 2 CTAs per
// SM, 17% occupancy) and every item began with a dependent index chain
// (item -> perm -> gradient row) that stalled the warp.
// Here each warp owns a ring of R row-sized shared-memory slots. A producer
// step resolves the pointers of the next 32 ring entries in parallel — one
// lane per entry, entries spanning as many items as they cover (a single-row
// item is 2 entries: the table row and its gradient row) — and issues one
// bulk copy per free slot; the consumer step folds the slots in order. The
// ring keeps R rows (8-16 KB) in flight per warp with ~60 registers, so an
// SM holds ~190 KB of row traffic in flight — above what HBM3e needs to run
// at full bandwidth — and the index chain of the next batch resolves while
// the current batch's rows are still landing.
//
// Work: each warp takes an equal share of the one-occurrence rows
// (`singles`) and the work items (rows of 2+ occurrences, and the fixed
// `chunk`-occurrence chunks of hot rows) whose first occurrence falls in its
// equal share of the sorted occurrence range — a balanced static split with
// no queue. Multi-chunk rows leave f64 partials; the warp completing a row's
// last chunk adds them in chunk order (as k_sgd_warp / k_sgd_combine), so
// results are bit-identical to the other update kernels.
#pragma once

#include "kernels.cuh"

namespace fsx {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
// arm the barrier's phase with the byte count the bulk copy will complete
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}

// first work item whose first occurrence is >= target (items are in sorted
// occurrence order): a 32-ary search, one probe per lane per round
__device__ __forceinline__ uint64_t first_item_at(const SgdItem* work, uint64_t n, uint64_t target, unsigned lane) {
  uint64_t lo = 0, hi = n;
  while (hi - lo > 32) {
    const uint64_t step = (hi - lo + 31) / 32;
    const uint64_t probe = lo + (lane + 1) * step - 1;
    const bool below = probe < hi && work[probe].kb < target;
    const uint32_t m = __ballot_sync(0xffffffffu, below);
    const uint64_t nlo = lo + static_cast<uint64_t>(__popc(m)) * step;
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  const bool below = lo + lane < hi && work[lo + lane].kb < target;
  return lo + __popc(__ballot_sync(0xffffffffu, below));
}

template <class T>
struct StreamItems {
  const SgdItem* work;
  const SgdItem* singles;
  uint64_t w0, nwi, s0;  // this warp's work items [w0, w0+nwi), then singles from s0
  __device__ __forceinline__ const SgdItem* at(uint64_t v) const {
    return v < nwi ? work + w0 + v : singles + s0 + (v - nwi);
  }
};

// ring entries of an item: the destination table row first when the item
// updates it in place (single-chunk item, table mode), then one gradient row
// per occurrence. Items whose destination lies outside the shard do nothing.
__device__ __forceinline__ uint32_t item_entries(const SgdItem& it, bool table_mode) {
  const bool single = (it.q & kSgdSingleChunk) != 0;
  if (single && !it.dst) return 0;
  return (single && table_mode ? 1u : 0u) + (it.ke - it.kb);
}

template <class T, int NV, int R>
__global__ void __launch_bounds__(128, 6) k_sgd_stream(SgdArgs<T> a, uint32_t* __restrict__ done, uint32_t rb) {
  FSX_PDL_ENTER();
  constexpr unsigned kFull = 0xffffffffu;
  constexpr int VE = static_cast<int>(16 / sizeof(T));
  using V = VecOf<T, VE>;
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned lane = threadIdx.x & 31u, wib = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const uint32_t bar0 = smem_addr(smem) + wib * R * 8;
  const uint32_t slot0 = smem_addr(smem) + ((wpc * R * 8 + 127) & ~127u) + wib * R * rb;
  const unsigned char* slots = smem + ((wpc * R * 8 + 127) & ~127u) + wib * R * rb;
  if (lane < static_cast<unsigned>(R)) mbar_init(bar0 + 8 * lane, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();

  const bool table_mode = a.seg_out == nullptr;
  const uint32_t dim = a.g.dim;
  const uint32_t vpr = dim / VE;
  const uint64_t W = static_cast<uint64_t>(gridDim.x) * wpc;
  const uint64_t w = static_cast<uint64_t>(blockIdx.x) * wpc + wib;
  const uint64_t nwork = *a.d_work_n, nsing = *a.d_single_n;
  const uint64_t nocc = a.rs.seg_start[*a.rs.d_u];
  StreamItems<T> items{a.work, a.singles, 0, 0, nsing * w / W};
  const uint64_t s1 = nsing * (w + 1) / W;
  items.w0 = first_item_at(a.work, nwork, nocc * w / W, lane);
  items.nwi = first_item_at(a.work, nwork, nocc * (w + 1) / W, lane) - items.w0;
  const uint64_t nitems = items.nwi + (s1 - items.s0);

  // ---- producer state: cursor (item pi, entry pk), resolved batch ----
  uint64_t pi = 0;
  uint32_t pk = 0;
  const char* bptr = nullptr;  // lane l: source of batch entry l
  uint32_t bcnt = 0, boff = 0;  // batch size, entries already issued
  uint32_t issued = 0, consumed = 0;

  // resolve the next (up to) 32 entries: lane j reads item pi + j, a scan of
  // the entry counts gives each lane l its entry's item and offset
  auto resolve = [&]() {
    bcnt = 0;
    boff = 0;
    while (bcnt == 0 && pi < nitems) {
      SgdItem it{};
      const bool have = pi + lane < nitems;
      if (have) it = *items.at(pi + lane);
      uint32_t n = have ? item_entries(it, table_mode) : 0u;
      if (lane == 0) n -= pk;
      uint32_t incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= static_cast<unsigned>(o)) incl += y;
      }
      const uint32_t total = __shfl_sync(kFull, incl, 31);
      const uint32_t cnt = min(total, 32u);
      if (cnt == 0) {  // 32 items with nothing to move
        pi += 32;
        pk = 0;
        continue;
      }
      // item of entry `lane`: first j with incl[j] > lane
      unsigned j = 0;
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const uint32_t v = __shfl_sync(kFull, incl, j + st - 1);
        if (v <= lane) j += st;
      }
      j = min(j, 31u);
      const uint32_t excl = __shfl_sync(kFull, incl - n, j);
      const uint32_t kb = __shfl_sync(kFull, it.kb, j);
      const bool has_old = __shfl_sync(kFull, (it.q & kSgdSingleChunk) && table_mode ? 1u : 0u, j) != 0;
      const char* dst = reinterpret_cast<const char*>(
          __shfl_sync(kFull, reinterpret_cast<unsigned long long>(it.dst), j));
      SgdItem first{};
      first.kb = kb;
      first.g0 = reinterpret_cast<const char*>(__shfl_sync(kFull, reinterpret_cast<unsigned long long>(it.g0), j));
      const uint32_t e = lane - excl + (j == 0 ? pk : 0u);  // entry inside its item
      const char* src = nullptr;
      if (lane < cnt) {
        if (has_old && e == 0) {
          src = dst;
        } else {
          const uint32_t k = kb + e - (has_old ? 1u : 0u);
          src = reinterpret_cast<const char*>(k == kb ? a.first_grad(first) : a.grad(k));
        }
      }
      bptr = src;
      bcnt = cnt;
      // advance past the batch: the last entry's item and offset
      const uint32_t jl = __shfl_sync(kFull, j, cnt - 1);
      const uint32_t el = __shfl_sync(kFull, e, cnt - 1);
      const uint32_t nl = __shfl_sync(kFull, have ? item_entries(it, table_mode) : 0u, jl);
      if (el + 1 == nl) {
        pi += jl + 1;
        pk = 0;
      } else {
        pi += jl;
        pk = el + 1;
      }
    }
  };
  // issue bulk copies into the free slots, in entry order
  auto produce = [&]() {
    while (true) {
      if (boff == bcnt) {
        resolve();
        if (bcnt == 0) return;
      }
      const uint32_t free_slots = R - (issued - consumed);
      if (free_slots == 0) return;
      const uint32_t n = min(free_slots, bcnt - boff);
      if (lane >= boff && lane < boff + n) {
        const uint32_t slot = (issued + (lane - boff)) % R;
        mbar_expect_tx(bar0 + 8 * slot, rb);
        bulk_g2s(slot0 + slot * rb, bptr, rb, bar0 + 8 * slot);
      }
      issued += n;
      boff += n;
    }
  };
  produce();

  // ---- consumer: items in order, entries in order ----
  for (uint64_t ci = 0; ci < nitems; ++ci) {
    const SgdItem it = *items.at(ci);
    const uint32_t ne = item_entries(it, table_mode);
    if (ne == 0) continue;
    const bool single = (it.q & kSgdSingleChunk) != 0;
    const bool has_old = single && table_mode;
    V old[NV];
    double acc[NV][VE];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int x = 0; x < VE; ++x) acc[v][x] = 0.0;
    for (uint32_t e = 0; e < ne; ++e) {
      const uint32_t slot = consumed % R;
      mbar_wait(bar0 + 8 * slot, (consumed / R) & 1u);
      const V* row = reinterpret_cast<const V*>(slots + static_cast<size_t>(slot) * rb);
      V g[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (lane + 32u * v < vpr) g[v] = row[lane + 32u * v];
      __syncwarp();  // every lane has read the slot: it may be refilled
      ++consumed;
      if (has_old && e == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) old[v] = g[v];
      } else {
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int x = 0; x < VE; ++x) acc[v][x] = __dadd_rn(acc[v][x], static_cast<double>(g[v].v[x]));
      }
      if (issued - consumed <= R / 2) produce();
    }
    if (single) {
      T* dst = reinterpret_cast<T*>(it.dst);
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (lane + 32u * v < vpr) sgd_store_vec<T, VE>(a, it.u, dst, (lane + 32u * v) * VE, acc[v], old[v]);
    } else {
      const uint64_t base = a.part_base[it.u];
      double* pp = a.partials + (base + (it.q & ~kSgdSingleChunk)) * dim;
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (lane + 32u * v < vpr) {
#pragma unroll
          for (int x = 0; x < VE; ++x) pp[(lane + 32u * v) * VE + x] = acc[v][x];
        }
      __syncwarp();
      unsigned arrived = 0;
      if (lane == 0) {
        __threadfence();
        arrived = atomicAdd(done + it.u, 1u);
      }
      arrived = __shfl_sync(kFull, arrived, 0);
      const uint32_t len = a.rs.seg_start[it.u + 1] - a.rs.seg_start[it.u];
      const uint32_t nch = (len + a.chunk - 1) / a.chunk;
      if (arrived == nch - 1) {  // last chunk of the row: combine in chunk order
        __threadfence();
        const double* pb = a.partials + base * dim;
#pragma unroll
        for (int v = 0; v < NV; ++v)
          if (lane + 32u * v < vpr) {
            const uint32_t col = (lane + 32u * v) * VE;
            double c[VE];
#pragma unroll
            for (int x = 0; x < VE; ++x) c[x] = 0.0;
            for (uint32_t q = 0; q < nch; ++q)
#pragma unroll
              for (int x = 0; x < VE; ++x) c[x] = __dadd_rn(c[x], __ldcg(pb + static_cast<uint64_t>(q) * dim + col + x));
            sgd_apply_vec<T, VE>(a, it.u, col, c);
          }
        if (lane == 0) done[it.u] = 0;
      }
    }
    if (issued == consumed) produce();  // ring drained (short items): refill before the next wait
  }
}

}  // namespace fsx
