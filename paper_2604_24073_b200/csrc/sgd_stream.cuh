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
// Here the plan (built on the side lane, a whole iteration ahead at one rank)
// flattens the update into ring entries — per row its table row (when
// updated in place) then one gradient row per occurrence — so the update
// kernel's producer has no index chain left: it reads 32 entry addresses
// with one coalesced load per batch (the next batch's in flight) and issues
// one bulk copy per free slot of its warp's ring of R row-sized
// shared-memory slots; the consumer folds the slots in order. The ring keeps
// R rows (8-16 KB) in flight per warp, so an SM holds ~160 KB of row traffic
// in flight — above what HBM3e needs to run at full bandwidth.
//
// Work: the items (rows, and the fixed `chunk`-occurrence chunks of hot rows)
// are in row order; each warp takes the items whose cost (entries + a fixed
// per-item cost) falls in its equal share — a balanced static split with no
// queue. Chunks of hot rows leave f64 partials that k_sgd_combine adds in
// chunk order right after (the association of k_sgd_warp / k_sgd_flat), so
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
// 16-byte async global -> shared copy (LDGSTS, L2 only) and the arrive that
// fires on the barrier once this thread's earlier async copies have landed
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
template <class V>
__device__ __forceinline__ void lds_vec(uint32_t addr, V& out) {
  static_assert(sizeof(V) == 16, "16-byte vectors");
  uint32_t* w = reinterpret_cast<uint32_t*>(&out);
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
               : "r"(addr)
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

__device__ __forceinline__ uint64_t item_ent(const SgdItem* it) {
  return static_cast<uint64_t>(reinterpret_cast<uintptr_t>(it->g0));
}

// ring entries of an item: the destination table row first when the item
// updates it in place (single-chunk item, table mode), then one gradient row
// per occurrence. Items whose destination lies outside the shard do nothing.
__device__ __forceinline__ uint32_t item_entries(const SgdItem& it, bool table_mode) {
  const bool single = (it.q & kSgdSingleChunk) != 0;
  if (single && !it.dst) return 0;
  return (single && table_mode ? 1u : 0u) + (it.ke - it.kb);
}

// Ring entry -> source address: absolute (table rows, resolved gradient
// rows) or an occurrence index tagged in bit 0 (plain gradient arrays: one
// multiply-add, no load).
template <class T>
__device__ __forceinline__ const void* entry_src(const SgdArgs<T>& a, uint64_t tag) {
  if (tag & 1u) return a.gr.row(static_cast<uint32_t>(tag >> 1));
  return reinterpret_cast<const void*>(static_cast<uintptr_t>(tag));
}

// Work split: an item's cost is its entries plus kStreamItemCost (the
// per-item work: descriptor, table-row store or partial, loop setup); warp w
// takes the items whose cost prefix ent(i) + kStreamItemCost * i falls in
// its equal share — a balanced static split. (Measured on B200, config 4 at
// one rank, kernel alone: static 80 us; the same work handed out from one
// atomic counter 100-108 us — ~3,000 warps serialise on it.)
__device__ __forceinline__ uint64_t first_item_at(const SgdItem* work, uint64_t n, uint64_t target, unsigned lane) {
  uint64_t lo = 0, hi = n;
  while (hi - lo > 32) {
    const uint64_t step = (hi - lo + 31) / 32;
    const uint64_t probe = lo + (lane + 1) * step - 1;
    const bool below = probe < hi && item_ent(work + probe) + kStreamItemCost * probe < target;
    const uint32_t m = __ballot_sync(0xffffffffu, below);
    const uint64_t nlo = lo + static_cast<uint64_t>(__popc(m)) * step;
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  const bool below = lo + lane < hi && item_ent(work + lo + lane) + kStreamItemCost * (lo + lane) < target;
  return lo + __popc(__ballot_sync(0xffffffffu, below));
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// kBulk: one bulk copy (TMA) per ring entry; else the warp moves each entry
// with 16-byte LDGSTS. kFused: the warp that completes a hot row's last
// chunk adds the row's partials (else k_sgd_combine runs after the kernel).
template <class T, int NV, int R, int MINB, bool kBulk, bool kFused>
__global__ void __launch_bounds__(128, MINB) k_sgd_stream(SgdArgs<T> a, uint32_t rb, uint32_t* __restrict__ done,
                                                         unsigned long long* span) {
  FSX_PDL_ENTER();
  // span (fsx_ctx_kernel_span): [0] ~first warp start, [1] last warp end (ns)
  if (span && (threadIdx.x & 31u) == 0) atomicMax(span, ~global_ns());
  constexpr int VE = static_cast<int>(16 / sizeof(T));
  using V = VecOf<T, VE>;
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned lane = threadIdx.x & 31u, wib = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  // layout: [wpc][R] mbarriers, then [wpc][R] slots of rb bytes
  const uint32_t bar0 = smem_addr(smem) + wib * R * 8;
  const uint32_t slot0 = smem_addr(smem) + ((wpc * R * 8 + 127) & ~127u) + wib * R * rb;
  if (lane < static_cast<unsigned>(R)) mbar_init(bar0 + 8 * lane, kBulk ? 1u : 32u);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();

  const bool table_mode = a.seg_out == nullptr;
  const uint32_t dim = a.g.dim;
  const uint32_t vpr = dim / VE;
  const uint64_t W = static_cast<uint64_t>(gridDim.x) * wpc;
  const uint64_t w = static_cast<uint64_t>(blockIdx.x) * wpc + wib;
  const uint64_t nitems = *a.d_work_n, nent = *a.d_single_n;
  const uint64_t cost = nent + kStreamItemCost * nitems;
  const uint64_t i0 = first_item_at(a.work, nitems, cost * w / W, lane);
  const uint64_t i1 = first_item_at(a.work, nitems, cost * (w + 1) / W, lane);
  const uint64_t e_end = i1 < nitems ? item_ent(a.work + i1) : nent;

  // ---- producer: entries [e_cur, e_end) in batches of 32, one load per
  // lane, the next batch's tags in flight while the current batch issues ----
  uint64_t e_cur = i0 < nitems ? item_ent(a.work + i0) : e_end;
  uint64_t bbase = e_cur;
  uint64_t tag_cur = bbase + lane < e_end ? a.ent[bbase + lane] : 0;
  uint64_t tag_nxt = bbase + 32 + lane < e_end ? a.ent[bbase + 32 + lane] : 0;
  uint32_t issued = 0, consumed = 0;
  auto produce = [&]() {
    uint32_t free_slots = R - (issued - consumed);
    while (free_slots && e_cur < e_end) {
      const uint32_t off = static_cast<uint32_t>(e_cur - bbase);
      const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(min(free_slots, 32u - off)), e_end - e_cur));
      if constexpr (kBulk) {
        if (lane >= off && lane < off + n) {
          const uint32_t slot = (issued + (lane - off)) % R;
          mbar_expect_tx(bar0 + 8 * slot, rb);
          bulk_g2s(slot0 + slot * rb, entry_src(a, tag_cur), rb, bar0 + 8 * slot);
        }
      } else {
        // the whole warp moves each entry, 16 bytes per lane per vector, and
        // every lane arrives on the slot's barrier when its copies landed
        const char* src = static_cast<const char*>(entry_src(a, tag_cur));
        for (uint32_t j = 0; j < n; ++j) {
          const char* sj = reinterpret_cast<const char*>(
              __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(src), off + j));
          const uint32_t slot = (issued + j) % R;
#pragma unroll
          for (int v = 0; v < NV; ++v)
            if (lane + 32u * v < vpr) cp_async16(slot0 + slot * rb + (lane + 32u * v) * 16u, sj + (lane + 32u * v) * 16u);
          cp_async_arrive(bar0 + 8 * slot);
        }
      }
      issued += n;
      e_cur += n;
      free_slots -= n;
      if (e_cur - bbase == 32) {
        bbase += 32;
        tag_cur = tag_nxt;
        tag_nxt = bbase + 32 + lane < e_end ? a.ent[bbase + 32 + lane] : 0;
      }
    }
  };
  produce();

  // ---- consumer: items in order (the next descriptor in flight) ----
  // slot k: shared address slot0 + k * rb; lane l reads 16-byte vectors
  // l, l + 32, ... of the row (conflict-free)
  auto take = [&](V (&g)[NV]) {
    const uint32_t slot = consumed % R;
    mbar_wait(bar0 + 8 * slot, (consumed / R) & 1u);
    const uint32_t addr = slot0 + slot * rb + lane * 16u;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (lane + 32u * v < vpr) lds_vec(addr + v * 512u, g[v]);
    ++consumed;
  };
  SgdItem nx{};
  if (i0 < i1) nx = a.work[i0];
  for (uint64_t ci = i0; ci < i1; ++ci) {
    const SgdItem it = nx;
    if (ci + 1 < i1) nx = a.work[ci + 1];
    const uint32_t ne = item_entries(it, table_mode);
    if (ne == 0) continue;
    const bool single = (it.q & kSgdSingleChunk) != 0;
    const bool has_old = single && table_mode;
    V old[NV];
    if (has_old) {
      take(old);
      __syncwarp();  // every lane has read the slot: it may be refilled
    }
    double acc[NV][VE];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int x = 0; x < VE; ++x) acc[v][x] = 0.0;
    const uint32_t ng = ne - (has_old ? 1u : 0u);
    for (uint32_t e = 0; e < ng; ++e) {
      V g0[NV];
      take(g0);
      __syncwarp();  // every lane has read the slot: it may be refilled
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int x = 0; x < VE; ++x) acc[v][x] = __dadd_rn(acc[v][x], static_cast<double>(g0[v].v[x]));
      if (issued - consumed <= R / 2) produce();
    }
    if (single) {
      T* dst = reinterpret_cast<T*>(it.dst);
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (lane + 32u * v < vpr) sgd_store_vec<T, VE>(a, it.u, dst, (lane + 32u * v) * VE, acc[v], old[v]);
      continue;
    }
    // one chunk of a hot row: its f64 partial
    const uint64_t base = a.part_base[it.u];
    double* pp = a.partials + (base + it.q) * dim;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (lane + 32u * v < vpr) {
        double2* p2 = reinterpret_cast<double2*>(pp + (lane + 32u * v) * VE);
#pragma unroll
        for (int x = 0; x < VE; x += 2) p2[x / 2] = make_double2(acc[v][x], acc[v][x + 1]);
      }
    if constexpr (kFused) {
      // the warp completing the row's last chunk adds the partials in chunk
      // order, 4 partials' loads in flight per step
      __syncwarp();
      unsigned arrived = 0;
      if (lane == 0) {
        __threadfence();
        arrived = atomicAdd(done + it.u, 1u);
      }
      arrived = __shfl_sync(0xffffffffu, arrived, 0);
      const uint32_t len = a.rs.seg_start[it.u + 1] - a.rs.seg_start[it.u];
      const uint32_t nch = (len + a.chunk - 1) / a.chunk;
      if (arrived == nch - 1) {
        __threadfence();
        const double* pb = a.partials + base * dim;
#pragma unroll
        for (int v = 0; v < NV; ++v)
          if (lane + 32u * v < vpr) {
            const uint32_t col = (lane + 32u * v) * VE;
            double c[VE];
#pragma unroll
            for (int x = 0; x < VE; ++x) c[x] = 0.0;
            for (uint32_t q0 = 0; q0 < nch; q0 += 4) {
              double2 t[4][VE / 2];
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (q0 + j < nch)
#pragma unroll
                  for (int x = 0; x < VE / 2; ++x)
                    t[j][x] = __ldcg(reinterpret_cast<const double2*>(pb + static_cast<uint64_t>(q0 + j) * dim + col) + x);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (q0 + j < nch)
#pragma unroll
                  for (int x = 0; x < VE / 2; ++x) {
                    c[2 * x] = __dadd_rn(c[2 * x], t[j][x].x);
                    c[2 * x + 1] = __dadd_rn(c[2 * x + 1], t[j][x].y);
                  }
            }
            sgd_apply_vec<T, VE>(a, it.u, col, c);
          }
        if (lane == 0) done[it.u] = 0;
      }
    }
  }
  // reduce-only outputs may be peer windows (direct CO_G): visible system-wide
  // before the stream's flag write that follows the kernel
  if (!table_mode) __threadfence_system();
  if (span && lane == 0) atomicMax(span + 1, global_ns());
}

}  // namespace fsx
