// Sort + unique of an id multiset with everything the hot path derives from
// it: the stable permutation (sorted position -> occurrence), the sorted
// unique ids, the segment of each unique id in sorted order, and every
// occurrence's slot. Replaces sorted_unique + the lower_bound slotting of
// apply_gradients (embedding.cpp:12-16, 157-166).
#pragma once

#include "kernels.cuh"

namespace fsx {

// key[j] = id[j] / p  (local row index; same order as the global id because
// every id on a shard has the same residue) or the raw id. Invalid ids (not
// owned / out of range) are flagged when `validate`.
template <class K>
__global__ void k_make_keys(const uint64_t* __restrict__ ids, uint64_t n_cap, const uint64_t* d_n,
                            ShardGeom g, int local, int validate, K* __restrict__ keys,
                            DevErr* err) { FSX_PDL_ENTER();
  const uint64_t n = scan_n(n_cap, d_n);
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t id = ids[j];
    if (validate && !g.owns(id))
      report(err, id >= g.total_rows ? kErrRowRange : kErrNotOwned, id,
             id >= g.total_rows ? g.total_rows : static_cast<unsigned long long>(g.shard));
    keys[j] = static_cast<K>(local ? id / static_cast<uint64_t>(g.p) : id);
  }
}

struct SortedIds {
  // sort buffers (32- or 64-bit keys depending on nbits)
  DevBuf<uint32_t> k32a, k32b;
  DevBuf<uint64_t> k64a, k64b;
  DevBuf<uint32_t> va, vb;
  RadixScratch radix;
  ScanScratch scan;
  // results
  uint32_t* perm = nullptr;       // sorted position -> occurrence
  DevBuf<uint64_t> uniq;          // sorted unique keys (local index or raw id)
  DevBuf<uint64_t> uniq_g;        // sorted unique global ids
  DevBuf<uint32_t> seg_start;     // [U+1]
  DevBuf<uint32_t> inverse;       // occurrence -> slot
  DevBuf<uint64_t> d_counts;      // [0] live n (input), [1] U
  uint64_t cap = 0;

  void reserve(uint64_t n_cap) {
    if (n_cap <= cap && d_counts.p) return;
    cap = n_cap > 0 ? n_cap : 1;
    k32a.alloc(cap); k32b.alloc(cap); va.alloc(cap); vb.alloc(cap);
    k64a.release(); k64b.release();
    uniq.alloc(cap); uniq_g.alloc(cap); seg_start.alloc(cap + 1); inverse.alloc(cap);
    if (!d_counts.p) d_counts.alloc(4);
    // every scratch buffer is sized up front: a lazy cudaMalloc/cudaFree in
    // the middle of a multi-rank iteration can serialize the device
    radix.counts.ensure(static_cast<size_t>(ceil_div(cap, kRadixTile)) * kRadixBins + kRadixBins);
    radix.ensure_onesweep(cap, 4);
    scan.ensure(cap, 1);
  }
  void reserve64() {
    k64a.ensure(cap);
    k64b.ensure(cap);
  }
  uint64_t* d_n() { return d_counts.p; }
  uint64_t* d_u() { return d_counts.p + 1; }

  // ids: n_cap-capacity input, live count at *d_n() (caller fills it, or
  // pass host n via set_n). nbits: significant key bits.
  // keys_ready: k32a already holds the 32-bit keys (the caller's fused pass)
  void run(Ctx* ctx, const uint64_t* ids, uint64_t n_cap, const ShardGeom& g, bool local,
           bool validate, int nbits, cudaStream_t s, bool keys_ready = false) {
    reserve(n_cap);
    const unsigned grid = grid_for(ctx, n_cap, 256, 8);
    uint64_t* totals = d_counts.p + 1;  // scan total -> U
    if (nbits <= 32) {
      if (!keys_ready)
        FSX_LAUNCH(ctx, k_make_keys<uint32_t>, grid, 256, 0, s, ids, n_cap, d_n(), g, local ? 1 : 0,
                   validate ? 1 : 0, k32a.p, ctx->d_err);
      uint32_t* ko;
      radix_sort_pairs<uint32_t>(ctx, k32a.p, va.p, k32b.p, vb.p, n_cap, d_n(), nbits, radix, s,
                                 &ko, &perm);
      UniqueOp<uint32_t> op{ko, perm, d_n(), uniq.p, uniq_g.p, local ? (uint64_t)g.p : 1ull,
                            local ? (uint64_t)g.shard : 0ull, seg_start.p, inverse.p};
      run_scan(ctx, op, n_cap, d_n(), scan, totals, s);
    } else {
      if (k64a.n < cap || k64b.n < cap) raise(FSX_ERR_CONFIG, "fsx: 64-bit sort keys need reserve64()");
      FSX_LAUNCH(ctx, k_make_keys<uint64_t>, grid, 256, 0, s, ids, n_cap, d_n(), g, local ? 1 : 0,
                 validate ? 1 : 0, k64a.p, ctx->d_err);
      uint64_t* ko;
      radix_sort_pairs<uint64_t>(ctx, k64a.p, va.p, k64b.p, vb.p, n_cap, d_n(), nbits, radix, s,
                                 &ko, &perm);
      UniqueOp<uint64_t> op{ko, perm, d_n(), uniq.p, uniq_g.p, local ? (uint64_t)g.p : 1ull,
                            local ? (uint64_t)g.shard : 0ull, seg_start.p, inverse.p};
      run_scan(ctx, op, n_cap, d_n(), scan, totals, s);
    }
  }
};

}  // namespace fsx
