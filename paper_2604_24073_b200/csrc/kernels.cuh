// Hot-path kernels of the embedding shard (K1-K11 in SURVEY §2.3).
//
// Layout in HBM: a shard is one row-major [local_rows x dim] array of T
// (float or double), global row g at local row g / p (embedding.hpp:20-21).
// Ids are u64; occurrence indices and positions are u32.
//
// Roofline: every kernel here is HBM/L2-bandwidth or latency bound; none is a
// dense contraction (no tensor cores). Row copies use 16-byte vector loads
// (ld.global.nc.v4) and stores, one warp per row, several rows in flight per
// warp so each lane keeps >= 4 independent 16-B requests outstanding.
#pragma once

#include "radix.cuh"

namespace fsx {

// ---- shard geometry on the device -------------------------------------------
struct ShardGeom {
  uint64_t total_rows;
  uint64_t local_rows;
  uint32_t dim;
  int p;
  int shard;
  __host__ __device__ bool owns(uint64_t g) const {
    return g < total_rows && static_cast<int>(g % static_cast<uint64_t>(p)) == shard;
  }
};

// ---- splitmix64 table init (embedding.cpp:59-64, 108-119) --------------------
__device__ __forceinline__ uint64_t splitmix(uint64_t& s) {
  s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double initial_value_dev(uint64_t seed, uint64_t row, uint32_t d) {
  uint64_t st = seed + row * 0x9e3779b97f4a7c15ULL + (static_cast<uint64_t>(d) + 1) * 0xbf58476d1ce4e5b9ULL;
  splitmix(st);
  const double u = __dmul_rn(static_cast<double>(splitmix(st) >> 11), 0x1.0p-53);
  return __dmul_rn(__dsub_rn(u, 0.5), 0.2);
}

template <class T>
__global__ void k_init_table(T* __restrict__ vals, ShardGeom g, uint64_t seed) { FSX_PDL_ENTER();
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  const uint64_t wid = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t l = wid; l < g.local_rows; l += warps) {
    const uint64_t row = static_cast<uint64_t>(g.shard) + l * static_cast<uint64_t>(g.p);
    T* dst = vals + l * g.dim;
    for (uint32_t d = lane; d < g.dim; d += 32) dst[d] = static_cast<T>(initial_value_dev(seed, row, d));
  }
}

// ---- vectorised row copy ------------------------------------------------------
template <int VB>
struct VecT;
template <>
struct VecT<16> { using type = uint4; };
template <>
struct VecT<8> { using type = uint2; };
template <>
struct VecT<4> { using type = uint32_t; };

__device__ __forceinline__ uint4 ldg_nc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_nc(const uint2* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ldg_nc(const uint32_t* p) { return __ldg(p); }
// plain (coherent) loads for buffers written earlier in the same kernel chain
// by another stream / peer: .nc is only safe for data read-only during the
// kernel, which every caller guarantees.

// Copy `row_bytes` for each item i in [0, n): dst(i) <- src(i). A Map returns
// nullptr from src() to skip an item. Each warp takes 32 items per round: lane
// j resolves item base+j (the Map's index chain, once per item, 32 chains in
// parallel), then the warp copies the live rows kRowsPerWarp at a time with
// every row's loads in flight before the stores.
constexpr int kRowsPerWarp = 8;

template <class Map, int VB>
__global__ void __launch_bounds__(256, 4) k_copy_rows(Map map, uint64_t n_cap, const uint64_t* d_n,
                                                   uint32_t row_bytes) { FSX_PDL_ENTER();
  using V = typename VecT<VB>::type;
  const uint64_t n = scan_n(n_cap, d_n);
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  const uint64_t wid = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t nvec = row_bytes / VB;
  for (uint64_t base = wid * 32; base < n; base += warps * 32) {
    const uint64_t i = base + lane;
    const V* s = nullptr;
    V* d = nullptr;
    if (i < n) {
      s = reinterpret_cast<const V*>(map.src(i));
      if (s) d = reinterpret_cast<V*>(map.dst(i));
    }
    unsigned live = __ballot_sync(0xffffffffu, s != nullptr);
    while (live) {
      const V* src[kRowsPerWarp];
      V* dst[kRowsPerWarp];
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) {
        const int j = live ? __ffs(live) - 1 : 0;
        const bool ok = live != 0;
        live &= live - 1;
        src[r] = reinterpret_cast<const V*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(s), j));
        dst[r] = reinterpret_cast<V*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(d), j));
        if (!ok) src[r] = nullptr;
      }
      for (uint32_t c = lane; c < nvec; c += 32) {
        V v[kRowsPerWarp];
#pragma unroll
        for (int r = 0; r < kRowsPerWarp; ++r)
          if (src[r]) v[r] = ldg_nc(src[r] + c);
#pragma unroll
        for (int r = 0; r < kRowsPerWarp; ++r)
          if (src[r]) dst[r][c] = v[r];
      }
    }
  }
}

inline int vec_bytes_for(uint32_t row_bytes) {
  if (row_bytes % 16 == 0) return 16;
  if (row_bytes % 8 == 0) return 8;
  return 4;
}

template <class Map>
void launch_copy_rows(Ctx* ctx, const Map& map, uint64_t n_cap, const uint64_t* d_n,
                      uint32_t row_bytes, cudaStream_t s) {
  if (n_cap == 0) return;
  const int vb = vec_bytes_for(row_bytes);
  const unsigned grid = grid_for(ctx, n_cap, 8 * 32, ctx->copy_per_sm);
  switch (vb) {
    case 16: FSX_LAUNCH(ctx, (k_copy_rows<Map, 16>), grid, 256, 0, s, map, n_cap, d_n, row_bytes); break;
    case 8: FSX_LAUNCH(ctx, (k_copy_rows<Map, 8>), grid, 256, 0, s, map, n_cap, d_n, row_bytes); break;
    default: FSX_LAUNCH(ctx, (k_copy_rows<Map, 4>), grid, 256, 0, s, map, n_cap, d_n, row_bytes); break;
  }
}

// lookup (embedding.cpp:139-146): out[k] = row(ids[k]); bad ids flagged.
struct GatherByIdMap {
  const char* table;
  const uint64_t* ids;
  char* out;
  uint32_t row_bytes;
  ShardGeom g;
  DevErr* err;
  __device__ const char* src(uint64_t i) const {
    const uint64_t id = ids[i];
    if (!g.owns(id)) {
      report(err, id >= g.total_rows ? kErrRowRange : kErrNotOwned, id,
             id >= g.total_rows ? g.total_rows : static_cast<unsigned long long>(g.shard));
      return nullptr;
    }
    return table + (id / static_cast<uint64_t>(g.p)) * row_bytes;
  }
  __device__ char* dst(uint64_t i) const { return out + i * row_bytes; }
};

// ---- sort + unique -----------------------------------------------------------
// After a stable sort: flag the first occurrence of each key, emit the unique
// keys, segment starts and every item's slot.
template <class K>
struct UniqueOp {
  static constexpr int NC = 1;
  const K* keys;          // sorted
  const uint32_t* perm;   // sorted payload (original index), nullable
  const uint64_t* d_n;    // live item count (device)
  uint64_t* uniq;         // nullable: unique keys (widened)
  uint64_t* uniq_g;       // nullable: unique keys mapped key*mul + add
  uint64_t mul, add;
  uint32_t* seg_start;    // nullable, capacity U+1
  uint32_t* inverse;      // nullable: inverse[perm[k]] = slot
  __device__ void count(uint64_t k, uint32_t (&c)[1]) const {
    c[0] = (k == 0 || keys[k] != keys[k - 1]) ? 1u : 0u;
  }
  __device__ void emit(uint64_t k, const uint32_t (&ex)[1], const uint32_t (&c)[1],
                       const uint32_t (&tot)[1]) const {
    const uint32_t slot = ex[0] + c[0] - 1;
    if (c[0]) {
      const uint64_t key = static_cast<uint64_t>(keys[k]);
      if (uniq) uniq[slot] = key;
      if (uniq_g) uniq_g[slot] = key * mul + add;
      if (seg_start) seg_start[slot] = static_cast<uint32_t>(k);
    }
    if (inverse) inverse[perm ? perm[k] : k] = slot;
    if (seg_start && k + 1 == *d_n) seg_start[slot + 1] = static_cast<uint32_t>(k + 1);
  }
};

// ---- owner partition (route_to_shard_major requester half, :194-204) --------
template <int NC_>
struct OwnerPartitionOp {
  static constexpr int NC = NC_;
  static_assert(NC <= 16, "world too large");
  const uint64_t* ids;
  uint64_t total_rows;
  int p;
  const uint64_t* totals;  // filled by the scan's phase 2 before emit runs
  uint64_t* send_ids;
  uint32_t* send_pos;
  DevErr* err;
  __device__ void count(uint64_t i, uint32_t (&c)[NC]) const {
    const uint64_t id = ids[i];
    const int o = static_cast<int>(id % static_cast<uint64_t>(p));
#pragma unroll
    for (int q = 0; q < NC; ++q) c[q] = (q == o && id < total_rows) ? 1u : 0u;
  }
  __device__ void emit(uint64_t i, const uint32_t (&ex)[NC], const uint32_t (&c)[NC],
                       const uint32_t (&tot)[NC]) const {
    const uint64_t id = ids[i];
    if (id >= total_rows) {
      report(err, kErrRowRange, id, total_rows);
      return;
    }
    const int o = static_cast<int>(id % static_cast<uint64_t>(p));
    uint64_t base = 0;
    for (int q = 0; q < o; ++q) base += tot[q];
    uint32_t r = 0;
#pragma unroll
    for (int q = 0; q < NC; ++q)
      if (q == o) r = ex[q];
    send_ids[base + r] = id;
    send_pos[base + r] = static_cast<uint32_t>(i);
  }
};

// ---- collision (embedding.cpp:82-93) -----------------------------------------
// a, b sorted unique. flag_a[i] = a[i] in b; flag_b[j] = b[j] in a.
__global__ void k_intersect_flags(const uint64_t* __restrict__ a, const uint64_t* d_na,
                                  const uint64_t* __restrict__ b, const uint64_t* d_nb,
                                  uint8_t* __restrict__ flag_a, uint8_t* __restrict__ flag_b,
                                  uint32_t* __restrict__ partner_a = nullptr);

// compaction of a sorted list by a byte flag: out_true / out_false keep order
struct SplitByFlagOp {
  static constexpr int NC = 2;
  const uint64_t* v;
  const uint8_t* flag;
  uint64_t* out_true;   // nullable
  uint64_t* out_false;  // nullable
  __device__ void count(uint64_t i, uint32_t (&c)[2]) const {
    const uint32_t f = flag[i] ? 1u : 0u;
    c[0] = f;
    c[1] = 1u - f;
  }
  __device__ void emit(uint64_t i, const uint32_t (&ex)[2], const uint32_t (&c)[2],
                       const uint32_t (&tot)[2]) const {
    if (c[0]) {
      if (out_true) out_true[ex[0]] = v[i];
    } else if (out_false) {
      out_false[ex[1]] = v[i];
    }
  }
};

// ---- deterministic segmented reduce + SGD (embedding.cpp:148-181) -------------
// Rows are segments of a stable sort of occurrences by id, so within a segment
// occurrences are in (source rank, position) order. Each row's gradient is
// summed in f64 in that order (chunk == 0), or, for rows longer than `chunk`
// occurrences, as ceil(len/chunk) sequential chunk sums added in chunk order
// (fixed association, identical in both engine modes). Then
//   row = row - lr * acc      (f64, no FMA; one rounding to T for f32 tables)
// and a non-finite result is flagged.
// Gradient row of occurrence j: base + src_off(j) + idx(j) * row_bytes. With
// occ_src == nullptr and occ_idx == nullptr this is a plain [M x dim] array.
template <class T>
struct GradRows {
  const char* base;
  uint64_t slot_bytes;      // stride between per-source receive slots
  const uint8_t* occ_src;   // nullable: source slot of occurrence j
  const uint32_t* occ_idx;  // nullable: row of occurrence j inside its slot
  uint32_t row_bytes;
  // nullable: occurrences from source `self_src` read the caller's gradient
  // rows directly (row self_pos[r] of self_base) instead of a staged copy
  const char* self_base = nullptr;
  const uint32_t* self_pos = nullptr;
  int self_src = -1;
  __device__ __forceinline__ const T* row(uint32_t j) const {
    const int s = occ_src ? occ_src[j] : 0;
    const uint64_t r = occ_idx ? occ_idx[j] : j;
    if (self_base && s == self_src)
      return reinterpret_cast<const T*>(self_base + static_cast<uint64_t>(self_pos[r]) * row_bytes);
    return reinterpret_cast<const T*>(base + static_cast<uint64_t>(s) * slot_bytes + r * row_bytes);
  }
};

struct RowSegments {
  const uint64_t* uniq_local;  // sorted local row index per slot
  const uint32_t* seg_start;   // [U+1] into the sorted occurrence order
  const uint32_t* perm;        // sorted position -> occurrence j (nullable: identity)
  const uint64_t* d_u;         // live row count U (device)
  const uint8_t* select;       // nullable: update only rows with select[u] == want
  uint8_t want;
  const uint32_t* inverse = nullptr;  // nullable: occurrence -> row slot (k_stream_entries)
};

// Work lists. A selected row with exactly one occurrence becomes a "single"
// (a pure gather-update: gradient row -> destination row); any other row
// contributes ceil(len / chunk) items (1 when chunk == 0 or len <= chunk),
// and multi-chunk rows are listed for the combine pass. Items are emitted
// fully resolved — occurrence range, first gradient row, destination row —
// so the update kernels' index chains start at the item itself.
struct SgdItem {
  uint32_t u, q, kb, ke;  // row slot, chunk index (bit 31: single-chunk row), occurrence range
  char* dst;              // single-chunk rows: destination row; nullptr: none
  const char* g0;         // gradient row of occurrence kb
};
constexpr uint32_t kSgdSingleChunk = 0x80000000u;

// k_sgd_stream work split: cost = ring entries + kStreamItemCost per item
constexpr uint64_t kStreamItemCost = 2;

#ifndef FSX_PLAN_IPT
#define FSX_PLAN_IPT 2
#endif
struct SgdPlanOp {
  static constexpr int NC = 4;
  static constexpr int kIPT = FSX_PLAN_IPT;  // tens of thousands of rows: spread over every SM
  RowSegments rs;
  uint32_t chunk;
  SgdItem* singles;     // one-occurrence rows
  SgdItem* work;        // every other row / chunk
  uint32_t* multi;      // rows with > 1 chunk
  uint32_t* part_base;  // first partial slot of row u
  char* table;          // table base (row pitch row_bytes)
  uint32_t row_bytes;
  uint64_t local_rows;
  char* const* seg_out; // nullable: reduce-only destinations
  const char* const* gptr;  // nullable: gradient row per sorted occurrence
                            // (nullptr: items carry no gradient pointer; the
                            // update kernels resolve rows from perm)
  // Stream plan (k_sgd_stream, sgd_stream.cuh) when `ent` is set: every row
  // — one-occurrence rows included — becomes work items in row order; c0
  // counts the row's ring entries (its table row when updated in place, then
  // one gradient row per occurrence), each item carries its first entry's
  // offset in `g0`, the table-row entry is written here and the row's first
  // gradient entry goes to row_ent[u] (~0: none) for k_stream_entries.
  uint64_t* ent = nullptr;
  uint32_t* row_ent = nullptr;
  __device__ uint32_t len(uint64_t u) const { return rs.seg_start[u + 1] - rs.seg_start[u]; }
  __device__ bool selected(uint64_t u) const { return !rs.select || rs.select[u] == rs.want; }
  __device__ char* single_dst(uint64_t u) const {
    if (seg_out) return seg_out[u];
    const uint64_t l = rs.uniq_local[u];
    return l < local_rows ? table + l * row_bytes : nullptr;  // never outside the shard
  }
  // c0: singles (stream plan: entries), c1: work items, c2: multi-chunk rows, c3: partial slots
  __device__ void count(uint64_t u, uint32_t (&c)[4]) const {
    c[0] = c[1] = c[2] = c[3] = 0;
    if (!selected(u)) return;
    const uint32_t n = len(u);
    if (ent) {
      const uint32_t k = (chunk == 0 || n <= chunk) ? 1u : (n + chunk - 1) / chunk;
      c[0] = k > 1 ? n : (single_dst(u) ? n + (seg_out ? 0u : 1u) : 0u);
      c[1] = k;
      c[2] = k > 1 ? 1u : 0u;
      c[3] = k > 1 ? k : 0u;
      return;
    }
    if (n == 1) { c[0] = 1; return; }
    const uint32_t k = (chunk == 0 || n <= chunk) ? 1u : (n + chunk - 1) / chunk;
    c[1] = k;
    c[2] = k > 1 ? 1u : 0u;
    c[3] = k > 1 ? k : 0u;
  }
  __device__ void emit(uint64_t u, const uint32_t (&ex)[4], const uint32_t (&c)[4],
                       const uint32_t (&tot)[4]) const {
    if (ent) {
      emit_stream(u, ex, c);
      return;
    }
    if (c[0] == 0 && c[1] == 0) return;
    const uint32_t s = rs.seg_start[u], e = rs.seg_start[u + 1];
    char* dst = nullptr;
    if (c[0] == 1 || c[1] == 1) {
      if (seg_out) {
        dst = seg_out[u];
      } else {
        const uint64_t l = rs.uniq_local[u];
        dst = l < local_rows ? table + l * row_bytes : nullptr;  // never outside the shard
      }
    }
    // first gradient row: a pointer (resolved plans), or, for plans built
    // ahead of the gradients, the occurrence index tagged in bit 0 — the
    // update kernels then skip the perm load
    const char* g0 = gptr ? gptr[s]
                          : reinterpret_cast<const char*>((static_cast<uintptr_t>(rs.perm ? rs.perm[s] : s) << 1) | 1u);
    if (c[0]) {
      singles[ex[0]] = SgdItem{static_cast<uint32_t>(u), kSgdSingleChunk, s, e, dst, g0};
      return;
    }
    if (c[1] == 1) {
      work[ex[1]] = SgdItem{static_cast<uint32_t>(u), kSgdSingleChunk, s, e, dst, g0};
    } else {
      // chunks of a hot row: plain stores (no dependent loads in this loop)
      for (uint32_t q = 0; q < c[1]; ++q) {
        const uint32_t kb = s + q * chunk;
        work[ex[1] + q] = SgdItem{static_cast<uint32_t>(u), q, kb, min(e, kb + chunk), nullptr, nullptr};
      }
    }
    if (c[2]) {
      multi[ex[2]] = static_cast<uint32_t>(u);
      part_base[u] = ex[3];
    }
  }
  __device__ void emit_stream(uint64_t u, const uint32_t (&ex)[4], const uint32_t (&c)[4]) const {
    if (c[1] == 0) {
      row_ent[u] = ~0u;
      return;
    }
    const uint32_t s = rs.seg_start[u], e = rs.seg_start[u + 1];
    if (c[1] == 1) {
      char* dst = single_dst(u);
      const bool old = dst && !seg_out;
      work[ex[1]] = SgdItem{static_cast<uint32_t>(u), kSgdSingleChunk, s, e, dst,
                            reinterpret_cast<const char*>(static_cast<uintptr_t>(ex[0]))};
      if (old) ent[ex[0]] = reinterpret_cast<uintptr_t>(dst);
      row_ent[u] = dst ? ex[0] + (old ? 1u : 0u) : ~0u;
      return;
    }
    for (uint32_t q = 0; q < c[1]; ++q) {
      const uint32_t kb = s + q * chunk;
      work[ex[1] + q] = SgdItem{static_cast<uint32_t>(u), q, kb, min(e, kb + chunk), nullptr,
                                reinterpret_cast<const char*>(static_cast<uintptr_t>(ex[0] + q * chunk))};
    }
    multi[ex[2]] = static_cast<uint32_t>(u);
    part_base[u] = ex[3];
    row_ent[u] = ex[0];
  }
};

// Gradient entries of a stream plan, one thread per sorted occurrence k: the
// row is found by a search of seg_start, the entry holds the gradient row's
// address (resolved plans) or the occurrence index tagged in bit 0 (plans
// built ahead of the gradients: the update adds the base at issue time).
// remap (nullable): the gradient row of occurrence j is row remap[j] of the
// gradient array (pooled backward: every token of a bag takes the bag's row)
static __global__ void k_stream_entries(const uint32_t* __restrict__ seg_start, const uint64_t* d_u,
                                 const uint32_t* __restrict__ perm, const uint32_t* __restrict__ inverse,
                                 const char* const* __restrict__ gptr, const uint32_t* __restrict__ row_ent,
                                 uint64_t* __restrict__ ent, const uint32_t* __restrict__ remap) {
  FSX_PDL_ENTER();
  const uint64_t U = *d_u;
  const uint64_t n = seg_start[U];
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t lo = 0;  // the row u of sorted position k
    const uint32_t j = perm ? perm[k] : static_cast<uint32_t>(k);
    if (inverse) {
      lo = inverse[j];
    } else {  // last row u with seg_start[u] <= k
      uint64_t hi = U;
      while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (seg_start[mid] <= k) lo = mid; else hi = mid;
      }
    }
    const uint32_t r = row_ent[lo];
    if (r == ~0u) continue;
    ent[r + (k - seg_start[lo])] = gptr ? reinterpret_cast<uintptr_t>(gptr[k])
                                        : (static_cast<uint64_t>(remap ? remap[j] : j) << 1) | 1u;
  }
}

// Gradient row of every occurrence in sorted order (perm -> source / rank ->
// row), resolved once by a fully parallel pass
template <class T>
__global__ void k_grad_ptrs(GradRows<T> gr, const uint32_t* __restrict__ perm,
                            const uint32_t* __restrict__ seg_start, const uint64_t* d_u,
                            const T** __restrict__ gptr) { FSX_PDL_ENTER();
  const uint64_t n = seg_start[*d_u];
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    gptr[k] = gr.row(perm ? perm[k] : static_cast<uint32_t>(k));
}

template <class T>
struct SgdArgs {
  T* table;
  ShardGeom g;
  double lr;
  RowSegments rs;
  GradRows<T> gr;
  uint32_t chunk;
  const SgdItem* singles;
  const uint64_t* d_single_n; // device: number of one-occurrence rows (scan total 0)
  const SgdItem* work;
  const uint64_t* d_work_n;   // device: number of work items (scan total 1)
  const uint32_t* multi;
  const uint64_t* d_multi_n;  // device: number of multi-chunk rows (scan total 2)
  const uint32_t* part_base;
  double* partials;           // [work items x dim] f64
  T* rows_out;                // nullable: post-update rows by slot [U x dim]
  DevErr* err;
  char* const* seg_out;       // nullable: reduce-only mode — segment u's sum is
                              // written (as T) to seg_out[u] instead of updating
  const T* const* gptr;       // nullable: gradient row per sorted occurrence
                              // (k_grad_ptrs); nullptr: gr.row(perm[k])
  const uint64_t* ent = nullptr;  // stream plan: ring entries (k_sgd_stream)
  __device__ __forceinline__ const T* grad(uint32_t k) const {
    return gptr ? gptr[k] : gr.row(rs.perm ? rs.perm[k] : k);
  }
  // gradient row of an item's first occurrence (SgdItem::g0: pointer,
  // tagged occurrence index, or nullptr)
  __device__ __forceinline__ const T* first_grad(const SgdItem& it) const {
    const uintptr_t g = reinterpret_cast<uintptr_t>(it.g0);
    if (g & 1u) return gr.row(static_cast<uint32_t>(g >> 1));
    return g ? reinterpret_cast<const T*>(g) : grad(it.kb);
  }
};

// isfinite of a stored value without widening it (an fp32 value is finite
// exactly when its f64 widening is): one integer test for fp32
__device__ __forceinline__ bool finite_val(float x) { return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u; }
__device__ __forceinline__ bool finite_val(double x) { return isfinite(x); }

// vector of VE elements of T moved as one 4/8/16-byte access
template <class T, int VE>
struct alignas(sizeof(T) * VE) VecOf {
  T v[VE];
};

template <class T, int VE>
__device__ __forceinline__ void sgd_apply_vec(const SgdArgs<T>& a, uint32_t u, uint32_t col,
                                              const double (&acc)[VE]) {
  if (a.seg_out) {
    VecOf<T, VE> r;
#pragma unroll
    for (int e = 0; e < VE; ++e) r.v[e] = static_cast<T>(acc[e]);
    *reinterpret_cast<VecOf<T, VE>*>(reinterpret_cast<T*>(a.seg_out[u]) + col) = r;
    return;
  }
  const uint64_t l = a.rs.uniq_local[u];
  if (l >= a.g.local_rows) return;  // never write outside the shard
  VecOf<T, VE>* cell = reinterpret_cast<VecOf<T, VE>*>(a.table + l * a.g.dim + col);
  VecOf<T, VE> r = *cell;
  bool bad = false;
#pragma unroll
  for (int e = 0; e < VE; ++e) {
    const double v = __dsub_rn(static_cast<double>(r.v[e]), __dmul_rn(a.lr, acc[e]));
    r.v[e] = static_cast<T>(v);
    bad |= !finite_val(r.v[e]);
  }
  *cell = r;
  if (a.rows_out)
    *reinterpret_cast<VecOf<T, VE>*>(a.rows_out + static_cast<uint64_t>(u) * a.g.dim + col) = r;
  if (bad) report(a.err, kErrNonFinite, l * static_cast<uint64_t>(a.g.p) + a.g.shard, 0);
}

// Store of one updated vector into a resolved destination row `dst`
// (table row, or seg_out row in reduce-only mode); `old` = the row's current
// value (table mode). Same arithmetic as sgd_apply_vec.
template <class T, int VE>
__device__ __forceinline__ void sgd_store_vec(const SgdArgs<T>& a, uint32_t u, T* dst, uint32_t col,
                                              const double (&acc)[VE], VecOf<T, VE> old) {
  VecOf<T, VE> r;
  if (a.seg_out) {
#pragma unroll
    for (int e = 0; e < VE; ++e) r.v[e] = static_cast<T>(acc[e]);
    *reinterpret_cast<VecOf<T, VE>*>(dst + col) = r;
    return;
  }
  bool bad = false;
#pragma unroll
  for (int e = 0; e < VE; ++e) {
    r.v[e] = static_cast<T>(__dsub_rn(static_cast<double>(old.v[e]), __dmul_rn(a.lr, acc[e])));
    bad |= !finite_val(r.v[e]);
  }
  *reinterpret_cast<VecOf<T, VE>*>(dst + col) = r;
  if (a.rows_out)
    *reinterpret_cast<VecOf<T, VE>*>(a.rows_out + static_cast<uint64_t>(u) * a.g.dim + col) = r;
  if (bad) report(a.err, kErrNonFinite, a.rs.uniq_local[u] * static_cast<uint64_t>(a.g.p) + a.g.shard, 0);
}

// Thread per (item, VE-column vector): every thread runs its own short index
// chain (item -> gradient rows) and moves one 16-byte vector per occurrence,
// so the grid's loads are independent — the memory-level parallelism a
// gather/scatter over Zipf rows needs. The 64 threads of one 1 KB row share
// the item load through L1.
//
// k_sgd_single: one-occurrence rows, two items per thread in flight.
template <class T, int VE>
__global__ void __launch_bounds__(256) k_sgd_single(SgdArgs<T> a, uint32_t vpr_shift) { FSX_PDL_ENTER();
  using V = VecOf<T, VE>;
  const uint64_t n = *a.d_single_n;
  const uint32_t dim = a.g.dim;
  const uint32_t vpr = dim / VE;
  const uint64_t total = n * vpr;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i0 < total; i0 += 2 * stride) {
    uint64_t ix[2] = {i0, i0 + stride};
    SgdItem it[2];
    uint32_t col[2];
    bool ok[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ok[h] = ix[h] < total;
      const uint64_t w = vpr_shift != 0xffffffffu ? ix[h] >> vpr_shift : ix[h] / vpr;
      col[h] = static_cast<uint32_t>(ix[h] - w * vpr) * VE;
      if (ok[h]) it[h] = a.singles[w];
    }
    V g[2], old[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ok[h] = ok[h] && it[h].dst != nullptr;
      if (ok[h]) {
        const T* g0 = a.first_grad(it[h]);
        g[h] = *reinterpret_cast<const V*>(g0 + col[h]);
        if (!a.seg_out) old[h] = *reinterpret_cast<const V*>(reinterpret_cast<const T*>(it[h].dst) + col[h]);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (ok[h]) {
        double acc[VE];
#pragma unroll
        for (int x = 0; x < VE; ++x) acc[x] = __dadd_rn(0.0, static_cast<double>(g[h].v[x]));
        sgd_store_vec<T, VE>(a, it[h].u, reinterpret_cast<T*>(it[h].dst), col[h], acc, old[h]);
      }
  }
}

// k_sgd_flat: rows of 2+ occurrences (or one chunk of a hot row), summed in
// order in f64 with kFlatBatch loads in flight; multi-chunk rows leave
// partials for k_sgd_combine.
constexpr int kFlatBatch = 8;
template <class T, int VE>
__global__ void __launch_bounds__(256, 3) k_sgd_flat(SgdArgs<T> a, uint32_t vpr_shift) { FSX_PDL_ENTER();
  using V = VecOf<T, VE>;
  const uint64_t nwork = *a.d_work_n;
  const uint32_t dim = a.g.dim;
  const uint32_t vpr = dim / VE;  // vectors per row
  const uint64_t total = nwork * vpr;
  for (uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t w = vpr_shift != 0xffffffffu ? idx >> vpr_shift : idx / vpr;
    const uint32_t col = static_cast<uint32_t>(idx - w * vpr) * VE;
    const SgdItem item = a.work[w];
    T* dst = reinterpret_cast<T*>(item.dst);
    const bool single = (item.q & kSgdSingleChunk) != 0;
    V old{};
    if (single && dst && !a.seg_out) old = *reinterpret_cast<const V*>(dst + col);  // in flight with the gradients
    double acc[VE];
#pragma unroll
    for (int x = 0; x < VE; ++x) acc[x] = 0.0;
    // software pipeline: the next batch's gradient-row pointers load while
    // this batch's gradient vectors are in flight
    const T* gp[kFlatBatch];
#pragma unroll
    for (int t = 0; t < kFlatBatch; ++t)
      gp[t] = item.kb + t < item.ke ? (t == 0 ? a.first_grad(item) : a.grad(item.kb + t)) : nullptr;
    for (uint32_t k0 = item.kb; k0 < item.ke; k0 += kFlatBatch) {
      V g[kFlatBatch];
#pragma unroll
      for (int t = 0; t < kFlatBatch; ++t)
        if (k0 + t < item.ke) g[t] = *reinterpret_cast<const V*>(gp[t] + col);
      const uint32_t k1 = k0 + kFlatBatch;
#pragma unroll
      for (int t = 0; t < kFlatBatch; ++t) gp[t] = k1 + t < item.ke ? a.grad(k1 + t) : nullptr;
#pragma unroll
      for (int t = 0; t < kFlatBatch; ++t)
        if (k0 + t < item.ke) {
#pragma unroll
          for (int x = 0; x < VE; ++x) acc[x] = __dadd_rn(acc[x], static_cast<double>(g[t].v[x]));
        }
    }
    if (single) {
      if (dst) sgd_store_vec<T, VE>(a, item.u, dst, col, acc, old);
    } else {
      double* p = a.partials + (static_cast<uint64_t>(a.part_base[item.u]) + item.q) * dim + col;
#pragma unroll
      for (int x = 0; x < VE; ++x) p[x] = acc[x];
    }
  }
}

// k_sgd_warp: the work items of k_sgd_flat (rows of 2+ occurrences, chunks of
// hot rows), one warp per item. Lane l resolves the gradient row of occurrence
// kb + l (32 index chains in parallel instead of one per 16-byte vector), the
// warp then streams the rows U at a time — lane l moves vectors l, l + 32, …
// (VPL per lane) — so per gradient vector a lane issues one load, VE
// conversions and VE adds. The next item and its row pointers load while the
// current item's rows are in flight. A multi-chunk row's chunks leave f64
// partials; the warp that completes the row's last chunk (arrival counter
// `done[u]`, reset by that warp) adds them in chunk order — the association
// k_sgd_combine uses — and applies the row: no separate combine pass.
template <class T, int VE, int VPL, int U, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_sgd_warp(SgdArgs<T> a, uint32_t* __restrict__ done) { FSX_PDL_ENTER();
  using V = VecOf<T, VE>;
  constexpr unsigned kFull = 0xffffffffu;
  const uint64_t nwork = *a.d_work_n;
  const uint32_t dim = a.g.dim;
  const uint32_t vpr = dim / VE;
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  if (w >= nwork) return;
  SgdItem it = a.work[w];
  const T* myp = it.kb + lane < it.ke ? a.grad(it.kb + lane) : nullptr;
  while (true) {
    const uint64_t wn = w + nw;
    SgdItem nx{};
    if (wn < nwork) nx = a.work[wn];
    const bool single = (it.q & kSgdSingleChunk) != 0;
    T* dst = reinterpret_cast<T*>(it.dst);
    V old[VPL];
    if (single && dst && !a.seg_out) {
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        if (lane + 32u * v < vpr) old[v] = *reinterpret_cast<const V*>(dst + (lane + 32u * v) * VE);
    }
    double acc[VPL][VE];
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int x = 0; x < VE; ++x) acc[v][x] = 0.0;
    const T* myp_nx = nullptr;
    bool nx_resolved = false;
    for (uint32_t k0 = it.kb; k0 < it.ke; k0 += 32) {
      const uint32_t nk = min(32u, it.ke - k0);
      if (k0 != it.kb) myp = k0 + lane < it.ke ? a.grad(k0 + lane) : nullptr;
      for (uint32_t t0 = 0; t0 < nk; t0 += U) {
        V g[U][VPL];
#pragma unroll
        for (int t = 0; t < U; ++t) {
          const T* p = reinterpret_cast<const T*>(
              __shfl_sync(kFull, reinterpret_cast<unsigned long long>(myp), t0 + t));
          if (t0 + t < nk) {
#pragma unroll
            for (int v = 0; v < VPL; ++v)
              if (lane + 32u * v < vpr) g[t][v] = *reinterpret_cast<const V*>(p + (lane + 32u * v) * VE);
          }
        }
        if (!nx_resolved) {  // next item's pointers load behind this batch
          nx_resolved = true;
          if (wn < nwork && nx.kb + lane < nx.ke) myp_nx = a.grad(nx.kb + lane);
        }
#pragma unroll
        for (int t = 0; t < U; ++t)
          if (t0 + t < nk) {
#pragma unroll
            for (int v = 0; v < VPL; ++v)
#pragma unroll
              for (int x = 0; x < VE; ++x) acc[v][x] = __dadd_rn(acc[v][x], static_cast<double>(g[t][v].v[x]));
          }
      }
    }
    if (!nx_resolved && wn < nwork && nx.kb + lane < nx.ke) myp_nx = a.grad(nx.kb + lane);
    if (single) {
      if (dst) {
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (lane + 32u * v < vpr) sgd_store_vec<T, VE>(a, it.u, dst, (lane + 32u * v) * VE, acc[v], old[v]);
      }
    } else {
      const uint64_t base = a.part_base[it.u];
      double* pp = a.partials + (base + it.q) * dim;
#pragma unroll
      for (int v = 0; v < VPL; ++v)
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
        for (int v = 0; v < VPL; ++v)
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
    if (wn >= nwork) break;
    w = wn;
    it = nx;
    myp = myp_nx;
  }
}

// one CTA per multi-chunk row, each thread owning VE columns: the row's chunk
// partials are summed in chunk order (8 loads in flight per thread)
template <class T, int VE>
__global__ void __launch_bounds__(128) k_sgd_combine(SgdArgs<T> a) { FSX_PDL_ENTER();
  const uint64_t nm = *a.d_multi_n;
  const uint32_t dim = a.g.dim;
  for (uint64_t m = blockIdx.x; m < nm; m += gridDim.x) {
    const uint32_t u = a.multi[m];
    const uint32_t len = a.rs.seg_start[u + 1] - a.rs.seg_start[u];
    const uint32_t nch = (len + a.chunk - 1) / a.chunk;
    const double* base = a.partials + static_cast<uint64_t>(a.part_base[u]) * dim;
    for (uint32_t col = threadIdx.x * VE; col < dim; col += blockDim.x * VE) {
      double acc[VE];
#pragma unroll
      for (int x = 0; x < VE; ++x) acc[x] = 0.0;
      uint32_t q = 0;
      for (; q + 8 <= nch; q += 8) {
        double t[8][VE];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int x = 0; x < VE; ++x) t[j][x] = base[static_cast<uint64_t>(q + j) * dim + col + x];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int x = 0; x < VE; ++x) acc[x] = __dadd_rn(acc[x], t[j][x]);
      }
      for (; q < nch; ++q)
#pragma unroll
        for (int x = 0; x < VE; ++x) acc[x] = __dadd_rn(acc[x], base[static_cast<uint64_t>(q) * dim + col + x]);
      sgd_apply_vec<T, VE>(a, u, col, acc);
    }
  }
}

}  // namespace fsx
