// Device side of the embedding engines (SynchronizedEmbedding /
// PrioritizedEmbedding, embedding.cpp:235-607).
//
// Wire format of every message slot (one per (channel, peer)):
//   [u64 n][u64 reserved][payload]
// payload = n u64 ids                       (IDS)
//         | n rows                          (ROWS, GRADS, CO_G, EX_G)
//         | n u64 ids, pad16, n rows        (EX, CO_R; rows at 16+align16(8n))
//         | n u8 flags                      (MASK)
// The reference's [u64 count][ids][rows] (embedding.cpp:29-55) with the ids
// 16-byte aligned so rows move as 128-bit vectors.
#pragma once

#include "table.cuh"

namespace fsx {

constexpr int kMaxRanks = 16;
constexpr uint64_t kHdr = 16;

__host__ __device__ __forceinline__ uint64_t align16(uint64_t x) { return (x + 15) & ~uint64_t(15); }
__host__ __device__ __forceinline__ uint64_t idrows_rows_off(uint64_t n) { return kHdr + align16(8 * n); }

// per-peer slot base addresses of one channel as seen by this rank
struct Slots {
  char* p[kMaxRanks];
};
struct CSlots {
  const char* p[kMaxRanks];
};

__device__ __forceinline__ uint64_t slot_n(const char* s) { return *reinterpret_cast<const uint64_t*>(s); }

// ---- headers ---------------------------------------------------------------
// n of destination d = counts[d * stride] (device); one thread per slot.
static __global__ void k_write_headers(Slots dst, int p, const uint64_t* counts, int stride,
                                uint64_t cap, DevErr* err) { FSX_PDL_ENTER();
  const int d = threadIdx.x;
  if (d < p) {
    const uint64_t n = counts[d * stride];
    if (n > cap) report(err, kErrCapacity, n, cap);
    reinterpret_cast<uint64_t*>(dst.p[d])[0] = n;
    reinterpret_cast<uint64_t*>(dst.p[d])[1] = 0;
  }
}

// ---- requester: route (embedding.cpp:194-212) -------------------------------
// stable partition by owner straight into the IDS send slots
template <int NC_>
struct RouteOp {
  static constexpr int NC = NC_;
  const uint64_t* ids;
  uint64_t total_rows;
  int p;
  const uint64_t* totals;   // per-owner counts (scan phase 2)
  Slots send;               // IDS send slots
  uint32_t* send_pos;       // grouped k -> position j
  uint8_t* send_dst;        // grouped k -> owner
  uint64_t cap;
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
    if (r >= cap) {
      report(err, kErrCapacity, static_cast<unsigned long long>(r) + 1, cap);
      return;
    }
    reinterpret_cast<uint64_t*>(send.p[o] + kHdr)[r] = id;
    send_pos[base + r] = static_cast<uint32_t>(i);
    send_dst[base + r] = static_cast<uint8_t>(o);
  }
};

// ---- owner: flatten received ids (embedding.cpp:214-229) ----------------------
// cnt[0] = M, cnt[2+s] = n_s, off[s] prefix (cnt[2+p+s])
static __global__ void k_recv_prefix(CSlots slots, int p, uint64_t cap, uint64_t* cnt, DevErr* err) { FSX_PDL_ENTER();
  if (threadIdx.x == 0) {
    uint64_t off = 0;
    for (int s = 0; s < p; ++s) {
      const uint64_t n = slot_n(slots.p[s]);
      if (n > cap) report(err, kErrCapacity, n, cap);
      cnt[2 + s] = n;
      cnt[2 + kMaxRanks + s] = off;
      off += n <= cap ? n : cap;
    }
    cnt[0] = off;
  }
}

static __global__ void k_flatten_recv(CSlots slots, int p, uint64_t cap, const uint64_t* cnt, ShardGeom g,
                               uint64_t* __restrict__ ids, uint8_t* __restrict__ occ_src,
                               uint32_t* __restrict__ occ_idx, DevErr* err) { FSX_PDL_ENTER();
  const uint64_t total = static_cast<uint64_t>(p) * cap;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(i / cap);
    const uint64_t idx = i - static_cast<uint64_t>(s) * cap;
    if (idx >= cnt[2 + s]) continue;
    const uint64_t id = reinterpret_cast<const uint64_t*>(slots.p[s] + kHdr)[idx];
    if (!g.owns(id)) report(err, kErrRecvNotOwned, id, g.shard);
    const uint64_t j = cnt[2 + kMaxRanks + s] + idx;
    ids[j] = id;
    occ_src[j] = static_cast<uint8_t>(s);
    occ_idx[j] = static_cast<uint32_t>(idx);
  }
}

// src bitmask per unique row: bit s set iff source s requested it
static __global__ void k_src_bits(const uint32_t* __restrict__ inverse, const uint8_t* __restrict__ occ_src,
                           const uint64_t* d_m, uint32_t* __restrict__ bits) { FSX_PDL_ENTER();
  const uint64_t m = *d_m;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < m;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    atomicOr(&bits[inverse[j]], 1u << occ_src[j]);
}

// ---- owner: per-source pack lists -------------------------------------------
// Over the unique rows of the NEXT batch: counters 2s (bit s, exclusive) and
// 2s+1 (bit s, collision). Emits entry lists: ex_list / co_list, ordered by
// source then rank (rank = position inside that source's message).
struct PackEntry {
  uint32_t u;
  uint32_t rank;
  uint32_t src;
  uint32_t pad;
};

template <int NC_>
struct OwnerPackOp {
  static constexpr int NC = NC_;  // 2 * kMax(p)
  const uint32_t* bits;
  const uint8_t* co;          // co flag per unique row of the batch
  int p;
  const uint64_t* totals;     // [NC] from phase 2
  PackEntry* ex_list;
  PackEntry* co_list;
  uint32_t* rank_us;          // [u][kMaxRanks]: position of row u in source s's message
  __device__ void count(uint64_t u, uint32_t (&c)[NC]) const {
    const uint32_t b = bits[u];
    const uint32_t f = co[u] ? 1u : 0u;
#pragma unroll
    for (int q = 0; q < NC / 2; ++q) {
      const uint32_t has = (b >> q) & 1u;
      c[2 * q] = has & (1u - f);
      c[2 * q + 1] = has & f;
    }
  }
  __device__ void emit(uint64_t u, const uint32_t (&ex)[NC], const uint32_t (&c)[NC],
                       const uint32_t (&tot)[NC]) const {
    const uint32_t b = bits[u];
    const uint32_t f = co[u] ? 1u : 0u;
    uint64_t base_ex = 0, base_co = 0;
#pragma unroll
    for (int q = 0; q < NC / 2; ++q) {
      if ((b >> q) & 1u) {
        PackEntry e{static_cast<uint32_t>(u), ex[2 * q + f], static_cast<uint32_t>(q), 0};
        if (f) co_list[base_co + e.rank] = e;
        else ex_list[base_ex + e.rank] = e;
        rank_us[u * kMaxRanks + q] = e.rank;
      }
      base_ex += tot[2 * q];
      base_co += tot[2 * q + 1];
    }
  }
};

// Per-occurrence messages back to the requesters, in each source's own send
// order (occurrence j of the owner batch = element occ_idx[j] of source
// occ_src[j]'s id message):
//  IDX  (next batch): where the occurrence's row sits in this owner's E_ex /
//       E_co message to that source: rank | collision << 31. Replaces the
//       reference's merge-time lower_bound by id (embedding.cpp:465-482).
//  MASK (current batch): the occurrence's collision flag, i.e. mask_co_
//       membership (embedding.cpp:392-401, 530) as one byte per occurrence.
static __global__ void k_idx_pack(const uint32_t* __restrict__ inverse,
                                  const uint8_t* __restrict__ occ_src,
                                  const uint32_t* __restrict__ occ_idx, const uint64_t* d_m,
                                  const uint32_t* __restrict__ rank_us,
                                  const uint8_t* __restrict__ co, Slots send, int self) { FSX_PDL_ENTER();
  const uint64_t m = *d_m;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < m;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t u = inverse[j];
    const int s = occ_src[j];
    // self rows are merged straight from the table: only their collision bit
    const uint32_t v = (s == self ? 0u : rank_us[static_cast<uint64_t>(u) * kMaxRanks + s]) |
                       (co[u] ? 0x80000000u : 0u);
    reinterpret_cast<uint32_t*>(send.p[s] + kHdr)[occ_idx[j]] = v;
  }
}

static __global__ void k_mask_pack(const uint32_t* __restrict__ inverse,
                                   const uint8_t* __restrict__ occ_src,
                                   const uint32_t* __restrict__ occ_idx, const uint64_t* d_m,
                                   const uint8_t* __restrict__ co, Slots send) { FSX_PDL_ENTER();
  const uint64_t m = *d_m;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < m;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    reinterpret_cast<uint8_t*>(send.p[occ_src[j]] + kHdr)[occ_idx[j]] = co && co[inverse[j]] ? 1 : 0;
}

// per-occurrence rank inside its (source, flag) class, flat recv order:
// counters 2s (exclusive) / 2s+1 (collision)
template <int NC_>
struct OccRankOp {
  static constexpr int NC = NC_;
  const uint8_t* occ_src;
  const uint32_t* inverse;
  const uint8_t* co;          // nullable -> all exclusive
  uint32_t* occ_rank;
  __device__ void count(uint64_t j, uint32_t (&c)[NC]) const {
    const int s = occ_src[j];
    const uint32_t f = co ? (co[inverse[j]] ? 1u : 0u) : 0u;
#pragma unroll
    for (int q = 0; q < NC; ++q) c[q] = (q == 2 * s + static_cast<int>(f)) ? 1u : 0u;
  }
  __device__ void emit(uint64_t j, const uint32_t (&ex)[NC], const uint32_t (&c)[NC],
                       const uint32_t (&tot)[NC]) const {
    const int s = occ_src[j];
    const uint32_t f = co ? (co[inverse[j]] ? 1u : 0u) : 0u;
    uint32_t r = 0;
#pragma unroll
    for (int q = 0; q < NC; ++q)
      if (q == 2 * s + static_cast<int>(f)) r = ex[q];
    occ_rank[j] = r;
  }
};

// ---- requester: collision flag of every sent occurrence (MASK messages) ----
static __global__ void k_req_flags(CSlots mask, const uint8_t* __restrict__ send_dst,
                                   const uint64_t* __restrict__ send_off, uint64_t n,
                                   uint8_t* __restrict__ flag, DevErr* err) { FSX_PDL_ENTER();
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int d = send_dst[k];
    const uint64_t q = k - send_off[d];
    if (q == 0 && slot_n(mask.p[d]) != send_off[d + 1] - send_off[d])
      report(err, kErrMaskOverlap, slot_n(mask.p[d]), send_off[d + 1] - send_off[d]);
    flag[k] = reinterpret_cast<const uint8_t*>(mask.p[d] + kHdr)[q];
  }
}

// split counters over the grouped send order: 2d + flag
template <int NC_>
struct SplitOp {
  static constexpr int NC = NC_;
  const uint8_t* send_dst;
  const uint8_t* flag;       // per grouped k (nullable -> all exclusive)
  uint32_t* split_rank;      // grouped k -> rank in its (dst, flag) message
  __device__ uint32_t f(uint64_t k) const { return flag ? (flag[k] ? 1u : 0u) : 0u; }
  __device__ void count(uint64_t k, uint32_t (&c)[NC]) const {
    const int d = send_dst[k];
    const uint32_t fl = f(k);
#pragma unroll
    for (int q = 0; q < NC; ++q) c[q] = (q == 2 * d + static_cast<int>(fl)) ? 1u : 0u;
  }
  __device__ void emit(uint64_t k, const uint32_t (&ex)[NC], const uint32_t (&c)[NC],
                       const uint32_t (&tot)[NC]) const {
    const int d = send_dst[k];
    const uint32_t fl = f(k);
    uint32_t r = 0;
#pragma unroll
    for (int q = 0; q < NC; ++q)
      if (q == 2 * d + static_cast<int>(fl)) r = ex[q];
    split_rank[k] = r;
  }
};

// ---- row movers (all go through k_copy_rows) ----------------------------------
// sync forward, owner side: per received occurrence, its row into the ROWS
// send slot of its source at its index (embedding.cpp:245-248)
struct OwnerLookupMap {
  const char* table;
  const uint64_t* ids;
  const uint8_t* occ_src;
  const uint32_t* occ_idx;
  Slots send;
  uint32_t row_bytes;
  int p;
  __device__ const char* src(uint64_t j) const {
    return table + (ids[j] / static_cast<uint64_t>(p)) * row_bytes;
  }
  __device__ char* dst(uint64_t j) const {
    return send.p[occ_src[j]] + kHdr + static_cast<uint64_t>(occ_idx[j]) * row_bytes;
  }
};

// sync forward, requester side: reply row k of owner d -> out[send_pos[k]]
// (embedding.cpp:252-264)
struct RequesterScatterMap {
  CSlots recv;
  const uint32_t* send_pos;
  const uint8_t* send_dst;
  const uint64_t* send_off;  // per owner start in the grouped order (device)
  char* out;
  uint32_t row_bytes;
  __device__ const char* src(uint64_t k) const {
    const int d = send_dst[k];
    return recv.p[d] + kHdr + (k - send_off[d]) * row_bytes;
  }
  __device__ char* dst(uint64_t k) const { return out + static_cast<uint64_t>(send_pos[k]) * row_bytes; }
};

// backward, requester side: grads of grouped k into GRADS / CO_G / EX_G send
// slots (embedding.cpp:276-286, 526-536). split_rank == nullptr: sync pack.
struct GradPackMap {
  const char* grads;
  const uint32_t* send_pos;
  const uint8_t* send_dst;
  const uint64_t* send_off;
  const uint8_t* flag;        // per grouped k; nullable: everything to `ex`
  const uint32_t* split_rank; // nullable: rank = k - send_off[d]
  Slots co, ex;
  uint32_t row_bytes;
  int part;                   // 0: every row; 1: exclusive only; 2: collision only
  int skip_dst = -1;          // rows for this owner are not staged (read in place)
  __device__ const char* src(uint64_t k) const {
    const bool f = flag && flag[k];
    if ((part == 1 && f) || (part == 2 && !f)) return nullptr;
    if (send_dst[k] == skip_dst) return nullptr;
    return grads + static_cast<uint64_t>(send_pos[k]) * row_bytes;
  }
  __device__ char* dst(uint64_t k) const {
    const int d = send_dst[k];
    const bool f = flag && flag[k];
    const uint64_t r = split_rank ? split_rank[k] : k - send_off[d];
    return (f ? co.p[d] : ex.p[d]) + kHdr + r * row_bytes;
  }
};

// owner pack of [ids][rows] messages (EX prefetch, E_co) from the entry lists
struct IdRowPackMap {
  const char* table;
  const uint64_t* uniq_local;
  const uint64_t* uniq_g;
  const PackEntry* list;
  Slots send;
  const uint64_t* totals;  // per-source counts: totals[2*s + which]
  int which;
  uint32_t row_bytes;
  int self;                // rows for this rank itself are never copied: its
                           // merge reads them from the table (MergeMap)
  __device__ const char* src(uint64_t i) const {
    const PackEntry e = list[i];
    if (static_cast<int>(e.src) == self) return nullptr;
    // the id rides in the same pass
    reinterpret_cast<uint64_t*>(send.p[e.src] + kHdr)[e.rank] = uniq_g[e.u];
    return table + uniq_local[e.u] * row_bytes;
  }
  __device__ char* dst(uint64_t i) const {
    const PackEntry e = list[i];
    const uint64_t n = totals[2 * e.src + which];
    return send.p[e.src] + idrows_rows_off(n) + static_cast<uint64_t>(e.rank) * row_bytes;
  }
};

// requester merge (embedding.cpp:453-484): occurrence k of owner d takes row
// IDX[d][q] of that owner's E_ex or E_co message; the id stored next to the
// row must be the id asked for ("missing from both prefetched buffers").
// Rows this rank owns itself are read straight from the table: at merge time
// the table holds exactly what E_ex / E_co would carry (exclusive rows of i
// are not updated between their prefetch and this merge; collision rows were
// updated before E_co was released), so self traffic moves no rows at all.
struct MergeMap {
  CSlots idx, ex, co;
  const char* table;
  const uint32_t* send_pos;
  const uint8_t* send_dst;
  const uint64_t* send_off;
  const uint64_t* ids;  // batch ids (position order)
  char* out;
  uint32_t row_bytes;
  int self, p;
  DevErr* err;
  int part;  // 0: every row; 1: exclusive rows only; 2: collision rows only
  __device__ const char* src(uint64_t k) const {
    const int d = send_dst[k];
    const uint64_t q = k - send_off[d];
    const uint32_t v = reinterpret_cast<const uint32_t*>(idx.p[d] + kHdr)[q];
    const bool is_co = (v & 0x80000000u) != 0;
    if ((part == 1 && is_co) || (part == 2 && !is_co)) return nullptr;
    if (d == self) return table + (ids[send_pos[k]] / static_cast<uint64_t>(p)) * row_bytes;
    const char* s = is_co ? co.p[d] : ex.p[d];
    const uint64_t r = v & 0x7fffffffu;
    const uint64_t n = slot_n(s);
    const uint64_t want = ids[send_pos[k]];
    if (r >= n || reinterpret_cast<const uint64_t*>(s + kHdr)[r] != want) {
      report(err, kErrMissingRow, want, 0);
      return nullptr;
    }
    return s + idrows_rows_off(n) + r * row_bytes;
  }
  __device__ char* dst(uint64_t k) const { return out + static_cast<uint64_t>(send_pos[k]) * row_bytes; }
};

// ---- pre-summed collision gradients (FSX_ENGINE_PRESUM) ----------------------
// The collision chain is the exposed part of the protocol: its bytes are one
// gradient row per collision OCCURRENCE (embedding.cpp:526-546). With PRESUM
// each requester first sums its own occurrences of each collision row, so the
// chain carries one row per (source, collision row) and the owner adds at
// most p rows per collision row. Association: per (row, source) the
// source's occurrences in position order (chunked like the owner reduce),
// then the sources in rank order — fixed, hence deterministic, but different
// from the reference's single left fold, so this mode is held to the fp32
// tolerance, not bitwise.
//
// GRP message (owner -> requester s), built from the owner's sorted order:
//   [u64 n_slots][u64 n_occ][u32 seg[n_slots + 1]][pad16][u32 list[n_occ]]
// list = s's collision occurrences (its own send-order indices) grouped by
// row, rows ascending, positions ascending within a row; seg = slot starts.
__host__ __device__ __forceinline__ uint64_t grp_list_off(uint64_t n_slots) {
  return kHdr + align16(4 * (n_slots + 1));
}

template <int NC_>
struct GroupOp {
  static constexpr int NC = NC_;  // 2 counters per source
  const uint32_t* perm;           // sorted position -> occurrence j
  const uint32_t* inverse;        // occurrence -> row slot u
  const uint32_t* seg_start;      // row segments in sorted order
  const uint8_t* occ_src;
  const uint32_t* occ_idx;
  const uint8_t* co;              // collision flag per row
  Slots send;                     // GRP send slots
  uint32_t* slot_us;              // [u][kMaxRanks] -> slot of (row, source)
  __device__ void classify(uint64_t k, int& s, bool& is_co, bool& first) const {
    const uint32_t j = perm[k];
    const uint32_t u = inverse[j];
    s = occ_src[j];
    is_co = co[u] != 0;
    first = is_co && (k == seg_start[u] || occ_src[perm[k - 1]] != s);
  }
  __device__ void count(uint64_t k, uint32_t (&c)[NC]) const {
    int s;
    bool is_co, first;
    classify(k, s, is_co, first);
#pragma unroll
    for (int q = 0; q < NC / 2; ++q) {
      c[2 * q] = (q == s && is_co) ? 1u : 0u;
      c[2 * q + 1] = (q == s && first) ? 1u : 0u;
    }
  }
  __device__ void emit(uint64_t k, const uint32_t (&ex)[NC], const uint32_t (&c)[NC],
                       const uint32_t (&tot)[NC]) const {
    int s;
    bool is_co, first;
    classify(k, s, is_co, first);
    if (!is_co) return;
    uint32_t r_occ = 0, r_slot = 0, n_slots = 0;
#pragma unroll
    for (int q = 0; q < NC / 2; ++q)
      if (q == s) { r_occ = ex[2 * q]; r_slot = ex[2 * q + 1]; n_slots = tot[2 * q + 1]; }
    char* msg = send.p[s];
    reinterpret_cast<uint32_t*>(msg + grp_list_off(n_slots))[r_occ] = occ_idx[perm[k]];
    if (first) {
      reinterpret_cast<uint32_t*>(msg + kHdr)[r_slot] = r_occ;
      slot_us[static_cast<uint64_t>(inverse[perm[k]]) * kMaxRanks + s] = r_slot;
    }
  }
};

// headers + closing seg entry: tot[2s] = n_occ, tot[2s+1] = n_slots
static __global__ void k_grp_headers(Slots send, int p, const uint64_t* tot) { FSX_PDL_ENTER();
  const int s = threadIdx.x;
  if (s < p) {
    const uint64_t n_occ = tot[2 * s], n_slots = tot[2 * s + 1];
    reinterpret_cast<uint64_t*>(send.p[s])[0] = n_slots;
    reinterpret_cast<uint64_t*>(send.p[s])[1] = n_occ;
    reinterpret_cast<uint32_t*>(send.p[s] + kHdr)[n_slots] = static_cast<uint32_t>(n_occ);
  }
}

// requester: per-owner bases of the received GRP messages.
// bases[0..p] slot prefix, bases[17..17+p] occurrence prefix, bases[34+d] = n_slots_d
static __global__ void k_grp_bases(CSlots grp, int p, uint64_t* bases) { FSX_PDL_ENTER();
  if (threadIdx.x == 0) {
    uint64_t s = 0, o = 0;
    for (int d = 0; d < p; ++d) {
      bases[d] = s;
      bases[17 + d] = o;
      const uint64_t ns = reinterpret_cast<const uint64_t*>(grp.p[d])[0];
      bases[34 + d] = ns;
      s += ns;
      o += reinterpret_cast<const uint64_t*>(grp.p[d])[1];
    }
    bases[p] = s;
    bases[17 + p] = o;
    bases[16] = s;  // live segment count for the reduce
  }
}

// requester: collision flag of every sent occurrence + the flattened segment
// view (one segment per (owner, slot)) the chunked reduce consumes:
// seg_flat[] (starts into perm_flat), perm_flat[] (batch positions),
// out_ptr[] (the CO_G staging row each segment sum is written to)
static __global__ void k_grp_flatten(CSlots grp, int p, uint64_t cap, const uint64_t* bases,
                                     const uint64_t* send_off, const uint32_t* send_pos, Slots cog,
                                     uint32_t row_bytes, uint8_t* flag, uint32_t* seg_flat,
                                     uint32_t* perm_flat, char** out_ptr) { FSX_PDL_ENTER();
  const uint64_t total = static_cast<uint64_t>(p) * (cap + 1);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int d = static_cast<int>(i / (cap + 1));
    const uint64_t q = i - static_cast<uint64_t>(d) * (cap + 1);
    const char* m = grp.p[d];
    const uint64_t n_slots = reinterpret_cast<const uint64_t*>(m)[0];
    const uint64_t n_occ = reinterpret_cast<const uint64_t*>(m)[1];
    const uint32_t* seg = reinterpret_cast<const uint32_t*>(m + kHdr);
    const uint32_t* list = reinterpret_cast<const uint32_t*>(m + grp_list_off(n_slots));
    if (q < n_slots) {
      seg_flat[bases[d] + q] = static_cast<uint32_t>(bases[17 + d] + seg[q]);
      out_ptr[bases[d] + q] = cog.p[d] + kHdr + q * row_bytes;
    }
    if (q < n_occ) {
      const uint64_t k = send_off[d] + list[q];
      flag[k] = 1;
      perm_flat[bases[17 + d] + q] = send_pos[k];
    }
    if (d == p - 1 && q == 0) seg_flat[bases[p]] = static_cast<uint32_t>(bases[17 + p]);
  }
}

// owner: collision rows get the sum of the sources' pre-summed rows, sources
// in rank order, then row -= lr * acc (f64, one rounding). Fused E_co pack
// (eco.partner != nullptr): the updated row is also written straight into the
// E_co message of every next-iteration requester of that row (the same bytes
// IdRowPackMap would copy out of the table afterwards).
struct EcoOut {
  const uint32_t* partner;   // oc row -> row of the next owner batch; nullable: no E_co
  const uint32_t* bits;      // next batch: requester bits per row
  const uint32_t* rank_us;   // next batch: position of the row in each requester's E_co
  const uint64_t* totals;    // next batch pack totals: [2s+1] = E_co rows for s
  const uint64_t* uniq_g;    // next batch: global id per row
  Slots send;                // COR send slots
  int self;
};

template <class T, int VE, int P>  // P >= p: per-source registers
__global__ void __launch_bounds__(128) k_co_apply(T* __restrict__ table, ShardGeom g, double lr,
                                                   const uint64_t* __restrict__ uniq_local,
                                                   const uint64_t* d_nco, const uint32_t* __restrict__ co_rows,
                                                   const uint32_t* __restrict__ bits,
                                                   const uint32_t* __restrict__ slot_us, CSlots cog,
                                                   int p, EcoOut eco, DevErr* err) { FSX_PDL_ENTER();
  using V = VecOf<T, VE>;
  const uint64_t n_co = *d_nco;  // collision rows (k_collide_count's list)
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  const uint64_t wid = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t rb = g.dim * sizeof(T);
  for (uint64_t k = wid; k < n_co; k += warps) {
    const uint64_t u = co_rows[k];
    const uint32_t b = bits[u];
    const uint64_t l = uniq_local[u];
    if (l >= g.local_rows) continue;
    // lane s < p: this row's slot in source s's CO_G message (and, fused,
    // its position in requester s's E_co message); broadcast before the
    // column loop, which only some lanes enter when dim < 32 * VE
    const bool in_b = lane < static_cast<unsigned>(p) && ((b >> lane) & 1u);
    const uint32_t my_slot = in_b ? slot_us[u * kMaxRanks + lane] : 0u;
    uint32_t nb = 0, npos = 0;
    if (eco.partner) {
      const uint32_t un = eco.partner[u];
      nb = eco.bits[un] & ~(1u << eco.self);
      const bool in_nb = lane < static_cast<unsigned>(p) && ((nb >> lane) & 1u);
      if (in_nb) {
        npos = eco.rank_us[un * kMaxRanks + lane];
        reinterpret_cast<uint64_t*>(eco.send.p[lane] + kHdr)[npos] = eco.uniq_g[un];
      }
    }
    uint32_t slot[P], pos[P];
#pragma unroll
    for (int s = 0; s < P; ++s) {
      slot[s] = __shfl_sync(0xffffffffu, my_slot, s);
      pos[s] = __shfl_sync(0xffffffffu, npos, s);
    }
    for (uint32_t col = lane * VE; col < g.dim; col += 32 * VE) {
      // issue every source's load before the ordered sum
      V v[P];
#pragma unroll
      for (int s = 0; s < P; ++s)
        if (s < p && ((b >> s) & 1u))
          v[s] = *reinterpret_cast<const V*>(cog.p[s] + kHdr + static_cast<uint64_t>(slot[s]) * rb +
                                             col * sizeof(T));
      double acc[VE];
#pragma unroll
      for (int x = 0; x < VE; ++x) acc[x] = 0.0;
#pragma unroll
      for (int s = 0; s < P; ++s)
        if (s < p && ((b >> s) & 1u)) {
#pragma unroll
          for (int x = 0; x < VE; ++x) acc[x] = __dadd_rn(acc[x], static_cast<double>(v[s].v[x]));
        }
      V* cell = reinterpret_cast<V*>(table + l * g.dim + col);
      V r = *cell;
      bool bad = false;
#pragma unroll
      for (int x = 0; x < VE; ++x) {
        r.v[x] = static_cast<T>(__dsub_rn(static_cast<double>(r.v[x]), __dmul_rn(lr, acc[x])));
        bad |= !finite_val(r.v[x]);
      }
      *cell = r;
      if (bad) report(err, kErrNonFinite, l * static_cast<uint64_t>(g.p) + g.shard, 0);
#pragma unroll
      for (int s = 0; s < P; ++s)
        if (s < p && ((nb >> s) & 1u))
          *reinterpret_cast<V*>(eco.send.p[s] + idrows_rows_off(eco.totals[2 * s + 1]) +
                                static_cast<uint64_t>(pos[s]) * rb + col * sizeof(T)) = r;
    }
  }
  // E_co may have gone straight to peer windows: visible system-wide before
  // the stream's flag write that follows this kernel
  if (eco.partner) __threadfence_system();
}

}  // namespace fsx
