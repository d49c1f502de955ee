// Host side of the embedding engines: SynchronizedEmbedding (blocking
// baseline, embedding.cpp:235-297) and PrioritizedEmbedding (collision-first
// protocol, embedding.cpp:301-607) over the device kernels in
// engine_kernels.cuh, plus the copy-engine all-to-all transport.
//
// Streams per rank:
//   C  the caller's compute stream: merge (forward) and gradient split/pack
//      (backward) — the only embedding work the model waits on;
//   H  high priority side lane: the collision chain (collision gradients ->
//      owner update -> E_co rows back to the next iteration's requesters);
//   L  low priority side lane: deferred exclusive updates, routing and dedup
//      of iteration i+1, collision detection, exclusive prefetch, masks.
// Cross-stream order is expressed with CUDA events; cross-rank order with
// stream memory operations on flag words in the peers' receive windows
// (cuStreamWriteValue32 after each copy-engine copy, cuStreamWaitValue32 on
// the receiving lane) — no SM ever spins and no kernel touches a peer.
#include <algorithm>
#include <numeric>
#include <deque>
#include <functional>
#include <thread>
#include <chrono>
#include <condition_variable>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <vector>

#include <dlfcn.h>

#include "capi_util.cuh"
#include "engine_kernels.cuh"
#include "nccl.h"

namespace fsx {

enum Channel : int { CH_IDS, CH_ROWS, CH_GRADS, CH_EX, CH_MASK, CH_COG, CH_EXG, CH_COR, CH_IDX, CH_GRP, CH_AG, NCH };

// ---- NCCL, loaded at run time (baseline transport only) ----------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  static NcclApi& get() {
    static NcclApi a = [] {
      NcclApi n;
      // prefer the NCCL torch already loaded into this process
      n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
      if (!n.h) n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!n.h) return n;
      n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(n.h, "ncclGetUniqueId"));
      n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(n.h, "ncclCommInitRank"));
      n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(n.h, "ncclCommDestroy"));
      n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(n.h, "ncclGroupStart"));
      n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(n.h, "ncclGroupEnd"));
      n.Send = reinterpret_cast<decltype(n.Send)>(dlsym(n.h, "ncclSend"));
      n.Recv = reinterpret_cast<decltype(n.Recv)>(dlsym(n.h, "ncclRecv"));
      n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(n.h, "ncclGetErrorString"));
      return n;
    }();
    if (!a.h || !a.Send) raise(FSX_ERR_CONFIG, "fsx: libnccl.so.2 not available for the NCCL baseline");
    return a;
  }
};

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    raise(FSX_ERR_COLLECTIVE, std::string("nccl: ") + what + ": " + NcclApi::get().GetErrorString(r));
}

namespace {

__global__ void k_prefix(const uint64_t* cnt, int p, int stride, uint64_t* off) { FSX_PDL_ENTER();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
    for (int d = 0; d < p; ++d) {
      off[d] = s;
      s += cnt[d * stride];
    }
    off[p] = s;
  }
}

// out[0] = sum of even entries, out[1] = sum of odd entries of t[0..2p)
__global__ void k_sum_pairs(const uint64_t* t, int p, uint64_t* out) { FSX_PDL_ENTER();
  if (threadIdx.x == 0) {
    uint64_t a = 0, b = 0;
    for (int d = 0; d < p; ++d) {
      a += t[2 * d];
      b += t[2 * d + 1];
    }
    out[0] = a;
    out[1] = b;
  }
}


// One rank: the owner partition of route_to_shard_major (embedding.cpp:194-212)
// is the identity — every id goes to self in its original order. One pass
// writes the IDS message, send_pos = j, send_dst = 0 and the counts
// (tot[0] = n, send_off = {0, n}).
__global__ void k_route_self(const uint64_t* __restrict__ ids, uint64_t n, uint64_t total_rows, Slots send,
                             uint32_t* __restrict__ send_pos, uint8_t* __restrict__ send_dst,
                             uint64_t* tot, DevErr* err) { FSX_PDL_ENTER();
  const uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i0 == 0) {
    tot[0] = n;
    tot[16] = 0;
    tot[17] = n;
    reinterpret_cast<uint64_t*>(send.p[0])[0] = n;
    reinterpret_cast<uint64_t*>(send.p[0])[1] = 0;
  }
  uint64_t* msg = reinterpret_cast<uint64_t*>(send.p[0] + kHdr);
  for (uint64_t i = i0; i < n; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t id = ids[i];
    if (id >= total_rows) report(err, kErrRowRange, id, total_rows);
    msg[i] = id;
    send_pos[i] = static_cast<uint32_t>(i);
    send_dst[i] = 0;
  }
}

// compute_collision (embedding.cpp:82-93) on the owner's sorted unique rows:
// co[u] for rows of a also in b (b's flag and a's partner row set alongside),
// plus the counts the statistics need — collision rows (misc[0]) and the
// occurrences of a on them (misc[1]) — warp-aggregated.
__global__ void k_collide_count(const uint64_t* __restrict__ a, const uint64_t* d_na,
                                const uint64_t* __restrict__ b, const uint64_t* d_nb,
                                const uint32_t* __restrict__ seg_a, uint8_t* __restrict__ flag_a,
                                uint8_t* __restrict__ flag_b, uint32_t* __restrict__ partner_a,
                                unsigned long long* misc, uint32_t* __restrict__ co_rows) { FSX_PDL_ENTER();
  const uint64_t na = *d_na, nb = *d_nb;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n_round = (na + 31) & ~uint64_t{31};
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_round; i += stride) {
    bool hit = false;
    unsigned long long occ = 0;
    if (i < na) {
      const uint64_t x = a[i];
      uint64_t lo = 0, hi = nb;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (b[mid] < x) lo = mid + 1; else hi = mid;
      }
      hit = lo < nb && b[lo] == x;
      flag_a[i] = hit ? 1 : 0;
      if (hit) {
        flag_b[lo] = 1;
        partner_a[i] = static_cast<uint32_t>(lo);
        occ = seg_a[i + 1] - seg_a[i];
      }
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, hit);
    for (int o = 16; o > 0; o >>= 1) occ += __shfl_xor_sync(0xffffffffu, occ, o);
    unsigned long long base = 0;
    if ((threadIdx.x & 31u) == 0 && ballot) {
      base = atomicAdd(misc, static_cast<unsigned long long>(__popc(ballot)));
      atomicAdd(misc + 1, occ);
    }
    // the collision rows as a list (warp-aggregated append; the collision
    // update's rows are independent, so their order is immaterial)
    base = __shfl_sync(0xffffffffu, base, 0);
    if (hit) co_rows[base + __popc(ballot & ((1u << (threadIdx.x & 31u)) - 1u))] = static_cast<uint32_t>(i);
  }
}

// one rank: the split / occurrence-rank totals of the statistics from the
// collision counts ([0] exclusive, [1] collision occurrences)
__global__ void k_self_split_totals(const uint64_t* d_n, const uint64_t* misc, int with_co, uint64_t* split_tot,
                                    uint64_t* occ_tot) { FSX_PDL_ENTER();
  if (threadIdx.x == 0) {
    const uint64_t n = *d_n, c = with_co ? misc[1] : 0;
    split_tot[0] = occ_tot[0] = n - c;
    split_tot[1] = occ_tot[1] = c;
  }
}

// one rank: receive = the own IDS message as the owner batch — occurrence j
// is id j from source 0 — and its 32-bit sort keys (local row = id), in one
// pass (k_recv_prefix + k_flatten_recv + k_make_keys at p > 1)
__global__ void k_self_receive(const char* __restrict__ slot, uint64_t cap, uint64_t* __restrict__ cnt,
                               uint64_t* __restrict__ d_n, uint64_t* __restrict__ ids,
                               uint8_t* __restrict__ occ_src, uint32_t* __restrict__ occ_idx,
                               uint32_t* __restrict__ keys, DevErr* err) { FSX_PDL_ENTER();
  const uint64_t n_msg = reinterpret_cast<const uint64_t*>(slot)[0];
  const uint64_t n = n_msg <= cap ? n_msg : cap;
  const uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i0 == 0) {
    if (n_msg > cap) report(err, kErrCapacity, n_msg, cap);
    cnt[0] = n;
    cnt[2] = n;
    cnt[2 + kMaxRanks] = 0;
    *d_n = n;
  }
  const uint64_t* msg = reinterpret_cast<const uint64_t*>(slot + kHdr);
  for (uint64_t j = i0; j < n; j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t id = msg[j];
    ids[j] = id;
    occ_src[j] = 0;
    occ_idx[j] = static_cast<uint32_t>(j);
    keys[j] = static_cast<uint32_t>(id);
  }
}

// receive (embedding.cpp:214-229) at p > 1 in one pass: each thread finds its
// source's offset from the p headers itself (k_recv_prefix), flattens the id
// (k_flatten_recv) and writes its 32-bit sort key (k_make_keys, local row)
__global__ void k_receive_keys(CSlots slots, int p, uint64_t cap, ShardGeom g, uint64_t* __restrict__ cnt,
                               uint64_t* __restrict__ d_n, uint64_t* __restrict__ ids,
                               uint8_t* __restrict__ occ_src, uint32_t* __restrict__ occ_idx,
                               uint32_t* __restrict__ keys, DevErr* err) { FSX_PDL_ENTER();
  const uint64_t total = static_cast<uint64_t>(p) * cap;
  const uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i0 == 0) {
    uint64_t off = 0;
    for (int s = 0; s < p; ++s) {
      const uint64_t n = slot_n(slots.p[s]);
      if (n > cap) report(err, kErrCapacity, n, cap);
      cnt[2 + s] = n;
      cnt[2 + kMaxRanks + s] = off;
      off += n <= cap ? n : cap;
    }
    cnt[0] = off;
    *d_n = off;
  }
  for (uint64_t i = i0; i < total; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(i / cap);
    const uint64_t idx = i - static_cast<uint64_t>(s) * cap;
    const uint64_t ns = slot_n(slots.p[s]);
    if (idx >= ns || idx >= cap) continue;
    uint64_t base = 0;
    for (int q = 0; q < s; ++q) {
      const uint64_t nq = slot_n(slots.p[q]);
      base += nq <= cap ? nq : cap;
    }
    const uint64_t id = reinterpret_cast<const uint64_t*>(slots.p[s] + kHdr)[idx];
    if (!g.owns(id)) report(err, kErrRecvNotOwned, id, g.shard);
    const uint64_t j = base + idx;
    ids[j] = id;
    occ_src[j] = static_cast<uint8_t>(s);
    occ_idx[j] = static_cast<uint32_t>(idx);
    keys[j] = static_cast<uint32_t>(id / static_cast<uint64_t>(g.p));
  }
}

// IterationStats.blocking_bytes (embedding.cpp:498-593) in the reference's
// accounting (8-byte values): collision grads sent + received, E_co
// messages sent + received.
// (single rank: E_co is a message to self carrying every collision row)
__global__ void k_blocking_bytes(int p, uint64_t rb8, const uint64_t* split_tot,
                                 const uint64_t* occ_tot, const uint64_t* pack_tot, CSlots cor_recv,
                                 const uint64_t* co_count, int have_grads, int have_eco, uint64_t* out) { FSX_PDL_ENTER();
  if (threadIdx.x != 0) return;
  uint64_t b = 0;
  if (have_grads)
    for (int d = 0; d < p; ++d) b += rb8 * (split_tot[2 * d + 1] + occ_tot[2 * d + 1]);
  if (have_eco) {
    if (p == 1) {
      b += 2 * (8 + co_count[0] * (8 + rb8));
    } else {
      for (int d = 0; d < p; ++d)
        b += 8 + pack_tot[2 * d + 1] * (8 + rb8) + 8 + slot_n(cor_recv.p[d]) * (8 + rb8);
    }
  }
  *out = b;
}

}  // namespace

// ---- per-batch state -----------------------------------------------------------
struct ReqBatch {  // requester view of one iteration's ids
  uint64_t n = 0;
  DevBuf<uint64_t> ids;
  DevBuf<uint32_t> send_pos, split_rank;
  DevBuf<uint8_t> send_dst, flag;  // flag: collision flag per grouped occurrence
  DevBuf<uint64_t> tot;        // [0..16) send counts, [16..33) send_off
  DevBuf<uint64_t> split_tot;  // [32]
  ScanScratch scan;
  std::vector<uint64_t> h_send, h_split;
  bool has_flags = false;
  int ex_par = -1, cor_par = -1, idx_par = -1;  // channel parities of E_ex / E_co / IDX
  // PRESUM: flattened (owner, slot) segments of the collision occurrences
  DevBuf<uint32_t> seg_flat, perm_flat;
  DevBuf<char*> out_ptr;
  DevBuf<uint64_t> bases;  // k_grp_bases layout
  std::vector<uint64_t> h_slots;  // collision rows per owner (pre-summed message rows)
  SgdScratch plan;  // PRESUM: work lists of the collision pre-sum, built on L
  // split sizes arrive asynchronously: pinned mirror [2*16 split | 16 slots]
  // written by a D2H copy on L; the first reader waits on ev_sizes
  uint64_t* hp_sizes = nullptr;
  cudaEvent_t ev_sizes = nullptr;
  bool sizes_pending = false, sizes_slots = false;
  // PRESUM, direct CO_G: the pre-sum kernel stores each (owner, row) sum
  // straight into the owner's receive window (fixed when the masks are built)
  bool cog_direct = false;
  void sizes(int p) {
    if (!sizes_pending) return;
    FSX_CUDA(cudaEventSynchronize(ev_sizes));
    h_split.assign(hp_sizes, hp_sizes + 2 * p);
    if (sizes_slots) h_slots.assign(hp_sizes + 32, hp_sizes + 32 + p);
    sizes_pending = false;
  }
  ~ReqBatch() {
    if (hp_sizes) cudaFreeHost(hp_sizes);
    if (ev_sizes) cudaEventDestroy(ev_sizes);
  }
  void reserve(uint64_t cap) {
    if (ids.n >= cap && ids.p) return;
    ids.alloc(cap); send_pos.alloc(cap); split_rank.alloc(cap); send_dst.alloc(cap); flag.alloc(cap);
    tot.alloc(48); split_tot.alloc(32);
    seg_flat.alloc(cap + kMaxRanks + 1); perm_flat.alloc(cap); out_ptr.alloc(cap + kMaxRanks); bases.alloc(64);
  }
  const uint64_t* send_off() const { return tot.p + 16; }
};

struct OwnBatch {  // owner view: occurrences received for this shard
  DevBuf<uint64_t> ids;
  DevBuf<uint8_t> occ_src, co;
  DevBuf<uint32_t> occ_idx, occ_rank, bits;
  DevBuf<uint64_t> cnt;  // k_recv_prefix layout: [0]=M, [2+s]=n_s, [2+16+s]=off_s
  DevBuf<uint64_t> misc; // [0] co count, [8..40) pack totals (2p), [40..72) occ totals, [72..88) mask totals
  DevBuf<PackEntry> ex_list, co_list;
  DevBuf<uint32_t> rank_us;  // [unique row][kMaxRanks] position in each source's message
  DevBuf<uint32_t> slot_us;  // PRESUM: [unique row][kMaxRanks] slot in the GRP message
  DevBuf<uint32_t> partner;  // collision row -> its row in the next owner batch
  DevBuf<uint32_t> co_rows;  // the collision rows (any order; count misc[0])
  SortedIds srt;
  ScanScratch scan;
  SgdScratch plan;               // one rank: the update's work lists, built on L
  cudaEvent_t ev_plan = nullptr; // ahead of the backward that applies them
  std::vector<uint64_t> h_recv, h_pack, h_mask;
  bool has_co = false;
  uint64_t m_cap = 0;
  void reserve(uint64_t cap) {
    if (m_cap >= cap && ids.p) return;
    m_cap = cap;
    ids.alloc(cap); occ_src.alloc(cap); co.alloc(cap); occ_idx.alloc(cap); occ_rank.alloc(cap);
    bits.alloc(cap); cnt.alloc(2 + 2 * kMaxRanks + 8); misc.alloc(128); ex_list.alloc(cap);
    co_list.alloc(cap);
    rank_us.alloc(cap * kMaxRanks);
    slot_us.alloc(cap * kMaxRanks);
    partner.alloc(cap);
    co_rows.alloc(cap);
    srt.reserve(cap);
  }
  uint64_t* pack_tot() { return misc.p + 8; }
  uint64_t* occ_tot() { return misc.p + 40; }
  uint64_t* mask_tot() { return misc.p + 72; }
  uint64_t* grp_tot() { return misc.p + 96; }
};

struct PeerView {
  char* base = nullptr;       // peer's receive window (mapped)
  uint32_t* flags = nullptr;  // peer's flag words (mapped)
  bool ipc = false;
  void* local = nullptr;      // in-process peer engine (host mailbox signalling)
};

// In-process signalling: ranks that are threads of one process (the
// reference's InProcessFabric shape, several ranks may share a GPU) hand each
// other CUDA events through a host mailbox instead of flag words. A receiver
// only ever waits on an event that was already recorded, so no stream can park
// on work that is queued behind it (flag waits between streams of ONE GPU can
// deadlock when the streams share a hardware queue).
struct Hub {
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::tuple<const void*, int, uint32_t, int>, cudaEvent_t> box;  // (dst engine, ch, seq, src)
  static Hub& get() {
    static Hub h;
    return h;
  }
  void post(const void* dst, int ch, uint32_t seq, int src, cudaEvent_t ev) {
    {
      std::lock_guard<std::mutex> lk(mu);
      box[{dst, ch, seq, src}] = ev;
    }
    cv.notify_all();
  }
  cudaEvent_t take(const void* dst, int ch, uint32_t seq, int src) {
    static const int timeout_s = [] {
      const char* v = std::getenv("FSX_HUB_TIMEOUT_S");
      return v ? std::atoi(v) : 300;
    }();
    std::unique_lock<std::mutex> lk(mu);
    const auto key = std::make_tuple(dst, ch, seq, src);
    if (!cv.wait_for(lk, std::chrono::seconds(timeout_s), [&] { return box.count(key) > 0; }))
      raise(FSX_ERR_COLLECTIVE, "collective aborted: no message from rank " + std::to_string(src) +
                                    " on channel " + std::to_string(ch) + " (timeout)");
    cudaEvent_t ev = box[key];
    box.erase(key);
    return ev;
  }
};

// Host side lane: one thread per engine that issues the low-priority lane's
// work (route / dedup / collide / prefetch / masks of iteration i+1 and the
// deferred exclusive update). With more than one rank those steps need host
// round trips for copy-engine sizes; on this thread they never stall the
// caller, which only issues compute-stream work and waits (in backward) for
// the masks of its own iteration — by then its model compute is queued.
struct SideLane {
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<std::function<void()>> q;
  uint64_t posted = 0, done = 0;
  bool stop = false;
  std::exception_ptr err;
  void start(int device) {
    th = std::thread([this, device] {
      cudaSetDevice(device);
      for (;;) {
        std::function<void()> f;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return stop || !q.empty(); });
          if (q.empty()) return;
          f = std::move(q.front());
          q.pop_front();
        }
        try {
          f();
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          if (!err) err = std::current_exception();
        }
        {
          std::lock_guard<std::mutex> lk(mu);
          ++done;
        }
        cv.notify_all();
      }
    });
  }
  // returns a ticket: wait_for(ticket) returns once this job has run
  uint64_t post(std::function<void()> f) {
    uint64_t t;
    {
      std::lock_guard<std::mutex> lk(mu);
      q.push_back(std::move(f));
      t = ++posted;
    }
    cv.notify_all();
    return t;
  }
  void drain() { wait_for(~uint64_t{0}); }
  void wait_for(uint64_t ticket) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return done >= (ticket < posted ? ticket : posted); });
    if (err) {
      auto e = err;
      err = nullptr;
      std::rethrow_exception(e);
    }
  }
  ~SideLane() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    if (th.joinable()) th.join();
  }
};

// FSX_HOST_PROF=1 (diagnostic): host nanoseconds per category, printed when
// the engine is destroyed — where a host-bound step's enqueue time goes
enum HostProfSlot { HP_FWD, HP_BWD, HP_WAIT_SIDE, HP_SIDE_JOB, HP_SIZES, HP_FETCH, HP_A2A, HP_N };

struct Engine {
  Ctx* ctx = nullptr;
  bool host_prof = std::getenv("FSX_HOST_PROF") != nullptr;
  bool trace_copies = std::getenv("FSX_TRACE_COPIES") != nullptr;
  bool ce_fork = std::getenv("FSX_CE_FORK") == nullptr || std::atoi(std::getenv("FSX_CE_FORK")) != 0;
  std::atomic<uint64_t> hp_ns[HP_N] = {};
  std::atomic<uint64_t> hp_calls[HP_N] = {};
  struct HostTimer {
    Engine* e;
    int slot;
    std::chrono::steady_clock::time_point t0;
    HostTimer(Engine* en, int k) : e(en->host_prof ? en : nullptr), slot(k) {
      if (e) t0 = std::chrono::steady_clock::now();
    }
    ~HostTimer() {
      if (!e) return;
      e->hp_ns[slot] += static_cast<uint64_t>(
          std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
      ++e->hp_calls[slot];
    }
  };
  std::unique_ptr<SideLane> side;  // p > 1 only
  std::mutex ev_mu;                // event pools are shared by both host threads
  Table* t = nullptr;
  fsx_engine_config cfg{};
  int p = 1, me = 0;
  bool debug = std::getenv("FSX_DEBUG") != nullptr;
  uint64_t cap = 0;       // ids per rank per iteration
  uint32_t rb = 0;        // row bytes
  // receive window (IPC-exportable): per channel [2 parities][p slots][slot]
  char* win = nullptr;
  size_t win_bytes = 0;
  size_t ch_off[NCH] = {};
  size_t ch_slot[NCH] = {};
  uint32_t* flags = nullptr;  // [NCH][kMaxRanks], inside win
  size_t flags_off = 0;
  DevBuf<char> stage;         // send staging, same layout as the channel region of win
  PeerView peer[kMaxRanks];
  ncclComm_t nccl = nullptr;  // FSX_TRANSPORT_NCCL (blocking baseline)
  bool ids_ready = false;     // device ids handed to forward need no stream ordering
  static bool is_host_ptr(const void* ptr) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
      cudaGetLastError();
      return true;  // unregistered host memory
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
  }
  uint32_t seq[NCH] = {};
  cudaStream_t lo = nullptr, hi = nullptr, ux = nullptr;  // ux: deferred exclusive updates
  // lo2: the side lane's part 2 (pack lists, E_ex prefetch, IDX) on its own
  // stream, forked from L after the collision: the next iteration's part 1
  // (route, ids all-to-all, dedup) then overlaps it instead of queueing
  // behind its transfers. FSX_SPLIT_LANE=0: part 2 back on L (A/B).
  cudaStream_t lo2 = nullptr;
  bool split_lane = true;
  cudaStream_t l2() const { return split_lane && lo2 ? lo2 : lo; }
  cudaEvent_t ev_collided = nullptr;  // L: after the collision of (i, i+1)
  // us: the caller's-stream row movers re-issued at the highest priority
  // (FSX_C_PRIO: 1 = the one-rank update, 2 = + the merge), so the side lane
  // (mid priority) does not take the SMs those kernels' CTAs wait for
  cudaStream_t us = nullptr;
  int c_prio = 0;
  int self_serial = 0;
  cudaStream_t boost(cudaStream_t c, int level) {
    if (c_prio < level) return c;
    wait(us, record(c));
    return us;
  }
  void unboost(cudaStream_t c, cudaStream_t s) {
    if (s != c) wait(c, record(s));
  }
  // per-(lane, peer) copy streams: a lane's copies never queue behind another
  // lane's (the collision chain must not wait for prefetch or deferred
  // traffic issued earlier on the same peer)
  static constexpr int kLanes = 5;  // L, H, ux, caller, L2
  cudaStream_t cstream[kLanes][kMaxRanks] = {};
  // copy-stream set of a lane: the prioritized engine's caller stream runs no
  // all-to-all of its own (raw fsx_a2a_ce / all-gather calls borrow H's set),
  // the blocking engine uses only the caller's — fewer streams keep every
  // used stream on its own hardware queue at 8 ranks (CUDA_DEVICE_MAX_CONNECTIONS)
  int lane_map[kLanes] = {0, 1, 2, 3, 4};
  int lane_of(cudaStream_t s) const {
    return lane_map[s == lo ? 0 : s == hi ? 1 : s == ux ? 2 : (lo2 && s == lo2) ? 4 : 3];
  }
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  // exposed-wait timing on the compute stream
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> waits;
  std::vector<cudaEvent_t> timing_pool;
  size_t timing_next = 0;
  // live phase timing (fsx_engine_set_profiling)
  bool prof = false;
  // one span: its events, the lane it ran on (0 caller, 1 L, 2 H, 3 X, 4 the
  // top-priority lane), the channel of an all-to-all (-1 otherwise) and the
  // host time it was issued (timeline traces: fsx_engine_trace)
  struct SpanRec {
    cudaEvent_t first, second;
    int lane, ch;
    int64_t host_ns;
  };
  std::vector<SpanRec> spans[FSX_NUM_PHASES];
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_next = 0;
  cudaEvent_t prof_event() {
    std::lock_guard<std::mutex> lk(ev_mu);
    if (prof_next == prof_pool.size()) {
      cudaEvent_t e;
      FSX_CUDA(cudaEventCreate(&e));
      prof_pool.push_back(e);
    }
    return prof_pool[prof_next++];
  }
  int lane_code(cudaStream_t s) const {
    if (s == lo) return 1;
    if (s == hi) return 2;
    if (s == ux) return 3;
    if (us && s == us) return 4;
    if (lo2 && s == lo2) return 6;
    for (int l = 0; l < kLanes; ++l)
      for (int d = 0; d < p; ++d)
        if (cstream[l][d] && s == cstream[l][d]) return 5;
    return 0;
  }
  struct Span {
    Engine* e;
    int phase, ch;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    int64_t hns = 0;
    Span(Engine* eng, int ph, cudaStream_t st, int chan = -1) : e(eng), phase(ph), ch(chan), s(st) {
      if (e->prof && (ch < 1000 || st)) {
        hns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                  std::chrono::steady_clock::now().time_since_epoch()).count();
        a = e->prof_event();
        FSX_CUDA(cudaEventRecord(a, s));
      }
    }
    ~Span() {
      if (a) {
        cudaEvent_t b = e->prof_event();
        cudaEventRecord(b, s);
        std::lock_guard<std::mutex> lk(e->ev_mu);
        e->spans[phase].push_back(SpanRec{a, b, e->lane_code(s), ch, hns});
      }
    }
  };
  // protocol state
  ReqBatch rq[3];
  OwnBatch ow[3];
  int iter = 0;
  bool forward_done = false;
  bool has_pending = false;
  int exg_par = -1;
  cudaEvent_t ev_ex_ready = nullptr, ev_co_ready = nullptr, ev_mask = nullptr, ev_split = nullptr;
  // stats: pinned chunks of kStatsChunk iterations x 3, never moved or freed
  // while iterations run (cudaFreeHost would synchronize the device)
  static constexpr int kStatsChunk = 1024;
  std::vector<uint64_t*> h_stats;
  DevBuf<uint64_t> d_stats;  // ring of 3 x 4
  int stats_n = 0;
  uint64_t* stat_row(int i) { return h_stats[i / kStatsChunk] + 3 * (i % kStatsChunk); }
  ScanScratch scan;

  ReqBatch& R(int i) { return rq[((i % 3) + 3) % 3]; }
  OwnBatch& O(int i) { return ow[((i % 3) + 3) % 3]; }

  char* recv_slot(int ch, int par, int src) const {
    return win + ch_off[ch] + (static_cast<size_t>(par) * p + src) * ch_slot[ch];
  }
  char* stage_slot(int ch, int par, int dst) const {
    // self slot of the staging area is unused: self messages go straight to
    // this rank's own receive slot
    if (dst == me) return recv_slot(ch, par, dst);
    return stage.p + ch_off[ch] + (static_cast<size_t>(par) * p + dst) * ch_slot[ch];
  }
  Slots send_slots(int ch, int par) const {
    Slots s{};
    for (int d = 0; d < p; ++d) s.p[d] = stage_slot(ch, par, d);
    return s;
  }
  CSlots recv_slots(int ch, int par) const {
    CSlots s{};
    for (int d = 0; d < p; ++d) s.p[d] = recv_slot(ch, par, d);
    return s;
  }
  int next_par(int ch) { return static_cast<int>(++seq[ch] & 1u); }

  cudaEvent_t record(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(ev_mu);
    if (ev_next == ev_pool.size()) {
      cudaEvent_t e;
      FSX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev_pool.push_back(e);
    }
    // Handles kept across an iteration (ev_merged, ev_next_ready, the deferred
    // split, ev_pack) are waited on after both host threads recorded up to
    // ~20 + 8p more events; the ring must not wrap within that window.
    const size_t ring = std::max<size_t>(256, 128 * static_cast<size_t>(p));
    cudaEvent_t e = ev_pool[ev_next];
    ev_next = (ev_next + 1) % ring;
    if (ev_pool.size() < ring && ev_next == 0) ev_next = ev_pool.size();
    FSX_CUDA(cudaEventRecord(e, s));
    return e;
  }
  void wait(cudaStream_t s, cudaEvent_t e) {
    if (e) FSX_CUDA(cudaStreamWaitEvent(s, e, 0));
  }
  cudaEvent_t timing_event() {
    // pairs accumulate across iterations until fsx_engine_exposed_ms reads
    // them; only then is the pool recycled
    if (timing_next == timing_pool.size()) {
      cudaEvent_t e;
      FSX_CUDA(cudaEventCreate(&e));
      timing_pool.push_back(e);
    }
    return timing_pool[timing_next++];
  }
  // compute stream waits on embedding traffic; the pair measures the stall
  void exposed_wait(cudaStream_t c, std::initializer_list<cudaEvent_t> evs) {
    Span sp(this, FSX_PHASE_EXPOSED, c);
    cudaEvent_t a = timing_event(), b = timing_event();
    FSX_CUDA(cudaEventRecord(a, c));
    for (cudaEvent_t e : evs) wait(c, e);
    FSX_CUDA(cudaEventRecord(b, c));
    waits.emplace_back(a, b);
  }

  std::vector<uint64_t> fetch(const uint64_t* d, int n, cudaStream_t s) {
    HostTimer ht(this, HP_FETCH);
    if (debug)
      std::fprintf(stderr, "[fsx r%d] fetch on %s\n", me, s == lo ? "L" : s == hi ? "H" : "C");
    std::vector<uint64_t> h(n);
    FSX_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, s));
    FSX_CUDA(cudaStreamSynchronize(s));
    return h;
  }

  // copy-engine all-to-all of channel `ch` (parity `par`): bytes[d] to rank d.
  // Self messages are already in place. Returns after enqueueing; `s` then
  // waits for every peer's message to this rank.
  // Byte all-to-all of channel `ch` (parity `par`): bytes[d] to rank d; self
  // messages are already in place. recv_bytes (NCCL only) = what each peer
  // sends here. On the caller's compute stream the whole exchange is blocking
  // main-lane communication and is timed as exposed (sim.cpp:25-35).
  void a2a(int ch, int par, const std::vector<uint64_t>& bytes, cudaStream_t s,
           const std::vector<uint64_t>* recv_bytes = nullptr) {
    if (p == 1) return;
    cudaEvent_t t0 = nullptr;
    if (s == cur_c) {
      t0 = timing_event();
      FSX_CUDA(cudaEventRecord(t0, s));
    }
    if (nccl) {
      a2a_nccl(ch, par, bytes, recv_bytes, s);
    } else {
      a2a_ce(ch, par, bytes, s);
    }
    if (t0) {
      cudaEvent_t t1 = timing_event();
      FSX_CUDA(cudaEventRecord(t1, s));
      waits.emplace_back(t0, t1);
    }
  }

  void a2a_nccl(int ch, int par, const std::vector<uint64_t>& bytes,
                const std::vector<uint64_t>* recv_bytes, cudaStream_t s) {
    Span sp(this, FSX_PHASE_A2A, s, ch);
    NcclApi& N = NcclApi::get();
    std::vector<uint64_t> rb_local;
    if (!recv_bytes) {
      // size round first (comm.cpp:328-341): every peer's 16-byte header
      nccl_check(N.GroupStart(), "group start");
      for (int k = 1; k < p; ++k) {
        const int d = (me + k) % p;
        nccl_check(N.Send(stage_slot(ch, par, d), kHdr, ncclChar, d, nccl, s), "send header");
        nccl_check(N.Recv(recv_slot(ch, par, d), kHdr, ncclChar, d, nccl, s), "recv header");
      }
      nccl_check(N.GroupEnd(), "group end");
      rb_local.assign(p, 0);
      std::vector<uint64_t> hdr(2 * p);
      for (int d = 0; d < p; ++d)
        if (d != me) FSX_CUDA(cudaMemcpyAsync(&hdr[2 * d], recv_slot(ch, par, d), kHdr, cudaMemcpyDeviceToHost, s));
      FSX_CUDA(cudaStreamSynchronize(s));
      for (int d = 0; d < p; ++d)
        if (d != me) rb_local[d] = hdr[2 * d] * elem_bytes(ch);
      recv_bytes = &rb_local;
      nccl_check(N.GroupStart(), "group start");
      for (int k = 1; k < p; ++k) {
        const int d = (me + k) % p;
        if (bytes[d] > kHdr)
          nccl_check(N.Send(stage_slot(ch, par, d) + kHdr, bytes[d] - kHdr, ncclChar, d, nccl, s), "send");
        if ((*recv_bytes)[d])
          nccl_check(N.Recv(recv_slot(ch, par, d) + kHdr, (*recv_bytes)[d], ncclChar, d, nccl, s), "recv");
      }
      nccl_check(N.GroupEnd(), "group end");
      return;
    }
    nccl_check(N.GroupStart(), "group start");
    for (int k = 1; k < p; ++k) {
      const int d = (me + k) % p;
      if (bytes[d]) nccl_check(N.Send(stage_slot(ch, par, d), bytes[d], ncclChar, d, nccl, s), "send");
      if ((*recv_bytes)[d]) nccl_check(N.Recv(recv_slot(ch, par, d), (*recv_bytes)[d], ncclChar, d, nccl, s), "recv");
    }
    nccl_check(N.GroupEnd(), "group end");
  }
  // payload bytes per counted element of a channel (after the header)
  uint64_t elem_bytes(int ch) const { return ch == CH_IDS ? 8 : ch == CH_MASK ? 1 : ch == CH_IDX ? 4 : rb; }
  bool presum() const { return (cfg.flags & FSX_ENGINE_PRESUM) != 0; }

  void a2a_ce(int ch, int par, const std::vector<uint64_t>& bytes, cudaStream_t s) {
    HostTimer ht(this, HP_A2A);
    const uint32_t v = seq[ch];
    if (debug)
      std::fprintf(stderr, "[fsx r%d] a2a ch=%d seq=%u par=%d stream=%s\n", me, ch, v, par,
                   s == lo ? "L" : s == hi ? "H" : "C");
    Span sp(this, FSX_PHASE_A2A, s, ch);
    // Each peer's copy + flag on its own copy stream, joined back into `s`.
    // A GPU's copy engine runs one peer copy at a time anyway (measured: the
    // p-1 copies of an all-to-all serialise even on separate streams), but
    // the fork keeps `s` free for work that does not need the copies.
    // FSX_CE_FORK=0: the copies straight on `s` (3 host calls per peer fewer;
    // A/B at N=2/4 within run-to-run spread: profiles/r2_split_lane_ab.txt).
    cudaEvent_t fork = ce_fork ? record(s) : nullptr;
    for (int k = 1; k < p; ++k) {
      const int d = (me + k) % p;  // stagger destinations across the NVSwitch
      const PeerView& pv = peer[d];
      if (!pv.base) raise(FSX_ERR_COLLECTIVE, "all_to_all: peer " + std::to_string(d) + " not connected");
      cudaStream_t cs = ce_fork ? cstream[lane_of(s)][d] : s;
      if (ce_fork) wait(cs, fork);
      char* dst = pv.base + ch_off[ch] + (static_cast<size_t>(par) * p + me) * ch_slot[ch];
      {
        // FSX_TRACE_COPIES: a span per copy for fsx_engine_trace (not in the phase sums)
        Span cp(this, FSX_PHASE_A2A, trace_copies ? cs : nullptr, 1000 + 16 * ch + d);
        if (bytes[d]) FSX_CUDA(cudaMemcpyAsync(dst, stage_slot(ch, par, d), bytes[d], cudaMemcpyDefault, cs));
      }
      if (pv.local) {
        cudaEvent_t ev;
        FSX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        FSX_CUDA(cudaEventRecord(ev, cs));
        Hub::get().post(pv.local, ch, v, me, ev);
      } else {
        FSX_CU(drv::write_value32()(reinterpret_cast<CUstream>(cs),
                                    reinterpret_cast<CUdeviceptr>(pv.flags + ch * kMaxRanks + me), v,
                                    CU_STREAM_WRITE_VALUE_DEFAULT));
      }
      // the sender's staging slot is reused two uses later: `s` must not run
      // ahead of this copy
      if (ce_fork) wait(s, record(cs));
    }
    for (int k = 1; k < p; ++k) {
      const int src = (me + p - k) % p;
      if (peer[src].local) {
        cudaEvent_t ev = Hub::get().take(this, ch, v, src);
        FSX_CUDA(cudaStreamWaitEvent(s, ev, 0));
        FSX_CUDA(cudaEventDestroy(ev));
      } else {
        FSX_CU(drv::wait_value32()(reinterpret_cast<CUstream>(s),
                                   reinterpret_cast<CUdeviceptr>(flags + ch * kMaxRanks + src), v,
                                   CU_STREAM_WAIT_VALUE_GEQ));
      }
    }
  }

  // ---- copy-engine all-gather (comm.cpp:185-306 analogue) -------------------
  // Every rank's chunk (16-byte header + payload) sits in its own receive slot
  // `me` of channel CH_AG (parity par); afterwards slot d holds rank d's chunk
  // on every rank. ring == false: each rank copies its chunk straight to every
  // peer (NVSwitch: full bandwidth to each). ring == true: the reference's
  // SmFree schedule (comm.cpp:214-236) — p-1 stages, at stage st rank r
  // forwards chunk (r - st) mod p to r + 1, each stage gated on the previous
  // stage's arrival from r - 1. Flag values: one sequence number per stage.
  uint32_t ag_calls = 0;
  void all_gather_ce(int par, uint64_t bytes, bool ring, cudaStream_t s) {
    if (p == 1) return;
    Span sp(this, FSX_PHASE_A2A, s);
    const int ch = CH_AG;
    auto peer_slot = [&](int d, int chunk) {
      return peer[d].base + ch_off[ch] + (static_cast<size_t>(par) * p + chunk) * ch_slot[ch];
    };
    auto send = [&](cudaStream_t cs, int d, int chunk, uint64_t n, uint32_t v) {
      const PeerView& pv = peer[d];
      if (!pv.base) raise(FSX_ERR_COLLECTIVE, "all_gather: peer " + std::to_string(d) + " not connected");
      if (n) FSX_CUDA(cudaMemcpyAsync(peer_slot(d, chunk), recv_slot(ch, par, chunk), n, cudaMemcpyDefault, cs));
      if (pv.local) {
        cudaEvent_t ev;
        FSX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        FSX_CUDA(cudaEventRecord(ev, cs));
        Hub::get().post(pv.local, ch, v, me, ev);
      } else {
        FSX_CU(drv::write_value32()(reinterpret_cast<CUstream>(cs),
                                    reinterpret_cast<CUdeviceptr>(pv.flags + ch * kMaxRanks + me), v,
                                    CU_STREAM_WRITE_VALUE_DEFAULT));
      }
    };
    auto recv_wait = [&](cudaStream_t ws, int src, uint32_t v) {
      if (peer[src].local) {
        cudaEvent_t ev = Hub::get().take(this, ch, v, src);
        FSX_CUDA(cudaStreamWaitEvent(ws, ev, 0));
        FSX_CUDA(cudaEventDestroy(ev));
      } else {
        FSX_CU(drv::wait_value32()(reinterpret_cast<CUstream>(ws),
                                   reinterpret_cast<CUdeviceptr>(flags + ch * kMaxRanks + src), v,
                                   CU_STREAM_WAIT_VALUE_GEQ));
      }
    };
    cudaEvent_t fork = record(s);
    if (!ring) {
      const uint32_t v = ++seq[ch];
      for (int k = 1; k < p; ++k) {
        const int d = (me + k) % p;
        cudaStream_t cs = cstream[lane_of(s)][d];
        wait(cs, fork);
        send(cs, d, me, kHdr + bytes, v);
        wait(s, record(cs));
      }
      for (int k = 1; k < p; ++k) recv_wait(s, (me + p - k) % p, v);
      return;
    }
    // ring: chunk sizes differ per rank, so every stage moves the whole slot
    // prefix the largest chunk can occupy (bytes is the caller's bound)
    const int right = (me + 1) % p, left = (me + p - 1) % p;
    cudaStream_t cs = cstream[lane_of(s)][right];
    wait(cs, fork);
    const uint32_t v0 = seq[ch];
    for (int st = 0; st < p - 1; ++st) {
      if (st > 0) recv_wait(cs, left, v0 + st);  // chunk (me - st) arrived at stage st - 1
      send(cs, right, ((me - st) % p + p) % p, kHdr + bytes, v0 + st + 1);
    }
    seq[ch] = v0 + p - 1;
    recv_wait(s, left, v0 + p - 1);
    wait(s, record(cs));
  }

  int nc2() const { return p <= 4 ? 8 : 16; }  // counters for 2p classes

  // ---- requester: route a batch (embedding.cpp:185-212) ----------------------
  // exact: fetch the per-owner counts (the blocking paths size their row
  // messages by them). Otherwise the IDS copies are bounded by n — every
  // owner's message has at most n ids — and no host round trip is taken,
  // unless that bound is large (then the exact sizes are cheaper).
  static constexpr uint64_t kBoundedCopyMax = 2ull << 20;
  int route(ReqBatch& r, const uint64_t* d_ids, uint64_t n, cudaStream_t s, bool exact = true) {
    Span sp(this, FSX_PHASE_ROUTE, s);
    if (n > cap) raise(FSX_ERR_INVALID_ARGUMENT, "embedding: batch of " + std::to_string(n) +
                                                    " ids exceeds engine capacity " + std::to_string(cap));
    r.reserve(cap);
    r.n = n;
    r.has_flags = false;
    if (n && d_ids != r.ids.p) FSX_CUDA(cudaMemcpyAsync(r.ids.p, d_ids, n * 8, cudaMemcpyDeviceToDevice, s));
    const int par = next_par(CH_IDS);
    Slots send = send_slots(CH_IDS, par);
    FSX_CUDA(cudaMemsetAsync(r.tot.p, 0, 48 * 8, s));
    if (p == 1) {
      FSX_LAUNCH(ctx, k_route_self, grid_for(ctx, n ? n : 1, 256, 8), 256, 0, s, r.ids.p, n, t->g.total_rows, send,
                 r.send_pos.p, r.send_dst.p, r.tot.p, ctx->d_err);
      return par;
    }
    if (p <= 8) {
      RouteOp<8> op{r.ids.p, t->g.total_rows, p, r.tot.p, send, r.send_pos.p, r.send_dst.p, cap, ctx->d_err};
      run_scan(ctx, op, n, nullptr, r.scan, r.tot.p, s);
    } else {
      RouteOp<16> op{r.ids.p, t->g.total_rows, p, r.tot.p, send, r.send_pos.p, r.send_dst.p, cap, ctx->d_err};
      run_scan(ctx, op, n, nullptr, r.scan, r.tot.p, s);
    }
    FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, send, p, r.tot.p, 1, cap, ctx->d_err);
    FSX_LAUNCH(ctx, k_prefix, 1, 32, 0, s, r.tot.p, p, 1, r.tot.p + 16);
    if (p > 1) {
      std::vector<uint64_t> bytes(p);
      if (exact || 8 * n > kBoundedCopyMax) {
        r.h_send = fetch(r.tot.p, p, s);
        for (int d = 0; d < p; ++d) bytes[d] = kHdr + 8 * r.h_send[d];
      } else {
        r.h_send.clear();
        for (int d = 0; d < p; ++d) bytes[d] = kHdr + 8 * n;
      }
      a2a(CH_IDS, par, bytes, s);
    }
    return par;
  }

  // ---- owner: receive + dedup (embedding.cpp:214-229) -------------------------
  // exact: fetch the per-source counts (blocking paths); the prioritized
  // IDX / MASK messages are bounded by the capacity instead
  void receive(OwnBatch& o, int ids_par, cudaStream_t s, bool exact = true) {
    Span sp(this, FSX_PHASE_DEDUP, s);
    o.reserve(static_cast<uint64_t>(p) * cap);
    o.has_co = false;
    CSlots slots = recv_slots(CH_IDS, ids_par);
    if (p == 1 && t->key_bits() <= 32) {
      o.srt.reserve(o.m_cap);
      FSX_LAUNCH(ctx, k_self_receive, grid_for(ctx, cap, 256, 8), 256, 0, s, slots.p[0], cap, o.cnt.p, o.srt.d_n(),
                 o.ids.p, o.occ_src.p, o.occ_idx.p, o.srt.k32a.p, ctx->d_err);
      o.srt.run(ctx, o.ids.p, o.m_cap, t->g, true, false, t->key_bits(), s, /*keys_ready=*/true);
    } else if (t->key_bits() <= 32) {
      o.srt.reserve(o.m_cap);
      FSX_LAUNCH(ctx, k_receive_keys, grid_for(ctx, static_cast<uint64_t>(p) * cap, 256, 8), 256, 0, s, slots, p,
                 cap, t->g, o.cnt.p, o.srt.d_n(), o.ids.p, o.occ_src.p, o.occ_idx.p, o.srt.k32a.p, ctx->d_err);
      o.srt.run(ctx, o.ids.p, o.m_cap, t->g, true, false, t->key_bits(), s, /*keys_ready=*/true);
    } else {
      FSX_LAUNCH(ctx, k_recv_prefix, 1, 32, 0, s, slots, p, cap, o.cnt.p, ctx->d_err);
      FSX_CUDA(cudaMemcpyAsync(o.srt.d_n(), o.cnt.p, 8, cudaMemcpyDeviceToDevice, s));
      FSX_LAUNCH(ctx, k_flatten_recv, grid_for(ctx, static_cast<uint64_t>(p) * cap, 256, 8), 256, 0, s,
                 slots, p, cap, o.cnt.p, t->g, o.ids.p, o.occ_src.p, o.occ_idx.p, ctx->d_err);
      o.srt.run(ctx, o.ids.p, o.m_cap, t->g, true, false, t->key_bits(), s);
    }
    if (p > 1 || presum()) {  // requester bits per row: one source at p = 1
      FSX_CUDA(cudaMemsetAsync(o.bits.p, 0, o.m_cap * 4, s));
      FSX_LAUNCH(ctx, k_src_bits, grid_for(ctx, o.m_cap, 256, 8), 256, 0, s, o.srt.inverse.p,
                 o.occ_src.p, o.srt.d_n(), o.bits.p);
    }
    if (p > 1 && exact) o.h_recv = fetch(o.cnt.p + 2, p, s);
    else o.h_recv.clear();
  }
  // bytes of a per-occurrence message of `elem` bytes to every source
  std::vector<uint64_t> occ_msg_bytes(const OwnBatch& o, uint64_t elem) const {
    std::vector<uint64_t> bytes(p);
    for (int d = 0; d < p; ++d) bytes[d] = kHdr + elem * (o.h_recv.empty() ? cap : o.h_recv[d]);
    return bytes;
  }

  // full-row deterministic update of an owner batch from a grads channel
  // self_grads != nullptr: this rank's own occurrences read the caller's
  // gradient rows in place (row self_pos[e] for element e of its own message)
  void update(OwnBatch& o, int ch, int par, const uint8_t* select, uint8_t want, bool by_rank,
              cudaStream_t s, int phase = FSX_PHASE_UPDATE, const void* self_grads = nullptr,
              const uint32_t* self_pos = nullptr) {
    Span sp(this, phase, s);
    RowSegments rs{o.srt.uniq.p, o.srt.seg_start.p, o.srt.perm, o.srt.d_u(), select, want, o.srt.inverse.p};
    const uint64_t m = o.m_cap;
    const char* sb = static_cast<const char*>(self_grads);
    if (t->dtype == FSX_F32) {
      GradRows<float> gr{recv_slot(ch, par, 0) + kHdr, ch_slot[ch], o.occ_src.p,
                         by_rank ? o.occ_rank.p : o.occ_idx.p, rb, sb, self_pos, sb ? me : -1};
      sgd_update_rows<float>(ctx, *t, rs, m, m, gr, cfg.reduce_chunk, sgd_for(s), nullptr, s);
    } else {
      GradRows<double> gr{recv_slot(ch, par, 0) + kHdr, ch_slot[ch], o.occ_src.p,
                          by_rank ? o.occ_rank.p : o.occ_idx.p, rb, sb, self_pos, sb ? me : -1};
      sgd_update_rows<double>(ctx, *t, rs, m, m, gr, cfg.reduce_chunk, sgd_for(s), nullptr, s);
    }
  }
  // one rank: the whole update of an owner batch reads the caller's gradient
  // array in occurrence order (row j of the array is occurrence j), so its
  // work lists depend on the batch's row segments alone and are built on L a
  // whole iteration early; the backward only runs the update kernels.
  bool self_plan() const { return p == 1 && !presum(); }
  void plan_self(OwnBatch& o, cudaStream_t s) {
    RowSegments rs{o.srt.uniq.p, o.srt.seg_start.p, o.srt.perm, o.srt.d_u(), nullptr, 0, o.srt.inverse.p};
    if (t->dtype == FSX_F32)
      sgd_plan<float>(ctx, *t, rs, o.m_cap, o.m_cap, nullptr, cfg.reduce_chunk, o.plan, s);
    else
      sgd_plan<double>(ctx, *t, rs, o.m_cap, o.m_cap, nullptr, cfg.reduce_chunk, o.plan, s);
    o.ev_plan = record(s);
  }
  void apply_self(OwnBatch& o, const void* grads, cudaStream_t c0) {
    exposed_wait(c0, {o.ev_plan});
    cudaStream_t c = boost(c0, 1);
    {
      Span sp(this, FSX_PHASE_CO_UPDATE, c);
      RowSegments rs{o.srt.uniq.p, o.srt.seg_start.p, o.srt.perm, o.srt.d_u(), nullptr, 0};
      if (t->dtype == FSX_F32) {
        GradRows<float> gr{static_cast<const char*>(grads), 0, nullptr, nullptr, rb};
        sgd_apply<float>(ctx, *t, rs, o.m_cap, o.m_cap, gr, cfg.reduce_chunk, o.plan, nullptr, c);
      } else {
        GradRows<double> gr{static_cast<const char*>(grads), 0, nullptr, nullptr, rb};
        sgd_apply<double>(ctx, *t, rs, o.m_cap, o.m_cap, gr, cfg.reduce_chunk, o.plan, nullptr, c);
      }
    }
    unboost(c0, c);
  }
  SgdScratch sgd[3];  // one per lane that updates: ux, hi, compute
  SgdScratch& sgd_for(cudaStream_t s) { return sgd[s == ux ? 0 : s == hi ? 1 : 2]; }

  // ---- sync building blocks ---------------------------------------------------------
  // owner lookup per occurrence -> ROWS -> requester scatter (embedding.cpp:244-264)
  void serve_blocking(ReqBatch& r, OwnBatch& o, void* d_out, cudaStream_t s) {
    Span sp(this, FSX_PHASE_SERVE, s);
    const int par = next_par(CH_ROWS);
    Slots send = send_slots(CH_ROWS, par);
    OwnerLookupMap lm{static_cast<const char*>(t->values), o.ids.p, o.occ_src.p, o.occ_idx.p, send, rb, p};
    launch_copy_rows(ctx, lm, o.m_cap, o.srt.d_n(), rb, s);
    FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, send, p, o.cnt.p + 2, 1, cap, ctx->d_err);
    if (p > 1) {
      std::vector<uint64_t> bytes(p), rbytes(p);
      for (int d = 0; d < p; ++d) {
        bytes[d] = kHdr + rb * o.h_recv[d];
        rbytes[d] = kHdr + rb * r.h_send[d];
      }
      a2a(CH_ROWS, par, bytes, s, &rbytes);
    }
    RequesterScatterMap sm{recv_slots(CH_ROWS, par), r.send_pos.p, r.send_dst.p, r.send_off(),
                           static_cast<char*>(d_out), rb};
    launch_copy_rows(ctx, sm, r.n, nullptr, rb, s);
  }

  // requester grads -> GRADS -> owner full update (embedding.cpp:276-295)
  // The gradients of this rank's own rows are never staged: the update reads
  // them from the caller's buffer (valid for the whole call: the update runs
  // on the caller's stream).
  void update_blocking(ReqBatch& r, OwnBatch& o, const void* d_grads, cudaStream_t s) {
    Span sp(this, FSX_PHASE_UPDATE, s);
    const int par = next_par(CH_GRADS);
    Slots send = send_slots(CH_GRADS, par);
    const uint64_t self_off = p > 1 ? std::accumulate(r.h_send.begin(), r.h_send.begin() + me, uint64_t{0}) : 0;
    if (p > 1) {
      GradPackMap gm{static_cast<const char*>(d_grads), r.send_pos.p, r.send_dst.p, r.send_off(),
                     nullptr, nullptr, send, send, rb, 0, me};
      launch_copy_rows(ctx, gm, r.n, nullptr, rb, s);
      FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, send, p, r.tot.p, 1, cap, ctx->d_err);
    }
    if (p > 1) {
      std::vector<uint64_t> bytes(p), rbytes(p);
      for (int d = 0; d < p; ++d) {
        bytes[d] = kHdr + rb * r.h_send[d];
        rbytes[d] = kHdr + rb * o.h_recv[d];
      }
      a2a(CH_GRADS, par, bytes, s, &rbytes);
    }
    update(o, CH_GRADS, par, nullptr, 0, false, s, FSX_PHASE_UPDATE, d_grads, r.send_pos.p + self_off);
  }

  // ---- prioritized building blocks ----------------------------------------------------
  // collision of (cur, next) owner batches + pack lists + EX prefetch of next
  // (embedding.cpp:360-390)
  void collide(OwnBatch& oc, OwnBatch& on, cudaStream_t s) {
    Span sp(this, FSX_PHASE_COLLIDE, s);
    FSX_CUDA(cudaMemsetAsync(on.co.p, 0, on.m_cap, s));
    FSX_CUDA(cudaMemsetAsync(oc.misc.p, 0, 16, s));
    FSX_LAUNCH(ctx, k_collide_count, grid_for(ctx, oc.m_cap, 256, 8), 256, 0, s, oc.srt.uniq_g.p,
               oc.srt.d_u(), on.srt.uniq_g.p, on.srt.d_u(), oc.srt.seg_start.p, oc.co.p, on.co.p, oc.partner.p,
               reinterpret_cast<unsigned long long*>(oc.misc.p), oc.co_rows.p);
    oc.has_co = true;
    on.has_co = false;
  }
  // pack lists + E_ex prefetch + IDX of the next batch (its collision flags
  // come from collide)
  // (a) pack lists of the next batch + their sizes on the host: all the
  // collision chain's E_co pack needs (ev_pack)
  void prefetch_pack(OwnBatch& on, cudaStream_t s) {
    ev_pack = nullptr;
    if (p == 1) return;
    Span sp(this, FSX_PHASE_COLLIDE, s);
    FSX_CUDA(cudaMemsetAsync(on.pack_tot(), 0, 32 * 8, s));
    if (nc2() == 8) {
      OwnerPackOp<8> op{on.bits.p, on.co.p, p, on.pack_tot(), on.ex_list.p, on.co_list.p, on.rank_us.p};
      run_scan(ctx, op, on.m_cap, on.srt.d_u(), on.scan, on.pack_tot(), s);
    } else {
      OwnerPackOp<16> op{on.bits.p, on.co.p, p, on.pack_tot(), on.ex_list.p, on.co_list.p, on.rank_us.p};
      run_scan(ctx, op, on.m_cap, on.srt.d_u(), on.scan, on.pack_tot(), s);
    }
    FSX_LAUNCH(ctx, k_sum_pairs, 1, 32, 0, s, on.pack_tot(), p, on.misc.p + 2);
    ev_pack = record(s);
    on.h_pack = fetch(on.pack_tot(), 2 * p, s);
  }
  cudaEvent_t ev_pack = nullptr;
  // (b) E_ex prefetch + IDX of the next batch
  void prefetch(OwnBatch& on, ReqBatch& rn, cudaStream_t s) {
    Span sp(this, FSX_PHASE_COLLIDE, s);
    if (p == 1) {
      // single rank: every message would go to self, and self rows are
      // merged straight from the table — no pack lists, no copies. IDX still
      // carries each occurrence's collision bit (the merge's two halves).
      // The merge must see the deferred exclusive update first.
      const int ipar = next_par(CH_IDX);
      FSX_LAUNCH(ctx, k_idx_pack, grid_for(ctx, on.m_cap, 256, 8), 256, 0, s, on.srt.inverse.p, on.occ_src.p,
                 on.occ_idx.p, on.srt.d_n(), on.rank_us.p, on.co.p, send_slots(CH_IDX, ipar), me);
      wait(s, ev_ex_applied);
      rn.ex_par = -1;
      rn.idx_par = ipar;
      return;
    }
    const int par = next_par(CH_EX);
    Slots send = send_slots(CH_EX, par);
    FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, send, p, on.pack_tot(), 2, cap, ctx->d_err);
    IdRowPackMap pm{static_cast<const char*>(t->values), on.srt.uniq.p, on.srt.uniq_g.p, on.ex_list.p,
                    send, on.pack_tot(), 0, rb, me};
    wait(s, ev_ex_applied);  // rows of the previous exclusive set may be prefetched now
    {
      Span sp2(this, FSX_PHASE_PREFETCH, s);
      launch_copy_rows(ctx, pm, on.m_cap * static_cast<uint64_t>(p), on.misc.p + 2, rb, s);
    }
    // IDX: per-occurrence row positions for the next merge, packed before
    // the E_ex copies are queued on this stream (the copies run in its order)
    const int ipar = next_par(CH_IDX);
    Slots isend = send_slots(CH_IDX, ipar);
    FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, isend, p, on.cnt.p + 2, 1, cap, ctx->d_err);
    FSX_LAUNCH(ctx, k_idx_pack, grid_for(ctx, on.m_cap, 256, 8), 256, 0, s, on.srt.inverse.p, on.occ_src.p,
               on.occ_idx.p, on.srt.d_n(), on.rank_us.p, on.co.p, isend, me);
    {
      std::vector<uint64_t> bytes(p);
      for (int d = 0; d < p; ++d) bytes[d] = idrows_rows_off(on.h_pack[2 * d]) + rb * on.h_pack[2 * d];
      a2a(CH_EX, par, bytes, s);
    }
    rn.ex_par = par;
    a2a(CH_IDX, ipar, occ_msg_bytes(on, 4), s);
    rn.idx_par = ipar;
  }

  // MASK messages for the current batch + requester flags + split plan
  // (embedding.cpp:392-408, 524-536)
  void masks_and_split(OwnBatch& oc, ReqBatch& rc, bool with_co, cudaStream_t s) {
    Span sp(this, FSX_PHASE_MASKS, s);
    rc.cog_direct = false;
    if (p == 1 && !presum()) {
      // one rank: the update needs no masks or split plan (it runs whole on
      // the caller's stream); only the statistics need the totals
      // (collision occurrences counted by k_collide_count)
      FSX_LAUNCH(ctx, k_self_split_totals, 1, 32, 0, s, oc.srt.d_n(), oc.misc.p, with_co ? 1 : 0, rc.split_tot.p,
                 oc.occ_tot());
      rc.has_flags = false;
      rc.cog_direct = false;
      return;
    }
    if (with_co && presum()) {
      rc.cog_direct = cog_direct && p > 1;
      // GRP messages: each source's collision occurrences grouped by row
      const int par = next_par(CH_GRP);
      Slots send = send_slots(CH_GRP, par);
      FSX_CUDA(cudaMemsetAsync(oc.grp_tot(), 0, 32 * 8, s));
      if (nc2() == 8) {
        GroupOp<8> op{oc.srt.perm, oc.srt.inverse.p, oc.srt.seg_start.p, oc.occ_src.p, oc.occ_idx.p,
                      oc.co.p, send, oc.slot_us.p};
        run_scan(ctx, op, oc.m_cap, oc.srt.d_n(), oc.scan, oc.grp_tot(), s);
      } else {
        GroupOp<16> op{oc.srt.perm, oc.srt.inverse.p, oc.srt.seg_start.p, oc.occ_src.p, oc.occ_idx.p,
                       oc.co.p, send, oc.slot_us.p};
        run_scan(ctx, op, oc.m_cap, oc.srt.d_n(), oc.scan, oc.grp_tot(), s);
      }
      FSX_LAUNCH(ctx, k_grp_headers, 1, 32, 0, s, send, p, oc.grp_tot());
      if (p > 1) {
        // bounded copies (the whole slot) when small: no host round trip
        std::vector<uint64_t> bytes(p, ch_slot[CH_GRP]);
        if (ch_slot[CH_GRP] > kBoundedCopyMax) {
          const std::vector<uint64_t> g = fetch(oc.grp_tot(), 2 * p, s);
          for (int d = 0; d < p; ++d) bytes[d] = grp_list_off(g[2 * d + 1]) + 4 * g[2 * d];
        }
        a2a(CH_GRP, par, bytes, s);
      }
      FSX_CUDA(cudaMemsetAsync(rc.flag.p, 0, rc.n ? rc.n : 1, s));
      CSlots grp = recv_slots(CH_GRP, par);
      FSX_LAUNCH(ctx, k_grp_bases, 1, 32, 0, s, grp, p, rc.bases.p);
      FSX_LAUNCH(ctx, k_grp_flatten, grid_for(ctx, static_cast<uint64_t>(p) * (cap + 1), 256, 8), 256, 0, s,
                 grp, p, cap, rc.bases.p, rc.send_off(), rc.send_pos.p,
                 cog_direct && p > 1 ? remote_slots(CH_COG, cog_par_next()) : send_slots(CH_COG, cog_par_next()),
                 rb, rc.flag.p, rc.seg_flat.p, rc.perm_flat.p, rc.out_ptr.p);
      // the pre-sum's work lists: the segments and the caller's gradient
      // positions are known now, the gradients only at the backward
      RowSegments prs{nullptr, rc.seg_flat.p, rc.perm_flat.p, rc.bases.p + 16, nullptr, 0};
      if (t->dtype == FSX_F32)
        sgd_plan<float>(ctx, *t, prs, rc.n, rc.n, nullptr, cfg.reduce_chunk, rc.plan, s, rc.out_ptr.p);
      else
        sgd_plan<double>(ctx, *t, prs, rc.n, rc.n, nullptr, cfg.reduce_chunk, rc.plan, s, rc.out_ptr.p);
    } else if (with_co) {
      const int par = next_par(CH_MASK);
      Slots send = send_slots(CH_MASK, par);
      FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, send, p, oc.cnt.p + 2, 1, cap, ctx->d_err);
      FSX_LAUNCH(ctx, k_mask_pack, grid_for(ctx, oc.m_cap, 256, 8), 256, 0, s, oc.srt.inverse.p,
                 oc.occ_src.p, oc.occ_idx.p, oc.srt.d_n(), oc.co.p, send);
      if (p > 1) a2a(CH_MASK, par, occ_msg_bytes(oc, 1), s);
      if (rc.n)
        FSX_LAUNCH(ctx, k_req_flags, grid_for(ctx, rc.n, 256, 8), 256, 0, s, recv_slots(CH_MASK, par),
                   rc.send_dst.p, rc.send_off(), rc.n, rc.flag.p, ctx->d_err);
    }
    rc.has_flags = with_co;
    const uint8_t* flag = with_co ? rc.flag.p : nullptr;
    // split plan (ranks of each occurrence in its (owner, flag) message)
    FSX_CUDA(cudaMemsetAsync(rc.split_tot.p, 0, 32 * 8, s));
    if (nc2() == 8) {
      SplitOp<8> op{rc.send_dst.p, flag, rc.split_rank.p};
      run_scan(ctx, op, rc.n, nullptr, rc.scan, rc.split_tot.p, s);
    } else {
      SplitOp<16> op{rc.send_dst.p, flag, rc.split_rank.p};
      run_scan(ctx, op, rc.n, nullptr, rc.scan, rc.split_tot.p, s);
    }
    // owner side: per-occurrence rank within (source, flag)
    FSX_CUDA(cudaMemsetAsync(oc.occ_tot(), 0, 32 * 8, s));
    if (nc2() == 8) {
      OccRankOp<8> op{oc.occ_src.p, oc.srt.inverse.p, with_co ? oc.co.p : nullptr, oc.occ_rank.p};
      run_scan(ctx, op, oc.m_cap, oc.srt.d_n(), oc.scan, oc.occ_tot(), s);
    } else {
      OccRankOp<16> op{oc.occ_src.p, oc.srt.inverse.p, with_co ? oc.co.p : nullptr, oc.occ_rank.p};
      run_scan(ctx, op, oc.m_cap, oc.srt.d_n(), oc.scan, oc.occ_tot(), s);
    }
    if (p > 1) {
      // split counts (+ collision rows per owner) go to pinned memory without
      // a host round trip here: only the gradient all-to-alls of the coming
      // backward need them, and they read them through rc.sizes()
      rc.sizes_slots = with_co && presum();
      FSX_CUDA(cudaMemcpyAsync(rc.hp_sizes, rc.split_tot.p, 16 * p, cudaMemcpyDeviceToHost, s));
      if (rc.sizes_slots)
        FSX_CUDA(cudaMemcpyAsync(rc.hp_sizes + 32, rc.bases.p + 34, 8 * p, cudaMemcpyDeviceToHost, s));
      FSX_CUDA(cudaEventRecord(rc.ev_sizes, s));
      rc.sizes_pending = true;
    }
  }
  // the CO_G parity the coming backward will use (next_par is taken there)
  int cog_par_next() const { return static_cast<int>((seq[CH_COG] + 1) & 1u); }

  // owner, PRESUM: collision rows from the sources' pre-summed rows; with
  // `on` the E_co messages of the next iteration are packed in the same pass
  // E_co written by the collision update straight into the requesters'
  // receive windows (their slot `me`, over NVLink) instead of local staging +
  // a copy-engine all-to-all: the transfer rides the update's own stores and
  // leaves the chain; signal_direct then only raises the flags.
  // FSX_ECO_DIRECT=1 (opt-in): the collision update stores E_co rows straight
  // into the peers' windows over NVLink — SM-issued communication. Off by
  // default: every byte between ranks then moves on the copy engines (0 SMs).
  // FSX_COG_DIRECT=1 (opt-in, PRESUM): likewise the pre-sum kernel stores the
  // collision gradients into the owners' windows. The copy engines run one
  // copy at a time per GPU (measured: a rank's p-1 copies of an all-to-all
  // serialise), so on the collision chain the fused stores cut the transfer
  // to the kernels' own NVLink stores and one flag round.
  bool eco_direct = false;
  bool cog_direct = false;
  Slots remote_slots(int ch, int par) const {
    Slots r{};
    for (int d = 0; d < p; ++d)
      r.p[d] = d == me ? recv_slot(ch, par, me)
                       : peer[d].base + ch_off[ch] + (static_cast<size_t>(par) * p + me) * ch_slot[ch];
    return r;
  }
  // flags of a channel whose payload the sender's kernels already stored into
  // the peers' windows (ordered by `s`), then wait for every peer's
  void signal_direct(int ch, cudaStream_t s) {
    Span sp(this, FSX_PHASE_A2A, s, ch);
    const uint32_t v = seq[ch];
    for (int k = 1; k < p; ++k) {
      const int d = (me + k) % p;
      const PeerView& pv = peer[d];
      if (pv.local) {
        cudaEvent_t ev;  // one per receiver: the Hub hands it over and the receiver destroys it
        FSX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        FSX_CUDA(cudaEventRecord(ev, s));
        Hub::get().post(pv.local, ch, v, me, ev);
      } else {
        FSX_CU(drv::write_value32()(reinterpret_cast<CUstream>(s),
                                    reinterpret_cast<CUdeviceptr>(pv.flags + ch * kMaxRanks + me), v,
                                    CU_STREAM_WRITE_VALUE_DEFAULT));
      }
    }
    for (int k = 1; k < p; ++k) {
      const int src = (me + p - k) % p;
      if (peer[src].local) {
        cudaEvent_t ev = Hub::get().take(this, ch, v, src);
        FSX_CUDA(cudaStreamWaitEvent(s, ev, 0));
        FSX_CUDA(cudaEventDestroy(ev));
      } else {
        FSX_CU(drv::wait_value32()(reinterpret_cast<CUstream>(s),
                                   reinterpret_cast<CUdeviceptr>(flags + ch * kMaxRanks + src), v,
                                   CU_STREAM_WAIT_VALUE_GEQ));
      }
    }
  }

  void co_apply(OwnBatch& oc, int cog_par, cudaStream_t s, OwnBatch* on = nullptr, int cor_par = -1) {
    CSlots cog = recv_slots(CH_COG, cog_par);
    EcoOut eco{};
    eco.self = me;
    if (on) {
      eco = EcoOut{oc.partner.p, on->bits.p, on->rank_us.p, on->pack_tot(), on->srt.uniq_g.p,
                   eco_direct ? remote_slots(CH_COR, cor_par) : send_slots(CH_COR, cor_par), me};
      FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, eco.send, p, on->pack_tot() + 1, 2, cap, ctx->d_err);
    }
    const unsigned grid = grid_for(ctx, oc.m_cap, 4, 16);
    const bool v16 = rb % 16 == 0;
#define FSX_CO_APPLY_P(T, VE, P)                                                                     \
  FSX_LAUNCH(ctx, (k_co_apply<T, VE, P>), grid, 128, 0, s, static_cast<T*>(t->values), t->g, t->lr,   \
             oc.srt.uniq.p, oc.misc.p, oc.co_rows.p, oc.bits.p, oc.slot_us.p, cog, p, eco, ctx->d_err)
#define FSX_CO_APPLY(T, VE)                                    \
  do {                                                         \
    if (p <= 2) FSX_CO_APPLY_P(T, VE, 2);                      \
    else if (p <= 4) FSX_CO_APPLY_P(T, VE, 4);                 \
    else if (p <= 8) FSX_CO_APPLY_P(T, VE, 8);                 \
    else FSX_CO_APPLY_P(T, VE, 16);                            \
  } while (0)
    if (t->dtype == FSX_F32) {
      if (v16) FSX_CO_APPLY(float, 4); else FSX_CO_APPLY(float, 1);
    } else {
      if (v16) FSX_CO_APPLY(double, 2); else FSX_CO_APPLY(double, 1);
    }
#undef FSX_CO_APPLY_P
#undef FSX_CO_APPLY
  }

  // collision half first (its chain is the exposed one), then the exclusive
  // half, which overlaps the collision all-to-all
  void split_co(ReqBatch& r, const void* d_grads, int cog_par, cudaStream_t s) {
    Span sp(this, FSX_PHASE_SPLIT, s);
    Slots co = r.cog_direct ? remote_slots(CH_COG, cog_par) : send_slots(CH_COG, cog_par);
    if (!r.has_flags) {
      FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, co, p, r.split_tot.p + 1, 2, cap, ctx->d_err);
      return;
    }
    if (!presum()) {
      GradPackMap gm{static_cast<const char*>(d_grads), r.send_pos.p, r.send_dst.p, r.send_off(),
                     r.flag.p, r.split_rank.p, co, co, rb, 2};
      launch_copy_rows(ctx, gm, r.n, nullptr, rb, s);
      FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, co, p, r.split_tot.p + 1, 2, cap, ctx->d_err);
      return;
    }
    // pre-sum the collision occurrences of each (owner, row) straight into
    // the CO_G messages (same chunked reduce as the owner, reduce-only mode)
    RowSegments rs{nullptr, r.seg_flat.p, r.perm_flat.p, r.bases.p + 16, nullptr, 0};
    const uint64_t segs_cap = r.n;  // a segment holds >= 1 occurrence
    // work lists planned on L (masks_and_split); gradient row j = occurrence j
    if (t->dtype == FSX_F32) {
      GradRows<float> gr{static_cast<const char*>(d_grads), 0, nullptr, nullptr, rb};
      sgd_apply<float>(ctx, *t, rs, segs_cap, r.n, gr, cfg.reduce_chunk, r.plan, nullptr, s, r.out_ptr.p);
    } else {
      GradRows<double> gr{static_cast<const char*>(d_grads), 0, nullptr, nullptr, rb};
      sgd_apply<double>(ctx, *t, rs, segs_cap, r.n, gr, cfg.reduce_chunk, r.plan, nullptr, s, r.out_ptr.p);
    }
    FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, co, p, r.bases.p + 34, 1, cap, ctx->d_err);
  }
  void split_ex(ReqBatch& r, const void* d_grads, int exg_par, cudaStream_t s) {
    Span sp(this, FSX_PHASE_SPLIT, s);
    Slots ex = send_slots(CH_EXG, exg_par);
    GradPackMap gm{static_cast<const char*>(d_grads), r.send_pos.p, r.send_dst.p, r.send_off(),
                   r.has_flags ? r.flag.p : nullptr, r.split_rank.p, ex, ex, rb, 1};
    launch_copy_rows(ctx, gm, r.n, nullptr, rb, s);
    FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, ex, p, r.split_tot.p, 2, cap, ctx->d_err);
  }


  // owner: E_co rows of the next batch (embedding.cpp:560-590)
  int send_eco(OwnBatch& on, cudaStream_t s) {
    Span sp(this, FSX_PHASE_ECO, s);
    if (p == 1) return -1;  // the merge reads the updated rows from the table
    const int par = next_par(CH_COR);
    Slots send = send_slots(CH_COR, par);
    FSX_LAUNCH(ctx, k_write_headers, 1, 32, 0, s, send, p, on.pack_tot() + 1, 2, cap, ctx->d_err);
    IdRowPackMap pm{static_cast<const char*>(t->values), on.srt.uniq.p, on.srt.uniq_g.p, on.co_list.p,
                    send, on.pack_tot(), 1, rb, me};
    launch_copy_rows(ctx, pm, on.m_cap * static_cast<uint64_t>(p), on.misc.p + 3, rb, s);
    if (p > 1) {
      std::vector<uint64_t> bytes(p);
      for (int d = 0; d < p; ++d) bytes[d] = idrows_rows_off(on.h_pack[2 * d + 1]) + rb * on.h_pack[2 * d + 1];
      a2a(CH_COR, par, bytes, s);
    }
    return par;
  }

  // requester: merge E_ex / E_co into batch-major rows (embedding.cpp:453-484)
  void merge(ReqBatch& r, void* d_out, cudaStream_t s0, int part = 0) {
    cudaStream_t s = boost(s0, 2);
    merge_on(r, d_out, s, part);
    unboost(s0, s);
  }
  void merge_on(ReqBatch& r, void* d_out, cudaStream_t s, int part) {
    Span sp(this, FSX_PHASE_MERGE, s);
    if (r.idx_par < 0) raise(FSX_ERR_PROTOCOL, "embedding: merge without IDX messages");
    CSlots co{};
    if (p > 1) co = r.cor_par >= 0 ? recv_slots(CH_COR, r.cor_par) : recv_slots(CH_EX, r.ex_par);
    MergeMap mm{recv_slots(CH_IDX, r.idx_par), recv_slots(CH_EX, r.ex_par), co,
                static_cast<const char*>(t->values), r.send_pos.p, r.send_dst.p, r.send_off(), r.ids.p,
                static_cast<char*>(d_out), rb, me, p, ctx->d_err, part};
    launch_copy_rows(ctx, mm, r.n, nullptr, rb, s);
  }

  // ---- protocol --------------------------------------------------------------------
  cudaStream_t cur_c = nullptr;
  cudaEvent_t ev_merged = nullptr;   // C: after the last merge / bootstrap serve
  cudaEvent_t ev_next_ready = nullptr;  // L: owner batch i+1 built + pack lists
  int pending_iter = -1;             // owner batch whose exclusive grads are deferred
  cudaEvent_t ev_pending_split = nullptr;

  void sync_forward(const uint64_t* ids, uint64_t n, void* out, cudaStream_t c) {
    ReqBatch& r = R(0);
    OwnBatch& o = O(0);
    const int par = route(r, ids, n, c);
    receive(o, par, c);
    serve_blocking(r, o, out, c);
    forward_done = true;
  }

  void sync_backward(const void* grads, cudaStream_t c) {
    if (!forward_done) raise(FSX_ERR_PROTOCOL, "embedding: backward before forward");
    update_blocking(R(0), O(0), grads, c);
    forward_done = false;
    ++iter;
  }

  void prio_forward(const uint64_t* ids_cur, uint64_t n_cur, const uint64_t* ids_next,
                    uint64_t n_next, void* out, cudaStream_t c) {
    if (forward_done) raise(FSX_ERR_PROTOCOL, "embedding: forward called twice in one iteration");
    // E_ex of this batch: recorded by the previous forward's side-lane prep
    wait_next_ready();
    cur_ex_ready = rn_ex_ready;
    const int i = iter;
    ReqBatch& rc = R(i);
    OwnBatch& oc = O(i);
    const bool bootstrap = i == 0;
    cudaEvent_t ev_cur = nullptr;
    if (bootstrap) {
      if (ids_cur && is_host_ptr(ids_cur)) {
        rc.reserve(cap);
        if (n_cur > cap)
          raise(FSX_ERR_INVALID_ARGUMENT, "embedding: batch of " + std::to_string(n_cur) +
                                              " ids exceeds engine capacity " + std::to_string(cap));
        if (n_cur) FSX_CUDA(cudaMemcpyAsync(rc.ids.p, ids_cur, n_cur * 8, cudaMemcpyHostToDevice, c));
        ids_cur = rc.ids.p;
      }
      const int par = route(rc, ids_cur, n_cur, c);
      receive(oc, par, c);
      rc.cor_par = -1;
      ev_cur = record(c);
    } else if (rc.n != n_cur) {
      raise(FSX_ERR_PROTOCOL, "embedding: current batch does not match the prefetched ids");
    }
    // ---- side lane L: prepare iteration i+1 (embedding.cpp:355-420) ----
    // The next batch's ids are copied now (the caller's buffer is free once
    // forward returns). Host ids: H2D on L, no tie to the caller's stream.
    // Device ids: ordered after everything the caller enqueued so far,
    // unless the caller declared them ready (fsx_engine_set_ids_ready) —
    // that tie would serialise this prep behind the previous backward.
    const bool next_host = ids_next && is_host_ptr(ids_next);
    if (ids_next && !next_host && !ids_ready) wait(lo, record(c));
    wait(lo, ev_cur);
    wait(lo, ev_merged);  // slots of the parity reused below were read by the last merge
    if (ids_next) {
      ReqBatch& rn = R(i + 1);
      if (n_next > cap)
        raise(FSX_ERR_INVALID_ARGUMENT, "embedding: batch of " + std::to_string(n_next) +
                                            " ids exceeds engine capacity " + std::to_string(cap));
      rn.reserve(cap);
      if (n_next)
        FSX_CUDA(cudaMemcpyAsync(rn.ids.p, ids_next, n_next * 8,
                                 next_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, lo));
    }
    stats_reserve(i + 1);
    const bool with_next = ids_next != nullptr;
    // part 1 (what the backward of i waits for): route + dedup of i+1, the
    // collision of (i, i+1), masks + split plan of i. Part 2 (needed only by
    // the merge of i+1 and the E_co pack): pack lists, E_ex prefetch, IDX.
    auto prep1 = [this, i, bootstrap, with_next, n_next]() {
      ReqBatch& rc2 = R(i);
      OwnBatch& oc2 = O(i);
      // part 2 of the previous prep (on L2) still reads O(i) (its collision
      // flags and scan scratch), which the collision / masks below rewrite
      const cudaEvent_t prev2 = split_lane ? ev_next_ready : nullptr;
      if (with_next) {
        ReqBatch& rn = R(i + 1);
        OwnBatch& on = O(i + 1);
        const int par = route(rn, rn.ids.p, n_next, lo, false);
        receive(on, par, lo, false);
        rn.cor_par = -1;
        wait(lo, prev2);
        collide(oc2, on, lo);
        ev_collided = record(lo);
        if (!bootstrap) masks_and_split(oc2, rc2, true, lo);
      } else {
        wait(lo, prev2);
        oc2.has_co = false;
        if (!bootstrap) masks_and_split(oc2, rc2, false, lo);
      }
      ev_mask = bootstrap ? nullptr : record(lo);
      // (host zeroing of the row: before the backward's stats copy is issued)
      stats_forward(i, with_next);
    };
    const Deferred dfr = take_deferred();
    auto prep2a = [this, dfr, with_next, i]() {
      // the deferred exclusive update of i-1 after the masks: it has a whole
      // iteration of slack and would only slow the chain the backward waits on
      apply_deferred(dfr);
      if (with_next) {
        if (l2() != lo) wait(l2(), ev_collided);
        prefetch_pack(O(i + 1), l2());
      } else {
        ev_pack = nullptr;
      }
    };
    auto prep2 = [this, i, with_next]() {
      if (with_next) {
        ReqBatch& rn = R(i + 1);
        OwnBatch& on = O(i + 1);
        prefetch(on, rn, l2());
        if (self_plan()) plan_self(on, l2());
        ev_next_ready = record(l2());
        rn_ex_ready = ev_next_ready;
      } else {
        ev_next_ready = nullptr;
        rn_ex_ready = nullptr;
      }
    };
    cudaEvent_t ex_ready_cur = cur_ex_ready;  // E_ex(i), recorded by the previous prep
    if (side) {
      ticket_mask = side->post([this, prep1] { HostTimer ht(this, HP_SIDE_JOB); prep1(); });
      ticket_pack = side->post([this, prep2a] { HostTimer ht(this, HP_SIDE_JOB); prep2a(); });
      ticket_next = side->post([this, prep2] { HostTimer ht(this, HP_SIDE_JOB); prep2(); });
    } else {
      prep1();
      prep2a();
      prep2();
    }
    // ---- compute stream C: serve iteration i ----
    if (bootstrap) {
      serve_blocking(rc, oc, out, c);
    } else {
      // exclusive rows first: they only wait for the prefetch, so this half of
      // the merge overlaps the tail of the collision chain
      exposed_wait(c, {ex_ready_cur});
      merge(rc, out, c, 1);
      exposed_wait(c, {cur_co_ready});
      merge(rc, out, c, 2);
    }
    ev_merged = record(c);
    forward_done = true;
    has_next = ids_next != nullptr;
  }
  cudaEvent_t cur_ex_ready = nullptr, cur_co_ready = nullptr, rn_ex_ready = nullptr;
  uint64_t ticket_mask = 0, ticket_pack = 0, ticket_next = 0;  // side-lane jobs of the last forward
  void wait_pack_ready() {
    HostTimer ht(this, HP_WAIT_SIDE);
    if (side) side->wait_for(ticket_pack);
  }
  void wait_next_ready() {
    HostTimer ht(this, HP_WAIT_SIDE);
    if (side) side->wait_for(ticket_next);
  }
  bool has_next = false;

  // deferred exclusive gradients of the previous iteration (embedding.cpp:314-339),
  // on their own lane: they only have to land before the next exclusive
  // prefetch reads rows, so routing / dedup / collision overlap with them
  cudaEvent_t ev_ex_applied = nullptr;
  cudaEvent_t ev_hchain = nullptr;  // end of the last backward's collision chain
  // The deferred state is taken by the caller's thread when the forward posts
  // the side-lane job (the next backward overwrites it while that job waits).
  struct Deferred {
    bool pending = false;
    int iter = -1, par = -1;
    cudaEvent_t split = nullptr, hchain = nullptr;
  };
  Deferred take_deferred() {
    Deferred d{has_pending, pending_iter, exg_par, ev_pending_split, ev_hchain};
    has_pending = false;
    return d;
  }
  void apply_deferred(const Deferred& d) {
    ev_ex_applied = nullptr;
    if (!d.pending) return;
    OwnBatch& op = O(d.iter);
    ReqBatch& rp = R(d.iter);
    wait(ux, d.split);
    // the collision chain of that iteration has the links first: the
    // exclusive gradients have a whole iteration of slack
    if (d.hchain) wait(ux, d.hchain);
    if (p > 1) {
      std::vector<uint64_t> bytes(p);
      {
        HostTimer ht(this, HP_SIZES);
        rp.sizes(p);
      }
      for (int d2 = 0; d2 < p; ++d2) bytes[d2] = kHdr + rb * rp.h_split[2 * d2];
      a2a(CH_EXG, d.par, bytes, ux);
    }
    update(op, CH_EXG, d.par, op.has_co ? op.co.p : nullptr, 0, true, ux, FSX_PHASE_EX_UPDATE);
    ev_ex_applied = record(ux);
  }

  void prio_backward(const void* grads, cudaStream_t c) {
    if (!forward_done) raise(FSX_ERR_PROTOCOL, "embedding: backward before forward");
    if (side) {
      HostTimer ht(this, HP_WAIT_SIDE);
      side->wait_for(ticket_mask);  // masks + split counts of this iteration are issued
    }
    const int i = iter;
    ReqBatch& rc = R(i);
    OwnBatch& oc = O(i);
    cudaEvent_t ev_chain_start = nullptr;
    bool have_grads = false;
    int fused_cor = -1;  // E_co packed by the collision update itself
    if (i == 0) {
      update_blocking(rc, oc, grads, c);  // bootstrap: one synchronized update
      ev_chain_start = record(c);
      has_pending = false;
    } else if (p == 1) {
      // single rank: nothing to hide behind a transfer, so the whole update
      // (collision rows first in row order is immaterial: rows are disjoint)
      // runs at once on the caller's stream, reading the gradients in place.
      // It needs neither the masks nor the split plan (only the statistics
      // do, on H below), so it does not wait for the side lane.
      // FSX_SELF_SERIAL (A/B): 1 = the update waits for the side lane's
      // route / dedup / collision of i+1 (ev_mask), 2 = for its whole prep
      // (ev_next_ready), so the update kernel does not share the SMs with it
      if (self_serial == 1 && ev_mask) wait(c, ev_mask);
      if (self_serial == 2) {
        wait_next_ready();
        if (ev_next_ready) wait(c, ev_next_ready);
      }
      if (self_plan())
        apply_self(oc, grads, c);
      else
        update(oc, CH_GRADS, 0, nullptr, 0, false, c, FSX_PHASE_CO_UPDATE, grads, rc.send_pos.p);
      ev_chain_start = record(c);
      has_pending = false;
      have_grads = true;
    } else {
      exposed_wait(c, {ev_mask});
      const int cog = next_par(CH_COG);
      exg_par = next_par(CH_EXG);
      split_co(rc, grads, cog, c);
      ev_chain_start = record(c);
      split_ex(rc, grads, exg_par, c);
      ev_pending_split = record(c);
      pending_iter = i;
      has_pending = true;
      if (oc.has_co) {
        // collision chain, high priority (embedding.cpp:539-557)
        wait(hi, ev_chain_start);
        if (presum()) {
          if (p > 1 && rc.cog_direct) {
            signal_direct(CH_COG, hi);  // the pre-sum already stored the rows
          } else if (p > 1) {
            std::vector<uint64_t> bytes(p);
            {
              HostTimer ht(this, HP_SIZES);
              rc.sizes(p);
            }
            for (int d = 0; d < p; ++d) bytes[d] = kHdr + rb * rc.h_slots[d];
            a2a(CH_COG, cog, bytes, hi);
          }
          Span sp(this, FSX_PHASE_CO_UPDATE, hi);
          if (has_next && p > 1) {
            wait_pack_ready();
            wait(hi, ev_pack);
            fused_cor = next_par(CH_COR);
            co_apply(oc, cog, hi, &O(i + 1), fused_cor);
          } else {
            co_apply(oc, cog, hi);
          }
        } else {
          if (p > 1) {
            std::vector<uint64_t> bytes(p);
            {
              HostTimer ht(this, HP_SIZES);
              rc.sizes(p);
            }
            for (int d = 0; d < p; ++d) bytes[d] = kHdr + rb * rc.h_split[2 * d + 1];
            a2a(CH_COG, cog, bytes, hi);
          }
          update(oc, CH_COG, cog, oc.co.p, 1, true, hi, FSX_PHASE_CO_UPDATE);
        }
        have_grads = true;
      }
    }
    wait_pack_ready();
    if (has_next) {
      // E_co^{i+1}: fresh collision rows to the next iteration's requesters
      OwnBatch& on = O(i + 1);
      ReqBatch& rn = R(i + 1);
      wait(hi, ev_chain_start);
      if (ev_pack) wait(hi, ev_pack);
      if (fused_cor >= 0) {
        Span sp(this, FSX_PHASE_ECO, hi);
        if (eco_direct) {
          signal_direct(CH_COR, hi);
        } else {
          std::vector<uint64_t> bytes(p);
          for (int d = 0; d < p; ++d) bytes[d] = idrows_rows_off(on.h_pack[2 * d + 1]) + rb * on.h_pack[2 * d + 1];
          a2a(CH_COR, fused_cor, bytes, hi);
        }
        rn.cor_par = fused_cor;
      } else {
        rn.cor_par = send_eco(on, hi);
      }
      cur_co_ready = record(hi);
      if (p == 1) wait(hi, ev_mask);  // split counts for the statistics
      stats_backward(i, have_grads, true, rc, oc, on, rn.cor_par, hi);
    } else {
      cur_co_ready = nullptr;
      if (p == 1 && i > 0) wait(hi, ev_mask);
      stats_backward(i, have_grads, false, rc, oc, oc, -1, i == 0 ? c : hi);
    }
    ev_hchain = have_grads || has_next ? record(hi) : nullptr;
    forward_done = false;
    ++iter;
  }

  // every lane's issued work (side-lane jobs included) ordered before the
  // caller's stream `c`: no protocol effect, for timing regions that must end
  // only when the engine is idle
  void join(cudaStream_t c) {
    if (side) side->drain();
    for (cudaStream_t s : {lo, hi, ux, us, lo2})
      if (s) wait(c, record(s));
    for (int l = 0; l < kLanes; ++l)
      for (int d = 0; d < p; ++d)
        if (cstream[l][d]) wait(c, record(cstream[l][d]));
  }

  void finalize(cudaStream_t c) {
    if (side) side->drain();
    apply_deferred(take_deferred());
    wait(c, record(lo));
    if (lo2) wait(c, record(lo2));
    wait(c, record(hi));
    wait(c, record(ux));
  }

  // ---- stats (IterationStats, embedding.hpp:119-124) ----------------------------
  void stats_reserve(int n) {
    while (static_cast<int>(h_stats.size()) * kStatsChunk < n) {
      uint64_t* h = nullptr;
      FSX_CUDA(cudaHostAlloc(&h, kStatsChunk * 3 * 8, cudaHostAllocDefault));
      std::memset(h, 0, kStatsChunk * 3 * 8);
      h_stats.push_back(h);
    }
  }
  void stats_forward(int i, bool with_next) {
    stats_reserve(i + 1);
    stats_n = i + 1;
    uint64_t* dst = stat_row(i);
    dst[0] = dst[1] = dst[2] = 0;
    if (with_next) {
      FSX_CUDA(cudaMemcpyAsync(dst, O(i).misc.p, 8, cudaMemcpyDeviceToHost, lo));
      FSX_CUDA(cudaMemcpyAsync(dst + 1, O(i + 1).srt.d_u(), 8, cudaMemcpyDeviceToHost, lo));
    }
  }
  void stats_backward(int i, bool have_grads, bool have_eco, ReqBatch& rc, OwnBatch& oc,
                      OwnBatch& on, int cor_par, cudaStream_t s) {
    if (!have_grads && !have_eco) return;
    uint64_t* d = d_stats.p + 4 * (i % 3);
    CSlots cor{};
    if (cor_par >= 0) cor = recv_slots(CH_COR, cor_par);
    FSX_LAUNCH(ctx, k_blocking_bytes, 1, 32, 0, s, p, 8ull * t->g.dim, rc.split_tot.p, oc.occ_tot(),
               on.pack_tot(), cor, oc.misc.p, have_grads ? 1 : 0, have_eco ? 1 : 0, d);
    FSX_CUDA(cudaMemcpyAsync(stat_row(i) + 2, d, 8, cudaMemcpyDeviceToHost, s));
  }

  ~Engine() {
    if (host_prof) {
      static const char* names[HP_N] = {"forward", "backward", "wait_side", "side_jobs", "sizes_sync", "fetch_sync",
                                        "a2a_issue"};
      std::fprintf(stderr, "[fsx host r%d]", me);
      for (int k = 0; k < HP_N; ++k)
        std::fprintf(stderr, " %s %.3f ms/%llu", names[k], 1e-6 * static_cast<double>(hp_ns[k].load()),
                     static_cast<unsigned long long>(hp_calls[k].load()));
      std::fprintf(stderr, "\n");
    }
    side.reset();
    cudaDeviceSynchronize();
    for (int d = 0; d < kMaxRanks; ++d)
      if (peer[d].ipc && peer[d].base) cudaIpcCloseMemHandle(peer[d].base);
    if (nccl) NcclApi::get().CommDestroy(nccl);
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto e : timing_pool) cudaEventDestroy(e);
    for (auto e : prof_pool) cudaEventDestroy(e);
    if (lo) cudaStreamDestroy(lo);
    if (lo2) cudaStreamDestroy(lo2);
    if (hi) cudaStreamDestroy(hi);
    if (ux) cudaStreamDestroy(ux);
    if (us) cudaStreamDestroy(us);
    for (auto& lane : cstream)
      for (auto cs : lane)
        if (cs) cudaStreamDestroy(cs);
    if (win) cudaFree(win);
    for (auto* h : h_stats) cudaFreeHost(h);
  }
};

}  // namespace fsx

using namespace fsx;

struct fsx_engine : Engine {};

namespace {
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

struct ExportBlob {
  uint64_t magic;
  int32_t p, me, mode, pad;
  uint64_t win_bytes, flags_off;
  uint64_t ch_off[NCH], ch_slot[NCH];
  cudaIpcMemHandle_t handle;
};
constexpr uint64_t kBlobMagic = 0x46535857494e3031ull;  // "FSXWIN01"
}  // namespace

extern "C" {

int fsx_engine_create(fsx_ctx* ctx, fsx_table* table, const fsx_engine_config* cfg, fsx_engine** out) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  if (!cfg || (cfg->mode != FSX_MODE_SYNC && cfg->mode != FSX_MODE_PRIO))
    raise(FSX_ERR_INVALID_ARGUMENT, "fsx: bad engine mode");
  if (cfg->transport != FSX_TRANSPORT_CE && cfg->transport != FSX_TRANSPORT_NCCL)
    raise(FSX_ERR_CONFIG, "fsx: unknown transport");
  if (cfg->transport == FSX_TRANSPORT_NCCL && cfg->mode != FSX_MODE_SYNC)
    raise(FSX_ERR_CONFIG, "fsx: the NCCL transport is the blocking baseline (synchronized mode only)");
  if (table->g.p != ctx->world || table->g.shard != ctx->rank)
    raise(FSX_ERR_INVALID_ARGUMENT, "fsx: table shard does not match the context rank/world");
  if (ctx->world > kMaxRanks) raise(FSX_ERR_INVALID_ARGUMENT, "fsx: at most 16 ranks");
  auto e = std::make_unique<fsx_engine>();
  e->ctx = ctx;
  e->t = table;
  e->cfg = *cfg;
  e->p = ctx->world;
  e->me = ctx->rank;
  e->cap = std::max<uint64_t>(cfg->max_occurrences, 1);
  e->rb = table->row_bytes();
  if (const char* v = std::getenv("FSX_ECO_DIRECT")) e->eco_direct = std::atoi(v) != 0;
  if (const char* v = std::getenv("FSX_COG_DIRECT")) e->cog_direct = std::atoi(v) != 0;
  const bool prio = cfg->mode == FSX_MODE_PRIO;
  const uint64_t cap = e->cap, rb = e->rb;
  auto round256 = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  uint64_t slot[NCH] = {};
  slot[CH_IDS] = kHdr + cap * 8;
  slot[CH_ROWS] = kHdr + cap * rb;
  slot[CH_GRADS] = kHdr + cap * rb;
  slot[CH_AG] = kHdr + std::max<uint64_t>(cap * 8, 1u << 16);  // fsx_allgather_ce chunks
  if (prio) {
    slot[CH_EX] = idrows_rows_off(cap) + cap * rb;
    slot[CH_MASK] = kHdr + align16(cap);
    slot[CH_IDX] = kHdr + align16(4 * cap);
    if (cfg->flags & FSX_ENGINE_PRESUM) slot[CH_GRP] = grp_list_off(cap) + 4 * cap;
    slot[CH_COG] = kHdr + cap * rb;
    slot[CH_EXG] = kHdr + cap * rb;
    slot[CH_COR] = idrows_rows_off(cap) + cap * rb;
  }
  size_t off = 0;
  for (int ch = 0; ch < NCH; ++ch) {
    e->ch_slot[ch] = round256(slot[ch]);
    e->ch_off[ch] = off;
    off += 2 * static_cast<size_t>(e->p) * e->ch_slot[ch];
  }
  e->flags_off = off;
  e->win_bytes = off + round256(NCH * kMaxRanks * sizeof(uint32_t));
  FSX_CUDA(cudaMalloc(&e->win, e->win_bytes));
  e->flags = reinterpret_cast<uint32_t*>(e->win + e->flags_off);
  FSX_CUDA(cudaMemset(e->flags, 0, NCH * kMaxRanks * sizeof(uint32_t)));
  if (e->p > 1) e->stage.alloc(off);
  // Priorities (lower number = higher): the collision chain highest, the
  // next-iteration prep above the caller's compute (it gates the next merge),
  // the deferred exclusive update lowest (it has an iteration of slack).
  int least = 0, greatest = 0;
  FSX_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  const int mid = greatest < least ? greatest + 1 : greatest;
  FSX_CUDA(cudaStreamCreateWithPriority(&e->lo, cudaStreamNonBlocking, mid));
  // (one rank: no transfers in part 2, measured neutral — kept on L)
  e->split_lane = e->p > 1;
  if (const char* v = std::getenv("FSX_SPLIT_LANE")) e->split_lane = std::atoi(v) != 0;
  if (prio && e->split_lane) FSX_CUDA(cudaStreamCreateWithPriority(&e->lo2, cudaStreamNonBlocking, mid));
  FSX_CUDA(cudaStreamCreateWithPriority(&e->hi, cudaStreamNonBlocking, greatest));
  FSX_CUDA(cudaStreamCreateWithPriority(&e->ux, cudaStreamNonBlocking, least));
  FSX_CUDA(cudaStreamCreateWithPriority(&e->us, cudaStreamNonBlocking, greatest));
  if (const char* v = std::getenv("FSX_C_PRIO")) e->c_prio = std::atoi(v);
  if (const char* v = std::getenv("FSX_SELF_SERIAL")) e->self_serial = std::atoi(v);
  // one copy stream per peer: outgoing copies of an all-to-all run on
  // several copy engines at once instead of queueing on one
  for (int l = 0; l < Engine::kLanes; ++l) e->lane_map[l] = prio ? (l == 3 ? 1 : l) : 3;
  if (!e->lo2) e->lane_map[4] = e->lane_map[0];
  for (int l = 0; l < Engine::kLanes; ++l) {
    if (prio ? l == 3 : l != 3) continue;
    for (int d = 0; d < e->p; ++d)
      if (d != e->me) FSX_CUDA(cudaStreamCreateWithPriority(&e->cstream[l][d], cudaStreamNonBlocking, greatest));
  }
  if (e->p > 1) {
    e->side = std::make_unique<SideLane>();
    e->side->start(ctx->device);
  }
  e->d_stats.alloc(16);
  const uint64_t m = static_cast<uint64_t>(e->p) * cap;
  for (int k = 0; k < 3; ++k) {
    FSX_CUDA(cudaHostAlloc(&e->rq[k].hp_sizes, 48 * 8, cudaHostAllocDefault));
    FSX_CUDA(cudaEventCreateWithFlags(&e->rq[k].ev_sizes, cudaEventDisableTiming));
    e->rq[k].reserve(cap);
    if (prio && (cfg->flags & FSX_ENGINE_PRESUM)) e->rq[k].plan.reserve(cap, cap, table->g.dim, cfg->reduce_chunk);
    e->rq[k].scan.ensure(cap, 16);
    e->ow[k].reserve(m);
    e->ow[k].scan.ensure(m, 16);
  }
  for (auto& s : e->sgd) s.reserve(m, m, table->g.dim, cfg->reduce_chunk);
  if (prio && e->self_plan())
    for (int k = 0; k < 3; ++k) e->ow[k].plan.reserve(m, m, table->g.dim, cfg->reduce_chunk);
  e->stats_reserve(4 * Engine::kStatsChunk);
  FSX_CUDA(cudaDeviceSynchronize());
  *out = e.release();
  FSX_API_END
}

int fsx_engine_destroy(fsx_engine* e) {
  FSX_API_BEGIN
  if (!e) return FSX_OK;
  DeviceGuard dg(e->ctx->device);
  delete e;
  FSX_API_END
}

int fsx_engine_connect_local(fsx_engine* e, int peer, fsx_engine* other) {
  FSX_API_BEGIN
  if (peer < 0 || peer >= e->p || other->p != e->p || other->me != peer || other->win_bytes != e->win_bytes)
    raise(FSX_ERR_COLLECTIVE, "fsx: peer engine layout mismatch");
  DeviceGuard dg(e->ctx->device);
  if (other->ctx->device != e->ctx->device) {
    cudaError_t rc = cudaDeviceEnablePeerAccess(other->ctx->device, 0);
    if (rc != cudaSuccess && rc != cudaErrorPeerAccessAlreadyEnabled) FSX_CUDA(rc);
    cudaGetLastError();
  }
  e->peer[peer].base = other->win;
  e->peer[peer].flags = other->flags;
  e->peer[peer].ipc = false;
  e->peer[peer].local = other;
  FSX_API_END
}

int fsx_engine_export(fsx_engine* e, void* blob, uint64_t* len) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  ExportBlob b{};
  b.magic = kBlobMagic;
  b.p = e->p;
  b.me = e->me;
  b.mode = e->cfg.mode;
  b.win_bytes = e->win_bytes;
  b.flags_off = e->flags_off;
  for (int ch = 0; ch < NCH; ++ch) {
    b.ch_off[ch] = e->ch_off[ch];
    b.ch_slot[ch] = e->ch_slot[ch];
  }
  FSX_CUDA(cudaIpcGetMemHandle(&b.handle, e->win));
  std::memcpy(blob, &b, sizeof b);
  *len = sizeof b;
  FSX_API_END
}

int fsx_engine_connect_ipc(fsx_engine* e, int peer, const void* blob, uint64_t len) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  ExportBlob b{};
  if (len != sizeof b) raise(FSX_ERR_COLLECTIVE, "fsx: bad peer blob");
  std::memcpy(&b, blob, sizeof b);
  if (b.magic != kBlobMagic || b.p != e->p || b.me != peer || b.win_bytes != e->win_bytes ||
      b.flags_off != e->flags_off)
    raise(FSX_ERR_COLLECTIVE, "fsx: peer " + std::to_string(peer) + " window layout mismatch");
  void* base = nullptr;
  FSX_CUDA(cudaIpcOpenMemHandle(&base, b.handle, cudaIpcMemLazyEnablePeerAccess));
  e->peer[peer].base = static_cast<char*>(base);
  e->peer[peer].flags = reinterpret_cast<uint32_t*>(static_cast<char*>(base) + b.flags_off);
  e->peer[peer].ipc = true;
  FSX_API_END
}

int fsx_nccl_unique_id(void* id128) {
  FSX_API_BEGIN
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  nccl_check(NcclApi::get().GetUniqueId(&id), "get unique id");
  std::memcpy(id128, &id, 128);
  FSX_API_END
}

int fsx_engine_connect_nccl(fsx_engine* e, const void* id128) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  if (e->cfg.transport != FSX_TRANSPORT_NCCL)
    raise(FSX_ERR_CONFIG, "fsx: engine was not created for the NCCL transport");
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  nccl_check(NcclApi::get().CommInitRank(&e->nccl, e->p, id, e->me), "comm init");
  FSX_API_END
}

int fsx_engine_forward(fsx_engine* e, const uint64_t* d_ids_cur, uint64_t n_cur,
                       const uint64_t* d_ids_next, uint64_t n_next, void* d_out, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  e->cur_c = S(stream);
  Engine::HostTimer ht(e, HP_FWD);
  if (e->cfg.mode == FSX_MODE_SYNC)
    e->sync_forward(d_ids_cur, n_cur, d_out, S(stream));
  else
    e->prio_forward(d_ids_cur, n_cur, d_ids_next, n_next, d_out, S(stream));
  FSX_API_END
}

int fsx_engine_backward(fsx_engine* e, const void* d_grads, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  e->cur_c = S(stream);
  Engine::HostTimer ht(e, HP_BWD);
  if (e->cfg.mode == FSX_MODE_SYNC)
    e->sync_backward(d_grads, S(stream));
  else
    e->prio_backward(d_grads, S(stream));
  FSX_API_END
}

int fsx_engine_finalize(fsx_engine* e, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  if (e->cfg.mode == FSX_MODE_PRIO) e->finalize(S(stream));
  FSX_API_END
}

int fsx_engine_stats(fsx_engine* e, int iter, uint64_t* out3) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  if (e->side) e->side->drain();
  if (iter < 0 || iter >= e->stats_n) raise(FSX_ERR_OUT_OF_RANGE, "fsx: no stats for iteration " + std::to_string(iter));
  FSX_CUDA(cudaDeviceSynchronize());
  std::memcpy(out3, e->stat_row(iter), 24);
  FSX_API_END
}

int fsx_engine_exposed_ms(fsx_engine* e, double* ms) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  if (e->side) e->side->drain();
  double total = 0;
  for (auto& w : e->waits) {
    FSX_CUDA(cudaEventSynchronize(w.second));
    float x = 0;
    FSX_CUDA(cudaEventElapsedTime(&x, w.first, w.second));
    total += x;
  }
  *ms = total;
  e->waits.clear();
  e->timing_next = 0;
  FSX_API_END
}

// Timeline dump of every recorded span: (phase, start ms, end ms) relative
// to the earliest span start; consumes the spans like fsx_engine_phase_ms.
int fsx_engine_spans(fsx_engine* e, double* out, uint64_t max_spans, uint64_t* n_out) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  if (e->side) e->side->drain();
  FSX_CUDA(cudaDeviceSynchronize());
  cudaEvent_t base = nullptr;
  float best = 0;
  for (auto& v : e->spans)
    for (auto& sp : v) {
      if (!base) { base = sp.first; continue; }
      float x = 0;
      FSX_CUDA(cudaEventElapsedTime(&x, base, sp.first));
      if (x < best) best = x;
    }
  uint64_t k = 0;
  for (int ph = 0; ph < FSX_NUM_PHASES; ++ph) {
    for (auto& sp : e->spans[ph]) {
      if (k >= max_spans) break;
      float a = 0, b = 0;
      FSX_CUDA(cudaEventElapsedTime(&a, base, sp.first));
      FSX_CUDA(cudaEventElapsedTime(&b, base, sp.second));
      out[3 * k] = ph;
      out[3 * k + 1] = a - best;
      out[3 * k + 2] = b - best;
      ++k;
    }
    e->spans[ph].clear();
  }
  e->prof_next = 0;
  *n_out = k;
  FSX_API_END
}

// Timeline trace: per span (phase, lane, channel, GPU start ms, GPU end ms,
// host issue ms), GPU times relative to the earliest span start and host
// issue times in CLOCK_MONOTONIC ms; consumes the spans like fsx_engine_spans.
int fsx_engine_trace(fsx_engine* e, double* out, uint64_t max_spans, uint64_t* n_out) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  if (e->side) e->side->drain();
  FSX_CUDA(cudaDeviceSynchronize());
  cudaEvent_t base = nullptr;
  float best = 0;
  for (auto& v : e->spans)
    for (auto& sp : v) {
      if (!base) { base = sp.first; continue; }
      float x = 0;
      FSX_CUDA(cudaEventElapsedTime(&x, base, sp.first));
      if (x < best) best = x;
    }
  uint64_t k = 0;
  for (int ph = 0; ph < FSX_NUM_PHASES; ++ph) {
    for (auto& sp : e->spans[ph]) {
      if (k >= max_spans) break;
      float a = 0, b = 0;
      FSX_CUDA(cudaEventElapsedTime(&a, base, sp.first));
      FSX_CUDA(cudaEventElapsedTime(&b, base, sp.second));
      double* o = out + 6 * k;
      o[0] = ph;
      o[1] = sp.lane;
      o[2] = sp.ch;
      o[3] = a - best;
      o[4] = b - best;
      o[5] = sp.host_ns * 1e-6;  // CLOCK_MONOTONIC ms
      ++k;
    }
    e->spans[ph].clear();
  }
  e->prof_next = 0;
  *n_out = k;
  FSX_API_END
}

int fsx_engine_join(fsx_engine* e, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  e->join(S(stream));
  FSX_API_END
}

int fsx_engine_set_ids_ready(fsx_engine* e, int ready) {
  FSX_API_BEGIN
  e->ids_ready = ready != 0;
  FSX_API_END
}

int fsx_engine_set_eco_direct(fsx_engine* e, int on) {
  FSX_API_BEGIN
  if (e->forward_done) raise(FSX_ERR_PROTOCOL, "fsx: E_co mode changes between iterations only");
  e->eco_direct = (on & 1) != 0;
  e->cog_direct = (on & 2) != 0;
  FSX_API_END
}

int fsx_engine_set_profiling(fsx_engine* e, int on) {
  FSX_API_BEGIN
  e->prof = on != 0;
  FSX_API_END
}

int fsx_engine_phase_ms(fsx_engine* e, int phase, double* total_ms, uint64_t* count) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  if (e->side) e->side->drain();
  if (phase < 0 || phase >= FSX_NUM_PHASES) raise(FSX_ERR_OUT_OF_RANGE, "fsx: bad phase");
  double t = 0;
  uint64_t c = 0;
  for (auto& sp : e->spans[phase]) {
    if (sp.ch >= 1000) continue;  // per-copy trace spans
    FSX_CUDA(cudaEventSynchronize(sp.second));
    float x = 0;
    FSX_CUDA(cudaEventElapsedTime(&x, sp.first, sp.second));
    t += x;
    ++c;
  }
  *total_ms = t;
  *count = c;
  e->spans[phase].clear();
  bool any = false;
  for (auto& v : e->spans) any = any || !v.empty();
  if (!any) e->prof_next = 0;  // recycle the event pool once every phase was read
  FSX_API_END
}

uint64_t fsx_engine_slot_bytes(const fsx_engine* e) { return e ? e->ch_slot[CH_GRADS] - kHdr : 0; }

// Byte all-to-all over the engine's GRADS channel (comm.cpp:308-365 shape:
// size round, then payloads); collective, between iterations only.
int fsx_allgather_ce(fsx_engine* e, const void* d_send, uint64_t send_bytes, uint64_t max_bytes, void* d_recv,
                     uint64_t slot_bytes, uint64_t* h_recv_bytes, int ring, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t cap = e->ch_slot[CH_AG] - kHdr;
  if (max_bytes < send_bytes) max_bytes = send_bytes;
  if (max_bytes > cap || max_bytes > slot_bytes)
    raise(FSX_ERR_COLLECTIVE, "all_gather: payload of " + std::to_string(max_bytes) +
                                  " bytes exceeds the slot capacity");
  if (e->side) e->side->drain();
  const int p = e->p, me = e->me;
  const int par = static_cast<int>(++e->ag_calls & 1u);
  char* mine = e->recv_slot(CH_AG, par, me);
  const uint64_t hdr[2] = {send_bytes, 0};
  FSX_CUDA(cudaMemcpyAsync(mine, hdr, kHdr, cudaMemcpyHostToDevice, s));
  if (send_bytes) FSX_CUDA(cudaMemcpyAsync(mine + kHdr, d_send, send_bytes, cudaMemcpyDeviceToDevice, s));
  FSX_CUDA(cudaStreamSynchronize(s));  // the host header above is stack memory
  e->all_gather_ce(par, max_bytes, ring != 0, s);
  std::vector<uint64_t> h(2 * p);
  for (int d = 0; d < p; ++d)
    FSX_CUDA(cudaMemcpyAsync(&h[2 * d], e->recv_slot(CH_AG, par, d), kHdr, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  for (int d = 0; d < p; ++d) {
    if (h[2 * d] > max_bytes)
      raise(FSX_ERR_COLLECTIVE, "all_gather: rank " + std::to_string(d) + " sent " + std::to_string(h[2 * d]) +
                                    " bytes, above the agreed bound " + std::to_string(max_bytes));
    h_recv_bytes[d] = h[2 * d];
    if (h[2 * d])
      FSX_CUDA(cudaMemcpyAsync(static_cast<char*>(d_recv) + d * slot_bytes, e->recv_slot(CH_AG, par, d) + kHdr,
                               h[2 * d], cudaMemcpyDeviceToDevice, s));
  }
  FSX_CUDA(cudaStreamSynchronize(s));
  FSX_API_END
}

int fsx_a2a_ce(fsx_engine* e, const void* d_send, const uint64_t* h_send_offsets,
               const uint64_t* h_send_bytes, void* d_recv, uint64_t slot_bytes, uint64_t* h_recv_bytes,
               void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t cap = e->ch_slot[CH_GRADS] - kHdr;
  const int p = e->p;
  for (int d = 0; d < p; ++d)
    if (h_send_bytes[d] > cap || h_send_bytes[d] > slot_bytes)
      raise(FSX_ERR_COLLECTIVE, "all_to_all: payload of " + std::to_string(h_send_bytes[d]) +
                                    " bytes exceeds the slot capacity");
  const int par = e->next_par(CH_GRADS);
  std::vector<uint64_t> bytes(p);
  for (int d = 0; d < p; ++d) {
    char* slot = e->stage_slot(CH_GRADS, par, d);
    const uint64_t hdr[2] = {h_send_bytes[d], 0};
    FSX_CUDA(cudaMemcpyAsync(slot, hdr, kHdr, cudaMemcpyHostToDevice, s));
    if (h_send_bytes[d])
      FSX_CUDA(cudaMemcpyAsync(slot + kHdr, static_cast<const char*>(d_send) + h_send_offsets[d],
                               h_send_bytes[d], cudaMemcpyDeviceToDevice, s));
    bytes[d] = kHdr + h_send_bytes[d];
  }
  FSX_CUDA(cudaStreamSynchronize(s));  // host headers above are stack memory
  e->a2a(CH_GRADS, par, bytes, s);
  std::vector<uint64_t> hdr(2 * p);
  for (int d = 0; d < p; ++d)
    FSX_CUDA(cudaMemcpyAsync(&hdr[2 * d], e->recv_slot(CH_GRADS, par, d), kHdr, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  for (int d = 0; d < p; ++d) {
    h_recv_bytes[d] = hdr[2 * d];
    if (hdr[2 * d])
      FSX_CUDA(cudaMemcpyAsync(static_cast<char*>(d_recv) + d * slot_bytes, e->recv_slot(CH_GRADS, par, d) + kHdr,
                               hdr[2 * d], cudaMemcpyDeviceToDevice, s));
  }
  FSX_CUDA(cudaStreamSynchronize(s));
  FSX_API_END
}

// The engine's copy-engine all-to-all alone (measurement, e.g. against NCCL's
// copy-engine collectives): bytes_per_peer from each staging slot of the
// GRADS channel to every peer, as the protocol's own exchanges move them
// (kernels have written the staging slots; here they hold whatever they
// hold). Enqueue only — no host synchronisation; collective.
int fsx_engine_a2a_staged(fsx_engine* e, uint64_t bytes_per_peer, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(e->ctx->device);
  if (bytes_per_peer + kHdr > e->ch_slot[CH_GRADS])
    raise(FSX_ERR_COLLECTIVE, "all_to_all: payload of " + std::to_string(bytes_per_peer) +
                                  " bytes exceeds the slot capacity");
  const int par = e->next_par(CH_GRADS);
  std::vector<uint64_t> bytes(e->p, kHdr + bytes_per_peer);
  e->a2a(CH_GRADS, par, bytes, static_cast<cudaStream_t>(stream));
  FSX_API_END
}

}  // extern "C"
