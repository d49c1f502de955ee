/* fsx.h — C ABI of the B200-native FreeScale embedding hot path (libfsx.so).
 *
 * Plain pointers and sizes only: no torch, no C++ types. Device pointers are
 * CUDA device addresses on the context's device; host pointers are ordinary
 * (preferably pinned) host memory. Streams are cudaStream_t passed as void*.
 * Every entry point returns an int status (FSX_OK or a negative class code);
 * fsx_last_error() returns the message of the calling thread's last failure.
 * The status classes map 1:1 onto the reference's exception classes so the
 * C++ and Python shims rethrow the same class with the same text
 * (SURVEY §8(b) "Errors").
 *
 * Reference interfaces replaced (paths under /root/reference/proj):
 *   table   — embedding::ShardView                 include/freescale/embedding.hpp:59-90
 *   sort    — sorted_unique / IndexSet::shard_major src/embedding.cpp:12-16, 66-80
 *   collide — compute_collision / collision_pct    include/freescale/embedding.hpp:51-57
 *   route   — route_to_shard_major                 include/freescale/embedding.hpp:107-110
 *   engine  — SynchronizedEmbedding / PrioritizedEmbedding
 *                                                  include/freescale/embedding.hpp:126-189
 *   a2a     — comm::Communicator::all_to_all       include/freescale/comm.hpp:126-128
 *   partition — fbs_partition / vbs_partition / autotune_update / identity
 *                                                  include/freescale/partition.hpp:50-74
 *   cost    — sim::CostModel::compute_time_for_lengths  include/freescale/sim.hpp:24-35
 */
#ifndef FSX_H
#define FSX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (reference exception class in brackets) --------------- */
#define FSX_OK 0
#define FSX_ERR_INVALID_ARGUMENT (-1) /* std::invalid_argument           */
#define FSX_ERR_DOMAIN (-2)           /* std::domain_error               */
#define FSX_ERR_OUT_OF_RANGE (-3)     /* std::out_of_range               */
#define FSX_ERR_PROTOCOL (-4)         /* freescale::ProtocolError        */
#define FSX_ERR_COLLECTIVE (-5)       /* freescale::CollectiveError      */
#define FSX_ERR_CONFIG (-6)           /* freescale::ConfigError          */
#define FSX_ERR_CUDA (-7)             /* CUDA runtime/driver failure     */
#define FSX_ERR_NOMEM (-8)            /* device allocation failed        */
#define FSX_ERR_IO (-9)               /* freescale::IoError              */

/* element type of table values, rows and gradients */
#define FSX_F32 0
#define FSX_F64 1

/* engine protocol (embedding.hpp:126-189) */
#define FSX_MODE_SYNC 0 /* SynchronizedEmbedding: blocking, per-occurrence traffic */
#define FSX_MODE_PRIO 1 /* PrioritizedEmbedding: collision-first, side lanes      */

/* engine transport for N > 1 ranks */
#define FSX_TRANSPORT_CE 0   /* copy-engine peer copies + stream mem-op flags, 0 SMs */
#define FSX_TRANSPORT_NCCL 1 /* NCCL send/recv kernels (baseline only)               */

const char* fsx_last_error(void);
/* library build string: arch, git-less version, compile flags */
const char* fsx_version(void);

/* ---- context: one per rank (= one per GPU in production) ------------------ */
typedef struct fsx_ctx fsx_ctx;

int fsx_ctx_create(int device, int rank, int world, fsx_ctx** out);
int fsx_ctx_destroy(fsx_ctx* ctx);
/* Synchronize the context's device and surface any kernel-raised error
 * (out-of-range / not-owned row ids, non-finite updates, protocol breaks)
 * with the reference's exception class and message. */
int fsx_ctx_sync(fsx_ctx* ctx);
/* number of kernels this context has launched (for bench gpu_launches) */
uint64_t fsx_ctx_launches(const fsx_ctx* ctx);
/* The row-update kernel's own span (first CTA start -> last CTA end, device
 * globaltimer) per launch, recorded without host synchronisation while on:
 * returns the mean (us) and count of the launches since the last call, then
 * switches recording on / off (measurement only; synchronizes when reading). */
int fsx_ctx_kernel_span(fsx_ctx* ctx, int on, double* mean_us, uint64_t* n);

/* ---- primitives (hot-path kernels, exposed for parity tests) -------------- */

/* K1+K2: sorted unique of n u64 keys. Writes the unique keys ascending to
 * d_unique (capacity n), optionally each input's slot in d_unique to
 * d_inverse (u32, capacity n), and the unique count to *h_num_unique.
 * Synchronous on `stream`. Replaces sorted_unique (embedding.cpp:12-16). */
int fsx_sort_unique_u64(fsx_ctx* ctx, const uint64_t* d_keys, uint64_t n, uint64_t* d_unique,
                        uint32_t* d_inverse, uint64_t* h_num_unique, void* stream);

/* K3: compute_collision (embedding.cpp:82-93) on two raw shard-major id
 * lists: both are sorted+uniqued on the device, then split into
 * co = U(cur) ∩ U(next), ex_cur = U(cur) \ co, ex_next = U(next) \ co, all
 * ascending. Capacities: d_co, d_ex_cur >= n_cur; d_ex_next >= n_next.
 * h_counts[0..4] = |co|, |ex_cur|, |ex_next|, |U(cur)|, |U(next)|. */
int fsx_collision_split(fsx_ctx* ctx, const uint64_t* d_cur, uint64_t n_cur,
                        const uint64_t* d_next, uint64_t n_next, uint64_t* d_co,
                        uint64_t* d_ex_cur, uint64_t* d_ex_next, uint64_t* h_counts,
                        void* stream);

/* K4: the requester half of route_to_shard_major (embedding.cpp:194-204):
 * stable partition of n ids by owner = id mod num_shards. Writes the ids
 * grouped by owner in original order to d_send_ids, their flat positions to
 * d_send_pos, per-owner counts to h_send_counts[num_shards]. Raises
 * FSX_ERR_DOMAIN ("embedding: row id X out of range ...") for ids >= total_rows. */
int fsx_route_by_owner(fsx_ctx* ctx, const uint64_t* d_ids, uint64_t n, uint64_t total_rows,
                       int num_shards, uint64_t* d_send_ids, uint32_t* d_send_pos,
                       uint64_t* h_send_counts, void* stream);

/* ---- table: one shard of a row-wise sharded table (ShardView) -------------- */
typedef struct fsx_table fsx_table;

/* ShardView ctor (embedding.cpp:108-119): allocates local_rows x dim values
 * on the device and fills them with initial_value(seed, global_row, d)
 * (splitmix64, exact in f64; FSX_F32 rounds that value once). */
int fsx_table_create(fsx_ctx* ctx, uint64_t total_rows, uint32_t dim, int num_shards, int shard,
                     double learning_rate, uint64_t seed, int dtype, fsx_table** out);
int fsx_table_destroy(fsx_table* t);
uint64_t fsx_table_local_rows(const fsx_table* t);
/* device address of the local_rows x dim value array (row-major) */
void* fsx_table_values(fsx_table* t);

/* K5: ShardView::lookup (embedding.cpp:139-146): d_out[k] = row(ids[k]).
 * Out-of-range / not-owned ids raise FSX_ERR_DOMAIN at the next sync point
 * (this call synchronizes when `sync` != 0). */
int fsx_table_gather(fsx_table* t, const uint64_t* d_ids, uint64_t n, void* d_out, void* stream,
                     int sync);

/* K8: ShardView::apply_gradients (embedding.cpp:148-181): each row's
 * gradients summed in occurrence order, then row -= lr*acc, non-finite check.
 * Optional outputs: sorted unique ids (d_unique, capacity n) and their
 * post-update rows (d_rows, capacity n*dim); *h_num_unique if non-null.
 * Synchronous. */
int fsx_table_sgd_update(fsx_table* t, const uint64_t* d_ids, uint64_t n, const void* d_grads,
                         uint64_t* d_unique, void* d_rows, uint64_t* h_num_unique, void* stream);

/* values() as f64 host array [local_rows x dim] (lazy D2H mirror). */
int fsx_table_download(fsx_table* t, double* h_values);
/* overwrite the shard from a host f64 array (test / checkpoint-restore aid) */
int fsx_table_upload(fsx_table* t, const double* h_values);

/* ---- pooled (bag) lookup + scatter: BASELINE config 3 ------- */
/* No reference operator (the reference's toy model mean-pools whole samples,
 * pipeline.cpp:59-67); restated in oracle/fsx_oracle.c fso_pooled_*.
 * forward: d_out[b] (n_bags x dim, the table's type) = sum of row(ids[k]) over
 * k in [offs[b], offs[b+1]) in token order (f64, one rounding); it also plans
 * the backward (tokens sorted by row). Bad ids raise FSX_ERR_DOMAIN at the next
 * sync (fsx_ctx_sync). backward: token k of bag b takes gradient row
 * d_bag_grads[b]; rows are updated as fsx_table_sgd_update with the chunk
 * association `reduce_chunk` (0: one left fold per row). Asynchronous on
 * `stream`; one forward per backward. */
typedef struct fsx_pooled fsx_pooled;
int fsx_pooled_create(fsx_table* t, uint64_t max_occurrences, uint64_t max_bags, uint32_t reduce_chunk,
                      fsx_pooled** out);
int fsx_pooled_destroy(fsx_pooled* p);
int fsx_pooled_forward(fsx_pooled* p, const uint64_t* d_ids, const uint64_t* d_bag_offsets, uint64_t n_bags,
                       uint64_t n_ids, void* d_out, void* stream);
int fsx_pooled_backward(fsx_pooled* p, const void* d_bag_grads, void* stream);

/* ---- engines: Synchronized / Prioritized embedding ------------------------ */
typedef struct fsx_engine fsx_engine;

/* engine flags */
#define FSX_ENGINE_PRESUM 1u /* prioritized: requesters pre-sum their collision
                                gradients per row before the collision
                                all-to-all (one row per (source, row) on the
                                blocking chain instead of one per occurrence).
                                Fixed two-level association: fp32 tolerance,
                                not bitwise with the reference. */

typedef struct fsx_engine_config {
  int mode;                  /* FSX_MODE_SYNC | FSX_MODE_PRIO */
  int transport;             /* FSX_TRANSPORT_CE | FSX_TRANSPORT_NCCL (N>1) */
  uint64_t max_occurrences;  /* capacity: ids per rank per iteration */
  uint32_t reduce_chunk;     /* 0: reference order (one sequential sum per
                                row); k>0: rows with more than k occurrences
                                are summed as fixed k-occurrence chunks, then
                                chunk partials in order (deterministic, shared
                                by both modes) */
  uint32_t flags;            /* FSX_ENGINE_* */
} fsx_engine_config;

int fsx_engine_create(fsx_ctx* ctx, fsx_table* table, const fsx_engine_config* cfg,
                      fsx_engine** out);
int fsx_engine_destroy(fsx_engine* e);

/* Peer wiring (N > 1). In-process ranks connect directly; separate
 * processes exchange the opaque blob from fsx_engine_export (CUDA IPC
 * handles of the receive windows) through any out-of-band channel. Every
 * rank must connect every peer before the first forward. */
int fsx_engine_connect_local(fsx_engine* e, int peer, fsx_engine* peer_engine);
int fsx_engine_export(fsx_engine* e, void* blob, uint64_t* len); /* blob capacity >= 4096 */
int fsx_engine_connect_ipc(fsx_engine* e, int peer, const void* blob, uint64_t len);
/* NCCL baseline transport: 128-byte ncclUniqueId from rank 0, shared by all */
int fsx_nccl_unique_id(void* id128);
int fsx_engine_connect_nccl(fsx_engine* e, const void* id128);

/* forward (embedding.hpp:129, 181): ids of this iteration (d_ids_cur, n_cur)
 * and, for the prioritized engine, of the next one (d_ids_next, n_next; pass
 * NULL on the final iteration). Writes n_cur x dim rows batch-major to d_out
 * on `stream` (the caller's compute stream). Host returns once the work is
 * enqueued; device-side errors surface at fsx_ctx_sync / later calls.
 * Id pointers may be device memory or (pinned) host memory; host ids are
 * copied on the engine's side lane. Device ids are ordered after the work
 * already on `stream` unless fsx_engine_set_ids_ready(e, 1) declared that the
 * caller passes only completed buffers. */
int fsx_engine_forward(fsx_engine* e, const uint64_t* d_ids_cur, uint64_t n_cur,
                       const uint64_t* d_ids_next, uint64_t n_next, void* d_out, void* stream);
/* backward: n_cur x dim gradients of the last forward, on `stream`. */
int fsx_engine_backward(fsx_engine* e, const void* d_grads, void* stream);
/* flush deferred exclusive gradients after the last backward (prioritized) */
int fsx_engine_finalize(fsx_engine* e, void* stream);
/* IterationStats of iteration `iter` (embedding.hpp:119-124): [collision_rows,
 * unique_next_rows, blocking_bytes]; synchronizes. Returns FSX_ERR_OUT_OF_RANGE
 * past the last forward. */
int fsx_engine_stats(fsx_engine* e, int iter, uint64_t* out3);
/* exposed embedding communication: total ms the caller's stream spent
 * blocked on embedding traffic since the last call — waits on the side lanes'
 * results (prioritized) and blocking all-to-alls on the caller's stream
 * (synchronized) — measured with CUDA event pairs around each wait; the
 * reference's Main/Wait + blocking collective time (sim.cpp:25-35).
 * Synchronizes; resets the accumulator. */
int fsx_engine_exposed_ms(fsx_engine* e, double* ms);

/* Live per-phase device timing (CUDA event pairs on the stream each phase
 * runs on). Off by default; when on, every phase launch is bracketed. */
#define FSX_PHASE_MERGE 0     /* C: resolve + batch-major merge (K6)            */
#define FSX_PHASE_SPLIT 1     /* C: gradient split / pack (K7)                  */
#define FSX_PHASE_CO_UPDATE 2 /* H: collision-row SGD (K8)                       */
#define FSX_PHASE_EX_UPDATE 3 /* L: deferred exclusive-row SGD (K8)             */
#define FSX_PHASE_PREFETCH 4  /* L: exclusive prefetch pack (K5)                */
#define FSX_PHASE_ECO 5       /* H: E_co pack (K9)                              */
#define FSX_PHASE_ROUTE 6     /* requester route + per-owner dedup (K1 K2 K4)   */
#define FSX_PHASE_DEDUP 7     /* owner flatten + sort/unique + src bits (K1 K2) */
#define FSX_PHASE_COLLIDE 8   /* collision flags + pack plans (K3)              */
#define FSX_PHASE_MASKS 9     /* masks + split / occurrence ranks (K10)         */
#define FSX_PHASE_SERVE 10    /* C: blocking per-occurrence lookup + scatter    */
#define FSX_PHASE_UPDATE 11   /* C: blocking full update                        */
#define FSX_PHASE_A2A 12      /* copy-engine transfers (any lane)               */
#define FSX_PHASE_EXPOSED 13  /* C: compute stream stalled on embedding traffic   */
#define FSX_NUM_PHASES 14
int fsx_engine_set_profiling(fsx_engine* e, int on);
/* Collision chain's transfers (prioritized engine, between iterations, the
 * same on every rank), a bit mask: 0 (default) = staged + copy-engine
 * all-to-alls (0 SMs); bit 0 = the collision update kernel stores each updated
 * E_co row straight into the requesters' windows over NVLink; bit 1 (PRESUM) =
 * the pre-sum kernel stores the collision gradients straight into the owners'
 * windows. Direct stores are SM-issued communication riding the compute
 * kernels (no extra kernel, one hop less, no copy-engine serialisation). */
int fsx_engine_set_eco_direct(fsx_engine* e, int on);
/* timeline of the recorded spans: out[3k..3k+2] = (phase, start ms, end ms)
 * relative to the earliest span; consumes them (synchronizes) */
int fsx_engine_spans(fsx_engine* e, double* out, uint64_t max_spans, uint64_t* n_spans);
/* the same spans with their lane and host issue time: out[6k..6k+5] =
 * (phase, lane (0 caller, 1 L, 2 H, 3 X, 4 top-priority, 5 a copy stream, 6 L2),
 * all-to-all channel (one copy: 1000 + 16 * channel + destination) or -1, GPU start ms, GPU end ms relative to the earliest span, host issue
 * time in CLOCK_MONOTONIC ms); consumes them */
int fsx_engine_trace(fsx_engine* e, double* out, uint64_t max_spans, uint64_t* n_spans);
/* device ids handed to forward are complete (no pending writes on any stream) */
/* Orders everything the engine has issued on its own lanes (side-lane jobs,
 * priority lanes, copy-engine streams) before `stream`. No protocol effect:
 * lets a caller end a timing region only when the engine is idle. */
int fsx_engine_join(fsx_engine* e, void* stream);
int fsx_engine_set_ids_ready(fsx_engine* e, int ready);
/* total ms and number of spans of `phase` since the last call for that
 * phase (synchronizes; resets the phase) */
int fsx_engine_phase_ms(fsx_engine* e, int phase, double* total_ms, uint64_t* spans);

/* ---- load balancer (partition.cpp, sim.hpp) -------------------------------- */

/* K12: CostModel::compute_time_for_lengths (sim.hpp:24-35) for each of
 * `num_groups` consecutive groups of lengths (group g = lens[offsets[g] ..
 * offsets[g+1])): h_out[g] = c0 + c1*sum(L) + c2*sum(L^2), bit-exact f64. */
int fsx_cost_estimate(fsx_ctx* ctx, const uint64_t* d_lens, const uint64_t* h_offsets,
                      int num_groups, double c0, double c1, double c2, double* h_out,
                      void* stream);

/* K13: fbs_partition (partition.cpp:157-176). Samples g = 0..m-1 carry
 * (uih_len, origin_rank, local_index). Outputs: h_assignment[m] (rank of g),
 * h_order[m] = receive_order flattened rank-major (each rank m/n entries). */
int fsx_fbs_partition(fsx_ctx* ctx, const uint64_t* h_lens, const int32_t* h_origin,
                      const int32_t* h_local, uint64_t m, int num_ranks, int32_t* h_assignment,
                      uint64_t* h_order, void* stream);

/* K14: vbs_partition (partition.cpp:178-209) without autotune state, or with
 * an initialized one when h_tuned_sizes != NULL (sizes summing to m).
 * alpha: exact device weights for alpha in {1,2}; otherwise pass the
 * per-sorted-position weights in h_weights (host std::pow, NULL for 1/2).
 * h_sizes_out[num_ranks] receives the segment sizes used. */
int fsx_vbs_partition(fsx_ctx* ctx, const uint64_t* h_lens, const int32_t* h_origin,
                      const int32_t* h_local, uint64_t m, int num_ranks, double alpha,
                      const int32_t* h_tuned_sizes, int32_t* h_sizes_out, int32_t* h_assignment,
                      uint64_t* h_order, void* stream);

/* autotune_update (partition.cpp:211-269) — n <= 64, host f64, no FMA */
int fsx_autotune_update(int n, int32_t* sizes, double* ema_local, double* ema_global, int step,
                        double delta, double decay, const double* local_times);

/* ---- raw copy-engine all-to-all (comm.cpp:308-365 analogue) ---------------- */
/* The engine's copy-engine all-to-all of bytes_per_peer from its GRADS
 * staging slots to every peer, exactly as the protocol's exchanges run
 * (enqueue only, no host synchronisation; collective) — a measurement entry
 * point for comparisons with other transports (tools/nccl_ce_compare.py). */
int fsx_engine_a2a_staged(fsx_engine* e, uint64_t bytes_per_peer, void* stream);
/* Each engine also exposes its transport as a plain byte all-to-all over the
 * engine's windows: send_bytes[d] bytes from d_send + send_offsets[d] go to
 * rank d; on return d_recv + d * slot_bytes holds what rank d sent here and
 * h_recv_bytes[d] its size. Collective: every rank calls it. Capacity:
 * slot_bytes <= the engine's window slot (max_occurrences * 8 * dim... see
 * fsx_engine_slot_bytes). Used by the balancer's stage-3 sample shuffle. */
uint64_t fsx_engine_slot_bytes(const fsx_engine* e);
int fsx_a2a_ce(fsx_engine* e, const void* d_send, const uint64_t* h_send_offsets,
               const uint64_t* h_send_bytes, void* d_recv, uint64_t slot_bytes,
               uint64_t* h_recv_bytes, void* stream);

/* ---- jagged reshuffle (jagged.hpp:89-248) ------------------- */
/* Device layout: values = elem_bytes-sized elements back to back, offsets =
 * u64 [n+1] exclusive prefix of the lengths. */
/* offsets of a length array (the JaggedTensor constructor's prefix, jagged.hpp:23-34) */
int fsx_jagged_offsets(fsx_ctx* ctx, const uint64_t* d_lengths, uint64_t n, uint64_t* d_offsets,
                       uint64_t* h_total, void* stream);
/* indexed_permute (jagged.hpp:89-111): output segment j = input segment
 * perm[j] (repetition allowed). Writes out lengths/offsets, *h_out_total; with
 * d_out_values == NULL only sizes. FSX_ERR_OUT_OF_RANGE ("indexed_permute:
 * segment index K out of range (have N)") before anything moves. */
int fsx_jagged_permute(fsx_ctx* ctx, const void* d_values, uint32_t elem_bytes, const uint64_t* d_offsets,
                       uint64_t n_segs, const uint64_t* d_perm, uint64_t n_perm, void* d_out_values,
                       uint64_t out_capacity, uint64_t* d_out_lengths, uint64_t* d_out_offsets,
                       uint64_t* h_out_total, void* stream);
/* keyed_transpose's permutation (jagged.hpp:227-248): feature_major != 0 maps
 * (f, s) at f*S+s to s*F+f, else the inverse */
int fsx_keyed_transpose_perm(fsx_ctx* ctx, uint64_t num_keys, uint64_t num_samples, int feature_major,
                             uint64_t* d_perm, void* stream);

/* ---- copy-engine all-gather (comm.cpp:185-306 analogue) --------------------- */
/* Collective: every rank contributes send_bytes bytes (<= max_bytes, the bound
 * every rank passes identically); on return d_recv + d * slot_bytes holds rank
 * d's bytes and h_recv_bytes[d] their size. ring = 0: direct copies to every
 * peer (all_gather, comm.cpp:185-259 — on NVSwitch each peer link runs at full
 * bandwidth); ring = 1: the reference's SmFree ring, p-1 forwarding stages
 * (ring_all_gather, comm.cpp:214-236 / 261-306). 0 SMs: copy engines and stream
 * memory operations only. CollectiveError if a chunk exceeds the bound or the
 * engine's all-gather slot (max(8 * max_occurrences, 64 KiB) bytes). */
int fsx_allgather_ce(fsx_engine* e, const void* d_send, uint64_t send_bytes, uint64_t max_bytes, void* d_recv,
                     uint64_t slot_bytes, uint64_t* h_recv_bytes, int ring, void* stream);

/* ---- workload-file replay ----------------------------------- */
/* Replaces workload::Reader::next_iteration (workload.hpp:131-140,
 * workload.cpp:500-549) for the engine's input. Host part: walk the length
 * prefixes of one iteration's bytes (h_bytes = the file from the iteration's
 * first byte): h_rank_samples[num_ranks] = samples per rank, h_rec_off[k] =
 * byte offset of record k's body (capacity cap; NULL only counts),
 * *h_consumed = the iteration's size. FSX_ERR_IO with the reference's text
 * ("workload: file truncated; last complete record is iteration I, rank R,
 * sample S") on a short file. No device work. */
int fsx_workload_scan(const uint8_t* h_bytes, uint64_t nbytes, int num_ranks, int iteration,
                      uint64_t* h_rank_samples, uint64_t* h_rec_off, uint64_t cap, uint64_t* h_n_records,
                      uint64_t* h_consumed);
/* Device part: d_bytes = the same iteration's bytes in HBM, d_rec_off = the
 * scan's offsets. Per record: d_uih_len[n], d_labels[n] (may be NULL); batch-major
 * d_offsets[n + 1] (u64 exclusive prefix) and d_values (uih ids, capacity cap;
 * NULL only sizes, *h_total = id count). FSX_ERR_IO "workload: record has
 * trailing bytes at iteration I, rank R, sample S" (decode_sample consumed less
 * than the record) or "workload: record truncated". Synchronizes `stream`. */
int fsx_workload_decode(fsx_ctx* ctx, const uint8_t* d_bytes, uint64_t nbytes, const uint64_t* d_rec_off,
                        uint64_t n, int iteration, const uint64_t* h_rank_samples, int num_ranks,
                        uint64_t* d_uih_len, uint64_t* d_offsets, double* d_labels, uint64_t* d_values,
                        uint64_t cap, uint64_t* h_total, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FSX_H */
