// One shard of a row-wise sharded embedding table on the device (ShardView,
// embedding.hpp:59-90) and its update machinery.
#pragma once

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "sgd_stream.cuh"
#include "sorter.cuh"

namespace fsx {

struct SgdScratch {
  DevBuf<SgdItem> work, singles;
  DevBuf<const void*> gptr;  // gradient row per sorted occurrence
  DevBuf<uint32_t> multi, part_base;
  DevBuf<uint32_t> done;     // k_sgd_warp: chunks arrived per row (kept zeroed)
  DevBuf<double> partials;
  DevBuf<uint64_t> ent;      // stream plan: ring entries (k_sgd_stream)
  DevBuf<uint32_t> row_ent;  // stream plan: first gradient entry per row
  bool stream_plan = false;  // the last plan is a stream plan
  DevBuf<uint64_t> d_tot;  // [0] singles (stream plan: entries), [1] work items, [2] multi rows, [3] partial slots
  ScanScratch scan;
  uint64_t cap_rows = 0, cap_work = 0, cap_occ = 0;
  bool resolved = false;  // the last plan stored gradient-row pointers
  uint32_t dim = 0;
  void reserve(uint64_t rows, uint64_t occ, uint32_t d, uint32_t chunk) {
    const uint64_t w = rows + (chunk ? occ / chunk + 1 : 0);
    if (rows > cap_rows || w > cap_work || d != dim || occ > cap_occ) {
      cap_occ = occ > cap_occ ? occ : cap_occ;
      cap_rows = rows > cap_rows ? rows : cap_rows;
      cap_work = w > cap_work ? w : cap_work;
      dim = d;
      work.alloc(cap_work); singles.alloc(cap_rows); multi.alloc(cap_rows); part_base.alloc(cap_rows);
      done.alloc(cap_rows);
      FSX_CUDA(cudaMemset(done.p, 0, cap_rows * sizeof(uint32_t)));
      gptr.alloc(occ > rows ? occ : rows);
      ent.alloc(occ + rows + 1);
      row_ent.alloc(rows + 1);
      // a row with k > 1 chunks has > (k-1)*chunk occurrences: slots <= 2*occ/chunk
      partials.alloc(chunk ? (2 * occ / chunk + 1) * d : 1);
    }
    if (!d_tot.p) d_tot.alloc(4);
    scan.ensure(rows, 4);
  }
};

struct Table {
  Ctx* ctx = nullptr;
  ShardGeom g{};
  int dtype = FSX_F32;
  double lr = 0.0;
  uint64_t seed = 0;
  void* values = nullptr;
  size_t elem = 4;
  uint32_t row_bytes() const { return static_cast<uint32_t>(g.dim * elem); }
  int key_bits() const { return bits_for(g.local_rows > 0 ? g.local_rows - 1 : 0); }

  ~Table() {
    if (values) cudaFree(values);
  }
};

// Segmented deterministic SGD over the rows of `rs` (selected rows only),
// gradients from `gr`, in two halves:
//  sgd_plan  — the work lists (plan scan). With resolve_grads the gradient row
//              of every occurrence is resolved first (k_grad_ptrs) and stored
//              in the items; without it the plan depends on the row segments
//              alone, so it can be built ahead of time (before the gradients
//              exist) and the update kernels resolve gr.row(perm[k]) — for a
//              plain [M x dim] gradient array that is one multiply-add.
//  sgd_apply — the chunk kernels + combine over a plan.
// seg_out != nullptr: reduce only — each segment's gradient sum (same
// chunked association) goes to seg_out[u]; the table is not touched.
// k_sgd_stream handles rows of 1, 2 or 4 16-byte vectors per lane
template <class T>
bool use_stream(const Ctx* ctx, const Table& t) {
  const uint32_t rb = t.row_bytes();
  const unsigned vpl = (rb / 16 + 31) / 32;
  return ctx->sgd_stream && rb % 16 == 0 && (vpl == 1 || vpl == 2 || vpl == 4);
}

template <class T>
void sgd_plan(Ctx* ctx, Table& t, const RowSegments& rs, uint64_t rows_cap, uint64_t occ_cap,
              const GradRows<T>* resolve_grads, uint32_t chunk, SgdScratch& s, cudaStream_t stream,
              char* const* seg_out = nullptr, const uint32_t* grad_remap = nullptr) {
  if (rows_cap == 0) return;
  s.reserve(rows_cap, occ_cap, t.g.dim, chunk);
  s.stream_plan = use_stream<T>(ctx, t);
  const T** gptr = nullptr;
  if (resolve_grads) {
    gptr = reinterpret_cast<const T**>(s.gptr.p);
    FSX_LAUNCH(ctx, k_grad_ptrs<T>, grid_for(ctx, occ_cap, 256, 8), 256, 0, stream, *resolve_grads, rs.perm,
               rs.seg_start, rs.d_u, gptr);
  }
  s.resolved = gptr != nullptr;
  SgdPlanOp plan{rs, chunk, s.singles.p, s.work.p, s.multi.p, s.part_base.p, static_cast<char*>(t.values),
                 t.row_bytes(), t.g.local_rows, seg_out, reinterpret_cast<const char* const*>(gptr)};
  if (s.stream_plan) {
    plan.ent = s.ent.p;
    plan.row_ent = s.row_ent.p;
  }
  run_scan(ctx, plan, rows_cap, rs.d_u, s.scan, s.d_tot.p, stream);
  if (s.stream_plan)
    FSX_LAUNCH(ctx, k_stream_entries, grid_for(ctx, occ_cap, 256, 8), 256, 0, stream, rs.seg_start, rs.d_u, rs.perm,
               rs.inverse, reinterpret_cast<const char* const*>(gptr), s.row_ent.p, s.ent.p, grad_remap);
}

// persistent grid of k_sgd_stream: as many 4-warp CTAs per SM as shared
// memory allows, capped by ctx->stream_per_sm
template <class T, int NV, int R, int MINB, bool kBulk, bool kFused>
void launch_sgd_stream(Ctx* ctx, const SgdArgs<T>& a, uint32_t rb, uint32_t* done, cudaStream_t stream) {
  constexpr int kWarps = 4;
  const size_t smem = ((kWarps * R * 8 + 127) & ~static_cast<size_t>(127)) + static_cast<size_t>(kWarps) * R * rb;
  // function attributes are per device: one entry per (device, ring size)
  // (in-process ranks on several GPUs each set them on their own device)
  static std::mutex m;
  static std::unordered_map<size_t, int>* occ = new std::unordered_map<size_t, int>();
  int per_sm;
  {
    std::lock_guard<std::mutex> g(m);
    const size_t key = smem * 1024 + static_cast<size_t>(ctx->device);
    auto it = occ->find(key);
    if (it == occ->end()) {
      if (smem > 48 * 1024)
        FSX_CUDA(cudaFuncSetAttribute(k_sgd_stream<T, NV, R, MINB, kBulk, kFused>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
      // the ring is the point of the kernel: ask for the largest shared carveout
      FSX_CUDA(cudaFuncSetAttribute(k_sgd_stream<T, NV, R, MINB, kBulk, kFused>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    cudaSharedmemCarveoutMaxShared));
      int b = 0;
      FSX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_sgd_stream<T, NV, R, MINB, kBulk, kFused>, kWarps * 32, smem));
      if (std::getenv("FSX_DEBUG"))
        std::fprintf(stderr, "[fsx] k_sgd_stream<%d,%d,%d> smem %zu B/CTA: %d CTAs/SM\n", static_cast<int>(sizeof(T)),
                     NV, R, smem, b);
      it = occ->emplace(key, b > 0 ? b : 1).first;
    }
    per_sm = it->second;
  }
  per_sm = std::min<int>(per_sm, static_cast<int>(ctx->stream_per_sm));
  // kernel span (fsx_ctx_kernel_span): each launch gets a slot of the
  // context's ring; the kernel stores ~first start and last end (globaltimer
  // ns) with atomicMax, so a zeroed slot needs no per-launch initialisation
  unsigned long long* span = nullptr;
  if (ctx->span_on && ctx->span_next < Ctx::kSpanSlots) span = ctx->d_span + 2 * ctx->span_next++;
  FSX_LAUNCH(ctx, (k_sgd_stream<T, NV, R, MINB, kBulk, kFused>), static_cast<unsigned>(ctx->num_sms * per_sm), kWarps * 32, smem,
             stream, a, rb, done, span);
}

template <class T>
void sgd_apply(Ctx* ctx, Table& t, const RowSegments& rs, uint64_t rows_cap, uint64_t occ_cap,
               const GradRows<T>& gr, uint32_t chunk, SgdScratch& s, T* rows_out, cudaStream_t stream,
               char* const* seg_out = nullptr) {
  if (rows_cap == 0) return;
  const T** gptr = s.resolved ? reinterpret_cast<const T**>(s.gptr.p) : nullptr;
  SgdArgs<T> a{static_cast<T*>(t.values), t.g, t.lr, rs, gr, chunk, s.singles.p, s.d_tot.p, s.work.p,
               s.d_tot.p + 1, s.multi.p, s.d_tot.p + 2, s.part_base.p, s.partials.p, rows_out, ctx->d_err,
               seg_out, gptr};
  const uint64_t work_cap = rows_cap + (chunk ? occ_cap / chunk + 1 : 0);
  const unsigned g2 = grid_for(ctx, rows_cap, 1, 8);
  const uint32_t rb = t.row_bytes();
  constexpr int VE16 = static_cast<int>(16 / sizeof(T));
  const int ve = rb % 16 == 0 ? VE16 : 1;
  // one thread per (work item, vector); the grid streams over all of them
  const unsigned vpr = t.g.dim / static_cast<unsigned>(ve);
  const uint32_t shift = (vpr & (vpr - 1)) == 0 ? static_cast<uint32_t>(__builtin_ctz(vpr)) : 0xffffffffu;
  const unsigned g0 = grid_for(ctx, rows_cap * vpr / 2, 256, ctx->single_per_sm);
  const unsigned g1 = grid_for(ctx, work_cap * vpr, 256, ctx->flat_per_sm);
  const unsigned vpl = (vpr + 31) / 32;
  if (s.stream_plan) {
    // one persistent kernel, rows staged by bulk copies (sgd_stream.cuh)
    a.ent = s.ent.p;
    // Default (B200 A/B at config 4, one rank): rings of 16 rows, 3 CTAs of
    // 4 warps per SM (12 warps x 16 KB in flight per SM), hot-row combine
    // fused. Fewer, deeper rings leave registers and shared memory on every
    // SM for the side lane's latency-bound kernels (route / dedup / collide
    // of the next iteration), which the update otherwise starves.
    // FSX_STREAM_VARIANT (tuning): 1 = 8-row rings at 5 CTAs per SM,
    // 2 = separate k_sgd_combine, 3 = LDGSTS instead of bulk copies,
    // 4 = 12-row rings at 4 CTAs per SM.
    const unsigned var = ctx->stream_variant;
    const bool fused = var != 2;
    uint32_t* done = s.done.p;
    if (vpl == 1)
      launch_sgd_stream<T, 1, 16, 5, true, true>(ctx, a, rb, done, stream);
    else if (vpl == 2 && var == 1)
      launch_sgd_stream<T, 2, 8, 5, true, true>(ctx, a, rb, done, stream);
    else if (vpl == 2 && var == 2)
      launch_sgd_stream<T, 2, 16, 3, true, false>(ctx, a, rb, done, stream);
    else if (vpl == 2 && var == 4)
      launch_sgd_stream<T, 2, 12, 4, true, true>(ctx, a, rb, done, stream);
    else if (vpl == 2 && var == 3)
      launch_sgd_stream<T, 2, 16, 3, false, true>(ctx, a, rb, done, stream);
    else if (vpl == 2)
      launch_sgd_stream<T, 2, 16, 3, true, true>(ctx, a, rb, done, stream);
    else
      launch_sgd_stream<T, 4, 8, 3, true, true>(ctx, a, rb, done, stream);
    if (chunk && !fused) {  // hot rows: chunk partials in chunk order
      if (t.g.dim % 2 == 0)
        FSX_LAUNCH(ctx, (k_sgd_combine<T, 2>), g2, 128, 0, stream, a);
      else
        FSX_LAUNCH(ctx, (k_sgd_combine<T, 1>), g2, 128, 0, stream, a);
    }
    return;
  }
  if (ve == VE16 && ctx->sgd_warp && vpl <= 4 && vpl != 3) {
    // warp per work item, combine fused (k_sgd_warp)
    FSX_LAUNCH(ctx, (k_sgd_single<T, VE16>), g0, 256, 0, stream, a, shift);
    const unsigned gw = grid_for(ctx, work_cap * 32, 256, ctx->warp_per_sm);
    if (vpl == 1)
      FSX_LAUNCH(ctx, (k_sgd_warp<T, VE16, 1, 4>), gw, 256, 0, stream, a, s.done.p);
    else if (vpl == 2 && ctx->warp_variant == 1)
      FSX_LAUNCH(ctx, (k_sgd_warp<T, VE16, 2, 2, 3>), gw, 256, 0, stream, a, s.done.p);
    else if (vpl == 2 && ctx->warp_variant == 2)
      FSX_LAUNCH(ctx, (k_sgd_warp<T, VE16, 2, 4, 3>), gw, 256, 0, stream, a, s.done.p);
    else if (vpl == 2 && ctx->warp_variant == 3)
      FSX_LAUNCH(ctx, (k_sgd_warp<T, VE16, 2, 2, 4>), gw, 256, 0, stream, a, s.done.p);
    else if (vpl == 2)
      FSX_LAUNCH(ctx, (k_sgd_warp<T, VE16, 2, 4>), gw, 256, 0, stream, a, s.done.p);
    else
      FSX_LAUNCH(ctx, (k_sgd_warp<T, VE16, 4, 2>), gw, 256, 0, stream, a, s.done.p);
    return;
  }
  if (ve == VE16) {
    FSX_LAUNCH(ctx, (k_sgd_single<T, VE16>), g0, 256, 0, stream, a, shift);
    FSX_LAUNCH(ctx, (k_sgd_flat<T, VE16>), g1, 256, 0, stream, a, shift);
  } else {
    FSX_LAUNCH(ctx, (k_sgd_single<T, 1>), g0, 256, 0, stream, a, shift);
    FSX_LAUNCH(ctx, (k_sgd_flat<T, 1>), g1, 256, 0, stream, a, shift);
  }
  if (chunk) {
    if (t.g.dim % 2 == 0)
      FSX_LAUNCH(ctx, (k_sgd_combine<T, 2>), g2, 128, 0, stream, a);
    else
      FSX_LAUNCH(ctx, (k_sgd_combine<T, 1>), g2, 128, 0, stream, a);
  }
}

template <class T>
void sgd_update_rows(Ctx* ctx, Table& t, const RowSegments& rs, uint64_t rows_cap,
                     uint64_t occ_cap, const GradRows<T>& gr, uint32_t chunk, SgdScratch& s,
                     T* rows_out, cudaStream_t stream, char* const* seg_out = nullptr) {
  sgd_plan<T>(ctx, t, rs, rows_cap, occ_cap, &gr, chunk, s, stream, seg_out);
  sgd_apply<T>(ctx, t, rs, rows_cap, occ_cap, gr, chunk, s, rows_out, stream, seg_out);
}

}  // namespace fsx

// opaque C-ABI handles (include/fsx.h) are the internal objects
struct fsx_ctx : fsx::Ctx {};
struct fsx_table : fsx::Table {};
