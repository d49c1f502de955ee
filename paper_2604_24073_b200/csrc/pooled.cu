// Pooled (bag) embedding on one shard — BASELINE config 3's lookup: every
// (sample, table) bag of ids is sum-pooled into one row, and the backward
// scatters each bag's gradient row to all of its tokens before the
// row-wise SGD (the reference has only a toy mean-pool over whole samples,
// pipeline.cpp:59-67; this is the production operator that config 3 names:
// a pooled lookup whose result is one row per bag, so the owner-to-requester
// traffic of a table-wise shard is bags x D instead of tokens x D).
//
//   forward : pooled[b] = sum over the bag's tokens k, in order, of row(ids[k])
//             (f64, the chunk association below, one rounding to the table type)
//   backward: every token k of bag b takes gradient row g[b]; rows are then
//             updated exactly as ShardView::apply_gradients
//             (embedding.cpp:148-181) with the engine's chunk association
//
// The forward is the update kernels' segmented reduce in reduce-only mode over
// bags (so its association is theirs: tokens left-folded from 0.0 in order,
// bags longer than `reduce_chunk` tokens as chunk partials folded in chunk
// order), then sorts the tokens by row (the update plan), so the backward is
// one update launch.
#include <cstdint>
#include <memory>
#include <string>

#include "capi_util.cuh"
#include "common.cuh"
#include "table.cuh"

namespace fsx {
namespace {

// Per bag: its start as a u32 segment offset, its output row's address (the
// reduce-only destinations) and a zero row for an empty bag; per token: its
// local table row (the gradient-row index the segmented reduce reads) and
// its bag (the backward's gradient row). A bad id reads row 0 and raises the
// reference's domain_error at the next sync. Warp per bag.
__global__ void k_pool_prep(ShardGeom g, const uint64_t* __restrict__ ids, const uint64_t* __restrict__ offs,
                            uint64_t n_bags, char* out, uint32_t row_bytes, uint32_t* __restrict__ bag_start,
                            char** __restrict__ seg_out, uint32_t* __restrict__ row_of,
                            uint32_t* __restrict__ bag_of, uint64_t* __restrict__ d_nbags, DevErr* err) {
  FSX_PDL_ENTER();
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t w0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w0 == 0 && lane == 0) {
    *d_nbags = n_bags;
    bag_start[n_bags] = static_cast<uint32_t>(offs[n_bags]);
  }
  for (uint64_t b = w0; b < n_bags; b += warps) {
    const uint64_t k0 = offs[b], k1 = offs[b + 1];
    char* row = out + b * row_bytes;
    if (lane == 0) {
      bag_start[b] = static_cast<uint32_t>(k0);
      seg_out[b] = row;
    }
    if (k0 == k1)
      for (uint32_t x = lane * 4; x < row_bytes; x += 128) *reinterpret_cast<uint32_t*>(row + x) = 0u;
    for (uint64_t k = k0 + lane; k < k1; k += 32) {
      const uint64_t id = ids[k];
      bag_of[k] = static_cast<uint32_t>(b);
      uint32_t r = 0;
      if (g.owns(id))
        r = static_cast<uint32_t>(id / static_cast<uint64_t>(g.p));
      else
        report(err, id >= g.total_rows ? kErrRowRange : kErrNotOwned, id,
               id >= g.total_rows ? g.total_rows : static_cast<unsigned long long>(g.shard));
      row_of[k] = r;
    }
  }
}

}  // namespace
}  // namespace fsx

using namespace fsx;

struct fsx_pooled {
  Table* t = nullptr;
  uint64_t cap_occ = 0, cap_bags = 0;
  uint32_t chunk = 0;
  SortedIds srt;          // the backward's tokens sorted by row
  SgdScratch fplan, plan; // forward (bags) and backward (rows) work lists
  DevBuf<uint32_t> bag_of, row_of, bag_start;
  DevBuf<char*> seg_out;
  DevBuf<uint64_t> d_nbags;
  bool planned = false;
  uint64_t n_occ = 0, n_bags = 0;
};

namespace {

// forward: the segmented reduce of the update kernels in reduce-only mode —
// segments = bags (tokens already in bag order: identity permutation),
// "gradient" rows = the tokens' table rows, the same fixed chunk association
// (k_sgd_stream: rows staged by bulk copies, balanced across warps, hot bags
// split into chunks), each bag's f64 sum rounded once into its output row.
// Then the backward's plan: tokens sorted by row.
template <class T>
void pooled_forward(fsx_pooled* p, const uint64_t* d_ids, const uint64_t* d_offs, uint64_t n_bags, uint64_t n,
                    void* d_out, cudaStream_t s) {
  Table& t = *p->t;
  Ctx* ctx = t.ctx;
  const uint32_t rb = t.row_bytes();
  FSX_LAUNCH(ctx, k_pool_prep, grid_for(ctx, n_bags * 32, 256, 8), 256, 0, s, t.g, d_ids, d_offs, n_bags,
             static_cast<char*>(d_out), rb, p->bag_start.p, p->seg_out.p, p->row_of.p, p->bag_of.p,
             p->d_nbags.p, ctx->d_err);
  if (n) {
    RowSegments bags{nullptr, p->bag_start.p, nullptr, p->d_nbags.p, nullptr, 0, p->bag_of.p};
    sgd_plan<T>(ctx, t, bags, n_bags, n, nullptr, p->chunk, p->fplan, s, p->seg_out.p, p->row_of.p);
    GradRows<T> rows{static_cast<const char*>(t.values), 0, nullptr, p->fplan.stream_plan ? nullptr : p->row_of.p,
                     rb};
    sgd_apply<T>(ctx, t, bags, n_bags, n, rows, p->chunk, p->fplan, nullptr, s, p->seg_out.p);
  }
  // the backward's plan: tokens sorted by row (stable: bag order within a
  // row), the update work lists with each token's gradient row = its bag's
  FSX_CUDA(cudaMemcpyAsync(p->srt.d_n(), &p->n_occ, 8, cudaMemcpyHostToDevice, s));
  p->srt.run(ctx, d_ids, n, t.g, true, false, t.key_bits(), s);
  RowSegments rs{p->srt.uniq.p, p->srt.seg_start.p, p->srt.perm, p->srt.d_u(), nullptr, 0, p->srt.inverse.p};
  sgd_plan<T>(ctx, t, rs, n, n, nullptr, p->chunk, p->plan, s, nullptr, p->bag_of.p);
}

template <class T>
void pooled_backward(fsx_pooled* p, const void* d_bag_grads, cudaStream_t s) {
  Table& t = *p->t;
  RowSegments rs{p->srt.uniq.p, p->srt.seg_start.p, p->srt.perm, p->srt.d_u(), nullptr, 0, p->srt.inverse.p};
  // stream plans carry each token's bag row already (the remap); the other
  // update kernels resolve it through occ_idx
  GradRows<T> gr{static_cast<const char*>(d_bag_grads), 0, nullptr, p->plan.stream_plan ? nullptr : p->bag_of.p,
                 t.row_bytes()};
  sgd_apply<T>(t.ctx, t, rs, p->n_occ, p->n_occ, gr, p->chunk, p->plan, nullptr, s);
}

}  // namespace

extern "C" {

int fsx_pooled_create(fsx_table* t, uint64_t max_occurrences, uint64_t max_bags, uint32_t reduce_chunk,
                      fsx_pooled** out) {
  FSX_API_BEGIN
  DeviceGuard dg(t->ctx->device);
  if (max_occurrences >= (1ull << 32) || max_bags >= (1ull << 32))
    raise(FSX_ERR_CONFIG, "pooled: capacity beyond 2^32 tokens or bags");
  auto p = std::make_unique<fsx_pooled>();
  p->t = t;
  p->cap_occ = max_occurrences > 0 ? max_occurrences : 1;
  p->cap_bags = max_bags > 0 ? max_bags : 1;
  p->chunk = reduce_chunk;
  p->srt.reserve(p->cap_occ);
  p->bag_of.alloc(p->cap_occ);
  p->row_of.alloc(p->cap_occ);
  p->bag_start.alloc(p->cap_bags + 1);
  p->seg_out.alloc(p->cap_bags);
  p->d_nbags.alloc(1);
  *out = p.release();
  FSX_API_END
}

int fsx_pooled_destroy(fsx_pooled* p) {
  FSX_API_BEGIN
  if (!p) return FSX_OK;
  DeviceGuard dg(p->t->ctx->device);
  FSX_CUDA(cudaDeviceSynchronize());
  delete p;
  FSX_API_END
}

int fsx_pooled_forward(fsx_pooled* p, const uint64_t* d_ids, const uint64_t* d_bag_offsets, uint64_t n_bags,
                       uint64_t n_ids, void* d_out, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(p->t->ctx->device);
  if (n_ids > p->cap_occ || n_bags > p->cap_bags)
    raise(FSX_ERR_INVALID_ARGUMENT, "pooled: " + std::to_string(n_ids) + " ids in " + std::to_string(n_bags) +
                                        " bags exceed the capacity (" + std::to_string(p->cap_occ) + " ids, " +
                                        std::to_string(p->cap_bags) + " bags)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  p->n_occ = n_ids;
  p->n_bags = n_bags;
  p->planned = true;  // (an empty batch has nothing to plan)
  if (n_bags == 0) return FSX_OK;
  p->planned = false;
  if (p->t->dtype == FSX_F32)
    pooled_forward<float>(p, d_ids, d_bag_offsets, n_bags, n_ids, d_out, s);
  else
    pooled_forward<double>(p, d_ids, d_bag_offsets, n_bags, n_ids, d_out, s);
  p->planned = true;
  FSX_API_END
}

int fsx_pooled_backward(fsx_pooled* p, const void* d_bag_grads, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(p->t->ctx->device);
  if (!p->planned) raise(FSX_ERR_PROTOCOL, "pooled: backward before forward");
  if (p->n_occ == 0) return FSX_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p->t->dtype == FSX_F32)
    pooled_backward<float>(p, d_bag_grads, s);
  else
    pooled_backward<double>(p, d_bag_grads, s);
  p->planned = false;
  FSX_API_END
}

}  // extern "C"
