// Pooled (bag) embedding on one shard — BASELINE config 3's lookup: every
// (sample, table) bag of ids is sum-pooled into one row, and the backward
// scatters each bag's gradient row to all of its tokens before the
// row-wise SGD (the reference has only a toy mean-pool over whole samples,
// pipeline.cpp:59-67; this is the production operator that config 3 names:
// a pooled lookup whose result is one row per bag, so the owner-to-requester
// traffic of a table-wise shard is bags x D instead of tokens x D).
//
//   forward : pooled[b] = sum over the bag's tokens k, in order, of row(ids[k])
//             (f64 left fold from 0.0, one rounding to the table type)
//   backward: every token k of bag b takes gradient row g[b]; rows are then
//             updated exactly as ShardView::apply_gradients
//             (embedding.cpp:148-181) with the engine's chunk association
//
// The forward sorts the bag tokens by row (the update plan) right behind the
// pooled gather, so the backward is one update launch.
#include <cstdint>
#include <memory>
#include <string>

#include "capi_util.cuh"
#include "common.cuh"
#include "table.cuh"

namespace fsx {
namespace {

// warp per bag: lanes hold the 16-byte vectors of the row (NV per lane), U
// rows of the bag in flight per step; the token -> bag map for the backward
// is written on the way
template <class T, int NV, int U>
__global__ void __launch_bounds__(256) k_pool_bags(const T* __restrict__ table, ShardGeom g,
                                                   const uint64_t* __restrict__ ids,
                                                   const uint64_t* __restrict__ offs, uint64_t n_bags,
                                                   T* __restrict__ out, uint32_t* __restrict__ bag_of,
                                                   DevErr* err) {
  FSX_PDL_ENTER();
  constexpr int VE = static_cast<int>(16 / sizeof(T));
  using V = VecOf<T, VE>;
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t vpr = g.dim / VE;
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t b = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; b < n_bags; b += warps) {
    const uint64_t k0 = offs[b], k1 = offs[b + 1];
    double acc[NV][VE];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int x = 0; x < VE; ++x) acc[v][x] = 0.0;
    for (uint64_t kb = k0; kb < k1; kb += 32) {
      const uint32_t nk = static_cast<uint32_t>(min(static_cast<uint64_t>(32), k1 - kb));
      // lane l: token kb + l's row (validated: a bad id contributes nothing
      // and raises the reference's domain_error at the next sync)
      const T* myrow = nullptr;
      if (lane < nk) {
        const uint64_t id = ids[kb + lane];
        bag_of[kb + lane] = static_cast<uint32_t>(b);
        if (g.owns(id))
          myrow = table + (id / static_cast<uint64_t>(g.p)) * g.dim;
        else
          report(err, id >= g.total_rows ? kErrRowRange : kErrNotOwned, id,
                 id >= g.total_rows ? g.total_rows : static_cast<unsigned long long>(g.shard));
      }
      for (uint32_t t0 = 0; t0 < nk; t0 += U) {
        V r[U][NV];
        bool live[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const T* p = reinterpret_cast<const T*>(
              __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(myrow), (t0 + u) & 31u));
          live[u] = t0 + u < nk && p != nullptr;
#pragma unroll
          for (int v = 0; v < NV; ++v)
            if (live[u] && lane + 32u * v < vpr) r[u][v] = *reinterpret_cast<const V*>(p + (lane + 32u * v) * VE);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (live[u]) {
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
              for (int x = 0; x < VE; ++x) acc[v][x] = __dadd_rn(acc[v][x], static_cast<double>(r[u][v].v[x]));
          }
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (lane + 32u * v < vpr) {
        V o;
#pragma unroll
        for (int x = 0; x < VE; ++x) o.v[x] = static_cast<T>(acc[v][x]);
        *reinterpret_cast<V*>(out + b * g.dim + (lane + 32u * v) * VE) = o;
      }
  }
}

// scalar fallback for rows that are not whole 16-byte vectors: thread per
// (bag, column), tokens in order
template <class T>
__global__ void k_pool_bags_scalar(const T* __restrict__ table, ShardGeom g, const uint64_t* __restrict__ ids,
                                   const uint64_t* __restrict__ offs, uint64_t n_bags, T* __restrict__ out,
                                   uint32_t* __restrict__ bag_of, DevErr* err) {
  FSX_PDL_ENTER();
  const uint64_t total = n_bags * g.dim;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t b = i / g.dim;
    const uint32_t d = static_cast<uint32_t>(i - b * g.dim);
    double acc = 0.0;
    for (uint64_t k = offs[b]; k < offs[b + 1]; ++k) {
      const uint64_t id = ids[k];
      if (d == 0) bag_of[k] = static_cast<uint32_t>(b);
      if (!g.owns(id)) {
        if (d == 0)
          report(err, id >= g.total_rows ? kErrRowRange : kErrNotOwned, id,
                 id >= g.total_rows ? g.total_rows : static_cast<unsigned long long>(g.shard));
        continue;
      }
      acc = __dadd_rn(acc, static_cast<double>(table[(id / static_cast<uint64_t>(g.p)) * g.dim + d]));
    }
    out[i] = static_cast<T>(acc);
  }
}

}  // namespace
}  // namespace fsx

using namespace fsx;

struct fsx_pooled {
  Table* t = nullptr;
  uint64_t cap_occ = 0, cap_bags = 0;
  uint32_t chunk = 0;
  SortedIds srt;
  SgdScratch plan;
  DevBuf<uint32_t> bag_of;
  DevBuf<uint64_t> d_n;
  bool planned = false;
  uint64_t n_occ = 0, n_bags = 0;
};

namespace {

template <class T>
void pooled_forward(fsx_pooled* p, const uint64_t* d_ids, const uint64_t* d_offs, uint64_t n_bags, uint64_t n,
                    void* d_out, cudaStream_t s) {
  Table& t = *p->t;
  Ctx* ctx = t.ctx;
  constexpr int VE = static_cast<int>(16 / sizeof(T));
  const uint32_t rb = t.row_bytes();
  const unsigned vpl = (rb / 16 + 31) / 32;
  if (rb % 16 == 0 && vpl <= 2) {
    const unsigned grid = grid_for(ctx, n_bags * 32, 256, 8);
    if (vpl == 1)
      FSX_LAUNCH(ctx, (k_pool_bags<T, 1, 8>), grid, 256, 0, s, static_cast<const T*>(t.values), t.g, d_ids, d_offs,
                 n_bags, static_cast<T*>(d_out), p->bag_of.p, ctx->d_err);
    else
      FSX_LAUNCH(ctx, (k_pool_bags<T, 2, 4>), grid, 256, 0, s, static_cast<const T*>(t.values), t.g, d_ids, d_offs,
                 n_bags, static_cast<T*>(d_out), p->bag_of.p, ctx->d_err);
  } else {
    FSX_LAUNCH(ctx, k_pool_bags_scalar<T>, grid_for(ctx, n_bags * t.g.dim, 256, 8), 256, 0, s,
               static_cast<const T*>(t.values), t.g, d_ids, d_offs, n_bags, static_cast<T*>(d_out), p->bag_of.p,
               ctx->d_err);
  }
  (void)VE;
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
  p->planned = false;
  if (n_bags == 0) return FSX_OK;
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
  if (!p->planned && p->n_bags) raise(FSX_ERR_PROTOCOL, "pooled: backward before forward");
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
