// libfsx core: context, error mapping, primitives (K1-K5, K8, K11) and the
// table object behind the C ABI in include/fsx.h.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "capi_util.cuh"
#include "table.cuh"

namespace fsx {

std::string describe(const DevErr& e, int* code) {
  auto u = [](unsigned long long v) { return std::to_string(v); };
  switch (e.kind) {
    case kErrRowRange:
      *code = FSX_ERR_DOMAIN;
      return "embedding: row id " + u(e.a) + " out of range (table has " + u(e.b) + " rows)";
    case kErrNotOwned:
      *code = FSX_ERR_DOMAIN;
      return "embedding: row id " + u(e.a) + " is not owned by shard " + u(e.b);
    case kErrNonFinite:
      *code = FSX_ERR_DOMAIN;
      return "embedding: non-finite value after update of row " + u(e.a);
    case kErrRecvNotOwned:
      *code = FSX_ERR_PROTOCOL;
      return "embedding: received row " + u(e.a) + " that this shard does not own";
    case kErrMissingRow:
      *code = FSX_ERR_PROTOCOL;
      return "embedding: row " + u(e.a) + " missing from both prefetched buffers";
    case kErrCapacity:
      *code = FSX_ERR_COLLECTIVE;
      return "fsx: buffer capacity exceeded (need " + u(e.a) + ", have " + u(e.b) + ")";
    case kErrMissingCoRow:
      *code = FSX_ERR_PROTOCOL;
      return "embedding: collision row " + u(e.a) + " missing from the update result";
    case kErrMaskOverlap:
      *code = FSX_ERR_PROTOCOL;
      return "embedding: a row appears in both collision and exclusive masks";
    case kErrSegIndex:  // jagged.hpp:93-96
      *code = FSX_ERR_OUT_OF_RANGE;
      return "indexed_permute: segment index " + u(e.a) + " out of range (have " + u(e.b) + ")";
    default:
      *code = FSX_ERR_CUDA;
      return "fsx: unknown device error " + std::to_string(e.kind);
  }
}

void Ctx::check_error(cudaStream_t s) {
  FSX_CUDA(cudaMemcpyAsync(h_err, d_err, sizeof(DevErr), cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  if (h_err->kind != kErrNone) {
    DevErr e = *h_err;
    FSX_CUDA(cudaMemsetAsync(d_err, 0, sizeof(DevErr), s));
    FSX_CUDA(cudaStreamSynchronize(s));
    int code = FSX_ERR_CUDA;
    std::string msg = describe(e, &code);
    raise(code, msg);
  }
}

// ---- K3 ----------------------------------------------------------------------
__global__ void k_intersect_flags(const uint64_t* __restrict__ a, const uint64_t* d_na,
                                  const uint64_t* __restrict__ b, const uint64_t* d_nb,
                                  uint8_t* __restrict__ flag_a, uint8_t* __restrict__ flag_b,
                                  uint32_t* __restrict__ partner_a) { FSX_PDL_ENTER();
  const uint64_t na = *d_na, nb = *d_nb;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < na;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t x = a[i];
    uint64_t lo = 0, hi = nb;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (b[mid] < x) lo = mid + 1; else hi = mid;
    }
    const bool hit = lo < nb && b[lo] == x;
    flag_a[i] = hit ? 1 : 0;
    if (hit && flag_b) flag_b[lo] = 1;
    if (hit && partner_a) partner_a[i] = static_cast<uint32_t>(lo);
  }
}

}  // namespace fsx

using namespace fsx;


namespace {

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// First offending occurrence in reference order, for exact error messages on
// the synchronous primitives (lookup walks ids in order, embedding.cpp:141-143;
// apply_gradients walks sorted unique ids, :168-169).
void raise_first_bad(const Table& t, const uint64_t* d_ids, uint64_t n, bool sorted_order) {
  std::vector<uint64_t> h(n);
  if (n) FSX_CUDA(cudaMemcpy(h.data(), d_ids, n * 8, cudaMemcpyDeviceToHost));
  if (sorted_order) std::sort(h.begin(), h.end());
  for (uint64_t id : h) {
    if (id >= t.g.total_rows)
      raise(FSX_ERR_DOMAIN, "embedding: row id " + std::to_string(id) + " out of range (table has " +
                                std::to_string(t.g.total_rows) + " rows)");
    if (static_cast<int>(id % static_cast<uint64_t>(t.g.p)) != t.g.shard)
      raise(FSX_ERR_DOMAIN, "embedding: row id " + std::to_string(id) +
                                " is not owned by shard " + std::to_string(t.g.shard));
  }
}

template <class T>
void table_sgd(Table& t, const uint64_t* d_ids, uint64_t n, const void* d_grads, uint64_t* d_unique,
               void* d_rows, uint64_t* h_num_unique, cudaStream_t s) {
  Ctx* ctx = t.ctx;
  SortedIds srt;
  srt.reserve(n);
  FSX_CUDA(cudaMemcpyAsync(srt.d_n(), &n, 8, cudaMemcpyHostToDevice, s));
  srt.run(ctx, d_ids, n, t.g, true, true, t.key_bits(), s);
  try {
    ctx->check_error(s);
  } catch (const Error&) {
    raise_first_bad(t, d_ids, n, true);
    throw;
  }
  RowSegments rs{srt.uniq.p, srt.seg_start.p, srt.perm, srt.d_u(), nullptr, 0};
  GradRows<T> gr{static_cast<const char*>(d_grads), 0, nullptr, nullptr, t.row_bytes()};
  SgdScratch sc;
  sgd_update_rows<T>(ctx, t, rs, n, n, gr, 0, sc, static_cast<T*>(d_rows), s);
  uint64_t u = 0;
  FSX_CUDA(cudaMemcpyAsync(&u, srt.d_u(), 8, cudaMemcpyDeviceToHost, s));
  if (d_unique && n) FSX_CUDA(cudaMemcpyAsync(d_unique, srt.uniq_g.p, n * 8, cudaMemcpyDeviceToDevice, s));
  ctx->check_error(s);
  if (h_num_unique) *h_num_unique = u;
}

}  // namespace

extern "C" {

const char* fsx_last_error(void) { return capi_last_error(); }

const char* fsx_version(void) {
  return "libfsx 0.1 sm_100a (" __DATE__ ") nvcc " FSX_STR(__CUDACC_VER_MAJOR__) "." FSX_STR(
      __CUDACC_VER_MINOR__);
}

int fsx_ctx_create(int device, int rank, int world, fsx_ctx** out) {
  FSX_API_BEGIN
  if (world < 1 || rank < 0 || rank >= world) raise(FSX_ERR_INVALID_ARGUMENT, "fsx: bad rank/world");
  FSX_CUDA(cudaSetDevice(device));
  auto c = std::make_unique<fsx_ctx>();
  c->device = device;
  c->rank = rank;
  c->world = world;
  FSX_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  auto env_u = [](const char* k, unsigned d) {
    const char* v = std::getenv(k);
    return v && std::atoi(v) > 0 ? static_cast<unsigned>(std::atoi(v)) : d;
  };
  c->copy_per_sm = env_u("FSX_COPY_PER_SM", c->copy_per_sm);
  c->single_per_sm = env_u("FSX_SINGLE_PER_SM", c->single_per_sm);
  c->flat_per_sm = env_u("FSX_FLAT_PER_SM", c->flat_per_sm);
  c->warp_per_sm = env_u("FSX_WARP_PER_SM", c->warp_per_sm);
  c->warp_variant = env_u("FSX_WARP_VARIANT", c->warp_variant);
  if (const char* v = std::getenv("FSX_SGD_WARP")) c->sgd_warp = std::atoi(v) != 0;
  if (const char* v = std::getenv("FSX_SGD_STREAM")) c->sgd_stream = std::atoi(v) != 0;
  c->stream_per_sm = env_u("FSX_STREAM_PER_SM", c->stream_per_sm);
  c->stream_variant = env_u("FSX_STREAM_VARIANT", c->stream_variant);
  // onesweep radix passes: on (bench A/B on B200, after the one-rank side
  // lane was slimmed: 0.274 -> 0.259 ms at N = 1; on at N = 4 as well)
  c->onesweep = true;
  if (const char* v = std::getenv("FSX_ONESWEEP")) c->onesweep = std::atoi(v) != 0;
  if (const char* v = std::getenv("FSX_PDL")) c->pdl = std::atoi(v) != 0;
  FSX_CUDA(cudaMalloc(&c->d_err, sizeof(DevErr)));
  FSX_CUDA(cudaMemset(c->d_err, 0, sizeof(DevErr)));
  FSX_CUDA(cudaMallocHost(&c->h_err, sizeof(DevErr)));
  std::memset(c->h_err, 0, sizeof(DevErr));
  *out = c.release();
  FSX_API_END
}

int fsx_ctx_destroy(fsx_ctx* ctx) {
  FSX_API_BEGIN
  if (!ctx) return FSX_OK;
  DeviceGuard dg(ctx->device);
  if (ctx->d_span) cudaFree(ctx->d_span);
  cudaFree(ctx->d_err);
  cudaFreeHost(ctx->h_err);
  delete ctx;
  FSX_API_END
}

int fsx_ctx_sync(fsx_ctx* ctx) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  FSX_CUDA(cudaDeviceSynchronize());
  ctx->check_error(nullptr);
  FSX_API_END
}

uint64_t fsx_ctx_launches(const fsx_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

int fsx_ctx_kernel_span(fsx_ctx* ctx, int on, double* mean_us, uint64_t* n) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  double tot = 0;
  uint64_t k = 0;
  if (ctx->span_on && ctx->span_next) {
    // every launch of the window has run: read the slots
    FSX_CUDA(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(2 * ctx->span_next);
    FSX_CUDA(cudaMemcpy(h.data(), ctx->d_span, h.size() * 8, cudaMemcpyDeviceToHost));
    for (uint64_t j = 0; j < ctx->span_next; ++j) {
      const unsigned long long a = ~h[2 * j], b = h[2 * j + 1];
      if (h[2 * j] && b > a) {
        tot += 1e-3 * static_cast<double>(b - a);
        ++k;
      }
    }
  }
  if (mean_us) *mean_us = k ? tot / static_cast<double>(k) : 0.0;
  if (n) *n = k;
  ctx->span_on = on != 0;
  ctx->span_next = 0;
  if (ctx->span_on) {
    if (!ctx->d_span) FSX_CUDA(cudaMalloc(&ctx->d_span, 2 * 8 * fsx::Ctx::kSpanSlots));
    FSX_CUDA(cudaMemset(ctx->d_span, 0, 2 * 8 * fsx::Ctx::kSpanSlots));
  }
  FSX_API_END
}

int fsx_sort_unique_u64(fsx_ctx* ctx, const uint64_t* d_keys, uint64_t n, uint64_t* d_unique,
                        uint32_t* d_inverse, uint64_t* h_num_unique, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  cudaStream_t s = S(stream);
  if (n == 0) {
    if (h_num_unique) *h_num_unique = 0;
    return FSX_OK;
  }
  // significant bits from the maximum key
  std::vector<uint64_t> h(1);
  DevBuf<uint64_t> dmax(1);
  {
    // small reduction via the scan machinery would be overkill: one pass of
    // atomicMax over u64 keys
    FSX_CUDA(cudaMemsetAsync(dmax.p, 0, 8, s));
    capi_launch_max_u64(ctx, d_keys, n, dmax.p, s);
    FSX_CUDA(cudaMemcpyAsync(h.data(), dmax.p, 8, cudaMemcpyDeviceToHost, s));
    FSX_CUDA(cudaStreamSynchronize(s));
  }
  SortedIds srt;
  srt.reserve(n);
  srt.reserve64();
  FSX_CUDA(cudaMemcpyAsync(srt.d_n(), &n, 8, cudaMemcpyHostToDevice, s));
  ShardGeom g{~0ull, 0, 1, 1, 0};
  srt.run(ctx, d_keys, n, g, false, false, bits_for(h[0]), s);
  uint64_t u = 0;
  FSX_CUDA(cudaMemcpyAsync(&u, srt.d_u(), 8, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  if (d_unique) FSX_CUDA(cudaMemcpyAsync(d_unique, srt.uniq.p, u * 8, cudaMemcpyDeviceToDevice, s));
  if (d_inverse) FSX_CUDA(cudaMemcpyAsync(d_inverse, srt.inverse.p, n * 4, cudaMemcpyDeviceToDevice, s));
  ctx->check_error(s);
  if (h_num_unique) *h_num_unique = u;
  FSX_API_END
}

int fsx_collision_split(fsx_ctx* ctx, const uint64_t* d_cur, uint64_t n_cur,
                        const uint64_t* d_next, uint64_t n_next, uint64_t* d_co,
                        uint64_t* d_ex_cur, uint64_t* d_ex_next, uint64_t* h_counts,
                        void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  cudaStream_t s = S(stream);
  DevBuf<uint64_t> ua(n_cur ? n_cur : 1), ub(n_next ? n_next : 1);
  uint64_t na = 0, nb = 0;
  if (n_cur) FSX_CHECK_RC(fsx_sort_unique_u64(ctx, d_cur, n_cur, ua.p, nullptr, &na, stream));
  if (n_next) FSX_CHECK_RC(fsx_sort_unique_u64(ctx, d_next, n_next, ub.p, nullptr, &nb, stream));
  DevBuf<uint64_t> cnt(8);
  uint64_t hc[2] = {na, nb};
  FSX_CUDA(cudaMemcpyAsync(cnt.p, hc, 16, cudaMemcpyHostToDevice, s));
  DevBuf<uint8_t> fa(na ? na : 1), fb(nb ? nb : 1);
  FSX_CUDA(cudaMemsetAsync(fb.p, 0, nb ? nb : 1, s));
  FSX_LAUNCH(ctx, k_intersect_flags, grid_for(ctx, na, 256, 8), 256, 0, s, ua.p, cnt.p, ub.p,
             cnt.p + 1, fa.p, fb.p, nullptr);
  ScanScratch sc;
  SplitByFlagOp opa{ua.p, fa.p, d_co, d_ex_cur};
  run_scan(ctx, opa, na, cnt.p, sc, cnt.p + 2, s);
  SplitByFlagOp opb{ub.p, fb.p, nullptr, d_ex_next};
  run_scan(ctx, opb, nb, cnt.p + 1, sc, cnt.p + 4, s);
  uint64_t t[6] = {0, 0, 0, 0, 0, 0};
  FSX_CUDA(cudaMemcpyAsync(t, cnt.p, 48, cudaMemcpyDeviceToHost, s));
  ctx->check_error(s);
  if (na == 0) t[2] = t[3] = 0;
  if (nb == 0) t[4] = t[5] = 0;
  h_counts[0] = t[2];
  h_counts[1] = t[3];
  h_counts[2] = t[5];
  h_counts[3] = na;
  h_counts[4] = nb;
  FSX_API_END
}

int fsx_route_by_owner(fsx_ctx* ctx, const uint64_t* d_ids, uint64_t n, uint64_t total_rows,
                       int num_shards, uint64_t* d_send_ids, uint32_t* d_send_pos,
                       uint64_t* h_send_counts, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  cudaStream_t s = S(stream);
  if (num_shards < 1 || num_shards > 16)
    raise(FSX_ERR_INVALID_ARGUMENT, "fsx: route_by_owner supports 1..16 shards");
  DevBuf<uint64_t> tot(16);
  FSX_CUDA(cudaMemsetAsync(tot.p, 0, 16 * 8, s));
  ScanScratch sc;
  if (num_shards <= 8) {
    OwnerPartitionOp<8> op{d_ids, total_rows, num_shards, tot.p, d_send_ids, d_send_pos, ctx->d_err};
    run_scan(ctx, op, n, nullptr, sc, tot.p, s);
  } else {
    OwnerPartitionOp<16> op{d_ids, total_rows, num_shards, tot.p, d_send_ids, d_send_pos, ctx->d_err};
    run_scan(ctx, op, n, nullptr, sc, tot.p, s);
  }
  uint64_t h[16];
  FSX_CUDA(cudaMemcpyAsync(h, tot.p, 16 * 8, cudaMemcpyDeviceToHost, s));
  try {
    ctx->check_error(s);
  } catch (const Error&) {
    std::vector<uint64_t> hid(n);
    if (n) FSX_CUDA(cudaMemcpy(hid.data(), d_ids, n * 8, cudaMemcpyDeviceToHost));
    for (uint64_t id : hid)
      if (id >= total_rows)
        raise(FSX_ERR_DOMAIN, "embedding: row id " + std::to_string(id) +
                                  " out of range (table has " + std::to_string(total_rows) + " rows)");
    throw;
  }
  for (int q = 0; q < num_shards; ++q) h_send_counts[q] = h[q];
  FSX_API_END
}

// ---- table ---------------------------------------------------------------------
int fsx_table_create(fsx_ctx* ctx, uint64_t total_rows, uint32_t dim, int num_shards, int shard,
                     double learning_rate, uint64_t seed, int dtype, fsx_table** out) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  if (num_shards < 1 || shard < 0 || shard >= num_shards)
    raise(FSX_ERR_INVALID_ARGUMENT, "embedding: shard id out of range");
  if (dim < 1) raise(FSX_ERR_INVALID_ARGUMENT, "embedding: dim must be >= 1");
  if (dtype != FSX_F32 && dtype != FSX_F64) raise(FSX_ERR_INVALID_ARGUMENT, "fsx: bad dtype");
  auto t = std::make_unique<fsx_table>();
  t->ctx = ctx;
  const uint64_t s = static_cast<uint64_t>(shard);
  const uint64_t local = total_rows > s ? (total_rows - 1 - s) / static_cast<uint64_t>(num_shards) + 1 : 0;
  t->g = ShardGeom{total_rows, local, dim, num_shards, shard};
  t->dtype = dtype;
  t->elem = dtype == FSX_F32 ? 4 : 8;
  t->lr = learning_rate;
  t->seed = seed;
  const size_t bytes = std::max<size_t>(local * dim * t->elem, 16);
  FSX_CUDA(cudaMalloc(&t->values, bytes));
  if (local) {
    const unsigned grid = grid_for(ctx, local, 8, 32);
    if (dtype == FSX_F32)
      FSX_LAUNCH(ctx, k_init_table<float>, grid, 256, 0, nullptr, static_cast<float*>(t->values), t->g, seed);
    else
      FSX_LAUNCH(ctx, k_init_table<double>, grid, 256, 0, nullptr, static_cast<double*>(t->values), t->g, seed);
  }
  FSX_CUDA(cudaDeviceSynchronize());
  *out = t.release();
  FSX_API_END
}

int fsx_table_destroy(fsx_table* t) {
  FSX_API_BEGIN
  if (!t) return FSX_OK;
  DeviceGuard dg(t->ctx->device);
  delete t;
  FSX_API_END
}

uint64_t fsx_table_local_rows(const fsx_table* t) { return t ? t->g.local_rows : 0; }
void* fsx_table_values(fsx_table* t) { return t ? t->values : nullptr; }

int fsx_table_gather(fsx_table* t, const uint64_t* d_ids, uint64_t n, void* d_out, void* stream,
                     int sync) {
  FSX_API_BEGIN
  DeviceGuard dg(t->ctx->device);
  cudaStream_t s = S(stream);
  GatherByIdMap m{static_cast<const char*>(t->values), d_ids, static_cast<char*>(d_out),
                  t->row_bytes(), t->g, t->ctx->d_err};
  launch_copy_rows(t->ctx, m, n, nullptr, t->row_bytes(), s);
  if (sync) {
    try {
      t->ctx->check_error(s);
    } catch (const Error&) {
      raise_first_bad(*t, d_ids, n, false);
      throw;
    }
  }
  FSX_API_END
}

int fsx_table_sgd_update(fsx_table* t, const uint64_t* d_ids, uint64_t n, const void* d_grads,
                         uint64_t* d_unique, void* d_rows, uint64_t* h_num_unique, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(t->ctx->device);
  if (n == 0) {
    if (h_num_unique) *h_num_unique = 0;
    return FSX_OK;
  }
  if (t->dtype == FSX_F32)
    table_sgd<float>(*t, d_ids, n, d_grads, d_unique, d_rows, h_num_unique, S(stream));
  else
    table_sgd<double>(*t, d_ids, n, d_grads, d_unique, d_rows, h_num_unique, S(stream));
  FSX_API_END
}

int fsx_table_download(fsx_table* t, double* h_values) {
  FSX_API_BEGIN
  DeviceGuard dg(t->ctx->device);
  const uint64_t n = t->g.local_rows * t->g.dim;
  if (n == 0) return FSX_OK;
  FSX_CUDA(cudaDeviceSynchronize());
  if (t->dtype == FSX_F64) {
    FSX_CUDA(cudaMemcpy(h_values, t->values, n * 8, cudaMemcpyDeviceToHost));
  } else {
    std::vector<float> tmp(n);
    FSX_CUDA(cudaMemcpy(tmp.data(), t->values, n * 4, cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < n; ++i) h_values[i] = static_cast<double>(tmp[i]);
  }
  FSX_API_END
}

int fsx_table_upload(fsx_table* t, const double* h_values) {
  FSX_API_BEGIN
  DeviceGuard dg(t->ctx->device);
  const uint64_t n = t->g.local_rows * t->g.dim;
  if (n == 0) return FSX_OK;
  FSX_CUDA(cudaDeviceSynchronize());
  if (t->dtype == FSX_F64) {
    FSX_CUDA(cudaMemcpy(t->values, h_values, n * 8, cudaMemcpyHostToDevice));
  } else {
    std::vector<float> tmp(n);
    for (uint64_t i = 0; i < n; ++i) tmp[i] = static_cast<float>(h_values[i]);
    FSX_CUDA(cudaMemcpy(t->values, tmp.data(), n * 4, cudaMemcpyHostToDevice));
  }
  FSX_API_END
}

}  // extern "C"
