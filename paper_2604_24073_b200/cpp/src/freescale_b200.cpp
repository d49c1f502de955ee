// The reference's C++ API (drop-in headers under cpp/include/freescale/)
// implemented over libfsx's C ABI (include/fsx.h). Host vectors cross the
// boundary only where the reference API returns them by value; all hot-path
// work runs in libfsx's sm_100a kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <limits>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>

#include "freescale/embedding.hpp"
#include "freescale/partition.hpp"
#include "fsx.h"

namespace freescale {

[[noreturn]] void throw_fsx_status(int code) {
  const std::string msg = fsx_last_error();
  switch (code) {
    case FSX_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case FSX_ERR_DOMAIN: throw std::domain_error(msg);
    case FSX_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case FSX_ERR_PROTOCOL: throw ProtocolError(msg);
    case FSX_ERR_COLLECTIVE: throw CollectiveError(msg);
    case FSX_ERR_CONFIG: throw ConfigError(msg);
    case FSX_ERR_IO: throw IoError(msg);
    default: throw std::runtime_error(msg);
  }
}

namespace {

void cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + cudaGetErrorString(e));
}

template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  Dev() = default;
  explicit Dev(size_t count) { alloc(count); }
  ~Dev() { if (p) cudaFree(p); }
  void alloc(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    if (count) cuda_ok(cudaMalloc(&p, count * sizeof(T)));
  }
  void ensure(size_t count) { if (count > n) alloc(count); }
};

template <class T>
void h2d(T* d, const T* h, size_t n) {
  if (n) cuda_ok(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice));
}
template <class T>
void d2h(T* h, const T* d, size_t n) {
  if (n) cuda_ok(cudaMemcpy(h, d, n * sizeof(T), cudaMemcpyDeviceToHost));
}

// one context per (thread's current device) for the free functions
fsx_ctx* thread_ctx() {
  thread_local fsx_ctx* ctx = nullptr;
  thread_local int dev = -1;
  int cur = 0;
  cuda_ok(cudaGetDevice(&cur));
  if (!ctx || dev != cur) {
    fsx_ok(fsx_ctx_create(cur, 0, 1, &ctx));
    dev = cur;
  }
  return ctx;
}

std::vector<std::uint64_t> sorted_unique_dev(const std::vector<std::uint64_t>& v) {
  if (v.empty()) return {};
  Dev<std::uint64_t> d(v.size()), u(v.size());
  h2d(d.p, v.data(), v.size());
  std::uint64_t nu = 0;
  fsx_ok(fsx_sort_unique_u64(thread_ctx(), d.p, v.size(), u.p, nullptr, &nu, nullptr));
  std::vector<std::uint64_t> out(nu);
  d2h(out.data(), u.p, nu);
  return out;
}

}  // namespace

// ---- jagged reshuffle (jagged.hpp) ----------------------------------------------------
namespace jagged_detail {

void permute(const void* values, std::size_t elem_bytes, std::span<const std::size_t> lengths,
             std::span<const std::size_t> perm, std::vector<unsigned char>& out_values,
             std::vector<std::size_t>& out_lengths) {
  const std::size_t nseg = lengths.size(), np = perm.size();
  // the reference validates every index before moving anything
  for (std::size_t idx : perm)
    if (idx >= nseg)
      throw std::out_of_range("indexed_permute: segment index " + std::to_string(idx) + " out of range (have " +
                              std::to_string(nseg) + ")");
  out_lengths.assign(np, 0);
  out_values.clear();
  if (np == 0) return;
  fsx_ctx* ctx = thread_ctx();
  std::vector<std::uint64_t> h_len(lengths.begin(), lengths.end()), h_perm(perm.begin(), perm.end());
  std::uint64_t total_in = 0;
  for (auto l : h_len) total_in += l;
  Dev<std::uint64_t> d_len(nseg + 1), d_off(nseg + 1), d_perm(np), d_olen(np), d_ooff(np + 1);
  Dev<unsigned char> d_vals(total_in * elem_bytes + 16);
  h2d(d_len.p, h_len.data(), nseg);
  h2d(d_perm.p, h_perm.data(), np);
  if (total_in) h2d(d_vals.p, static_cast<const unsigned char*>(values), total_in * elem_bytes);
  std::uint64_t tot = 0;
  fsx_ok(fsx_jagged_offsets(ctx, d_len.p, nseg, d_off.p, &tot, nullptr));
  std::uint64_t out_total = 0;
  fsx_ok(fsx_jagged_permute(ctx, d_vals.p, static_cast<std::uint32_t>(elem_bytes), d_off.p, nseg, d_perm.p, np,
                            nullptr, 0, d_olen.p, d_ooff.p, &out_total, nullptr));  // sizing
  Dev<unsigned char> d_out(out_total * elem_bytes + 16);
  fsx_ok(fsx_jagged_permute(ctx, d_vals.p, static_cast<std::uint32_t>(elem_bytes), d_off.p, nseg, d_perm.p, np,
                            d_out.p, out_total, d_olen.p, d_ooff.p, &out_total, nullptr));
  std::vector<std::uint64_t> olen(np);
  d2h(olen.data(), d_olen.p, np);
  out_lengths.assign(olen.begin(), olen.end());
  out_values.resize(out_total * elem_bytes);
  if (out_total) d2h(out_values.data(), d_out.p, out_values.size());
}

std::vector<std::size_t> transpose_perm(std::size_t num_keys, std::size_t num_samples, bool feature_major) {
  const std::size_t n = num_keys * num_samples;
  std::vector<std::size_t> perm(n);
  if (n == 0) return perm;
  Dev<std::uint64_t> d(n);
  fsx_ok(fsx_keyed_transpose_perm(thread_ctx(), num_keys, num_samples, feature_major ? 1 : 0, d.p, nullptr));
  std::vector<std::uint64_t> h(n);
  d2h(h.data(), d.p, n);
  perm.assign(h.begin(), h.end());
  return perm;
}

}  // namespace jagged_detail

// ---- embedding -----------------------------------------------------------------------
namespace embedding {

// embedding.cpp:59-64 restated (a pure host function of the API)
double initial_value(std::uint64_t seed, std::uint64_t row, std::uint32_t d) {
  auto mix = [](std::uint64_t& s) {
    s += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  std::uint64_t st = seed + row * 0x9e3779b97f4a7c15ULL + (static_cast<std::uint64_t>(d) + 1) * 0xbf58476d1ce4e5b9ULL;
  mix(st);
  const double u = static_cast<double>(mix(st) >> 11) * 0x1.0p-53;
  return (u - 0.5) * 0.2;
}

IndexSet IndexSet::batch_major(IdJagged ids) {
  IndexSet s;
  s.layout = IndexLayout::BatchMajor;
  s.unique_ids = sorted_unique_dev(ids.values());
  s.ids = std::move(ids);
  return s;
}

IndexSet IndexSet::shard_major(IdJagged ids) {
  IndexSet s = batch_major(std::move(ids));
  s.layout = IndexLayout::ShardMajor;
  return s;
}

CollisionSplit compute_collision(const IndexSet& cur, const IndexSet& next) {
  if (cur.layout != IndexLayout::ShardMajor || next.layout != IndexLayout::ShardMajor)
    throw std::invalid_argument("compute_collision: both index sets must be shard-major");
  const auto& a = cur.unique_ids;
  const auto& b = next.unique_ids;
  Dev<std::uint64_t> da(a.size() + 1), db(b.size() + 1), co(a.size() + 1), ec(a.size() + 1), en(b.size() + 1);
  h2d(da.p, a.data(), a.size());
  h2d(db.p, b.data(), b.size());
  std::uint64_t cnt[5] = {};
  fsx_ok(fsx_collision_split(thread_ctx(), da.p, a.size(), db.p, b.size(), co.p, ec.p, en.p, cnt, nullptr));
  CollisionSplit s;
  s.collision.resize(cnt[0]);
  s.exclusive_cur.resize(cnt[1]);
  s.exclusive_next.resize(cnt[2]);
  d2h(s.collision.data(), co.p, cnt[0]);
  d2h(s.exclusive_cur.data(), ec.p, cnt[1]);
  d2h(s.exclusive_next.data(), en.p, cnt[2]);
  return s;
}

double collision_pct(const IndexSet& cur, const IndexSet& next) {
  if (cur.layout != IndexLayout::ShardMajor || next.layout != IndexLayout::ShardMajor)
    throw std::invalid_argument("collision_pct: both index sets must be shard-major");
  if (next.unique_ids.empty()) throw std::invalid_argument("collision_pct: next iteration uses no rows");
  return static_cast<double>(compute_collision(cur, next).collision.size()) /
         static_cast<double>(next.unique_ids.size());
}

ShardView::ShardView(TableGeometry geom, int shard_id, double lr, std::uint64_t seed)
    : geom_(geom), shard_(shard_id), lr_(lr) {
  int dev = 0;
  cuda_ok(cudaGetDevice(&dev));
  fsx_ok(fsx_ctx_create(dev, shard_id, geom.num_shards, &ctx_));
  own_ctx_ = true;
  fsx_ok(fsx_table_create(ctx_, geom.total_rows, geom.dim, geom.num_shards, shard_id, lr, seed, FSX_F64, &table_));
}

ShardView::~ShardView() {
  if (table_) fsx_table_destroy(table_);
  if (own_ctx_) fsx_ctx_destroy(ctx_);
}

const std::vector<double>& ShardView::values() const {
  mirror_.resize(local_rows() * geom_.dim);
  fsx_ok(fsx_table_download(table_, mirror_.data()));
  return mirror_;
}

std::span<const double> ShardView::row(std::uint64_t g) const {
  if (g >= geom_.total_rows)
    throw std::domain_error("embedding: row id " + std::to_string(g) + " out of range (table has " +
                            std::to_string(geom_.total_rows) + " rows)");
  if (geom_.owner(g) != shard_)
    throw std::domain_error("embedding: row id " + std::to_string(g) + " is not owned by shard " +
                            std::to_string(shard_));
  const auto& v = values();
  return std::span<const double>(v.data() + geom_.local_index(g) * geom_.dim, geom_.dim);
}

std::vector<double> ShardView::lookup(std::span<const std::uint64_t> ids) const {
  std::vector<double> out(ids.size() * geom_.dim);
  if (ids.empty()) return out;
  Dev<std::uint64_t> d(ids.size());
  Dev<double> o(out.size());
  h2d(d.p, ids.data(), ids.size());
  fsx_ok(fsx_table_gather(table_, d.p, ids.size(), o.p, nullptr, 1));
  d2h(out.data(), o.p, out.size());
  return out;
}

ShardView::UpdateResult ShardView::apply_gradients(std::span<const std::uint64_t> ids,
                                                   std::span<const double> grads) {
  const std::uint32_t dim = geom_.dim;
  if (grads.size() != ids.size() * dim)
    throw std::invalid_argument("embedding: gradient shape " + std::to_string(grads.size()) +
                                " misaligned with " + std::to_string(ids.size()) + " ids x dim " +
                                std::to_string(dim));
  UpdateResult res;
  if (ids.empty()) return res;
  Dev<std::uint64_t> d(ids.size()), u(ids.size());
  Dev<double> g(grads.size()), rows(grads.size());
  h2d(d.p, ids.data(), ids.size());
  h2d(g.p, grads.data(), grads.size());
  std::uint64_t nu = 0;
  fsx_ok(fsx_table_sgd_update(table_, d.p, ids.size(), g.p, u.p, rows.p, &nu, nullptr));
  res.unique_ids.resize(nu);
  res.rows.resize(nu * dim);
  d2h(res.unique_ids.data(), u.p, nu);
  d2h(res.rows.data(), rows.p, nu * dim);
  return res;
}

// ---- engines --------------------------------------------------------------------------
EngineBase::EngineBase(ShardView& shard, comm::Communicator& comm, int mode) : shard_(shard), comm_(comm) {
  if (comm.world_size() != shard.geometry().num_shards || comm.rank() != shard.shard_id())
    throw std::invalid_argument("embedding: shard geometry does not match the communicator");
  cuda_ok(cudaStreamCreateWithFlags(reinterpret_cast<cudaStream_t*>(&stream_), cudaStreamNonBlocking));
  mode_ = mode;
}

EngineBase::~EngineBase() {
  if (eng_) fsx_engine_destroy(eng_);
  cudaFree(d_ids_);
  cudaFree(d_next_);
  cudaFree(d_rows_);
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
}

void EngineBase::ensure(std::size_t n) {
  if (eng_) {
    if (n > cap_)
      throw std::invalid_argument("embedding: batch of " + std::to_string(n) +
                                  " ids exceeds the engine capacity " + std::to_string(cap_));
    return;
  }
  // Lazy, collective creation on the first forward: every rank agrees on one
  // capacity (identical receive-window layouts), then wires its peers.
  const int mode = mode_;
  std::vector<std::uint8_t> mine(8);
  const std::uint64_t want = std::max<std::uint64_t>(4 * n + 1024, 1 << 16);
  std::memcpy(mine.data(), &want, 8);
  auto& fab = comm_.transport().fabric();
  std::uint64_t cap = 0;
  for (const auto& b : fab.exchange(comm_.rank(), mine)) {
    std::uint64_t v = 0;
    std::memcpy(&v, b.data(), 8);
    cap = std::max(cap, v);
  }
  cap_ = cap;
  fsx_engine_config cfg{mode, FSX_TRANSPORT_CE, cap_, 0, 0};
  fsx_ok(fsx_engine_create(shard_.ctx(), shard_.handle(), &cfg, &eng_));
  std::vector<std::uint8_t> me(sizeof(void*));
  std::memcpy(me.data(), &eng_, sizeof(void*));
  const auto all = fab.exchange(comm_.rank(), me);
  for (int p = 0; p < comm_.world_size(); ++p) {
    if (p == comm_.rank()) continue;
    fsx_engine* other = nullptr;
    std::memcpy(&other, all[static_cast<size_t>(p)].data(), sizeof(void*));
    fsx_ok(fsx_engine_connect_local(eng_, p, other));
  }
  fab.exchange(comm_.rank(), {});
  cuda_ok(cudaMalloc(&d_ids_, cap_ * 8));
  cuda_ok(cudaMalloc(&d_next_, cap_ * 8));
  cuda_ok(cudaMalloc(&d_rows_, cap_ * shard_.geometry().dim * 8));
}

std::vector<double> EngineBase::run_forward(const IdJagged& cur, const IdJagged* next) {
  const auto& c = cur.values();
  ensure(std::max<std::size_t>(c.size(), next ? next->values().size() : 0));
  auto s = static_cast<cudaStream_t>(stream_);
  if (!c.empty()) cuda_ok(cudaMemcpyAsync(d_ids_, c.data(), c.size() * 8, cudaMemcpyHostToDevice, s));
  if (next && !next->values().empty())
    cuda_ok(cudaMemcpyAsync(d_next_, next->values().data(), next->values().size() * 8, cudaMemcpyHostToDevice, s));
  fsx_ok(fsx_engine_forward(eng_, d_ids_, c.size(), next ? d_next_ : nullptr, next ? next->values().size() : 0,
                            d_rows_, s));
  std::vector<double> out(c.size() * shard_.geometry().dim);
  if (!out.empty()) cuda_ok(cudaMemcpyAsync(out.data(), d_rows_, out.size() * 8, cudaMemcpyDeviceToHost, s));
  cuda_ok(cudaStreamSynchronize(s));
  fsx_ok(fsx_ctx_sync(shard_.ctx()));
  n_cur_ = c.size();
  have_cur_ = true;
  return out;
}

void EngineBase::run_backward(std::span<const double> grads) {
  if (!have_cur_) throw ProtocolError("embedding: backward before forward");
  if (grads.size() != n_cur_ * shard_.geometry().dim)
    throw std::invalid_argument("embedding: gradient count does not match forward occurrences");
  auto s = static_cast<cudaStream_t>(stream_);
  if (!grads.empty()) cuda_ok(cudaMemcpyAsync(d_rows_, grads.data(), grads.size() * 8, cudaMemcpyHostToDevice, s));
  fsx_ok(fsx_engine_backward(eng_, d_rows_, s));
  cuda_ok(cudaStreamSynchronize(s));
  have_cur_ = false;
}

SynchronizedEmbedding::SynchronizedEmbedding(ShardView& shard, comm::Communicator& comm)
    : EngineBase(shard, comm, FSX_MODE_SYNC) {}

std::vector<double> SynchronizedEmbedding::forward(const IdJagged& ids) { return run_forward(ids, nullptr); }
void SynchronizedEmbedding::backward(std::span<const double> grads) { run_backward(grads); }

PrioritizedEmbedding::PrioritizedEmbedding(ShardView& shard, comm::Communicator& comm, comm::CollectiveMode)
    : EngineBase(shard, comm, FSX_MODE_PRIO) {}

std::vector<double> PrioritizedEmbedding::forward(const IdJagged& cur, const IdJagged* next) {
  if (forward_done_) throw ProtocolError("embedding: forward called twice in one iteration");
  auto out = run_forward(cur, next);
  forward_done_ = true;
  ++iters_;
  return out;
}

void PrioritizedEmbedding::backward(std::span<const double> grads) {
  if (!forward_done_) throw ProtocolError("embedding: backward before forward");
  run_backward(grads);
  forward_done_ = false;
}

void PrioritizedEmbedding::finalize() {
  if (!eng_) return;
  auto s = static_cast<cudaStream_t>(stream_);
  fsx_ok(fsx_engine_finalize(eng_, s));
  cuda_ok(cudaStreamSynchronize(s));
  fsx_ok(fsx_ctx_sync(shard_.ctx()));
}

const std::vector<IterationStats>& PrioritizedEmbedding::stats() const {
  stats_.clear();
  for (int i = 0; i < iters_; ++i) {
    std::uint64_t v[3] = {};
    fsx_ok(fsx_engine_stats(eng_, i, v));
    IterationStats st{v[0], v[1], v[2], v[1] ? static_cast<double>(v[0]) / static_cast<double>(v[1]) : 0.0};
    stats_.push_back(st);
  }
  return stats_;
}

std::vector<double> gather_full_table(comm::Communicator& comm, const ShardView& shard) {
  const auto& geom = shard.geometry();
  const auto& v = shard.values();
  std::vector<std::uint8_t> mine(v.size() * 8);
  if (!v.empty()) std::memcpy(mine.data(), v.data(), mine.size());
  auto parts = comm.transport().fabric().exchange(comm.rank(), std::move(mine));
  std::vector<double> full(geom.total_rows * geom.dim);
  for (int s = 0; s < geom.num_shards; ++s) {
    const auto& b = parts[static_cast<size_t>(s)];
    const std::uint64_t rows = geom.local_rows(s);
    if (b.size() != rows * geom.dim * 8)
      throw ProtocolError("embedding: shard " + std::to_string(s) + " checkpoint size mismatch");
    for (std::uint64_t l = 0; l < rows; ++l)
      std::memcpy(full.data() + (s + l * geom.num_shards) * geom.dim, b.data() + l * geom.dim * 8, geom.dim * 8);
  }
  return full;
}

std::vector<std::uint8_t> checkpoint_bytes(const TableGeometry& geom, std::span<const double> t) {
  std::vector<std::uint8_t> out(24 + t.size() * 8);
  const std::uint64_t h[3] = {geom.total_rows, geom.dim, static_cast<std::uint64_t>(geom.num_shards)};
  std::memcpy(out.data(), h, 24);
  if (!t.empty()) std::memcpy(out.data() + 24, t.data(), t.size() * 8);
  return out;
}

// ---- routing (embedding.cpp:185-231) ---------------------------------------------------
ShardRouting route_to_shard_major(comm::Communicator& comm, const TableGeometry& geom, const IdJagged& batch_ids,
                                  const comm::CollectiveOptions& opts) {
  const int p = comm.world_size();
  ShardRouting r;
  r.batch_ids = batch_ids;
  const auto& flat = batch_ids.values();
  const std::size_t n = flat.size();
  r.occ_shard.resize(n);
  r.send_positions.resize(static_cast<std::size_t>(p));
  r.send_ids.resize(static_cast<std::size_t>(p));
  r.unique_per_shard.resize(static_cast<std::size_t>(p));
  fsx_ctx* ctx = comm.transport().ctx() ? comm.transport().ctx() : thread_ctx();
  if (n) {
    // stable owner partition on the GPU; range errors raise the reference's text
    Dev<std::uint64_t> d_ids(n), d_send(n);
    Dev<std::uint32_t> d_pos(n);
    h2d(d_ids.p, flat.data(), n);
    std::vector<std::uint64_t> counts(static_cast<std::size_t>(p));
    fsx_ok(fsx_route_by_owner(ctx, d_ids.p, n, geom.total_rows, p, d_send.p, d_pos.p, counts.data(), nullptr));
    std::vector<std::uint64_t> send(n);
    std::vector<std::uint32_t> pos(n);
    d2h(send.data(), d_send.p, n);
    d2h(pos.data(), d_pos.p, n);
    std::size_t at = 0;
    for (int s = 0; s < p; ++s) {
      const std::size_t c = counts[static_cast<std::size_t>(s)];
      auto& sp = r.send_positions[static_cast<std::size_t>(s)];
      auto& si = r.send_ids[static_cast<std::size_t>(s)];
      sp.assign(pos.begin() + static_cast<std::ptrdiff_t>(at), pos.begin() + static_cast<std::ptrdiff_t>(at + c));
      si.assign(send.begin() + static_cast<std::ptrdiff_t>(at), send.begin() + static_cast<std::ptrdiff_t>(at + c));
      for (std::size_t q : sp) r.occ_shard[q] = s;
      r.unique_per_shard[static_cast<std::size_t>(s)] = sorted_unique_dev(si);
      at += c;
    }
  }
  std::vector<comm::Bytes> payloads(static_cast<std::size_t>(p));
  for (int s = 0; s < p; ++s) payloads[static_cast<std::size_t>(s)] = comm::pack_u64s(r.send_ids[static_cast<std::size_t>(s)]);
  const auto got = comm.all_to_all(payloads, opts);
  std::vector<std::uint64_t> values;
  std::vector<std::size_t> lengths(static_cast<std::size_t>(p));
  r.recv_unique_per_src.resize(static_cast<std::size_t>(p));
  for (int src = 0; src < p; ++src) {
    const auto ids = comm::unpack_u64s(got[static_cast<std::size_t>(src)]);
    for (std::uint64_t id : ids)
      if (geom.owner(id) != comm.rank())
        throw ProtocolError("embedding: received row " + std::to_string(id) + " that this shard does not own");
    lengths[static_cast<std::size_t>(src)] = ids.size();
    r.recv_unique_per_src[static_cast<std::size_t>(src)] = sorted_unique_dev(ids);
    values.insert(values.end(), ids.begin(), ids.end());
  }
  r.shard_ids = IndexSet::shard_major(IdJagged(std::move(values), std::move(lengths)));
  return r;
}

}  // namespace embedding

// ---- partition / sim --------------------------------------------------------------------
namespace partition {

namespace {
void unpack(std::span<const GlobalSampleMeta> metas, std::vector<std::uint64_t>& l, std::vector<int32_t>& o,
            std::vector<int32_t>& x) {
  for (const auto& m : metas) {
    l.push_back(m.uih_len);
    o.push_back(m.origin_rank);
    x.push_back(m.local_index);
  }
}
PartitionPlan make_plan(int n, const std::vector<int32_t>& a, const std::vector<std::uint64_t>& order,
                        const std::vector<std::size_t>& sizes) {
  PartitionPlan p;
  p.num_ranks = n;
  p.assignment.assign(a.begin(), a.end());
  std::size_t at = 0;
  for (std::size_t s : sizes) {
    p.receive_order.emplace_back(order.begin() + static_cast<std::ptrdiff_t>(at),
                                 order.begin() + static_cast<std::ptrdiff_t>(at + s));
    at += s;
  }
  return p;
}
}  // namespace

std::vector<std::vector<std::vector<int>>> PartitionPlan::exchange_lists(std::span<const GlobalSampleMeta> metas) const {
  std::vector<std::vector<std::vector<int>>> lists(static_cast<size_t>(num_ranks),
                                                   std::vector<std::vector<int>>(static_cast<size_t>(num_ranks)));
  for (int dst = 0; dst < num_ranks; ++dst)
    for (std::size_t g : receive_order[static_cast<size_t>(dst)])
      lists[static_cast<size_t>(metas[g].origin_rank)][static_cast<size_t>(dst)].push_back(metas[g].local_index);
  return lists;
}

void PartitionPlan::validate(std::size_t num_samples, bool fixed_batch) const {
  if (num_ranks < 1) throw std::invalid_argument("partition plan: num_ranks < 1");
  if (assignment.size() != num_samples)
    throw std::invalid_argument("partition plan: assignment covers " + std::to_string(assignment.size()) +
                                " samples, expected " + std::to_string(num_samples) + " (samples lost or duplicated)");
  if (receive_order.size() != static_cast<std::size_t>(num_ranks))
    throw std::invalid_argument("partition plan: receive_order must have one list per rank");
  std::vector<int> seen(num_samples, 0);
  for (int r = 0; r < num_ranks; ++r)
    for (std::size_t g : receive_order[static_cast<size_t>(r)]) {
      if (g >= num_samples) throw std::invalid_argument("partition plan: sample index " + std::to_string(g) + " out of range");
      if (assignment[g] != r)
        throw std::invalid_argument("partition plan: sample " + std::to_string(g) + " listed under rank " +
                                    std::to_string(r) + " but assigned to rank " + std::to_string(assignment[g]));
      if (++seen[g] > 1) throw std::invalid_argument("partition plan: sample " + std::to_string(g) + " assigned more than once");
    }
  for (std::size_t g = 0; g < num_samples; ++g)
    if (!seen[g]) throw std::invalid_argument("partition plan: sample " + std::to_string(g) + " not assigned to any rank");
  if (fixed_batch && num_samples % static_cast<std::size_t>(num_ranks) == 0) {
    const std::size_t per = num_samples / static_cast<std::size_t>(num_ranks);
    for (int r = 0; r < num_ranks; ++r)
      if (receive_order[static_cast<size_t>(r)].size() != per)
        throw std::invalid_argument("partition plan: rank " + std::to_string(r) + " receives " +
                                    std::to_string(receive_order[static_cast<size_t>(r)].size()) +
                                    " samples, expected " + std::to_string(per));
  }
}

PartitionPlan fbs_partition(std::span<const GlobalSampleMeta> metas, int n) {
  std::vector<std::uint64_t> l;
  std::vector<int32_t> o, x;
  unpack(metas, l, o, x);
  std::vector<int32_t> a(metas.size());
  std::vector<std::uint64_t> order(metas.size());
  fsx_ok(fsx_fbs_partition(thread_ctx(), l.data(), o.data(), x.data(), metas.size(), n, a.data(), order.data(), nullptr));
  return make_plan(n, a, order, std::vector<std::size_t>(static_cast<size_t>(n), metas.size() / static_cast<size_t>(n)));
}

PartitionPlan vbs_partition(std::span<const GlobalSampleMeta> metas, int n, double alpha, AutoTuneState* tune) {
  std::vector<std::uint64_t> l;
  std::vector<int32_t> o, x;
  unpack(metas, l, o, x);
  const std::size_t m = metas.size();
  const bool tuned = tune && tune->initialized && tune->local_batch_size.size() == static_cast<size_t>(n) &&
                     std::accumulate(tune->local_batch_size.begin(), tune->local_batch_size.end(), std::size_t{0},
                                     [](std::size_t a, int b) { return a + static_cast<std::size_t>(b); }) == m;
  std::vector<int32_t> ts, sizes(static_cast<size_t>(std::max(n, 1))), a(std::max<std::size_t>(m, 1));
  std::vector<std::uint64_t> order(std::max<std::size_t>(m, 1));
  if (tuned) ts.assign(tune->local_batch_size.begin(), tune->local_batch_size.end());
  fsx_ok(fsx_vbs_partition(thread_ctx(), l.data(), o.data(), x.data(), m, n, alpha, tuned ? ts.data() : nullptr,
                           sizes.data(), a.data(), order.data(), nullptr));
  if (tune && !tuned) {
    tune->local_batch_size.assign(sizes.begin(), sizes.begin() + n);
    tune->ema_local.assign(static_cast<size_t>(n), 0.0);
    tune->ema_global = 0.0;
    tune->initialized = true;
  }
  a.resize(m);
  order.resize(m);
  return make_plan(n, a, order, std::vector<std::size_t>(sizes.begin(), sizes.begin() + n));
}

void autotune_update(AutoTuneState& tune, std::span<const double> times) {
  if (!tune.initialized) throw ProtocolError("autotune: state not initialized");
  const auto n = tune.local_batch_size.size();
  if (times.size() != n)
    throw std::invalid_argument("autotune: expected " + std::to_string(n) + " times, got " + std::to_string(times.size()));
  std::vector<int32_t> s(tune.local_batch_size.begin(), tune.local_batch_size.end());
  fsx_ok(fsx_autotune_update(static_cast<int>(n), s.data(), tune.ema_local.data(), &tune.ema_global, tune.step,
                             tune.delta, tune.decay, times.data()));
  tune.local_batch_size.assign(s.begin(), s.end());
}

PartitionPlan identity_partition(std::span<const GlobalSampleMeta> metas, int n) {
  std::vector<std::vector<std::size_t>> order(static_cast<size_t>(n));
  for (std::size_t g = 0; g < metas.size(); ++g) order[static_cast<size_t>(metas[g].origin_rank)].push_back(g);
  for (auto& o : order)
    std::sort(o.begin(), o.end(), [&](std::size_t a, std::size_t b) { return metas[a].local_index < metas[b].local_index; });
  PartitionPlan p;
  p.num_ranks = n;
  p.assignment.assign(metas.size(), -1);
  for (int r = 0; r < n; ++r)
    for (auto g : order[static_cast<size_t>(r)]) p.assignment[g] = r;
  p.receive_order = std::move(order);
  return p;
}

PartitionPlan custom_partition(const PartitionFn& fn, std::span<const GlobalSampleMeta> metas, int n) {
  PartitionPlan plan = fn(metas, n);
  plan.validate(metas.size(), false);
  return plan;
}

double plan_max_weight(const PartitionPlan& plan, std::span<const GlobalSampleMeta> metas, double alpha) {
  double mx = 0;
  for (const auto& o : plan.receive_order) {
    double w = 0;
    for (std::size_t g : o) w += std::pow(static_cast<double>(metas[g].uih_len), alpha);
    mx = std::max(mx, w);
  }
  return mx;
}

// Every split into `segments` non-empty contiguous runs (cut positions
// strictly increasing in (0, m)), the smallest maximum run sum; sequential
// prefix sums as the DP uses. Test oracle of vbs_partition's DP.
double min_max_contiguous_bruteforce(std::span<const double> weights, int segments) {
  const std::size_t m = weights.size();
  std::vector<double> prefix(m + 1, 0.0);
  for (std::size_t i = 0; i < m; ++i) prefix[i + 1] = prefix[i] + weights[i];
  if (segments == 1) return prefix[m];
  const std::size_t ncut = static_cast<std::size_t>(segments) - 1;
  std::vector<std::size_t> cut(ncut);
  double best = std::numeric_limits<double>::infinity();
  std::function<void(std::size_t, std::size_t)> place = [&](std::size_t k, std::size_t first) {
    if (k == ncut) {
      double worst = 0;
      std::size_t from = 0;
      for (std::size_t c : cut) {
        worst = std::max(worst, prefix[c] - prefix[from]);
        from = c;
      }
      best = std::min(best, std::max(worst, prefix[m] - prefix[from]));
      return;
    }
    for (std::size_t c = first; c + (ncut - k) <= m; ++c) {
      cut[k] = c;
      place(k + 1, c + 1);
    }
  };
  place(0, 1);
  return best;
}

}  // namespace partition

namespace sim {

std::vector<double> CostModel::compute_times(const std::vector<std::vector<std::uint64_t>>& batches) const {
  std::vector<std::uint64_t> flat, off{0};
  for (const auto& b : batches) {
    flat.insert(flat.end(), b.begin(), b.end());
    off.push_back(flat.size());
  }
  std::vector<double> out(batches.size());
  if (batches.empty()) return out;
  Dev<std::uint64_t> d(flat.size() + 1);
  h2d(d.p, flat.data(), flat.size());
  fsx_ok(fsx_cost_estimate(thread_ctx(), d.p, off.data(), static_cast<int>(batches.size()), c0, c1, c2, out.data(),
                           nullptr));
  return out;
}

}  // namespace sim
}  // namespace freescale
