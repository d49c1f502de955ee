// Rank fabric, copy-engine collectives and host metric helpers behind the
// drop-in headers comm.hpp / tcp.hpp / sim.hpp (reference: src/comm.cpp,
// src/tcp.cpp, src/sim.cpp). See comm.hpp for the B200 mapping.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <sstream>
#include <thread>

#include "freescale/comm.hpp"
#include "freescale/sim.hpp"
#include "freescale/tcp.hpp"
#include "fsx.h"

namespace freescale::comm {

namespace {

void cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + cudaGetErrorString(e));
}

std::uint64_t max_of(const std::vector<std::vector<std::uint8_t>>& blobs) {
  std::uint64_t m = 0;
  for (const auto& b : blobs) {
    std::uint64_t v = 0;
    if (b.size() >= 8) std::memcpy(&v, b.data(), 8);
    m = std::max(m, v);
  }
  return m;
}

std::vector<std::uint8_t> u64_blob(std::uint64_t v) {
  std::vector<std::uint8_t> b(8);
  std::memcpy(b.data(), &v, 8);
  return b;
}

}  // namespace

// A rank's copy-engine collective windows: a libfsx engine (blocking mode,
// 8-byte rows) whose IDS/GRADS/all-gather windows carry the Communicator's
// byte collectives, plus device staging. Grown collectively when a
// collective's agreed bound exceeds the slot.
struct CommWindows {
  fsx_table* table = nullptr;
  fsx_engine* eng = nullptr;
  std::uint64_t cap = 0;  // payload bytes per slot
  char* d_send = nullptr;
  char* d_recv = nullptr;
  cudaStream_t s = nullptr;

  ~CommWindows() { release(); }
  void release() {
    if (eng) fsx_engine_destroy(eng);
    if (table) fsx_table_destroy(table);
    if (d_send) cudaFree(d_send);
    if (d_recv) cudaFree(d_recv);
    if (s) cudaStreamDestroy(s);
    eng = nullptr;
    table = nullptr;
    d_send = d_recv = nullptr;
    s = nullptr;
    cap = 0;
  }

  // Collective: every rank passes its need; all agree on the max (the size
  // round) and, if it exceeds the slot, rebuild and rewire together.
  static std::uint64_t agree(Transport& t, std::uint64_t need) {
    InProcessFabric& fab = t.fabric();
    const std::uint64_t bound = max_of(fab.exchange(t.rank(), u64_blob(need)));
    CommWindows* w = t.windows();
    if (w && w->cap >= bound) return bound;
    std::uint64_t cap = 1 << 16;
    while (cap < bound) cap <<= 1;
    if (!w) {
      t.win_ = std::make_unique<CommWindows>();
      w = t.win_.get();
    }
    w->release();
    const int p = t.world_size(), me = t.rank();
    cuda_ok(cudaSetDevice(t.device()));
    fsx_ok(fsx_table_create(t.ctx(), static_cast<std::uint64_t>(p), 1, p, me, 0.0, 0, FSX_F64, &w->table));
    fsx_engine_config cfg{FSX_MODE_SYNC, FSX_TRANSPORT_CE, cap / 8, 0, 0};
    fsx_ok(fsx_engine_create(t.ctx(), w->table, &cfg, &w->eng));
    std::vector<std::uint8_t> me_ptr(sizeof(void*));
    std::memcpy(me_ptr.data(), &w->eng, sizeof(void*));
    const auto all = fab.exchange(me, me_ptr);
    for (int d = 0; d < p; ++d) {
      if (d == me) continue;
      fsx_engine* other = nullptr;
      std::memcpy(&other, all[static_cast<size_t>(d)].data(), sizeof(void*));
      fsx_ok(fsx_engine_connect_local(w->eng, d, other));
    }
    fab.exchange(me, {});  // every rank wired before the first transfer
    w->cap = cap;
    cuda_ok(cudaMalloc(&w->d_send, static_cast<size_t>(p) * cap));
    cuda_ok(cudaMalloc(&w->d_recv, static_cast<size_t>(p) * cap));
    cuda_ok(cudaStreamCreateWithFlags(&w->s, cudaStreamNonBlocking));
    return bound;
  }
};

Transport::~Transport() = default;

InProcessFabric& Transport::fabric() const {
  if (!fabric_) throw ConfigError("comm: this transport is not part of an in-process fabric");
  return *fabric_;
}

void Transport::send(int dst, std::uint64_t tag, Bytes payload, double, CostClass) {
  if (dst < 0 || dst >= world_) throw CollectiveError("send: destination rank " + std::to_string(dst) + " out of range");
  fabric().post(rank_, dst, tag, std::move(payload));
}

Delivery Transport::recv(int src, std::uint64_t tag) {
  if (src < 0 || src >= world_) throw CollectiveError("recv: source rank " + std::to_string(src) + " out of range");
  return Delivery{fabric().take(src, rank_, tag), 0.0};
}

InProcessFabric::InProcessFabric(int world_size, LinkParams) : world_(world_size) {
  if (world_size < 1) throw std::invalid_argument("fabric: world_size must be >= 1");
  int ndev = 1;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) ndev = 1;
  for (int r = 0; r < world_size; ++r) {
    std::unique_ptr<Transport> t(new Transport());
    t->rank_ = r;
    t->world_ = world_size;
    t->device_ = r % ndev;
    t->fabric_ = this;
    fsx_ok(fsx_ctx_create(t->device_, r, world_size, &t->ctx_));
    eps_.push_back(std::move(t));
  }
}

InProcessFabric::~InProcessFabric() {
  for (auto& t : eps_) {
    t->win_.reset();
    fsx_ctx_destroy(t->ctx_);
  }
}

Transport& InProcessFabric::transport(int rank) { return *eps_.at(static_cast<size_t>(rank)); }

void InProcessFabric::set_link(int, int, LinkParams) {}  // the NVLink fabric's costs are measured

std::uint64_t InProcessFabric::message_count() const {
  auto* self = const_cast<InProcessFabric*>(this);
  std::lock_guard<std::mutex> lk(self->mu_);
  return messages_;
}

void InProcessFabric::reset_message_count() {
  std::lock_guard<std::mutex> lk(mu_);
  messages_ = 0;
}

void InProcessFabric::count_messages(std::uint64_t n) {
  std::lock_guard<std::mutex> lk(mu_);
  messages_ += n;
}

void InProcessFabric::poison(const std::string& why) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    poisoned_ = true;
    poison_msg_ = "collective aborted: " + why;
  }
  cv_.notify_all();
}

std::vector<std::vector<std::uint8_t>> InProcessFabric::exchange(int rank, std::vector<std::uint8_t> mine) {
  std::unique_lock<std::mutex> lk(mu_);
  if (poisoned_) throw CollectiveError(poison_msg_);
  const std::uint64_t my_round = round_;
  if (blobs_.empty()) blobs_.resize(static_cast<size_t>(world_));
  blobs_[static_cast<size_t>(rank)] = std::move(mine);
  if (++arrived_ == world_) {
    last_ = std::move(blobs_);
    blobs_.clear();
    arrived_ = 0;
    ++round_;
    cv_.notify_all();
  } else {
    cv_.wait(lk, [&] { return round_ != my_round || poisoned_; });
    if (round_ == my_round) throw CollectiveError(poison_msg_);
  }
  return last_;
}

void InProcessFabric::post(int src, int dst, std::uint64_t tag, Bytes payload) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    if (poisoned_) throw CollectiveError(poison_msg_);
    mail_[{src, dst, tag}].push_back(std::move(payload));
    ++messages_;
  }
  cv_.notify_all();
}

Bytes InProcessFabric::take(int src, int dst, std::uint64_t tag) {
  std::unique_lock<std::mutex> lk(mu_);
  auto& q = mail_[{src, dst, tag}];
  cv_.wait(lk, [&] { return !q.empty() || poisoned_; });
  if (q.empty()) throw CollectiveError(poison_msg_);
  Bytes b = std::move(q.front());
  q.pop_front();
  return b;
}

void InProcessFabric::run(const std::function<void(int)>& body) {
  std::vector<std::exception_ptr> errs(static_cast<size_t>(world_));
  std::vector<std::thread> th;
  for (int r = 0; r < world_; ++r) {
    th.emplace_back([&, r] {
      try {
        cuda_ok(cudaSetDevice(eps_[static_cast<size_t>(r)]->device_));
        body(r);
      } catch (...) {
        errs[static_cast<size_t>(r)] = std::current_exception();
        poison("rank " + std::to_string(r) + " failed");
      }
    });
  }
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// ---- collectives ---------------------------------------------------------------------
std::vector<Bytes> Communicator::gather_ce(const Bytes& local, std::uint64_t bound, bool ring) {
  const int p = world_size();
  CommWindows::agree(t_, bound);
  CommWindows* w = t_.windows();
  if (!local.empty()) cuda_ok(cudaMemcpyAsync(w->d_send, local.data(), local.size(), cudaMemcpyHostToDevice, w->s));
  std::vector<std::uint64_t> got(static_cast<size_t>(p));
  fsx_ok(fsx_allgather_ce(w->eng, w->d_send, local.size(), bound, w->d_recv, w->cap, got.data(), ring ? 1 : 0, w->s));
  std::vector<Bytes> out(static_cast<size_t>(p));
  for (int d = 0; d < p; ++d) {
    out[static_cast<size_t>(d)].resize(got[static_cast<size_t>(d)]);
    if (got[static_cast<size_t>(d)])
      cuda_ok(cudaMemcpyAsync(out[static_cast<size_t>(d)].data(), w->d_recv + static_cast<size_t>(d) * w->cap,
                              got[static_cast<size_t>(d)], cudaMemcpyDeviceToHost, w->s));
  }
  cuda_ok(cudaStreamSynchronize(w->s));
  t_.fabric().count_messages(static_cast<std::uint64_t>(p - 1));
  return out;
}

std::vector<Bytes> Communicator::all_gather(const Bytes& local, const CollectiveOptions&) {
  if (world_size() == 1) return {local};
  // size round: every rank learns the largest chunk (the slot bound)
  const std::uint64_t bound = max_of(t_.fabric().exchange(rank(), u64_blob(local.size())));
  t_.fabric().count_messages(static_cast<std::uint64_t>(world_size() - 1));
  return gather_ce(local, bound, false);
}

std::vector<Bytes> Communicator::ring_all_gather(const Bytes& local, std::span<const std::uint64_t> sizes,
                                                 const CollectiveOptions&) {
  const int p = world_size();
  if (sizes.size() != static_cast<std::size_t>(p))
    throw CollectiveError("ring_all_gather: need one chunk size per rank");
  if (local.size() != sizes[static_cast<size_t>(rank())])
    throw CollectiveError("ring_all_gather: local chunk size " + std::to_string(local.size()) +
                          " disagrees with sizes[" + std::to_string(rank()) + "] = " +
                          std::to_string(sizes[static_cast<size_t>(rank())]));
  if (p == 1) return {local};
  const std::uint64_t bound = *std::max_element(sizes.begin(), sizes.end());
  auto out = gather_ce(local, bound, true);
  for (int d = 0; d < p; ++d)
    if (out[static_cast<size_t>(d)].size() != sizes[static_cast<size_t>(d)])
      throw CollectiveError("ring_all_gather: rank " + std::to_string(d) + " sent " +
                            std::to_string(out[static_cast<size_t>(d)].size()) + " bytes, announced " +
                            std::to_string(sizes[static_cast<size_t>(d)]));
  return out;
}

std::vector<Bytes> Communicator::all_to_all(const std::vector<Bytes>& send, const CollectiveOptions&) {
  const int p = world_size();
  if (send.size() != static_cast<std::size_t>(p)) throw CollectiveError("all_to_all: need one payload per destination rank");
  if (p == 1) return send;
  std::uint64_t mine = 0;
  for (const auto& b : send) mine = std::max<std::uint64_t>(mine, b.size());
  // size round, then the payload round on the copy engines
  t_.fabric().count_messages(static_cast<std::uint64_t>(p - 1));
  CommWindows::agree(t_, mine);
  CommWindows* w = t_.windows();
  std::vector<std::uint64_t> off(static_cast<size_t>(p)), nb(static_cast<size_t>(p)), got(static_cast<size_t>(p));
  for (int d = 0; d < p; ++d) {
    off[static_cast<size_t>(d)] = static_cast<std::uint64_t>(d) * w->cap;
    nb[static_cast<size_t>(d)] = send[static_cast<size_t>(d)].size();
    if (nb[static_cast<size_t>(d)])
      cuda_ok(cudaMemcpyAsync(w->d_send + off[static_cast<size_t>(d)], send[static_cast<size_t>(d)].data(),
                              nb[static_cast<size_t>(d)], cudaMemcpyHostToDevice, w->s));
  }
  fsx_ok(fsx_a2a_ce(w->eng, w->d_send, off.data(), nb.data(), w->d_recv, w->cap, got.data(), w->s));
  std::vector<Bytes> out(static_cast<size_t>(p));
  for (int d = 0; d < p; ++d) {
    out[static_cast<size_t>(d)].resize(got[static_cast<size_t>(d)]);
    if (got[static_cast<size_t>(d)])
      cuda_ok(cudaMemcpyAsync(out[static_cast<size_t>(d)].data(), w->d_recv + static_cast<size_t>(d) * w->cap,
                              got[static_cast<size_t>(d)], cudaMemcpyDeviceToHost, w->s));
  }
  cuda_ok(cudaStreamSynchronize(w->s));
  t_.fabric().count_messages(static_cast<std::uint64_t>(p - 1));
  return out;
}

std::vector<double> Communicator::all_reduce_sum(std::span<const double> local, const CollectiveOptions& opts) {
  const auto parts = all_gather(pack_f64s(local), opts);
  for (const auto& b : parts)
    if (b.size() != local.size() * sizeof(double))
      throw CollectiveError("all_reduce_sum: vector length mismatch across ranks");
  std::vector<double> out(local.size(), 0.0);
  for (const auto& b : parts) {  // fixed rank order: bitwise deterministic
    const auto v = unpack_f64s(b);
    for (std::size_t i = 0; i < out.size(); ++i) out[i] += v[i];
  }
  return out;
}

double Communicator::time_max(double t) {
  if (!t_.in_fabric() || world_size() == 1) return t;
  std::vector<std::uint8_t> b(sizeof(double));
  std::memcpy(b.data(), &t, sizeof(double));
  double m = t;
  for (const auto& x : t_.fabric().exchange(rank(), b)) {
    double v;
    std::memcpy(&v, x.data(), sizeof(double));
    m = std::max(m, v);
  }
  return m;
}

void Communicator::log_compute(double duration, double penalty) {
  if (!clock_) return;
  const Interval iv = clock_->advance_compute(duration, penalty);
  if (log_) log_->append(Event{iteration_, rank(), Channel::Main, EventKind::Compute, Category::Dense, iv.start, iv.end, 0});
}

Bytes pack_u64s(std::span<const std::uint64_t> v) {
  Bytes b(v.size() * 8);
  if (!v.empty()) std::memcpy(b.data(), v.data(), b.size());
  return b;
}

std::vector<std::uint64_t> unpack_u64s(const Bytes& b) {
  if (b.size() % 8) throw CollectiveError("unpack_u64s: payload not a multiple of 8 bytes");
  std::vector<std::uint64_t> v(b.size() / 8);
  if (!v.empty()) std::memcpy(v.data(), b.data(), b.size());
  return v;
}

Bytes pack_f64s(std::span<const double> v) {
  Bytes b(v.size() * 8);
  if (!v.empty()) std::memcpy(b.data(), v.data(), b.size());
  return b;
}

std::vector<double> unpack_f64s(const Bytes& b) {
  if (b.size() % 8) throw CollectiveError("unpack_f64s: payload not a multiple of 8 bytes");
  std::vector<double> v(b.size() / 8);
  if (!v.empty()) std::memcpy(v.data(), b.data(), b.size());
  return v;
}

// ---- tcp.hpp ---------------------------------------------------------------------------
TcpTransport::TcpTransport(int, const std::vector<std::pair<std::string, std::uint16_t>>&) {
  throw ConfigError(
      "tcp transport: not part of the B200 build (one box; ranks exchange over NVLink through "
      "InProcessFabric or one process per GPU)");
}
TcpTransport::~TcpTransport() = default;
void TcpTransport::shutdown() {}

std::vector<std::pair<std::string, std::uint16_t>> local_peer_table(int world_size, std::uint16_t base_port) {
  std::vector<std::pair<std::string, std::uint16_t>> t;
  for (int r = 0; r < world_size; ++r) t.emplace_back("127.0.0.1", static_cast<std::uint16_t>(base_port + r));
  return t;
}

}  // namespace freescale::comm

// ---- sim.hpp (host helpers) ---------------------------------------------------------------
namespace freescale::sim {

double qps(std::uint64_t samples_processed, double duration_us) {
  if (duration_us <= 0) throw std::invalid_argument("qps: duration must be > 0");
  return static_cast<double>(samples_processed) / duration_us * 1e6;
}

std::string metric_csv_header() {
  return "iteration,rank_count,batch_size,max_uih,mode,sparsity,straggler_pct,collision_pct,"
         "exposed_ids_us,exposed_emb_us,exposed_grad_us,exposed_balancer_us,iteration_us,qps";
}

namespace {
std::string num9(double v) {
  std::ostringstream os;
  os.precision(9);
  os << v;
  return os.str();
}
// shortest round-trip decimal, with a trailing ".0" for integral values (the
// reference's JSON writer's number format)
std::string json_num(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}
}  // namespace

std::string metric_csv_row(const MetricRecord& r) {
  std::ostringstream os;
  os << r.iteration << ',' << r.rank_count << ',' << r.batch_size << ',' << r.max_uih << ',' << r.mode << ','
     << num9(r.sparsity) << ',' << num9(r.straggler_pct) << ',' << num9(r.collision_pct) << ','
     << num9(r.exposed_ids_us) << ',' << num9(r.exposed_emb_us) << ',' << num9(r.exposed_grad_us) << ','
     << num9(r.exposed_balancer_us) << ',' << num9(r.iteration_us) << ',' << num9(r.qps);
  return os.str();
}

std::string metric_json_line(const MetricRecord& r) {
  // keys in sorted order, as the reference's JSON object writes them
  std::ostringstream os;
  os << "{\"batch_size\":" << r.batch_size << ",\"collision_pct\":" << json_num(r.collision_pct)
     << ",\"exposed_balancer_us\":" << json_num(r.exposed_balancer_us)
     << ",\"exposed_emb_us\":" << json_num(r.exposed_emb_us) << ",\"exposed_grad_us\":" << json_num(r.exposed_grad_us)
     << ",\"exposed_ids_us\":" << json_num(r.exposed_ids_us) << ",\"iteration\":" << r.iteration
     << ",\"iteration_us\":" << json_num(r.iteration_us) << ",\"max_uih\":" << r.max_uih << ",\"mode\":\"" << r.mode
     << "\",\"qps\":" << json_num(r.qps) << ",\"rank_count\":" << r.rank_count
     << ",\"sparsity\":" << json_num(r.sparsity) << ",\"straggler_pct\":" << json_num(r.straggler_pct) << "}";
  return os.str();
}

LinearFit linear_fit(std::span<const double> xs, std::span<const double> ys) {
  if (xs.size() != ys.size() || xs.size() < 2) throw std::invalid_argument("linear_fit: need >= 2 paired points");
  const double n = static_cast<double>(xs.size());
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  for (std::size_t i = 0; i < xs.size(); ++i) {
    sx += xs[i];
    sy += ys[i];
    sxx += xs[i] * xs[i];
    sxy += xs[i] * ys[i];
  }
  LinearFit f;
  const double den = n * sxx - sx * sx;
  f.slope = den != 0 ? (n * sxy - sx * sy) / den : 0.0;
  f.intercept = (sy - f.slope * sx) / n;
  // residual and total sums of squares about the fit and the mean
  const double ybar = sy / n;
  double ss_res = 0, ss_tot = 0;
  for (std::size_t i = 0; i < xs.size(); ++i) {
    const double e = ys[i] - (f.slope * xs[i] + f.intercept);
    const double c = ys[i] - ybar;
    ss_res += e * e;
    ss_tot += c * c;
  }
  f.r2 = ss_tot > 0 ? 1.0 - ss_res / ss_tot : 1.0;
  return f;
}

}  // namespace freescale::sim
