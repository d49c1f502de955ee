// Drop-in header: rank fabric + collectives (proj/include/freescale/comm.hpp,
// same names, signatures and exception classes).
//
// B200 mapping. The reference's InProcessFabric runs ranks as threads over
// mailboxes; here each rank thread drives one GPU context (ranks share GPUs
// when there are fewer GPUs than ranks). The Communicator's byte collectives
// move their payloads with the copy engines between the ranks' device windows
// (libfsx fsx_a2a_ce / fsx_allgather_ce: cudaMemcpyAsync peer copies + stream
// memory-op flags, 0 SMs) — the single-box analogue of the reference's SmFree
// path. Sizes travel first (the reference's 8-byte size round, comm.cpp:
// 328-341) on the host, so every rank agrees on the slot bound; payloads never
// leave HBM between the ranks. Transport::send / recv remain available as host
// point-to-point messages (the reference's mailbox semantics: exactly once,
// FIFO per (src, dst, tag)).
//
// Logical time: the reference is a simulator whose collectives advance a
// per-rank logical clock by a link-cost model. On B200 the hot path is timed on
// the device (fsx_engine_exposed_ms); the clock here is bookkeeping only —
// collectives do not advance it, wait_handle / log_compute do as in the
// reference.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <string>
#include <tuple>
#include <vector>

#include "freescale/errors.hpp"
#include "freescale/events.hpp"

struct fsx_ctx;

namespace freescale::comm {

using Bytes = std::vector<std::uint8_t>;

enum class CollectiveMode : std::uint8_t { Fused, SmFree };
enum class CostClass : std::uint8_t { Normal, Staged, Free };

// the reference's link-cost parameters (carried for API parity; the B200
// fabric's costs are measured, not modelled)
struct LinkParams {
  double latency_us = 5.0;
  double bandwidth_bytes_per_us = 25000.0;
  double copy_cost_us_per_mb = 40.0;
};

struct Delivery {
  Bytes payload;
  double arrival = 0.0;
};

class InProcessFabric;
struct CommWindows;  // a rank's copy-engine collective windows (libfsx engine)

// One rank's endpoint (comm.hpp:41-49).
class Transport {
 public:
  virtual ~Transport();
  virtual int rank() const { return rank_; }
  virtual int world_size() const { return world_; }
  // host point-to-point message; FIFO per (src, dst, tag)
  virtual void send(int dst, std::uint64_t tag, Bytes payload, double send_time, CostClass cost);
  virtual Delivery recv(int src, std::uint64_t tag);

  // B200 endpoint: the rank's GPU context and fabric (null for transports
  // that are not part of an in-process fabric)
  int device() const { return device_; }
  fsx_ctx* ctx() const { return ctx_; }
  InProcessFabric& fabric() const;
  bool in_fabric() const { return fabric_ != nullptr; }
  CommWindows* windows() const { return win_.get(); }

 protected:
  Transport() = default;

 private:
  friend class InProcessFabric;
  friend struct CommWindows;
  friend class Communicator;
  int rank_ = 0, world_ = 1, device_ = 0;
  fsx_ctx* ctx_ = nullptr;
  InProcessFabric* fabric_ = nullptr;
  std::unique_ptr<CommWindows> win_;
};

class InProcessFabric {
 public:
  explicit InProcessFabric(int world_size, LinkParams link = {});
  ~InProcessFabric();
  InProcessFabric(const InProcessFabric&) = delete;
  InProcessFabric& operator=(const InProcessFabric&) = delete;

  int world_size() const { return world_; }
  Transport& transport(int rank);
  void set_link(int src, int dst, LinkParams link);
  // point-to-point transfers the collectives and send() issued (every rank)
  std::uint64_t message_count() const;
  void reset_message_count();
  void poison(const std::string& why);
  void run(const std::function<void(int)>& body);

  // Host rendezvous used by the collectives' size rounds, the engines'
  // wiring and the checkpoint gather: every rank contributes one blob, all
  // get all (rank order).
  std::vector<std::vector<std::uint8_t>> exchange(int rank, std::vector<std::uint8_t> mine);
  void count_messages(std::uint64_t n);
  void post(int src, int dst, std::uint64_t tag, Bytes payload);
  Bytes take(int src, int dst, std::uint64_t tag);

 private:
  int world_;
  std::vector<std::unique_ptr<Transport>> eps_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::uint64_t round_ = 0;
  int arrived_ = 0;
  std::vector<std::vector<std::uint8_t>> blobs_, last_;
  bool poisoned_ = false;
  std::string poison_msg_;
  std::uint64_t messages_ = 0;
  std::map<std::tuple<int, int, std::uint64_t>, std::deque<Bytes>> mail_;
};

struct CollectiveOptions {
  Channel channel = Channel::Main;
  Category category = Category::None;
  CollectiveMode mode = CollectiveMode::Fused;
  bool synchronizing = false;
};

// An overlapped collective's result and the time its producer finished.
template <typename T>
struct Handle {
  T value{};
  double ready_time = 0.0;
  Category category = Category::None;
  std::uint64_t bytes = 0;
};

// Per-rank collective facade (comm.hpp:105-164). Every rank issues the same
// collectives in the same order.
class Communicator {
 public:
  explicit Communicator(Transport& transport, RankClock* clock = nullptr, EventLog* log = nullptr)
      : t_(transport), clock_(clock), log_(log) {}

  int rank() const { return t_.rank(); }
  int world_size() const { return t_.world_size(); }
  Transport& transport() const { return t_; }
  RankClock* clock() const { return clock_; }
  void set_iteration(int iteration) { iteration_ = iteration; }
  int iteration() const { return iteration_; }

  // every rank's chunk, in rank order (direct copy-engine all-gather)
  std::vector<Bytes> all_gather(const Bytes& local, const CollectiveOptions& opts);
  // the reference's SmFree ring: p-1 forwarding stages; sizes[r] = rank r's
  // chunk size on every rank; bitwise equal to all_gather
  std::vector<Bytes> ring_all_gather(const Bytes& local, std::span<const std::uint64_t> sizes,
                                     const CollectiveOptions& opts);
  // send[d] -> rank d; slot s of the result = what rank s sent here
  std::vector<Bytes> all_to_all(const std::vector<Bytes>& send, const CollectiveOptions& opts);
  // elementwise sum in rank order 0..p-1 (bitwise deterministic)
  std::vector<double> all_reduce_sum(std::span<const double> local, const CollectiveOptions& opts);
  // everyone leaves with the max over ranks of t
  double time_max(double t);

  template <typename T>
  double wait_handle(const Handle<T>& h) {
    if (clock_ == nullptr) return 0.0;
    const Interval iv = clock_->wait_until(h.ready_time);
    if (iv.end > iv.start && log_ != nullptr)
      log_->append(Event{iteration_, rank(), Channel::Main, EventKind::Wait, h.category, iv.start, iv.end, h.bytes});
    return iv.end - iv.start;
  }
  void log_compute(double duration, double penalty = 1.0);
  double now_main() const { return clock_ ? clock_->main_time() : 0.0; }

 private:
  std::vector<Bytes> gather_ce(const Bytes& local, std::uint64_t bound, bool ring);
  Transport& t_;
  RankClock* clock_;
  EventLog* log_;
  int iteration_ = 0;
};

Bytes pack_u64s(std::span<const std::uint64_t> v);
std::vector<std::uint64_t> unpack_u64s(const Bytes& b);
Bytes pack_f64s(std::span<const double> v);
std::vector<double> unpack_f64s(const Bytes& b);

}  // namespace freescale::comm
