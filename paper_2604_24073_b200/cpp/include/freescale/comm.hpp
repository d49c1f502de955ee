// Drop-in header: rank fabric + communicator (proj/include/freescale/comm.hpp).
// The reference's InProcessFabric runs ranks as threads over mailboxes; on a
// B200 box each rank thread drives one GPU context (ranks share GPUs when
// there are fewer GPUs than ranks) and the engines move bytes with copy
// engines between the ranks' device windows. The fabric keeps the
// reference's run(body) contract: one thread per rank, poison on failure, the
// lowest failing rank's exception rethrown.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "freescale/errors.hpp"

struct fsx_ctx;

namespace freescale::comm {

enum class CollectiveMode : std::uint8_t { Fused, SmFree };

class InProcessFabric;

// One rank's endpoint (comm.hpp:41-49 role): rank, world, its GPU context.
class Transport {
 public:
  int rank() const { return rank_; }
  int world_size() const { return world_; }
  int device() const { return device_; }
  fsx_ctx* ctx() const { return ctx_; }
  InProcessFabric& fabric() const { return *fabric_; }

 private:
  friend class InProcessFabric;
  int rank_ = 0, world_ = 1, device_ = 0;
  fsx_ctx* ctx_ = nullptr;
  InProcessFabric* fabric_ = nullptr;
};

class InProcessFabric {
 public:
  explicit InProcessFabric(int world_size);
  ~InProcessFabric();
  InProcessFabric(const InProcessFabric&) = delete;
  InProcessFabric& operator=(const InProcessFabric&) = delete;

  int world_size() const { return world_; }
  Transport& transport(int rank);
  void poison(const std::string& why);
  void run(const std::function<void(int)>& body);

  // Collective host exchange used by the engines' wiring and the checkpoint
  // gather: every rank contributes one blob, all get all (rank order).
  std::vector<std::vector<std::uint8_t>> exchange(int rank, std::vector<std::uint8_t> mine);

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
};

// Per-rank facade (comm.hpp:105-164): identity of the rank + the fabric.
class Communicator {
 public:
  explicit Communicator(Transport& t) : t_(t) {}
  int rank() const { return t_.rank(); }
  int world_size() const { return t_.world_size(); }
  Transport& transport() const { return t_; }

 private:
  Transport& t_;
};

}  // namespace freescale::comm
