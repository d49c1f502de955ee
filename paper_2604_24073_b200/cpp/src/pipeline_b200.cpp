// Drop-in implementation of freescale/pipeline.hpp, freescale/balancer.hpp
// and sim::Timeline (references: proj/src/pipeline.cpp, balancer.cpp,
// sim.cpp). The loop, the hook points, the toy model's evaluation order and
// the dense reduction follow the reference so run() returns its checkpoints
// bit for bit; the embedding engines underneath are the drop-in's GPU ones.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>

#include "freescale/balancer.hpp"
#include "freescale/embedding.hpp"
#include "freescale/pipeline.hpp"
#include "freescale/rng.hpp"
#include "freescale/sim.hpp"

namespace freescale {

// ---- sim::Timeline (sim.cpp:10-104) ---------------------------------------------
namespace sim {

Timeline::Timeline(EventLog log, std::vector<double> boundaries)
    : log_(std::move(log)), boundaries_(std::move(boundaries)) {
  if (boundaries_.empty()) throw std::invalid_argument("timeline: missing boundaries");
}

double Timeline::iteration_duration(int i) const {
  return boundaries_.at(static_cast<std::size_t>(i) + 1) - boundaries_.at(static_cast<std::size_t>(i));
}

double Timeline::straggler_pct(int i) const {
  const double dur = iteration_duration(i);
  if (dur <= 0) throw std::invalid_argument("straggler_pct: zero-duration iteration");
  if (num_ranks() == 0) throw std::invalid_argument("straggler_pct: no ranks");
  double idle = 0;
  for (int r = 0; r < num_ranks(); ++r) {
    double busy = 0;
    for (const Event& e : log_.rank_events(r))
      if (e.iteration == i && e.channel == Channel::Main && e.kind == EventKind::Compute) busy += e.end - e.start;
    idle += std::max(0.0, dur - busy);
  }
  return idle / (dur * num_ranks());
}

double Timeline::mean_straggler_pct() const {
  if (num_iterations() == 0) return 0;
  double t = 0;
  for (int i = 0; i < num_iterations(); ++i) t += straggler_pct(i);
  return t / num_iterations();
}

ExposedBreakdown Timeline::exposed_comm(int i) const {
  ExposedBreakdown x;
  for (int r = 0; r < num_ranks(); ++r)
    for (const Event& e : log_.rank_events(r)) {
      if (e.iteration != i || e.channel != Channel::Main || e.kind == EventKind::Compute) continue;
      const double d = e.end - e.start;
      switch (e.category) {
        case Category::Ids: x.ids_us += d; break;
        case Category::Embedding: x.embedding_us += d; break;
        case Category::Gradient: x.gradient_us += d; break;
        case Category::Balancer: x.balancer_us += d; break;
        case Category::Dense: x.dense_us += d; break;
        case Category::None: break;
      }
    }
  return x;
}

ExposedBreakdown Timeline::exposed_comm_total() const {
  ExposedBreakdown t;
  for (int i = 0; i < num_iterations(); ++i) {
    const ExposedBreakdown e = exposed_comm(i);
    t.ids_us += e.ids_us;
    t.embedding_us += e.embedding_us;
    t.gradient_us += e.gradient_us;
    t.balancer_us += e.balancer_us;
    t.dense_us += e.dense_us;
  }
  return t;
}

void Timeline::check_causality() const {
  for (int r = 0; r < num_ranks(); ++r) {
    double last[2] = {-1, -1};
    for (const Event& e : log_.rank_events(r)) {
      if (e.end < e.start) throw std::logic_error("timeline: event ends before it starts on rank " + std::to_string(r));
      double& l = last[e.channel == Channel::Main ? 0 : 1];
      if (e.start + 1e-9 < l) throw std::logic_error("timeline: overlapping events on one channel of rank " + std::to_string(r));
      l = e.end;
    }
  }
}

}  // namespace sim

// ---- pipeline (pipeline.cpp) ------------------------------------------------------
namespace pipeline {

namespace {
std::mutex& registry_mu() {
  static std::mutex m;
  return m;
}
std::map<std::string, partition::PartitionFn>& registry() {
  static std::map<std::string, partition::PartitionFn> r;
  return r;
}
}  // namespace

void register_partitioner(const std::string& name, partition::PartitionFn fn) {
  std::lock_guard<std::mutex> g(registry_mu());
  registry()[name] = std::move(fn);
}

const partition::PartitionFn* find_partitioner(const std::string& name) {
  std::lock_guard<std::mutex> g(registry_mu());
  auto it = registry().find(name);
  return it == registry().end() ? nullptr : &it->second;
}

ToyModel ToyModel::init(std::uint32_t dim, std::uint64_t seed) {
  ToyModel m;
  m.dim = dim;
  std::uint64_t st = seed ^ 0xd15ea5e0f1e1dULL;  // pipeline.cpp:36-42
  for (std::uint32_t d = 0; d < dim; ++d) m.w.push_back((rng_double(st) - 0.5) * 0.2);
  return m;
}

double ToyModel::predict(const workload::Sample&, std::span<const double> pooled) const {
  double y = 0;
  for (std::uint32_t d = 0; d < dim; ++d) y += pooled[d] * w[d];
  return y;
}

ToyModel::Result ToyModel::forward_backward(const workload::Batch& batch, std::span<const double> emb,
                                            std::uint64_t global_samples) const {
  // the reference's evaluation order (pipeline.cpp:51-90): pooled sums over a
  // sample's rows in order, the projection summed over d in order
  Result r;
  r.dense_grad_sum.assign(dim, 0.0);
  r.emb_grads.assign(emb.size(), 0.0);
  const double n = static_cast<double>(global_samples);
  std::vector<double> pooled(dim);
  std::size_t row = 0;
  for (const workload::Sample& s : batch.samples) {
    const std::size_t L = s.uih.size();
    std::fill(pooled.begin(), pooled.end(), 0.0);
    for (std::size_t k = 0; k < L; ++k)
      for (std::uint32_t d = 0; d < dim; ++d) pooled[d] += emb[(row + k) * dim + d];
    if (L)
      for (std::uint32_t d = 0; d < dim; ++d) pooled[d] /= static_cast<double>(L);
    const double err = predict(s, pooled) - s.label;
    r.loss_sum += err * err;
    for (std::uint32_t d = 0; d < dim; ++d) r.dense_grad_sum[d] += 2.0 * err * pooled[d];
    if (L) {
      const double scale = 2.0 * err / (static_cast<double>(L) * n);
      for (std::size_t k = 0; k < L; ++k)
        for (std::uint32_t d = 0; d < dim; ++d) r.emb_grads[(row + k) * dim + d] = scale * w[d];
    }
    row += L;
  }
  if (row * dim != emb.size()) throw std::invalid_argument("toy model: embedding rows do not match batch occurrences");
  return r;
}

std::vector<double> dense_grad_sync(comm::Communicator& comm, std::span<const double> grad_sum,
                                    std::uint64_t global_samples) {
  auto g = comm.all_reduce_sum(grad_sum, {Channel::Main, Category::Dense, comm::CollectiveMode::Fused, true});
  for (double& x : g) x /= static_cast<double>(global_samples);
  return g;
}

namespace {

std::vector<std::uint8_t> full_blob(const std::vector<std::uint8_t>& table, const std::vector<double>& w) {
  std::vector<std::uint8_t> out(table);
  const auto* p = reinterpret_cast<const std::uint8_t*>(w.data());
  out.insert(out.end(), p, p + w.size() * sizeof(double));
  return out;
}

}  // namespace

RunResult run(const std::vector<std::vector<workload::Batch>>& iterations, const workload::WorkloadSpec& wspec,
              const RunConfig& config) {
  const int world = wspec.num_ranks;
  const int n_it = static_cast<int>(iterations.size());
  for (const auto& it : iterations)
    if (it.size() != static_cast<std::size_t>(world))
      throw std::invalid_argument("pipeline: iteration without one batch per rank");
  const std::uint64_t global = static_cast<std::uint64_t>(world) * static_cast<std::uint64_t>(wspec.batch_size);
  const embedding::TableGeometry geom{config.table_rows, config.dim, world};
  RunResult res;
  res.samples_processed = static_cast<std::uint64_t>(n_it) * global;
  if (n_it == 0) {
    std::vector<double> full(config.table_rows * config.dim);
    for (std::uint64_t g = 0; g < config.table_rows; ++g)
      for (std::uint32_t d = 0; d < config.dim; ++d)
        full[g * config.dim + d] = embedding::initial_value(config.model_seed, g, d);
    res.table_checkpoint = embedding::checkpoint_bytes(geom, full);
    res.final_dense = ToyModel::init(config.dim, config.model_seed).w;
    res.full_checkpoint = full_blob(res.table_checkpoint, res.final_dense);
    return res;
  }
  // per-iteration collision share of the raw workload (metric records)
  std::vector<double> collision(static_cast<std::size_t>(n_it), 0.0);
  {
    std::vector<std::uint64_t> prev;
    for (int i = 0; i < n_it; ++i) {
      auto cur = workload::unique_rows(iterations[static_cast<std::size_t>(i)]);
      if (i > 0 && !cur.empty()) collision[static_cast<std::size_t>(i)] = workload::collision_fraction(prev, cur);
      prev = std::move(cur);
    }
  }

  comm::InProcessFabric fabric(world, config.cost.link);
  EventLog log(world);
  std::vector<RankClock> clocks(static_cast<std::size_t>(world));
  std::vector<double> bounds(static_cast<std::size_t>(n_it) + 1, 0.0), losses(static_cast<std::size_t>(n_it), 0.0);
  std::vector<std::vector<double>> sparsity(static_cast<std::size_t>(world), std::vector<double>(static_cast<std::size_t>(n_it), 0.0));
  std::vector<double> dense;
  std::vector<std::uint8_t> table_blob;

  fabric.run([&](int rank) {
    RankClock& clock = clocks[static_cast<std::size_t>(rank)];
    comm::Communicator comm(fabric.transport(rank), &clock, &log);
    embedding::ShardView shard(geom, rank, config.lr_embedding, config.model_seed);
    ToyModel model = ToyModel::init(config.dim, config.model_seed);
    std::optional<embedding::SynchronizedEmbedding> sync;
    std::optional<embedding::PrioritizedEmbedding> prio;
    if (config.mode == Mode::Synchronized)
      sync.emplace(shard, comm);
    else
      prio.emplace(shard, comm, config.cost.collective_mode);
    HookRegistry hooks;
    std::optional<balancer::Balancer> bal;
    if (config.balancer_enabled) {
      balancer::BalancerConfig bc;
      bc.partition = config.partition;
      bc.alpha = config.alpha;
      bc.autotune_step = config.autotune_step;
      bc.autotune_delta = config.autotune_delta;
      bc.autotune_decay = config.autotune_decay;
      bc.mode = config.cost.collective_mode;
      // the prioritized forward routes the next batch's ids: one more batch ahead
      bc.lead = config.prefetch_depth + (config.mode == Mode::Prioritized ? 1 : 0);
      bal.emplace(comm, bc,
                  [&, rank](int i) -> const workload::Batch* {
                    return i >= 0 && i < n_it ? &iterations[static_cast<std::size_t>(i)][static_cast<std::size_t>(rank)]
                                              : nullptr;
                  },
                  n_it);
      bal->install_hooks(hooks);
    }
    for (int i = 0; i < n_it; ++i) {
      comm.set_iteration(i);
      const HookContext hc{i, rank};
      hooks.fire(HookPoint::DataLoad, hc);
      const workload::Batch batch = bal ? bal->take(i) : iterations[static_cast<std::size_t>(i)][static_cast<std::size_t>(rank)];
      std::vector<std::uint64_t> lengths;
      for (const auto& s : batch.samples) lengths.push_back(s.uih.size());
      if (!lengths.empty() && batch.max_uih_len() > 0)
        sparsity[static_cast<std::size_t>(rank)][static_cast<std::size_t>(i)] = workload::measure_sparsity(lengths);
      hooks.fire(HookPoint::PreForward, hc);
      const IdJagged cur = batch.uih_ids();
      std::vector<double> rows;
      if (sync) {
        rows = sync->forward(cur);
      } else {
        std::optional<IdJagged> next;
        if (i + 1 < n_it)
          next = bal ? bal->peek(i + 1)->uih_ids()
                     : iterations[static_cast<std::size_t>(i) + 1][static_cast<std::size_t>(rank)].uih_ids();
        rows = prio->forward(cur, next ? &*next : nullptr);
      }
      const double compute_us = config.cost.compute_time_for_lengths(lengths);
      comm.log_compute(compute_us / 3.0, config.cost.overlap_penalty);
      const ToyModel::Result g = model.forward_backward(batch, rows, global);
      hooks.fire(HookPoint::PostForward, hc);
      comm.log_compute(compute_us * 2.0 / 3.0, config.cost.overlap_penalty);
      if (sync)
        sync->backward(g.emb_grads);
      else
        prio->backward(g.emb_grads);
      hooks.fire(HookPoint::PostBackward, hc);
      // optimizer step: one reduction of the dense sums, the loss and the sample count
      std::vector<double> payload(g.dense_grad_sum);
      payload.push_back(g.loss_sum);
      payload.push_back(static_cast<double>(batch.samples.size()));
      const auto red = comm.all_reduce_sum(payload, {Channel::Main, Category::Dense, comm::CollectiveMode::Fused, true});
      const double count = red[config.dim + 1];
      if (count != static_cast<double>(global))
        throw ProtocolError("pipeline: sample conservation violated (" + std::to_string(count) + " vs " +
                            std::to_string(global) + ")");
      for (std::uint32_t d = 0; d < config.dim; ++d) model.w[d] -= config.lr_dense * red[d] / static_cast<double>(global);
      if (rank == 0) {
        losses[static_cast<std::size_t>(i)] = red[config.dim] / static_cast<double>(global);
        bounds[static_cast<std::size_t>(i) + 1] = clock.main_time();
      }
      if (bal) bal->report_compute_time(compute_us);
      hooks.fire(HookPoint::OptimizerStep, hc);
      hooks.fire(HookPoint::Metrics, hc);
    }
    if (prio) prio->finalize();
    const auto full = embedding::gather_full_table(comm, shard);
    const auto ws = comm.all_gather(comm::pack_f64s(model.w), {Channel::Main, Category::None, comm::CollectiveMode::Fused, true});
    for (const auto& x : ws)
      if (x != ws[0]) throw ProtocolError("pipeline: dense weights diverged across ranks");
    if (rank == 0) {
      dense = model.w;
      table_blob = embedding::checkpoint_bytes(geom, full);
    }
  });

  sim::Timeline tl(std::move(log), bounds);
  for (int i = 0; i < n_it; ++i) {
    sim::MetricRecord m;
    m.iteration = i;
    m.rank_count = world;
    m.batch_size = wspec.batch_size;
    m.max_uih = wspec.max_uih;
    m.mode = mode_name(config.mode);
    double sp = 0;
    for (int r = 0; r < world; ++r) sp += sparsity[static_cast<std::size_t>(r)][static_cast<std::size_t>(i)];
    m.sparsity = sp / world;
    m.straggler_pct = tl.iteration_duration(i) > 0 ? tl.straggler_pct(i) : 0.0;
    m.collision_pct = collision[static_cast<std::size_t>(i)];
    const auto x = tl.exposed_comm(i);
    m.exposed_ids_us = x.ids_us;
    m.exposed_emb_us = x.embedding_us;
    m.exposed_grad_us = x.gradient_us;
    m.exposed_balancer_us = x.balancer_us;
    m.iteration_us = tl.iteration_duration(i);
    m.qps = m.iteration_us > 0 ? sim::qps(global, m.iteration_us) : 0.0;
    res.records.push_back(std::move(m));
  }
  res.losses = std::move(losses);
  res.final_dense = dense;
  res.table_checkpoint = table_blob;
  res.full_checkpoint = full_blob(table_blob, dense);
  res.total_us = tl.total_duration();
  res.timeline.emplace(std::move(tl));
  return res;
}

}  // namespace pipeline

// ---- balancer (balancer.cpp) -------------------------------------------------------
namespace balancer {

using comm::Bytes;

Balancer::Balancer(comm::Communicator& comm, BalancerConfig config,
                   std::function<const workload::Batch*(int)> raw_batches, int num_iterations)
    : comm_(comm), cfg_(std::move(config)), source_(std::move(raw_batches)), iterations_(num_iterations) {
  if (cfg_.lead < 1) throw ConfigError("balancer: lead must be >= 1");
  tune_.step = cfg_.autotune_step;
  tune_.delta = cfg_.autotune_delta;
  tune_.decay = cfg_.autotune_decay;
}

Balancer::Work* Balancer::find(int index, bool create) {
  for (Work& p : work_)
    if (p.iteration == index) return &p;
  if (!create || index >= iterations_) return nullptr;
  Work p;
  p.iteration = index;
  p.source = source_(index);
  if (!p.source) throw ProtocolError("balancer: no raw batch for iteration " + std::to_string(index));
  work_.push_back(std::move(p));
  return &work_.back();
}

void Balancer::fire(int index, int stage) {
  if (index < 0 || index >= iterations_) return;
  Work* p = find(index, stage == 0);
  if (!p) return;
  ++fired_[stage];
  if (stage == 0) gather_lengths(*p);
  else if (stage == 1) gather_candidates_and_plan(*p);
  else exchange_samples(*p);
}

void Balancer::install_hooks(pipeline::HookRegistry& hooks) {
  const int lead = cfg_.lead;
  hooks.add(pipeline::HookPoint::DataLoad, [this, lead](const pipeline::HookContext& c) {
    if (c.iteration != 0) return;
    for (int j = 0; j < lead && j < iterations_; ++j)
      for (int s = 0; s < 3; ++s) fire(j, s);
    fire(lead, 0);
  });
  hooks.add(pipeline::HookPoint::PreForward, [this, lead](const pipeline::HookContext& c) { fire(c.iteration + lead, 1); });
  hooks.add(pipeline::HookPoint::PostForward, [this, lead](const pipeline::HookContext& c) { fire(c.iteration + lead, 2); });
  hooks.add(pipeline::HookPoint::OptimizerStep,
            [this, lead](const pipeline::HookContext& c) { fire(c.iteration + lead + 1, 0); });
}

void Balancer::gather_lengths(Work& p) {
  if (p.at != Stage::Idle) throw ProtocolError("balancer: stage 1 fired out of order");
  // [B, uih lengths, candidate counts] as u64, then the last compute time (f64)
  std::vector<std::uint64_t> v{p.source->samples.size()};
  for (const auto& s : p.source->samples) v.push_back(s.uih.size());
  for (const auto& s : p.source->samples) v.push_back(s.candidates.size());
  Bytes msg = comm::pack_u64s(v);
  const std::size_t at = msg.size();
  msg.resize(at + 8);
  std::memcpy(msg.data() + at, &compute_us_, 8);
  const auto all = comm_.all_gather(msg, {Channel::Side, Category::Balancer, cfg_.mode, false});
  const int world = comm_.world_size();
  p.metas.clear();
  p.candidate_counts.clear();
  p.rank_compute_us.assign(static_cast<std::size_t>(world), 0.0);
  for (int r = 0; r < world; ++r) {
    const Bytes& b = all[static_cast<std::size_t>(r)];
    if (b.size() < 16) throw ProtocolError("balancer: short stage-1 payload");
    const auto u = comm::unpack_u64s(Bytes(b.begin(), b.end() - 8));
    std::memcpy(&p.rank_compute_us[static_cast<std::size_t>(r)], b.data() + b.size() - 8, 8);
    const std::size_t B = static_cast<std::size_t>(u.at(0));
    if (u.size() != 1 + 2 * B) throw ProtocolError("balancer: stage-1 payload shape mismatch");
    for (std::size_t k = 0; k < B; ++k) {
      partition::GlobalSampleMeta m;
      m.origin_rank = r;
      m.local_index = static_cast<int>(k);
      m.uih_len = u[1 + k];
      m.num_candidates = static_cast<std::uint32_t>(u[1 + B + k]);
      p.metas.push_back(std::move(m));
      p.candidate_counts.push_back(u[1 + B + k]);
    }
  }
  p.at = Stage::LengthsGathered;
}

void Balancer::gather_candidates_and_plan(Work& p) {
  if (p.at != Stage::LengthsGathered) throw ProtocolError("balancer: stage 2 before stage 1");
  std::vector<std::uint64_t> mine;
  for (const auto& s : p.source->samples)
    for (const auto& c : s.candidates) mine.push_back(c.size());
  const auto all = comm_.all_gather(comm::pack_u64s(mine), {Channel::Side, Category::Balancer, cfg_.mode, false});
  std::size_t m = 0;
  for (int r = 0; r < comm_.world_size(); ++r) {
    const auto lens = comm::unpack_u64s(all[static_cast<std::size_t>(r)]);
    const std::size_t first = m;
    std::uint64_t announced = 0;
    while (m < p.metas.size() && p.metas[m].origin_rank == r) announced += p.metas[m++].num_candidates;
    if (lens.size() != announced)
      throw ProtocolError("balancer: rank " + std::to_string(r) + " sent " + std::to_string(lens.size()) +
                          " candidate lengths, stage 1 announced " + std::to_string(announced));
    std::size_t at = 0;
    for (std::size_t k = first; k < m; ++k) {
      p.metas[k].candidate_lens.assign(lens.begin() + static_cast<std::ptrdiff_t>(at),
                                       lens.begin() + static_cast<std::ptrdiff_t>(at + p.metas[k].num_candidates));
      at += p.metas[k].num_candidates;
    }
  }
  const int world = comm_.world_size();
  const std::string& part = cfg_.partition;
  if (part == "fbs") {
    p.plan = partition::fbs_partition(p.metas, world);
  } else if (part == "vbs") {
    if (tune_.initialized && std::any_of(p.rank_compute_us.begin(), p.rank_compute_us.end(), [](double t) { return t > 0; })) {
      std::vector<double> t(p.rank_compute_us);
      for (double& x : t) x = std::max(x, 1e-9);
      partition::autotune_update(tune_, t);
    }
    p.plan = partition::vbs_partition(p.metas, world, cfg_.alpha, &tune_);
  } else if (part == "none") {
    p.plan = partition::identity_partition(p.metas, world);
  } else if (part.rfind("custom:", 0) == 0) {
    const partition::PartitionFn* fn = pipeline::find_partitioner(part.substr(7));
    if (!fn) throw ConfigError("balancer: unknown custom partitioner '" + part.substr(7) + "'");
    p.plan = partition::custom_partition(*fn, p.metas, world);
  } else {
    throw ConfigError("balancer: unknown partition '" + part + "'");
  }
  p.plan.validate(p.metas.size(), part == "fbs");
  p.at = Stage::CandidatesGathered;
}

void Balancer::exchange_samples(Work& p) {
  if (p.at != Stage::CandidatesGathered) throw ProtocolError("balancer: stage 3 before stage 2");
  const auto lists = p.plan.exchange_lists(p.metas);
  const auto& sends = lists[static_cast<std::size_t>(comm_.rank())];
  std::vector<Bytes> out(static_cast<std::size_t>(comm_.world_size()));
  std::vector<std::uint8_t> rec;
  for (std::size_t dst = 0; dst < out.size(); ++dst)
    for (int local : sends[dst]) {
      rec.clear();
      workload::encode_sample(p.source->samples.at(static_cast<std::size_t>(local)), rec);
      const std::uint32_t n = static_cast<std::uint32_t>(rec.size());
      const std::size_t at = out[dst].size();
      out[dst].resize(at + 4 + n);
      std::memcpy(out[dst].data() + at, &n, 4);
      std::memcpy(out[dst].data() + at + 4, rec.data(), n);
    }
  p.records.value = comm_.all_to_all(out, {Channel::Side, Category::Balancer, cfg_.mode, false});
  p.records.category = Category::Balancer;
  p.records.ready_time = comm_.clock() ? comm_.clock()->side_time() : 0.0;
  p.records.bytes = 0;
  for (const Bytes& b : p.records.value) p.records.bytes += b.size();
  p.at = Stage::Shuffled;
}

workload::Batch Balancer::build_batch(Work& p) {
  const int me = comm_.rank();
  std::vector<std::size_t> at(p.records.value.size(), 0);
  workload::Batch out;
  out.rank = me;
  for (std::size_t g : p.plan.receive_order[static_cast<std::size_t>(me)]) {
    const std::size_t src = static_cast<std::size_t>(p.metas[g].origin_rank);
    const Bytes& blob = p.records.value[src];
    if (at[src] + 4 > blob.size()) throw ProtocolError("balancer: stage-3 payload shorter than the plan");
    std::uint32_t n = 0;
    std::memcpy(&n, blob.data() + at[src], 4);
    at[src] += 4;
    if (at[src] + n > blob.size()) throw ProtocolError("balancer: stage-3 record truncated");
    std::size_t used = 0;
    out.samples.push_back(workload::decode_sample(blob.data() + at[src], n, used));
    if (used != n) throw ProtocolError("balancer: stage-3 record has trailing bytes");
    at[src] += n;
  }
  for (std::size_t src = 0; src < at.size(); ++src)
    if (at[src] != p.records.value[src].size())
      throw ProtocolError("balancer: stage-3 payload from rank " + std::to_string(src) + " longer than the plan");
  return out;
}

workload::Batch Balancer::take(int iteration) {
  Work* p = find(iteration, false);
  if (!p || p->at != Stage::Shuffled)
    throw ProtocolError("balancer: batch " + std::to_string(iteration) + " consumed before stage 3 completed");
  comm_.wait_handle(p->records);
  workload::Batch out = p->assembled ? std::move(*p->assembled) : build_batch(*p);
  while (!work_.empty() && work_.front().iteration <= iteration) work_.pop_front();
  return out;
}

const workload::Batch* Balancer::peek(int iteration) {
  Work* p = find(iteration, false);
  if (!p) return nullptr;
  if (p->at != Stage::Shuffled)
    throw ProtocolError("balancer: peek at batch " + std::to_string(iteration) + " before stage 3 completed");
  if (!p->assembled) p->assembled = build_batch(*p);
  return &*p->assembled;
}

}  // namespace balancer
}  // namespace freescale
