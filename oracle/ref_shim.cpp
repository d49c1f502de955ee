// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI shim over the *unmodified* reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It exists so
// that pytest (via ctypes) can (1) pin the plain-C restatement in
// oracle/fsx_oracle.c against the reference itself, (2) regenerate the golden
// fixtures under tests/golden/, and (3) serve as the `cpu_baseline` /
// `--impl reference` arm of bench.py. Nothing on the product path links this.
//
// Every function drives the reference through its own public API
// (proj/include/freescale/*.hpp); the mapping is cited per function.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "freescale/comm.hpp"
#include "freescale/embedding.hpp"
#include "freescale/partition.hpp"
#include "freescale/pipeline.hpp"
#include "freescale/rng.hpp"
#include "freescale/sim.hpp"
#include "freescale/workload.hpp"

using namespace freescale;

namespace {

thread_local std::string g_err;

// 0 ok; negative codes mirror include/fsx.h's exception classes.
int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define SHIM_TRY try {
#define SHIM_CATCH                                                   \
  }                                                                  \
  catch (const ProtocolError& e) { return fail(e, -4); }             \
  catch (const CollectiveError& e) { return fail(e, -5); }           \
  catch (const ConfigError& e) { return fail(e, -6); }               \
  catch (const std::invalid_argument& e) { return fail(e, -1); }     \
  catch (const std::domain_error& e) { return fail(e, -2); }         \
  catch (const std::out_of_range& e) { return fail(e, -3); }         \
  catch (const std::exception& e) { return fail(e, -9); }            \
  return 0;

// ids laid out [iter][rank] as one flat array + per-(iter,rank) lengths. Each
// per-rank batch becomes a single-segment IdJagged (segmentation is irrelevant
// to the embedding engines: they only consume values()).
std::vector<std::vector<IdJagged>> unflatten(const std::uint64_t* ids, const std::uint64_t* lens,
                                             int iters, int world) {
  std::vector<std::vector<IdJagged>> out(static_cast<std::size_t>(iters));
  std::size_t at = 0;
  for (int i = 0; i < iters; ++i) {
    for (int r = 0; r < world; ++r) {
      const std::size_t n = lens[static_cast<std::size_t>(i * world + r)];
      std::vector<std::uint64_t> v(ids + at, ids + at + n);
      at += n;
      out[static_cast<std::size_t>(i)].push_back(IdJagged(std::move(v), {n}));
    }
  }
  return out;
}

}  // namespace

extern "C" {

const char* fsref_last_error() { return g_err.c_str(); }

// embedding.cpp:59-64
double fsref_initial_value(std::uint64_t seed, std::uint64_t row, std::uint32_t d) {
  return embedding::initial_value(seed, row, d);
}

// embedding.cpp:82-93 via IndexSet::shard_major (:74-80). Output buffers must
// hold at least ncur / nnext entries.
int fsref_compute_collision(const std::uint64_t* cur, std::uint64_t ncur, const std::uint64_t* next,
                            std::uint64_t nnext, std::uint64_t* co, std::uint64_t* nco,
                            std::uint64_t* exc, std::uint64_t* nexc, std::uint64_t* exn,
                            std::uint64_t* nexn, std::uint64_t* ucur, std::uint64_t* nucur,
                            std::uint64_t* unext, std::uint64_t* nunext) {
  SHIM_TRY
  auto a = embedding::IndexSet::shard_major(IdJagged(std::vector<std::uint64_t>(cur, cur + ncur), {ncur}));
  auto b = embedding::IndexSet::shard_major(IdJagged(std::vector<std::uint64_t>(next, next + nnext), {nnext}));
  auto s = embedding::compute_collision(a, b);
  auto put = [](const std::vector<std::uint64_t>& v, std::uint64_t* dst, std::uint64_t* n) {
    if (!v.empty()) std::memcpy(dst, v.data(), v.size() * 8);
    *n = v.size();
  };
  put(s.collision, co, nco);
  put(s.exclusive_cur, exc, nexc);
  put(s.exclusive_next, exn, nexn);
  put(a.unique_ids, ucur, nucur);
  put(b.unique_ids, unext, nunext);
  SHIM_CATCH
}

// ShardView ctor + apply_gradients (embedding.cpp:108-119, 148-181): a fresh
// shard, one update, then the update result and the full shard values.
int fsref_apply_gradients(std::uint64_t total_rows, std::uint32_t dim, int num_shards, int shard,
                          double lr, std::uint64_t seed, const std::uint64_t* ids, std::uint64_t n,
                          const double* grads, std::uint64_t ngrads, std::uint64_t* uniq,
                          std::uint64_t* nuniq, double* rows, double* values) {
  SHIM_TRY
  embedding::TableGeometry g{total_rows, dim, num_shards};
  embedding::ShardView view(g, shard, lr, seed);
  auto res = view.apply_gradients(std::span<const std::uint64_t>(ids, n),
                                  std::span<const double>(grads, ngrads));
  *nuniq = res.unique_ids.size();
  if (!res.unique_ids.empty()) {
    std::memcpy(uniq, res.unique_ids.data(), res.unique_ids.size() * 8);
    std::memcpy(rows, res.rows.data(), res.rows.size() * 8);
  }
  if (values != nullptr && !view.values().empty())
    std::memcpy(values, view.values().data(), view.values().size() * 8);
  SHIM_CATCH
}

// ShardView::lookup (embedding.cpp:139-146).
int fsref_lookup(std::uint64_t total_rows, std::uint32_t dim, int num_shards, int shard,
                 std::uint64_t seed, const std::uint64_t* ids, std::uint64_t n, double* out) {
  SHIM_TRY
  embedding::TableGeometry g{total_rows, dim, num_shards};
  embedding::ShardView view(g, shard, 0.1, seed);
  auto rows = view.lookup(std::span<const std::uint64_t>(ids, n));
  if (!rows.empty()) std::memcpy(out, rows.data(), rows.size() * 8);
  SHIM_CATCH
}

// route_to_shard_major (embedding.cpp:185-231) on an InProcessFabric. Per rank
// r the outputs are written at the rank's slot:
//   occ_shard[r][N_r]                     (flat, concatenated over ranks)
//   recv_ids[r][...]   recv_lens[r][p]    shard_ids values + per-src lengths
//   uniq[r][...]       nuniq[r]           shard_ids.unique_ids
// Buffers are sized by the caller: occ_shard Σ N_r, recv_ids/uniq Σ N_r each
// (a shard never receives more than all occurrences).
int fsref_route(int world, std::uint64_t total_rows, const std::uint64_t* ids,
                const std::uint64_t* lens, int* occ_shard, std::uint64_t* recv_ids,
                std::uint64_t* recv_lens, std::uint64_t* uniq, std::uint64_t* nuniq) {
  SHIM_TRY
  auto batches = unflatten(ids, lens, 1, world);
  embedding::TableGeometry g{total_rows, 1, world};
  comm::InProcessFabric fabric(world);
  std::vector<embedding::ShardRouting> routes(static_cast<std::size_t>(world));
  fabric.run([&](int rank) {
    comm::Communicator c(fabric.transport(rank));
    routes[static_cast<std::size_t>(rank)] =
        embedding::route_to_shard_major(c, g, batches[0][static_cast<std::size_t>(rank)], {});
  });
  std::size_t occ_at = 0, recv_at = 0, uniq_at = 0;
  for (int r = 0; r < world; ++r) {
    const auto& rt = routes[static_cast<std::size_t>(r)];
    for (int s : rt.occ_shard) occ_shard[occ_at++] = s;
    const auto& vals = rt.shard_ids.ids.values();
    for (auto v : vals) recv_ids[recv_at++] = v;
    for (int s = 0; s < world; ++s) recv_lens[r * world + s] = rt.shard_ids.ids.length(static_cast<std::size_t>(s));
    for (auto v : rt.shard_ids.unique_ids) uniq[uniq_at++] = v;
    nuniq[r] = rt.shard_ids.unique_ids.size();
  }
  SHIM_CATCH
}

// tests/test_embedding.cpp:22-63 (run_engine): drive Synchronized or
// Prioritized embedding over per-(iteration, rank) id batches with gradient
// fixture g = 0.125*row + 0.0625, finalize, gather the full table.
// stats (prioritized only, rank 0): per iteration [collision_rows,
// unique_next_rows, blocking_bytes].
int fsref_run_engine(int prioritized, int world, int iters, const std::uint64_t* ids,
                     const std::uint64_t* lens, std::uint64_t total_rows, std::uint32_t dim,
                     double lr, std::uint64_t seed, double grad_scale, double grad_shift,
                     double* table_out, std::uint64_t* stats_out) {
  SHIM_TRY
  auto batches = unflatten(ids, lens, iters, world);
  embedding::TableGeometry geom{total_rows, dim, world};
  comm::InProcessFabric fabric(world);
  std::vector<std::vector<double>> tables(static_cast<std::size_t>(world));
  std::vector<embedding::IterationStats> stats;
  fabric.run([&](int rank) {
    comm::Communicator c(fabric.transport(rank));
    embedding::ShardView shard(geom, rank, lr, seed);
    std::optional<embedding::SynchronizedEmbedding> sync;
    std::optional<embedding::PrioritizedEmbedding> prio;
    if (prioritized) prio.emplace(shard, c); else sync.emplace(shard, c);
    for (int i = 0; i < iters; ++i) {
      const IdJagged& cur = batches[static_cast<std::size_t>(i)][static_cast<std::size_t>(rank)];
      std::vector<double> rows;
      if (prioritized) {
        const IdJagged* next = i + 1 < iters ? &batches[static_cast<std::size_t>(i) + 1][static_cast<std::size_t>(rank)] : nullptr;
        rows = prio->forward(cur, next);
      } else {
        rows = sync->forward(cur);
      }
      std::vector<double> grads(rows.size());
      for (std::size_t k = 0; k < rows.size(); ++k) grads[k] = grad_scale * rows[k] + grad_shift;
      if (prioritized) prio->backward(grads); else sync->backward(grads);
    }
    if (prio) prio->finalize();
    tables[static_cast<std::size_t>(rank)] = embedding::gather_full_table(c, shard);
    if (rank == 0 && prio) stats = prio->stats();
  });
  if (!tables[0].empty()) std::memcpy(table_out, tables[0].data(), tables[0].size() * 8);
  if (stats_out != nullptr) {
    for (std::size_t i = 0; i < stats.size(); ++i) {
      stats_out[3 * i + 0] = stats[i].collision_rows;
      stats_out[3 * i + 1] = stats[i].unique_next_rows;
      stats_out[3 * i + 2] = stats[i].blocking_bytes;
    }
  }
  SHIM_CATCH
}

// workload::generate_all (workload.cpp:142-241), uniform length distribution,
// flattened to the [iter][rank] layout used above. ids_out must hold
// iters*world*batch*max_uih values.
int fsref_generate_uniform(int world, int batch, std::uint64_t max_uih, std::uint64_t lo,
                           std::uint64_t hi, std::uint64_t table_rows, double target_collision,
                           int has_target, std::uint64_t seed, int iters, std::uint64_t* ids_out,
                           std::uint64_t* lens_out) {
  SHIM_TRY
  workload::WorkloadSpec spec;
  spec.num_ranks = world;
  spec.batch_size = batch;
  spec.max_uih = max_uih;
  spec.dist = workload::DistSpec::uniform(lo, hi);
  spec.table_rows = table_rows;
  if (has_target) spec.target_collision = target_collision;
  spec.seed = seed;
  spec.num_iterations = iters;
  std::size_t at = 0;
  int slot = 0;
  for (const auto& it : workload::generate_all(spec)) {
    for (const auto& b : it) {
      const auto v = b.uih_ids().values();
      for (auto x : v) ids_out[at++] = x;
      lens_out[slot++] = v.size();
    }
  }
  SHIM_CATCH
}

// Empirical length draw (workload.cpp:111-131) for the cfg2 UIH lengths:
// batch lengths of a generator with DistSpec::empirical(hist).
int fsref_generate_lengths(const double* hist, std::uint64_t nhist, std::uint64_t max_uih, int world,
                           int batch, std::uint64_t seed, std::uint64_t* lens_out,
                           std::uint64_t* ncand_out) {
  SHIM_TRY
  workload::WorkloadSpec spec;
  spec.num_ranks = world;
  spec.batch_size = batch;
  spec.max_uih = max_uih;
  spec.dist = workload::DistSpec::empirical(std::vector<double>(hist, hist + nhist));
  spec.table_rows = 1 << 20;
  spec.seed = seed;
  spec.num_iterations = 1;
  workload::Generator gen(spec);
  auto it = gen.next_iteration();
  std::size_t at = 0;
  for (const auto& b : it)
    for (const auto& s : b.samples) {
      lens_out[at] = s.uih.size();
      if (ncand_out) ncand_out[at] = s.candidates.size();
      ++at;
    }
  SHIM_CATCH
}

namespace {
std::vector<partition::GlobalSampleMeta> metas_of(const std::uint64_t* lens, const int* origin,
                                                  const int* local, std::uint64_t m) {
  std::vector<partition::GlobalSampleMeta> metas(m);
  for (std::uint64_t i = 0; i < m; ++i) {
    metas[i].origin_rank = origin[i];
    metas[i].local_index = local[i];
    metas[i].uih_len = lens[i];
  }
  return metas;
}
void put_plan(const partition::PartitionPlan& plan, int* assignment, std::uint64_t* order,
              std::uint64_t* order_lens) {
  std::size_t at = 0;
  for (std::size_t g = 0; g < plan.assignment.size(); ++g) assignment[g] = plan.assignment[g];
  for (std::size_t r = 0; r < plan.receive_order.size(); ++r) {
    order_lens[r] = plan.receive_order[r].size();
    for (auto g : plan.receive_order[r]) order[at++] = g;
  }
}
}  // namespace

// partition.cpp:157-176
int fsref_fbs(const std::uint64_t* lens, const int* origin, const int* local, std::uint64_t m,
              int n, int* assignment, std::uint64_t* order, std::uint64_t* order_lens) {
  SHIM_TRY
  auto metas = metas_of(lens, origin, local, m);
  put_plan(partition::fbs_partition(metas, n), assignment, order, order_lens);
  SHIM_CATCH
}

// partition.cpp:178-209 (no autotune state, or a state given by sizes/emas).
// tune_io (optional, n ints): in = local_batch_size of an initialized state
// (tune_init=1), out = state after the call.
int fsref_vbs(const std::uint64_t* lens, const int* origin, const int* local, std::uint64_t m,
              int n, double alpha, int use_tune, int tune_init, int* tune_sizes,
              int* assignment, std::uint64_t* order, std::uint64_t* order_lens) {
  SHIM_TRY
  auto metas = metas_of(lens, origin, local, m);
  partition::AutoTuneState st;
  if (use_tune && tune_init) {
    st.local_batch_size.assign(tune_sizes, tune_sizes + n);
    st.ema_local.assign(static_cast<std::size_t>(n), 0.0);
    st.initialized = true;
  }
  auto plan = partition::vbs_partition(metas, n, alpha, use_tune ? &st : nullptr);
  if (use_tune) for (int r = 0; r < n; ++r) tune_sizes[r] = st.local_batch_size[static_cast<std::size_t>(r)];
  put_plan(plan, assignment, order, order_lens);
  SHIM_CATCH
}

// partition.cpp:211-269; runs `rounds` updates, times[rounds][n].
int fsref_autotune(int n, int* sizes, double* ema_local, double* ema_global, int step, double delta,
                   double decay, const double* times, int rounds) {
  SHIM_TRY
  partition::AutoTuneState st;
  st.local_batch_size.assign(sizes, sizes + n);
  st.ema_local.assign(ema_local, ema_local + n);
  st.ema_global = *ema_global;
  st.step = step;
  st.delta = delta;
  st.decay = decay;
  st.initialized = true;
  for (int k = 0; k < rounds; ++k)
    partition::autotune_update(st, std::span<const double>(times + static_cast<std::size_t>(k) * n, static_cast<std::size_t>(n)));
  for (int r = 0; r < n; ++r) {
    sizes[r] = st.local_batch_size[static_cast<std::size_t>(r)];
    ema_local[r] = st.ema_local[static_cast<std::size_t>(r)];
  }
  *ema_global = st.ema_global;
  SHIM_CATCH
}

// partition.cpp:292-319
double fsref_bruteforce(const double* w, std::uint64_t m, int segments) {
  return partition::min_max_contiguous_bruteforce(std::span<const double>(w, m), segments);
}

// sim.hpp:24-35
double fsref_cost(double c0, double c1, double c2, const std::uint64_t* lens, std::uint64_t n) {
  sim::CostModel cm;
  cm.c0 = c0;
  cm.c1 = c1;
  cm.c2 = c2;
  return cm.compute_time_for_lengths(std::span<const std::uint64_t>(lens, n));
}

// CPU baseline arm for bench.py: prioritized engine (embedding.cpp:301-607),
// one rank per thread on an InProcessFabric, over the given [iter][rank]
// batches. Returns per-iteration wall µs (max over ranks) in iter_us and the
// per-iteration occurrences served + unique rows updated (summed over ranks)
// in work_rows. Table init (ShardView ctor) is excluded from the timing.
int fsref_bench_engine(int prioritized, int world, int iters, const std::uint64_t* ids,
                       const std::uint64_t* lens, std::uint64_t total_rows, std::uint32_t dim,
                       double lr, std::uint64_t seed, double* iter_us) {
  SHIM_TRY
  auto batches = unflatten(ids, lens, iters, world);
  embedding::TableGeometry geom{total_rows, dim, world};
  comm::InProcessFabric fabric(world);
  std::vector<std::vector<double>> per_rank(static_cast<std::size_t>(world), std::vector<double>(static_cast<std::size_t>(iters)));
  fabric.run([&](int rank) {
    comm::Communicator c(fabric.transport(rank));
    embedding::ShardView shard(geom, rank, lr, seed);
    std::optional<embedding::SynchronizedEmbedding> sync;
    std::optional<embedding::PrioritizedEmbedding> prio;
    if (prioritized) prio.emplace(shard, c); else sync.emplace(shard, c);
    for (int i = 0; i < iters; ++i) {
      auto t0 = std::chrono::steady_clock::now();
      const IdJagged& cur = batches[static_cast<std::size_t>(i)][static_cast<std::size_t>(rank)];
      std::vector<double> rows;
      if (prioritized) {
        const IdJagged* next = i + 1 < iters ? &batches[static_cast<std::size_t>(i) + 1][static_cast<std::size_t>(rank)] : nullptr;
        rows = prio->forward(cur, next);
      } else {
        rows = sync->forward(cur);
      }
      std::vector<double> grads(rows.size());
      for (std::size_t k = 0; k < rows.size(); ++k) grads[k] = 0.125 * rows[k] + 0.0625;
      if (prioritized) prio->backward(grads); else sync->backward(grads);
      auto t1 = std::chrono::steady_clock::now();
      per_rank[static_cast<std::size_t>(rank)][static_cast<std::size_t>(i)] =
          std::chrono::duration<double, std::micro>(t1 - t0).count();
    }
  });
  for (int i = 0; i < iters; ++i) {
    double mx = 0;
    for (int r = 0; r < world; ++r) mx = std::max(mx, per_rank[static_cast<std::size_t>(r)][static_cast<std::size_t>(i)]);
    iter_us[i] = mx;
  }
  SHIM_CATCH
}

// workload::save_workload (workload.cpp:551-557) of generate_all's output for a
// uniform-length spec: a file written by the reference's own Writer, for the
// workload-file replay parity tests.
int fsref_save_workload_uniform(const char* path, int world, int batch, std::uint64_t max_uih,
                                std::uint64_t lo, std::uint64_t hi, std::uint64_t table_rows,
                                std::uint64_t seed, int iters) {
  SHIM_TRY
  workload::WorkloadSpec spec;
  spec.num_ranks = world;
  spec.batch_size = batch;
  spec.max_uih = max_uih;
  spec.dist = workload::DistSpec::uniform(lo, hi);
  spec.table_rows = table_rows;
  spec.seed = seed;
  spec.num_iterations = iters;
  workload::save_workload(path, spec, workload::generate_all(spec));
  SHIM_CATCH
}

// workload::load_workload (workload.cpp:559-564) flattened [iter][rank][sample]:
// counts_out[iter*ranks + rank] = samples, lens_out / labels_out per sample,
// ids_out = uih ids in order. Sizing: with ids_out == nullptr only the totals
// (n_ids, n_samples, dims[0] = ranks, dims[1] = iterations) are written.
int fsref_load_workload(const char* path, std::uint64_t* ids_out, std::uint64_t* lens_out,
                        double* labels_out, std::uint64_t* counts_out, std::uint64_t* n_ids,
                        std::uint64_t* n_samples, int* dims) {
  SHIM_TRY
  auto [spec, its] = workload::load_workload(path);
  dims[0] = spec.num_ranks;
  dims[1] = spec.num_iterations;
  std::uint64_t ni = 0, ns = 0, slot = 0;
  for (const auto& it : its)
    for (const auto& b : it) {
      if (ids_out) counts_out[slot] = b.samples.size();
      ++slot;
      for (const auto& s : b.samples) {
        if (ids_out) {
          lens_out[ns] = s.uih.size();
          labels_out[ns] = s.label;
          for (auto x : s.uih) ids_out[ni++] = x;
        } else {
          ni += s.uih.size();
        }
        ++ns;
      }
    }
  *n_ids = ni;
  *n_samples = ns;
  SHIM_CATCH
}

// ---- pipeline::run (pipeline.cpp:118-323) -----------------------------------------
// The workload is the reference's own generator (generate_all of a uniform-
// length spec); pipeline_samples exports it sample by sample so the B200
// harness runs the same batches: per sample (iteration, rank order) its uih
// length, candidate-list count, label; then all uih ids; then the candidate
// list lengths; then all candidate ids. Sizing: with ids == nullptr only the
// totals are written (n[0] samples, n[1] uih ids, n[2] candidate lists,
// n[3] candidate ids).
namespace {
workload::WorkloadSpec pipeline_spec(int world, int batch, std::uint64_t max_uih, std::uint64_t lo,
                                     std::uint64_t hi, std::uint64_t table_rows, double target, int has_target,
                                     std::uint64_t seed, int iters) {
  workload::WorkloadSpec spec;
  spec.num_ranks = world;
  spec.batch_size = batch;
  spec.max_uih = max_uih;
  spec.dist = workload::DistSpec::uniform(lo, hi);
  spec.table_rows = table_rows;
  if (has_target) spec.target_collision = target;
  spec.seed = seed;
  spec.num_iterations = iters;
  return spec;
}
}  // namespace

int fsref_pipeline_samples(int world, int batch, std::uint64_t max_uih, std::uint64_t lo, std::uint64_t hi,
                           std::uint64_t table_rows, double target, int has_target, std::uint64_t seed, int iters,
                           std::uint64_t* uih_len, std::uint64_t* n_cand, double* label, std::uint64_t* ids,
                           std::uint64_t* cand_len, std::uint64_t* cand_ids, std::uint64_t* n) {
  SHIM_TRY
  const auto spec = pipeline_spec(world, batch, max_uih, lo, hi, table_rows, target, has_target, seed, iters);
  std::uint64_t ns = 0, ni = 0, nc = 0, nci = 0;
  for (const auto& it : workload::generate_all(spec))
    for (const auto& b : it)
      for (const auto& smp : b.samples) {
        if (ids) {
          uih_len[ns] = smp.uih.size();
          n_cand[ns] = smp.candidates.size();
          label[ns] = smp.label;
          for (auto x : smp.uih) ids[ni++] = x;
          for (const auto& c : smp.candidates) {
            cand_len[nc++] = c.size();
            for (auto x : c) cand_ids[nci++] = x;
          }
        } else {
          ni += smp.uih.size();
          nc += smp.candidates.size();
          for (const auto& c : smp.candidates) nci += c.size();
        }
        ++ns;
      }
  n[0] = ns;
  n[1] = ni;
  n[2] = nc;
  n[3] = nci;
  SHIM_CATCH
}

// pipeline::run over that workload. partition: 0 fbs, 1 vbs, 2 none.
// Outputs: the full checkpoint (table checkpoint + dense weights; ckpt_len
// bytes, capacity ckpt_cap), per-iteration losses, final dense weights.
int fsref_pipeline_run(int world, int batch, std::uint64_t max_uih, std::uint64_t lo, std::uint64_t hi,
                       std::uint64_t wl_table_rows, double target, int has_target, std::uint64_t seed, int iters,
                       int prioritized, int balancer, int partition, double alpha, std::uint32_t dim,
                       std::uint64_t table_rows, double lr_emb, double lr_dense, std::uint64_t model_seed,
                       double c0, double c1, double c2, std::uint8_t* ckpt, std::uint64_t ckpt_cap,
                       std::uint64_t* ckpt_len, double* losses, double* dense) {
  SHIM_TRY
  const auto spec = pipeline_spec(world, batch, max_uih, lo, hi, wl_table_rows, target, has_target, seed, iters);
  pipeline::RunConfig cfg;
  cfg.mode = prioritized ? pipeline::Mode::Prioritized : pipeline::Mode::Synchronized;
  cfg.balancer_enabled = balancer != 0;
  cfg.partition = partition == 0 ? "fbs" : partition == 1 ? "vbs" : "none";
  cfg.alpha = alpha;
  cfg.dim = dim;
  cfg.table_rows = table_rows;
  cfg.lr_embedding = lr_emb;
  cfg.lr_dense = lr_dense;
  cfg.model_seed = model_seed;
  cfg.cost.c0 = c0;
  cfg.cost.c1 = c1;
  cfg.cost.c2 = c2;
  const auto res = pipeline::run(workload::generate_all(spec), spec, cfg);
  *ckpt_len = res.full_checkpoint.size();
  if (ckpt && ckpt_cap >= res.full_checkpoint.size())
    std::memcpy(ckpt, res.full_checkpoint.data(), res.full_checkpoint.size());
  for (std::size_t i = 0; i < res.losses.size(); ++i) losses[i] = res.losses[i];
  for (std::size_t d = 0; d < res.final_dense.size(); ++d) dense[d] = res.final_dense[d];
  SHIM_CATCH
}

}  // extern "C"
