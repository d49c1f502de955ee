// The reference's own test cases (proj/tests/test_embedding.cpp,
// test_partition.cpp, test_sim.cpp), rewritten against the drop-in headers:
// the same calls a reference user makes, now executed by libfsx on the GPU.
// Built and run by tests/test_gpu_dropin.py; exit 0 iff every check passes.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <optional>
#include <string>
#include <vector>

#include "freescale/embedding.hpp"
#include "freescale/partition.hpp"

using namespace freescale;
using namespace freescale::embedding;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                              \
  do {                                                                        \
    if (c) ++g_pass;                                                          \
    else { ++g_fail; std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c); } \
  } while (0)
template <class E, class F>
bool throws(F f, const char* sub = nullptr) {
  try { f(); } catch (const E& e) { return !sub || std::string(e.what()).find(sub) != std::string::npos; }
  catch (...) { return false; }
  return false;
}

static IndexSet shard_set(std::vector<std::vector<std::uint64_t>> segs) {
  return IndexSet::shard_major(IdJagged::from_segments(segs));
}

// test_embedding.cpp:22-63
static std::vector<double> run_engine(bool prio, const std::vector<std::vector<IdJagged>>& ids,
                                      TableGeometry geom, double lr, std::uint64_t seed) {
  const int world = geom.num_shards, iters = static_cast<int>(ids.size());
  comm::InProcessFabric fabric(world);
  std::vector<std::vector<double>> tables(static_cast<size_t>(world));
  fabric.run([&](int rank) {
    comm::Communicator c(fabric.transport(rank));
    ShardView shard(geom, rank, lr, seed);
    std::optional<SynchronizedEmbedding> sync;
    std::optional<PrioritizedEmbedding> pr;
    if (prio) pr.emplace(shard, c); else sync.emplace(shard, c);
    for (int i = 0; i < iters; ++i) {
      const IdJagged& cur = ids[static_cast<size_t>(i)][static_cast<size_t>(rank)];
      std::vector<double> rows = prio ? pr->forward(cur, i + 1 < iters ? &ids[static_cast<size_t>(i) + 1][static_cast<size_t>(rank)] : nullptr)
                                      : sync->forward(cur);
      std::vector<double> g(rows.size());
      for (size_t k = 0; k < rows.size(); ++k) g[k] = 0.125 * rows[k] + 0.0625;
      if (prio) pr->backward(g); else sync->backward(g);
    }
    if (pr) pr->finalize();
    tables[static_cast<size_t>(rank)] = gather_full_table(c, shard);
  });
  for (int r = 1; r < world; ++r) CHECK(tables[static_cast<size_t>(r)] == tables[0]);
  return tables[0];
}

static std::uint64_t lcg(std::uint64_t& s) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return s >> 33; }

int main() {
  // ---- collision (test_embedding.cpp:79-108)
  {
    auto s = compute_collision(shard_set({{1, 2, 3}}), shard_set({{2, 4}}));
    CHECK((s.collision == std::vector<std::uint64_t>{2}));
    CHECK((s.exclusive_cur == std::vector<std::uint64_t>{1, 3}));
    CHECK((s.exclusive_next == std::vector<std::uint64_t>{4}));
    CHECK(compute_collision(shard_set({{1}}), shard_set({{2}})).collision.empty());
    auto same = compute_collision(shard_set({{5, 6}}), shard_set({{6, 5}}));
    CHECK((same.collision == std::vector<std::uint64_t>{5, 6}) && same.exclusive_cur.empty());
    CHECK(throws<std::invalid_argument>([] { compute_collision(IndexSet::batch_major(IdJagged::from_segments({{1}})), shard_set({{1}})); }));
    CHECK(std::abs(collision_pct(shard_set({{1, 2, 3}}), shard_set({{2, 4}})) - 0.5) < 1e-12);
    CHECK(throws<std::invalid_argument>([] { collision_pct(shard_set({{1}}), shard_set({std::vector<std::uint64_t>{}})); }));
  }
  // ---- lookup / apply_gradients (test_embedding.cpp:131-170)
  {
    TableGeometry geom{4, 2, 1};
    ShardView shard(geom, 0, 1.0, 9);
    auto rows = shard.lookup(std::vector<std::uint64_t>{2, 0});
    CHECK(rows[0] == shard.row(2)[0] && rows[1] == shard.row(2)[1] && rows[2] == shard.row(0)[0]);
    CHECK(shard.lookup(std::vector<std::uint64_t>{}).empty());
    auto dup = shard.lookup(std::vector<std::uint64_t>{1, 1});
    CHECK(dup[0] == dup[2] && dup[1] == dup[3]);
    CHECK(throws<std::domain_error>([&] { shard.lookup(std::vector<std::uint64_t>{4}); }, "row id 4"));
    CHECK(shard.row(3)[1] == initial_value(9, 3, 1));
  }
  {
    TableGeometry geom{2, 2, 1};
    ShardView shard(geom, 0, 1.0, 1);
    const double v0 = shard.row(0)[0], v1 = shard.row(0)[1];
    shard.apply_gradients(std::vector<std::uint64_t>{0}, std::vector<double>{v0 - 1.0, v1 - 1.0});
    CHECK(std::abs(shard.row(0)[0] - 1.0) < 1e-12);
    auto res = shard.apply_gradients(std::vector<std::uint64_t>{0}, std::vector<double>{0.5, 0.0});
    CHECK(std::abs(res.rows[0] - 0.5) < 1e-12 && std::abs(res.rows[1] - 1.0) < 1e-12);
    const std::vector<double> before(shard.values());
    shard.apply_gradients(std::vector<std::uint64_t>{0, 1}, std::vector<double>{0, 0, 0, 0});
    CHECK(shard.values() == before);
    ShardView a(geom, 0, 0.5, 3), b(geom, 0, 0.5, 3);
    a.apply_gradients(std::vector<std::uint64_t>{1, 1}, std::vector<double>{0.25, 0.5, 0.125, 0.25});
    b.apply_gradients(std::vector<std::uint64_t>{1}, std::vector<double>{0.25, 0.5});
    b.apply_gradients(std::vector<std::uint64_t>{1}, std::vector<double>{0.125, 0.25});
    CHECK(a.values() == b.values());
    CHECK(throws<std::invalid_argument>([&] { a.apply_gradients(std::vector<std::uint64_t>{0}, std::vector<double>{1.0}); }));
  }
  // ---- synchronized single rank == dense table (test_embedding.cpp:209-235)
  {
    TableGeometry geom{8, 2, 1};
    const double lr = 0.5;
    std::vector<double> dense(16);
    for (std::uint64_t g = 0; g < 8; ++g)
      for (std::uint32_t d = 0; d < 2; ++d) dense[g * 2 + d] = initial_value(11, g, d);
    std::vector<std::vector<IdJagged>> ids;
    std::uint64_t rng = 77;
    for (int i = 0; i < 4; ++i) {
      std::vector<std::uint64_t> flat(6);
      for (auto& x : flat) x = lcg(rng) % 8;
      ids.push_back({IdJagged(flat, {3, 3})});
      std::vector<double> rows(12), acc(16, 0.0);
      for (size_t k = 0; k < 6; ++k) for (int d = 0; d < 2; ++d) rows[k * 2 + d] = dense[flat[k] * 2 + d];
      for (size_t k = 0; k < 6; ++k) for (int d = 0; d < 2; ++d) acc[flat[k] * 2 + d] += 0.125 * rows[k * 2 + d] + 0.0625;
      for (size_t g = 0; g < 8; ++g) for (int d = 0; d < 2; ++d) dense[g * 2 + d] -= lr * acc[g * 2 + d];
    }
    CHECK(run_engine(false, ids, geom, lr, 11) == dense);
    CHECK(run_engine(true, ids, geom, lr, 11) == dense);
  }
  // ---- parity prioritized == synchronized across ranks (test_embedding.cpp:253-282)
  for (int ranks : {1, 2, 4}) {
    std::uint64_t rng = 99 + ranks;
    std::vector<std::vector<IdJagged>> ids;
    for (int i = 0; i < 7; ++i) {
      std::vector<IdJagged> per;
      for (int r = 0; r < ranks; ++r) {
        std::vector<std::uint64_t> v(lcg(rng) % 13);
        for (auto& x : v) x = lcg(rng) % 64;
        per.push_back(IdJagged(v, {v.size()}));
      }
      ids.push_back(per);
    }
    TableGeometry geom{64, 3, ranks};
    CHECK(run_engine(false, ids, geom, 0.125, 5) == run_engine(true, ids, geom, 0.125, 5));
  }
  {
    TableGeometry geom{16, 2, 2};
    std::vector<std::vector<IdJagged>> one = {{IdJagged::from_segments({{1, 2}}), IdJagged::from_segments({{3, 1}})}};
    CHECK(run_engine(false, one, geom, 0.5, 7) == run_engine(true, one, geom, 0.5, 7));
    auto two = one;
    two.push_back({IdJagged::from_segments({{2, 2, 5}}), IdJagged::from_segments({{1}})});
    CHECK(run_engine(false, two, geom, 0.5, 7) == run_engine(true, two, geom, 0.5, 7));
  }
  // ---- protocol order errors (test_embedding.cpp:329-342)
  {
    TableGeometry geom{4, 1, 1};
    comm::InProcessFabric fabric(1);
    fabric.run([&](int rank) {
      comm::Communicator c(fabric.transport(rank));
      ShardView shard(geom, rank, 0.1, 1);
      PrioritizedEmbedding prio(shard, c);
      std::vector<double> g{0.0};
      CHECK(throws<ProtocolError>([&] { prio.backward(g); }));
      auto ids = IdJagged::from_segments({{1}});
      prio.forward(ids, nullptr);
      CHECK(throws<ProtocolError>([&] { prio.forward(ids, nullptr); }));
    });
  }
  // ---- checkpoint header (test_embedding.cpp:344-352)
  {
    TableGeometry geom{4, 2, 2};
    std::vector<double> table(8, 1.5);
    auto blob = checkpoint_bytes(geom, table);
    std::uint64_t rows = 0;
    std::memcpy(&rows, blob.data(), 8);
    CHECK(blob.size() == 24 + 64 && rows == 4);
  }
  // ---- partition (test_partition.cpp:38-139)
  {
    using namespace freescale::partition;
    auto metas = [](std::vector<std::uint64_t> l, int n) {
      std::vector<GlobalSampleMeta> m(l.size());
      const size_t per = (l.size() + n - 1) / n;
      for (size_t i = 0; i < l.size(); ++i) { m[i].origin_rank = int(i / per); m[i].local_index = int(i % per); m[i].uih_len = l[i]; }
      return m;
    };
    auto m1 = metas({9, 7, 5, 3}, 2);
    auto p1 = fbs_partition(m1, 2);
    p1.validate(4, true);
    std::uint64_t t0 = 0, t1 = 0;
    for (auto g : p1.receive_order[0]) t0 += m1[g].uih_len;
    for (auto g : p1.receive_order[1]) t1 += m1[g].uih_len;
    CHECK(t0 == 12 && t1 == 12);
    CHECK((fbs_partition(metas({3, 9, 1}, 1), 1).receive_order[0] == std::vector<std::size_t>{1, 0, 2}));
    CHECK(throws<std::invalid_argument>([&] { fbs_partition(metas({1, 2, 3}, 2), 2); }));
    auto m2 = metas({4, 3, 2, 1}, 2);
    auto p2 = vbs_partition(m2, 2, 1.0);
    CHECK(std::abs(plan_max_weight(p2, m2, 1.0) - 6.0) < 1e-12 && p2.receive_order[0].size() == 1);
    CHECK(throws<std::invalid_argument>([&] { vbs_partition(metas({5, 4}, 2), 3, 1.0); }));
    AutoTuneState tune;
    tune.local_batch_size = {4, 4};
    tune.ema_local = {0, 0};
    tune.initialized = true;
    autotune_update(tune, std::vector<double>{12, 8});
    CHECK((tune.local_batch_size == std::vector<int>{3, 5}));
    sim::CostModel cm;
    cm.c0 = 50; cm.c1 = 0.01; cm.c2 = 1e-6;
    std::vector<std::uint64_t> lens{16, 8192, 97, 1000};
    CHECK(cm.compute_time_for_lengths(lens) == 0x1.a656496ededafp+7);
  }
  std::printf("dropin: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
