// Test helper for the drop-in workload.hpp (tests/test_cpu_workload_dropin.py):
//   workload_tool gen <world> <batch> <max_uih> <lo> <hi> <table_rows> <target|-1> <seed> <iters> <file>
//       generate_all of a uniform-length spec, save_workload to <file> and the
//       flat dump (below) to <file>.flat
//   workload_tool load <file>
//       load_workload of <file>, the flat dump to <file>.flat
// Flat dump (little-endian u64 unless noted): counts (samples, uih ids,
// candidates, candidate ids), then per sample uih_len, n_cand, label (f64
// bits), then uih ids, candidate lengths, candidate ids — samples in
// (iteration, rank, sample) order, the layout of oracle Reference.pipeline_samples.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "freescale/workload.hpp"

using namespace freescale::workload;

static int dump(const std::vector<std::vector<Batch>>& all, const std::string& path) {
  std::vector<std::uint64_t> len, nc, lab, ids, cl, cid;
  for (const auto& it : all)
    for (const Batch& b : it)
      for (const Sample& s : b.samples) {
        len.push_back(s.uih.size());
        nc.push_back(s.candidates.size());
        std::uint64_t bits;
        std::memcpy(&bits, &s.label, 8);
        lab.push_back(bits);
        ids.insert(ids.end(), s.uih.begin(), s.uih.end());
        for (const auto& c : s.candidates) {
          cl.push_back(c.size());
          cid.insert(cid.end(), c.begin(), c.end());
        }
      }
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return 2;
  const std::uint64_t head[4] = {len.size(), ids.size(), cl.size(), cid.size()};
  std::fwrite(head, 8, 4, f);
  for (const auto* v : {&len, &nc, &lab, &ids, &cl, &cid}) std::fwrite(v->data(), 8, v->size(), f);
  std::fclose(f);
  return 0;
}

int main(int argc, char** argv) {
  try {
    if (argc == 12 && std::string(argv[1]) == "gen") {
      WorkloadSpec s;
      s.num_ranks = std::atoi(argv[2]);
      s.batch_size = std::atoi(argv[3]);
      s.max_uih = std::strtoull(argv[4], nullptr, 10);
      s.dist = DistSpec::uniform(std::strtoull(argv[5], nullptr, 10), std::strtoull(argv[6], nullptr, 10));
      s.table_rows = std::strtoull(argv[7], nullptr, 10);
      const double t = std::atof(argv[8]);
      if (t >= 0) s.target_collision = t;
      s.seed = std::strtoull(argv[9], nullptr, 10);
      s.num_iterations = std::atoi(argv[10]);
      const auto all = generate_all(s);
      save_workload(argv[11], s, all);
      return dump(all, std::string(argv[11]) + ".flat");
    }
    if (argc == 3 && std::string(argv[1]) == "load") {
      const auto [spec, all] = load_workload(argv[2]);
      return dump(all, std::string(argv[2]) + ".flat");
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "usage: workload_tool gen ... | load <file>\n");
  return 2;
}
