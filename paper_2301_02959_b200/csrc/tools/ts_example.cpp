// ts_example — the drop-in C++ flow end to end (what a tiershard user writes):
// synthesize a Zipf table, plan it (host, bit-exact with the reference),
// sample a workload, then train the tiered sequence embedding on the GPU
// through tiershard/device.hpp.  Prints one JSON line.
//
// Usage: ts_example [rows] [dim] [batch] [steps]
#include <cstdio>
#include <cstdlib>
#include <memory>

#include "tiershard/device.hpp"
#include "tiershard/error.hpp"
#include "tiershard/planner.hpp"
#include "tiershard/simulator.hpp"

int main(int argc, char** argv) {
  namespace ts = tiershard;
  const uint64_t rows = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 100000;
  const uint32_t dim = argc > 2 ? static_cast<uint32_t>(std::atoi(argv[2])) : 64;
  const uint32_t batch = argc > 3 ? static_cast<uint32_t>(std::atoi(argv[3])) : 128;
  const int steps = argc > 4 ? std::atoi(argv[4]) : 3;
  try {
    auto dist = std::make_shared<ts::RowDistribution>(ts::synthesize_zipf(rows, 1.05, 32.0, 1));
    ts::Topology topo;
    topo.a2a_global = topo.a2a_intra = topo.ar_global = topo.ar_cross = ts::kGiB;
    ts::CostModelConfig cfg;
    cfg.local_batch = batch;
    cfg.embedding_dim = dim;
    const ts::ShardingPlan plan = ts::plan_2tier(*dist, cfg, topo);
    const ts::Workload wl = ts::sample_workload(dist, cfg, topo, 7, static_cast<uint32_t>(steps));
    ts::DeviceOptions opt;
    opt.optimizer = ts::Optimizer::kRowwiseAdagrad;
    opt.max_occurrences = uint64_t{batch} * 64 * 4;
    ts::SequenceEmbedding table(plan, *dist, topo, cfg, opt);
    ts::IterationBatch b;
    double loss = 0.0;
    uint64_t occ = 0;
    for (int s = 0; s < steps; ++s) {
      wl.materialize_iteration(static_cast<uint32_t>(s), b);
      loss = table.train_step_host(b.rows);
      occ += b.rows.size();
    }
    const std::vector<uint64_t> c = table.counters();
    std::printf("{\"dp_cut\": %llu, \"occurrences\": %llu, \"last_loss\": %.17g, \"served\": %llu, "
                "\"distinct\": %llu}\n",
                static_cast<unsigned long long>(plan.dp_cut), static_cast<unsigned long long>(occ), loss,
                static_cast<unsigned long long>(c[5]), static_cast<unsigned long long>(c[6]));
  } catch (const ts::Error& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 3;
  }
  return 0;
}
