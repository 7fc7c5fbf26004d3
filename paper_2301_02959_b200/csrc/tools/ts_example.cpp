// ts_example — the drop-in C++ flow end to end (what a tiershard user writes):
// synthesize a Zipf table, plan it (host, bit-exact with the reference),
// sample a workload, then train the tiered sequence embedding on the GPU
// through tiershard/device.hpp.  Prints one JSON line.
//
// Usage: ts_example [rows] [dim] [batch] [steps]
//        ts_example --plan PLAN.json ASSIGNMENT.csv [steps]
//        ts_example --group N W [rows] [steps]
//   The third form runs a U = N*W-rank job in this process: one thread per
//   rank over a DeviceGroup (rank g on GPU g % device count), each rank
//   stepping its slice of the reference Workload's iterations through
//   train_steps_host; it prints the summed losses and counter columns.
//   The second form imports a plan from the reference's on-disk formats
//   (load_device_plan) and feeds raw (table_id, row_id) keys through a
//   KeyMap; it runs the table on one GPU (topology collapsed to 1 x 1, every
//   tier local) -- a U-GPU job keeps the plan's topology, one rank per process.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <thread>

#include "tiershard/device.hpp"
#include "tiershard/error.hpp"
#include "tiershard/planner.hpp"
#include "tiershard/simulator.hpp"

namespace {

int run_from_plan(const char* plan_json, const char* assignment_csv, int steps) {
  namespace ts = tiershard;
  ts::DevicePlan dp = ts::load_device_plan(plan_json, assignment_csv);
  dp.topology.num_nodes = 1;  // one GPU: every tier local
  dp.topology.gpus_per_node = 1;
  dp.topology.a2a_global = dp.topology.a2a_intra = dp.topology.ar_global = dp.topology.ar_cross = ts::kGiB;
  std::fill(dp.placement.begin(), dp.placement.end(), 0);
  const uint64_t n = dp.table_ids.size();
  const uint64_t occ = uint64_t{dp.cost_model.local_batch} * 16;
  ts::DeviceOptions opt;
  opt.max_occurrences = occ;
  ts::SequenceEmbedding table(dp, opt);
  ts::KeyMap keys(dp);
  std::mt19937_64 rng(17);
  std::vector<uint32_t> h_t(occ);
  std::vector<uint64_t> h_r(occ);
  uint32_t* d_t = nullptr;
  uint64_t* d_r = nullptr;
  float* d_out = nullptr;
  const auto ok = [](cudaError_t e) {
    if (e != cudaSuccess) throw ts::Error(std::string("cuda: ") + cudaGetErrorString(e));
  };
  ok(cudaMalloc(&d_t, sizeof(uint32_t) * occ));
  ok(cudaMalloc(&d_r, sizeof(uint64_t) * occ));
  ok(cudaMalloc(&d_out, sizeof(float) * occ * table.dim()));
  double loss = 0.0;
  for (int s = 0; s < steps; ++s) {
    for (uint64_t i = 0; i < occ; ++i) {  // raw keys of plan rows, hot rows first-weighted
      const uint64_t k = (rng() % n) * (rng() % n) / n;
      h_t[i] = dp.table_ids[k];
      h_r[i] = dp.row_ids[k];
    }
    ok(cudaMemcpy(d_t, h_t.data(), sizeof(uint32_t) * occ, cudaMemcpyHostToDevice));
    ok(cudaMemcpy(d_r, h_r.data(), sizeof(uint64_t) * occ, cudaMemcpyHostToDevice));
    table.forward_keys(keys, d_t, d_r, occ, d_out);
    table.backward(d_out);  // grad = out: loss 0.5 |out|^2
    table.synchronize();
    std::vector<float> h_out(occ * table.dim());
    ok(cudaMemcpy(h_out.data(), d_out, sizeof(float) * h_out.size(), cudaMemcpyDeviceToHost));
    loss = 0.0;
    for (float v : h_out) loss += 0.5 * double(v) * double(v);
  }
  cudaFree(d_t);
  cudaFree(d_r);
  cudaFree(d_out);
  std::printf("{\"rows\": %llu, \"dp_cut\": %llu, \"flex_cut\": %llu, \"occurrences\": %llu, "
              "\"last_loss\": %.17g}\n",
              static_cast<unsigned long long>(n), static_cast<unsigned long long>(dp.plan.dp_cut),
              static_cast<unsigned long long>(dp.plan.flex_cut),
              static_cast<unsigned long long>(occ * steps), loss);
  return 0;
}

int run_group(uint32_t nodes, uint32_t w, uint64_t rows, int steps) {
  namespace ts = tiershard;
  const uint32_t u = nodes * w, batch = 64, dim = 64;
  auto dist = std::make_shared<ts::RowDistribution>(ts::synthesize_zipf(rows, 1.05, 32.0, 1));
  ts::Topology topo;
  topo.num_nodes = nodes;
  topo.gpus_per_node = w;
  topo.a2a_global = topo.a2a_intra = topo.ar_global = topo.ar_cross = ts::kGiB;
  ts::CostModelConfig cfg;
  cfg.local_batch = batch;
  cfg.embedding_dim = dim;
  const ts::ShardingPlan plan = ts::plan_2tier(*dist, cfg, topo);
  const ts::Workload wl = ts::sample_workload(dist, cfg, topo, 7, static_cast<uint32_t>(steps));
  std::vector<ts::IterationBatch> iters(static_cast<size_t>(steps));
  uint64_t max_occ = 1;
  for (int s = 0; s < steps; ++s) {
    wl.materialize_iteration(static_cast<uint32_t>(s), iters[s]);
    for (uint32_t g = 0; g < u; ++g) {
      max_occ = std::max<uint64_t>(max_occ, iters[s].sample_offsets[(g + 1) * batch] - iters[s].sample_offsets[g * batch]);
    }
  }
  int devices = 1;
  if (cudaGetDeviceCount(&devices) != cudaSuccess || devices < 1) throw ts::Error("no CUDA device");
  ts::DeviceGroup group(u);
  std::vector<double> loss(u, 0.0);
  std::vector<std::vector<uint64_t>> counters(u);
  std::vector<std::exception_ptr> errors(u);
  std::vector<std::thread> threads;
  for (uint32_t g = 0; g < u; ++g) {
    threads.emplace_back([&, g] {
      try {
        ts::DeviceOptions opt;
        opt.device = static_cast<int>(g % static_cast<uint32_t>(devices));
        opt.rank = g;
        opt.group = &group;
        opt.max_occurrences = max_occ;
        ts::SequenceEmbedding table(plan, *dist, topo, cfg, opt);
        std::vector<const uint32_t*> ptrs;
        std::vector<uint64_t> occ;
        for (const ts::IterationBatch& b : iters) {
          const uint64_t lo = b.sample_offsets[g * batch], hi = b.sample_offsets[(g + 1) * batch];
          ptrs.push_back(b.rows.data() + lo);
          occ.push_back(hi - lo);
        }
        const std::vector<double> l = table.train_steps_host(ptrs, occ);
        loss[g] = l.back();
        table.synchronize();
        counters[g] = table.counters();
      } catch (...) {
        errors[g] = std::current_exception();
        group.abort();
      }
    });
  }
  for (auto& t : threads) t.join();
  for (auto& e : errors) {
    if (e) std::rethrow_exception(e);
  }
  std::vector<uint64_t> sum(7 * u, 0);
  double total = 0.0;
  for (uint32_t g = 0; g < u; ++g) {
    total += loss[g];
    for (size_t i = 0; i < sum.size(); ++i) sum[i] += counters[g][i];
  }
  uint64_t served = 0;
  for (uint32_t g = 0; g < u; ++g) served += sum[5 * u + g];
  std::printf("{\"ranks\": %u, \"devices\": %d, \"dp_cut\": %llu, \"last_loss_sum\": %.17g, "
              "\"last_iteration_occurrences\": %llu, \"served\": %llu}\n",
              u, devices, static_cast<unsigned long long>(plan.dp_cut), total,
              static_cast<unsigned long long>(iters.back().rows.size()), static_cast<unsigned long long>(served));
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  namespace ts = tiershard;
  if (argc > 1 && std::strcmp(argv[1], "--group") == 0) {
    if (argc < 4) {
      std::fprintf(stderr, "usage: %s --group N W [rows] [steps]\n", argv[0]);
      return 2;
    }
    try {
      return run_group(static_cast<uint32_t>(std::atoi(argv[2])), static_cast<uint32_t>(std::atoi(argv[3])),
                       argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 50000, argc > 5 ? std::atoi(argv[5]) : 3);
    } catch (const ts::Error& e) {
      std::printf("{\"error\": \"%s\"}\n", e.what());
      return 3;
    }
  }
  if (argc > 1 && std::strcmp(argv[1], "--plan") == 0) {
    if (argc < 4) {
      std::fprintf(stderr, "usage: %s --plan PLAN.json ASSIGNMENT.csv [steps]\n", argv[0]);
      return 2;
    }
    try {
      return run_from_plan(argv[2], argv[3], argc > 4 ? std::atoi(argv[4]) : 3);
    } catch (const ts::Error& e) {
      std::printf("{\"error\": \"%s\"}\n", e.what());
      return 3;
    }
  }
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
