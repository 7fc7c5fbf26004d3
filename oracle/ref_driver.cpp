// ref_driver — JSON front-end over the UNMODIFIED reference library
// (tiershard v0.1.0, /root/reference/proj), compiled by oracle/Makefile into
// oracle/_ref/.  Test infrastructure only: it is the checker the parity tests,
// the golden-fixture generator (tests/golden/make_golden.py) and bench.py's
// reference arm run.  It calls nothing but the reference's public API:
//
//   synthesize_zipf / merge          proj/include/tiershard/distribution.hpp:88-98
//   find_breakpoints                 proj/include/tiershard/cost_model.hpp:100
//   build_frontier / find_points     proj/include/tiershard/planner.hpp:46-63
//   plan_2tier / plan_3tier /        proj/include/tiershard/planner.hpp:125-147
//     plan_for_budget / predict_cost
//   sample_workload / Workload       proj/include/tiershard/simulator.hpp:38-66
//   assign_rows                      proj/include/tiershard/simulator.hpp:83-86
//   simulate / compare_to_baseline / proj/include/tiershard/simulator.hpp:136-172
//     compare
//   to_json(...)                     proj/include/tiershard/json_io.hpp:22-29
//
// Usage: ref_driver SPEC.json [OUT.json]     (OUT defaults to stdout)
// The spec format is documented in oracle/README.md; our own product driver
// (paper_2301_02959_b200 ts_driver) accepts the same spec and emits the same
// keys so the tests can compare the two documents field by field.

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"
#include "tiershard/cost_model.hpp"
#include "tiershard/distribution.hpp"
#include "tiershard/error.hpp"
#include "tiershard/hashing.hpp"
#include "tiershard/json_io.hpp"
#include "tiershard/planner.hpp"
#include "tiershard/simulator.hpp"
#include "tiershard/topology.hpp"
#include "tiershard/version.hpp"

using nlohmann::json;
namespace ts = tiershard;

namespace {

double now_s() {
  using clk = std::chrono::steady_clock;
  return std::chrono::duration<double>(clk::now().time_since_epoch()).count();
}

ts::Topology topo_from(const json& j) {
  ts::Topology t;
  t.num_nodes = j.at("num_nodes").get<uint32_t>();
  t.gpus_per_node = j.at("gpus_per_node").get<uint32_t>();
  t.a2a_global = j.at("a2a_global_gibs").get<double>() * ts::kGiB;
  t.a2a_intra = j.at("a2a_intra_gibs").get<double>() * ts::kGiB;
  t.ar_global = j.at("ar_global_gibs").get<double>() * ts::kGiB;
  t.ar_cross = j.at("ar_cross_gibs").get<double>() * ts::kGiB;
  t.validate();
  return t;
}

ts::CostModelConfig cfg_from(const json& j) {
  ts::CostModelConfig c;
  if (j.contains("local_batch")) c.local_batch = j["local_batch"];
  if (j.contains("embedding_dim")) c.embedding_dim = j["embedding_dim"];
  if (j.contains("scalar_bytes")) c.scalar_bytes = j["scalar_bytes"];
  if (j.contains("dp_replication_multiplier"))
    c.dp_replication_multiplier = j["dp_replication_multiplier"];
  if (j.contains("dynamic_pass_count")) c.dynamic_pass_count = j["dynamic_pass_count"];
  if (j.contains("static_pass_count")) c.static_pass_count = j["static_pass_count"];
  if (j.contains("include_id_bytes")) c.include_id_bytes = j["include_id_bytes"];
  if (j.contains("bytes_per_id")) c.bytes_per_id = j["bytes_per_id"];
  if (j.contains("count_dynamic_memory")) c.count_dynamic_memory = j["count_dynamic_memory"];
  c.validate();
  return c;
}

// Order-sensitive digest of the canonical row order (table, row, p bits).
uint64_t dist_digest(const ts::RowDistribution& d) {
  uint64_t h = 0x243F6A8885A308D3ull;
  for (const ts::RowRecord& r : d.rows()) {
    uint64_t pb;
    std::memcpy(&pb, &r.probability, 8);
    h = ts::mix64(h ^ r.table_id);
    h = ts::mix64(h ^ r.row_id);
    h = ts::mix64(h ^ pb);
  }
  return h;
}

uint64_t placement_digest(const std::vector<ts::RowPlacement>& p) {
  uint64_t h = 0x13198A2E03707344ull;
  for (const ts::RowPlacement& x : p) {
    h = ts::mix64(h ^ static_cast<uint64_t>(x.tier));
    h = ts::mix64(h ^ x.owner_gpu);
    h = ts::mix64(h ^ x.flex_slot);
  }
  return h;
}

json sim_json(const ts::SimReport& r) {
  json j;
  j["seed"] = r.seed;
  j["hash_seed"] = r.hash_seed;
  j["num_iterations"] = r.num_iterations;
  json its = json::array();
  for (const auto& m : r.iterations) its.push_back(ts::to_json(m));
  j["iterations"] = its;
  j["mean"] = ts::to_json(r.mean);
  return j;
}

template <typename T>
void dump_vec(const std::string& path, const std::vector<T>& v) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw ts::ConfigError("ref_driver: cannot write " + path);
  f.write(reinterpret_cast<const char*>(v.data()),
          static_cast<std::streamsize>(v.size() * sizeof(T)));
}

json run(const json& spec) {
  json out;
  out["tool"] = "tiershard-reference";
  out["version"] = std::string(ts::kVersion);
  json timing;

  if (spec.value("hash_vectors", false)) {
    // Known answers of the integer primitives (hashing.hpp, rng.hpp).
    ts::SplitMix64 rng(7);
    const uint64_t r0 = rng.next_u64();
    const uint64_t r1 = rng.next_u64();
    json pois = json::array();
    ts::SplitMix64 prng(11);
    for (double mean : {0.5, 3.0, 9.99, 10.0, 32.0, 1024.0}) {
      json draws = json::array();
      for (int k = 0; k < 8; ++k) draws.push_back(ts::poisson(prng, mean));
      pois.push_back({{"mean", mean}, {"draws", draws}});
    }
    out["hash"] = {{"mix64_0", ts::mix64(0)},
                   {"mix64_1", ts::mix64(1)},
                   {"row_key_hash_0_0_2", ts::row_key_hash(0, 0, 2)},
                   {"row_key_hash_3_12345_2", ts::row_key_hash(3, 12345, 2)},
                   {"derive_seed_7_0", ts::derive_seed(7, 0)},
                   {"splitmix64_7", {r0, r1}},
                   {"poisson_seed11", pois}};
    return out;
  }

  // ---- distribution -------------------------------------------------------
  double t0 = now_s();
  std::vector<ts::RowDistribution> parts;
  for (const json& t : spec.at("tables")) {
    parts.push_back(ts::synthesize_zipf(
        t.at("rows").get<uint64_t>(), t.at("exponent").get<double>(),
        t.at("target_length").get<double>(), t.at("seed").get<uint64_t>(),
        t.value("table_id", 0u)));
  }
  auto dist = std::make_shared<ts::RowDistribution>(
      parts.size() == 1 ? std::move(parts[0]) : ts::merge(parts));
  parts.clear();
  timing["synth_merge_s"] = now_s() - t0;

  const ts::RowDistribution& d = *dist;
  json jd;
  jd["rows"] = d.rows().size();
  jd["capacity"] = d.capacity();
  jd["num_samples"] = d.num_samples();
  jd["expected_length"] = d.expected_length();
  jd["digest"] = dist_digest(d);
  json head = json::array();
  const size_t nh = std::min<size_t>(d.rows().size(), spec.value("head_rows", 16));
  for (size_t i = 0; i < nh; ++i) {
    const auto& r = d.rows()[i];
    head.push_back({r.table_id, r.row_id, r.probability});
  }
  jd["head"] = head;
  out["distribution"] = jd;

  const ts::Topology topo = topo_from(spec.at("topology"));
  const ts::CostModelConfig cfg = cfg_from(spec.value("cost_model", json::object()));

  // ---- breakpoints + frontier ----------------------------------------------
  const ts::Breakpoints bp = ts::find_breakpoints(cfg, topo);
  out["breakpoints"] = ts::to_json(bp);
  t0 = now_s();
  if (spec.value("frontier", true)) {
    const ts::Frontier fr = ts::build_frontier(d, cfg, topo, ts::Strategy::kDataParallel);
    const ts::FrontierLandmarks lm = ts::find_points(fr, d, cfg, topo);
    out["landmarks"] = {{"a", lm.a}, {"b", lm.b}, {"c", lm.c}, {"d", lm.d}};
    json samples = json::array();
    std::vector<size_t> ks = {0, lm.a, lm.b, lm.c, lm.d};
    for (const json& k : spec.value("frontier_points", json::array())) ks.push_back(k);
    for (size_t k : ks) {
      if (k < fr.size()) samples.push_back({k, fr.memory_at(k), fr.comm_at(k)});
    }
    out["frontier_dp"] = samples;
    if (topo.has_fast_intra_tier()) {
      const ts::Frontier ff = ts::build_frontier(d, cfg, topo, ts::Strategy::kFlex);
      json fs = json::array();
      for (size_t k : ks) {
        if (k < ff.size()) fs.push_back({k, ff.memory_at(k), ff.comm_at(k)});
      }
      out["frontier_flex"] = fs;
    }
  }
  timing["frontier_s"] = now_s() - t0;

  // ---- plan ------------------------------------------------------------------
  t0 = now_s();
  const std::string goal = spec.value("goal", std::string("2tier"));
  ts::ShardingPlan plan;
  if (goal == "2tier") {
    plan = ts::plan_2tier(d, cfg, topo);
  } else if (goal == "3tier") {
    plan = ts::plan_3tier(d, cfg, topo);
  } else if (goal == "budget") {
    plan = ts::plan_for_budget(d, cfg, topo, spec.at("budget_bytes").get<double>(),
                               spec.value("allow_flex", false));
  } else if (goal == "rw" || goal == "cuts") {
    plan.dp_cut = goal == "rw" ? 0 : spec.at("dp_cut").get<uint64_t>();
    plan.flex_cut = goal == "rw" ? 0 : spec.at("flex_cut").get<uint64_t>();
    plan.total_rows = d.rows().size();
    plan.goal = goal;
    plan.predicted = ts::predict_cost(d, plan.dp_cut, plan.flex_cut, cfg, topo);
  } else {
    throw ts::ConfigError("ref_driver: unknown goal " + goal);
  }
  timing["plan_s"] = now_s() - t0;
  json jp;
  jp["dp_cut"] = plan.dp_cut;
  jp["flex_cut"] = plan.flex_cut;
  jp["total_rows"] = plan.total_rows;
  jp["goal"] = plan.goal;
  jp["warnings"] = plan.warnings;
  jp["achieved_memory_bytes"] =
      plan.achieved_memory_bytes ? json(*plan.achieved_memory_bytes) : json();
  jp["achieved_comm_seconds"] =
      plan.achieved_comm_seconds ? json(*plan.achieved_comm_seconds) : json();
  jp["predicted"] = ts::to_json(plan.predicted);
  out["plan"] = jp;
  out["coverage"] = {
      {"dp", ts::to_json(ts::coverage_report(plan, d).dp)},
      {"flex", ts::to_json(ts::coverage_report(plan, d).flex)},
      {"rw", ts::to_json(ts::coverage_report(plan, d).rw)}};

  const uint64_t hash_seed = spec.value("hash_seed", ts::kDefaultPlacementSeed);
  const auto placements = ts::assign_rows(plan, d, topo, hash_seed);
  out["placements_digest"] = placement_digest(placements);

  const std::string dump_dir = spec.value("dump_dir", std::string());
  if (!dump_dir.empty()) {
    std::vector<uint8_t> tier(placements.size());
    std::vector<uint32_t> owner(placements.size()), slot(placements.size());
    for (size_t i = 0; i < placements.size(); ++i) {
      tier[i] = static_cast<uint8_t>(placements[i].tier);
      owner[i] = placements[i].owner_gpu;
      slot[i] = placements[i].flex_slot;
    }
    dump_vec(dump_dir + "/placements.tier.u8", tier);
    dump_vec(dump_dir + "/placements.owner.u32", owner);
    dump_vec(dump_dir + "/placements.slot.u32", slot);
    std::vector<uint32_t> dt(d.rows().size());
    std::vector<uint64_t> dr(d.rows().size());
    std::vector<double> dpv(d.rows().size());
    for (size_t i = 0; i < d.rows().size(); ++i) {
      dt[i] = d.rows()[i].table_id;
      dr[i] = d.rows()[i].row_id;
      dpv[i] = d.rows()[i].probability;
    }
    dump_vec(dump_dir + "/dist.table.u32", dt);
    dump_vec(dump_dir + "/dist.row.u64", dr);
    dump_vec(dump_dir + "/dist.p.f64", dpv);
  }

  // ---- workload + simulation -------------------------------------------------
  if (!spec.contains("workload")) {
    out["timing"] = timing;
    return out;
  }
  const json& jw = spec["workload"];
  const uint64_t wseed = jw.value("seed", uint64_t{7});
  const uint32_t iters = jw.value("iterations", 1u);
  unsigned threads = spec.value("threads", 1u);
  if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
  timing["threads"] = threads;

  t0 = now_s();
  const ts::Workload wl = ts::sample_workload(dist, cfg, topo, wseed, iters);
  timing["workload_build_s"] = now_s() - t0;

  if (jw.value("materialize_pass", true)) {
    ts::IterationBatch batch;
    json occ = json::array();
    t0 = now_s();
    for (uint32_t it = 0; it < iters; ++it) {
      wl.materialize_iteration(it, batch);
      occ.push_back(batch.occurrences());
      if (!dump_dir.empty() && jw.value("dump_batches", false)) {
        dump_vec(dump_dir + "/batch_" + std::to_string(it) + ".rows.u32", batch.rows);
        dump_vec(dump_dir + "/batch_" + std::to_string(it) + ".offsets.u64",
                 batch.sample_offsets);
      }
    }
    timing["materialize_total_s_1thread"] = now_s() - t0;
    out["occurrences"] = occ;
  }

  if (jw.value("materialize_parallel", false)) {
    // the sampling share of simulate(): every iteration materialized by the
    // same number of threads pulling iterations from an atomic counter, the
    // way simulate()'s pool does (simulator.cpp:336-364), without routing --
    // bench.py subtracts it to time routing + accounting alone
    std::atomic<uint32_t> next{0};
    std::atomic<uint64_t> occ_sum{0};
    t0 = now_s();
    std::vector<std::thread> pool;
    for (unsigned k = 0; k < threads; ++k) {
      pool.emplace_back([&] {
        ts::IterationBatch batch;
        for (uint32_t it = next++; it < iters; it = next++) {
          wl.materialize_iteration(it, batch);
          occ_sum += batch.occurrences();
        }
      });
    }
    for (auto& th : pool) th.join();
    timing["materialize_parallel_s"] = now_s() - t0;
    timing["materialize_parallel_occurrences"] = occ_sum.load();
  }

  if (spec.value("simulate", true)) {
    t0 = now_s();
    const ts::SimReport rep = ts::simulate(plan, wl, cfg, topo, hash_seed, threads);
    timing["simulate_s"] = now_s() - t0;
    out["sim"] = sim_json(rep);
    out["discrepancies"] = ts::to_json(ts::compare(plan.predicted, rep, 0.02));
    if (spec.value("baseline", false)) {
      ts::ShardingPlan rw;
      rw.total_rows = d.rows().size();
      rw.goal = "rw";
      rw.predicted = ts::predict_cost(d, 0, 0, cfg, topo);
      const ts::SimReport base = ts::simulate(rw, wl, cfg, topo, hash_seed, threads);
      out["baseline_sim"] = sim_json(base);
      out["comparison"] = ts::to_json(ts::compare_to_baseline(base, rep));
    }
  }
  out["timing"] = timing;
  return out;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver SPEC.json [OUT.json]\n");
    return 2;
  }
  auto emit = [&](const json& j) {
    if (argc >= 3) {
      std::ofstream(argv[2]) << j.dump() << "\n";
    } else {
      std::cout << j.dump() << "\n";
    }
  };
  try {
    std::ifstream in(argv[1]);
    if (!in) throw ts::ConfigError(std::string("cannot open ") + argv[1]);
    emit(run(json::parse(in)));
  } catch (const ts::ValidationError& e) {
    emit(json{{"error", "ValidationError"}, {"what", e.what()}});
    return 3;
  } catch (const ts::ConfigError& e) {
    emit(json{{"error", "ConfigError"}, {"what", e.what()}});
    return 3;
  } catch (const ts::Error& e) {
    emit(json{{"error", "Error"}, {"what", e.what()}});
    return 3;
  } catch (const std::exception& e) {
    emit(json{{"error", "std::exception"}, {"what", e.what()}});
    return 3;
  }
  return 0;
}
