// ts_driver — JSON front-end over THIS library's public C++ API
// (include/tiershard/*.hpp), accepting the same spec as oracle/ref_driver and
// emitting the same keys, so tests can diff the product against the compiled
// reference document-for-document.  simulate() here routes every iteration
// on the GPU (csrc/device/router.cu); the planner and workload sampling run
// on the host.
//
// Usage: ts_driver SPEC.json [OUT.json]
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <string>
#include <algorithm>
#include <thread>
#include <vector>

#include "json.hpp"
#include "tiershard/cost_model.hpp"
#include "tiershard/device.hpp"
#include "tiershard/distribution.hpp"
#include "tiershard/error.hpp"
#include "tiershard/hashing.hpp"
#include "tiershard/planner.hpp"
#include "tiershard/rng.hpp"
#include "tiershard/simulator.hpp"
#include "tiershard/topology.hpp"
#include "tiershard/version.hpp"

using Json = nlohmann::json;
namespace ts = tiershard;

namespace {

double seconds_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

Json tier_json(const ts::TierSummary& t) {
  return Json{{"rows", t.row_count}, {"expected_length", t.expected_length}, {"coverage", t.coverage}};
}

Json report_json(const ts::CostReport& r) {
  Json j;
  j["tiers"] = {{"dp", tier_json(r.dp)}, {"flex", tier_json(r.flex)}, {"rw", tier_json(r.rw)}};
#define F(x) j[#x] = r.x
  F(static_memory_bytes); F(baseline_static_memory_bytes); F(peak_dynamic_memory_bytes);
  F(baseline_peak_dynamic_memory_bytes); F(rows_accessed_scalars); F(input_id_count);
  F(baseline_input_id_count); F(global_a2a_bytes); F(intra_a2a_bytes); F(ar_global_bytes);
  F(ar_cross_bytes); F(global_a2a_seconds); F(intra_a2a_seconds); F(ar_global_seconds);
  F(ar_cross_seconds); F(baseline_global_a2a_bytes); F(baseline_global_a2a_seconds);
  F(global_a2a_reduction); F(total_seconds); F(total_seconds_critical); F(baseline_total_seconds);
  F(latency_improvement); F(latency_improvement_critical);
#undef F
  return j;
}

Json metrics_json(const ts::IterationMetrics& m) {
  Json j;
#define F(x) j[#x] = m.x
  F(global_a2a_send_max); F(global_a2a_recv_max); F(global_a2a_bytes_mean); F(global_a2a_total);
  F(intra_a2a_send_max); F(intra_a2a_recv_max); F(intra_a2a_bytes_mean); F(intra_a2a_total);
  F(ar_global_bytes); F(ar_cross_bytes_max); F(ar_cross_bytes_mean); F(global_a2a_seconds);
  F(intra_a2a_seconds); F(ar_global_seconds); F(ar_cross_seconds); F(total_seconds);
  F(total_seconds_critical); F(peak_dynamic_memory_bytes); F(rows_accessed_scalars_min);
  F(rows_accessed_scalars_max); F(rows_accessed_scalars_mean); F(load_imbalance);
  F(distinct_rows_min); F(distinct_rows_max); F(distinct_rows_mean); F(distinct_row_imbalance);
#undef F
  return j;
}

Json comparison_json(const ts::SimComparison& c) {
  Json j;
#define F(x) j[#x] = c.x
  F(baseline_global_a2a_bytes); F(plan_global_a2a_bytes); F(global_a2a_reduction);
  F(baseline_total_seconds); F(plan_total_seconds); F(plan_total_seconds_critical);
  F(latency_improvement); F(latency_improvement_critical); F(baseline_peak_dynamic_memory_bytes);
  F(plan_peak_dynamic_memory_bytes);
#undef F
  return j;
}

Json sim_json(const ts::SimReport& r) {
  Json its = Json::array();
  for (const auto& m : r.iterations) its.push_back(metrics_json(m));
  return Json{{"seed", r.seed}, {"hash_seed", r.hash_seed}, {"num_iterations", r.num_iterations},
              {"iterations", its}, {"mean", metrics_json(r.mean)}};
}

ts::Topology parse_topology(const Json& j) {
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

ts::CostModelConfig parse_cfg(const Json& j) {
  ts::CostModelConfig c;
  c.local_batch = j.value("local_batch", c.local_batch);
  c.embedding_dim = j.value("embedding_dim", c.embedding_dim);
  c.scalar_bytes = j.value("scalar_bytes", c.scalar_bytes);
  c.dp_replication_multiplier = j.value("dp_replication_multiplier", c.dp_replication_multiplier);
  c.dynamic_pass_count = j.value("dynamic_pass_count", c.dynamic_pass_count);
  c.static_pass_count = j.value("static_pass_count", c.static_pass_count);
  c.include_id_bytes = j.value("include_id_bytes", c.include_id_bytes);
  c.bytes_per_id = j.value("bytes_per_id", c.bytes_per_id);
  c.count_dynamic_memory = j.value("count_dynamic_memory", c.count_dynamic_memory);
  c.validate();
  return c;
}

uint64_t digest_rows(const ts::RowDistribution& d) {
  uint64_t h = 0x243F6A8885A308D3ull;
  for (const auto& r : d.rows()) {
    uint64_t pb;
    std::memcpy(&pb, &r.probability, 8);
    h = ts::mix64(ts::mix64(ts::mix64(h ^ r.table_id) ^ r.row_id) ^ pb);
  }
  return h;
}

uint64_t digest_placements(const std::vector<ts::RowPlacement>& p) {
  uint64_t h = 0x13198A2E03707344ull;
  for (const auto& x : p) {
    h = ts::mix64(ts::mix64(ts::mix64(h ^ static_cast<uint64_t>(x.tier)) ^ x.owner_gpu) ^ x.flex_slot);
  }
  return h;
}

template <typename T>
void write_binary(const std::string& path, const std::vector<T>& v) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw ts::ConfigError("ts_driver: cannot write " + path);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

// All-to-all bytes of one iteration under three shardings of the same rows:
// the plan, pure row-wise (owner = h % U) and table-wise (owner = table % U,
// builder-defined: the reference has no TW strategy).
// "reference convention" counts every non-replicated occurrence (self sends
// included, simulator.cpp:234-243); "off_device" counts only occurrences whose
// server is another GPU — the bytes that actually cross NVLink.  One
// direction, one pass, embedding payload only.
Json traffic_json(const ts::IterationBatch& b, const ts::RowDistribution& d,
                  const std::vector<ts::RowPlacement>& pl, uint32_t u, uint32_t w,
                  const ts::CostModelConfig& cfg, uint64_t hash_seed) {
  const double row_bytes = static_cast<double>(cfg.embedding_dim) * cfg.scalar_bytes;
  uint64_t plan_global = 0, plan_intra = 0, plan_global_off = 0, plan_intra_off = 0;
  uint64_t rw_off = 0, tw_off = 0, total = 0;
  // per-server sends, self-inclusive (the reference's convention) and
  // off-device only: the most loaded server is the all-to-all's critical path
  std::vector<uint64_t> rw_send(u, 0), tw_send(u, 0), plan_send(u, 0);
  std::vector<uint64_t> rw_send_off(u, 0), tw_send_off(u, 0), plan_send_off(u, 0);
  for (uint32_t g = 0; g < u; ++g) {
    const uint64_t lo = b.sample_offsets[uint64_t{g} * b.local_batch];
    const uint64_t hi = b.sample_offsets[uint64_t{g + 1} * b.local_batch];
    const uint32_t node_base = (g / w) * w;
    for (uint64_t k = lo; k < hi; ++k) {
      const uint32_t r = b.rows[k];
      const ts::RowRecord& rec = d.rows()[r];
      ++total;
      const uint32_t rw_owner = static_cast<uint32_t>(ts::row_key_hash(rec.table_id, rec.row_id, hash_seed) % u);
      const uint32_t tw_owner = rec.table_id % u;
      rw_off += rw_owner != g;
      tw_off += tw_owner != g;
      ++rw_send[rw_owner];
      ++tw_send[tw_owner];
      rw_send_off[rw_owner] += rw_owner != g;
      tw_send_off[tw_owner] += tw_owner != g;
      const ts::RowPlacement& p = pl[r];
      if (p.tier == ts::Tier::kRowWise) {
        ++plan_global;
        plan_global_off += p.owner_gpu != g;
        ++plan_send[p.owner_gpu];
        plan_send_off[p.owner_gpu] += p.owner_gpu != g;
      } else if (p.tier == ts::Tier::kFlex) {
        const uint32_t server = node_base + p.flex_slot;
        ++plan_intra;
        plan_intra_off += server != g;
        ++plan_send[server];
        plan_send_off[server] += server != g;
      }
    }
  }
  auto maxv = [](const std::vector<uint64_t>& v) { return *std::max_element(v.begin(), v.end()); };
  return Json{{"occurrences", total},
              {"row_bytes", row_bytes},
              {"reference_convention",
               {{"plan_global_bytes", plan_global * row_bytes},
                {"plan_intra_bytes", plan_intra * row_bytes},
                {"rw_global_bytes", total * row_bytes}}},
              {"off_device",
               {{"plan_global_bytes", plan_global_off * row_bytes},
                {"plan_intra_bytes", plan_intra_off * row_bytes},
                {"rw_bytes", rw_off * row_bytes},
                {"tw_bytes", tw_off * row_bytes}}},
              {"max_send_bytes",
               {{"plan", maxv(plan_send) * row_bytes},
                {"rw", maxv(rw_send) * row_bytes},
                {"tw", maxv(tw_send) * row_bytes}}},
              {"max_send_off_device_bytes",
               {{"plan", maxv(plan_send_off) * row_bytes},
                {"rw", maxv(rw_send_off) * row_bytes},
                {"tw", maxv(tw_send_off) * row_bytes}}}};
}

Json run(const Json& spec) {
  Json out;
  Json timing;
  out["tool"] = "tiershard-b200";
  out["version"] = std::string(ts::kVersion);
  if (spec.value("hash_vectors", false)) {
    ts::SplitMix64 rng(7);
    const uint64_t r0 = rng.next_u64();
    const uint64_t r1 = rng.next_u64();
    Json pois = Json::array();
    ts::SplitMix64 prng(11);
    for (double mean : {0.5, 3.0, 9.99, 10.0, 32.0, 1024.0}) {
      Json draws = Json::array();
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

  double t0 = seconds_now();
  std::vector<ts::RowDistribution> parts;
  for (const Json& t : spec.at("tables")) {
    parts.push_back(ts::synthesize_zipf(t.at("rows").get<uint64_t>(), t.at("exponent").get<double>(),
                                        t.at("target_length").get<double>(),
                                        t.at("seed").get<uint64_t>(), t.value("table_id", 0u)));
  }
  auto dist = std::make_shared<ts::RowDistribution>(parts.size() == 1 ? std::move(parts[0])
                                                                      : ts::merge(parts));
  parts.clear();
  timing["synth_merge_s"] = seconds_now() - t0;
  const ts::RowDistribution& d = *dist;
  Json head = Json::array();
  const size_t nh = std::min<size_t>(d.rows().size(), spec.value("head_rows", 16));
  for (size_t i = 0; i < nh; ++i) head.push_back({d.rows()[i].table_id, d.rows()[i].row_id, d.rows()[i].probability});
  out["distribution"] = {{"rows", d.rows().size()}, {"capacity", d.capacity()},
                         {"num_samples", d.num_samples()}, {"expected_length", d.expected_length()},
                         {"digest", digest_rows(d)}, {"head", head}};

  const ts::Topology topo = parse_topology(spec.at("topology"));
  const ts::CostModelConfig cfg = parse_cfg(spec.value("cost_model", Json::object()));
  const ts::Breakpoints bp = ts::find_breakpoints(cfg, topo);
  out["breakpoints"] = {{"p_mem_dp", bp.p_mem_dp ? Json(*bp.p_mem_dp) : Json()},
                        {"p_comm_dp", bp.p_comm_dp},
                        {"flex_mem_price_bytes", bp.flex_mem_price_bytes},
                        {"p_comm_flex", bp.p_comm_flex ? Json(*bp.p_comm_flex) : Json()}};

  t0 = seconds_now();
  if (spec.value("frontier", true)) {
    const ts::Frontier fr = ts::build_frontier(d, cfg, topo, ts::Strategy::kDataParallel);
    const ts::FrontierLandmarks lm = ts::find_points(fr, d, cfg, topo);
    out["landmarks"] = {{"a", lm.a}, {"b", lm.b}, {"c", lm.c}, {"d", lm.d}};
    std::vector<size_t> ks = {0, lm.a, lm.b, lm.c, lm.d};
    for (const Json& k : spec.value("frontier_points", Json::array())) ks.push_back(k);
    Json s = Json::array();
    for (size_t k : ks) if (k < fr.size()) s.push_back({k, fr.memory_at(k), fr.comm_at(k)});
    out["frontier_dp"] = s;
    if (topo.has_fast_intra_tier()) {
      const ts::Frontier ff = ts::build_frontier(d, cfg, topo, ts::Strategy::kFlex);
      Json f = Json::array();
      for (size_t k : ks) if (k < ff.size()) f.push_back({k, ff.memory_at(k), ff.comm_at(k)});
      out["frontier_flex"] = f;
    }
  }
  timing["frontier_s"] = seconds_now() - t0;

  t0 = seconds_now();
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
    throw ts::ConfigError("ts_driver: unknown goal " + goal);
  }
  timing["plan_s"] = seconds_now() - t0;
  out["plan"] = {{"dp_cut", plan.dp_cut}, {"flex_cut", plan.flex_cut}, {"total_rows", plan.total_rows},
                 {"goal", plan.goal}, {"warnings", plan.warnings},
                 {"achieved_memory_bytes", plan.achieved_memory_bytes ? Json(*plan.achieved_memory_bytes) : Json()},
                 {"achieved_comm_seconds", plan.achieved_comm_seconds ? Json(*plan.achieved_comm_seconds) : Json()},
                 {"predicted", report_json(plan.predicted)}};
  const ts::CoverageReport cov = ts::coverage_report(plan, d);
  out["coverage"] = {{"dp", tier_json(cov.dp)}, {"flex", tier_json(cov.flex)}, {"rw", tier_json(cov.rw)}};
  const uint64_t hash_seed = spec.value("hash_seed", ts::kDefaultPlacementSeed);
  const auto placements = ts::assign_rows(plan, d, topo, hash_seed);
  out["placements_digest"] = digest_placements(placements);

  if (spec.contains("preview")) {
    // GPU planner preview of this spec's (cost model, topology) plus any
    // what-if overrides, beside the authoritative host plans of each
    std::vector<ts::WhatIf> wi{{cfg, topo}};
    for (const Json& o : spec["preview"].value("what_if", Json::array())) {
      wi.push_back({o.contains("cost_model") ? parse_cfg(o["cost_model"]) : cfg,
                    o.contains("topology") ? parse_topology(o["topology"]) : topo});
    }
    t0 = seconds_now();
    const std::vector<ts::PlanPreview> pv = ts::preview_plans(d, wi);
    timing["preview_s"] = seconds_now() - t0;
    Json arr = Json::array();
    for (size_t i = 0; i < pv.size(); ++i) {
      const ts::ShardingPlan p2 = ts::plan_2tier(d, wi[i].cost_model, wi[i].topology);
      const ts::ShardingPlan p3 = ts::plan_3tier(d, wi[i].cost_model, wi[i].topology);
      const ts::Frontier fr = ts::build_frontier(d, wi[i].cost_model, wi[i].topology, ts::Strategy::kDataParallel);
      const ts::FrontierLandmarks lm = ts::find_points(fr, d, wi[i].cost_model, wi[i].topology);
      arr.push_back({{"gpu", {{"a", pv[i].landmarks.a}, {"b", pv[i].landmarks.b}, {"c", pv[i].landmarks.c},
                              {"dp_cut_2tier", pv[i].dp_cut_2tier}, {"dp_cut_3tier", pv[i].dp_cut_3tier},
                              {"flex_cut_3tier", pv[i].flex_cut_3tier},
                              {"reduction_2tier", pv[i].reduction_2tier},
                              {"reduction_3tier", pv[i].reduction_3tier}}},
                     {"host", {{"a", lm.a}, {"b", lm.b}, {"c", lm.c}, {"dp_cut_2tier", p2.dp_cut},
                               {"dp_cut_3tier", p3.dp_cut}, {"flex_cut_3tier", p3.flex_cut},
                               {"reduction_2tier", p2.predicted.global_a2a_reduction},
                               {"reduction_3tier", p3.predicted.global_a2a_reduction}}}});
    }
    out["preview"] = arr;
  }

  if (spec.contains("export_dir")) {
    // Bench/test preparation: the device remap bytes the planner emits, the
    // cuts, and materialized batches — everything bench.py needs to drive
    // the C-ABI without re-implementing the host API in Python.
    t0 = seconds_now();
    const std::string dir = spec["export_dir"].get<std::string>();
    std::vector<uint8_t> dest(placements.size());
    for (size_t i = 0; i < placements.size(); ++i) {
      dest[i] = static_cast<uint8_t>(placements[i].tier == ts::Tier::kFlex ? placements[i].flex_slot
                                                                          : placements[i].owner_gpu);
    }
    write_binary(dir + "/dest.u8", dest);
    if (spec.value("export_alias", false)) {  // the Workload's alias table (GPU sampler input)
      std::vector<double> w(d.rows().size());
      for (size_t i = 0; i < w.size(); ++i) w[i] = d.rows()[i].probability;
      const ts::AliasTable at(w);
      const std::vector<double> prob(at.probabilities().begin(), at.probabilities().end());
      const std::vector<uint32_t> idx(at.aliases().begin(), at.aliases().end());
      write_binary(dir + "/alias.prob.f64", prob);
      write_binary(dir + "/alias.idx.u32", idx);
      out["expected_length"] = d.expected_length();
    }
    const Json& jw = spec.at("workload");
    const uint32_t iters = jw.value("iterations", 1u);
    const ts::Workload wl = ts::sample_workload(dist, cfg, topo, jw.value("seed", uint64_t{7}), iters);
    std::vector<ts::IterationBatch> batches(iters);
    {
      std::vector<std::thread> pool;
      for (uint32_t it = 0; it < iters; ++it) {
        pool.emplace_back([&, it] { wl.materialize_iteration(it, batches[it]); });
      }
      for (auto& th : pool) th.join();
    }
    Json occ = Json::array();
    Json traffic = Json::array();
    const uint32_t u = topo.total_gpus(), w = topo.gpus_per_node;
    for (uint32_t it = 0; it < iters; ++it) {
      const auto& b = batches[it];
      write_binary(dir + "/batch_" + std::to_string(it) + ".rows.u32", b.rows);
      write_binary(dir + "/batch_" + std::to_string(it) + ".offsets.u64", b.sample_offsets);
      occ.push_back(b.occurrences());
      traffic.push_back(traffic_json(b, d, placements, u, w, cfg, hash_seed));
    }
    out["export"] = {{"dir", dir}, {"iterations", iters}, {"occurrences", occ}, {"traffic", traffic},
                     {"n_rows", d.rows().size()}, {"num_gpus", u}, {"gpus_per_node", w},
                     {"local_batch", cfg.local_batch}, {"embedding_dim", cfg.embedding_dim}};
    timing["export_s"] = seconds_now() - t0;
  }

  if (!spec.contains("workload") || spec.contains("export_dir")) {
    out["timing"] = timing;
    return out;
  }
  const Json& jw = spec["workload"];
  const uint32_t iters = jw.value("iterations", 1u);
  unsigned threads = spec.value("threads", 1u);
  if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
  timing["threads"] = threads;
  t0 = seconds_now();
  const ts::Workload wl = ts::sample_workload(dist, cfg, topo, jw.value("seed", uint64_t{7}), iters);
  timing["workload_build_s"] = seconds_now() - t0;
  {
    ts::IterationBatch batch;
    Json occ = Json::array();
    t0 = seconds_now();
    for (uint32_t it = 0; it < iters; ++it) {
      wl.materialize_iteration(it, batch);
      occ.push_back(batch.occurrences());
    }
    timing["materialize_total_s_1thread"] = seconds_now() - t0;
    out["occurrences"] = occ;
  }
  if (spec.value("simulate", true)) {
    t0 = seconds_now();
    const ts::SimReport rep = ts::simulate(plan, wl, cfg, topo, hash_seed, threads);
    timing["simulate_s"] = seconds_now() - t0;
    out["sim"] = sim_json(rep);
    Json disc = Json::array();
    for (const auto& x : ts::compare(plan.predicted, rep, 0.02)) {
      disc.push_back({{"metric", x.metric}, {"predicted", x.predicted}, {"simulated", x.simulated},
                      {"relative_error", x.relative_error}, {"flagged", x.flagged}});
    }
    out["discrepancies"] = disc;
    if (spec.value("baseline", false)) {
      ts::ShardingPlan rw;
      rw.total_rows = d.rows().size();
      rw.goal = "rw";
      rw.predicted = ts::predict_cost(d, 0, 0, cfg, topo);
      const ts::SimReport base = ts::simulate(rw, wl, cfg, topo, hash_seed, threads);
      out["baseline_sim"] = sim_json(base);
      out["comparison"] = comparison_json(ts::compare_to_baseline(base, rep));
    }
  }
  out["timing"] = timing;
  return out;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ts_driver SPEC.json [OUT.json]\n");
    return 2;
  }
  auto emit = [&](const Json& j) {
    if (argc >= 3) {
      std::ofstream(argv[2]) << j.dump() << "\n";
    } else {
      std::cout << j.dump() << "\n";
    }
  };
  try {
    std::ifstream in(argv[1]);
    if (!in) throw ts::ConfigError(std::string("cannot open ") + argv[1]);
    emit(run(Json::parse(in)));
  } catch (const ts::ValidationError& e) {
    emit(Json{{"error", "ValidationError"}, {"what", e.what()}});
    return 3;
  } catch (const ts::ConfigError& e) {
    emit(Json{{"error", "ConfigError"}, {"what", e.what()}});
    return 3;
  } catch (const ts::Error& e) {
    emit(Json{{"error", "Error"}, {"what", e.what()}});
    return 3;
  } catch (const std::exception& e) {
    emit(Json{{"error", "std::exception"}, {"what", e.what()}});
    return 3;
  }
  return 0;
}
