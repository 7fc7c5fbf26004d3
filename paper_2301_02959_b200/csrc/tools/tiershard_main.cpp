// tiershard — command-line front end over the tiershard API (SURVEY.md §8(f)
// row 3; the reference declares this tool, proj/tools/CMakeLists.txt:1, but
// ships no source; its contract is SPEC.md's `cli` module).
//
//   tiershard synth       --manifest M [--out DIR]
//       Zipf tables of the manifest -> DIR/table_<id>.csv histograms
//       (write_histogram) plus DIR/manifest_echo.json.
//   tiershard plan        --manifest M [--out DIR]
//       merged distribution -> plan goal -> DIR/plan.json, frontier.csv,
//       coverage.csv, assignment.csv; coverage table on stdout, plan
//       warnings on stderr.
//   tiershard simulate    --manifest M [--plan P] [--out DIR] [--threads N]
//       baseline-RW and plan simulations on identical seeds (the routing
//       loop runs on the GPU) -> DIR/sim_report.json, sim.csv,
//       baseline_sim.csv, discrepancies.json; summary on stdout.
//   tiershard compare     --manifest M [--plan P] [--threads N]
//       predicted vs simulated metrics (compare, 2 % tolerance) on stdout.
//   tiershard breakpoints --manifest M
//       Breakpoints of the manifest's cost model and topology (JSON, stdout).
//   tiershard preview     --manifest M [--plan SWEEP.json]
//       GPU planner preview (device.hpp preview_plans) for the manifest's
//       configuration and every what-if of SWEEP.json (a list of
//       {"cost_model": {...}, "topology": {...}} overrides); JSON on stdout.
//
// DIR defaults to the manifest's output_dir (relative to the manifest).  The
// plan of simulate/compare is P, else DIR/plan.json, else planned in
// memory.  Exit 0 on success, 2 on usage errors, 3 on tiershard errors
// (message on stderr).
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <string>

#include "tiershard/device.hpp"
#include "tiershard/error.hpp"
#include "tiershard/json_io.hpp"
#include "tiershard/manifest.hpp"
#include "tiershard/planner.hpp"
#include "tiershard/simulator.hpp"
#include "tiershard/version.hpp"

namespace ts = tiershard;
namespace fs = std::filesystem;

namespace {

struct Args {
  std::string command;
  fs::path manifest, out, plan;
  unsigned threads = 1;
};

[[noreturn]] void usage(const char* msg) {
  std::fprintf(stderr,
               "tiershard %s: %s\n"
               "usage: tiershard {synth|plan|simulate|compare|breakpoints|preview} --manifest PATH "
               "[--out DIR] [--plan PATH] [--threads N]\n",
               std::string(ts::kVersion).c_str(), msg);
  std::exit(2);
}

Args parse(int argc, char** argv) {
  if (argc < 2) usage("missing command");
  Args a;
  a.command = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    if (i + 1 >= argc) usage(("missing value for " + k).c_str());
    const char* v = argv[++i];
    if (k == "--manifest") a.manifest = v;
    else if (k == "--out") a.out = v;
    else if (k == "--plan") a.plan = v;
    else if (k == "--threads") a.threads = static_cast<unsigned>(std::max(1, std::atoi(v)));
    else usage(("unknown flag " + k).c_str());
  }
  if (a.manifest.empty()) usage("--manifest is required");
  return a;
}

fs::path out_dir(const Args& a, const ts::Manifest& m) {
  fs::path d = a.out.empty() ? m.output_dir : a.out;
  if (a.out.empty() && d.is_relative()) d = m.base_dir / d;
  fs::create_directories(d);
  return d;
}

ts::ShardingPlan make_plan(const ts::Manifest& m, const ts::RowDistribution& d, const ts::Topology& topo) {
  const std::string& goal = m.plan_goal;
  if (goal == "2tier" || goal == "frontier") return ts::plan_2tier(d, m.cost_model, topo);
  if (goal == "3tier") return ts::plan_3tier(d, m.cost_model, topo);
  if (goal.rfind("budget:", 0) == 0) {
    return ts::plan_for_budget(d, m.cost_model, topo, std::stod(goal.substr(7)), m.budget_allow_flex);
  }
  throw ts::ConfigError("manifest: unknown plan goal '" + goal + "' (2tier | 3tier | frontier | budget:<bytes>)");
}

ts::PlanDocument plan_document(const ts::Manifest& m, const ts::RowDistribution& d, const ts::Topology& topo,
                               const ts::ShardingPlan& plan, const ts::Frontier& fr,
                               const ts::FrontierLandmarks& lm) {
  ts::PlanDocument doc;
  doc.tool_version = std::string(ts::kVersion);
  doc.plan = plan;
  doc.topology = topo;
  doc.cost_model = m.cost_model;
  for (const ts::TableSpec& spec : m.tables) {
    const ts::RowDistribution t = ts::build_table(m, spec);
    doc.tables.push_back({spec.table_id, spec.rows, t.num_samples(), t.expected_length()});
  }
  doc.capacity = d.capacity();
  doc.total_expected_length = d.expected_length();
  doc.seed = m.seed;
  doc.hash_seed = m.hash_seed;
  doc.landmarks = lm;
  doc.landmark_points = {fr.point(lm.a), fr.point(lm.b), fr.point(lm.c), fr.point(lm.d)};
  return doc;
}

int cmd_synth(const Args& a) {
  const ts::Manifest m = ts::load_manifest(a.manifest);
  if (m.tables.empty()) throw ts::ConfigError("empty manifest: no tables declared");
  const fs::path dir = out_dir(a, m);
  for (const ts::TableSpec& spec : m.tables) {
    if (!spec.zipf) continue;  // histogram tables are inputs already
    const fs::path p = dir / ("table_" + std::to_string(spec.table_id) + ".csv");
    ts::write_histogram(ts::build_table(m, spec), p);
    std::cout << p.string() << "\n";
  }
  // manifest echo: the same tables as histogram references
  nlohmann::json echo;
  echo["tool_version"] = std::string(ts::kVersion);
  echo["seed"] = m.seed;
  nlohmann::json tables = nlohmann::json::array();
  for (const ts::TableSpec& spec : m.tables) {
    const ts::RowDistribution t = ts::build_table(m, spec);
    tables.push_back({{"table_id", spec.table_id},
                      {"rows", spec.rows},
                      {"histogram", spec.zipf ? "table_" + std::to_string(spec.table_id) + ".csv"
                                              : spec.histogram->string()},
                      {"num_samples", t.num_samples()}});
  }
  echo["tables"] = tables;
  std::ofstream(dir / "manifest_echo.json") << echo.dump(2) << "\n";
  return 0;
}

int cmd_plan(const Args& a) {
  const ts::Manifest m = ts::load_manifest(a.manifest);
  const ts::Topology topo = ts::manifest_topology(m);
  const ts::RowDistribution d = ts::build_merged_distribution(m);
  const fs::path dir = out_dir(a, m);
  const ts::Frontier fr = ts::build_frontier(d, m.cost_model, topo, ts::Strategy::kDataParallel);
  const ts::FrontierLandmarks lm = ts::find_points(fr, d, m.cost_model, topo);
  const ts::ShardingPlan plan = make_plan(m, d, topo);
  for (const std::string& w : plan.warnings) std::cerr << "warning: " << w << "\n";
  ts::save_plan_document(plan_document(m, d, topo, plan, fr, lm), d, dir / "plan.json");
  ts::write_frontier_csv(fr, d, lm, dir / "frontier.csv");
  const ts::CoverageReport cov = ts::coverage_report(plan, d);
  ts::write_coverage_csv(cov, dir / "coverage.csv");
  ts::write_assignment_csv(plan, d, dir / "assignment.csv");
  std::cout << ts::format_coverage_table(cov);
  return 0;
}

// The plan to simulate: --plan, else DIR/plan.json, else planned now.  A
// loaded plan must describe the manifest's tables (ids, E) and rows.
ts::ShardingPlan plan_for_sim(const Args& a, const ts::Manifest& m, const ts::RowDistribution& d,
                              const ts::Topology& topo, const fs::path& dir) {
  fs::path p = a.plan;
  if (p.empty() && fs::exists(dir / "plan.json")) p = dir / "plan.json";
  if (p.empty()) return make_plan(m, d, topo);
  if (!fs::exists(p)) throw ts::ConfigError("plan: cannot open '" + p.string() + "'");
  const ts::PlanDocument doc = ts::load_plan_document(p);
  bool same = doc.tables.size() == m.tables.size();
  for (size_t i = 0; same && i < m.tables.size(); ++i) {
    same = doc.tables[i].table_id == m.tables[i].table_id && doc.tables[i].rows == m.tables[i].rows;
  }
  if (!same || doc.plan.total_rows != d.rows().size()) {
    throw ts::ValidationError("simulate: plan '" + p.string() + "' does not match the manifest's tables");
  }
  return doc.plan;
}

int cmd_simulate(const Args& a, bool compare_only) {
  const ts::Manifest m = ts::load_manifest(a.manifest);
  const ts::Topology topo = ts::manifest_topology(m);
  auto dist = std::make_shared<ts::RowDistribution>(ts::build_merged_distribution(m));
  const fs::path dir = out_dir(a, m);
  const ts::ShardingPlan plan = plan_for_sim(a, m, *dist, topo, dir);
  const ts::Workload wl = ts::sample_workload(dist, m.cost_model, topo, m.seed, m.sim_iterations);
  const ts::SimReport rep = ts::simulate(plan, wl, m.cost_model, topo, m.hash_seed, a.threads);
  const std::vector<ts::MetricDiscrepancy> diffs = ts::compare(plan.predicted, rep, 0.02);
  if (compare_only) {
    std::printf("%-32s %14s %14s %10s\n", "metric", "predicted", "simulated", "rel_err");
    for (const ts::MetricDiscrepancy& x : diffs) {
      std::printf("%-32s %14.6g %14.6g %9.3f%%%s\n", x.metric.c_str(), x.predicted, x.simulated,
                  x.relative_error * 100.0, x.flagged ? "  FLAGGED" : "");
    }
    return 0;
  }
  ts::ShardingPlan rw;
  rw.total_rows = dist->rows().size();
  rw.goal = "rw";
  rw.predicted = ts::predict_cost(*dist, 0, 0, m.cost_model, topo);
  const ts::SimReport base = ts::simulate(rw, wl, m.cost_model, topo, m.hash_seed, a.threads);
  const ts::SimComparison cmp = ts::compare_to_baseline(base, rep);
  std::ofstream(dir / "sim_report.json") << ts::sim_report_json(base, rep, cmp).dump(2) << "\n";
  std::ofstream(dir / "discrepancies.json") << ts::to_json(diffs).dump(2) << "\n";
  ts::write_sim_csv(rep, dir / "sim.csv");
  ts::write_sim_csv(base, dir / "baseline_sim.csv");
  std::printf("global a2a bytes / iteration: baseline %.6g, plan %.6g (reduction %.3f%%)\n",
              cmp.baseline_global_a2a_bytes, cmp.plan_global_a2a_bytes, cmp.global_a2a_reduction * 100.0);
  std::printf("total seconds / iteration:    baseline %.6g, plan %.6g (%.3fx; %.3fx with overlappable "
              "collectives hidden)\n",
              cmp.baseline_total_seconds, cmp.plan_total_seconds, cmp.latency_improvement,
              cmp.latency_improvement_critical);
  return 0;
}

// GPU planner preview over a what-if sweep: --plan names a JSON list of
// {"cost_model": {...}, "topology": {...}} overrides of the manifest's
// (either key optional); the manifest's own configuration comes first.
int cmd_preview(const Args& a) {
  const ts::Manifest m = ts::load_manifest(a.manifest);
  const ts::Topology topo = ts::manifest_topology(m);
  const ts::RowDistribution d = ts::build_merged_distribution(m);
  std::vector<ts::WhatIf> wi{{m.cost_model, topo}};
  if (!a.plan.empty()) {
    std::ifstream in(a.plan);
    if (!in) throw ts::ConfigError("preview: cannot open '" + a.plan.string() + "'");
    nlohmann::json sweep;
    try {
      sweep = nlohmann::json::parse(in);
    } catch (const nlohmann::json::parse_error& e) {
      throw ts::ConfigError(std::string("preview: invalid JSON: ") + e.what());
    }
    for (const nlohmann::json& o : sweep) {
      ts::WhatIf w{m.cost_model, topo};
      if (o.contains("cost_model")) {
        const nlohmann::json& c = o["cost_model"];
        if (c.contains("local_batch")) w.cost_model.local_batch = c["local_batch"].get<uint32_t>();
        if (c.contains("embedding_dim")) w.cost_model.embedding_dim = c["embedding_dim"].get<uint32_t>();
        if (c.contains("scalar_bytes")) w.cost_model.scalar_bytes = c["scalar_bytes"].get<uint32_t>();
        if (c.contains("dp_replication_multiplier")) {
          w.cost_model.dp_replication_multiplier = c["dp_replication_multiplier"].get<double>();
        }
      }
      if (o.contains("topology")) {
        const nlohmann::json& t = o["topology"];
        w.topology.num_nodes = t.value("num_nodes", w.topology.num_nodes);
        w.topology.gpus_per_node = t.value("gpus_per_node", w.topology.gpus_per_node);
        if (t.contains("a2a_global_gibs")) w.topology.a2a_global = t["a2a_global_gibs"].get<double>() * ts::kGiB;
        if (t.contains("a2a_intra_gibs")) w.topology.a2a_intra = t["a2a_intra_gibs"].get<double>() * ts::kGiB;
        if (t.contains("ar_global_gibs")) w.topology.ar_global = t["ar_global_gibs"].get<double>() * ts::kGiB;
        if (t.contains("ar_cross_gibs")) w.topology.ar_cross = t["ar_cross_gibs"].get<double>() * ts::kGiB;
      }
      wi.push_back(w);
    }
  }
  const std::vector<ts::PlanPreview> pv = ts::preview_plans(d, wi);
  nlohmann::json out = nlohmann::json::array();
  for (size_t i = 0; i < pv.size(); ++i) {
    out.push_back({{"cost_model", ts::to_json(wi[i].cost_model)},
                   {"topology", ts::to_json(wi[i].topology)},
                   {"landmarks", {{"a", pv[i].landmarks.a}, {"b", pv[i].landmarks.b}, {"c", pv[i].landmarks.c},
                                  {"d", pv[i].landmarks.d}}},
                   {"plan_2tier", {{"dp_cut", pv[i].dp_cut_2tier},
                                   {"global_a2a_reduction", pv[i].reduction_2tier}}},
                   {"plan_3tier", {{"dp_cut", pv[i].dp_cut_3tier}, {"flex_cut", pv[i].flex_cut_3tier},
                                   {"global_a2a_reduction", pv[i].reduction_3tier}}}});
  }
  std::cout << out.dump(2) << "\n";
  return 0;
}

int cmd_breakpoints(const Args& a) {
  const ts::Manifest m = ts::load_manifest(a.manifest);
  const ts::Topology topo = ts::manifest_topology(m);
  std::cout << ts::to_json(ts::find_breakpoints(m.cost_model, topo)).dump(2) << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const Args a = parse(argc, argv);
  try {
    if (a.command == "synth") return cmd_synth(a);
    if (a.command == "plan") return cmd_plan(a);
    if (a.command == "simulate") return cmd_simulate(a, false);
    if (a.command == "compare") return cmd_simulate(a, true);
    if (a.command == "breakpoints") return cmd_breakpoints(a);
    if (a.command == "preview") return cmd_preview(a);
    usage(("unknown command " + a.command).c_str());
  } catch (const ts::ValidationError& e) {
    std::fprintf(stderr, "tiershard: ValidationError: %s\n", e.what());
  } catch (const ts::ConfigError& e) {
    std::fprintf(stderr, "tiershard: ConfigError: %s\n", e.what());
  } catch (const ts::Error& e) {
    std::fprintf(stderr, "tiershard: Error: %s\n", e.what());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "tiershard: %s\n", e.what());
  }
  return 3;
}
