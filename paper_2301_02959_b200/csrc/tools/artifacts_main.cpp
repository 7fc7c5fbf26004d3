// artifacts — manifest in, plan / CSV / simulation artefacts out.
//
// One client source compiled twice: against libtiershard_b200 (bin/ts_artifacts)
// and, by oracle/Makefile, against the unmodified reference library
// (oracle/_ref/ref_artifacts).  It uses only the public tiershard API
// (manifest.hpp, planner.hpp, simulator.hpp, json_io.hpp), so building it
// unchanged against both IS the source-compatibility check, and
// tests/test_io_parity.py diffs the two output directories byte for byte.
//
// Usage: artifacts MANIFEST.json OUT_DIR [THREADS]
// Writes OUT_DIR/{plan.json, plan_reloaded.json, frontier.csv, coverage.csv,
// coverage.txt, assignment.csv, sim.csv, sim_report.json, discrepancies.json};
// on a tiershard error writes OUT_DIR/error.txt ("<Kind>: <what>") and exits 3.
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "tiershard/error.hpp"
#include "tiershard/json_io.hpp"
#include "tiershard/manifest.hpp"
#include "tiershard/planner.hpp"
#include "tiershard/simulator.hpp"
#include "tiershard/version.hpp"

namespace ts = tiershard;
namespace fs = std::filesystem;

namespace {

void write_text(const fs::path& path, const std::string& text) {
  std::ofstream out(path);
  out << text;
}

ts::ShardingPlan plan_for_goal(const ts::Manifest& m, const ts::RowDistribution& d,
                               const ts::Topology& topo) {
  const std::string& goal = m.plan_goal;
  if (goal == "2tier" || goal == "frontier") return ts::plan_2tier(d, m.cost_model, topo);
  if (goal == "3tier") return ts::plan_3tier(d, m.cost_model, topo);
  if (goal.rfind("budget:", 0) == 0) {
    return ts::plan_for_budget(d, m.cost_model, topo, std::stod(goal.substr(7)), m.budget_allow_flex);
  }
  throw ts::ConfigError("artifacts: unknown plan goal '" + goal + "'");
}

void run(const fs::path& manifest_path, const fs::path& dir, unsigned threads) {
  const ts::Manifest m = ts::load_manifest(manifest_path);
  const ts::Topology topo = ts::manifest_topology(m);
  const ts::CostModelConfig& cfg = m.cost_model;
  auto dist = std::make_shared<ts::RowDistribution>(ts::build_merged_distribution(m));
  const ts::RowDistribution& d = *dist;

  ts::PlanDocument doc;
  doc.tool_version = std::string(ts::kVersion);
  doc.topology = topo;
  doc.cost_model = cfg;
  for (const ts::TableSpec& spec : m.tables) {
    const ts::RowDistribution t = ts::build_table(m, spec);
    doc.tables.push_back({spec.table_id, spec.rows, t.num_samples(), t.expected_length()});
  }
  doc.capacity = d.capacity();
  doc.total_expected_length = d.expected_length();
  doc.seed = m.seed;
  doc.hash_seed = m.hash_seed;

  const ts::Frontier fr = ts::build_frontier(d, cfg, topo, ts::Strategy::kDataParallel);
  const ts::FrontierLandmarks lm = ts::find_points(fr, d, cfg, topo);
  doc.landmarks = lm;
  doc.landmark_points = {fr.point(lm.a), fr.point(lm.b), fr.point(lm.c), fr.point(lm.d)};
  ts::write_frontier_csv(fr, d, lm, dir / "frontier.csv");

  doc.plan = plan_for_goal(m, d, topo);
  ts::save_plan_document(doc, d, dir / "plan.json");
  ts::PlanDocument back = ts::load_plan_document(dir / "plan.json");
  back.landmarks = doc.landmarks;
  back.landmark_points = doc.landmark_points;
  ts::save_plan_document(back, d, dir / "plan_reloaded.json");

  const ts::CoverageReport cov = ts::coverage_report(doc.plan, d);
  ts::write_coverage_csv(cov, dir / "coverage.csv");
  write_text(dir / "coverage.txt", ts::format_coverage_table(cov));
  ts::write_assignment_csv(doc.plan, d, dir / "assignment.csv");

  if (m.sim_iterations == 0) return;
  const ts::Workload wl = ts::sample_workload(dist, cfg, topo, m.seed, m.sim_iterations);
  const ts::SimReport rep = ts::simulate(doc.plan, wl, cfg, topo, m.hash_seed, threads);
  ts::ShardingPlan rw;
  rw.total_rows = d.rows().size();
  rw.goal = "rw";
  rw.predicted = ts::predict_cost(d, 0, 0, cfg, topo);
  const ts::SimReport base = ts::simulate(rw, wl, cfg, topo, m.hash_seed, threads);
  ts::write_sim_csv(rep, dir / "sim.csv");
  write_text(dir / "sim_report.json",
             ts::sim_report_json(base, rep, ts::compare_to_baseline(base, rep)).dump(2) + "\n");
  write_text(dir / "discrepancies.json",
             ts::to_json(ts::compare(doc.plan.predicted, rep, 0.02)).dump(2) + "\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s MANIFEST.json OUT_DIR [THREADS]\n", argv[0]);
    return 2;
  }
  const fs::path dir = argv[2];
  fs::create_directories(dir);
  const unsigned threads = argc > 3 ? static_cast<unsigned>(std::atoi(argv[3])) : 1u;
  const auto fail = [&](const char* kind, const std::exception& e) {
    write_text(dir / "error.txt", std::string(kind) + ": " + e.what() + "\n");
    return 3;
  };
  try {
    run(argv[1], dir, threads);
  } catch (const ts::ValidationError& e) {
    return fail("ValidationError", e);
  } catch (const ts::ConfigError& e) {
    return fail("ConfigError", e);
  } catch (const ts::Error& e) {
    return fail("Error", e);
  } catch (const std::exception& e) {
    return fail("std::exception", e);
  }
  return 0;
}
