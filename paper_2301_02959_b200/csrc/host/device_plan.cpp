// Plan import from on-disk artefacts: the plan
// document written by save_plan_document (/root/reference/proj/src/
// json_io.cpp:210-274) and the assignment CSV of write_assignment_csv
// (:380-394) are enough to rebuild every device remap table.  The placement
// byte follows assign_rows (simulator.cpp:82-108): RW owner =
// row_key_hash(table, row, hash_seed) % U, Flex slot = % W.
#include <charconv>
#include <cstring>
#include <fstream>
#include <string>

#include "json.hpp"
#include "parallel.hpp"
#include "tiershard/device.hpp"
#include "tiershard/error.hpp"
#include "tiershard/hashing.hpp"
#include "tiershard/json_io.hpp"

namespace tiershard {
namespace {

std::string read_file(const std::filesystem::path& path, const char* what) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ConfigError(std::string(what) + ": cannot open '" + path.string() + "'");
  in.seekg(0, std::ios::end);
  std::string text(static_cast<size_t>(in.tellg()), '\0');
  in.seekg(0);
  in.read(text.data(), static_cast<std::streamsize>(text.size()));
  return text;
}

// table_id,row_id,tier lines after the header; tiers as tier_name().
void parse_assignment(const std::string& text, DevicePlan& out, std::vector<uint8_t>& tiers) {
  static constexpr char kHeader[] = "table_id,row_id,tier\n";
  if (text.compare(0, sizeof(kHeader) - 1, kHeader) != 0) {
    throw ConfigError("assignment: expected header 'table_id,row_id,tier'");
  }
  const char* p = text.data() + sizeof(kHeader) - 1;
  const char* end = text.data() + text.size();
  uint64_t line = 1;
  while (p < end) {
    ++line;
    const auto bad = [&] { return ConfigError("assignment: malformed line " + std::to_string(line)); };
    uint32_t t = 0;
    uint64_t r = 0;
    auto res = std::from_chars(p, end, t);
    if (res.ec != std::errc() || res.ptr >= end || *res.ptr != ',') throw bad();
    res = std::from_chars(res.ptr + 1, end, r);
    if (res.ec != std::errc() || res.ptr >= end || *res.ptr != ',') throw bad();
    const char* q = res.ptr + 1;
    const char* nl = static_cast<const char*>(std::memchr(q, '\n', static_cast<size_t>(end - q)));
    if (!nl) nl = end;
    const std::string_view tier(q, static_cast<size_t>(nl - q));
    uint8_t code;
    if (tier == "dp") code = static_cast<uint8_t>(Tier::kDataParallel);
    else if (tier == "flex") code = static_cast<uint8_t>(Tier::kFlex);
    else if (tier == "rw") code = static_cast<uint8_t>(Tier::kRowWise);
    else throw bad();
    out.table_ids.push_back(t);
    out.row_ids.push_back(r);
    tiers.push_back(code);
    p = nl + (nl < end ? 1 : 0);
  }
}

}  // namespace

DevicePlan load_device_plan(const std::filesystem::path& plan_json,
                            const std::filesystem::path& assignment_csv) {
  const PlanDocument doc = load_plan_document(plan_json);
  DevicePlan out;
  out.plan = doc.plan;
  out.topology = doc.topology;
  out.cost_model = doc.cost_model;
  out.hash_seed = doc.hash_seed;

  std::vector<uint8_t> tiers;
  parse_assignment(read_file(assignment_csv, "assignment"), out, tiers);
  const uint64_t n = out.table_ids.size();
  if (n != out.plan.total_rows) {
    throw ValidationError("device plan: the assignment has " + std::to_string(n) +
                          " rows, the plan document total_rows " + std::to_string(out.plan.total_rows));
  }
  if (out.plan.dp_cut > out.plan.flex_cut || out.plan.flex_cut > n) {
    throw ValidationError("assign_rows: plan does not cover the distribution");
  }
  for (uint64_t i = 0; i < n; ++i) {
    const Tier want = i < out.plan.dp_cut ? Tier::kDataParallel
                                          : (i < out.plan.flex_cut ? Tier::kFlex : Tier::kRowWise);
    if (tiers[i] != static_cast<uint8_t>(want)) {
      throw ValidationError("device plan: assignment row " + std::to_string(i) + " is '" +
                            tier_name(static_cast<Tier>(tiers[i])) + "', the cuts say '" +
                            tier_name(want) + "'");
    }
  }
  // the document's explicit DP / Flex membership must list the same rows
  {
    const nlohmann::json j = nlohmann::json::parse(read_file(plan_json, "plan"));
    const auto check = [&](const char* key, uint64_t lo, uint64_t hi) {
      const nlohmann::json& list = j.at(key);
      if (list.size() != hi - lo) {
        throw ValidationError(std::string("device plan: ") + key + " lists " + std::to_string(list.size()) +
                              " rows, the cuts " + std::to_string(hi - lo));
      }
      for (uint64_t i = lo; i < hi; ++i) {
        const nlohmann::json& e = list[i - lo];
        if (e.at(0).get<uint32_t>() != out.table_ids[i] || e.at(1).get<uint64_t>() != out.row_ids[i]) {
          throw ValidationError(std::string("device plan: ") + key + " differs from the assignment at row " +
                                std::to_string(i));
        }
      }
    };
    check("dp_rows", 0, out.plan.dp_cut);
    check("flex_rows", out.plan.dp_cut, out.plan.flex_cut);
  }
  if (out.topology.total_gpus() > 256) throw ConfigError("device path: at most 256 GPUs");
  out.placement.assign(n, 0);
  const uint64_t u = out.topology.total_gpus(), w = out.topology.gpus_per_node;
  detail::parallel_for(n, [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      if (i < out.plan.dp_cut) continue;
      const uint64_t h = row_key_hash(out.table_ids[i], out.row_ids[i], out.hash_seed);
      out.placement[i] = static_cast<uint8_t>(i < out.plan.flex_cut ? h % w : h % u);
    }
  });
  return out;
}

}  // namespace tiershard
