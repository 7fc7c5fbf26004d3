// ts_plan_import — load_device_plan() from a plan document + assignment CSV
// (the reference's on-disk formats, json_io.hpp) and dump the device remap
// inputs it derives: OUT/{table.u32, row.u64, placement.u8} in canonical
// order plus OUT/summary.json (cuts, topology, hash seed).  Host only.
//
// Usage: ts_plan_import PLAN.json ASSIGNMENT.csv OUT_DIR
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <string>

#include "tiershard/device.hpp"
#include "tiershard/error.hpp"

namespace ts = tiershard;

template <typename T>
static void dump(const std::filesystem::path& p, const std::vector<T>& v) {
  std::ofstream f(p, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s PLAN.json ASSIGNMENT.csv OUT_DIR\n", argv[0]);
    return 2;
  }
  const std::filesystem::path dir = argv[3];
  std::filesystem::create_directories(dir);
  try {
    const ts::DevicePlan p = ts::load_device_plan(argv[1], argv[2]);
    dump(dir / "table.u32", p.table_ids);
    dump(dir / "row.u64", p.row_ids);
    dump(dir / "placement.u8", p.placement);
    std::ofstream(dir / "summary.json")
        << "{\"rows\": " << p.table_ids.size() << ", \"dp_cut\": " << p.plan.dp_cut
        << ", \"flex_cut\": " << p.plan.flex_cut << ", \"num_nodes\": " << p.topology.num_nodes
        << ", \"gpus_per_node\": " << p.topology.gpus_per_node << ", \"embedding_dim\": "
        << p.cost_model.embedding_dim << ", \"hash_seed\": " << p.hash_seed << ", \"goal\": \""
        << p.plan.goal << "\"}\n";
  } catch (const ts::ValidationError& e) {
    std::ofstream(dir / "error.txt") << "ValidationError: " << e.what() << "\n";
    return 3;
  } catch (const ts::ConfigError& e) {
    std::ofstream(dir / "error.txt") << "ConfigError: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::ofstream(dir / "error.txt") << "std::exception: " << e.what() << "\n";
    return 3;
  }
  return 0;
}
