// tiershard-b200 — lookup / update entry points of the tiered sequence
// embedding on B200 (C++ front door over include/tiershard_b200.h).
//
// The reference (tiershard 0.1.0) stops at planning and traffic simulation;
// this header adds what the north star asks for on top of the same API: a
// sharded table laid out by a ShardingPlan, with a forward (unpooled L x D
// gather + id/row exchange) and a backward (gradient dedup, replicated-tier
// reduction, fused row-wise optimizer).  Every entry point runs on the GPU;
// failures surface as tiershard::ConfigError / ValidationError / Error.
#pragma once

#include <array>
#include <cstdint>
#include <filesystem>
#include <vector>

#include "tiershard/cost_model.hpp"
#include "tiershard/distribution.hpp"
#include "tiershard/hashing.hpp"
#include "tiershard/planner.hpp"
#include "tiershard/topology.hpp"

struct ts_table;   // C-ABI handles
struct ts_keymap;
struct ts_sampler;
struct ts_group;

namespace tiershard {

enum class Optimizer { kSgd = 0, kRowwiseAdagrad = 1 };

using NcclUniqueId = std::array<uint8_t, 128>;

// Fresh communicator id: rank 0 calls it and ships it to the other ranks.
NcclUniqueId new_nccl_unique_id();

// In-process rank group: all N*W ranks as host threads of one process (any
// GPUs, several per GPU allowed), instead of one process per GPU over NCCL.
// Each rank's SequenceEmbedding is created, stepped and destroyed by its own
// thread; destroy the group after its tables.  abort() makes every pending
// collective of its tables fail at once (a rank's thread failed).
class DeviceGroup {
 public:
  explicit DeviceGroup(uint32_t ranks);
  ~DeviceGroup();
  DeviceGroup(const DeviceGroup&) = delete;
  DeviceGroup& operator=(const DeviceGroup&) = delete;
  void abort();
  ts_group* handle() const { return group_; }

 private:
  ts_group* group_ = nullptr;
};

struct DeviceOptions {
  int device = 0;
  uint32_t rank = 0;                 // this process's GPU index in [0, N*W)
  uint64_t weight_seed = 1234;       // seeded-hash initial weights
  Optimizer optimizer = Optimizer::kRowwiseAdagrad;
  float learning_rate = 0.01f;
  float epsilon = 1e-8f;
  uint64_t max_occurrences = uint64_t{1} << 22;  // per step, this rank
  const NcclUniqueId* nccl_id = nullptr;         // N*W > 1, one process per GPU
  const DeviceGroup* group = nullptr;            // N*W > 1, all ranks in this process
  // capacity (rows) of the buffer peers push this rank's remote gradients
  // into: e.g. the plan's expected remote occurrences + 25 %; 0 = the worst
  // case, (N*W-1) x max_occurrences.  A step that needs more grows it.
  uint64_t recv_rows_hint = 0;
};

// The per-row placement byte the planner emits for the device: RW owner
// (row_key_hash % U) for RW rows, Flex slot (% W) for Flex rows, 0 for DP.
std::vector<uint8_t> placement_bytes(const ShardingPlan& plan, const RowDistribution& dist,
                                     const Topology& topo,
                                     uint64_t hash_seed = kDefaultPlacementSeed);

// A plan imported from its on-disk artefacts (json_io.hpp): the plan
// document (cuts, topology, cost model, hash seed, DP / Flex membership) and
// the assignment CSV (every materialized row in canonical order with its
// tier).  Together they determine every device remap table without the
// distribution: canonical index = CSV line, tier = CSV column (checked
// against the cuts and the document's dp_rows / flex_rows), placement byte =
// row_key_hash(table, row, hash_seed) % U (RW) or % W (Flex), as assign_rows.
struct DevicePlan {
  ShardingPlan plan;  // dp_cut, flex_cut, total_rows, goal, predicted
  Topology topology;
  CostModelConfig cost_model;
  uint64_t hash_seed = kDefaultPlacementSeed;
  std::vector<uint32_t> table_ids;  // canonical order
  std::vector<uint64_t> row_ids;
  std::vector<uint8_t> placement;   // device placement byte per canonical row
};

// ConfigError on unreadable files; ValidationError when the CSV and the
// document disagree (row count, tiers vs cuts, DP / Flex membership).
DevicePlan load_device_plan(const std::filesystem::path& plan_json,
                            const std::filesystem::path& assignment_csv);

// Raw (table_id, row_id) keys -> canonical row indices on one GPU.
class KeyMap {
 public:
  KeyMap(const std::vector<uint32_t>& table_ids, const std::vector<uint64_t>& row_ids, int device = 0);
  explicit KeyMap(const DevicePlan& plan, int device = 0) : KeyMap(plan.table_ids, plan.row_ids, device) {}
  ~KeyMap();
  KeyMap(const KeyMap&) = delete;
  KeyMap& operator=(const KeyMap&) = delete;

  // Device pointers; absent keys map to 0xFFFFFFFF.  Returns the number of
  // absent keys (synchronises the stream; nullptr = the map's own stream).
  uint64_t lookup(const uint32_t* d_table_ids, const uint64_t* d_row_ids, uint64_t n,
                  uint32_t* d_canon, void* stream = nullptr) const;
  ts_keymap* handle() const { return map_; }

 private:
  ts_keymap* map_ = nullptr;
};

// GPU workload sampler (throughput runs; tiershard_b200.h ts_sampler_*): the
// reference Workload's per-sample law (Poisson(L) length, alias draws over
// the same AliasTable) on per-sample streams, so a U-GPU job can sample each
// rank's samples on its own GPU.  Not the host Workload's stream.
class DeviceSampler {
 public:
  DeviceSampler(const RowDistribution& dist, uint64_t seed, int device = 0);
  ~DeviceSampler();
  DeviceSampler(const DeviceSampler&) = delete;
  DeviceSampler& operator=(const DeviceSampler&) = delete;

  // Samples [sample_begin, sample_begin + samples) of `iteration` into d_rows
  // (device, canonical rows) and d_offsets (device, samples + 1, optional).
  // Returns the occurrence count; ValidationError beyond `capacity`.
  uint64_t sample(uint32_t iteration, uint64_t sample_begin, uint32_t samples, uint32_t* d_rows,
                  uint64_t capacity, uint64_t* d_offsets = nullptr, void* stream = nullptr);

 private:
  ts_sampler* sampler_ = nullptr;
};

// GPU planner preview for what-if sweeps (tiershard_b200.h
// ts_frontier_preview): landmarks, 2- and 3-tier cuts and predicted
// reductions for every (cost model, topology) pair over one distribution.
// The host planner (plan_2tier / plan_3tier) stays authoritative; a preview
// cut can differ from it by a row.
struct PlanPreview {
  FrontierLandmarks landmarks;
  uint64_t dp_cut_2tier = 0;
  uint64_t dp_cut_3tier = 0, flex_cut_3tier = 0;
  double reduction_2tier = 0.0, reduction_3tier = 0.0;
};
struct WhatIf {
  CostModelConfig cost_model;
  Topology topology;
};
std::vector<PlanPreview> preview_plans(const RowDistribution& dist, const std::vector<WhatIf>& what_if,
                                       int device = 0);

// One rank's shard of the tiered table.  Collective when N*W > 1.
class SequenceEmbedding {
 public:
  SequenceEmbedding(const ShardingPlan& plan, const RowDistribution& dist, const Topology& topo,
                    const CostModelConfig& cfg, const DeviceOptions& options,
                    uint64_t hash_seed = kDefaultPlacementSeed);
  // From an imported plan (topology, cost model and placement included).
  SequenceEmbedding(const DevicePlan& plan, const DeviceOptions& options);
  ~SequenceEmbedding();
  SequenceEmbedding(const SequenceEmbedding&) = delete;
  SequenceEmbedding& operator=(const SequenceEmbedding&) = delete;

  // Lookup: d_rows (device) holds this rank's occurrences as canonical row
  // indices; d_out (device) receives the unpooled [occurrences x D] rows.
  void forward(const uint32_t* d_rows, uint64_t occurrences, float* d_out);
  // Same with raw keys (device pointers), looked up through `keys`;
  // ValidationError when a key is absent from the plan.
  void forward_keys(const KeyMap& keys, const uint32_t* d_table_ids, const uint64_t* d_row_ids,
                    uint64_t occurrences, float* d_out);
  // Update for the last forward from d_grad [occurrences x D] (device).
  void backward(const float* d_grad);
  // Host-buffer step: copy, forward, loss 0.5*|out|^2, backward, read loss.
  double train_step_host(const std::vector<uint32_t>& rows);
  // The same over several batches in one call, each step's host-to-device
  // copy overlapping the previous step (pinned host memory copies
  // asynchronously); returns one loss per batch.
  std::vector<double> train_steps_host(const std::vector<const uint32_t*>& rows,
                                       const std::vector<uint64_t>& occurrences);

  // This rank's column of the reference's 7 x U counter block
  // (send/recv global, send/recv intra, dp_local, served, distinct).
  std::vector<uint64_t> counters() const;
  // Weights (and Adagrad state) of canonical rows stored on this rank.
  std::vector<float> read_rows(const std::vector<uint32_t>& rows,
                               std::vector<float>* state = nullptr) const;
  void synchronize() const;
  void* stream() const;  // cudaStream_t
  uint32_t dim() const { return dim_; }

 private:
  void create(uint64_t n_rows, uint64_t dp_cut, uint64_t flex_cut, const std::vector<uint8_t>& dest,
              const Topology& topo, const CostModelConfig& cfg, const DeviceOptions& options);
  ts_table* table_ = nullptr;
  uint32_t dim_ = 0;
  uint32_t gpus_ = 1;
};

}  // namespace tiershard
