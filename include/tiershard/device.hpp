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
#include <vector>

#include "tiershard/cost_model.hpp"
#include "tiershard/distribution.hpp"
#include "tiershard/hashing.hpp"
#include "tiershard/planner.hpp"
#include "tiershard/topology.hpp"

struct ts_table;  // C-ABI handle

namespace tiershard {

enum class Optimizer { kSgd = 0, kRowwiseAdagrad = 1 };

using NcclUniqueId = std::array<uint8_t, 128>;

// Fresh communicator id: rank 0 calls it and ships it to the other ranks.
NcclUniqueId new_nccl_unique_id();

struct DeviceOptions {
  int device = 0;
  uint32_t rank = 0;                 // this process's GPU index in [0, N*W)
  uint64_t weight_seed = 1234;       // seeded-hash initial weights
  Optimizer optimizer = Optimizer::kRowwiseAdagrad;
  float learning_rate = 0.01f;
  float epsilon = 1e-8f;
  uint64_t max_occurrences = uint64_t{1} << 22;  // per step, this rank
  const NcclUniqueId* nccl_id = nullptr;         // required when N*W > 1
};

// The per-row placement byte the planner emits for the device: RW owner
// (row_key_hash % U) for RW rows, Flex slot (% W) for Flex rows, 0 for DP.
std::vector<uint8_t> placement_bytes(const ShardingPlan& plan, const RowDistribution& dist,
                                     const Topology& topo,
                                     uint64_t hash_seed = kDefaultPlacementSeed);

// One rank's shard of the tiered table.  Collective when N*W > 1.
class SequenceEmbedding {
 public:
  SequenceEmbedding(const ShardingPlan& plan, const RowDistribution& dist, const Topology& topo,
                    const CostModelConfig& cfg, const DeviceOptions& options,
                    uint64_t hash_seed = kDefaultPlacementSeed);
  ~SequenceEmbedding();
  SequenceEmbedding(const SequenceEmbedding&) = delete;
  SequenceEmbedding& operator=(const SequenceEmbedding&) = delete;

  // Lookup: d_rows (device) holds this rank's occurrences as canonical row
  // indices; d_out (device) receives the unpooled [occurrences x D] rows.
  void forward(const uint32_t* d_rows, uint64_t occurrences, float* d_out);
  // Update for the last forward from d_grad [occurrences x D] (device).
  void backward(const float* d_grad);
  // Host-buffer step: copy, forward, loss 0.5*|out|^2, backward, read loss.
  double train_step_host(const std::vector<uint32_t>& rows);

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
  ts_table* table_ = nullptr;
  uint32_t dim_ = 0;
  uint32_t gpus_ = 1;
};

}  // namespace tiershard
