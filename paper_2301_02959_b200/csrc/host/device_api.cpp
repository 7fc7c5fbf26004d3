// C++ front door over the C-ABI table handle (tiershard/device.hpp).
#include "tiershard/device.hpp"

#include <cstring>

#include "capi_check.hpp"
#include "parallel.hpp"
#include "tiershard/cost_model.hpp"
#include "tiershard/error.hpp"
#include "tiershard/rng.hpp"
#include "tiershard/simulator.hpp"
#include "tiershard_b200.h"

namespace tiershard {

NcclUniqueId new_nccl_unique_id() {
  NcclUniqueId id{};
  detail::check(ts_nccl_unique_id(id.data()));
  return id;
}

std::vector<uint8_t> placement_bytes(const ShardingPlan& plan, const RowDistribution& dist,
                                     const Topology& topo, uint64_t hash_seed) {
  if (topo.total_gpus() > 256) throw ConfigError("device path: at most 256 GPUs");
  const std::vector<RowPlacement> pl = assign_rows(plan, dist, topo, hash_seed);
  std::vector<uint8_t> dest(pl.size(), 0);
  detail::parallel_for(pl.size(), [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      dest[i] = static_cast<uint8_t>(pl[i].tier == Tier::kFlex ? pl[i].flex_slot : pl[i].owner_gpu);
    }
  });
  return dest;
}

SequenceEmbedding::SequenceEmbedding(const ShardingPlan& plan, const RowDistribution& dist,
                                     const Topology& topo, const CostModelConfig& cfg,
                                     const DeviceOptions& options, uint64_t hash_seed) {
  cfg.validate();
  topo.validate();
  create(dist.rows().size(), plan.dp_cut, plan.flex_cut, placement_bytes(plan, dist, topo, hash_seed),
         topo, cfg, options);
}

SequenceEmbedding::SequenceEmbedding(const DevicePlan& plan, const DeviceOptions& options) {
  plan.cost_model.validate();
  plan.topology.validate();
  create(plan.table_ids.size(), plan.plan.dp_cut, plan.plan.flex_cut, plan.placement, plan.topology,
         plan.cost_model, options);
}

void SequenceEmbedding::create(uint64_t n_rows, uint64_t dp_cut, uint64_t flex_cut,
                               const std::vector<uint8_t>& dest, const Topology& topo,
                               const CostModelConfig& cfg, const DeviceOptions& options) {
  if (cfg.scalar_bytes != 4) throw ConfigError("device path: fp32 tables only (scalar_bytes = 4)");
  if (dest.size() != n_rows) throw ValidationError("device path: placement does not cover the rows");
  dim_ = cfg.embedding_dim;
  gpus_ = topo.total_gpus();
  ts_table_config c{};
  c.num_nodes = topo.num_nodes;
  c.gpus_per_node = topo.gpus_per_node;
  c.rank = options.rank;
  c.device = options.device;
  c.dim = cfg.embedding_dim;
  c.n_rows = n_rows;
  c.dp_cut = dp_cut;
  c.flex_cut = flex_cut;
  c.weight_seed = options.weight_seed;
  c.optimizer = options.optimizer == Optimizer::kSgd ? TS_OPT_SGD : TS_OPT_ROWWISE_ADAGRAD;
  c.lr = options.learning_rate;
  c.eps = options.epsilon;
  c.max_occurrences = options.max_occurrences;
  c.nccl_unique_id = options.nccl_id ? options.nccl_id->data() : nullptr;
  c.group = options.group ? options.group->handle() : nullptr;
  c.recv_rows_hint = options.recv_rows_hint;
  detail::check(ts_table_create(&table_, &c, dest.data()));
}

DeviceGroup::DeviceGroup(uint32_t ranks) { detail::check(ts_group_create(&group_, ranks)); }

DeviceGroup::~DeviceGroup() {
  if (group_) ts_group_destroy(group_);
}

void DeviceGroup::abort() { detail::check(ts_group_abort(group_)); }

std::vector<double> SequenceEmbedding::train_steps_host(const std::vector<const uint32_t*>& rows,
                                                        const std::vector<uint64_t>& occurrences) {
  if (rows.size() != occurrences.size()) throw ConfigError("train_steps_host: rows / occurrences size mismatch");
  std::vector<double> losses(rows.size());
  detail::check(ts_table_train_steps_host(table_, rows.data(), occurrences.data(),
                                          static_cast<uint32_t>(rows.size()), losses.data()));
  return losses;
}

SequenceEmbedding::~SequenceEmbedding() {
  if (table_) ts_table_destroy(table_);
}

void SequenceEmbedding::forward(const uint32_t* d_rows, uint64_t occurrences, float* d_out) {
  detail::check(ts_table_forward(table_, d_rows, occurrences, d_out));
}

void SequenceEmbedding::forward_keys(const KeyMap& keys, const uint32_t* d_table_ids,
                                     const uint64_t* d_row_ids, uint64_t occurrences, float* d_out) {
  detail::check(ts_table_forward_keys(table_, keys.handle(), d_table_ids, d_row_ids, occurrences, d_out));
}

KeyMap::KeyMap(const std::vector<uint32_t>& table_ids, const std::vector<uint64_t>& row_ids, int device) {
  if (table_ids.size() != row_ids.size()) throw ConfigError("KeyMap: table_ids / row_ids size mismatch");
  detail::check(ts_keymap_create(&map_, device, table_ids.size(), table_ids.data(), row_ids.data()));
}

KeyMap::~KeyMap() {
  if (map_) ts_keymap_destroy(map_);
}

uint64_t KeyMap::lookup(const uint32_t* d_table_ids, const uint64_t* d_row_ids, uint64_t n,
                        uint32_t* d_canon, void* stream) const {
  uint64_t misses = 0;
  detail::check(ts_keymap_lookup(map_, d_table_ids, d_row_ids, n, d_canon, stream, &misses));
  return misses;
}

DeviceSampler::DeviceSampler(const RowDistribution& dist, uint64_t seed, int device) {
  if (dist.rows().empty()) throw ValidationError("workload: distribution has no materialized rows");
  std::vector<double> w(dist.rows().size());  // as Workload's constructor (simulator.cpp)
  for (size_t i = 0; i < w.size(); ++i) w[i] = dist.rows()[i].probability;
  const AliasTable table(w);
  detail::check(ts_sampler_create(&sampler_, device, w.size(), table.probabilities().data(),
                                  table.aliases().data(), dist.expected_length(), seed));
}

DeviceSampler::~DeviceSampler() {
  if (sampler_) ts_sampler_destroy(sampler_);
}

uint64_t DeviceSampler::sample(uint32_t iteration, uint64_t sample_begin, uint32_t samples, uint32_t* d_rows,
                               uint64_t capacity, uint64_t* d_offsets, void* stream) {
  uint64_t occ = 0;
  detail::check(ts_sampler_iteration(sampler_, iteration, sample_begin, samples, d_rows, capacity, d_offsets,
                                     &occ, stream));
  return occ;
}

std::vector<PlanPreview> preview_plans(const RowDistribution& dist, const std::vector<WhatIf>& what_if,
                                       int device) {
  if (dist.rows().empty()) throw ValidationError("frontier: distribution has no materialized rows");
  if (!dist.is_sorted()) throw ValidationError("frontier: distribution is not in canonical order");
  std::vector<ts_frontier_query> q(what_if.size());
  for (size_t i = 0; i < what_if.size(); ++i) {
    const CostModelConfig& cfg = what_if[i].cost_model;
    const Topology& topo = what_if[i].topology;
    cfg.validate();
    topo.validate();
    // the DP memory marginal is affine in p (table_cost differenced)
    const double m0 = marginal_cost_dp(0.0, cfg, topo).memory_bytes;
    const double m1 = marginal_cost_dp(1.0, cfg, topo).memory_bytes;
    const Breakpoints bp = find_breakpoints(cfg, topo);
    q[i].mem_a = m0;
    q[i].mem_b = m1 - m0;
    q[i].p_comm_dp = bp.p_comm_dp;
    q[i].flex_price = bp.flex_mem_price_bytes;
    q[i].p_comm_flex = topo.has_fast_intra_tier() && bp.p_comm_flex ? *bp.p_comm_flex : -1.0;
  }
  std::vector<double> p(dist.rows().size());
  for (size_t i = 0; i < p.size(); ++i) p[i] = dist.rows()[i].probability;
  std::vector<ts_frontier_answer> a(q.size());
  detail::check(ts_frontier_preview(device, p.size(), p.data(), static_cast<uint32_t>(q.size()), q.data(),
                                    a.data()));
  std::vector<PlanPreview> out(q.size());
  for (size_t i = 0; i < q.size(); ++i) {
    out[i].landmarks.a = a[i].a;
    out[i].landmarks.b = a[i].b;
    out[i].landmarks.c = a[i].c;
    out[i].landmarks.d = p.size();
    out[i].dp_cut_2tier = a[i].b;
    out[i].dp_cut_3tier = a[i].dp_cut_3tier;
    out[i].flex_cut_3tier = a[i].flex_cut_3tier;
    out[i].reduction_2tier = a[i].reduction_2tier;
    out[i].reduction_3tier = a[i].reduction_3tier;
  }
  return out;
}

void SequenceEmbedding::backward(const float* d_grad) { detail::check(ts_table_backward(table_, d_grad)); }

double SequenceEmbedding::train_step_host(const std::vector<uint32_t>& rows) {
  double loss = 0.0;
  detail::check(ts_table_train_step_host(table_, rows.data(), rows.size(), &loss));
  return loss;
}

std::vector<uint64_t> SequenceEmbedding::counters() const {
  std::vector<uint64_t> c(size_t{TS_NUM_COUNTERS} * gpus_);
  detail::check(ts_table_counters(table_, c.data()));
  return c;
}

std::vector<float> SequenceEmbedding::read_rows(const std::vector<uint32_t>& rows,
                                                std::vector<float>* state) const {
  std::vector<float> w(rows.size() * dim_);
  if (state) state->assign(rows.size(), 0.0f);
  detail::check(ts_table_read_rows(table_, rows.data(), rows.size(), w.data(),
                                   state ? state->data() : nullptr));
  return w;
}

void SequenceEmbedding::synchronize() const { detail::check(ts_table_synchronize(table_)); }

void* SequenceEmbedding::stream() const {
  void* s = nullptr;
  detail::check(ts_table_stream(table_, &s));
  return s;
}

}  // namespace tiershard
