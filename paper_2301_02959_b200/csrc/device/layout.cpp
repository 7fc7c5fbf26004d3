// Host-only planning helpers of the U > 1 path (include/tiershard_b200.h):
// the shard layout every rank derives from the planner's placement bytes, and
// the per-step all-to-allv plan derived from the all-gathered bucket counts.
// Pure integer arithmetic; unit-tested on the CPU (tests/test_layout.py,
// including a gloo world-size-2 exchange-consistency test).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "layout.hpp"
#include "tiershard_b200.h"

namespace tsd {

void shard_layout(uint64_t n, uint64_t dp_cut, uint64_t flex_cut, const uint8_t* dest, uint32_t N,
                  uint32_t W, uint32_t g, uint32_t* local_id, ShardRows* rows) {
  const uint32_t U = N * W;
  std::vector<uint64_t> flex_total(W, 0), rw_total(U, 0);
  for (uint64_t i = dp_cut; i < flex_cut; ++i) {
    if (dest[i] >= W) throw LayoutError(TS_ERR_VALIDATION, "table: Flex slot byte out of range");
    ++flex_total[dest[i]];
  }
  for (uint64_t i = flex_cut; i < n; ++i) {
    if (dest[i] >= U) throw LayoutError(TS_ERR_VALIDATION, "table: RW owner byte out of range");
    ++rw_total[dest[i]];
  }
  if (local_id) {
    std::vector<uint64_t> flex_next(W, 0), rw_next(U, 0);
    for (uint64_t i = 0; i < dp_cut; ++i) local_id[i] = static_cast<uint32_t>(i);
    for (uint64_t i = dp_cut; i < flex_cut; ++i) {
      local_id[i] = static_cast<uint32_t>(dp_cut + flex_next[dest[i]]++);
    }
    for (uint64_t i = flex_cut; i < n; ++i) {
      const uint8_t o = dest[i];
      local_id[i] = static_cast<uint32_t>(dp_cut + flex_total[o % W] + rw_next[o]++);
    }
  }
  rows->dp = dp_cut;
  rows->flex = flex_total[g % W];
  rows->rw = rw_total[g];
}

void exchange_plan(uint32_t N, uint32_t W, uint32_t g, const uint32_t* all_starts, ExchangePlan* x) {
  const uint32_t U = N * W;
  const uint32_t stride = U + W + 2;  // nb + 1 entries per rank
  const uint32_t node = g / W, slot = g % W;
  auto start_of = [&](uint32_t p, uint32_t b) -> uint64_t { return all_starts[size_t{p} * stride + b]; };
  auto count_of = [&](uint32_t p, uint32_t b) -> uint64_t { return start_of(p, b + 1) - start_of(p, b); };
  x->send_off.assign(2 * U, 0);
  x->send_cnt.assign(2 * U, 0);
  x->recv_off.assign(2 * U, 0);
  x->recv_cnt.assign(2 * U, 0);
  for (uint32_t p = 0; p < U; ++p) {
    x->send_off[2 * p] = start_of(g, p);
    x->send_cnt[2 * p] = p == g ? 0 : count_of(g, p);
    if (p / W == node && p != g) {
      x->send_off[2 * p + 1] = start_of(g, U + p % W);
      x->send_cnt[2 * p + 1] = count_of(g, U + p % W);
    }
  }
  uint64_t acc = 0;
  x->recv_before = 0;
  for (uint32_t p = 0; p < U; ++p) {
    if (p == g) {
      x->recv_before = acc;
      continue;
    }
    x->recv_off[2 * p] = acc;
    x->recv_cnt[2 * p] = count_of(p, g);
    acc += x->recv_cnt[2 * p];
    if (p / W == node) {
      x->recv_off[2 * p + 1] = acc;
      x->recv_cnt[2 * p + 1] = count_of(p, U + slot);
      acc += x->recv_cnt[2 * p + 1];
    }
  }
  x->recv_total = acc;
  x->n_remote = start_of(g, U + W);
}

}  // namespace tsd

namespace tsd {
void set_last_error(const std::string& msg);  // capi_common.cu
}

namespace {

template <typename F>
ts_status host_guard(F&& f) {
  try {
    f();
    return TS_OK;
  } catch (const tsd::LayoutError& e) {
    tsd::set_last_error(e.what());
    return e.status;
  } catch (const std::exception& e) {
    tsd::set_last_error(e.what());
    return TS_ERR_INTERNAL;
  }
}

}  // namespace

namespace tsd {

uint64_t recv_capacity_rows(const ts_table_config& c) {
  const uint64_t U = uint64_t{c.num_nodes} * c.gpus_per_node;
  const uint64_t worst = (U - 1) * c.max_occurrences;
  return c.recv_rows_hint ? std::max<uint64_t>(1, std::min(c.recv_rows_hint, worst)) : std::max<uint64_t>(1, worst);
}

namespace {
uint64_t paged(uint64_t bytes) {
  constexpr uint64_t kPage = uint64_t{2} << 20;
  bytes = std::max<uint64_t>(bytes, 4);
  return bytes > (kPage >> 1) ? (bytes + kPage - 1) / kPage * kPage : bytes;
}
}  // namespace

ts_table_footprint table_footprint(const ts_table_config& c, uint64_t dp_rows, uint64_t flex_rows,
                                   uint64_t rw_rows, bool host_api) {
  ts_table_footprint f{};
  const uint64_t U = uint64_t{c.num_nodes} * c.gpus_per_node;
  const uint64_t D = c.dim, n = c.n_rows, occ = c.max_occurrences;
  const uint64_t local = std::max<uint64_t>(dp_rows + flex_rows + rw_rows, 1);
  f.weights = paged(4 * local * D);
  f.optimizer_state = c.optimizer == TS_OPT_ROWWISE_ADAGRAD ? paged(4 * local) : 0;
  f.remap = U > 1 ? paged(n) + paged(4 * n) : 0;
  // dedup / sort sized for the largest entry count: the batch, plus what
  // the rank serves for its peers at U > 1
  const uint64_t recv = U > 1 ? recv_capacity_rows(c) : 0;
  const uint64_t m = occ + recv;
  const uint64_t tiles = (m + 4095) / 4096;
  const uint64_t short_max = U == 1 ? 32 : 256;
  const uint64_t max_long = m / (short_max + 1) + 1;
  f.step_buffers = 4 * paged(4 * m)                       // keys / values ping-pong
                   + paged(8 * 4 * tiles * 512)             // look-back status
                   + 2 * paged(4 * (m + 1))                 // segment starts + keys
                   + paged(4 * (2 * ((m + 4095) / 4096) + 4 + ((m + 4095) / 4096 + 4095) / 4096 + 1 + 8))
                   + paged(4 * max_long) + paged(4 * (max_long + 1))
                   + paged(4 * (m / 256 + max_long + 1) * D)  // piece partials
                   + (U > 1 ? 2 * paged(4 * m) : 0);        // (key, source) entries
  if (U > 1) {
    f.exchange = 3 * paged(4 * occ)                 // bucket, order, request ids
                 + paged(4 * recv * D)              // gradient receive buffer
                 + 2 * paged(4 * recv);             // received ids / positions
    const uint64_t per_dp = (dp_rows + U - 1) / U;
    f.replicated = paged(4 * std::max<uint64_t>(U * per_dp, 1) * D) + paged(4 * std::max<uint64_t>(U * per_dp, 1));
    if (c.num_nodes > 1) {
      const uint64_t per_flex = (flex_rows + c.num_nodes - 1) / c.num_nodes;
      f.replicated += paged(4 * std::max<uint64_t>(c.num_nodes * per_flex, 1) * D) +
                      paged(4 * std::max<uint64_t>(c.num_nodes * per_flex, 1));
    }
  }
  // ts_table_train_step(s)_host: two id buffers and the table-owned output
  f.host_api = host_api ? 2 * paged(4 * occ) + paged(4 * occ * D) : 0;
  f.total = f.weights + f.optimizer_state + f.remap + f.step_buffers + f.exchange + f.replicated + f.host_api;
  return f;
}

}  // namespace tsd

extern "C" {

ts_status ts_table_plan_footprint(const ts_table_config* cfg, uint64_t dp_rows, uint64_t flex_rows,
                                  uint64_t rw_rows, int host_api, ts_table_footprint* out) {
  if (!cfg || !out) {
    tsd::set_last_error("ts_table_plan_footprint: null argument");
    return TS_ERR_CONFIG;
  }
  if (cfg->num_nodes == 0 || cfg->gpus_per_node == 0 || cfg->dim == 0 || cfg->max_occurrences == 0) {
    tsd::set_last_error("ts_table_plan_footprint: incomplete configuration");
    return TS_ERR_CONFIG;
  }
  *out = tsd::table_footprint(*cfg, dp_rows, flex_rows, rw_rows, host_api != 0);
  return TS_OK;
}


ts_status ts_shard_layout(uint64_t n_rows, uint64_t dp_cut, uint64_t flex_cut, const uint8_t* tier_dest,
                          uint32_t num_nodes, uint32_t gpus_per_node, uint32_t rank, uint32_t* local_id,
                          uint64_t* dp_rows, uint64_t* flex_rows, uint64_t* rw_rows) {
  return host_guard([&] {
    const uint64_t u = uint64_t{num_nodes} * gpus_per_node;
    if (num_nodes == 0 || gpus_per_node == 0 || u > 256 || rank >= u) {
      throw tsd::LayoutError(TS_ERR_CONFIG, "shard_layout: need 1 <= N*W <= 256 and rank < N*W");
    }
    if (dp_cut > flex_cut || flex_cut > n_rows) {
      throw tsd::LayoutError(TS_ERR_VALIDATION, "assign_rows: plan does not cover the distribution");
    }
    if (!tier_dest && n_rows > dp_cut) throw tsd::LayoutError(TS_ERR_CONFIG, "shard_layout: null placement table");
    tsd::ShardRows r;
    tsd::shard_layout(n_rows, dp_cut, flex_cut, tier_dest, num_nodes, gpus_per_node, rank, local_id, &r);
    if (dp_rows) *dp_rows = r.dp;
    if (flex_rows) *flex_rows = r.flex;
    if (rw_rows) *rw_rows = r.rw;
  });
}

ts_status ts_exchange_plan(uint32_t num_nodes, uint32_t gpus_per_node, uint32_t rank,
                           const uint32_t* all_starts, uint64_t* send_off, uint64_t* send_cnt,
                           uint64_t* recv_off, uint64_t* recv_cnt, uint64_t* recv_before,
                           uint64_t* recv_total) {
  return host_guard([&] {
    const uint32_t u = num_nodes * gpus_per_node;
    if (num_nodes == 0 || gpus_per_node == 0 || u > 256 || rank >= u || !all_starts) {
      throw tsd::LayoutError(TS_ERR_CONFIG, "exchange_plan: bad arguments");
    }
    tsd::ExchangePlan x;
    tsd::exchange_plan(num_nodes, gpus_per_node, rank, all_starts, &x);
    auto copy = [&](uint64_t* dst, const std::vector<uint64_t>& src) {
      if (dst) std::memcpy(dst, src.data(), sizeof(uint64_t) * src.size());
    };
    copy(send_off, x.send_off);
    copy(send_cnt, x.send_cnt);
    copy(recv_off, x.recv_off);
    copy(recv_cnt, x.recv_cnt);
    if (recv_before) *recv_before = x.recv_before;
    if (recv_total) *recv_total = x.recv_total;
  });
}

}  // extern "C"
