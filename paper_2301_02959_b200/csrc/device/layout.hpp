// Host-only shard-layout and exchange-plan arithmetic (layout.cpp).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tiershard_b200.h"

namespace tsd {

struct LayoutError : std::runtime_error {
  ts_status status;
  LayoutError(ts_status st, const std::string& m) : std::runtime_error(m), status(st) {}
};

struct ShardRows {
  uint64_t dp = 0, flex = 0, rw = 0;
};

// local_id may be nullptr (counts only).
void shard_layout(uint64_t n, uint64_t dp_cut, uint64_t flex_cut, const uint8_t* dest, uint32_t N,
                  uint32_t W, uint32_t g, uint32_t* local_id, ShardRows* rows);

struct ExchangePlan {
  std::vector<uint64_t> send_off, send_cnt, recv_off, recv_cnt;  // 2*U, [2p] RW, [2p+1] Flex
  uint64_t recv_before = 0, recv_total = 0, n_remote = 0;
};

// all_starts: [U][U+W+2] bucket starts of every rank.
void exchange_plan(uint32_t N, uint32_t W, uint32_t g, const uint32_t* all_starts, ExchangePlan* x);

// Gradient receive-buffer capacity (rows) of a U > 1 rank: the caller's
// recv_rows_hint, else the worst case (every peer's whole batch).
uint64_t recv_capacity_rows(const ts_table_config& c);

// Device bytes one rank of a table allocates (ts_table_create + the step
// buffers its entry points size), itemised; mirrors table.cu's allocations,
// each rounded like DevBuf / dev_alloc (whole 2 MiB pages above 1 MiB).
ts_table_footprint table_footprint(const ts_table_config& c, uint64_t dp_rows, uint64_t flex_rows,
                                   uint64_t rw_rows, bool host_api);

}  // namespace tsd
