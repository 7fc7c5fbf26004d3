// tiershard-b200 — integer mixing used for placement and seed derivation.
//
// These three functions are part of the plan contract: a row's RW owner and
// Flex slot are pure functions of (table_id, row_id, hash_seed), so a plan
// computed by the reference places every row exactly where this library does.
// Anchors: /root/reference/proj/include/tiershard/hashing.hpp:14-39.
// The device side (paper_2301_02959_b200/csrc/device/common.cuh) carries a
// __device__ copy of mix64 with the same constants.
#pragma once

#include <cstdint>

namespace tiershard {

namespace detail {
inline constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;  // 2^64 / phi
inline constexpr uint64_t kMixMul1 = 0xBF58476D1CE4E5B9ull;  // Stafford mix13
inline constexpr uint64_t kMixMul2 = 0x94D049BB133111EBull;
}  // namespace detail

// SplitMix64 output function applied to x + golden increment.
inline constexpr uint64_t mix64(uint64_t x) {
  uint64_t z = x + detail::kGolden;
  z = (z ^ (z >> 30)) * detail::kMixMul1;
  z = (z ^ (z >> 27)) * detail::kMixMul2;
  return z ^ (z >> 31);
}

// Placement key of one embedding row.  RW owner = key % U, Flex slot = key % W.
inline constexpr uint64_t row_key_hash(uint32_t table_id, uint64_t row_id,
                                       uint64_t seed) {
  const uint64_t table_salt = mix64(seed ^ (uint64_t{table_id} * detail::kGolden));
  return mix64(table_salt ^ row_id);
}

// Placement seed used when the caller does not pass one.
inline constexpr uint64_t kDefaultPlacementSeed = 2;

// Seed of the random stream that materializes iteration `index`.
inline constexpr uint64_t derive_seed(uint64_t seed, uint64_t index) {
  return mix64(seed ^ mix64(index + 1));
}

}  // namespace tiershard
