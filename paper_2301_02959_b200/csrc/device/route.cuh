// Training-path routing for U > 1 ranks: bucket every occurrence by where it
// is served (the per-occurrence decision of simulator.cpp:228-249), compact
// the remote ones per destination with one stable counting pass (the radix
// scatter with digit = bucket), and move rows between the compacted order and
// the unpooled [occ x dim] layout.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "embedding.cuh"

namespace tsd {

// Bucket ids: RW to server s -> s (s in [0,U)); Flex to slot t -> U + t;
// served locally (DP, own RW, own Flex slot) -> U + W  (sorted last).
struct BucketView {
  const uint8_t* dest = nullptr;
  uint64_t dp_cut = 0, flex_cut = 0;
  uint32_t u = 1, w = 1, rank = 0, slot = 0;
};

// bucket[i] for every occurrence + tier counts of this requester:
// tier_counts[0..2] += (#RW, #Flex, #DP) occurrences (u64 device).
void launch_bucket_keys(const uint32_t* rows, uint64_t occ, const BucketView& bv,
                        uint32_t* bucket, unsigned long long* tier_counts, cudaStream_t stream);

// ids[j] = local id at the serving rank of rows[order[j]], j < count.
void launch_remote_ids(const uint32_t* rows, const uint32_t* order, uint64_t count,
                       const uint32_t* local, uint32_t* ids, cudaStream_t stream);

// Same for j < *d_count (device scalar), launched for up to max_count.
void launch_remote_ids_upto(const uint32_t* rows, const uint32_t* order, uint64_t max_count,
                            const uint32_t* d_count, const uint32_t* local, uint32_t* ids,
                            cudaStream_t stream);

// The whole route in three kernels, no sort (nb <= kRouteMaxBuckets):
// per-tile bucket histograms (+ the tier counts), one scan of them
// (bucket-major) that also writes starts[0..nb] (starts[nb] = occ), and a
// stable scatter -- warp match ranks within each 512-occurrence chunk of a
// tile -- that writes order[] (occurrences stably by bucket, the order the
// counting sort gives) and, for the remote buckets, ids[j] = local id of
// rows[order[j]] at its server.  `hist` holds route_hist_elems(occ, nb).
constexpr uint32_t kRouteMaxBuckets = 32;
uint64_t route_hist_elems(uint64_t occ, uint32_t nb);
void launch_route_buckets(const uint32_t* rows, uint64_t occ, const BucketView& bv, uint32_t nb, uint32_t* hist,
                          uint32_t* order, uint32_t* starts, const uint32_t* local, uint32_t* ids,
                          unsigned long long* tier_counts, cudaStream_t stream);

// dst[dst_idx ? dst_idx[j] : j] = src[src_idx ? src_idx[j] : j] for j < count
// (rows of `dim` floats).
void launch_copy_rows(const float* src, const uint32_t* src_idx, float* dst,
                      const uint32_t* dst_idx, uint64_t count, uint32_t dim, cudaStream_t stream);

// Server-side dedup input in ascending source-rank order:
//   [recv entries from ranks < g][local entries][recv entries from ranks > g]
// local entry j (occurrence order[j], j < n_local): key = local id, val = order[j]
// recv entry r: key = recv_ids[r], val = n_occ + r.
void launch_build_entries(const uint32_t* rows, const uint32_t* local_order, uint64_t n_local,
                          const RemapView& rv, const uint32_t* recv_ids, uint64_t recv_before,
                          uint64_t recv_total, uint32_t n_occ, uint32_t* keys, uint32_t* vals,
                          cudaStream_t stream);

// out[b] = hist_scan[b * tiles] (start of bucket b after the single counting
// pass), out[nb] = occ.
void launch_bucket_starts(const uint32_t* hist_scan, uint64_t tiles, uint32_t nb, uint32_t occ,
                          uint32_t* out, cudaStream_t stream);

// dst[dst_idx[j]] = src[j] for j < count, plus per-block partial sums of
// dst^2 into loss_partials[grid] (the remote half of the synthetic loss).
void launch_scatter_rows_loss(const float* src, float* dst, const uint32_t* dst_idx, uint64_t count,
                              uint32_t dim, double* loss_partials, unsigned grid,
                              cudaStream_t stream);

}  // namespace tsd
