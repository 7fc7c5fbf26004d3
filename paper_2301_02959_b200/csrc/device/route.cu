// Training-path routing kernels for U > 1 (route.cuh).
#include "common.cuh"
#include "route.cuh"

namespace tsd {
namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
bucket_keys_kernel(const uint32_t* __restrict__ rows, uint64_t occ, BucketView bv,
                   uint32_t* __restrict__ bucket, unsigned long long* __restrict__ tier_counts) {
  __shared__ unsigned s_cnt[3];
  if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t local_bucket = bv.u + bv.w;
  unsigned c_rw = 0, c_flex = 0, c_dp = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < occ; i += stride) {
    const uint32_t c = __ldg(rows + i);
    uint32_t b;
    if (c < bv.dp_cut) {
      b = local_bucket;
      ++c_dp;
    } else {
      const uint32_t d = __ldg(bv.dest + c);
      if (c < bv.flex_cut) {
        b = d == bv.slot ? local_bucket : bv.u + d;
        ++c_flex;
      } else {
        b = d == bv.rank ? local_bucket : d;
        ++c_rw;
      }
    }
    bucket[i] = b;
  }
  atomicAdd(&s_cnt[0], c_rw);
  atomicAdd(&s_cnt[1], c_flex);
  atomicAdd(&s_cnt[2], c_dp);
  __syncthreads();
  if (threadIdx.x < 3 && s_cnt[threadIdx.x]) {
    atomicAdd(tier_counts + threadIdx.x, static_cast<unsigned long long>(s_cnt[threadIdx.x]));
  }
}

__global__ void __launch_bounds__(kThreads)
remote_ids_kernel(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ order,
                  uint64_t count, const uint32_t* __restrict__ local, uint32_t* __restrict__ ids) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; j < count; j += stride) {
    ids[j] = __ldg(local + __ldg(rows + __ldg(order + j)));
  }
}

__global__ void __launch_bounds__(kThreads)
remote_ids_upto_kernel(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ order,
                       uint64_t max_count, const uint32_t* __restrict__ d_count,
                       const uint32_t* __restrict__ local, uint32_t* __restrict__ ids) {
  const uint64_t count = min(static_cast<uint64_t>(*d_count), max_count);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; j < count; j += stride) {
    ids[j] = __ldg(local + __ldg(rows + __ldg(order + j)));
  }
}

// One warp per row, float4 lanes; 4 rows in flight per warp.
__global__ void __launch_bounds__(kThreads)
copy_rows_kernel(const float* __restrict__ src, const uint32_t* __restrict__ src_idx,
                 float* __restrict__ dst, const uint32_t* __restrict__ dst_idx, uint64_t count,
                 uint32_t dim) {
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  const uint32_t vecs = dim / 4;
  for (uint64_t j = gwarp; j < count; j += nwarps) {
    const uint64_t s = src_idx ? __ldg(src_idx + j) : j;
    const uint64_t d = dst_idx ? __ldg(dst_idx + j) : j;
    const float4* sp = reinterpret_cast<const float4*>(src + s * dim);
    float4* dp = reinterpret_cast<float4*>(dst + d * dim);
    for (uint32_t v = lane; v < vecs; v += 32) dp[v] = __ldg(sp + v);
  }
}

__global__ void __launch_bounds__(kThreads)
build_entries_kernel(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ local_order,
                     uint64_t n_local, RemapView rv, const uint32_t* __restrict__ recv_ids,
                     uint64_t recv_before, uint64_t recv_total, uint32_t n_occ,
                     uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint64_t total = n_local + recv_total;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; k < total; k += stride) {
    uint32_t key, val;
    if (k < recv_before) {
      key = recv_ids[k];
      val = n_occ + static_cast<uint32_t>(k);
    } else if (k < recv_before + n_local) {
      const uint32_t i = local_order[k - recv_before];
      const uint32_t c = rows[i];
      key = (rv.identity || c < rv.dp_cut) ? c : __ldg(rv.local + c);
      val = i;
    } else {
      const uint64_t r = k - n_local;
      key = recv_ids[r];
      val = n_occ + static_cast<uint32_t>(r);
    }
    keys[k] = key;
    vals[k] = val;
  }
}

__global__ void bucket_starts_kernel(const uint32_t* __restrict__ hist_scan, uint64_t tiles,
                                     uint32_t nb, uint32_t occ, uint32_t* __restrict__ out) {
  // an empty batch is not sorted at all (hist_scan holds a previous batch's
  // offsets): every bucket starts at 0
  for (uint32_t b = threadIdx.x; b <= nb; b += blockDim.x) {
    out[b] = b < nb && occ ? hist_scan[static_cast<uint64_t>(b) * tiles] : occ;
  }
}

__global__ void __launch_bounds__(kThreads)
scatter_rows_loss_kernel(const float* __restrict__ src, float* __restrict__ dst,
                         const uint32_t* __restrict__ dst_idx, uint64_t count, uint32_t dim,
                         double* __restrict__ loss_partials) {
  __shared__ float s_sq[kThreads / 32];
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  const uint32_t vecs = dim / 4;
  float sq = 0.0f;
  for (uint64_t j = gwarp; j < count; j += nwarps) {
    const float4* sp = reinterpret_cast<const float4*>(src + j * dim);
    float4* dp = reinterpret_cast<float4*>(dst + static_cast<uint64_t>(__ldg(dst_idx + j)) * dim);
    for (uint32_t v = lane; v < vecs; v += 32) {
      const float4 x = __ldg(sp + v);
      dp[v] = x;
      sq = __fmaf_rn(x.x, x.x, sq);
      sq = __fmaf_rn(x.y, x.y, sq);
      sq = __fmaf_rn(x.z, x.z, sq);
      sq = __fmaf_rn(x.w, x.w, sq);
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, m);
  if (lane == 0) s_sq[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) acc += static_cast<double>(s_sq[w]);
    loss_partials[blockIdx.x] = acc;
  }
}

// ---- fused route (launch_route_buckets) -------------------------------------
constexpr int kRouteThreads = 512;
constexpr int kRouteWarps = kRouteThreads / 32;
constexpr int kRouteItems = 8;
constexpr uint32_t kRouteTile = kRouteThreads * kRouteItems;  // occurrences per block: 8 chunks of 512

__device__ __forceinline__ uint32_t route_bucket(uint32_t c, const BucketView& bv, uint32_t local_bucket,
                                                 int* tier) {
  if (c < bv.dp_cut) {
    *tier = 2;
    return local_bucket;
  }
  const uint32_t d = __ldg(bv.dest + c);
  if (c < bv.flex_cut) {
    *tier = 1;
    return d == bv.slot ? local_bucket : bv.u + d;
  }
  *tier = 0;
  return d == bv.rank ? local_bucket : d;
}

// hist[b * tiles + tile] = occurrences of bucket b in the tile
__global__ void __launch_bounds__(kRouteThreads)
route_hist_kernel(const uint32_t* __restrict__ rows, uint64_t occ, BucketView bv, uint32_t nb,
                  uint32_t* __restrict__ hist, unsigned long long* __restrict__ tier_counts) {
  __shared__ unsigned s_cnt[kRouteMaxBuckets];
  __shared__ unsigned s_tier[3];
  const uint32_t tiles = static_cast<uint32_t>(gridDim.x);
  for (uint32_t b = threadIdx.x; b < kRouteMaxBuckets; b += kRouteThreads) s_cnt[b] = 0;
  if (threadIdx.x < 3) s_tier[threadIdx.x] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t local_bucket = nb - 1;
  unsigned tc[3] = {0, 0, 0};
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kRouteTile + threadIdx.x;
  // every load of the thread's kRouteItems occurrences in flight at once
  uint32_t c[kRouteItems], b[kRouteItems];
#pragma unroll
  for (int k = 0; k < kRouteItems; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * kRouteThreads;
    c[k] = i < occ ? __ldg(rows + i) : 0;
  }
#pragma unroll
  for (int k = 0; k < kRouteItems; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * kRouteThreads;
    b[k] = kRouteMaxBuckets;  // sentinel: past the batch
    if (i < occ) {
      int tier;
      b[k] = route_bucket(c[k], bv, local_bucket, &tier);
      ++tc[tier];
    }
  }
#pragma unroll
  for (int k = 0; k < kRouteItems; ++k) {
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, b[k]);
    if (b[k] < kRouteMaxBuckets && lane == static_cast<unsigned>(__ffs(peers) - 1)) {
      atomicAdd(&s_cnt[b[k]], __popc(peers));
    }
  }
  for (int t = 0; t < 3; ++t) {
    unsigned v = tc[t];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (lane == 0 && v) atomicAdd(&s_tier[t], v);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nb; b += kRouteThreads) {
    hist[static_cast<uint64_t>(b) * tiles + blockIdx.x] = s_cnt[b];
  }
  if (threadIdx.x < 3 && s_tier[threadIdx.x]) {
    atomicAdd(tier_counts + threadIdx.x, static_cast<unsigned long long>(s_tier[threadIdx.x]));
  }
}

// In-place exclusive scan of hist[0..n) (one block), starts[b] = hist[b *
// tiles] after it, starts[nb] = occ.
__global__ void __launch_bounds__(1024)
route_scan_kernel(uint32_t* __restrict__ hist, uint64_t tiles, uint32_t nb, uint32_t occ,
                  uint32_t* __restrict__ starts) {
  __shared__ uint32_t s_warp[32];
  const uint64_t n = tiles * nb;
  const uint64_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint64_t lo = min(n, per * threadIdx.x), hi = min(n, lo + per);
  uint32_t sum = 0;
  for (uint64_t j = lo; j < hi; ++j) sum += hist[j];
  // block exclusive scan of the per-thread sums
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= static_cast<unsigned>(o)) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (blockDim.x >> 5) ? s_warp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= static_cast<unsigned>(o)) w += v;
    }
    s_warp[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  uint32_t run = incl - sum + (warp ? s_warp[warp - 1] : 0);
  for (uint64_t j = lo; j < hi; ++j) {
    const uint32_t v = hist[j];
    hist[j] = run;
    run += v;
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b <= nb; b += blockDim.x) {
    starts[b] = (b < nb && tiles) ? hist[static_cast<uint64_t>(b) * tiles] : (b < nb ? 0u : occ);
  }
}

__global__ void __launch_bounds__(kRouteThreads)
route_scatter_kernel(const uint32_t* __restrict__ rows, uint64_t occ, BucketView bv, uint32_t nb,
                     const uint32_t* __restrict__ hist, uint32_t* __restrict__ order,
                     const uint32_t* __restrict__ local, uint32_t* __restrict__ ids) {
  __shared__ uint32_t s_base[kRouteMaxBuckets];              // next position per bucket
  __shared__ uint32_t s_wcnt[kRouteWarps][kRouteMaxBuckets];  // chunk counts -> warp offsets
  const uint32_t tiles = static_cast<uint32_t>(gridDim.x);
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t local_bucket = nb - 1;
  for (uint32_t b = threadIdx.x; b < nb; b += kRouteThreads) {
    s_base[b] = hist[static_cast<uint64_t>(b) * tiles + blockIdx.x];
  }
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kRouteTile;
  // loads first (rows, destinations, remote ids), all in flight at once
  uint32_t bk[kRouteItems], id[kRouteItems];
#pragma unroll
  for (int k = 0; k < kRouteItems; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * kRouteThreads + threadIdx.x;
    id[k] = i < occ ? __ldg(rows + i) : 0;
  }
#pragma unroll
  for (int k = 0; k < kRouteItems; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * kRouteThreads + threadIdx.x;
    int tier;
    bk[k] = i < occ ? route_bucket(id[k], bv, local_bucket, &tier) : kRouteMaxBuckets;
  }
#pragma unroll
  for (int k = 0; k < kRouteItems; ++k) {
    if (bk[k] < local_bucket) id[k] = __ldg(local + id[k]);
  }
#pragma unroll
  for (int k = 0; k < kRouteItems; ++k) {
    const uint32_t k0 = static_cast<uint32_t>(k) * kRouteThreads;
    if (base + k0 >= occ) break;  // uniform over the block
    for (uint32_t e = threadIdx.x; e < kRouteWarps * kRouteMaxBuckets; e += kRouteThreads) {
      (&s_wcnt[0][0])[e] = 0;
    }
    __syncthreads();
    const uint64_t i = base + k0 + threadIdx.x;
    const bool valid = i < occ;
    const uint32_t b = bk[k];
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, b);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    if (valid && lane == static_cast<unsigned>(__ffs(peers) - 1)) s_wcnt[warp][b] = __popc(peers);
    __syncthreads();
    for (uint32_t bb = threadIdx.x; bb < nb; bb += kRouteThreads) {  // warp offsets, bucket bb
      uint32_t run = s_base[bb];
      for (int w = 0; w < kRouteWarps; ++w) {
        const uint32_t v = s_wcnt[w][bb];
        s_wcnt[w][bb] = run;
        run += v;
      }
      s_base[bb] = run;
    }
    __syncthreads();
    if (valid) {
      const uint32_t pos = s_wcnt[warp][b] + rank;
      order[pos] = static_cast<uint32_t>(i);
      if (b != local_bucket) ids[pos] = id[k];
    }
    __syncthreads();
  }
}

unsigned grid_for(uint64_t n, unsigned per_block) {
  const uint64_t want = (n + per_block - 1) / per_block;
  const uint64_t cap = static_cast<uint64_t>(sm_count()) * 16;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(want, cap)));
}

}  // namespace

uint64_t route_hist_elems(uint64_t occ, uint32_t nb) {
  return std::max<uint64_t>(1, (occ + kRouteTile - 1) / kRouteTile) * nb;
}

void launch_route_buckets(const uint32_t* rows, uint64_t occ, const BucketView& bv, uint32_t nb, uint32_t* hist,
                          uint32_t* order, uint32_t* starts, const uint32_t* local, uint32_t* ids,
                          unsigned long long* tier_counts, cudaStream_t stream) {
  if (nb == 0 || nb > kRouteMaxBuckets) fail(TS_ERR_CONFIG, "route: bucket count out of range");
  const uint64_t tiles = (occ + kRouteTile - 1) / kRouteTile;
  if (tiles > 0x7FFFFFFFu) fail(TS_ERR_VALIDATION, "route: batch too large");
  if (tiles) {
    route_hist_kernel<<<static_cast<unsigned>(tiles), kRouteThreads, 0, stream>>>(rows, occ, bv, nb, hist,
                                                                                 tier_counts);
    TSD_LAUNCH_CHECK();
  }
  route_scan_kernel<<<1, 1024, 0, stream>>>(hist, tiles, nb, static_cast<uint32_t>(occ), starts);
  TSD_LAUNCH_CHECK();
  if (tiles) {
    route_scatter_kernel<<<static_cast<unsigned>(tiles), kRouteThreads, 0, stream>>>(rows, occ, bv, nb, hist,
                                                                                    order, local, ids);
    TSD_LAUNCH_CHECK();
  }
}

void launch_bucket_starts(const uint32_t* hist_scan, uint64_t tiles, uint32_t nb, uint32_t occ,
                          uint32_t* out, cudaStream_t stream) {
  bucket_starts_kernel<<<1, 256, 0, stream>>>(hist_scan, tiles, nb, occ, out);
  TSD_LAUNCH_CHECK();
}

void launch_scatter_rows_loss(const float* src, float* dst, const uint32_t* dst_idx, uint64_t count,
                              uint32_t dim, double* loss_partials, unsigned grid,
                              cudaStream_t stream) {
  scatter_rows_loss_kernel<<<grid, kThreads, 0, stream>>>(src, dst, dst_idx, count, dim, loss_partials);
  TSD_LAUNCH_CHECK();
}

void launch_bucket_keys(const uint32_t* rows, uint64_t occ, const BucketView& bv, uint32_t* bucket,
                        unsigned long long* tier_counts, cudaStream_t stream) {
  if (occ == 0) return;
  bucket_keys_kernel<<<grid_for(occ, kThreads * 4), kThreads, 0, stream>>>(rows, occ, bv, bucket,
                                                                           tier_counts);
  TSD_LAUNCH_CHECK();
}

void launch_remote_ids(const uint32_t* rows, const uint32_t* order, uint64_t count,
                       const uint32_t* local, uint32_t* ids, cudaStream_t stream) {
  if (count == 0) return;
  remote_ids_kernel<<<grid_for(count, kThreads * 4), kThreads, 0, stream>>>(rows, order, count, local, ids);
  TSD_LAUNCH_CHECK();
}

void launch_remote_ids_upto(const uint32_t* rows, const uint32_t* order, uint64_t max_count,
                            const uint32_t* d_count, const uint32_t* local, uint32_t* ids,
                            cudaStream_t stream) {
  if (max_count == 0) return;
  remote_ids_upto_kernel<<<grid_for(max_count, kThreads * 4), kThreads, 0, stream>>>(rows, order, max_count,
                                                                                   d_count, local, ids);
  TSD_LAUNCH_CHECK();
}

void launch_copy_rows(const float* src, const uint32_t* src_idx, float* dst, const uint32_t* dst_idx,
                      uint64_t count, uint32_t dim, cudaStream_t stream) {
  if (count == 0) return;
  copy_rows_kernel<<<grid_for(count, (kThreads / 32) * 4), kThreads, 0, stream>>>(
      src, src_idx, dst, dst_idx, count, dim);
  TSD_LAUNCH_CHECK();
}

void launch_build_entries(const uint32_t* rows, const uint32_t* local_order, uint64_t n_local,
                          const RemapView& rv, const uint32_t* recv_ids, uint64_t recv_before,
                          uint64_t recv_total, uint32_t n_occ, uint32_t* keys, uint32_t* vals,
                          cudaStream_t stream) {
  const uint64_t total = n_local + recv_total;
  if (total == 0) return;
  build_entries_kernel<<<grid_for(total, kThreads * 4), kThreads, 0, stream>>>(
      rows, local_order, n_local, rv, recv_ids, recv_before, recv_total, n_occ, keys, vals);
  TSD_LAUNCH_CHECK();
}

}  // namespace tsd
