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

unsigned grid_for(uint64_t n, unsigned per_block) {
  const uint64_t want = (n + per_block - 1) / per_block;
  const uint64_t cap = static_cast<uint64_t>(sm_count()) * 16;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(want, cap)));
}

}  // namespace

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
