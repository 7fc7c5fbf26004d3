// ts_frontier_preview: GPU planner preview for what-if sweeps (SURVEY.md
// §8(f) row 4).  The host planner (planner.cpp, bit-exact with the
// reference's /root/reference/proj/src/planner.cpp:15-260) stays
// authoritative; this answers "where would the cuts land" for many cost
// models / topologies over one canonical distribution at once.
//
// The DP memory marginal of a row is affine in its probability (table_cost
// differenced, cost_model.cpp): dmem(p) = A + B p.  So the DP frontier is
//   mem(k) = k A + B P(k),   P(k) = sum of the k most probable rows' p,
// and one fp64 prefix scan of p serves every query.  Per query (one thread):
//   a = first argmin of mem  = #rows with A + B p < 0 (p is non-increasing);
//   b = last k with mem(k) <= 0 (mem convex: binary search on [a, n]);
//   c = #rows with p >= p_comm_dp;
//   2-tier cut = b;  3-tier = DP [0, a), Flex while p >= p_comm_flex and
//   mem(a) + k * price <= 0 (planner.cpp plan_3tier);
//   predicted global-a2a reduction = covered P / total P.
// The scan's summation order differs from the host's sequential Neumaier
// sum, so a cut can move by a row where mem(k) crosses zero within rounding.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <vector>

#include "common.cuh"

namespace tsd {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr uint64_t kTile = uint64_t{kThreads} * kItems;

__device__ __forceinline__ double warp_sum(double v) {
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, m);
  return v;
}

// tile sums of p
__global__ void __launch_bounds__(kThreads)
tile_sum_kernel(const double* __restrict__ p, uint64_t n, double* __restrict__ sums) {
  __shared__ double s_w[kThreads / 32];
  const uint64_t base = blockIdx.x * kTile;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * kThreads + threadIdx.x;
    if (i < n) acc += p[i];
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31u) == 0) s_w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) t += s_w[w];
    sums[blockIdx.x] = t;
  }
}

// exclusive scan of the tile sums, one block, sequential chunks
__global__ void __launch_bounds__(1024)
tile_scan_kernel(double* __restrict__ sums, uint64_t tiles) {
  __shared__ double s[1024];
  double carry = 0.0;
  for (uint64_t base = 0; base < tiles; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const double v = i < tiles ? sums[i] : 0.0;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {  // Hillis-Steele inclusive
      const double t = threadIdx.x >= static_cast<unsigned>(off) ? s[threadIdx.x - off] : 0.0;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < tiles) sums[i] = carry + s[threadIdx.x] - v;
    carry += s[1023];
    __syncthreads();
  }
}

// P[k] = sum of p[0..k) for k in [0, n]
__global__ void __launch_bounds__(kThreads)
apply_scan_kernel(const double* __restrict__ p, uint64_t n, const double* __restrict__ tile_off,
                  double* __restrict__ prefix) {
  __shared__ double s[kTile];
  const uint64_t base = blockIdx.x * kTile;
  for (uint32_t j = threadIdx.x; j < kTile; j += kThreads) {
    const uint64_t i = base + j;
    s[j] = i < n ? p[i] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // sequential within the tile: ~4k adds, fp64, in order
    double run = tile_off[blockIdx.x];
    for (uint32_t j = 0; j < kTile && base + j < n; ++j) {
      prefix[base + j] = run;
      run += s[j];
    }
    if (base + kTile >= n) prefix[n] = run;
  }
}

__device__ __forceinline__ double mem_at(const ts_frontier_query& q, const double* prefix, uint64_t k) {
  return static_cast<double>(k) * q.mem_a + q.mem_b * prefix[k];
}

// #leading rows with pred(p) true, p non-increasing and pred monotone
template <typename Pred>
__device__ uint64_t count_leading(const double* p, uint64_t n, Pred pred) {
  uint64_t lo = 0, hi = n;  // answer in [lo, hi]
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (pred(p[mid])) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void query_kernel(const double* __restrict__ p, const double* __restrict__ prefix, uint64_t n,
                             const ts_frontier_query* __restrict__ qs, uint32_t nq,
                             ts_frontier_answer* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq) return;
  const ts_frontier_query q = qs[i];
  ts_frontier_answer r{};
  const double total = prefix[n];
  // a: first argmin of the (convex when mem_b <= 0) frontier
  uint64_t a;
  if (q.mem_b <= 0.0) {
    a = count_leading(p, n, [&](double x) { return q.mem_a + q.mem_b * x < 0.0; });
  } else {
    a = mem_at(q, prefix, n) < 0.0 ? n : 0;
  }
  // b: last k with mem(k) <= 0 -- increasing on [a, n] in the convex case
  uint64_t lo = a, hi = n;
  if (mem_at(q, prefix, a) > 0.0) {
    lo = 0;  // mem(0) = 0: only the origin qualifies
    hi = 0;
  }
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo + 1) / 2;
    if (mem_at(q, prefix, mid) <= 0.0) lo = mid; else hi = mid - 1;
  }
  const uint64_t b = lo;
  const uint64_t c = count_leading(p, n, [&](double x) { return x >= q.p_comm_dp; });
  uint64_t flex = b, dp3 = b;
  if (q.p_comm_flex >= 0.0) {  // heterogeneous tiers: the 3-tier plan
    dp3 = a;
    const double ma = mem_at(q, prefix, a);
    const uint64_t above = count_leading(p, n, [&](double x) { return x >= q.p_comm_flex; });
    uint64_t k_comm = above > a ? above - a : 0;
    uint64_t k_price = n - a;
    if (q.flex_price > 0.0) k_price = ma > 0.0 ? 0 : static_cast<uint64_t>(floor(-ma / q.flex_price));
    flex = a + min(k_comm, min(k_price, n - a));
  }
  r.a = a;
  r.b = b;
  r.c = c;
  r.dp_cut_3tier = dp3;
  r.flex_cut_3tier = flex;
  r.reduction_2tier = total > 0.0 ? prefix[b] / total : 0.0;
  r.reduction_3tier = total > 0.0 ? prefix[flex] / total : 0.0;
  out[i] = r;
}

}  // namespace
}  // namespace tsd

extern "C" ts_status ts_frontier_preview(int device, uint64_t n, const double* probabilities, uint32_t nq,
                                         const ts_frontier_query* queries, ts_frontier_answer* answers) {
  return tsd::guarded([&] {
    using namespace tsd;
    if (!n || !probabilities || (nq && (!queries || !answers))) {
      fail(TS_ERR_CONFIG, "ts_frontier_preview: null argument or empty distribution");
    }
    for (uint64_t i = 1; i < std::min<uint64_t>(n, 1u << 20); ++i) {  // cheap canonical-order check
      if (probabilities[i] > probabilities[i - 1]) {
        fail(TS_ERR_VALIDATION, "frontier: distribution is not in canonical order");
      }
    }
    use_device(device);
    const uint64_t tiles = (n + kTile - 1) / kTile;
    double *d_p = nullptr, *d_prefix = nullptr, *d_sums = nullptr;
    ts_frontier_query* d_q = nullptr;
    ts_frontier_answer* d_a = nullptr;
    cudaStream_t s = nullptr;
    const auto cleanup = [&] {
      if (s) cudaStreamSynchronize(s);
      cudaFree(d_p);
      cudaFree(d_prefix);
      cudaFree(d_sums);
      cudaFree(d_q);
      cudaFree(d_a);
      if (s) cudaStreamDestroy(s);
    };
    try {
      TSD_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      TSD_CUDA(dev_alloc(&d_p, sizeof(double) * n));
      TSD_CUDA(dev_alloc(&d_prefix, sizeof(double) * (n + 1)));
      TSD_CUDA(dev_alloc(&d_sums, sizeof(double) * tiles));
      TSD_CUDA(cudaMemcpyAsync(d_p, probabilities, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      tile_sum_kernel<<<static_cast<unsigned>(tiles), kThreads, 0, s>>>(d_p, n, d_sums);
      TSD_LAUNCH_CHECK();
      tile_scan_kernel<<<1, 1024, 0, s>>>(d_sums, tiles);
      TSD_LAUNCH_CHECK();
      apply_scan_kernel<<<static_cast<unsigned>(tiles), kThreads, 0, s>>>(d_p, n, d_sums, d_prefix);
      TSD_LAUNCH_CHECK();
      if (nq) {
        TSD_CUDA(dev_alloc(&d_q, sizeof(ts_frontier_query) * nq));
        TSD_CUDA(dev_alloc(&d_a, sizeof(ts_frontier_answer) * nq));
        TSD_CUDA(cudaMemcpyAsync(d_q, queries, sizeof(ts_frontier_query) * nq, cudaMemcpyHostToDevice, s));
        query_kernel<<<ceil_div(nq, 128), 128, 0, s>>>(d_p, d_prefix, n, d_q, nq, d_a);
        TSD_LAUNCH_CHECK();
        TSD_CUDA(cudaMemcpyAsync(answers, d_a, sizeof(ts_frontier_answer) * nq, cudaMemcpyDeviceToHost, s));
      }
      TSD_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}
