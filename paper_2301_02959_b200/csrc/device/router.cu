// ts_router_*: the reference's per-iteration routing + traffic-accounting
// loop (/root/reference/proj/src/simulator.cpp:215-257) as one sm_100a kernel
// over a whole iteration of a LOGICAL U-GPU cluster.
//
// Per occurrence (canonical row r, requester g = the GPU whose sample range
// holds it): tier from the cuts, server from the placement byte, then the six
// GpuCounters increments plus a first-touch test on a (server, row) bitmap for
// the distinct count (the reference's iteration stamps, :158-166, :250-255).
// Integer-only, so the counters are bit-exact by construction; the kernel is
// HBM/L2-bound on the 4 B index stream plus random 1 B remap reads.
//
// Counter aggregation: warp-level __match_any_sync on (counter, gpu) so each
// warp issues one shared-memory atomic per distinct key, then one global
// 64-bit atomic per (block, counter, gpu) at block exit.
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <vector>

#include "common.cuh"

namespace tsd {
namespace {

constexpr int kRouterThreads = 512;
constexpr int kMaxGpus = 256;
constexpr int kSmallU = 8;  // register-counter kernel up to one NVSwitch node

// Everything one routing launch reads.  The distinct-row bitmap is compact:
// an RW row has ONE server (its owner) whoever requests it, so one bit per
// RW row; a Flex row has one server per node (N bits), a DP row one per
// requester (U bits) -- (n - flex_cut) + N (flex_cut - dp_cut) + U dp_cut
// bits instead of U x n (C2 at U = 8: 10.5 MB instead of 80 MB to clear).
struct RouteParams {
  const uint32_t* rows;
  uint64_t occ;
  const uint64_t* req_begin;  // U + 1 occurrence bounds
  const uint8_t* dest;
  uint64_t n_rows, dp_cut, flex_cut;
  uint32_t u, w;
  uint32_t* seen;
  uint64_t flex_base, dp_base;  // bit offsets of the Flex / DP sections
  unsigned long long* counters;
  unsigned* bad_rows;
};

__device__ __forceinline__ void warp_count(unsigned* s_cnt, unsigned key, bool valid) {
  // Aggregate equal keys across the warp: the lowest lane of each group adds.
  const unsigned k = valid ? key : 0xFFFFFFFFu;
  const unsigned peers = __match_any_sync(0xFFFFFFFFu, k);
  if (valid && (peers & lanemask_lt()) == 0) atomicAdd(&s_cnt[key], __popc(peers));
}

// Tier (0 RW, 1 Flex, 2 DP) and server of canonical row r requested by g.
__device__ __forceinline__ void classify(const RouteParams& p, uint32_t r, uint32_t g, uint32_t& kind,
                                         uint32_t& server) {
  if (r < p.dp_cut) {
    kind = 2;
    server = g;
  } else if (r < p.flex_cut) {
    kind = 1;
    server = (g / p.w) * p.w + __ldg(p.dest + r);
  } else {
    kind = 0;
    server = __ldg(p.dest + r);
  }
}

// First touch of (server, r) this iteration (the reference's stamps,
// simulator.cpp:158-166,250-255): test, then claim with an atomic OR.
__device__ __forceinline__ bool first_touch(const RouteParams& p, uint32_t r, uint32_t kind, uint32_t g) {
  uint64_t bit;
  if (kind == 0) {
    bit = r - p.flex_cut;
  } else if (kind == 1) {
    bit = p.flex_base + static_cast<uint64_t>(g / p.w) * (p.flex_cut - p.dp_cut) + (r - p.dp_cut);
  } else {
    bit = p.dp_base + static_cast<uint64_t>(g) * p.dp_cut + r;
  }
  uint32_t* word = p.seen + (bit >> 5);
  const uint32_t m = 1u << (bit & 31);
  if ((*reinterpret_cast<volatile uint32_t*>(word) & m) != 0) return false;
  return (atomicOr(word, m) & m) == 0;
}

// General U (<= 256): warp-aggregated shared-memory counters.
__global__ void __launch_bounds__(kRouterThreads) route_count_kernel(RouteParams p) {
  __shared__ unsigned s_cnt[TS_NUM_COUNTERS * kMaxGpus];
  __shared__ uint64_t s_bounds[kMaxGpus + 1];
  const uint32_t u = p.u;
  for (unsigned i = threadIdx.x; i < TS_NUM_COUNTERS * u; i += blockDim.x) s_cnt[i] = 0;
  for (unsigned i = threadIdx.x; i <= u; i += blockDim.x) s_bounds[i] = p.req_begin[i];
  __syncthreads();

  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // Uniform trip count per warp: every lane runs the same iterations so the
  // match/ballot intrinsics always see the full warp.
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x; base < p.occ; base += stride) {
    const uint64_t idx = base + threadIdx.x;
    bool valid = idx < p.occ;
    uint32_t g = 0, server = 0, kind = 0;
    uint32_t r = 0;
    if (valid) {
      r = __ldg(p.rows + idx);
      if (r >= p.n_rows) {
        atomicAdd(p.bad_rows, 1u);
        valid = false;
      }
    }
    if (valid) {
      // requester: last g with bounds[g] <= idx (binary search)
      uint32_t lo = 0, hi = u;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_bounds[mid] <= idx) lo = mid; else hi = mid;
      }
      g = lo;
      classify(p, r, g, kind, server);
    }
    // requester-side counter: RECV_GLOBAL / RECV_INTRA / DP_LOCAL [g]
    const unsigned req_ctr = kind == 0 ? TS_CTR_RECV_GLOBAL
                                       : (kind == 1 ? TS_CTR_RECV_INTRA : TS_CTR_DP_LOCAL);
    warp_count(s_cnt, req_ctr * u + g, valid);
    // server-side: SEND_GLOBAL / SEND_INTRA [server] (none for DP), SERVED [server]
    const bool sends = valid && kind != 2;
    const unsigned send_ctr = kind == 0 ? TS_CTR_SEND_GLOBAL : TS_CTR_SEND_INTRA;
    warp_count(s_cnt, send_ctr * u + server, sends);
    warp_count(s_cnt, TS_CTR_SERVED * u + server, valid);
    warp_count(s_cnt, TS_CTR_DISTINCT * u + server, valid && first_touch(p, r, kind, g));
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < TS_NUM_COUNTERS * u; i += blockDim.x) {
    if (s_cnt[i]) atomicAdd(p.counters + i, static_cast<unsigned long long>(s_cnt[i]));
  }
}

template <int K>
__device__ __forceinline__ void add_at(uint32_t (&c)[K], uint32_t i, uint32_t v) {
#pragma unroll
  for (int k = 0; k < K; ++k) c[k] += i == static_cast<uint32_t>(k) ? v : 0u;
}

// U <= 8 (one NVSwitch node): per-thread register counters, no warp
// intrinsics on the per-occurrence path.  A thread's grid-stride indices
// ascend, so its requester only moves forward (the per-requester counts
// are flushed when it does); server-side counts are per-thread arrays of 8
// updated by predicated adds; SERVED is not counted at all -- it equals
// SEND_GLOBAL + SEND_INTRA + DP_LOCAL per GPU (a DP row is served by its
// requester) and the host derives it.  Warp shuffle + shared atomics once
// per thread at the end.
__global__ void __launch_bounds__(kRouterThreads) route_count_u8_kernel(RouteParams p) {
  __shared__ unsigned long long s_cnt[TS_NUM_COUNTERS * kSmallU];
  __shared__ uint64_t s_bounds[kSmallU + 1];
  const uint32_t u = p.u;
  for (unsigned i = threadIdx.x; i < TS_NUM_COUNTERS * kSmallU; i += blockDim.x) s_cnt[i] = 0;
  for (unsigned i = threadIdx.x; i <= u; i += blockDim.x) s_bounds[i] = p.req_begin[i];
  __syncthreads();

  uint32_t send_g[kSmallU] = {}, send_i[kSmallU] = {}, dist[kSmallU] = {};
  uint32_t req[3] = {0, 0, 0};
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t g = 0;
  while (g + 1 < u && s_bounds[g + 1] <= idx) ++g;
  const auto flush_req = [&](uint32_t gg) {
    if (req[0]) atomicAdd(&s_cnt[TS_CTR_RECV_GLOBAL * kSmallU + gg], static_cast<unsigned long long>(req[0]));
    if (req[1]) atomicAdd(&s_cnt[TS_CTR_RECV_INTRA * kSmallU + gg], static_cast<unsigned long long>(req[1]));
    if (req[2]) atomicAdd(&s_cnt[TS_CTR_DP_LOCAL * kSmallU + gg], static_cast<unsigned long long>(req[2]));
    req[0] = req[1] = req[2] = 0;
  };
  // kBatch independent occurrences per thread per trip (indices idx,
  // idx + stride, ...: still ascending): their index, placement-byte and
  // bitmap loads are issued together, so each thread keeps kBatch dependent
  // load chains in flight instead of one
  constexpr int kBatch = 4;
  for (; idx < p.occ; idx += kBatch * stride) {
    uint32_t r[kBatch];
    bool ok[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      const uint64_t i = idx + k * stride;
      ok[k] = i < p.occ;
      r[k] = ok[k] ? __ldg(p.rows + i) : 0u;
      if (ok[k] && r[k] >= p.n_rows) {
        atomicAdd(p.bad_rows, 1u);
        ok[k] = false;
      }
    }
    uint32_t d[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) d[k] = ok[k] && r[k] >= p.dp_cut ? __ldg(p.dest + r[k]) : 0u;
    uint32_t* word[kBatch];
    uint32_t mask[kBatch], server[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      word[k] = nullptr;
      mask[k] = 0;
      server[k] = 0;
      if (!ok[k]) continue;
      const uint64_t i = idx + k * stride;
      if (s_bounds[g + 1] <= i) {
        flush_req(g);
        do ++g; while (g + 1 < u && s_bounds[g + 1] <= i);
      }
      uint64_t bit;
      if (r[k] < p.dp_cut) {
        req[2] += 1;
        server[k] = g;
        bit = p.dp_base + static_cast<uint64_t>(g) * p.dp_cut + r[k];
      } else if (r[k] < p.flex_cut) {
        req[1] += 1;
        server[k] = (g / p.w) * p.w + d[k];
        add_at(send_i, server[k], 1u);
        bit = p.flex_base + static_cast<uint64_t>(g / p.w) * (p.flex_cut - p.dp_cut) + (r[k] - p.dp_cut);
      } else {
        req[0] += 1;
        server[k] = d[k];
        add_at(send_g, server[k], 1u);
        bit = r[k] - p.flex_cut;
      }
      word[k] = p.seen + (bit >> 5);
      mask[k] = 1u << (bit & 31);
    }
    uint32_t cur[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) cur[k] = word[k] ? *reinterpret_cast<volatile uint32_t*>(word[k]) : ~0u;
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      if ((cur[k] & mask[k]) == 0 && (atomicOr(word[k], mask[k]) & mask[k]) == 0) add_at(dist, server[k], 1u);
    }
  }
  flush_req(g);
  const unsigned lane = threadIdx.x & 31u;
#pragma unroll
  for (int s = 0; s < kSmallU; ++s) {
    uint32_t a = send_g[s], b = send_i[s], c = dist[s];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
      b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
      c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    }
    if (lane == 0) {
      if (a) atomicAdd(&s_cnt[TS_CTR_SEND_GLOBAL * kSmallU + s], static_cast<unsigned long long>(a));
      if (b) atomicAdd(&s_cnt[TS_CTR_SEND_INTRA * kSmallU + s], static_cast<unsigned long long>(b));
      if (c) atomicAdd(&s_cnt[TS_CTR_DISTINCT * kSmallU + s], static_cast<unsigned long long>(c));
    }
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < TS_NUM_COUNTERS * kSmallU; i += blockDim.x) {
    const unsigned ctr = i / kSmallU, gpu = i % kSmallU;
    if (gpu < u && s_cnt[i]) atomicAdd(p.counters + ctr * u + gpu, s_cnt[i]);
  }
}

}  // namespace
}  // namespace tsd

struct ts_router {
  int device = 0;
  uint64_t n_rows = 0, dp_cut = 0, flex_cut = 0;
  uint32_t num_nodes = 1, gpus_per_node = 1;
  uint8_t* d_dest = nullptr;
  uint32_t* d_seen = nullptr;
  uint64_t seen_words = 0, flex_base = 0, dp_base = 0;
  unsigned long long* d_counters = nullptr;
  unsigned* d_bad = nullptr;
  uint64_t* d_bounds = nullptr;
  uint32_t* d_rows = nullptr;
  uint64_t rows_capacity = 0;
  cudaStream_t stream = nullptr;
  // device time of the last iteration: [0] before the clears, [1] kernel
  // start, [2] kernel end (ts_router_last_timing)
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};

  uint32_t u() const { return num_nodes * gpus_per_node; }

  void run(const uint64_t* d_req_begin, const uint32_t* rows, uint64_t occ, uint64_t* counters) {
    using namespace tsd;
    const uint32_t U = u();
    TSD_CUDA(cudaEventRecord(ev[0], stream));
    TSD_CUDA(cudaMemsetAsync(d_counters, 0, sizeof(unsigned long long) * TS_NUM_COUNTERS * U, stream));
    TSD_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned), stream));
    TSD_CUDA(cudaMemsetAsync(d_seen, 0, sizeof(uint32_t) * seen_words, stream));
    TSD_CUDA(cudaEventRecord(ev[1], stream));
    const bool small = U <= kSmallU;
    if (occ > 0) {
      RouteParams p{rows, occ, d_req_begin, d_dest, n_rows, dp_cut, flex_cut, U, gpus_per_node,
                    d_seen, flex_base, dp_base, d_counters, d_bad};
      const unsigned blocks = static_cast<unsigned>(
          std::min<uint64_t>(ceil_div(occ, kRouterThreads), static_cast<uint64_t>(sm_count()) * 4));
      if (small) {
        // persistent: every resident block once (the grid-stride loop covers the rest)
        int per_sm = 0;
        TSD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, route_count_u8_kernel, kRouterThreads, 0));
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(
            ceil_div(occ, kRouterThreads), static_cast<uint64_t>(sm_count()) * std::max(per_sm, 1)));
        route_count_u8_kernel<<<grid, kRouterThreads, 0, stream>>>(p);
      } else {
        route_count_kernel<<<blocks, kRouterThreads, 0, stream>>>(p);
      }
      TSD_LAUNCH_CHECK();
    }
    TSD_CUDA(cudaEventRecord(ev[2], stream));
    unsigned bad = 0;
    TSD_CUDA(cudaMemcpyAsync(counters, d_counters, sizeof(uint64_t) * TS_NUM_COUNTERS * U,
                             cudaMemcpyDeviceToHost, stream));
    TSD_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost, stream));
    TSD_CUDA(cudaStreamSynchronize(stream));
    if (bad) fail(TS_ERR_VALIDATION, "router: batch references rows outside the plan");
    if (small) {  // SERVED = SEND_GLOBAL + SEND_INTRA + DP_LOCAL on every GPU
      for (uint32_t s = 0; s < U; ++s) {
        counters[TS_CTR_SERVED * U + s] = counters[TS_CTR_SEND_GLOBAL * U + s] +
                                          counters[TS_CTR_SEND_INTRA * U + s] + counters[TS_CTR_DP_LOCAL * U + s];
      }
    }
  }
};

extern "C" {

ts_status ts_router_create(ts_router** out, int device, uint64_t n_rows, uint64_t dp_cut,
                           uint64_t flex_cut, const uint8_t* tier_dest, uint32_t num_nodes,
                           uint32_t gpus_per_node) {
  return tsd::guarded([&] {
    using namespace tsd;
    if (!out) fail(TS_ERR_CONFIG, "ts_router_create: null output handle");
    *out = nullptr;
    const uint64_t u = uint64_t{num_nodes} * gpus_per_node;
    if (num_nodes == 0 || gpus_per_node == 0 || u > kMaxGpus) {
      fail(TS_ERR_CONFIG, "router: need 1 <= N*W <= 256 GPUs");
    }
    if (n_rows == 0 || n_rows > 0xFFFFFFFFull) fail(TS_ERR_VALIDATION, "router: need 1 <= rows < 2^32");
    if (dp_cut > flex_cut || flex_cut > n_rows) {
      fail(TS_ERR_VALIDATION, "assign_rows: plan does not cover the distribution");
    }
    if (!tier_dest) fail(TS_ERR_CONFIG, "router: null placement table");
    use_device(device);
    auto r = std::make_unique<ts_router>();
    r->device = device;
    r->n_rows = n_rows;
    r->dp_cut = dp_cut;
    r->flex_cut = flex_cut;
    r->num_nodes = num_nodes;
    r->gpus_per_node = gpus_per_node;
    r->flex_base = n_rows - flex_cut;
    r->dp_base = r->flex_base + uint64_t{num_nodes} * (flex_cut - dp_cut);
    r->seen_words = (r->dp_base + u * dp_cut + 31) / 32 + 1;
    TSD_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : r->ev) TSD_CUDA(cudaEventCreate(&e));
    TSD_CUDA(dev_alloc(&r->d_dest, n_rows));
    TSD_CUDA(dev_alloc(&r->d_seen, sizeof(uint32_t) * r->seen_words));
    TSD_CUDA(dev_alloc(&r->d_counters, sizeof(unsigned long long) * TS_NUM_COUNTERS * u));
    TSD_CUDA(dev_alloc(&r->d_bad, sizeof(unsigned)));
    TSD_CUDA(dev_alloc(&r->d_bounds, sizeof(uint64_t) * (u + 1)));
    TSD_CUDA(cudaMemcpy(r->d_dest, tier_dest, n_rows, cudaMemcpyHostToDevice));
    // validate placement bytes against U / W once, on the host copy
    for (uint64_t i = dp_cut; i < n_rows; ++i) {
      const uint32_t limit = i < flex_cut ? gpus_per_node : static_cast<uint32_t>(u);
      if (tier_dest[i] >= limit) fail(TS_ERR_VALIDATION, "router: placement byte out of range");
    }
    *out = r.release();
  });
}

ts_status ts_router_iteration(ts_router* r, uint32_t local_batch, const uint64_t* sample_offsets,
                              const uint32_t* rows, uint64_t occurrences, uint64_t* counters) {
  return tsd::guarded([&] {
    using namespace tsd;
    if (!r || !sample_offsets || !counters || (occurrences && !rows)) {
      fail(TS_ERR_CONFIG, "ts_router_iteration: null argument");
    }
    TSD_CUDA(cudaSetDevice(r->device));
    const uint32_t U = r->u();
    if (local_batch == 0) fail(TS_ERR_VALIDATION, "simulate: workload was sampled for a different shape");
    std::vector<uint64_t> bounds(U + 1);
    for (uint32_t g = 0; g <= U; ++g) bounds[g] = sample_offsets[uint64_t{g} * local_batch];
    if (bounds[U] != occurrences) fail(TS_ERR_VALIDATION, "router: sample offsets do not match rows");
    if (occurrences > r->rows_capacity) {
      if (r->d_rows) TSD_CUDA(cudaFree(r->d_rows));
      r->d_rows = nullptr;
      r->rows_capacity = occurrences + occurrences / 8;
      TSD_CUDA(dev_alloc(&r->d_rows, sizeof(uint32_t) * r->rows_capacity));
    }
    TSD_CUDA(cudaMemcpyAsync(r->d_bounds, bounds.data(), sizeof(uint64_t) * (U + 1),
                             cudaMemcpyHostToDevice, r->stream));
    if (occurrences) {
      TSD_CUDA(cudaMemcpyAsync(r->d_rows, rows, sizeof(uint32_t) * occurrences,
                               cudaMemcpyHostToDevice, r->stream));
    }
    r->run(r->d_bounds, r->d_rows, occurrences, counters);
  });
}

ts_status ts_router_iteration_device(ts_router* r, const uint64_t* d_requester_begin,
                                     const uint32_t* d_rows, uint64_t occurrences,
                                     uint64_t* counters) {
  return tsd::guarded([&] {
    using namespace tsd;
    if (!r || !d_requester_begin || !counters || (occurrences && !d_rows)) {
      fail(TS_ERR_CONFIG, "ts_router_iteration_device: null argument");
    }
    TSD_CUDA(cudaSetDevice(r->device));
    r->run(d_requester_begin, d_rows, occurrences, counters);
  });
}

ts_status ts_router_last_timing(ts_router* r, double* kernel_ms, double* total_ms) {
  return tsd::guarded([&] {
    if (!r) tsd::fail(TS_ERR_CONFIG, "ts_router_last_timing: null router");
    TSD_CUDA(cudaSetDevice(r->device));
    float k = 0.f, t = 0.f;
    TSD_CUDA(cudaEventElapsedTime(&k, r->ev[1], r->ev[2]));
    TSD_CUDA(cudaEventElapsedTime(&t, r->ev[0], r->ev[2]));
    if (kernel_ms) *kernel_ms = k;
    if (total_ms) *total_ms = t;
  });
}

ts_status ts_router_destroy(ts_router* r) {
  return tsd::guarded([&] {
    if (!r) return;
    cudaSetDevice(r->device);
    cudaFree(r->d_dest);
    cudaFree(r->d_seen);
    cudaFree(r->d_counters);
    cudaFree(r->d_bad);
    cudaFree(r->d_bounds);
    cudaFree(r->d_rows);
    for (cudaEvent_t e : r->ev) {
      if (e) cudaEventDestroy(e);
    }
    if (r->stream) cudaStreamDestroy(r->stream);
    delete r;
  });
}

}  // extern "C"
