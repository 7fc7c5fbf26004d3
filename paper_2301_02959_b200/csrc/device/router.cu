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

__device__ __forceinline__ void warp_count(unsigned* s_cnt, unsigned key, bool valid) {
  // Aggregate equal keys across the warp: the lowest lane of each group adds.
  const unsigned k = valid ? key : 0xFFFFFFFFu;
  const unsigned peers = __match_any_sync(0xFFFFFFFFu, k);
  if (valid && (peers & lanemask_lt()) == 0) atomicAdd(&s_cnt[key], __popc(peers));
}

__global__ void __launch_bounds__(kRouterThreads)
route_count_kernel(const uint32_t* __restrict__ rows, uint64_t occ,
                   const uint64_t* __restrict__ req_begin,  // U+1 occurrence bounds
                   const uint8_t* __restrict__ dest, uint64_t n_rows, uint64_t dp_cut,
                   uint64_t flex_cut, uint32_t u, uint32_t w, uint32_t* __restrict__ seen,
                   uint64_t seen_words, unsigned long long* __restrict__ counters,
                   unsigned* __restrict__ bad_rows) {
  __shared__ unsigned s_cnt[TS_NUM_COUNTERS * kMaxGpus];
  __shared__ uint64_t s_bounds[kMaxGpus + 1];
  for (unsigned i = threadIdx.x; i < TS_NUM_COUNTERS * u; i += blockDim.x) s_cnt[i] = 0;
  for (unsigned i = threadIdx.x; i <= u; i += blockDim.x) s_bounds[i] = req_begin[i];
  __syncthreads();

  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // Uniform trip count per warp: every lane runs the same iterations so the
  // match/ballot intrinsics always see the full warp.
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x; base < occ;
       base += stride) {
    const uint64_t idx = base + threadIdx.x;
    bool valid = idx < occ;
    uint32_t g = 0, server = 0, kind = 0;  // kind: 0 RW, 1 Flex, 2 DP
    uint32_t r = 0;
    if (valid) {
      r = __ldg(rows + idx);
      if (r >= n_rows) {
        atomicAdd(bad_rows, 1u);
        valid = false;
      }
    }
    if (valid) {
      // requester: last g with bounds[g] <= idx (binary search, U <= 256)
      uint32_t lo = 0, hi = u;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_bounds[mid] <= idx) lo = mid; else hi = mid;
      }
      g = lo;
      if (r < dp_cut) {
        kind = 2;
        server = g;
      } else if (r < flex_cut) {
        kind = 1;
        server = (g / w) * w + __ldg(dest + r);
      } else {
        kind = 0;
        server = __ldg(dest + r);
      }
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
    // distinct (server, row): test first, then claim with an atomic OR
    bool first_touch = false;
    if (valid) {
      uint32_t* word = seen + static_cast<uint64_t>(server) * seen_words + (r >> 5);
      const uint32_t bit = 1u << (r & 31);
      if ((*reinterpret_cast<volatile uint32_t*>(word) & bit) == 0) {
        first_touch = (atomicOr(word, bit) & bit) == 0;
      }
    }
    warp_count(s_cnt, TS_CTR_DISTINCT * u + server, first_touch);
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < TS_NUM_COUNTERS * u; i += blockDim.x) {
    if (s_cnt[i]) atomicAdd(counters + i, static_cast<unsigned long long>(s_cnt[i]));
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
  uint64_t seen_words = 0;
  unsigned long long* d_counters = nullptr;
  unsigned* d_bad = nullptr;
  uint64_t* d_bounds = nullptr;
  uint32_t* d_rows = nullptr;
  uint64_t rows_capacity = 0;
  cudaStream_t stream = nullptr;

  uint32_t u() const { return num_nodes * gpus_per_node; }

  void run(const uint64_t* d_req_begin, const uint32_t* rows, uint64_t occ, uint64_t* counters) {
    using namespace tsd;
    const uint32_t U = u();
    TSD_CUDA(cudaMemsetAsync(d_counters, 0, sizeof(unsigned long long) * TS_NUM_COUNTERS * U, stream));
    TSD_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned), stream));
    TSD_CUDA(cudaMemsetAsync(d_seen, 0, sizeof(uint32_t) * seen_words * U, stream));
    if (occ > 0) {
      const unsigned blocks = static_cast<unsigned>(
          std::min<uint64_t>(ceil_div(occ, kRouterThreads), static_cast<uint64_t>(sm_count()) * 4));
      route_count_kernel<<<blocks, kRouterThreads, 0, stream>>>(
          rows, occ, d_req_begin, d_dest, n_rows, dp_cut, flex_cut, U, gpus_per_node, d_seen,
          seen_words, d_counters, d_bad);
      TSD_LAUNCH_CHECK();
    }
    unsigned bad = 0;
    TSD_CUDA(cudaMemcpyAsync(counters, d_counters, sizeof(uint64_t) * TS_NUM_COUNTERS * U,
                             cudaMemcpyDeviceToHost, stream));
    TSD_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost, stream));
    TSD_CUDA(cudaStreamSynchronize(stream));
    if (bad) fail(TS_ERR_VALIDATION, "router: batch references rows outside the plan");
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
    r->seen_words = (n_rows + 31) / 32;
    TSD_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    TSD_CUDA(dev_alloc(&r->d_dest, n_rows));
    TSD_CUDA(dev_alloc(&r->d_seen, sizeof(uint32_t) * r->seen_words * u));
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
    if (r->stream) cudaStreamDestroy(r->stream);
    delete r;
  });
}

}  // extern "C"
