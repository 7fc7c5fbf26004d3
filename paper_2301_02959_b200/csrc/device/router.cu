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
#include <cstdlib>
#include <string>
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

// Bit of (server, r) in the compact distinct bitmap.
__device__ __forceinline__ uint64_t seen_bit(const RouteParams& p, uint32_t r, uint32_t kind, uint32_t g) {
  if (kind == 0) return r - p.flex_cut;
  if (kind == 1) return p.flex_base + static_cast<uint64_t>(g / p.w) * (p.flex_cut - p.dp_cut) + (r - p.dp_cut);
  return p.dp_base + static_cast<uint64_t>(g) * p.dp_cut + r;
}

// Marks (server, r) as served this iteration (the reference's stamps,
// simulator.cpp:158-166): a fire-and-forget atomic OR -- the result is not
// read, so it compiles to a RED and costs the routing loop no round trip.
// The distinct counts come from one pass over the bitmap afterwards
// (distinct_count_kernel).
__device__ __forceinline__ void mark(const RouteParams& p, uint64_t bit) {
  atomicOr(p.seen + (bit >> 5), 1u << (bit & 31));
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
  // match intrinsics always see the full warp.
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
      // test first: a Zipf-hot row would otherwise pile REDs onto one word
      const uint64_t bit = seen_bit(p, r, kind, g);
      if ((*reinterpret_cast<volatile uint32_t*>(p.seen + (bit >> 5)) & (1u << (bit & 31))) == 0) mark(p, bit);
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

// U <= 8 (one NVSwitch node).  Each block takes a contiguous chunk of ONE
// requester's occurrences (grid = U x blocks_per_req), so:
//   * the requester-side counts are three registers per thread;
//   * a shared-memory bitmap over the hottest canonical rows (r < kFilterRows:
//     canonical order is probability order, so these carry most of a Zipf
//     batch) filters the distinct marks -- a hot row reaches the global
//     bitmap once per block instead of once per occurrence;
//   * server-side counts are per-thread arrays of 8 updated by predicated
//     adds; SERVED is not counted at all -- it equals SEND_GLOBAL +
//     SEND_INTRA + DP_LOCAL per GPU (a DP row is served by its requester)
//     and the host derives it.
// No warp intrinsics on the per-occurrence path; warp shuffles + shared
// atomics once per thread at the end.
constexpr int kU8Threads = 512;
constexpr uint32_t kFilterRows = 1u << 19;  // 64 KB of shared memory (dynamic)
__global__ void __launch_bounds__(kU8Threads, 2) route_count_u8_kernel(RouteParams p, uint32_t blocks_per_req) {
  extern __shared__ uint32_t s_filter[];  // kFilterRows bits
  __shared__ unsigned long long s_cnt[TS_NUM_COUNTERS * kSmallU];
  const uint32_t g = blockIdx.x / blocks_per_req, part = blockIdx.x % blocks_per_req;
  for (unsigned i = threadIdx.x; i < kFilterRows / 32; i += blockDim.x) s_filter[i] = 0;
  for (unsigned i = threadIdx.x; i < TS_NUM_COUNTERS * kSmallU; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const uint64_t lo = p.req_begin[g], hi = p.req_begin[g + 1];
  const uint64_t chunk = (hi - lo + blocks_per_req - 1) / blocks_per_req;
  const uint64_t begin = lo + part * chunk, end = min(hi, begin + chunk);
  const uint32_t node_base = (g / p.w) * p.w;
  const uint64_t flex_sec = p.flex_base + static_cast<uint64_t>(g / p.w) * (p.flex_cut - p.dp_cut) - p.dp_cut;
  const uint64_t dp_sec = p.dp_base + static_cast<uint64_t>(g) * p.dp_cut;

  uint32_t send_g[kSmallU] = {}, send_i[kSmallU] = {};
  uint32_t req[3] = {0, 0, 0};
  bool bad = false;
  // one occurrence whose placement byte d is loaded (or unused for DP)
  const auto route_one = [&](uint32_t r, uint32_t d) {
    if (r >= p.n_rows) {
      bad = true;
      return;
    }
    uint64_t bit;
    if (r < p.dp_cut) {
      req[2] += 1;
      bit = dp_sec + r;
    } else if (r < p.flex_cut) {
      req[1] += 1;
      add_at(send_i, node_base + d, 1u);
      bit = flex_sec + r;
    } else {
      req[0] += 1;
      add_at(send_g, d, 1u);
      bit = r - p.flex_cut;
    }
    bool first = true;
    if (r < kFilterRows) {
      const uint32_t m = 1u << (r & 31);
      first = (atomicOr(&s_filter[r >> 5], m) & m) == 0;
    }
    if (first) mark(p, bit);
  };
  const auto dest_of = [&](uint32_t r) -> uint32_t {
    return r >= p.dp_cut && r < p.n_rows ? __ldg(p.dest + r) : 0u;
  };
  // body: 16 B-aligned uint4 loads of 4 indices, two per thread per trip,
  // and the next trip's two issued before this trip's placement bytes --
  // the index stream stays in flight behind the dependent byte loads
  const uint64_t a0 = min(end, (begin + 3) & ~uint64_t{3});
  const uint64_t a1 = max(a0, end & ~uint64_t{3});
  const uint4* vec = reinterpret_cast<const uint4*>(p.rows + a0);
  const uint64_t nvec = (a1 - a0) / 4;
  const uint4 zero4 = make_uint4(0, 0, 0, 0);
  uint64_t j = threadIdx.x;
  uint4 va = j < nvec ? __ldg(vec + j) : zero4;
  uint4 vb = j + kU8Threads < nvec ? __ldg(vec + j + kU8Threads) : zero4;
  for (; j < nvec; j += 2 * kU8Threads) {
    const uint64_t jn = j + 2 * kU8Threads;
    const uint4 na = jn < nvec ? __ldg(vec + jn) : zero4;
    const uint4 nb = jn + kU8Threads < nvec ? __ldg(vec + jn + kU8Threads) : zero4;
    const bool has_b = j + kU8Threads < nvec;
    const uint32_t r[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
    uint32_t d[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k] = (k < 4 || has_b) ? dest_of(r[k]) : 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k < 4 || has_b) route_one(r[k], d[k]);
    }
    va = na;
    vb = nb;
  }
  // unaligned head [begin, a0) and tail [a1, end): at most 3 + 3 indices
  if (threadIdx.x < a0 - begin) {
    const uint32_t r = __ldg(p.rows + begin + threadIdx.x);
    route_one(r, dest_of(r));
  }
  if (threadIdx.x < end - a1) {
    const uint32_t r = __ldg(p.rows + a1 + threadIdx.x);
    route_one(r, dest_of(r));
  }
  if (bad) atomicAdd(p.bad_rows, 1u);
  atomicAdd(&s_cnt[TS_CTR_RECV_GLOBAL * kSmallU + g], static_cast<unsigned long long>(req[0]));
  atomicAdd(&s_cnt[TS_CTR_RECV_INTRA * kSmallU + g], static_cast<unsigned long long>(req[1]));
  atomicAdd(&s_cnt[TS_CTR_DP_LOCAL * kSmallU + g], static_cast<unsigned long long>(req[2]));
  const unsigned lane = threadIdx.x & 31u;
#pragma unroll
  for (int s = 0; s < kSmallU; ++s) {
    uint32_t a = send_g[s], b = send_i[s];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
      b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
    }
    if (lane == 0) {
      if (a) atomicAdd(&s_cnt[TS_CTR_SEND_GLOBAL * kSmallU + s], static_cast<unsigned long long>(a));
      if (b) atomicAdd(&s_cnt[TS_CTR_SEND_INTRA * kSmallU + s], static_cast<unsigned long long>(b));
    }
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < TS_NUM_COUNTERS * kSmallU; i += blockDim.x) {
    const unsigned ctr = i / kSmallU, gpu = i % kSmallU;
    if (gpu < p.u && s_cnt[i]) atomicAdd(p.counters + ctr * p.u + gpu, s_cnt[i]);
  }
}

// Distinct counts for U <= 8 (see distinct_count_kernel below): one thread
// per bitmap word, per-thread register counters, one reduction at the end.
__global__ void __launch_bounds__(256) distinct_count_u8_kernel(RouteParams p, uint64_t words) {
  __shared__ unsigned long long s_cnt[kSmallU];
  if (threadIdx.x < kSmallU) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  uint32_t cnt[kSmallU] = {};
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t flex_rows = p.flex_cut - p.dp_cut;
  const uint64_t total_bits = p.dp_base + static_cast<uint64_t>(p.u) * p.dp_cut;
  for (uint64_t wi = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; wi < words; wi += stride) {
    uint32_t m = p.seen[wi];
    const uint64_t b0 = wi * 32;
    if (b0 + 32 > total_bits) m &= b0 >= total_bits ? 0u : (1u << (total_bits - b0)) - 1u;
    while (m) {
      const uint64_t bit = b0 + (__ffs(m) - 1);
      if (bit >= p.dp_base) {  // DP: every set bit up to the section end is one requester's
        const uint64_t g = (bit - p.dp_base) / p.dp_cut;
        const uint64_t end = p.dp_base + (g + 1) * p.dp_cut;
        uint32_t same = m;
        if (end < b0 + 32) same &= (1u << (end - b0)) - 1u;
        add_at(cnt, static_cast<uint32_t>(g), __popc(same));
        m &= ~same;
        continue;
      }
      uint32_t server;
      if (bit >= p.flex_base) {
        const uint64_t rel = bit - p.flex_base;
        server = static_cast<uint32_t>((rel / flex_rows) * p.w) + __ldg(p.dest + p.dp_cut + rel % flex_rows);
      } else {
        server = __ldg(p.dest + p.flex_cut + bit);
      }
      add_at(cnt, server, 1u);
      m &= m - 1;
    }
  }
  const unsigned lane = threadIdx.x & 31u;
#pragma unroll
  for (int s = 0; s < kSmallU; ++s) {
    uint32_t a = cnt[s];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
    if (lane == 0 && a) atomicAdd(&s_cnt[s], static_cast<unsigned long long>(a));
  }
  __syncthreads();
  if (threadIdx.x < p.u && s_cnt[threadIdx.x]) {
    atomicAdd(p.counters + TS_CTR_DISTINCT * p.u + threadIdx.x, s_cnt[threadIdx.x]);
  }
}

// Distinct (server, row) pairs per server from the marked bitmap: the RW
// section is one bit per RW row (server = its owner byte), the Flex section
// one bit per (node, Flex row) (server = node*W + slot byte), the DP section
// one bit per (requester, DP row) (server = requester).  One thread per
// 32-bit word: popcount when the word has one server, else per set bit.
__global__ void __launch_bounds__(256) distinct_count_kernel(RouteParams p, uint64_t words) {
  __shared__ unsigned s_cnt[kMaxGpus];
  for (unsigned i = threadIdx.x; i < p.u; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t flex_rows = p.flex_cut - p.dp_cut;
  const uint64_t total_bits = p.dp_base + static_cast<uint64_t>(p.u) * p.dp_cut;
  for (uint64_t wi = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; wi < words; wi += stride) {
    uint32_t m = p.seen[wi];
    while (m) {
      const int b = __ffs(m) - 1;
      const uint64_t bit = wi * 32 + b;
      if (bit >= total_bits) break;
      if (bit >= p.dp_base) {  // DP: the rest of the word up to the section end is one requester
        const uint64_t g = (bit - p.dp_base) / p.dp_cut;
        const uint64_t end = p.dp_base + (g + 1) * p.dp_cut;  // first bit of the next requester
        uint32_t same = m;
        if (end < wi * 32 + 32) same &= (1u << (end - wi * 32)) - 1u;
        atomicAdd(&s_cnt[g], __popc(same));
        m &= ~same;
        continue;
      }
      uint32_t server;
      if (bit >= p.flex_base) {
        const uint64_t rel = bit - p.flex_base;
        const uint64_t node = rel / flex_rows;
        server = static_cast<uint32_t>(node * p.w) + p.dest[p.dp_cut + rel % flex_rows];
      } else {
        server = p.dest[p.flex_cut + bit];
      }
      atomicAdd(&s_cnt[server], 1u);
      m &= m - 1;
    }
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < p.u; i += blockDim.x) {
    if (s_cnt[i]) atomicAdd(p.counters + TS_CTR_DISTINCT * p.u + i, static_cast<unsigned long long>(s_cnt[i]));
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
    // TIERSHARD_ROUTER=general forces the warp-aggregated kernel (A/B)
    static const bool force_general = [] {
      const char* e = std::getenv("TIERSHARD_ROUTER");
      return e && std::string(e) == "general";
    }();
    const bool small = U <= kSmallU && !force_general;
    if (occ > 0) {
      RouteParams p{rows, occ, d_req_begin, d_dest, n_rows, dp_cut, flex_cut, U, gpus_per_node,
                    d_seen, flex_base, dp_base, d_counters, d_bad};
      const unsigned blocks = static_cast<unsigned>(
          std::min<uint64_t>(ceil_div(occ, kRouterThreads), static_cast<uint64_t>(sm_count()) * 4));
      if (small) {
        // U x blocks_per_req blocks, each a contiguous chunk of one requester
        constexpr size_t kFilterBytes = kFilterRows / 8;
        static const bool attr_set = [] {
          TSD_CUDA(cudaFuncSetAttribute(route_count_u8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kFilterBytes)));
          return true;
        }();
        (void)attr_set;
        int per_sm = 0;
        TSD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, route_count_u8_kernel, kU8Threads,
                                                               kFilterBytes));
        const uint32_t bpr = static_cast<uint32_t>(std::max<uint64_t>(
            1, std::min<uint64_t>(ceil_div(occ, uint64_t{U} * kU8Threads * 16),
                                  ceil_div(static_cast<uint64_t>(sm_count()) * std::max(per_sm, 1), U))));
        const unsigned grid = U * bpr;
        route_count_u8_kernel<<<grid, kU8Threads, kFilterBytes, stream>>>(p, bpr);
      } else {
        route_count_kernel<<<blocks, kRouterThreads, 0, stream>>>(p);
      }
      TSD_LAUNCH_CHECK();
      const unsigned dgrid = static_cast<unsigned>(
          std::min<uint64_t>(ceil_div(seen_words, 256), static_cast<uint64_t>(sm_count()) * 8));
      if (small) {
        distinct_count_u8_kernel<<<dgrid, 256, 0, stream>>>(p, seen_words);
      } else {
        distinct_count_kernel<<<dgrid, 256, 0, stream>>>(p, seen_words);
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
