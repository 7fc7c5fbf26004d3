// Value-path kernels (embedding.cuh): unpooled gather, deterministic
// segment-reduce with fused row-wise SGD / Adagrad, dense replica updates.
//
// Lane layout used everywhere a warp owns one embedding row: lane l holds the
// VEC = dim/32 contiguous floats [l*VEC, (l+1)*VEC) — 128-bit accesses for
// dim >= 128, 64-bit for dim = 64.  The Adagrad sum of squares is the
// per-lane fma chain followed by the xor butterfly, exactly the order
// oracle/restate.c replays, so single-GPU results are bit-identical.
// Every floating-point op in the update is an explicit _rn intrinsic: no
// contraction or fast-math can change a bit.
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "embedding.cuh"
#include "primitives.cuh"

namespace tsd {
namespace {

constexpr int kThreads = 256;

template <int VEC>
__device__ __forceinline__ void load_lane(const float* p, float (&r)[VEC]) {
  if constexpr (VEC % 4 == 0) {
#pragma unroll
    for (int j = 0; j < VEC / 4; ++j) {
      const float4 t = *reinterpret_cast<const float4*>(p + 4 * j);
      r[4 * j] = t.x;
      r[4 * j + 1] = t.y;
      r[4 * j + 2] = t.z;
      r[4 * j + 3] = t.w;
    }
  } else if constexpr (VEC == 2) {
    const float2 t = *reinterpret_cast<const float2*>(p);
    r[0] = t.x;
    r[1] = t.y;
  } else {
    r[0] = *p;
  }
}

template <int VEC>
__device__ __forceinline__ void load_lane_ro(const float* p, float (&r)[VEC]) {
  if constexpr (VEC % 4 == 0) {
#pragma unroll
    for (int j = 0; j < VEC / 4; ++j) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(p + 4 * j));
      r[4 * j] = t.x;
      r[4 * j + 1] = t.y;
      r[4 * j + 2] = t.z;
      r[4 * j + 3] = t.w;
    }
  } else if constexpr (VEC == 2) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(p));
    r[0] = t.x;
    r[1] = t.y;
  } else {
    r[0] = __ldg(p);
  }
}

template <int VEC>
__device__ __forceinline__ void store_lane(float* p, const float (&r)[VEC]) {
  if constexpr (VEC % 4 == 0) {
#pragma unroll
    for (int j = 0; j < VEC / 4; ++j) {
      *reinterpret_cast<float4*>(p + 4 * j) =
          make_float4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
    }
  } else if constexpr (VEC == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(r[0], r[1]);
  } else {
    *p = r[0];
  }
}

// Streaming (evict-first) store of one lane's slice: the unpooled output is
// written once and not re-read before it has left L2 anyway, so it should
// not evict the Zipf-hot weight rows.
template <int VEC>
__device__ __forceinline__ void store_lane_stream(float* p, const float (&r)[VEC]) {
  if constexpr (VEC % 4 == 0) {
#pragma unroll
    for (int j = 0; j < VEC / 4; ++j) {
      stg_stream(reinterpret_cast<float4*>(p + 4 * j),
                 make_float4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]));
    }
  } else {
    store_lane<VEC>(p, r);
  }
}

// Canonical row -> local shard row of THIS rank, false if served remotely.
__device__ __forceinline__ bool resolve_local(const RemapView& rv, uint32_t c, uint32_t* lid) {
  if (rv.identity || c < rv.dp_cut) {
    *lid = c;
    return true;
  }
  const uint32_t d = __ldg(rv.dest + c);
  const bool mine = c < rv.flex_cut ? d == rv.slot : d == rv.rank;
  if (mine) *lid = __ldg(rv.local + c);
  return mine;
}

template <int DIM, int UNROLL>
__global__ void __launch_bounds__(kThreads)
gather_local_kernel(const uint32_t* __restrict__ rows, uint64_t occ,
                    const float* __restrict__ weights, float* __restrict__ out, RemapView rv,
                    double* __restrict__ loss_partials) {
  constexpr int VEC = DIM / 32;
  __shared__ float s_sq[kThreads / 32];
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  float sq = 0.0f;
  for (uint64_t base = gwarp * UNROLL; base < occ; base += nwarps * UNROLL) {
    uint32_t my_lid = 0;
    bool my_ok = false;
    if (lane < UNROLL && base + lane < occ) my_ok = resolve_local(rv, __ldg(rows + base + lane), &my_lid);
    float r[UNROLL][VEC];
    bool ok[UNROLL];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const uint32_t lid = __shfl_sync(0xFFFFFFFFu, my_lid, k);
      ok[k] = __shfl_sync(0xFFFFFFFFu, my_ok, k);
      if (ok[k]) load_lane_ro<VEC>(weights + static_cast<uint64_t>(lid) * DIM + lane * VEC, r[k]);
    }
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      if (ok[k]) {
        store_lane_stream<VEC>(out + (base + k) * DIM + lane * VEC, r[k]);
#pragma unroll
        for (int j = 0; j < VEC; ++j) sq = __fmaf_rn(r[k][j], r[k][j], sq);
      }
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, m);
  if (lane == 0) s_sq[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) acc += static_cast<double>(s_sq[w]);
    loss_partials[blockIdx.x] = acc;
  }
}

// ---------------------------------------------------------------------------
// Bulk-copy gather (TIERSHARD_GATHER=bulk): the same contract as
// gather_local_kernel, with the rows moved by the copy engine instead of
// registers.  Each warp owns a ring of kBulkStages shared-memory stages of
// 4 KB; one elected lane issues cp.async.bulk global->shared loads of a
// stage's rows (one 16-B-aligned row each), completing on the stage's
// mbarrier, then ONE cp.async.bulk shared->global store of the stage when
// its rows are consecutive in `out` (always at U = 1), else one per row.
// The lanes only read the stage once for the loss partial.  Loads of
// kBulkStages - 1 stages stay in flight behind each store.
// ---------------------------------------------------------------------------

constexpr int kBulkThreads = 128;
constexpr int kBulkMaxStages = 8;
constexpr uint32_t kBulkStageBytes = 4096;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int DIM>
__global__ void __launch_bounds__(kBulkThreads)
gather_bulk_kernel(const uint32_t* __restrict__ rows, uint64_t occ, const float* __restrict__ weights,
                   float* __restrict__ out, RemapView rv, double* __restrict__ loss_partials, int kBulkStages) {
  constexpr uint32_t kRowBytes = DIM * 4;
  constexpr int R = kBulkStageBytes / kRowBytes;  // rows per stage (<= 32)
  static_assert(R >= 1 && R <= 32, "stage holds 1..32 rows");
  constexpr int kWarps = kBulkThreads / 32;
  extern __shared__ __align__(128) uint8_t bulk_smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(bulk_smem);  // [kWarps][kBulkMaxStages]
  uint8_t* stages = bulk_smem + 8 * kWarps * kBulkMaxStages;  // [kWarps][kBulkStages][4 KB]
  __shared__ float s_sq[kWarps];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint64_t* my_bars = bars + warp * kBulkMaxStages;
  uint8_t* my_stages = stages + static_cast<size_t>(warp) * kBulkStages * kBulkStageBytes;
  if (lane == 0) {
    for (int st = 0; st < kBulkStages; ++st) mbar_init(my_bars + st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  const uint64_t gwarp = static_cast<uint64_t>(blockIdx.x) * kWarps + warp;
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kWarps;
  const uint64_t groups = (occ + R - 1) / R;
  // group j of this warp = global group gwarp + j * nwarps
  uint32_t ok_mask[kBulkMaxStages];  // valid local rows of the group in each stage (lane 0)
  const auto issue = [&](uint64_t j, int st) {
    const uint64_t gi = gwarp + j * nwarps;
    uint32_t lid = 0;
    bool ok = false;
    const uint64_t i = gi * R + lane;
    if (gi < groups && lane < static_cast<unsigned>(R) && i < occ) ok = resolve_local(rv, __ldg(rows + i), &lid);
    const uint32_t mask = __ballot_sync(0xFFFFFFFFu, ok);
    if (lane == 0) {
      ok_mask[st] = mask;
      mbar_expect_tx(my_bars + st, __popc(mask) * kRowBytes);
    }
    __syncwarp();
    // each valid lane issues its own row's copy (lanes >= R never valid)
    if (ok) {
      bulk_load(my_stages + st * kBulkStageBytes + lane * kRowBytes, weights + static_cast<uint64_t>(lid) * DIM,
                kRowBytes, my_bars + st);
    }
  };
  const uint64_t my_groups = gwarp < groups ? (groups - gwarp + nwarps - 1) / nwarps : 0;
  for (int st = 0; st < kBulkStages - 1; ++st) {
    if (static_cast<uint64_t>(st) < my_groups) issue(st, st);
  }
  float sq = 0.0f;
  uint32_t phase = 0;  // parity bits, one per stage
  for (uint64_t j = 0; j < my_groups; ++j) {
    const int st = static_cast<int>(j % kBulkStages);
    mbar_wait(my_bars + st, (phase >> st) & 1u);
    phase ^= 1u << st;
    const uint32_t mask = __shfl_sync(0xFFFFFFFFu, ok_mask[st], 0);
    // loss partial: lanes read the stage (rows k with mask bit k)
    const float4* sp = reinterpret_cast<const float4*>(my_stages + st * kBulkStageBytes);
#pragma unroll
    for (int q = 0; q < static_cast<int>(kBulkStageBytes / 16 / 32); ++q) {
      const int f4 = q * 32 + static_cast<int>(lane);
      const int row = f4 * 16 / static_cast<int>(kRowBytes);
      if ((mask >> row) & 1u) {
        const float4 v = sp[f4];
        sq = __fmaf_rn(v.x, v.x, sq);
        sq = __fmaf_rn(v.y, v.y, sq);
        sq = __fmaf_rn(v.z, v.z, sq);
        sq = __fmaf_rn(v.w, v.w, sq);
      }
    }
    const uint64_t gi = gwarp + j * nwarps;
    const uint64_t row0 = gi * R;
    if (lane == 0) {
      const uint64_t left = occ - row0;
      const uint32_t nrows = left < static_cast<uint64_t>(R) ? static_cast<uint32_t>(left) : static_cast<uint32_t>(R);
      const uint32_t full = nrows >= 32 ? 0xFFFFFFFFu : ((1u << nrows) - 1u);
      if (mask == full) {  // consecutive rows of out: one store for the stage
        bulk_store(out + row0 * DIM, my_stages + st * kBulkStageBytes, nrows * kRowBytes);
      } else {
        for (uint32_t m = mask; m; m &= m - 1) {
          const int k = __ffs(m) - 1;
          bulk_store(out + (row0 + k) * DIM, my_stages + st * kBulkStageBytes + k * kRowBytes, kRowBytes);
        }
      }
      bulk_commit();
      // the previous stage's store has read its shared memory: refill it
      bulk_wait_read<1>();
    }
    __syncwarp();
    const uint64_t jn = j + kBulkStages - 1;
    if (jn < my_groups) issue(jn, static_cast<int>(jn % kBulkStages));
  }
  if (lane == 0) bulk_wait_all();
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, m);
  if (lane == 0) s_sq[warp] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) acc += static_cast<double>(s_sq[w]);
    loss_partials[blockIdx.x] = acc;
  }
}

// Requester-pull gather (launch_gather_all): like gather_local_kernel, but
// an occurrence served by a peer is loaded from that peer's shard over
// NVLink instead of being skipped.
template <int DIM, int UNROLL>
__global__ void __launch_bounds__(kThreads)
gather_all_kernel(const uint32_t* __restrict__ rows, uint64_t occ, PeerWeights pw, float* __restrict__ out,
                  RemapView rv, double* __restrict__ loss_partials) {
  constexpr int VEC = DIM / 32;
  __shared__ float s_sq[kThreads / 32];
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  float sq = 0.0f;
  for (uint64_t base = gwarp * UNROLL; base < occ; base += nwarps * UNROLL) {
    uint32_t my_lid = 0, my_server = rv.rank;
    if (lane < UNROLL && base + lane < occ) {
      const uint32_t c = __ldg(rows + base + lane);
      if (c < rv.dp_cut) {
        my_lid = c;
      } else {
        const uint32_t d = __ldg(rv.dest + c);
        my_server = c < rv.flex_cut ? pw.node_base + d : d;
        my_lid = __ldg(rv.local + c);
      }
    }
    float r[UNROLL][VEC];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const uint32_t lid = __shfl_sync(0xFFFFFFFFu, my_lid, k);
      const uint32_t srv = __shfl_sync(0xFFFFFFFFu, my_server, k);
      if (base + k < occ) load_lane_ro<VEC>(pw.w[srv] + static_cast<uint64_t>(lid) * DIM + lane * VEC, r[k]);
    }
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      if (base + k < occ) {
        store_lane_stream<VEC>(out + (base + k) * DIM + lane * VEC, r[k]);
#pragma unroll
        for (int j = 0; j < VEC; ++j) sq = __fmaf_rn(r[k][j], r[k][j], sq);
      }
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, m);
  if (lane == 0) s_sq[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) acc += static_cast<double>(s_sq[w]);
    loss_partials[blockIdx.x] = acc;
  }
}

template <int DIM, int UNROLL>
__global__ void __launch_bounds__(kThreads)
pull_rows_kernel(const uint32_t* __restrict__ sorted_bucket, const uint32_t* __restrict__ order,
                 const uint32_t* __restrict__ ids, const uint32_t* __restrict__ d_count, uint64_t max_count,
                 PeerWeights pw, uint32_t u, float* __restrict__ out, double* __restrict__ loss_partials) {
  constexpr int VEC = DIM / 32;
  __shared__ float s_sq[kThreads / 32];
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t count = min(static_cast<uint64_t>(*d_count), max_count);
  const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  float sq = 0.0f;
  for (uint64_t base = gwarp * UNROLL; base < count; base += nwarps * UNROLL) {
    uint32_t my_srv = 0, my_lid = 0, my_pos = 0;
    if (lane < UNROLL && base + lane < count) {
      const uint64_t j = base + lane;
      const uint32_t b = __ldg(sorted_bucket + j);
      my_srv = b < u ? b : pw.node_base + (b - u);
      my_lid = __ldg(ids + j);
      my_pos = __ldg(order + j);
    }
    float r[UNROLL][VEC];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const uint32_t srv = __shfl_sync(0xFFFFFFFFu, my_srv, k);
      const uint32_t lid = __shfl_sync(0xFFFFFFFFu, my_lid, k);
      if (base + k < count) load_lane_ro<VEC>(pw.w[srv] + static_cast<uint64_t>(lid) * DIM + lane * VEC, r[k]);
    }
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const uint32_t pos = __shfl_sync(0xFFFFFFFFu, my_pos, k);
      if (base + k < count) {
        store_lane_stream<VEC>(out + static_cast<uint64_t>(pos) * DIM + lane * VEC, r[k]);
#pragma unroll
        for (int j = 0; j < VEC; ++j) sq = __fmaf_rn(r[k][j], r[k][j], sq);
      }
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, m);
  if (lane == 0) s_sq[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) acc += static_cast<double>(s_sq[w]);
    loss_partials[blockIdx.x] = acc;
  }
}

// Fixed-shape tree over the partials (thread t sums t, t+1024, ... in order,
// then a fixed shared-memory tree): deterministic for a fixed grid.
__global__ void __launch_bounds__(1024)
loss_finalize_kernel(const double* __restrict__ partials, unsigned count, double* __restrict__ loss,
                     double* __restrict__ mirror) {
  __shared__ double s[1024];
  double acc = 0.0;
  for (unsigned i = threadIdx.x; i < count; i += 1024) acc += partials[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (unsigned half = 512; half > 0; half >>= 1) {
    if (threadIdx.x < half) s[threadIdx.x] += s[threadIdx.x + half];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *loss = 0.5 * s[0];
    if (mirror) *mirror = 0.5 * s[0];
  }
}

// ---------------------------------------------------------------------------
// segment reduction + optimizer
// ---------------------------------------------------------------------------

template <int VEC>
__device__ __forceinline__ const float* grad_row(const GradSource& gs, uint32_t v, uint32_t dim) {
  if (v < gs.n_local) return gs.local + static_cast<uint64_t>(v) * dim;
  return gs.remote + static_cast<uint64_t>(v - gs.n_local) * dim;
}

// Where a dense-range row's reduced gradient goes (and its stamp, or null).
template <int DIM>
__device__ __forceinline__ float* dense_row(const DenseRange& d, uint32_t row, uint32_t** stamp) {
  const uint32_t r = row - d.lo;
  if (d.push_n) {
    const uint32_t o = d.interleave ? r % d.push_n : r / d.per;
    const uint32_t i = d.interleave ? r / d.push_n : r - o * d.per;
    const uint64_t slot = static_cast<uint64_t>(d.me) * d.per + i;
    *stamp = d.push_stamp[o] + slot;
    return d.push_grad[o] + slot * DIM;
  }
  *stamp = d.stamp ? d.stamp + r : nullptr;
  return d.grad + static_cast<uint64_t>(r) * DIM;
}

// Finishes one reduced row: dense-range rows park their gradient, others get
// the optimizer step.  All 32 lanes must call (Adagrad uses shuffles).
template <int DIM>
__device__ __forceinline__ void finish_row(uint32_t row, const float (&g)[DIM / 32],
                                           float* __restrict__ weights, float* __restrict__ state,
                                           const OptParams& opt, const DenseRange& d0,
                                           const DenseRange& d1) {
  constexpr int VEC = DIM / 32;
  const unsigned lane = threadIdx.x & 31u;
  if ((row >= d0.lo && row < d0.hi) || (row >= d1.lo && row < d1.hi)) {
    const DenseRange& d = row < d0.hi && row >= d0.lo ? d0 : d1;
    uint32_t* st = nullptr;
    store_lane<VEC>(dense_row<DIM>(d, row, &st) + lane * VEC, g);
    if (st && lane == 0) *st = d.epoch;
    return;
  }
  float* wp = weights + static_cast<uint64_t>(row) * DIM + lane * VEC;
  float w[VEC];
  load_lane<VEC>(wp, w);
  if (opt.optimizer == TS_OPT_SGD) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) w[j] = __fmaf_rn(-opt.lr, g[j], w[j]);
  } else {
    float q = 0.0f;
#pragma unroll
    for (int j = 0; j < VEC; ++j) q = __fmaf_rn(g[j], g[j], q);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) q = __fadd_rn(q, __shfl_xor_sync(0xFFFFFFFFu, q, m));
    const float G = __fadd_rn(state[row], __fdiv_rn(q, static_cast<float>(DIM)));
    __syncwarp();
    if (lane == 0) state[row] = G;
    const float denom = __fadd_rn(__fsqrt_rn(G), opt.eps);
#pragma unroll
    for (int j = 0; j < VEC; ++j) w[j] = __fmaf_rn(-opt.lr, __fdiv_rn(g[j], denom), w[j]);
  }
  store_lane<VEC>(wp, w);
}

// acc = sum of grad rows vals[s..e) left to right (acc starts from entry s).
template <int DIM>
__device__ __forceinline__ void sum_entries(const uint32_t* __restrict__ vals, uint32_t s,
                                            uint32_t e, const GradSource& gs,
                                            float (&acc)[DIM / 32]) {
  constexpr int VEC = DIM / 32;
  constexpr int B = DIM <= 128 ? 8 : 4;  // rows in flight per warp
  const unsigned lane = threadIdx.x & 31u;
  load_lane<VEC>(grad_row<VEC>(gs, __ldg(vals + s), DIM) + lane * VEC, acc);
  uint32_t k = s + 1;
  for (; k + B <= e; k += B) {
    const uint32_t my_v = lane < B ? __ldg(vals + k + lane) : 0u;
    float r[B][VEC];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const uint32_t v = __shfl_sync(0xFFFFFFFFu, my_v, b);
      load_lane<VEC>(grad_row<VEC>(gs, v, DIM) + lane * VEC, r[b]);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) acc[j] = __fadd_rn(acc[j], r[b][j]);
    }
  }
  for (; k < e; ++k) {
    float r[VEC];
    load_lane<VEC>(grad_row<VEC>(gs, __ldg(vals + k), DIM) + lane * VEC, r);
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = __fadd_rn(acc[j], r[j]);
  }
}

// ---------------------------------------------------------------------------
// Short segments, several per warp.  A group of G lanes owns one segment; lane
// l of the group holds the PER = DIM/G contiguous floats [l*PER, (l+1)*PER),
// i.e. the K = 32/G "virtual lanes" l*K .. l*K+K-1 of the oracle's 32-lane
// layout (V = DIM/32 floats each).  The Adagrad sum of squares is formed per
// virtual lane and combined by the same xor butterfly (levels 16..1 over the
// virtual index: cross-lane shuffles for m >= K, in-register for m < K), so
// the result is bit-identical to restate.c.
// ---------------------------------------------------------------------------

template <int DIM>
struct Grouping {
  static constexpr int G = DIM <= 128 ? 8 : (DIM == 256 ? 16 : 32);  // lanes per segment
  static constexpr int PER = DIM / G;                                 // floats per lane
  static constexpr int K = 32 / G;                                    // virtual lanes per lane
  static constexpr int V = DIM / 32;                                  // floats per virtual lane
  static constexpr int E = PER <= 8 ? 4 : (PER <= 16 ? 2 : 1);        // entries in flight
};

template <int PER>
__device__ __forceinline__ void load_vec(const float* p, float (&r)[PER]) {
  static_assert(PER % 4 == 0, "group lanes hold whole float4s");
#pragma unroll
  for (int j = 0; j < PER / 4; ++j) {
    const float4 t = *reinterpret_cast<const float4*>(p + 4 * j);
    r[4 * j] = t.x;
    r[4 * j + 1] = t.y;
    r[4 * j + 2] = t.z;
    r[4 * j + 3] = t.w;
  }
}

template <int PER>
__device__ __forceinline__ void store_vec(float* p, const float (&r)[PER]) {
#pragma unroll
  for (int j = 0; j < PER / 4; ++j) {
    *reinterpret_cast<float4*>(p + 4 * j) = make_float4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
  }
}

template <int DIM>
__device__ __forceinline__ void group_finish_row(uint32_t row, const float (&g)[Grouping<DIM>::PER],
                                                 unsigned gl, unsigned gmask,
                                                 float* __restrict__ weights,
                                                 float* __restrict__ state, const OptParams& opt,
                                                 const DenseRange& d0, const DenseRange& d1) {
  using Gp = Grouping<DIM>;
  constexpr int PER = Gp::PER, K = Gp::K, V = Gp::V;
  const uint64_t col = static_cast<uint64_t>(gl) * PER;
  if ((row >= d0.lo && row < d0.hi) || (row >= d1.lo && row < d1.hi)) {
    const DenseRange& d = row < d0.hi && row >= d0.lo ? d0 : d1;
    uint32_t* st = nullptr;
    store_vec<PER>(dense_row<DIM>(d, row, &st) + col, g);
    if (st && gl == 0) *st = d.epoch;
    return;
  }
  float* wp = weights + static_cast<uint64_t>(row) * DIM + col;
  float w[PER];
  load_vec<PER>(wp, w);
  if (opt.optimizer == TS_OPT_SGD) {
#pragma unroll
    for (int j = 0; j < PER; ++j) w[j] = __fmaf_rn(-opt.lr, g[j], w[j]);
  } else {
    float q[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float acc = 0.0f;
#pragma unroll
      for (int j = 0; j < V; ++j) acc = __fmaf_rn(g[k * V + j], g[k * V + j], acc);
      q[k] = acc;
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      if (m >= K) {
#pragma unroll
        for (int k = 0; k < K; ++k) q[k] = __fadd_rn(q[k], __shfl_xor_sync(gmask, q[k], m / K));
      } else {
        float nq[K];
#pragma unroll
        for (int k = 0; k < K; ++k) nq[k] = __fadd_rn(q[k], q[k ^ m]);
#pragma unroll
        for (int k = 0; k < K; ++k) q[k] = nq[k];
      }
    }
    const float G = __fadd_rn(state[row], __fdiv_rn(q[0], static_cast<float>(DIM)));
    __syncwarp(gmask);
    if (gl == 0) state[row] = G;
    const float denom = __fadd_rn(__fsqrt_rn(G), opt.eps);
#pragma unroll
    for (int j = 0; j < PER; ++j) w[j] = __fmaf_rn(-opt.lr, __fdiv_rn(g[j], denom), w[j]);
  }
  store_vec<PER>(wp, w);
}

// ---------------------------------------------------------------------------
// Short segments, two interleaved per lane group.  A group of G lanes owns
// segment pairs (j, j + ngroups); both pairs' metadata, first two gradient
// rows, weight rows and Adagrad state are issued before any is consumed, so a
// pair costs ~3 dependent memory round trips instead of ~4 per segment.  Per
// segment the fp32 summation order is unchanged (entries left to right).
// ---------------------------------------------------------------------------

template <int DIM, int G>
struct Grp {
  static constexpr int PER = DIM / G;  // floats per lane
  static constexpr int K = 32 / G;     // oracle virtual lanes per lane
  static constexpr int V = DIM / 32;   // floats per virtual lane
};

// Optimizer step on one row whose weights / state are already in registers.
template <int DIM, int G>
__device__ __forceinline__ void group_apply(uint32_t row, const float (&g)[Grp<DIM, G>::PER],
                                            float (&w)[Grp<DIM, G>::PER], float st, unsigned gl,
                                            unsigned gmask, float* __restrict__ weights,
                                            float* __restrict__ state, const OptParams& opt) {
  constexpr int PER = Grp<DIM, G>::PER, K = Grp<DIM, G>::K, V = Grp<DIM, G>::V;
  if (opt.optimizer == TS_OPT_SGD) {
#pragma unroll
    for (int j = 0; j < PER; ++j) w[j] = __fmaf_rn(-opt.lr, g[j], w[j]);
  } else {
    float q[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float acc = 0.0f;
#pragma unroll
      for (int j = 0; j < V; ++j) acc = __fmaf_rn(g[k * V + j], g[k * V + j], acc);
      q[k] = acc;
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      if (m >= K) {
#pragma unroll
        for (int k = 0; k < K; ++k) q[k] = __fadd_rn(q[k], __shfl_xor_sync(gmask, q[k], m / K));
      } else {
        float nq[K];
#pragma unroll
        for (int k = 0; k < K; ++k) nq[k] = __fadd_rn(q[k], q[k ^ m]);
#pragma unroll
        for (int k = 0; k < K; ++k) q[k] = nq[k];
      }
    }
    const float Gs = __fadd_rn(st, __fdiv_rn(q[0], static_cast<float>(DIM)));
    if (gl == 0) state[row] = Gs;
    const float denom = __fadd_rn(__fsqrt_rn(Gs), opt.eps);
#pragma unroll
    for (int j = 0; j < PER; ++j) w[j] = __fmaf_rn(-opt.lr, __fdiv_rn(g[j], denom), w[j]);
  }
  store_vec<PER>(weights + static_cast<uint64_t>(row) * DIM + static_cast<uint64_t>(gl) * PER, w);
}

__device__ __forceinline__ bool in_dense(uint32_t row, const DenseRange& d0, const DenseRange& d1) {
  return (row >= d0.lo && row < d0.hi) || (row >= d1.lo && row < d1.hi);
}

template <int DIM, int G>
__device__ __forceinline__ void dense_store(uint32_t row, const float (&g)[Grp<DIM, G>::PER], unsigned gl,
                                            const DenseRange& d0, const DenseRange& d1) {
  constexpr int PER = Grp<DIM, G>::PER;
  const DenseRange& d = (row >= d0.lo && row < d0.hi) ? d0 : d1;
  uint32_t* st = nullptr;
  store_vec<PER>(dense_row<DIM>(d, row, &st) + static_cast<uint64_t>(gl) * PER, g);
  if (st && gl == 0) *st = d.epoch;
}

// acc += rows vals[k..e) (left to right), two rows in flight.
template <int DIM, int G>
__device__ __forceinline__ void sum_tail(const uint32_t* __restrict__ vals, uint32_t k, uint32_t e,
                                         const GradSource& gs, uint64_t col,
                                         float (&acc)[Grp<DIM, G>::PER]) {
  constexpr int PER = Grp<DIM, G>::PER;
  for (; k + 2 <= e; k += 2) {
    float r0[PER], r1[PER];
    load_vec<PER>(grad_row<1>(gs, __ldg(vals + k), DIM) + col, r0);
    load_vec<PER>(grad_row<1>(gs, __ldg(vals + k + 1), DIM) + col, r1);
#pragma unroll
    for (int q = 0; q < PER; ++q) acc[q] = __fadd_rn(__fadd_rn(acc[q], r0[q]), r1[q]);
  }
  if (k < e) {
    float r0[PER];
    load_vec<PER>(grad_row<1>(gs, __ldg(vals + k), DIM) + col, r0);
#pragma unroll
    for (int q = 0; q < PER; ++q) acc[q] = __fadd_rn(acc[q], r0[q]);
  }
}

template <int DIM, int G>
__global__ void __launch_bounds__(kThreads)
seg_pair_kernel(const uint32_t* __restrict__ vals, const uint32_t* __restrict__ starts,
                const uint32_t* __restrict__ seg_keys, const uint32_t* __restrict__ d_lo,
                const uint32_t* __restrict__ d_hi, GradSource gs, float* __restrict__ weights,
                float* __restrict__ state, OptParams opt, DenseRange d0, DenseRange d1,
                uint32_t* __restrict__ long_list, uint32_t* __restrict__ long_count, uint32_t short_max) {
  constexpr int PER = Grp<DIM, G>::PER;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned group = lane / G, gl = lane % G;
  const unsigned gmask = G == 32 ? 0xFFFFFFFFu : (((1u << G) - 1u) << (group * G));
  const uint32_t seg_lo = *d_lo, seg_hi = *d_hi;
  const uint32_t gid = ((blockIdx.x * kThreads + threadIdx.x) >> 5) * (32 / G) + group;
  const uint32_t ngroups = ((gridDim.x * kThreads) >> 5) * (32 / G);
  const uint64_t col = static_cast<uint64_t>(gl) * PER;
  const bool adagrad = opt.optimizer != TS_OPT_SGD;
  for (uint32_t ja = seg_lo + gid; ja < seg_hi; ja += 2 * ngroups) {
    const uint32_t jb = ja + ngroups;
    const bool has_b = jb < seg_hi;
    // round 1: segment metadata of both
    const uint32_t sa = __ldg(starts + ja), ea = __ldg(starts + ja + 1), ka = __ldg(seg_keys + ja);
    const uint32_t sb = has_b ? __ldg(starts + jb) : 0u, eb = has_b ? __ldg(starts + jb + 1) : 0u;
    const uint32_t kb = has_b ? __ldg(seg_keys + jb) : 0u;
    const bool long_a = ea - sa > short_max, long_b = has_b && eb - sb > short_max;
    if (long_list && gl == 0) {
      if (long_a) long_list[atomicAdd(long_count, 1u)] = ja;
      if (long_b) long_list[atomicAdd(long_count, 1u)] = jb;
    }
    const bool do_a = !long_a, do_b = has_b && !long_b;
    const bool upd_a = do_a && !in_dense(ka, d0, d1), upd_b = do_b && !in_dense(kb, d0, d1);
    // round 2: first two entries' gradient rows, weight rows, state
    float acc_a[PER], acc_b[PER], r_a[PER], r_b[PER], w_a[PER], w_b[PER];
    float st_a = 0.0f, st_b = 0.0f;
    const bool two_a = do_a && ea - sa >= 2, two_b = do_b && eb - sb >= 2;
    if (do_a) load_vec<PER>(grad_row<1>(gs, __ldg(vals + sa), DIM) + col, acc_a);
    if (do_b) load_vec<PER>(grad_row<1>(gs, __ldg(vals + sb), DIM) + col, acc_b);
    if (two_a) load_vec<PER>(grad_row<1>(gs, __ldg(vals + sa + 1), DIM) + col, r_a);
    if (two_b) load_vec<PER>(grad_row<1>(gs, __ldg(vals + sb + 1), DIM) + col, r_b);
    if (upd_a) {
      load_vec<PER>(weights + static_cast<uint64_t>(ka) * DIM + col, w_a);
      if (adagrad) st_a = state[ka];
    }
    if (upd_b) {
      load_vec<PER>(weights + static_cast<uint64_t>(kb) * DIM + col, w_b);
      if (adagrad) st_b = state[kb];
    }
    if (two_a) {
#pragma unroll
      for (int q = 0; q < PER; ++q) acc_a[q] = __fadd_rn(acc_a[q], r_a[q]);
      sum_tail<DIM, G>(vals, sa + 2, ea, gs, col, acc_a);
    }
    if (two_b) {
#pragma unroll
      for (int q = 0; q < PER; ++q) acc_b[q] = __fadd_rn(acc_b[q], r_b[q]);
      sum_tail<DIM, G>(vals, sb + 2, eb, gs, col, acc_b);
    }
    if (do_a) {
      if (upd_a) group_apply<DIM, G>(ka, acc_a, w_a, st_a, gl, gmask, weights, state, opt);
      else dense_store<DIM, G>(ka, acc_a, gl, d0, d1);
    }
    if (do_b) {
      if (upd_b) group_apply<DIM, G>(kb, acc_b, w_b, st_b, gl, gmask, weights, state, opt);
      else dense_store<DIM, G>(kb, acc_b, gl, d0, d1);
    }
  }
  if (d0.push_n | d1.push_n) __threadfence_system();  // partials stored to peers
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
seg_short_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                 const uint32_t* __restrict__ starts, const uint32_t* __restrict__ d_lo,
                 const uint32_t* __restrict__ d_hi,
                 GradSource gs, float* __restrict__ weights, float* __restrict__ state,
                 OptParams opt, DenseRange d0, DenseRange d1, uint32_t* __restrict__ long_list,
                 uint32_t* __restrict__ long_count, uint32_t short_max) {
  using Gp = Grouping<DIM>;
  constexpr int G = Gp::G, PER = Gp::PER, E = Gp::E;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned group = lane / G, gl = lane % G;
  const unsigned gmask = G == 32 ? 0xFFFFFFFFu : (((1u << G) - 1u) << (group * G));
  const uint32_t seg_lo = *d_lo, seg_hi = *d_hi;
  const uint32_t gid = ((blockIdx.x * kThreads + threadIdx.x) >> 5) * (32 / G) + group;
  const uint32_t ngroups = ((gridDim.x * kThreads) >> 5) * (32 / G);
  const uint64_t col = static_cast<uint64_t>(gl) * PER;
  for (uint32_t j = seg_lo + gid; j < seg_hi; j += ngroups) {
    const uint32_t s = __ldg(starts + j), e = __ldg(starts + j + 1);
    if (e - s > short_max) {  // listed here, or beforehand (long_list == nullptr)
      if (long_list && gl == 0) long_list[atomicAdd(long_count, 1u)] = j;
      continue;
    }
    const uint32_t row = __ldg(keys + s);
    float acc[PER];
    load_vec<PER>(grad_row<1>(gs, __ldg(vals + s), DIM) + col, acc);
    uint32_t k = s + 1;
    for (; k + E <= e; k += E) {
      float r[E][PER];
#pragma unroll
      for (int b = 0; b < E; ++b) load_vec<PER>(grad_row<1>(gs, __ldg(vals + k + b), DIM) + col, r[b]);
#pragma unroll
      for (int b = 0; b < E; ++b) {
#pragma unroll
        for (int q = 0; q < PER; ++q) acc[q] = __fadd_rn(acc[q], r[b][q]);
      }
    }
    for (; k < e; ++k) {
      float r[PER];
      load_vec<PER>(grad_row<1>(gs, __ldg(vals + k), DIM) + col, r);
#pragma unroll
      for (int q = 0; q < PER; ++q) acc[q] = __fadd_rn(acc[q], r[q]);
    }
    group_finish_row<DIM>(row, acc, gl, gmask, weights, state, opt, d0, d1);
  }
  if (d0.push_n | d1.push_n) __threadfence_system();  // partials stored to peers
}

// Segments [*d_lo, *d_hi) longer than short_max entries -> long_list (warp
// ballot + one atomic per warp), so the piece path can start without waiting
// for the short kernel to discover them.
__global__ void __launch_bounds__(kThreads)
long_segments_kernel(const uint32_t* __restrict__ starts, const uint32_t* __restrict__ d_lo,
                     const uint32_t* __restrict__ d_hi, uint32_t short_max,
                     uint32_t* __restrict__ long_list, uint32_t* __restrict__ long_count) {
  const uint32_t lo = *d_lo, hi = *d_hi;
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t stride = gridDim.x * kThreads;
  for (uint32_t base = lo + (blockIdx.x * kThreads + threadIdx.x - lane); base < hi; base += stride) {
    const uint32_t j = base + lane;
    const bool is_long = j < hi && __ldg(starts + j + 1) - __ldg(starts + j) > short_max;
    const unsigned b = __ballot_sync(0xFFFFFFFFu, is_long);
    if (!b) continue;
    uint32_t pos = 0;
    if (lane == 0) pos = atomicAdd(long_count, static_cast<uint32_t>(__popc(b)));
    pos = __shfl_sync(0xFFFFFFFFu, pos, 0);
    if (is_long) long_list[pos + __popc(b & ((1u << lane) - 1u))] = j;
  }
}

// piece_off[i] = exclusive prefix of pieces over the long list.
__global__ void __launch_bounds__(1024)
long_prefix_kernel(const uint32_t* __restrict__ long_list, const uint32_t* __restrict__ long_count,
                   const uint32_t* __restrict__ starts, uint32_t* __restrict__ piece_off) {
  __shared__ uint32_t s_warp[1024 / 32 + 1];
  const uint32_t n = *long_count;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < n; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    uint32_t pieces = 0;
    if (i < n) {
      const uint32_t j = long_list[i];
      pieces = (starts[j + 1] - starts[j] + kPiece - 1) / kPiece;
    }
    uint32_t total;
    const uint32_t ex = block_exclusive_scan<1024>(pieces, s_warp, &total);
    if (i < n) piece_off[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) piece_off[n] = carry;
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
piece_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
             const uint32_t* __restrict__ starts, const uint32_t* __restrict__ long_list,
             const uint32_t* __restrict__ long_count, const uint32_t* __restrict__ piece_off, GradSource gs,
             float* __restrict__ partials, float* __restrict__ weights, float* __restrict__ state, OptParams opt,
             DenseRange d0, DenseRange d1) {
  constexpr int VEC = DIM / 32;
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t n = *long_count;
  const uint32_t total = piece_off[n];
  const uint32_t gwarp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * kThreads) >> 5;
  for (uint32_t p = gwarp; p < total; p += nwarps) {
    uint32_t lo = 0, hi = n;  // last i with piece_off[i] <= p
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (piece_off[mid] <= p) lo = mid; else hi = mid;
    }
    const uint32_t j = long_list[lo];
    const uint32_t seg_s = starts[j], seg_e = starts[j + 1];
    const uint32_t s = seg_s + (p - piece_off[lo]) * kPiece;
    const uint32_t e = min(s + kPiece, seg_e);
    float acc[VEC];
    sum_entries<DIM>(vals, s, e, gs, acc);
    if (piece_off[lo + 1] - piece_off[lo] == 1) {
      // a single-piece segment (a mid-length one the short kernel handed
      // over): its sum is complete -- the same left-to-right order as the
      // short path -- so apply it here
      finish_row<DIM>(keys[seg_s], acc, weights, state, opt, d0, d1);
    } else {
      store_lane<VEC>(partials + static_cast<uint64_t>(p) * DIM + lane * VEC, acc);
    }
  }
  if (d0.push_n | d1.push_n) __threadfence_system();  // partials stored to peers
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
long_combine_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ starts,
                    const uint32_t* __restrict__ long_list, const uint32_t* __restrict__ long_count,
                    const uint32_t* __restrict__ piece_off, const float* __restrict__ partials,
                    float* __restrict__ weights, float* __restrict__ state, OptParams opt,
                    DenseRange d0, DenseRange d1) {
  constexpr int VEC = DIM / 32;
  constexpr int B = 8;
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t n = *long_count;
  const uint32_t gwarp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * kThreads) >> 5;
  for (uint32_t i = gwarp; i < n; i += nwarps) {
    const uint32_t j = long_list[i];
    const uint32_t p0 = piece_off[i], p1 = piece_off[i + 1];
    if (p1 - p0 == 1) continue;  // applied by piece_kernel
    float acc[VEC];
    load_lane<VEC>(partials + static_cast<uint64_t>(p0) * DIM + lane * VEC, acc);
    uint32_t p = p0 + 1;
    for (; p + B <= p1; p += B) {
      float r[B][VEC];
#pragma unroll
      for (int b = 0; b < B; ++b)
        load_lane<VEC>(partials + static_cast<uint64_t>(p + b) * DIM + lane * VEC, r[b]);
#pragma unroll
      for (int b = 0; b < B; ++b) {
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = __fadd_rn(acc[q], r[b][q]);
      }
    }
    for (; p < p1; ++p) {
      float r[VEC];
      load_lane<VEC>(partials + static_cast<uint64_t>(p) * DIM + lane * VEC, r);
#pragma unroll
      for (int q = 0; q < VEC; ++q) acc[q] = __fadd_rn(acc[q], r[q]);
    }
    finish_row<DIM>(keys[starts[j]], acc, weights, state, opt, d0, d1);
  }
  if (d0.push_n | d1.push_n) __threadfence_system();  // partials stored to peers
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
dense_update_kernel(const float* __restrict__ grad, uint32_t rows, uint32_t row_lo,
                    float* __restrict__ weights, float* __restrict__ state, OptParams opt) {
  constexpr int VEC = DIM / 32;
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t gwarp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * kThreads) >> 5;
  const DenseRange none{};
  for (uint32_t r = gwarp; r < rows; r += nwarps) {
    float g[VEC];
    load_lane<VEC>(grad + static_cast<uint64_t>(r) * DIM + lane * VEC, g);
    finish_row<DIM>(row_lo + r, g, weights, state, opt, none, none);
  }
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
replica_update_kernel(ReplicaGroup grp, OptParams opt) {
  constexpr int VEC = DIM / 32;
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t me = static_cast<uint32_t>(grp.me), size = static_cast<uint32_t>(grp.size);
  const uint32_t lo = grp.per * me;
  // rows I own: slots [0, n)
  const uint32_t n = grp.interleave ? (grp.rows > me ? (grp.rows - me + size - 1) / size : 0u)
                                    : (lo < grp.rows ? min(grp.per, grp.rows - lo) : 0u);
  const uint32_t gwarp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * kThreads) >> 5;
  float* mine = grp.weights[grp.me];
  float* my_state = grp.state[grp.me];
  for (uint32_t base = gwarp * 32; base < n; base += nwarps * 32) {
    // 32 rows' stamps at once (coalesced), then the rows some member touched
    const uint32_t i = base + lane;
    uint32_t members = 0;
    if (i < n) {
#pragma unroll
      for (int k = 0; k < kMaxGradPeers; ++k) {
        if (k < grp.size && __ldg(grp.recv_stamp + static_cast<uint64_t>(k) * grp.per + i) == grp.epoch) {
          members |= 1u << k;
        }
      }
    }
    unsigned active = __ballot_sync(0xFFFFFFFFu, members != 0);
    while (active) {
      const int b = __ffs(active) - 1;
      active &= active - 1;
      const uint32_t m = __shfl_sync(0xFFFFFFFFu, members, b);
      const uint32_t row = grp.interleave ? (base + b) * size + me : lo + base + b;
      float part[kMaxGradPeers][VEC];
#pragma unroll
      for (int k = 0; k < kMaxGradPeers; ++k) {  // touched members' partials in flight
        if ((m >> k) & 1u) {
          load_lane<VEC>(grp.recv + (static_cast<uint64_t>(k) * grp.per + base + b) * DIM + lane * VEC, part[k]);
        }
      }
      float g[VEC];
      bool first = true;
#pragma unroll
      for (int k = 0; k < kMaxGradPeers; ++k) {
        if ((m >> k) & 1u) {
#pragma unroll
          for (int j = 0; j < VEC; ++j) g[j] = first ? part[k][j] : __fadd_rn(g[j], part[k][j]);
          first = false;
        }
      }
      finish_row<DIM>(row, g, mine, my_state, opt, DenseRange{}, DenseRange{});
      __syncwarp();
      const uint64_t off = static_cast<uint64_t>(row) * DIM + lane * VEC;
      float w[VEC];
      load_lane<VEC>(mine + off, w);
      const float st = my_state ? my_state[row] : 0.0f;
#pragma unroll
      for (int k = 0; k < kMaxGradPeers; ++k) {
        if (k < grp.size && k != grp.me) {
          store_lane<VEC>(grp.weights[k] + off, w);
          if (my_state && lane == 0) grp.state[k][row] = st;
        }
      }
    }
  }
  __threadfence_system();
}

__global__ void __launch_bounds__(kThreads)
init_weights_kernel(float* __restrict__ weights, uint64_t local_rows, uint32_t dim, uint64_t seed,
                    const uint32_t* __restrict__ l2c) {
  const uint64_t total = local_rows * dim;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += stride) {
    const uint64_t l = i / dim;
    const uint32_t d = static_cast<uint32_t>(i - l * dim);
    const uint64_t canon = l2c ? l2c[l] : l;
    weights[i] = init_weight(seed, canon, d, dim);
  }
}

template <typename F>
void dispatch_dim(uint32_t dim, F&& f) {
  switch (dim) {
    case 32: f(std::integral_constant<int, 32>{}); break;
    case 64: f(std::integral_constant<int, 64>{}); break;
    case 128: f(std::integral_constant<int, 128>{}); break;
    case 256: f(std::integral_constant<int, 256>{}); break;
    case 512: f(std::integral_constant<int, 512>{}); break;
    case 1024: f(std::integral_constant<int, 1024>{}); break;
    default:
      fail(TS_ERR_CONFIG, "embedding_dim " + std::to_string(dim) +
                              " unsupported by the device path (32, 64, 128, 256, 512, 1024)");
  }
}

unsigned persistent_grid(unsigned per_sm) { return static_cast<unsigned>(sm_count()) * per_sm; }

// Blocks per SM of the compute-stream persistent grids.  With U > 1 the table
// lowers it so the exchange / replica kernels on the (high-priority) comm
// stream always find free SM slots instead of queueing behind grids that
// never retire a block (one table per process, set at creation).
// blocks per SM of the persistent compute grids (TIERSHARD_COMPUTE_BLOCKS)
unsigned g_compute_blocks_per_sm = [] {
  const char* e = std::getenv("TIERSHARD_COMPUTE_BLOCKS");
  return e ? static_cast<unsigned>(std::max(1, std::atoi(e))) : 8u;
}();

}  // namespace

unsigned gather_grid(uint64_t occ) {
  const uint64_t want = (occ + 63) / 64;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, persistent_grid(g_compute_blocks_per_sm))));
}

void set_compute_blocks_per_sm(unsigned per_sm) { g_compute_blocks_per_sm = per_sm; }

void launch_gather_local(const uint32_t* rows, uint64_t occ, const float* weights, float* out,
                         const RemapView& remap, uint32_t dim, double* loss_partials,
                         unsigned grid, cudaStream_t stream, int bulk_stages) {
  dispatch_dim(dim, [&](auto D) {
    constexpr int DIM = decltype(D)::value;
    if (bulk_stages > 0) {
      // grid = blocks per SM x SMs, each block 4 warps with bulk_stages
      // stages of 4 KB each
      const int stages = std::min(kBulkMaxStages, std::max(2, bulk_stages));
      const size_t smem = 8 * (kBulkThreads / 32) * kBulkMaxStages +
                          static_cast<size_t>(kBulkThreads / 32) * stages * kBulkStageBytes;
      static const bool attr = [] {  // the largest ring, once per instantiation
        const size_t most = 8 * (kBulkThreads / 32) * kBulkMaxStages +
                            static_cast<size_t>(kBulkThreads / 32) * kBulkMaxStages * kBulkStageBytes;
        TSD_CUDA(cudaFuncSetAttribute(gather_bulk_kernel<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(most)));
        return true;
      }();
      (void)attr;
      gather_bulk_kernel<DIM><<<grid, kBulkThreads, smem, stream>>>(rows, occ, weights, out, remap,
                                                                     loss_partials, stages);
      return;
    }
    constexpr int UNROLL = DIM <= 128 ? 8 : (DIM <= 256 ? 4 : 2);
    gather_local_kernel<DIM, UNROLL><<<grid, kThreads, 0, stream>>>(rows, occ, weights, out, remap,
                                                                     loss_partials);
  });
  TSD_LAUNCH_CHECK();
}

void launch_gather_all(const uint32_t* rows, uint64_t occ, const PeerWeights& pw, float* out,
                       const RemapView& remap, uint32_t dim, double* loss_partials, unsigned grid,
                       cudaStream_t stream) {
  dispatch_dim(dim, [&](auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int UNROLL = DIM <= 128 ? 8 : (DIM <= 256 ? 4 : 2);
    gather_all_kernel<DIM, UNROLL><<<grid, kThreads, 0, stream>>>(rows, occ, pw, out, remap, loss_partials);
  });
  TSD_LAUNCH_CHECK();
}

void launch_pull_rows(const uint32_t* sorted_bucket, const uint32_t* order, const uint32_t* ids,
                      const uint32_t* d_count, uint64_t max_count, const PeerWeights& pw, uint32_t u,
                      float* out, uint32_t dim, double* loss_partials, unsigned grid, cudaStream_t stream) {
  if (max_count == 0) return;
  dispatch_dim(dim, [&](auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int UNROLL = DIM <= 128 ? 8 : (DIM <= 256 ? 4 : 2);
    pull_rows_kernel<DIM, UNROLL><<<grid, kThreads, 0, stream>>>(sorted_bucket, order, ids, d_count, max_count,
                                                                 pw, u, out, loss_partials);
  });
  TSD_LAUNCH_CHECK();
}

void launch_loss_finalize(const double* partials, unsigned count, double* loss, cudaStream_t stream,
                          double* mirror) {
  loss_finalize_kernel<<<1, 1024, 0, stream>>>(partials, count, loss, mirror);
  TSD_LAUNCH_CHECK();
}

// Number of segments whose key is < split_key (sorted keys, so a lower bound
// over the segment heads); out[0] = 0, out[1] = split.
__global__ void segment_split_kernel(const uint32_t* __restrict__ keys,
                                     const uint32_t* __restrict__ starts,
                                     const uint32_t* __restrict__ d_nseg, uint32_t split_key,
                                     uint32_t* __restrict__ out) {
  // One warp, 33-ary search: each round probes 32 evenly spaced segments in
  // parallel, so a 2^21-segment range resolves in ~4 dependent round trips.
  const unsigned lane = threadIdx.x & 31u;
  uint32_t lo = 0, hi = *d_nseg;  // answer in [lo, hi]
  while (hi > lo) {
    const uint32_t span = hi - lo;
    const uint32_t probe = lo + static_cast<uint32_t>((static_cast<uint64_t>(span) * (lane + 1)) / 33);
    const bool below = probe < hi && keys[starts[probe]] < split_key;
    const unsigned b = __ballot_sync(0xFFFFFFFFu, below);
    // probes are increasing: `below` holds for a prefix of lanes
    const int nb = __popc(b);
    const uint32_t new_lo = nb == 0 ? lo : lo + static_cast<uint32_t>((static_cast<uint64_t>(span) * nb) / 33) + 1;
    const uint32_t new_hi = nb == 32 ? hi : lo + static_cast<uint32_t>((static_cast<uint64_t>(span) * (nb + 1)) / 33);
    if (span <= 32) {  // finish linearly
      uint32_t ans = hi;
      for (uint32_t j = lo; j < hi; ++j) {
        if (!(keys[starts[j]] < split_key)) {
          ans = j;
          break;
        }
      }
      lo = hi = ans;
      break;
    }
    lo = new_lo;
    hi = new_hi;
  }
  if (lane == 0) {
    out[0] = 0;
    out[1] = lo;
  }
}

void launch_segment_split(const uint32_t* keys, const uint32_t* starts, const uint32_t* d_nseg,
                          uint32_t split_key, uint32_t* out, cudaStream_t stream) {
  segment_split_kernel<<<1, 32, 0, stream>>>(keys, starts, d_nseg, split_key, out);
  TSD_LAUNCH_CHECK();
}

// Short-segment kernel choice: TIERSHARD_SEG=single (default) | pair.
// Measured on B200 at C2 (N=1, segment_update phase): single 0.756 ms,
// pair G=16 0.861 ms, pair G=8 1.177 ms — the pair kernel's extra ILP costs
// more in occupancy (80 / 152 registers) than it buys; kept as an option.
// TIERSHARD_SEG_G = lanes per segment for the pair kernel at dim 128.
int seg_variant() {
  static const int v = [] {
    const char* e = std::getenv("TIERSHARD_SEG");
    return e && std::string(e) == "pair" ? 1 : 0;
  }();
  return v;
}
// Segments longer than `short_max` entries go to the warp-per-piece path
// (<= kPiece): the short kernel's 4-8 segments per warp finish together only
// when their lengths are alike.  Same sums either way (a single piece is
// summed left to right).  Measured at C2 (segment update + long path):
// N=1: 256 -> 0.712 ms, 64 -> 0.693, 32 -> 0.684, 16 -> 0.724, 8 -> 0.747;
// N=2 step: 256 -> 2.39 ms, 32 -> 2.455; N=4: 3.437 vs 3.417 (noise).
// Default: 32 on one GPU, 256 otherwise (TIERSHARD_SHORT_MAX overrides).
uint32_t short_max(uint32_t gpus) {
  const char* e = std::getenv("TIERSHARD_SHORT_MAX");
  const int x = e ? std::atoi(e) : (gpus == 1 ? 32 : static_cast<int>(kPiece));
  return static_cast<uint32_t>(std::min<int>(std::max(x, 1), static_cast<int>(kPiece)));
}
int seg_group_128() {
  static const int v = [] {
    const char* e = std::getenv("TIERSHARD_SEG_G");
    return e && std::string(e) == "8" ? 8 : 16;
  }();
  return v;
}

void launch_segment_update(const uint32_t* keys, const uint32_t* vals, const uint32_t* starts,
                           const uint32_t* seg_keys, const uint32_t* d_lo, const uint32_t* d_hi,
                           uint64_t n_entries, uint32_t dim, const GradSource& grads, float* weights,
                           float* state, const OptParams& opt, const DenseRange& dense0,
                           const DenseRange& dense1, const SegmentScratch& sc,
                           cudaStream_t stream) {
  if (n_entries == 0) return;
  if (sc.long_list) TSD_CUDA(cudaMemsetAsync(sc.long_count, 0, sizeof(uint32_t), stream));
  // with the long path concurrent (long_list == nullptr) the short kernel's
  // grid can leave SM slots to it: TIERSHARD_SHORT_BLOCKS blocks per SM.
  // Measured at C2, N=1 (4 resident at 64 registers): 8 -> 1.308 ms/step
  // (the piece kernel starts once first-wave blocks retire), 4 -> 1.322 (it
  // starts only at the end), 3 -> 1.305 (both run side by side and end
  // together), 2 -> 1.399.  Default: the compute grid (8 per SM).
  static const unsigned short_blocks = [] {
    const char* e = std::getenv("TIERSHARD_SHORT_BLOCKS");
    return e ? static_cast<unsigned>(std::max(1, std::atoi(e))) : 0u;
  }();
  const unsigned grid = persistent_grid(!sc.long_list && short_blocks ? short_blocks : g_compute_blocks_per_sm);
  dispatch_dim(dim, [&](auto D) {
    constexpr int DIM = decltype(D)::value;
    if (seg_variant() == 0 || DIM > 128) {
      seg_short_kernel<DIM><<<grid, kThreads, 0, stream>>>(keys, vals, starts, d_lo, d_hi, grads,
                                                           weights, state, opt, dense0, dense1,
                                                           sc.long_list, sc.long_count, sc.short_max);
    } else if (DIM == 128 && seg_group_128() == 16) {
      if constexpr (DIM == 128) {
        seg_pair_kernel<DIM, 16><<<grid, kThreads, 0, stream>>>(vals, starts, seg_keys, d_lo, d_hi, grads,
                                                               weights, state, opt, dense0, dense1,
                                                               sc.long_list, sc.long_count, sc.short_max);
      }
    } else {
      constexpr int G = 8;  // DIM <= 128 here
      if constexpr (DIM <= 128) seg_pair_kernel<DIM, G><<<grid, kThreads, 0, stream>>>(vals, starts, seg_keys, d_lo, d_hi, grads,
                                                            weights, state, opt, dense0, dense1,
                                                            sc.long_list, sc.long_count, sc.short_max);
    }
    TSD_LAUNCH_CHECK();
  });
}

void launch_segment_long(const uint32_t* keys, const uint32_t* vals, const uint32_t* starts,
                         uint64_t n_entries, uint32_t dim, const GradSource& grads, float* weights,
                         float* state, const OptParams& opt, const DenseRange& dense0,
                         const DenseRange& dense1, const SegmentScratch& sc, cudaStream_t stream) {
  if (n_entries == 0) return;
  const unsigned grid = persistent_grid(g_compute_blocks_per_sm);
  dispatch_dim(dim, [&](auto D) {
    constexpr int DIM = decltype(D)::value;
    if (!sc.prefixed) {
      long_prefix_kernel<<<1, 1024, 0, stream>>>(sc.long_list, sc.long_count, starts, sc.piece_off);
      TSD_LAUNCH_CHECK();
    }
    piece_kernel<DIM><<<grid, kThreads, 0, stream>>>(keys, vals, starts, sc.long_list, sc.long_count,
                                                     sc.piece_off, grads, sc.partials, weights, state, opt,
                                                     dense0, dense1);
    TSD_LAUNCH_CHECK();
    long_combine_kernel<DIM><<<grid, kThreads, 0, stream>>>(keys, starts, sc.long_list,
                                                            sc.long_count, sc.piece_off,
                                                            sc.partials, weights, state, opt,
                                                            dense0, dense1);
    TSD_LAUNCH_CHECK();
  });
}

void launch_long_segments(const uint32_t* starts, const uint32_t* d_lo, const uint32_t* d_hi,
                          uint64_t n_entries, const SegmentScratch& sc, cudaStream_t stream) {
  TSD_CUDA(cudaMemsetAsync(sc.long_count, 0, sizeof(uint32_t), stream));
  const unsigned grid = std::max<unsigned>(
      1, std::min<unsigned>(persistent_grid(4), static_cast<unsigned>(ceil_div(n_entries, kThreads))));
  long_segments_kernel<<<grid, kThreads, 0, stream>>>(starts, d_lo, d_hi, sc.short_max, sc.long_list,
                                                      sc.long_count);
  TSD_LAUNCH_CHECK();
  long_prefix_kernel<<<1, 1024, 0, stream>>>(sc.long_list, sc.long_count, starts, sc.piece_off);
  TSD_LAUNCH_CHECK();
}

void launch_dense_update(const float* grad, uint32_t rows, uint32_t row_lo, uint32_t dim,
                         float* weights, float* state, const OptParams& opt, cudaStream_t stream) {
  if (rows == 0) return;
  const unsigned grid = std::min<unsigned>(persistent_grid(8), ceil_div(rows, kThreads / 32));
  dispatch_dim(dim, [&](auto D) {
    constexpr int DIM = decltype(D)::value;
    dense_update_kernel<DIM><<<grid, kThreads, 0, stream>>>(grad, rows, row_lo, weights, state, opt);
  });
  TSD_LAUNCH_CHECK();
}

void launch_replica_update(const ReplicaGroup& grp, uint32_t dim, const OptParams& opt,
                           cudaStream_t stream) {
  if (grp.rows == 0 || grp.size == 0) return;
  const unsigned grid = std::max<unsigned>(
      1, std::min<unsigned>(persistent_grid(g_compute_blocks_per_sm), ceil_div(grp.per, kThreads)));
  dispatch_dim(dim, [&](auto D) {
    constexpr int DIM = decltype(D)::value;
    replica_update_kernel<DIM><<<grid, kThreads, 0, stream>>>(grp, opt);
  });
  TSD_LAUNCH_CHECK();
}

void launch_init_weights(float* weights, uint64_t local_rows, uint32_t dim, uint64_t seed,
                         const uint32_t* l2c, cudaStream_t stream) {
  if (local_rows == 0) return;
  init_weights_kernel<<<persistent_grid(8), kThreads, 0, stream>>>(weights, local_rows, dim, seed, l2c);
  TSD_LAUNCH_CHECK();
}

}  // namespace tsd
