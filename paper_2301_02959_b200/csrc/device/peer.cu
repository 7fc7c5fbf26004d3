// Peer-memory exchange kernels and CUDA-IPC plumbing (peer.cuh).
#include <cuda.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>

#include "common.cuh"
#include "peer.cuh"

namespace tsd {

namespace {

using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

GetRangeFn get_range_fn() {
  static GetRangeFn fn = [] {
    void* h = dlopen("libcuda.so.1", RTLD_LAZY | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_LAZY);
    if (!h) return static_cast<GetRangeFn>(nullptr);
    return reinterpret_cast<GetRangeFn>(dlsym(h, "cuMemGetAddressRange_v2"));
  }();
  return fn;
}

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
pull_requests_kernel(PullTable t, uint32_t* __restrict__ recv_ids, uint32_t* __restrict__ recv_pos) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < t.total; i += stride) {
    int s = 0;
    while (s + 1 < t.nseg && i >= t.seg[s + 1].dst_off) ++s;
    const PullSeg& g = t.seg[s];
    const uint64_t j = g.src_off + (i - g.dst_off);
    recv_ids[i] = g.ids[j];  // coalesced loads from the peer's HBM
    recv_pos[i] = g.pos[j];
  }
}

template <int VEC4>  // float4s per lane per row
__global__ void __launch_bounds__(kThreads)
serve_rows_kernel(const float* __restrict__ weights, const uint32_t* __restrict__ recv_ids,
                  const uint32_t* __restrict__ recv_pos, ServeTable st, uint32_t dim) {
  constexpr int kRows = 4;  // rows in flight per warp
  __shared__ float s_sq[kThreads / 32];
  const ServeTarget tg = st.t[blockIdx.y];
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  const uint32_t vecs = dim / 4;
  float sq = 0.0f;
  for (uint64_t r0 = tg.r_begin + gwarp * kRows; r0 < tg.r_end; r0 += nwarps * kRows) {
    float4 v[kRows][VEC4];
    uint32_t pos[kRows];
    bool ok[kRows];
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      const uint64_t r = r0 + k;
      ok[k] = r < tg.r_end;
      const uint32_t id = ok[k] ? __ldg(recv_ids + r) : 0u;
      pos[k] = ok[k] ? __ldg(recv_pos + r) : 0u;
      const float4* src = reinterpret_cast<const float4*>(weights + static_cast<uint64_t>(id) * dim);
#pragma unroll
      for (int q = 0; q < VEC4; ++q) {
        const uint32_t c = lane + 32u * q;
        if (ok[k] && c < vecs) v[k][q] = __ldg(src + c);
      }
    }
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      if (!ok[k]) continue;
      float4* dst = reinterpret_cast<float4*>(tg.out + static_cast<uint64_t>(pos[k]) * dim);
#pragma unroll
      for (int q = 0; q < VEC4; ++q) {
        const uint32_t c = lane + 32u * q;
        if (c < vecs) {
          dst[c] = v[k][q];  // NVLink store into the requester's output
          sq = __fmaf_rn(v[k][q].x, v[k][q].x, sq);
          sq = __fmaf_rn(v[k][q].y, v[k][q].y, sq);
          sq = __fmaf_rn(v[k][q].z, v[k][q].z, sq);
          sq = __fmaf_rn(v[k][q].w, v[k][q].w, sq);
        }
      }
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, m);
  if (lane == 0) s_sq[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) acc += static_cast<double>(s_sq[w]);
    tg.loss_slots[blockIdx.x] = acc;
  }
  __threadfence_system();  // peer stores visible before the completion barrier
}

template <int VEC4>
__global__ void __launch_bounds__(kThreads)
pull_grads_kernel(PullGrads pg, const uint32_t* __restrict__ recv_pos, uint64_t count,
                  float* __restrict__ dst, uint32_t dim) {
  constexpr int kRows = 4;
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  const uint32_t vecs = dim / 4;
  for (uint64_t r0 = gwarp * kRows; r0 < count; r0 += nwarps * kRows) {
    float4 v[kRows][VEC4];
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      const uint64_t r = r0 + k;
      if (r >= count) continue;
      int s = 0;
      while (s + 1 < pg.nsrc && r >= pg.src_start[s + 1]) ++s;
      const float4* src =
          reinterpret_cast<const float4*>(pg.src[s] + static_cast<uint64_t>(__ldg(recv_pos + r)) * dim);
#pragma unroll
      for (int q = 0; q < VEC4; ++q) {
        const uint32_t c = lane + 32u * q;
        if (c < vecs) v[k][q] = src[c];  // NVLink load from the requester's gradient
      }
    }
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      const uint64_t r = r0 + k;
      if (r >= count) continue;
      float4* d = reinterpret_cast<float4*>(dst + r * dim);
#pragma unroll
      for (int q = 0; q < VEC4; ++q) {
        const uint32_t c = lane + 32u * q;
        if (c < vecs) d[c] = v[k][q];
      }
    }
  }
}

__global__ void flag_barrier_kernel(FlagBarrier b, int channel, uint64_t value) {
  const int p = static_cast<int>(threadIdx.x);
  const int off = channel * kMaxPeerRanks;
  __threadfence_system();  // this rank's earlier peer stores before its flag
  if (p < b.n && p != b.me) {
    uint64_t* dst = b.peer_flags[p] + off + b.me;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(value) : "memory");
  }
  if (p < b.n && p != b.me) {
    const uint64_t* src = b.peer_flags[b.me] + off + p;
    uint64_t seen = 0;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(seen) : "l"(src) : "memory");
      if (seen >= value) break;
      __nanosleep(64);
    }
  }
  __syncwarp();
  __threadfence_system();
}

__global__ void mailbox_put_kernel(MailboxPut m, const uint32_t* __restrict__ src, uint32_t words, size_t offset) {
  for (int p = 0; p < m.n; ++p) {
    if (p == m.me) continue;
    uint32_t* dst = reinterpret_cast<uint32_t*>(m.peer_box[p] + offset);
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  }
  __threadfence_system();
}

}  // namespace

void launch_mailbox_put(const MailboxPut& m, const uint8_t* src, size_t bytes, size_t offset,
                        cudaStream_t stream) {
  mailbox_put_kernel<<<1, 128, 0, stream>>>(m, reinterpret_cast<const uint32_t*>(src),
                                           static_cast<uint32_t>(bytes / 4), offset);
  TSD_LAUNCH_CHECK();
}

void launch_flag_barrier(const FlagBarrier& b, int channel, uint64_t value, cudaStream_t stream) {
  flag_barrier_kernel<<<1, 32, 0, stream>>>(b, channel, value);
  TSD_LAUNCH_CHECK();
}

void launch_pull_grads(const PullGrads& pg, const uint32_t* recv_pos, uint64_t count, float* dst,
                       uint32_t dim, cudaStream_t stream) {
  if (count == 0) return;
  const unsigned grid = 2 * sm_count();  // the two SM slots reserved for the comm stream
  const uint32_t vec4 = (dim / 4 + 31) / 32;
  switch (vec4) {
    case 1: pull_grads_kernel<1><<<grid, kThreads, 0, stream>>>(pg, recv_pos, count, dst, dim); break;
    case 2: pull_grads_kernel<2><<<grid, kThreads, 0, stream>>>(pg, recv_pos, count, dst, dim); break;
    case 4: pull_grads_kernel<4><<<grid, kThreads, 0, stream>>>(pg, recv_pos, count, dst, dim); break;
    default: pull_grads_kernel<8><<<grid, kThreads, 0, stream>>>(pg, recv_pos, count, dst, dim); break;
  }
  TSD_LAUNCH_CHECK();
}

template <int VEC4>
__global__ void __launch_bounds__(kThreads)
push_grads_kernel(PushTable t, const uint32_t* __restrict__ order, const float* __restrict__ grad,
                  uint32_t dim) {
  constexpr int kRows = 4;  // local loads in flight per warp
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  const uint64_t total = t.run_start[t.n];
  const uint32_t vecs = dim / 4;
  for (uint64_t r0 = gwarp * kRows; r0 < total; r0 += nwarps * kRows) {
    float4 v[kRows][VEC4];
    float4* dst[kRows];
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      const uint64_t r = r0 + k;
      dst[k] = nullptr;
      if (r >= total) continue;
      int s = 0;
      while (s + 1 < t.n && r >= t.run_start[s + 1]) ++s;
      const uint64_t j = r - t.run_start[s];
      const float4* src = reinterpret_cast<const float4*>(
          grad + static_cast<uint64_t>(__ldg(order + t.run[s].src_begin + j)) * dim);
      dst[k] = reinterpret_cast<float4*>(t.run[s].dst + j * dim);
#pragma unroll
      for (int q = 0; q < VEC4; ++q) {
        const uint32_t c = lane + 32u * q;
        if (c < vecs) v[k][q] = __ldg(src + c);
      }
    }
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      if (!dst[k]) continue;
#pragma unroll
      for (int q = 0; q < VEC4; ++q) {
        const uint32_t c = lane + 32u * q;
        if (c < vecs) dst[k][c] = v[k][q];  // NVLink store into the server's receive buffer
      }
    }
  }
  __threadfence_system();
}

void launch_push_grads(const PushTable& t, const uint32_t* order, const float* grad, uint32_t dim,
                       cudaStream_t stream) {
  if (t.n == 0 || t.run_start[t.n] == 0) return;
  // one block per SM saturates NVLink stores (~700 GB/s) and leaves the rest
  // of every SM to the sort it overlaps (TIERSHARD_PUSH_BLOCKS = per SM)
  static const unsigned per_sm = [] {
    const char* e = std::getenv("TIERSHARD_PUSH_BLOCKS");
    return e ? static_cast<unsigned>(std::max(1, std::atoi(e))) : 1u;
  }();
  const unsigned grid = per_sm * sm_count();
  const uint32_t vec4 = (dim / 4 + 31) / 32;
  switch (vec4) {
    case 1: push_grads_kernel<1><<<grid, kThreads, 0, stream>>>(t, order, grad, dim); break;
    case 2: push_grads_kernel<2><<<grid, kThreads, 0, stream>>>(t, order, grad, dim); break;
    case 4: push_grads_kernel<4><<<grid, kThreads, 0, stream>>>(t, order, grad, dim); break;
    default: push_grads_kernel<8><<<grid, kThreads, 0, stream>>>(t, order, grad, dim); break;
  }
  TSD_LAUNCH_CHECK();
}

IpcExport export_pointer(const void* ptr) {
  IpcExport e;
  std::memset(&e, 0, sizeof(e));
  GetRangeFn fn = get_range_fn();
  if (!fn) fail(TS_ERR_CUDA, "peer exchange: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) {
    fail(TS_ERR_CUDA, "peer exchange: pointer is not a device allocation");
  }
  TSD_CUDA(cudaIpcGetMemHandle(&e.handle, reinterpret_cast<void*>(base)));
  e.offset = reinterpret_cast<uint64_t>(ptr) - base;
  e.base_id = base;
  return e;
}

IpcExport direct_export(const void* ptr) {
  IpcExport e;
  std::memset(&e, 0, sizeof(e));
  e.base_id = reinterpret_cast<uint64_t>(ptr);
  return e;
}

void* PeerMappings::open(int peer, const IpcExport& e) {
  if (direct_) return reinterpret_cast<char*>(e.base_id) + e.offset;
  // keyed by base address, validated by handle: an exporter that freed and
  // re-allocated at the same address sends a different handle, and the stale
  // mapping is replaced instead of reused
  const auto key = std::make_pair(peer, e.base_id);
  auto it = opened_.find(key);
  if (it != opened_.end() && std::memcmp(&it->second.handle, &e.handle, sizeof(e.handle)) != 0) {
    ++reopens_;
    TSD_CUDA(cudaIpcCloseMemHandle(it->second.base));
    opened_.erase(it);
    it = opened_.end();
  }
  if (it == opened_.end()) {
    void* p = nullptr;
    TSD_CUDA(cudaIpcOpenMemHandle(&p, e.handle, cudaIpcMemLazyEnablePeerAccess));
    ++opens_;
    it = opened_.emplace(key, Mapping{e.handle, p}).first;
  }
  return static_cast<char*>(it->second.base) + e.offset;
}

void PeerMappings::close(int peer, const IpcExport& e) {
  if (direct_) return;
  auto it = opened_.find(std::make_pair(peer, e.base_id));
  if (it == opened_.end()) return;
  cudaIpcCloseMemHandle(it->second.base);
  opened_.erase(it);
}

void PeerMappings::close_all() {
  if (std::getenv("TIERSHARD_DEBUG_IPC") && opens_) {
    std::fprintf(stderr, "tiershard: peer mappings: %llu opens, %llu handle changes\n",
                 static_cast<unsigned long long>(opens_), static_cast<unsigned long long>(reopens_));
  }
  for (auto& kv : opened_) cudaIpcCloseMemHandle(kv.second.base);
  opened_.clear();
}

void launch_pull_requests(const PullTable& t, uint32_t* recv_ids, uint32_t* recv_pos, cudaStream_t stream) {
  if (t.total == 0) return;
  const uint64_t want = (t.total + kThreads * 4 - 1) / (kThreads * 4);
  const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, 4 * sm_count())));
  pull_requests_kernel<<<grid, kThreads, 0, stream>>>(t, recv_ids, recv_pos);
  TSD_LAUNCH_CHECK();
}

unsigned serve_blocks() {
  static const unsigned v = [] {
    const char* e = std::getenv("TIERSHARD_SERVE_BLOCKS");
    const int b = e ? std::atoi(e) : 96;
    return static_cast<unsigned>(std::min<int>(std::max(b, 1), static_cast<int>(kServeGrid)));
  }();
  return v;
}

void launch_serve_rows(const float* weights, const uint32_t* recv_ids, const uint32_t* recv_pos,
                       const ServeTable& st, uint32_t dim, cudaStream_t stream) {
  if (st.n == 0) return;
  const dim3 grid(serve_blocks(), st.n);
  const uint32_t vec4 = (dim / 4 + 31) / 32;
  switch (vec4) {
    case 1: serve_rows_kernel<1><<<grid, kThreads, 0, stream>>>(weights, recv_ids, recv_pos, st, dim); break;
    case 2: serve_rows_kernel<2><<<grid, kThreads, 0, stream>>>(weights, recv_ids, recv_pos, st, dim); break;
    case 4: serve_rows_kernel<4><<<grid, kThreads, 0, stream>>>(weights, recv_ids, recv_pos, st, dim); break;
    default: serve_rows_kernel<8><<<grid, kThreads, 0, stream>>>(weights, recv_ids, recv_pos, st, dim); break;
  }
  TSD_LAUNCH_CHECK();
}

}  // namespace tsd
