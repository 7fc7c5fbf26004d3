// Device-wide scan, stable LSD radix sort and segment-start compaction
// (declarations and design notes in primitives.cuh).
#include "common.cuh"
#include "primitives.cuh"

namespace tsd {
namespace {

// ---------------------------------------------------------------------------
// exclusive scan
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kScanThreads)
scan_tile_sums_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t* __restrict__ sums) {
  __shared__ uint32_t s_warp[kScanThreads / 32 + 1];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile;
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * kScanThreads + threadIdx.x;
    if (i < n) acc += in[i];
  }
  uint32_t total;
  block_exclusive_scan<kScanThreads>(acc, s_warp, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// One block scans the tile sums in chunks, carrying the running total.
__global__ void __launch_bounds__(1024)
scan_single_block_kernel(uint32_t* __restrict__ sums, uint64_t ntiles, uint32_t* __restrict__ d_total) {
  __shared__ uint32_t s_warp[1024 / 32 + 1];
  uint32_t carry = 0;
  for (uint64_t base = 0; base < ntiles; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint32_t v = i < ntiles ? sums[i] : 0u;
    uint32_t total;
    const uint32_t ex = block_exclusive_scan<1024>(v, s_warp, &total);
    if (i < ntiles) sums[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) {
    sums[ntiles] = carry;
    if (d_total) *d_total = carry;
  }
}

__global__ void __launch_bounds__(kScanThreads)
scan_apply_kernel(const uint32_t* in, uint32_t* out, uint64_t n, const uint32_t* __restrict__ prefix) {
  __shared__ uint32_t s_warp[kScanThreads / 32 + 1];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile +
                        static_cast<uint64_t>(threadIdx.x) * kScanItems;
  uint32_t v[kScanItems];
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : 0u;
    acc += v[k];
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan<kScanThreads>(acc, s_warp, &total) + prefix[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

// ---------------------------------------------------------------------------
// radix sort
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kRadixThreads)
radix_hist_kernel(const uint32_t* __restrict__ keys, uint64_t n, int shift, uint32_t mask,
                  uint32_t* __restrict__ hist, uint32_t tiles) {
  __shared__ uint32_t s_h[kRadixBins];
  s_h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kRadixTile;
#pragma unroll 4
  for (int k = 0; k < kRadixItems; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * kRadixThreads + threadIdx.x;
    const bool valid = i < n;
    const uint32_t d = valid ? (keys[i] >> shift) & mask : 0xFFFFFFFFu;
    // Zipf-skewed keys put many equal digits in one warp: aggregate first.
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    if (valid && (peers & lanemask_lt()) == 0) atomicAdd(&s_h[d], __popc(peers));
  }
  __syncthreads();
  hist[static_cast<uint64_t>(threadIdx.x) * tiles + blockIdx.x] = s_h[threadIdx.x];
}

__global__ void __launch_bounds__(kRadixThreads)
radix_scatter_kernel(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                     uint64_t n, int shift, uint32_t mask, const uint32_t* __restrict__ hist,
                     const uint32_t* __restrict__ hist_scan, uint32_t tiles,
                     uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
  __shared__ uint32_t s_keys[kRadixTile];
  __shared__ uint32_t s_vals[kRadixTile];
  __shared__ uint32_t s_run[kRadixWarps][kRadixBins];
  __shared__ uint32_t s_tile_excl[kRadixBins];
  __shared__ uint32_t s_gbase[kRadixBins];
  __shared__ uint32_t s_warp[kRadixThreads / 32 + 1];

  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t tile_base = static_cast<uint64_t>(blockIdx.x) * kRadixTile;

#pragma unroll
  for (int w = 0; w < kRadixWarps; ++w) s_run[w][threadIdx.x] = 0;
  {
    const uint64_t hi = static_cast<uint64_t>(threadIdx.x) * tiles + blockIdx.x;
    uint32_t total;
    s_tile_excl[threadIdx.x] = block_exclusive_scan<kRadixThreads>(hist[hi], s_warp, &total);
    s_gbase[threadIdx.x] = hist_scan[hi];
  }
  __syncthreads();

  uint32_t k[kRadixItems], v[kRadixItems], rank[kRadixItems];
  const uint64_t sub_base = tile_base + static_cast<uint64_t>(warp) * kRadixSubTile;
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint64_t i = sub_base + static_cast<uint64_t>(r) * 32 + lane;
    const bool valid = i < n;
    k[r] = valid ? keys_in[i] : 0u;
    v[r] = valid ? (vals_in ? vals_in[i] : static_cast<uint32_t>(i)) : 0u;
    const uint32_t d = valid ? (k[r] >> shift) & mask : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    rank[r] = valid ? s_run[warp][d] + __popc(peers & lanemask_lt()) : 0u;
    __syncwarp();
    if (valid && (peers & lanemask_lt()) == 0) s_run[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    // order the warps' sub-tiles: per digit, prefix over warps
    uint32_t acc = s_tile_excl[threadIdx.x];
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      const uint32_t t = s_run[w][threadIdx.x];
      s_run[w][threadIdx.x] = acc;
      acc += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint64_t i = sub_base + static_cast<uint64_t>(r) * 32 + lane;
    if (i < n) {
      const uint32_t d = (k[r] >> shift) & mask;
      const uint32_t pos = s_run[warp][d] + rank[r];
      s_keys[pos] = k[r];
      s_vals[pos] = v[r];
    }
  }
  __syncthreads();
  const uint64_t left = n - tile_base;
  const uint32_t tile_n = left < kRadixTile ? static_cast<uint32_t>(left) : kRadixTile;
  for (uint32_t j = threadIdx.x; j < tile_n; j += kRadixThreads) {
    const uint32_t kk = s_keys[j];
    const uint32_t d = (kk >> shift) & mask;
    const uint32_t dst = s_gbase[d] + (j - s_tile_excl[d]);
    keys_out[dst] = kk;
    vals_out[dst] = s_vals[j];
  }
}

// ---------------------------------------------------------------------------
// segment starts
// ---------------------------------------------------------------------------

__device__ __forceinline__ bool is_head(const uint32_t* keys, uint64_t i) {
  return i == 0 || keys[i] != keys[i - 1];
}

__global__ void __launch_bounds__(kScanThreads)
heads_count_kernel(const uint32_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ tile_cnt) {
  __shared__ uint32_t s_warp[kScanThreads / 32 + 1];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile;
  uint32_t c = 0;
#pragma unroll 4
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * kScanThreads + threadIdx.x;
    if (i < n && is_head(keys, i)) ++c;
  }
  uint32_t total;
  block_exclusive_scan<kScanThreads>(c, s_warp, &total);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads)
heads_write_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                   const uint32_t* __restrict__ tile_off, uint32_t* __restrict__ starts,
                   const uint32_t* __restrict__ d_nseg) {
  __shared__ uint32_t s_warp[kScanThreads / 32 + 1];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile +
                        static_cast<uint64_t>(threadIdx.x) * kScanItems;
  uint32_t flags = 0, c = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = base + k;
    if (i < n && is_head(keys, i)) {
      flags |= 1u << k;
      ++c;
    }
  }
  uint32_t total;
  uint32_t pos = block_exclusive_scan<kScanThreads>(c, s_warp, &total) + tile_off[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (flags & (1u << k)) starts[pos++] = static_cast<uint32_t>(base + k);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) starts[*d_nseg] = static_cast<uint32_t>(n);
}

}  // namespace

void device_exclusive_scan(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* scratch,
                           uint32_t* d_total, cudaStream_t stream) {
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (n == 0) {
    if (d_total) TSD_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint32_t), stream));
    return;
  }
  scan_tile_sums_kernel<<<static_cast<unsigned>(tiles), kScanThreads, 0, stream>>>(in, n, scratch);
  TSD_LAUNCH_CHECK();
  scan_single_block_kernel<<<1, 1024, 0, stream>>>(scratch, tiles, d_total);
  TSD_LAUNCH_CHECK();
  scan_apply_kernel<<<static_cast<unsigned>(tiles), kScanThreads, 0, stream>>>(in, out, n, scratch);
  TSD_LAUNCH_CHECK();
}

void radix_sort_pairs(const uint32_t* keys_in, const uint32_t* vals_in, uint64_t n, int key_bits,
                      const RadixBuffers& buf, uint32_t** keys_out, uint32_t** vals_out,
                      cudaStream_t stream) {
  // Even passes write (keys_a, vals_a), odd passes (keys_b, vals_b); the
  // caller's input is only read.
  const uint32_t* cur_k = keys_in;
  const uint32_t* cur_v = vals_in;
  *keys_out = buf.keys_a;
  *vals_out = buf.vals_a;
  if (n == 0) return;
  const uint32_t tiles = static_cast<uint32_t>(radix_tiles(n));
  if (key_bits < 1) key_bits = 1;
  int pass = 0;
  for (int shift = 0; shift < key_bits; shift += 8, ++pass) {
    const int bits = key_bits - shift < 8 ? key_bits - shift : 8;
    const uint32_t mask = (1u << bits) - 1u;
    uint32_t* out_k = (pass & 1) ? buf.keys_b : buf.keys_a;
    uint32_t* out_v = (pass & 1) ? buf.vals_b : buf.vals_a;
    radix_hist_kernel<<<tiles, kRadixThreads, 0, stream>>>(cur_k, n, shift, mask, buf.hist, tiles);
    TSD_LAUNCH_CHECK();
    device_exclusive_scan(buf.hist, buf.hist_scan, static_cast<uint64_t>(kRadixBins) * tiles,
                          buf.scan_scratch, nullptr, stream);
    radix_scatter_kernel<<<tiles, kRadixThreads, 0, stream>>>(cur_k, cur_v, n, shift, mask,
                                                              buf.hist, buf.hist_scan, tiles,
                                                              out_k, out_v);
    TSD_LAUNCH_CHECK();
    cur_k = out_k;
    cur_v = out_v;
  }
  *keys_out = const_cast<uint32_t*>(cur_k);
  *vals_out = const_cast<uint32_t*>(cur_v);
}

void segment_starts(const uint32_t* sorted_keys, uint64_t n, uint32_t* starts, uint32_t* d_nseg,
                    uint32_t* tile_scratch, cudaStream_t stream) {
  if (n == 0) {
    TSD_CUDA(cudaMemsetAsync(d_nseg, 0, sizeof(uint32_t), stream));
    TSD_CUDA(cudaMemsetAsync(starts, 0, sizeof(uint32_t), stream));
    return;
  }
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  uint32_t* tile_cnt = tile_scratch;
  uint32_t* tile_off = tile_scratch + tiles + 1;
  uint32_t* scratch = tile_scratch + 2 * (tiles + 1);
  heads_count_kernel<<<static_cast<unsigned>(tiles), kScanThreads, 0, stream>>>(sorted_keys, n, tile_cnt);
  TSD_LAUNCH_CHECK();
  device_exclusive_scan(tile_cnt, tile_off, tiles, scratch, d_nseg, stream);
  heads_write_kernel<<<static_cast<unsigned>(tiles), kScanThreads, 0, stream>>>(sorted_keys, n, tile_off,
                                                                                starts, d_nseg);
  TSD_LAUNCH_CHECK();
}

}  // namespace tsd
