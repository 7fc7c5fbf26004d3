// Device-wide building blocks for the backward dedup (and the U>1 routing
// compaction): warp/block scans, a device exclusive scan, and a stable LSD
// radix sort of (u32 key, u32 value) pairs.
//
// Radix sort design (sm_100a, HBM-bound), "onesweep":
//   1. onesweep_hist    — ONE read of the keys builds the 256-bin histograms of
//                         every 8-bit pass (warp match_any aggregation);
//   2. onesweep_offsets — exclusive scan per pass -> global digit offsets;
//   3. onesweep_pass    — per pass, per 4096-item tile: stable in-tile ranking
//                         (each warp ranks its contiguous 512-item sub-tile
//                         with __match_any_sync; warps ordered by a per-digit
//                         prefix), decoupled look-back over earlier tiles for
//                         the tile's per-digit global offset (tile ids taken
//                         from an atomic counter in launch order, so the
//                         look-back always progresses), smem staging, then
//                         coalesced run write-out.  One read + one write of the
//                         pairs per pass.
// Stability: ranks follow input order inside a warp sub-tile, sub-tiles follow
// warp order, tiles follow tile order — so equal keys keep input order, which
// is what makes the segment sums deterministic (oracle/restate.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tsd {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

constexpr int kRadixThreads = 256;
// Items per thread of a radix tile (TSD_RADIX_ITEMS at build time, A/B).
#ifndef TSD_RADIX_ITEMS
#define TSD_RADIX_ITEMS 16
#endif
constexpr int kRadixItems = TSD_RADIX_ITEMS;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixSubTile = kRadixTile / kRadixWarps;  // 512 items per warp
constexpr int kRadixBins = 256;

// Scratch sizes (in u32 elements) the host must provide.
inline uint64_t scan_scratch_elems(uint64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }
inline uint64_t radix_tiles(uint64_t n) { return (n + kRadixTile - 1) / kRadixTile; }

// Exclusive scan of n u32 values in -> out (out may alias in).  `scratch`
// holds scan_scratch_elems(n) u32; the total is written to *d_total if
// d_total != nullptr.  Three launches; totals must fit in u32.
void device_exclusive_scan(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* scratch,
                           uint32_t* d_total, cudaStream_t stream);

constexpr int kMaxRadixPasses = 4;
constexpr int kMaxRadixBins = 512;  // 9-bit digits when they save a pass
// Digit width radix_sort_pairs uses for keys of `key_bits` bits (8 or 9).
int radix_digit_bits(int key_bits);

struct RadixBuffers {
  uint32_t* keys_a;    // n
  uint32_t* vals_a;    // n
  uint32_t* keys_b;    // n
  uint32_t* vals_b;    // n
  uint32_t* ghist;     // kMaxRadixPasses * kMaxRadixBins digit totals
  uint32_t* goff;      // kMaxRadixPasses * kMaxRadixBins exclusive digit offsets (goff[0..]
                       // of pass 0 are the bucket starts when one 8-bit pass sorts bucket ids)
  uint64_t* status;    // kMaxRadixPasses * radix_tiles(n) * kMaxRadixBins look-back words
  uint32_t* counters;  // kMaxRadixPasses dynamic tile counters
};

// Stable sort of n (key, value) pairs by the low `key_bits` bits of the keys
// (ceil(key_bits / 8) passes).  vals_in == nullptr means values 0..n-1.  The
// input is only read; the result pointers land in buf's a- or b-arrays.
void radix_sort_pairs(const uint32_t* keys_in, const uint32_t* vals_in, uint64_t n, int key_bits,
                      const RadixBuffers& buf, uint32_t** keys_out, uint32_t** vals_out,
                      cudaStream_t stream);

// Segment starts of sorted keys: starts[j] = first index of the j-th run of
// equal keys, starts[nseg] = n; *d_nseg receives nseg.  `flags_scratch`
// holds scan_scratch_elems(n) + radix_tiles-style tile counts (2 * n/4096+2).
// seg_keys (nullable) receives the key of every segment.
void segment_starts(const uint32_t* sorted_keys, uint64_t n, uint32_t* starts, uint32_t* seg_keys,
                    uint32_t* d_nseg, uint32_t* tile_scratch, cudaStream_t stream);
inline uint64_t segment_scratch_elems(uint64_t n) {
  return 2 * ((n + kScanTile - 1) / kScanTile) + 4 + scan_scratch_elems((n + kScanTile - 1) / kScanTile);
}

// ---------------------------------------------------------------------------
// warp / block scan helpers (inline, used by several kernels)
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t v) {
  const unsigned lane = threadIdx.x & 31u;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, off);
    if (lane >= static_cast<unsigned>(off)) v += t;
  }
  return v;
}

// Block-wide exclusive scan; all THREADS threads must call.  s_warp holds
// THREADS/32 u32.  Returns the exclusive prefix; *total gets the block sum.
template <int THREADS>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp,
                                                         uint32_t* total) {
  constexpr int kWarps = THREADS / 32;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t inc = warp_inclusive_scan(v);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < kWarps ? s_warp[lane] : 0u;
    const uint32_t winc = warp_inclusive_scan(w);
    if (lane < kWarps) s_warp[lane] = winc - w;
    if (lane == kWarps - 1) s_warp[kWarps] = winc;
  }
  __syncthreads();
  const uint32_t result = s_warp[warp] + inc - v;
  *total = s_warp[kWarps];
  __syncthreads();
  return result;
}

}  // namespace tsd
