// Device-wide scan, stable LSD radix sort and segment-start compaction
// (declarations and design notes in primitives.cuh).
#include <atomic>
#include <cstdlib>
#include <string>

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
// onesweep radix sort: one global histogram for every pass, then one kernel
// per pass that ranks its tile, finds the tile's per-digit prefix with a
// decoupled look-back over earlier tiles, and scatters.  Each pass reads the
// pairs once and writes them once (the classic hist + scan + scatter pass
// reads the keys twice and scans 256 x tiles counts).
// ---------------------------------------------------------------------------

// Lanes of the warp whose digit equals mine (warp multi-split by one ballot
// per digit bit — cheaper than __match_any_sync on sm_100).  Lanes with
// valid == false match nobody and get 0.
__device__ __forceinline__ unsigned digit_peers(uint32_t d, bool valid, int bits) {
  unsigned peers = __ballot_sync(0xFFFFFFFFu, valid);
  for (int b = 0; b < bits; ++b) {
    const bool bit = (d >> b) & 1u;
    const unsigned ones = __ballot_sync(0xFFFFFFFFu, bit);
    peers &= bit ? ones : ~ones;
  }
  return valid ? peers : 0u;
}

// True when every lane of the warp is valid and holds the same digit (the
// common case in the high-order passes of Zipf-skewed row ids).
__device__ __forceinline__ bool warp_uniform(uint32_t d, bool valid) {
  const uint32_t d0 = __shfl_sync(0xFFFFFFFFu, d, 0);
  return __all_sync(0xFFFFFFFFu, valid && d == d0);
}

constexpr uint64_t kFlagAgg = 1ull << 62;   // tile-local count published
constexpr uint64_t kFlagInc = 2ull << 62;   // inclusive prefix published
constexpr uint64_t kCountMask = (1ull << 62) - 1;

// Digit width of a sort: 8 bits (256 bins), or 9 bits (512 bins) when that
// saves a pass (25..27-bit keys: 3 passes instead of 4).
__device__ __forceinline__ int pass_bits(int key_bits, int pass, int digit_bits) {
  const int left = key_bits - digit_bits * pass;
  return left < digit_bits ? left : digit_bits;
}

// Digit histograms of every pass from ONE read of the keys.  Warps whose
// digits all agree add 32 at once; otherwise plain shared atomics (few
// conflicts when digits are spread).
template <int BINS>
__global__ void __launch_bounds__(kRadixThreads)
onesweep_hist_kernel(const uint32_t* __restrict__ keys, uint64_t n, int key_bits, int passes,
                     uint32_t* __restrict__ ghist) {
  constexpr int DIGIT_BITS = BINS == 512 ? 9 : 8;
  __shared__ uint32_t s_h[kMaxRadixPasses][BINS];
  for (int p = 0; p < passes; ++p) {
    for (int b = threadIdx.x; b < BINS; b += kRadixThreads) s_h[p][b] = 0;
  }
  __syncthreads();
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kRadixTile;
  const unsigned lane = threadIdx.x & 31u;
  uint32_t key[kRadixItems];
#pragma unroll
  for (int k = 0; k < kRadixItems; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * kRadixThreads + threadIdx.x;
    key[k] = i < n ? __ldg(keys + i) : 0u;
  }
  for (int p = 0; p < passes; ++p) {
    const uint32_t mask = (1u << pass_bits(key_bits, p, DIGIT_BITS)) - 1u;
#pragma unroll
    for (int k = 0; k < kRadixItems; ++k) {
      const bool valid = base + static_cast<uint64_t>(k) * kRadixThreads + threadIdx.x < n;
      const uint32_t d = (key[k] >> (DIGIT_BITS * p)) & mask;
      if (warp_uniform(d, valid)) {
        if (lane == 0) atomicAdd(&s_h[p][d], 32u);
      } else if (valid) {
        atomicAdd(&s_h[p][d], 1u);
      }
    }
  }
  __syncthreads();
  for (int p = 0; p < passes; ++p) {
    for (int b = threadIdx.x; b < BINS; b += kRadixThreads) {
      if (s_h[p][b]) atomicAdd(ghist + p * BINS + b, s_h[p][b]);
    }
  }
}

// Exclusive scan of each pass's digit totals (one block per pass; thread t
// owns the BINS/256 consecutive digits t*DPT ..).
template <int BINS>
__global__ void __launch_bounds__(kRadixThreads)
onesweep_offsets_kernel(const uint32_t* __restrict__ ghist, uint32_t* __restrict__ goff) {
  constexpr int DPT = BINS / kRadixThreads;
  __shared__ uint32_t s_warp[kRadixThreads / 32 + 1];
  const int p = blockIdx.x;
  uint32_t v[DPT], sum = 0;
#pragma unroll
  for (int k = 0; k < DPT; ++k) {
    v[k] = ghist[p * BINS + threadIdx.x * DPT + k];
    sum += v[k];
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan<kRadixThreads>(sum, s_warp, &total);
#pragma unroll
  for (int k = 0; k < DPT; ++k) {
    goff[p * BINS + threadIdx.x * DPT + k] = run;
    run += v[k];
  }
}

__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Shared memory of one pass (dynamic: 52 KB at 512 bins).
template <int BINS>
struct PassSmem {
  uint32_t keys[kRadixTile];
  uint32_t vals[kRadixTile];
  uint32_t run[kRadixWarps][BINS];
  uint32_t tile_excl[BINS];
  uint32_t gbase[BINS];
  uint32_t warp_scan[kRadixThreads / 32 + 1];
  uint32_t tile;
};

template <int BINS, int kWindow>
#ifndef TSD_RADIX_MINB
#define TSD_RADIX_MINB 3
#endif
__global__ void __launch_bounds__(kRadixThreads, TSD_RADIX_MINB)
onesweep_pass_kernel(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                     uint64_t n, int shift, int bits, const uint32_t* __restrict__ goff,
                     uint64_t* __restrict__ status, uint32_t* __restrict__ tile_counter,
                     uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
  constexpr int DPT = BINS / kRadixThreads;  // digits per thread (consecutive)
  extern __shared__ __align__(16) uint8_t smem_raw[];
  PassSmem<BINS>& sm = *reinterpret_cast<PassSmem<BINS>*>(smem_raw);

  const uint32_t mask = (1u << bits) - 1u;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  // Dynamic tile ids in launch order: every predecessor of a tile was
  // scheduled before it, so the look-back below always makes progress.
  if (threadIdx.x == 0) sm.tile = atomicAdd(tile_counter, 1u);
#pragma unroll
  for (int w = 0; w < kRadixWarps; ++w) {
#pragma unroll
    for (int k = 0; k < DPT; ++k) sm.run[w][threadIdx.x * DPT + k] = 0;
  }
  __syncthreads();
  const uint32_t tile = sm.tile;
  const uint64_t tile_base = static_cast<uint64_t>(tile) * kRadixTile;

  uint32_t k[kRadixItems], v[kRadixItems], rank[kRadixItems];
  const uint64_t sub_base = tile_base + static_cast<uint64_t>(warp) * kRadixSubTile;
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint64_t i = sub_base + static_cast<uint64_t>(r) * 32 + lane;
    const bool valid = i < n;
    k[r] = valid ? __ldg(keys_in + i) : 0u;
    v[r] = valid ? (vals_in ? __ldg(vals_in + i) : static_cast<uint32_t>(i)) : 0u;
  }
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const bool valid = sub_base + static_cast<uint64_t>(r) * 32 + lane < n;
    const uint32_t d = (k[r] >> shift) & mask;
    if (warp_uniform(d, valid)) {
      rank[r] = sm.run[warp][d] + lane;
      __syncwarp();
      if (lane == 0) sm.run[warp][d] += 32u;
    } else {
      const unsigned peers = digit_peers(d, valid, bits);
      rank[r] = valid ? sm.run[warp][d] + __popc(peers & lt) : 0u;
      __syncwarp();
      if (valid && (peers & lt) == 0) sm.run[warp][d] += __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();

  // Per digit (thread t: digits t*DPT ..): tile count, warp prefix, look-back.
  uint32_t count[DPT], sum = 0;
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const uint32_t d = threadIdx.x * DPT + q;
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      const uint32_t t = sm.run[w][d];
      sm.run[w][d] = c;
      c += t;
    }
    count[q] = c;
    sum += c;
  }
  uint64_t excl[DPT];
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const uint32_t d = threadIdx.x * DPT + q;
    uint64_t* my = status + static_cast<uint64_t>(tile) * BINS + d;
    excl[q] = 0;
    if (tile == 0) {
      st_relaxed_u64(my, kFlagInc | count[q]);
    } else {
      st_relaxed_u64(my, kFlagAgg | count[q]);
    }
  }
  if (tile != 0) {
#pragma unroll
    for (int q = 0; q < DPT; ++q) {
      const uint32_t d = threadIdx.x * DPT + q;
      // Windowed look-back: kWindow predecessor words in flight at once, then
      // consumed nearest-first until an inclusive prefix is found; a
      // not-yet-published word restarts the window at that tile.  Measured
      // at C2 (4.2M pairs, 4 x 8-bit passes): window 1 / 2 / 4 / 8 / 16 / 32
      // -> 0.223 / 0.218 / 0.217 / 0.230 / 0.286 / 0.399 ms per sort
      // (larger windows spill under the 3-blocks/SM register cap); default 4
      // (TIERSHARD_LOOKBACK).
      int64_t p = static_cast<int64_t>(tile) - 1;
      bool done = false;
      while (!done) {
        uint64_t sw[kWindow];
#pragma unroll
        for (int w = 0; w < kWindow; ++w) {
          sw[w] = p - w >= 0 ? ld_relaxed_u64(status + static_cast<uint64_t>(p - w) * BINS + d) : kFlagInc;
        }
        int used = 0;
#pragma unroll
        for (int w = 0; w < kWindow; ++w) {
          if (done || used != w) break;
          const uint64_t flag = sw[w] & ~kCountMask;
          if (flag == 0) break;  // not ready: re-poll from here
          excl[q] += sw[w] & kCountMask;
          done = flag == kFlagInc;
          ++used;
        }
        p -= used;
      }
      st_relaxed_u64(status + static_cast<uint64_t>(tile) * BINS + d, kFlagInc | (excl[q] + count[q]));
    }
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan<kRadixThreads>(sum, sm.warp_scan, &total);
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const uint32_t d = threadIdx.x * DPT + q;
    sm.tile_excl[d] = run;
    sm.gbase[d] = goff[d] + static_cast<uint32_t>(excl[q]);
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) sm.run[w][d] += run;
    run += count[q];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint64_t i = sub_base + static_cast<uint64_t>(r) * 32 + lane;
    if (i < n) {
      const uint32_t dd = (k[r] >> shift) & mask;
      const uint32_t pos = sm.run[warp][dd] + rank[r];
      sm.keys[pos] = k[r];
      sm.vals[pos] = v[r];
    }
  }
  __syncthreads();
  const uint64_t left = n - tile_base;
  const uint32_t tile_n = left < kRadixTile ? static_cast<uint32_t>(left) : kRadixTile;
  for (uint32_t j = threadIdx.x; j < tile_n; j += kRadixThreads) {
    const uint32_t kk = sm.keys[j];
    const uint32_t dd = (kk >> shift) & mask;
    const uint32_t dst = sm.gbase[dd] + (j - sm.tile_excl[dd]);
    keys_out[dst] = kk;
    vals_out[dst] = sm.vals[j];
  }
}

// ---------------------------------------------------------------------------
// segment starts
// ---------------------------------------------------------------------------

// Head flags of one warp sub-tile (512 consecutive items, 16 coalesced rounds
// of 32): bit `lane` of mask[r] is set when item base + 32r + lane starts a run.
__device__ __forceinline__ void head_masks(const uint32_t* __restrict__ keys, uint64_t n, uint64_t base,
                                           unsigned (&mask)[kScanItems], uint32_t (&key)[kScanItems]) {
  const unsigned lane = threadIdx.x & 31u;
#pragma unroll
  for (int r = 0; r < kScanItems; ++r) {
    const uint64_t i = base + static_cast<uint64_t>(r) * 32 + lane;
    key[r] = i < n ? __ldg(keys + i) : 0u;
  }
  const uint32_t before = (base > 0 && base - 1 < n) ? __ldg(keys + base - 1) : ~key[0];
#pragma unroll
  for (int r = 0; r < kScanItems; ++r) {
    const uint64_t i = base + static_cast<uint64_t>(r) * 32 + lane;
    uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, key[r], 1);
    const uint32_t last_prev_round = __shfl_sync(0xFFFFFFFFu, r == 0 ? before : key[r > 0 ? r - 1 : 0], 31);
    if (lane == 0) prev = r == 0 ? before : last_prev_round;
    const bool head = i < n && (i == 0 || key[r] != prev);
    mask[r] = __ballot_sync(0xFFFFFFFFu, head);
  }
}

__global__ void __launch_bounds__(kScanThreads)
heads_count_kernel(const uint32_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ tile_cnt) {
  __shared__ uint32_t s_cnt[kScanThreads / 32];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + static_cast<uint64_t>(warp) * 32 * kScanItems;
  unsigned mask[kScanItems];
  uint32_t key[kScanItems];
  head_masks(keys, n, base, mask, key);
  uint32_t c = 0;
#pragma unroll
  for (int r = 0; r < kScanItems; ++r) c += __popc(mask[r]);
  if (lane == 0) s_cnt[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t total = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) total += s_cnt[w];
    tile_cnt[blockIdx.x] = total;
  }
}

__global__ void __launch_bounds__(kScanThreads)
heads_write_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                   const uint32_t* __restrict__ tile_off, uint32_t* __restrict__ starts,
                   uint32_t* __restrict__ seg_keys, const uint32_t* __restrict__ d_nseg) {
  __shared__ uint32_t s_cnt[kScanThreads / 32];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + static_cast<uint64_t>(warp) * 32 * kScanItems;
  unsigned mask[kScanItems];
  uint32_t key[kScanItems];
  head_masks(keys, n, base, mask, key);
  uint32_t c = 0;
#pragma unroll
  for (int r = 0; r < kScanItems; ++r) c += __popc(mask[r]);
  if (lane == 0) s_cnt[warp] = c;
  __syncthreads();
  uint32_t pos = tile_off[blockIdx.x];
  for (unsigned w = 0; w < warp; ++w) pos += s_cnt[w];  // sub-tiles in warp order
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kScanItems; ++r) {
    if (mask[r] & (1u << lane)) {
      const uint32_t j = pos + __popc(mask[r] & lt);
      starts[j] = static_cast<uint32_t>(base + static_cast<uint64_t>(r) * 32 + lane);
      if (seg_keys) seg_keys[j] = key[r];
    }
    pos += __popc(mask[r]);
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

template <int BINS>
void radix_sort_pairs_bins(const uint32_t* keys_in, const uint32_t* vals_in, uint64_t n, int key_bits,
                           const RadixBuffers& buf, uint32_t** keys_out, uint32_t** vals_out,
                           cudaStream_t stream) {
  constexpr int DIGIT_BITS = BINS == 512 ? 9 : 8;
  const int passes = (key_bits + DIGIT_BITS - 1) / DIGIT_BITS;
  const uint32_t tiles = static_cast<uint32_t>(radix_tiles(n));
  TSD_CUDA(cudaMemsetAsync(buf.ghist, 0, sizeof(uint32_t) * kMaxRadixPasses * kMaxRadixBins, stream));
  TSD_CUDA(cudaMemsetAsync(buf.counters, 0, sizeof(uint32_t) * kMaxRadixPasses, stream));
  TSD_CUDA(cudaMemsetAsync(buf.status, 0, sizeof(uint64_t) * passes * tiles * BINS, stream));
  onesweep_hist_kernel<BINS><<<tiles, kRadixThreads, 0, stream>>>(keys_in, n, key_bits, passes, buf.ghist);
  TSD_LAUNCH_CHECK();
  onesweep_offsets_kernel<BINS><<<passes, kRadixThreads, 0, stream>>>(buf.ghist, buf.goff);
  TSD_LAUNCH_CHECK();
  static const int window = [] {
    const char* e = std::getenv("TIERSHARD_LOOKBACK");
    return e ? std::atoi(e) : 4;
  }();
  const uint32_t* cur_k = keys_in;
  const uint32_t* cur_v = vals_in;
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = DIGIT_BITS * pass;
    const int bits = key_bits - shift < DIGIT_BITS ? key_bits - shift : DIGIT_BITS;
    uint32_t* out_k = (pass & 1) ? buf.keys_b : buf.keys_a;
    uint32_t* out_v = (pass & 1) ? buf.vals_b : buf.vals_a;
    const auto launch = [&](auto kern) {
      // opt in to > 48 KB of shared memory, once per instantiation and device
      static std::atomic<uint64_t> configured{0};
      int dev = 0;
      TSD_CUDA(cudaGetDevice(&dev));
      const uint64_t bit = uint64_t{1} << (dev & 63);
      if (!(configured.load(std::memory_order_relaxed) & bit)) {
        TSD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(sizeof(PassSmem<BINS>))));
        configured.fetch_or(bit, std::memory_order_relaxed);
      }
      kern<<<tiles, kRadixThreads, sizeof(PassSmem<BINS>), stream>>>(
          cur_k, cur_v, n, shift, bits, buf.goff + pass * BINS,
          buf.status + static_cast<uint64_t>(pass) * tiles * BINS, buf.counters + pass, out_k, out_v);
    };
    if (window >= 8) launch(onesweep_pass_kernel<BINS, 8>);
    else if (window >= 4) launch(onesweep_pass_kernel<BINS, 4>);
    else if (window >= 2) launch(onesweep_pass_kernel<BINS, 2>);
    else launch(onesweep_pass_kernel<BINS, 1>);
    TSD_LAUNCH_CHECK();
    cur_k = out_k;
    cur_v = out_v;
  }
  *keys_out = const_cast<uint32_t*>(cur_k);
  *vals_out = const_cast<uint32_t*>(cur_v);
}

int radix_digit_bits(int key_bits) {
  static const bool allow9 = [] {
    const char* e = std::getenv("TIERSHARD_RADIX9");
    return !(e && std::string(e) == "0");
  }();
  // 9-bit digits only where they save a pass: 25..27 bits in 3 passes
  return allow9 && key_bits > 24 && key_bits <= 27 ? 9 : 8;
}

void radix_sort_pairs(const uint32_t* keys_in, const uint32_t* vals_in, uint64_t n, int key_bits,
                      const RadixBuffers& buf, uint32_t** keys_out, uint32_t** vals_out,
                      cudaStream_t stream) {
  // Even passes write (keys_a, vals_a), odd passes (keys_b, vals_b); the
  // caller's input is only read.
  *keys_out = buf.keys_a;
  *vals_out = buf.vals_a;
  if (n == 0) return;
  if (key_bits < 1) key_bits = 1;
  if (key_bits > 32) key_bits = 32;
  if (radix_digit_bits(key_bits) == 9) {
    radix_sort_pairs_bins<512>(keys_in, vals_in, n, key_bits, buf, keys_out, vals_out, stream);
  } else {
    radix_sort_pairs_bins<256>(keys_in, vals_in, n, key_bits, buf, keys_out, vals_out, stream);
  }
}

void segment_starts(const uint32_t* sorted_keys, uint64_t n, uint32_t* starts, uint32_t* seg_keys,
                    uint32_t* d_nseg, uint32_t* tile_scratch, cudaStream_t stream) {
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
                                                                                starts, seg_keys, d_nseg);
  TSD_LAUNCH_CHECK();
}

}  // namespace tsd
