// ts_sampler_*: GPU workload sampler for throughput
// runs where host materialization dominates (C4/C5: ~11 s per iteration on
// one core at C4).
//
// The reference's Workload::materialize_iteration (/root/reference/proj/src/
// simulator.cpp:54-71) draws, for every sample s of an iteration, a length
// Poisson(L) and then L alias draws (rng.cpp:15-115), all from ONE sequential
// SplitMix64 stream seeded with derive_seed(seed, iteration).  A sequential
// stream does not parallelise, so here every sample gets its own SplitMix64
// stream seeded with mix64(derive_seed(seed, iteration) ^ mix64(s + kSalt))
// and follows the reference's per-sample procedure on it exactly:
//   * the same Poisson algorithms (multiplication below mean 10, Hormann's
//     PTRD at and above), with the device's log / lgamma;
//   * the same alias-table draw (column = high half of u64 x n, coin = top 53
//     bits), on the reference's own table, built on the host and uploaded.
// The output is therefore distributed exactly as the reference's workload
// (same per-sample law, independent samples) but is not the same stream: it
// is for throughput runs only.  Host materialization stays the bit-exact path.
//
// Parallelism: SplitMix64 is counter-based (draw k of a stream seeded x is
// mix64(x + (k - 1) * golden)), so after one thread per sample runs the
// Poisson draw and records its stream position, a warp per sample fills the
// sample's rows with every lane jumping straight to its own draws.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "primitives.cuh"

namespace tsd {
namespace {

constexpr int kThreads = 256;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kSampleSalt = 0x53616d706c65ull;  // "Sample"

struct AliasEntry {
  double prob;
  uint32_t alias;
  uint32_t pad;
};

struct Stream {  // SplitMix64 (include/tiershard/rng.hpp)
  uint64_t state;
  __device__ __forceinline__ uint64_t next_u64() {
    state += kGolden;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  __device__ __forceinline__ double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
};

__device__ uint32_t poisson_dev(Stream& rng, double mean) {
  if (!(mean > 0.0)) return 0;
  if (mean < 10.0) {  // multiplication method (rng.cpp poisson_inversion)
    const double limit = exp(-mean);
    uint32_t k = 0;
    double prod = rng.next_double();
    while (prod > limit) {
      ++k;
      prod *= rng.next_double();
    }
    return k;
  }
  // PTRD (rng.cpp poisson_ptrd)
  const double smu = sqrt(mean);
  const double b = 0.931 + 2.53 * smu;
  const double a = -0.059 + 0.02483 * b;
  const double inv_alpha = 1.1239 + 1.1328 / (b - 3.4);
  const double v_r = 0.9277 - 3.6224 / (b - 2.0);
  for (;;) {
    const double u = rng.next_double() - 0.5;
    const double v = rng.next_double();
    const double us = 0.5 - fabs(u);
    const double k = floor((2.0 * a / us + b) * u + mean + 0.43);
    if (us >= 0.07 && v <= v_r) return static_cast<uint32_t>(k);
    if (k < 0.0 || (us < 0.013 && v > us)) continue;
    if (log(v * inv_alpha / (a / (us * us) + b)) <= k * log(mean) - mean - lgamma(k + 1.0)) {
      return static_cast<uint32_t>(k);
    }
  }
}

__global__ void __launch_bounds__(kThreads)
sample_lengths_kernel(uint64_t iter_seed, uint64_t sample_begin, uint32_t samples, double mean,
                      uint32_t* __restrict__ counts, uint64_t* __restrict__ states) {
  const uint32_t s = blockIdx.x * kThreads + threadIdx.x;
  if (s >= samples) return;
  Stream rng{mix64(iter_seed ^ mix64(sample_begin + s + kSampleSalt))};
  counts[s] = poisson_dev(rng, mean);
  states[s] = rng.state;  // stream position after the length draw
}

__global__ void __launch_bounds__(kThreads)
sample_rows_kernel(const uint64_t* __restrict__ states, const uint32_t* __restrict__ offsets,
                   const uint32_t* __restrict__ counts, uint32_t samples, const AliasEntry* __restrict__ table,
                   uint64_t n_rows, uint32_t* __restrict__ rows, uint64_t* __restrict__ offsets64) {
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5;
  for (uint64_t s = gwarp; s < samples; s += nwarps) {
    const uint64_t st = states[s];
    const uint32_t off = offsets[s], cnt = counts[s];
    if (offsets64 && lane == 0) {
      offsets64[s] = off;
      if (s + 1 == samples) offsets64[samples] = static_cast<uint64_t>(off) + cnt;
    }
    for (uint32_t j = lane; j < cnt; j += 32) {
      // draws 2j+1 (column) and 2j+2 (coin) after the recorded position
      const uint64_t u1 = mix64(st + (2ull * j) * kGolden);
      const uint64_t u2 = mix64(st + (2ull * j + 1) * kGolden);
      const uint64_t column = __umul64hi(u1, n_rows);
      const double coin = static_cast<double>(u2 >> 11) * 0x1.0p-53;
      const AliasEntry e = table[column];
      rows[off + j] = coin < e.prob ? static_cast<uint32_t>(column) : e.alias;
    }
  }
}

}  // namespace
}  // namespace tsd

struct ts_sampler {
  int device = 0;
  uint64_t n_rows = 0;
  double mean = 0.0;
  uint64_t seed = 0;
  tsd::AliasEntry* d_table = nullptr;
  uint32_t* d_counts = nullptr;
  uint32_t* d_offsets = nullptr;
  uint64_t* d_states = nullptr;
  uint32_t* d_scratch = nullptr;
  uint32_t* d_total = nullptr;
  uint32_t cap_samples = 0;
  cudaStream_t stream = nullptr;

  void free_step() {
    cudaFree(d_counts);
    cudaFree(d_offsets);
    cudaFree(d_states);
    cudaFree(d_scratch);
    d_counts = d_offsets = d_scratch = nullptr;
    d_states = nullptr;
    cap_samples = 0;
  }
  void destroy() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    free_step();
    cudaFree(d_table);
    cudaFree(d_total);
    if (stream) cudaStreamDestroy(stream);
  }
};

extern "C" {

ts_status ts_sampler_create(ts_sampler** out, int device, uint64_t n_rows, const double* alias_prob,
                            const uint32_t* alias_index, double expected_length, uint64_t seed) {
  return tsd::guarded([&] {
    using namespace tsd;
    if (!out || !n_rows || !alias_prob || !alias_index) fail(TS_ERR_CONFIG, "ts_sampler_create: null argument");
    *out = nullptr;
    if (n_rows >= 0xFFFFFFFFull) fail(TS_ERR_VALIDATION, "sampler: need rows < 2^32 - 1");
    if (!(expected_length > 0.0) || !std::isfinite(expected_length)) {
      fail(TS_ERR_VALIDATION, "workload: total expected length must be positive");
    }
    use_device(device);
    auto s = std::make_unique<ts_sampler>();
    s->device = device;
    s->n_rows = n_rows;
    s->mean = expected_length;
    s->seed = seed;
    try {
      TSD_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
      std::vector<AliasEntry> t(n_rows);
      for (uint64_t i = 0; i < n_rows; ++i) t[i] = AliasEntry{alias_prob[i], alias_index[i], 0};
      TSD_CUDA(dev_alloc(&s->d_table, sizeof(AliasEntry) * n_rows));
      TSD_CUDA(cudaMemcpyAsync(s->d_table, t.data(), sizeof(AliasEntry) * n_rows, cudaMemcpyHostToDevice,
                               s->stream));
      TSD_CUDA(dev_alloc(&s->d_total, sizeof(uint32_t)));
      TSD_CUDA(cudaStreamSynchronize(s->stream));
    } catch (...) {
      s->destroy();
      throw;
    }
    *out = s.release();
  });
}

ts_status ts_sampler_iteration(ts_sampler* s, uint32_t iteration, uint64_t sample_begin, uint32_t samples,
                               uint32_t* d_rows, uint64_t rows_capacity, uint64_t* d_offsets,
                               uint64_t* occurrences, void* stream) {
  return tsd::guarded([&] {
    using namespace tsd;
    if (!s || !occurrences || (samples && !d_rows)) fail(TS_ERR_CONFIG, "ts_sampler_iteration: null argument");
    TSD_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
    *occurrences = 0;
    if (samples == 0) {
      if (d_offsets) TSD_CUDA(cudaMemsetAsync(d_offsets, 0, sizeof(uint64_t), st));
      return;
    }
    if (samples > s->cap_samples) {
      TSD_CUDA(cudaStreamSynchronize(st));
      s->free_step();
      TSD_CUDA(dev_alloc(&s->d_counts, sizeof(uint32_t) * samples));
      TSD_CUDA(dev_alloc(&s->d_offsets, sizeof(uint32_t) * samples));
      TSD_CUDA(dev_alloc(&s->d_states, sizeof(uint64_t) * samples));
      TSD_CUDA(dev_alloc(&s->d_scratch, sizeof(uint32_t) * (scan_scratch_elems(samples) + 8)));
      s->cap_samples = samples;
    }
    // derive_seed(seed, iteration) (include/tiershard/hashing.hpp:40-42)
    const uint64_t iter_seed = mix64(s->seed ^ mix64(static_cast<uint64_t>(iteration) + 1));
    sample_lengths_kernel<<<ceil_div(samples, kThreads), kThreads, 0, st>>>(iter_seed, sample_begin, samples,
                                                                         s->mean, s->d_counts, s->d_states);
    TSD_LAUNCH_CHECK();
    device_exclusive_scan(s->d_counts, s->d_offsets, samples, s->d_scratch, s->d_total, st);
    uint32_t total = 0;
    TSD_CUDA(cudaMemcpyAsync(&total, s->d_total, sizeof(total), cudaMemcpyDeviceToHost, st));
    TSD_CUDA(cudaStreamSynchronize(st));
    if (total > rows_capacity) {
      fail(TS_ERR_VALIDATION, "sampler: " + std::to_string(total) + " occurrences exceed the row capacity " +
                                  std::to_string(rows_capacity));
    }
    const unsigned grid = std::max(1u, std::min<unsigned>(ceil_div(samples, kThreads / 32), 8 * sm_count()));
    sample_rows_kernel<<<grid, kThreads, 0, st>>>(s->d_states, s->d_offsets, s->d_counts, samples, s->d_table,
                                                  s->n_rows, d_rows, d_offsets);
    TSD_LAUNCH_CHECK();
    *occurrences = total;
  });
}

ts_status ts_sampler_destroy(ts_sampler* s) {
  return tsd::guarded([&] {
    if (!s) return;
    s->destroy();
    delete s;
  });
}

}  // extern "C"
