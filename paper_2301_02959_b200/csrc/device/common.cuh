// Shared device/host plumbing for the sm_100a path: error capture at the
// C-ABI boundary, the placement mixer, and small warp/bit helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "tiershard_b200.h"

namespace tsd {

// Internal failure carrying the C-ABI status it maps to.
struct Failure : std::runtime_error {
  ts_status status;
  Failure(ts_status st, const std::string& msg) : std::runtime_error(msg), status(st) {}
};

void set_last_error(const std::string& msg);

[[noreturn]] inline void fail(ts_status st, const std::string& msg) { throw Failure(st, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    const ts_status st = (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
                             ? TS_ERR_NO_DEVICE
                             : TS_ERR_CUDA;
    fail(st, std::string("CUDA error in ") + what + " (" + file + ":" + std::to_string(line) +
                 "): " + cudaGetErrorString(e));
  }
}

// Counts every kernel launch of the library (ts_kernel_launches()).
void note_launch();

#define TSD_CUDA(call) ::tsd::cuda_check((call), #call, __FILE__, __LINE__)
#define TSD_LAUNCH_CHECK()                                                   \
  do {                                                                       \
    ::tsd::note_launch();                                                    \
    ::tsd::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
  } while (0)

// Selects `device` after verifying it exists and is an sm_100-class part.
void use_device(int device);

// Runs `body`, mapping exceptions to a ts_status + thread-local message.
template <typename Body>
ts_status guarded(Body&& body) {
  try {
    body();
    return TS_OK;
  } catch (const Failure& f) {
    set_last_error(f.what());
    return f.status;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return TS_ERR_INTERNAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TS_ERR_INTERNAL;
  }
}

// Device copy of tiershard::mix64 (include/tiershard/hashing.hpp).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Initial weight contract (oracle/restate.h orc_init_weight).
__host__ __device__ __forceinline__ float init_weight(uint64_t seed, uint64_t canon, uint32_t d,
                                                      uint32_t dim) {
  const uint64_t u = mix64(seed ^ mix64(canon * static_cast<uint64_t>(dim) + d));
  const int32_t v = static_cast<int32_t>(u >> 40) - (1 << 23);
  return static_cast<float>(v) * (0.01f / 8388608.0f);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// 128-bit read-only load that bypasses L1 allocation (streamed operands).
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// 128-bit store with evict-first L2 policy (outputs not re-read soon).
__device__ __forceinline__ void stg_stream(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

inline unsigned ceil_div(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// cudaMalloc rounded up to whole 2 MiB pages for anything over 1 MiB.
// Measured on B200: a 2.0003 GiB buffer whose size was not a 2 MiB multiple
// made every NVLink access to it (peer stores into it, peer loads from it)
// about 2x slower than the same buffer rounded up (U = 4 host-buffer step
// 5.9 -> 3.9 ms), consistent with the allocation falling back to small pages.
inline cudaError_t dev_alloc(void** p, uint64_t bytes) {
  constexpr uint64_t kPage = uint64_t{2} << 20;
  if (bytes > (kPage >> 1)) bytes = (bytes + kPage - 1) / kPage * kPage;
  return cudaMalloc(p, bytes);
}
template <typename T>
inline cudaError_t dev_alloc(T** p, uint64_t bytes) {
  return dev_alloc(reinterpret_cast<void**>(p), bytes);
}

// Number of SMs on the current device (cached per device).
int sm_count();

}  // namespace tsd
