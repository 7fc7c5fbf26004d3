// C-ABI entry points shared by every handle: error reporting, build info,
// device discovery (include/tiershard_b200.h).
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cstring>
#include <string>

#include "common.cuh"

namespace tsd {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void use_device(int device) {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(TS_ERR_NO_DEVICE, "no CUDA device available (the tiershard-b200 device path has no CPU "
                           "fallback)");
  }
  if (device < 0 || device >= count) {
    fail(TS_ERR_CONFIG, "CUDA device " + std::to_string(device) + " out of range (" +
                            std::to_string(count) + " visible)");
  }
  TSD_CUDA(cudaSetDevice(device));
  int major = 0;
  TSD_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major != 10) {
    fail(TS_ERR_NO_DEVICE, "device " + std::to_string(device) +
                               " is not an sm_100 (Blackwell) part; this build targets sm_100a only");
  }
}

namespace {
std::atomic<int> g_sm_budget{0};
}

void set_sm_budget(int sms) { g_sm_budget.store(sms, std::memory_order_relaxed); }

int sm_count() {
  const int budget = g_sm_budget.load(std::memory_order_relaxed);
  if (budget > 0) return budget;
  int dev = 0, n = 0;
  TSD_CUDA(cudaGetDevice(&dev));
  TSD_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

}  // namespace tsd

extern "C" {

const char* ts_last_error(void) { return tsd::g_last_error.c_str(); }

int ts_abi_version(void) { return TS_ABI_VERSION; }

const char* ts_build_info(void) {
  static const std::string info = [] {
    int rt = 0;
    cudaRuntimeGetVersion(&rt);
    return std::string("tiershard-b200 abi=") + std::to_string(TS_ABI_VERSION) +
           " arch=sm_100a cudart=" + std::to_string(rt) +
           " nccl_headers=" + std::to_string(NCCL_VERSION_CODE);
  }();
  return info.c_str();
}

ts_status ts_device_count(int* count) {
  return tsd::guarded([&] {
    if (!count) tsd::fail(TS_ERR_CONFIG, "ts_device_count: null output");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

ts_status ts_nccl_unique_id(void* out128) {
  return tsd::guarded([&] {
    if (!out128) tsd::fail(TS_ERR_CONFIG, "ts_nccl_unique_id: null output");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
      tsd::fail(TS_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    }
    std::memcpy(out128, &id, sizeof(id));
  });
}

uint64_t ts_kernel_launches(void) { return tsd::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
