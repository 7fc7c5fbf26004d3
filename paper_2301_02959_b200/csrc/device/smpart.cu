// Green-context SM partitions (smpart.cuh).
#include <cuda.h>
#include <dlfcn.h>

#include <string>

#include "common.cuh"
#include "smpart.cuh"

namespace tsd {
namespace {

struct Driver {
  CUresult (*get_resource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*split)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned) = nullptr;
  CUresult (*gen_desc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
  CUresult (*create)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
  CUresult (*stream_create)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
  CUresult (*destroy)(CUgreenCtx) = nullptr;
  CUresult (*device_get)(CUdevice*, int) = nullptr;
  bool ok = false;
};

const Driver& driver() {
  static const Driver d = [] {
    Driver x;
    void* h = dlopen("libcuda.so.1", RTLD_LAZY | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_LAZY);
    if (!h) return x;
    x.get_resource = reinterpret_cast<decltype(x.get_resource)>(dlsym(h, "cuDeviceGetDevResource"));
    x.split = reinterpret_cast<decltype(x.split)>(dlsym(h, "cuDevSmResourceSplitByCount"));
    x.gen_desc = reinterpret_cast<decltype(x.gen_desc)>(dlsym(h, "cuDevResourceGenerateDesc"));
    x.create = reinterpret_cast<decltype(x.create)>(dlsym(h, "cuGreenCtxCreate"));
    x.stream_create = reinterpret_cast<decltype(x.stream_create)>(dlsym(h, "cuGreenCtxStreamCreate"));
    x.destroy = reinterpret_cast<decltype(x.destroy)>(dlsym(h, "cuGreenCtxDestroy"));
    x.device_get = reinterpret_cast<decltype(x.device_get)>(dlsym(h, "cuDeviceGet"));
    x.ok = x.get_resource && x.split && x.gen_desc && x.create && x.stream_create && x.destroy && x.device_get;
    return x;
  }();
  return d;
}

void check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) fail(TS_ERR_CUDA, std::string("SM partition: ") + what + " failed (" + std::to_string(r) + ")");
}

}  // namespace

SmPartition make_partition(int device, int k) {
  const Driver& d = driver();
  if (!d.ok) fail(TS_ERR_CUDA, "SM partition: green contexts are unavailable in this driver");
  SmPartition p;
  CUdevice dev;
  check(d.device_get(&dev, device), "cuDeviceGet");
  CUdevResource all;
  check(d.get_resource(dev, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
  CUdevResource part, rest;
  unsigned n = 1;
  check(d.split(&part, &n, &all, &rest, 0, static_cast<unsigned>(k)), "cuDevSmResourceSplitByCount");
  CUdevResourceDesc dk, dr;
  check(d.gen_desc(&dk, &part, 1), "cuDevResourceGenerateDesc");
  check(d.gen_desc(&dr, &rest, 1), "cuDevResourceGenerateDesc");
  CUgreenCtx gk, gr;
  check(d.create(&gk, dk, dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
  check(d.create(&gr, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
  p.green[0] = gk;
  p.green[1] = gr;
  p.sms[0] = static_cast<int>(part.sm.smCount);
  p.sms[1] = static_cast<int>(rest.sm.smCount);
  return p;
}

cudaStream_t partition_stream(const SmPartition& p, int part, int priority) {
  CUstream s = nullptr;
  check(driver().stream_create(&s, static_cast<CUgreenCtx>(p.green[part]), CU_STREAM_NON_BLOCKING, priority),
        "cuGreenCtxStreamCreate");
  return reinterpret_cast<cudaStream_t>(s);
}

void destroy_partition(SmPartition& p) {
  for (void*& g : p.green) {
    if (g) driver().destroy(static_cast<CUgreenCtx>(g));
    g = nullptr;
  }
}

}  // namespace tsd
