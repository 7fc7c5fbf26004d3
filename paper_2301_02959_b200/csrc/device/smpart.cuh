// SM partitions through green contexts (CUDA driver API, reached by dlsym
// like the rest of the library's driver calls): a stream created in a
// partition runs its kernels on that partition's SMs only.  Used to give
// the exchange / dedup kernels SMs of their own beside the persistent
// HBM-bound grids (TIERSHARD_SM_SPLIT=K, see table.cu).  Device memory,
// events and stream waits work across partitions (checked by
// tools/gc_probe on B200).
#pragma once

#include <cuda_runtime.h>

namespace tsd {

struct SmPartition {
  void* green[2] = {nullptr, nullptr};  // CUgreenCtx: [0] the K-SM part, [1] the rest
  int sms[2] = {0, 0};
  bool active() const { return green[0] != nullptr; }
};

// Splits `device`'s SMs into K and the rest (K rounded by the driver to its
// granularity); fails with TS_ERR_CUDA when green contexts are unavailable.
SmPartition make_partition(int device, int k);
// A non-blocking stream of partition `part` (0: K SMs, 1: the rest).
cudaStream_t partition_stream(const SmPartition& p, int part, int priority);
void destroy_partition(SmPartition& p);

// Grid sizing: persistent grids are sized by sm_count(); with a partition
// the library sizes them for the partition the HBM kernels run on.
void set_sm_budget(int sms);

}  // namespace tsd
