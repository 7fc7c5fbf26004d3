// In-process rank group: the transport a ts_table uses when every rank of a
// U = N*W job is a host thread of ONE process (ts_group_create).  It stands
// in for NCCL where NCCL cannot go -- several ranks on one GPU (NCCL rejects
// duplicate devices) -- so the whole U > 1 peer-memory path (routing into
// request lists, serve, gradient push, replicated-row reduction) runs and is
// checked against the oracle on a single device.  Ranks may also sit on
// different GPUs of the process (rank g on any ordinal): peer pointers are
// then plain UVA pointers with peer access enabled.
//
// What it provides, and how:
//   * host all-gather (collective, blocking): a shared staging buffer and a
//     generation barrier (mutex + condition variable);
//   * device rendezvous on a stream: every rank records an event on its
//     stream, a host barrier, then every rank makes its stream wait on every
//     other rank's event.  Work queued before the rendezvous on any rank's
//     stream completes before work queued after it on every rank's stream --
//     the ordering the NCCL 1-int all-reduce gives the multi-process path.
//     Two events per rank, used alternately: a rank can run at most one
//     rendezvous ahead of the slowest (the host barrier holds it), so the
//     event another rank is waiting on is never re-recorded under it.
//   * peer pointers: exported as raw device addresses (no CUDA IPC, which
//     refuses same-process handles).
// A rendezvous that does not complete within TIERSHARD_GROUP_TIMEOUT seconds
// (default 300) fails with TS_ERR_INTERNAL and poisons the group, so a rank
// that failed cannot leave the others blocked forever.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

struct ts_group;

namespace tsd {

// Rank `rank` joins `g` on `device` (creates its rendezvous events there).
// Fails when the rank is taken or out of range.
void group_attach(ts_group* g, uint32_t rank, int device);
void group_detach(ts_group* g, uint32_t rank);
uint32_t group_size(const ts_group* g);

// Host barrier over all ranks.
void group_wait(ts_group* g);
// all[p*bytes .. (p+1)*bytes) = rank p's `mine`, on every rank.
void group_allgather(ts_group* g, uint32_t rank, const void* mine, size_t bytes, void* all);
// Device rendezvous on `stream` (see above).
void group_barrier(ts_group* g, uint32_t rank, cudaStream_t stream);
// Marks the group unusable (a rank failed): every pending and later
// rendezvous fails at once.
void group_poison(ts_group* g);

}  // namespace tsd
