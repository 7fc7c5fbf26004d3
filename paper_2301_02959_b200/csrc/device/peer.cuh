// Peer-memory (NVLink P2P) exchange for U > 1 ranks on one NVSwitch node.
//
// Instead of staging rows through NCCL send/recv buffers, each server
//   1. pulls its requesters' request lists (local row id, output position)
//      straight out of their HBM (coalesced peer loads),
//   2. gathers the requested rows from its own shard and STORES them directly
//      into each requester's unpooled output (peer stores over NVLink), fused
//      with the requester's share of the loss partial sums;
// and in backward the segment-reduce kernel LOADS remote gradient rows
// directly from the requesters' gradient buffers.  A remote occurrence costs
// one local row read + one NVLink row transfer per direction, versus three
// HBM round trips plus the NCCL copy in the staged path.
//
// Peer buffers are CUDA-IPC mapped (one process per GPU).  User buffers are
// exported by allocation base + offset and opened once per allocation
// (cached), so steady-state steps do no IPC work.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <map>
#include <vector>

namespace tsd {

constexpr int kMaxPeerRanks = 8;  // P2P mode: one NVSwitch node

struct IpcExport {
  cudaIpcMemHandle_t handle;  // 64 B
  uint64_t offset;            // ptr - allocation base
  uint64_t base_id;           // base address in the exporting process (cache key)
};
static_assert(sizeof(IpcExport) == 80, "IpcExport is part of the all-gather payload");

// Export of the allocation containing `ptr`.
IpcExport export_pointer(const void* ptr);
// In-process export (ranks that are threads of one process, group.cuh): the
// raw device address; PeerMappings in direct mode hands it back unchanged.
IpcExport direct_export(const void* ptr);

// Per-peer cache of opened IPC allocations.
class PeerMappings {
 public:
  // Device pointer (valid in this process) for a peer's export.
  void* open(int peer, const IpcExport& e);
  // Drops the mapping of a peer allocation that moved (no-op if absent).
  void close(int peer, const IpcExport& e);
  void close_all();
  void set_direct(bool direct) { direct_ = direct; }
  bool direct() const { return direct_; }
  ~PeerMappings() { close_all(); }

 private:
  struct Mapping {
    cudaIpcMemHandle_t handle;
    void* base;
  };
  std::map<std::pair<int, uint64_t>, Mapping> opened_;  // (peer, base_id) -> mapping
  uint64_t opens_ = 0, reopens_ = 0;
  bool direct_ = false;
};

// Request lists a server pulls: for each source rank, a run of `count`
// entries starting at `src_off` in that rank's (ids, pos) arrays, written to
// [dst_off, dst_off + count) of the local recv arrays.
struct PullSeg {
  const uint32_t* ids;
  const uint32_t* pos;
  uint64_t src_off;
  uint64_t dst_off;
  uint64_t count;
};
struct PullTable {
  PullSeg seg[2 * kMaxPeerRanks];
  int nseg;
  uint64_t total;
};

void launch_pull_requests(const PullTable& t, uint32_t* recv_ids, uint32_t* recv_pos,
                          cudaStream_t stream);

// Serve: for every requester (grid.y), rows W[recv_ids[r]] for r in its
// recv range are stored into that requester's output at recv_pos[r]; the
// block's partial sum of squares goes to the requester's remote-loss slot
// [server][block].
struct ServeTarget {
  float* out;          // requester's unpooled output (peer pointer)
  double* loss_slots;  // requester's loss_remote + server * serve_grid (peer pointer)
  uint64_t r_begin;
  uint64_t r_end;
};
struct ServeTable {
  ServeTarget t[kMaxPeerRanks];
  int n;
};

// Loss-slot stride per requester (the largest serve grid); the grid used is
// serve_blocks() <= kServeGrid, fixed per process, so unused slots stay zero.
constexpr unsigned kServeGrid = 512;
unsigned serve_blocks();  // blocks per requester (TIERSHARD_SERVE_BLOCKS, default 96)

// Remote gradient rows pulled into local HBM: dst[r] = src[s(r)][pos[r]]
// where s(r) is the source whose range [src_start[s], src_start[s+1])
// holds r.  NVLink-bandwidth-bound gather, run on the comm stream beside the
// dedup sort so the segment kernels then read only local memory.
struct PullGrads {
  const float* src[kMaxPeerRanks];
  uint32_t src_start[kMaxPeerRanks + 1];
  int nsrc;
};
void launch_pull_grads(const PullGrads& pg, const uint32_t* recv_pos, uint64_t count, float* dst,
                       uint32_t dim, cudaStream_t stream);

// Push: the requester STORES the gradient rows of its remote occurrences
// into the servers' receive buffers (NVLink stores, fire-and-forget; peer
// stores sustain ~700 GB/s with one block per SM where peer loads need four).
// Run k moves `count` rows: row j comes from grad[order[src_begin + j]] and
// lands at dst + j * dim (dst = the server's receive buffer at this
// requester's slot).
struct PushRun {
  uint64_t src_begin;
  uint64_t count;
  float* dst;
};
struct PushTable {
  PushRun run[2 * kMaxPeerRanks];
  uint64_t run_start[2 * kMaxPeerRanks + 1];
  int n;
};
void launch_push_grads(const PushTable& t, const uint32_t* order, const float* grad, uint32_t dim,
                       cudaStream_t stream);

void launch_serve_rows(const float* weights, const uint32_t* recv_ids, const uint32_t* recv_pos,
                       const ServeTable& st, uint32_t dim, cudaStream_t stream);

// Device-side rendezvous over peer memory (one process per GPU): rank `me`
// stores `value` into slot [me] of every peer's flag mailbox (release,
// system scope) and one warp spins until every peer has stored it into its
// own mailbox (acquire).  Work queued before it on the stream, on every
// rank, completes before work queued after it -- the ordering of the NCCL
// 1-int all-reduce it replaces, with one 32-thread block instead of NCCL's
// grid and no host involvement.  `value` increases by one per rendezvous.
// Mailboxes have kFlagChannels independent channels (one per stream that
// runs rendezvous, so two streams' sequence numbers never interleave in one
// slot): channel c of rank p is peer_flags[p] + c * kMaxPeerRanks.
constexpr int kFlagChannels = 3;
struct FlagBarrier {
  uint64_t* peer_flags[kMaxPeerRanks];  // each rank's mailbox (ours at [me])
  int n;
  int me;
};
void launch_flag_barrier(const FlagBarrier& b, int channel, uint64_t value, cudaStream_t stream);

// All-gather through peer mailboxes: `bytes` (a multiple of 4) from `src`
// are stored at offset `offset` of every other rank's mailbox (one block;
// the flag rendezvous that follows publishes them).
struct MailboxPut {
  uint8_t* peer_box[kMaxPeerRanks];
  int n;
  int me;
};
void launch_mailbox_put(const MailboxPut& m, const uint8_t* src, size_t bytes, size_t offset,
                        cudaStream_t stream);

}  // namespace tsd
