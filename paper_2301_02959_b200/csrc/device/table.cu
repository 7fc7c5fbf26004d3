// ts_table_*: one rank's shard of the per-row tiered sequence-embedding table
// and its lookup (forward) / update (backward) entry points.
//
// HBM layout of rank g:
//   weights [local_rows x dim] fp32 = [DP rows 0..dp_cut) | Flex rows of slot
//   g%W | RW rows owned by g], each group in canonical order; Adagrad state
//   [local_rows] fp32; remap u32[n] + placement byte u8[n] (U > 1 only — with
//   U == 1 the local id IS the canonical index and no remap is stored).
//
// Forward (U == 1): one fused gather over all occurrences; the backward's
//   dedup sort (it needs only the ids) starts beside it on the aux stream.
// Forward (U > 1, one node, peer memory -- the default): bucket every
//   occurrence (DP / own -> local, RW -> owner, Flex -> node slot), one stable
//   counting pass compacts the remote ones per destination into request
//   lists in HBM; one NCCL all-gather of bucket starts + output export (the
//   step's single host sync); each server pulls its requesters' lists from
//   their HBM and STORES the rows into their outputs over NVLink while the
//   local rows are gathered; the dedup (entries, sort, heads) is prefetched
//   on the aux stream.
// Backward (peer memory): each requester stores the gradients of its remote
//   occurrences into the servers' fixed receive buffers (then a barrier);
//   the replicated rows' segments store their partials into the row owner's
//   receive slots (epoch-stamped), the owner reduces them in rank order,
//   updates and broadcasts; the rest are segment-reduced with the fused
//   optimizer in place.
// Staged path (no peer access, TIERSHARD_EXCHANGE=nccl): NCCL all-to-allv of
//   ids (world comm for RW, intra comm g/W for Flex) and rows, reverse
//   all-to-allv of gradients, dense DP (world) / Flex (cross comm g%W)
//   all-reduce and a dense update on every replica.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "embedding.cuh"
#include "group.cuh"
#include "primitives.cuh"
#include "layout.hpp"
#include "peer.cuh"
#include "route.cuh"
#include "smpart.cuh"

namespace tsd {
namespace {

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    fail(TS_ERR_NCCL, std::string("NCCL error in ") + what + ": " + ncclGetErrorString(r));
  }
}
#define TSD_NCCL(call) ::tsd::nccl_check((call), #call)

template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  uint64_t cap = 0;
  void ensure(uint64_t n) {
    if (n <= cap && ptr) return;
    if (ptr) TSD_CUDA(cudaFree(ptr));
    ptr = nullptr;
    // whole 2 MiB pages (dev_alloc): the spare tail becomes capacity
    constexpr uint64_t kPage = uint64_t{2} << 20;
    uint64_t bytes = sizeof(T) * std::max<uint64_t>(n, 1);
    if (bytes > (kPage >> 1)) bytes = (bytes + kPage - 1) / kPage * kPage;
    cap = bytes / sizeof(T);
    TSD_CUDA(dev_alloc(&ptr, bytes));
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

int bits_for(uint64_t max_value) {
  int b = 1;
  while (b < 32 && (uint64_t{1} << b) <= max_value) ++b;
  return b;
}

enum Phase : int {
  kPhaseRoute = 0,
  kPhaseGather,
  kPhaseExchangeFwd,
  kPhaseScatter,
  kPhaseExchangeBwd,
  kPhaseSort,
  kPhaseSegments,
  kPhaseSegmentUpdate,
  kPhaseAllReduce,
  kPhaseDenseUpdate,
  kPhaseReplicaUpdate,
  kPhaseSegmentLong,
  kPhaseRendezvous,
  kNumPhases
};

// In-process staged path (group transport): out[i] = sum of the group's
// buffers in group-rank order, the stand-in for ncclAllReduce.
struct SumSources {
  const float* src[kMaxPeerRanks];
  int n;
};
__global__ void sum_sources_kernel(float* __restrict__ out, SumSources s, uint64_t count) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    float v = s.src[0][i];
    for (int k = 1; k < s.n; ++k) v = __fadd_rn(v, s.src[k][i]);
    out[i] = v;
  }
}

__global__ void gather_scalars_kernel(const float* __restrict__ src, const uint32_t* __restrict__ idx,
                                      float* __restrict__ dst, uint64_t count) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    dst[i] = src[idx[i]];
  }
}

// U = 1 tier counts of a batch (RW, Flex, DP), for ts_table_counters: the
// forward does not bucket at U = 1, so they are counted on demand.
__global__ void count_tiers_kernel(const uint32_t* __restrict__ rows, uint64_t occ, uint64_t dp_cut,
                                   uint64_t flex_cut, unsigned long long* __restrict__ tiers) {
  unsigned long long c[3] = {0, 0, 0};
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < occ; i += stride) {
    const uint32_t r = rows[i];
    c[r < dp_cut ? 2 : (r < flex_cut ? 1 : 0)] += 1;
  }
  for (int k = 0; k < 3; ++k) {
    unsigned long long v = c[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31u) == 0 && v) atomicAdd(tiers + k, v);
  }
}

const char* const kPhaseNames[kNumPhases] = {
    "route",         "gather",         "exchange_fwd", "scatter",  "exchange_bwd",
    "dedup_sort",    "segment_starts", "segment_update", "allreduce", "dense_update",
    "replica_update", "segment_long", "rendezvous"};

}  // namespace
}  // namespace tsd

struct ts_table {
  ts_table_config cfg{};
  uint32_t U = 1, W = 1, N = 1, g = 0, slot = 0, node = 0;
  cudaStream_t stream = nullptr;  // compute stream (S)
  // TIERSHARD_SM_SPLIT=K: green-context SM partition -- the exchange (U > 1:
  // comm, rep) or dedup (U = 1: aux) streams on K SMs of their own, the
  // compute streams on the rest (grids sized for it).  allgather_bytes then
  // runs NCCL on a separate stream of the whole device.
  tsd::SmPartition smp;
  cudaStream_t nccl_st = nullptr;
  cudaStream_t dd = nullptr;  // the prefetched dedup's stream (K partition) when split, else aux
  cudaStream_t dedup_stream() const { return dd ? dd : aux; }
  cudaStream_t make_stream(int part, int priority) {
    if (smp.active()) return tsd::partition_stream(smp, part, priority);
    cudaStream_t st = nullptr;
    TSD_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, priority));
    return st;
  }
  cudaStream_t comm = nullptr;    // exchange / all-reduce stream (C), U > 1
  // U = 1: the dedup (sort + segment heads) needs only the row ids, so the
  // forward starts it on `aux` beside the gather; the backward waits for it.
  // TIERSHARD_DEDUP_IN_FORWARD=0 keeps it in the backward;
  // TIERSHARD_GATHER_BLOCKS = the gather's blocks per SM meanwhile.
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fwd0 = nullptr, ev_dedup = nullptr;
  bool dedup_in_forward = true;
  uint32_t seg_short_max = tsd::kPiece;  // tsd::short_max(U), set at creation
  bool dedup_ready = false;
  // Segments longer than seg_short_max are listed ahead of the segment
  // update (U = 1: with the dedup in the forward; U > 1: per segment range,
  // on aux) and their piece path runs on `aux` beside the short-segment
  // kernel (TIERSHARD_LONG_CONCURRENT=0 keeps both on the compute stream).
  bool long_concurrent = true;
  cudaEvent_t ev_seg0 = nullptr, ev_long = nullptr;
  tsd::SegmentScratch seg_scratch_view() const {
    tsd::SegmentScratch sc;
    sc.long_list = long_list.ptr;
    sc.long_count = long_count.ptr;
    sc.piece_off = piece_off.ptr;
    sc.partials = partials.ptr;
    sc.short_max = seg_short_max;
    return sc;
  }
  uint32_t* dd_keys = nullptr;
  uint32_t* dd_vals = nullptr;
  unsigned fwd_gather_grid = 0;
  int gather_bulk_stages = 2;  // 0 = register gather (set at creation)
  cudaEvent_t ev_ids = nullptr, ev_fwd = nullptr, ev_bwd0 = nullptr, ev_grads = nullptr,
              ev_dense = nullptr, ev_ar = nullptr;
  ncclComm_t world = nullptr, intra = nullptr, cross = nullptr;
  // in-process group transport (cfg.group): replaces the NCCL communicators
  // for the peer-memory path (group.cuh); `ready` = creation completed, so
  // destroy() may run its collective rendezvous
  ts_group* grp = nullptr;
  bool attached = false, ready = false;
  tsd::IpcExport export_ptr(const void* p) const {
    return grp ? tsd::direct_export(p) : tsd::export_pointer(p);
  }

  // shard
  uint64_t local_rows = 0, dp_rows = 0, flex_rows = 0, rw_rows = 0;
  float* d_w = nullptr;
  float* d_state = nullptr;
  uint8_t* d_dest = nullptr;
  uint32_t* d_local = nullptr;
  std::vector<uint32_t> h_local;  // canonical -> local id (U > 1)
  std::vector<uint8_t> h_dest;

  // step state
  const uint32_t* last_rows = nullptr;
  uint64_t last_occ = 0;
  float* last_out = nullptr;
  unsigned gather_grid = 0;

  tsd::DevBuf<double> loss_partials, d_loss;
  tsd::DevBuf<unsigned long long> tier_counts;  // RW, Flex, DP of this requester
  tsd::DevBuf<uint32_t> rows_dev;                // host-step staging
  tsd::DevBuf<float> host_out;                   // host-step output [max_occurrences x D]
  // pipelined host steps (ts_table_train_steps_host): second id buffer, copy
  // stream, per-buffer events, pinned loss landing area
  tsd::DevBuf<uint32_t> rows_dev2;
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
  double* h_loss_pinned = nullptr;  // host-mapped: the loss kernel writes it directly
  double* h_loss_dev = nullptr;     // its device alias
  double* loss_mirror = nullptr;    // this step's slot in it (set by the host-step loops)
  uint32_t h_loss_cap = 0;
  // dedup / sort
  tsd::DevBuf<uint32_t> keys_a, vals_a, keys_b, vals_b, ghist, goff, sort_counters;
  tsd::DevBuf<uint64_t> sort_status;
  tsd::DevBuf<uint32_t> starts, seg_keys, seg_scratch, nseg, seg_split;
  tsd::DevBuf<uint32_t> long_list, long_count, piece_off, entry_keys, entry_vals;
  tsd::DevBuf<float> partials;
  // U > 1 routing / exchange
  tsd::DevBuf<uint32_t> bucket, order, send_ids, recv_ids, bucket_start, all_counts;
  tsd::DevBuf<uint32_t> route_hist;  // per-tile bucket counts (launch_route_buckets)
  // TIERSHARD_ROUTE=sort: the peer path's route as bucket keys + radix sort
  bool route_sort = false;
  tsd::DevBuf<float> send_rows, recv_rows, dense_dp, dense_flex;
  tsd::DevBuf<uint32_t> stamp_dp, stamp_flex;  // per dense row: last epoch written (P2P)
  uint32_t epoch = 0;                          // backward steps (P2P)
  std::vector<uint32_t> h_counts;     // [U][NB] send counts of every rank
  std::vector<uint64_t> send_off, send_cnt, recv_off, recv_cnt;  // per peer (entries)
  uint64_t n_remote = 0, n_local_occ = 0, recv_total = 0, recv_before = 0;
  uint64_t last_entries = 0;
  std::array<uint64_t, 3> last_tiers{};  // RW, Flex, DP (host, after sync)

  // ---- peer-memory (NVLink P2P) exchange, U > 1 on one node ------------------
  bool p2p = false;
  tsd::PeerMappings peers;
  tsd::DevBuf<uint32_t> recv_pos;
  tsd::DevBuf<uint8_t> xfer;  // all-gather scratch [U x bytes]
  tsd::DevBuf<int32_t> barrier_buf;
  // peer-memory flag rendezvous (one process per GPU; TIERSHARD_BARRIER=nccl
  // keeps the NCCL all-reduce): mailbox of U u64 flags, exported at setup
  tsd::DevBuf<uint64_t> flag_box;
  tsd::FlagBarrier flag_barrier{};
  // per-step payload mailbox [U x step_payload_bytes] (flag mode): every
  // rank's bucket starts + output export, stored by the ranks themselves
  tsd::DevBuf<uint8_t> mbox;
  tsd::MailboxPut mbox_put{};
  bool flag_barriers = false;
  // TIERSHARD_FWD_COUNTS=mailbox: the forward's count exchange through the
  // mailboxes + a flag rendezvous, with the local gather queued before it;
  // default: the NCCL all-gather, gather after.  Measured at C2 (ms/step,
  // tools/mg_env_ab.sh): N=2 2.29 (all-gather) vs 2.32-2.45 (mailbox, 6-8
  // gather blocks/SM); N=4 3.27 vs 3.34 -- the early gather takes the SMs
  // the serve and the sort then wait for; the step is bound by the sum of
  // concurrent HBM + NVLink work, not by the exchange's latency.
  bool mailbox_counts = false;
  uint64_t barrier_seq = 0, step_barrier_seq = 0;
  // TIERSHARD_FWD=pull|serve (pull needs flag barriers or the group): the
  // requester loads its remote rows from their owners' shards over NVLink
  // (launch_pull_rows, on aux right after the route) instead of the owners
  // storing them into its output after the count exchange; the counts then
  // only feed the backward.  A rendezvous on the compute stream (channel 1)
  // after the route makes every rank's previous update visible before any
  // row is read.  Measured at C2, N=2 (ms/step): serve 2.28-2.32, pull
  // 2.58-2.65 -- the random peer LOADS reach ~205 GB/s in the step (1.12 ms
  // for 0.23 GB) where the serve's peer STORES reach ~350; a whole-batch
  // gather with the remote loads inline (launch_gather_all) was 2.40-2.44.
  // Kept as an option (tested), serve is the default.
  bool pull_forward = false;
  void forward_p2p_pull(const uint32_t* d_rows, uint64_t occ, float* d_out);
  std::vector<uint8_t> h_xfer;
  std::vector<const uint32_t*> peer_ids, peer_pos;  // peers' request lists (mapped)
  std::vector<double*> peer_loss;                   // peers' remote-loss slots (mapped)
  std::vector<const float*> peer_grad;              // peers' gradient buffers (mapped)
  std::vector<float*> peer_dense_dp, peer_dense_flex;  // peers' partial receive buffers (mapped)
  std::vector<uint32_t*> peer_stamp_dp, peer_stamp_flex;  // and their slot stamps
  std::vector<float*> peer_recv_rows;  // peers' gradient receive buffers (mapped; moved by regrow_recv)
  std::vector<uint64_t> peer_recv_cap;  // their capacities, in rows
  std::vector<tsd::IpcExport> peer_recv_export;
  uint64_t recv_regrows = 0;
  void regrow_recv(const std::vector<uint64_t>& need);
  void exchange_recv_exports();
  uint32_t per_dp = 0, per_flex = 0;  // replicated rows owned per group member
  // TIERSHARD_REPLICA_OWNER=block|interleave: which member owns (reduces,
  // updates, broadcasts) replicated row r -- r / per, or r % members
  bool replica_interleave = true;
  // TIERSHARD_PUSH_ROTATE=0: the gradient push visits servers in rank order
  bool push_rotate = true;
  std::vector<float*> peer_w, peer_state;           // peers' shards (mapped)
  tsd::IpcExport my_export{};                       // staging for the step payload
  bool export_in_slot = false;                      // my_export is in our payload slot
  uint64_t remote_loss_slots = 0;                   // U * kServeGrid
  // schedule knobs (env, read at creation; defaults = fastest measured):
  //   TIERSHARD_REPLICA=serial|concurrent  replica update after the DP
  //     segments on the compute stream, or on the comm stream beside the RW
  //     segments;  TIERSHARD_GRADS=push|pull  remote gradient rows reach
  //     their server by requester-side NVLink stores (push) or a
  //     server-side NVLink gather (pull).
  bool replica_concurrent = true;
  // TIERSHARD_REPLICA=deferred (flag barriers or the group): the replica
  // update runs on its own stream `rep` after the rendezvous and a second
  // rendezvous follows it there; the step returns without waiting for it.
  // The next forward's gather (and, with replicated Flex rows, its serve)
  // waits for that rendezvous -- every owner's broadcast landed -- so the
  // replica tail overlaps the next step's route, count exchange and serve.
  // The replicated-row receive slots are double-buffered by epoch parity:
  // step k+1's partials never land in the set step k's owners still read.
  // Measured at C2 (ms/step, sum over steps): N=2 2.286 vs 2.290
  // (concurrent), N=4 3.27 vs 3.28, 2x2 3.28 vs 3.32 -- the next gather
  // needs the DP replicas (78 % of its rows), so only the route and count
  // exchange overlap, and they compete with the broadcast.  Option, tested.
  bool replica_deferred = false, rep_pending = false;
  cudaStream_t rep = nullptr;
  cudaEvent_t ev_rv = nullptr, ev_rep = nullptr;
  uint64_t rep_barrier_seq = 0;
  uint64_t dp_set_elems = 0, flex_set_elems = 0;  // one receive set, in floats
  bool grads_push = true;
  bool push_first = false;

  size_t step_payload_bytes() const { return ((nb() + 1) * 4 + 7) / 8 * 8 + sizeof(tsd::IpcExport); }
  std::vector<uint8_t> allgather_bytes(const void* mine, size_t bytes);
  void barrier_on_comm();
  void setup_p2p();
  // staged path over the in-process group: sum of `count` floats of `buf`
  // over the group's members (ranks `members`, in order), in place
  tsd::DevBuf<float> ar_tmp;
  void group_allreduce(float* buf, uint64_t count, const std::vector<uint32_t>& members, cudaStream_t on);
  void forward_p2p(const uint32_t* d_rows, uint64_t occ, float* d_out);
  void backward_p2p(const float* d_grad);

  // timing
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
  std::vector<std::pair<int, int>> ev_used;  // (phase, pool index)
  std::vector<cudaStream_t> ev_stream;        // stream of each used pair
  double phase_ms[tsd::kNumPhases] = {};
  uint64_t phase_launches[tsd::kNumPhases] = {};

  uint32_t nb() const { return U + W + 1; }  // buckets incl. the local one

  // --- timing helpers --------------------------------------------------------
  int phase_begin(int phase, cudaStream_t on = nullptr) {
    if (!timing) return -1;
    if (!on) on = stream;
    const size_t idx = ev_used.size();
    if (idx >= ev_pool.size()) {
      cudaEvent_t a, b;
      TSD_CUDA(cudaEventCreate(&a));
      TSD_CUDA(cudaEventCreate(&b));
      ev_pool.emplace_back(a, b);
    }
    TSD_CUDA(cudaEventRecord(ev_pool[idx].first, on));
    ev_used.emplace_back(phase, static_cast<int>(idx));
    ev_stream.push_back(on);
    return static_cast<int>(idx);
  }
  void phase_end(int token) {
    if (token < 0) return;
    TSD_CUDA(cudaEventRecord(ev_pool[token].second, ev_stream[token]));
  }
  void collect_timing() {
    if (ev_used.empty()) return;
    TSD_CUDA(cudaStreamSynchronize(stream));
    if (comm) TSD_CUDA(cudaStreamSynchronize(comm));
    if (aux) TSD_CUDA(cudaStreamSynchronize(aux));
    // keep the timeline of the last step (offsets from its first event): a
    // step starts at the first phase recorded after the previous collection
    trace.clear();
    const cudaEvent_t origin = ev_pool[ev_used.front().second].first;
    for (size_t i = 0; i < ev_used.size(); ++i) {
      const auto [phase, idx] = ev_used[i];
      float ms = 0.f, t0 = 0.f, t1 = 0.f;
      TSD_CUDA(cudaEventElapsedTime(&ms, ev_pool[idx].first, ev_pool[idx].second));
      TSD_CUDA(cudaEventElapsedTime(&t0, origin, ev_pool[idx].first));
      TSD_CUDA(cudaEventElapsedTime(&t1, origin, ev_pool[idx].second));
      phase_ms[phase] += ms;
      phase_launches[phase] += 1;
      trace.push_back({phase, ev_stream[i] == stream ? 0 : 1, t0, t1});
    }
    ev_stream.clear();
    ev_used.clear();
  }
  struct TraceRec {
    int phase, stream_id;
    float t0, t1;
  };
  std::vector<TraceRec> trace;  // timeline of the last collected window

  tsd::RemapView remap_view() const {
    tsd::RemapView rv;
    rv.identity = U == 1;
    rv.dest = d_dest;
    rv.local = d_local;
    rv.dp_cut = cfg.dp_cut;
    rv.flex_cut = cfg.flex_cut;
    rv.rank = g;
    rv.slot = slot;
    return rv;
  }

  void ensure_sort_capacity(uint64_t m) {
    keys_a.ensure(m);
    vals_a.ensure(m);
    keys_b.ensure(m);
    vals_b.ensure(m);
    const uint64_t tiles = tsd::radix_tiles(m);
    ghist.ensure(tsd::kMaxRadixPasses * tsd::kMaxRadixBins);
    goff.ensure(tsd::kMaxRadixPasses * tsd::kMaxRadixBins);
    sort_counters.ensure(tsd::kMaxRadixPasses);
    sort_status.ensure(tsd::kMaxRadixPasses * tiles * tsd::kMaxRadixBins);
    starts.ensure(m + 1);
    seg_keys.ensure(m + 1);
    seg_scratch.ensure(tsd::segment_scratch_elems(m) + 8);
    const uint64_t max_long = m / (seg_short_max + 1) + 1;
    long_list.ensure(max_long);
    piece_off.ensure(max_long + 1);
    partials.ensure((m / tsd::kPiece + max_long + 1) * cfg.dim);
  }

  // ------------------------------------------------------------------------
  void create(const ts_table_config& c, const uint8_t* tier_dest);
  void dedup_local(cudaStream_t on);
  void dedup_p2p(cudaStream_t on);
  void segment_range_concurrent(const uint32_t* sk, const uint32_t* sv, const uint32_t* d_lo,
                                const uint32_t* d_hi, uint64_t m, const tsd::GradSource& gs,
                                const tsd::OptParams& opt, const tsd::DenseRange& d0,
                                const tsd::DenseRange& d1);
  void forward(const uint32_t* d_rows, uint64_t occ, float* d_out);
  void backward(const float* d_grad);
  // ---- cross-step dedup (U = 1, ts_table_train_steps_host) ---------------
  // The dedup of step s+1 needs only its ids, which the pipelined host path
  // has on the device one step ahead: it runs on `pre` beside step s's
  // segment update instead of beside step s+1's gather, so the gather gets
  // every SM.  Two dedup buffer sets alternate by step parity (the swap
  // below exchanges the table's members with `alt`); step s+1's dedup waits
  // for step s's gather to end, by which time step s-1's segment kernels --
  // the last readers of that set -- have finished.  TIERSHARD_LOOKAHEAD=1
  // enables it (measured no gain, see create()).
  struct DedupSet {
    tsd::DevBuf<uint32_t> keys_a, vals_a, keys_b, vals_b, ghist, goff, sort_counters, starts, seg_keys,
        seg_scratch, nseg, seg_split, long_list, long_count, piece_off;
    tsd::DevBuf<uint64_t> sort_status;
    uint32_t* dd_keys = nullptr;
    uint32_t* dd_vals = nullptr;
  } alt;
  bool lookahead = false, alt_ready = false, skip_fwd_dedup = false;
  cudaStream_t pre = nullptr;
  cudaEvent_t ev_pre[2] = {nullptr, nullptr}, ev_gather_done = nullptr;
  cudaEvent_t ev_dedup_cur = nullptr;  // the event the backward's dedup wait uses
  unsigned la_gather_grid = 0;
  void swap_dedup();
  void dedup_rows(cudaStream_t on, const uint32_t* rows, uint64_t occ);
  void train_steps_lookahead(uint32_t* const* buf, const uint32_t* const* h_rows, const uint64_t* occ,
                             uint32_t steps);
  // One training step (forward, then backward with grad = out).  At U = 1
  // with TIERSHARD_GRAPH=1 it is captured into a CUDA graph and replayed:
  // the step's ~20 kernels across the compute and aux streams become one
  // launch.
  // Each call re-captures (host work only) and updates the executable graph
  // in place -- the batch pointer and size change every step -- falling
  // back to a fresh instantiation when the topology changed.
  cudaGraphExec_t step_exec = nullptr;
  bool step_graph = false;
  uint64_t graph_updates = 0, graph_instantiations = 0;
  void train_step(const uint32_t* d_rows, uint64_t occ, float* d_out);
  void exchange(const void* send, const std::vector<uint64_t>& s_off,
                const std::vector<uint64_t>& s_cnt, void* recv,
                const std::vector<uint64_t>& r_off, const std::vector<uint64_t>& r_cnt,
                size_t elem_bytes, cudaStream_t on);
  void destroy();
};

// ---------------------------------------------------------------------------
// create
// ---------------------------------------------------------------------------

void ts_table::create(const ts_table_config& c, const uint8_t* tier_dest) {
  using namespace tsd;
  cfg = c;
  N = c.num_nodes;
  W = c.gpus_per_node;
  U = N * W;
  g = c.rank;
  slot = g % W;
  node = g / W;
  if (N == 0 || W == 0 || U > 256) fail(TS_ERR_CONFIG, "table: need 1 <= N*W <= 256 GPUs");
  if (g >= U) fail(TS_ERR_CONFIG, "table: rank out of range");
  if (c.dim == 0 || c.dim % 32 != 0 || c.dim > 1024 || (c.dim & (c.dim - 1)) != 0) {
    fail(TS_ERR_CONFIG, "embedding_dim " + std::to_string(c.dim) +
                            " unsupported by the device path (32, 64, 128, 256, 512, 1024)");
  }
  if (c.n_rows == 0 || c.n_rows > 0xFFFFFFFFull) fail(TS_ERR_VALIDATION, "table: need 1 <= rows < 2^32");
  if (c.dp_cut > c.flex_cut || c.flex_cut > c.n_rows) {
    fail(TS_ERR_VALIDATION, "assign_rows: plan does not cover the distribution");
  }
  if (c.optimizer != TS_OPT_SGD && c.optimizer != TS_OPT_ROWWISE_ADAGRAD) {
    fail(TS_ERR_CONFIG, "table: unknown optimizer");
  }
  if (c.max_occurrences == 0 || c.max_occurrences >= 0x7FFFFFFFull) {
    fail(TS_ERR_CONFIG, "table: max_occurrences must be in [1, 2^31)");
  }
  if (U > 1 && !c.nccl_unique_id && !c.group) {
    fail(TS_ERR_CONFIG, "table: U > 1 needs an NCCL unique id or an in-process group");
  }
  if (c.group && tsd::group_size(c.group) != U) fail(TS_ERR_CONFIG, "table: group size differs from N*W");
  if (U > 1 && !tier_dest) fail(TS_ERR_CONFIG, "table: U > 1 needs the placement table");
  use_device(c.device);
  {
    // default at U > 1 with one process per GPU (the flag-barrier peer
    // path): the exchange streams get 48 SMs at U = 2, 56 at U >= 4, of
    // their own.  Re-measured after the fused route and the 4-block gather
    // (medians): 1x2 K=40 2.109, 48 2.115, 56 2.148, 64 2.242; 1x4 48 2.79,
    // 56 2.728, 64 2.70-2.74, 72 2.856, 80 2.955; after the rotated push,
    // 2x2 3-tier 56 2.862-2.874, 64 2.939, 72 3.066.
    // Earlier, at C2 (ms/step, tools/mg_env_ab.sh): N=2 1x2
    // K=0 2.285, 40 2.231, 48 2.244, 56 2.304, 64 2.425; N=4 1x4 K=0 3.27,
    // 32 3.10, 40 2.97, 48 2.85-2.90, 64 2.95, 72 3.05; N=4 2x2 3-tier K=0
    // 3.30, 40 3.33, 48 3.31, 64 3.13.  The persistent HBM grids otherwise
    // hold every SM slot, and the serve / push / replica / rendezvous
    // kernels wait for them; at U = 1 a split only slows the dedup sort
    // and the long-segment path (1.23 -> 1.43-2.31 ms).
    const char* se = std::getenv("TIERSHARD_SM_SPLIT");
    const char* xe = std::getenv("TIERSHARD_EXCHANGE");
    const bool staged = xe && std::string(xe) == "nccl";
    const int k = se ? std::atoi(se) : ((U > 1 && !c.group && !staged) ? (U >= 4 ? 56 : 48) : 0);
    if (k > 0) {
      smp = make_partition(c.device, k);
      set_sm_budget(smp.sms[1]);
      TSD_CUDA(cudaStreamCreateWithFlags(&nccl_st, cudaStreamNonBlocking));
    }
  }
  stream = make_stream(1, 0);
  seg_short_max = tsd::short_max(U);
  {
    if (const char* e = std::getenv("TIERSHARD_DEDUP_IN_FORWARD")) dedup_in_forward = std::string(e) != "0";
    if (dedup_in_forward) {
      // aux priority (TIERSHARD_AUX_PRIORITY=high|low): at U = 1 the dedup
      // sort's blocks are dispatched ahead of the gather's (measured at C2
      // with 6 gather blocks per SM: 1.328 -> 1.307 ms/step); at U > 1 with
      // the SM partition too (the comm stream has SMs of its own), beside a
      // 4-blocks-per-SM gather: N=2 2.21 -> 2.17, N=4 2.86 -> 2.82 ms (medians)
      const char* pe = std::getenv("TIERSHARD_AUX_PRIORITY");
      const bool aux_high = pe ? std::string(pe) == "high" : (U == 1 || smp.active());
      int lo_pri = 0, hi_pri = 0;
      TSD_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
      aux = make_stream(1, aux_high ? hi_pri : lo_pri);
      // TIERSHARD_SM_SPLIT_DEDUP=1: the prefetched dedup on a stream of the
      // K partition, beside the exchange kernels.  Measured at C2, N=2 with
      // K = 32 / 40 / 48: 2.79 / 2.53 / 2.37 ms against 2.23 with the
      // dedup on the rest -- the latency-bound sort needs the SM count
      // TIERSHARD_SM_SPLIT_DEDUP=device (default at U = 2): on a stream of
      // the whole device (primary context), free to use either partition's
      // idle SMs.  Medians: 1x2 2.108 -> 2.087 ms; 1x4 2.70 -> 2.74 (the
      // sort then delays serve and push there), so U = 2 only
      const char* de = std::getenv("TIERSHARD_SM_SPLIT_DEDUP");
      if (!de && U == 2 && N == 1) de = "device";
      if (smp.active() && de && std::string(de) != "0") {
        if (std::string(de) == "device") {
          TSD_CUDA(cudaStreamCreateWithPriority(&dd, cudaStreamNonBlocking, hi_pri));
        } else {
          dd = make_stream(0, hi_pri);
        }
      }
      TSD_CUDA(cudaEventCreateWithFlags(&ev_fwd0, cudaEventDisableTiming));
      TSD_CUDA(cudaEventCreateWithFlags(&ev_dedup, cudaEventDisableTiming));
    }
    if (const char* e = std::getenv("TIERSHARD_LONG_CONCURRENT")) long_concurrent = std::string(e) != "0";
    long_concurrent = long_concurrent && aux;
    if (long_concurrent) {
      TSD_CUDA(cudaEventCreateWithFlags(&ev_seg0, cudaEventDisableTiming));
      TSD_CUDA(cudaEventCreateWithFlags(&ev_long, cudaEventDisableTiming));
    }
  }

  if (U == 1 && aux) {
    // measured at C2 (tools/la_ab.sh, tools/la_trace.py): e2e 2.85-2.97 M
    // with it against 2.87 M without, within noise -- the persistent
    // segment-update grids hold every SM slot, so step s+1's sort makes
    // almost no progress beside them (1.25 ms instead of 0.5) and ends up
    // beside step s+1's gather anyway.  Opt-in (TIERSHARD_LOOKAHEAD=1).
    const char* le = std::getenv("TIERSHARD_LOOKAHEAD");
    lookahead = le && std::string(le) == "1";
    if (lookahead) {
      pre = make_stream(0, 0);
      for (cudaEvent_t* e : {&ev_pre[0], &ev_pre[1], &ev_gather_done}) {
        TSD_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      }
    }
  }
  if (U == 1) {
    // measured at C2, N=1: 3.293 M samples/s with the graph, 3.307 M without
    // (and 2.94 / 2.96 M end to end) -- the step's launches already run ahead
    // of the device, so the graph only adds the per-step capture; opt-in
    const char* ge = std::getenv("TIERSHARD_GRAPH");
    step_graph = ge && std::string(ge) == "1";
  }

  // ---- local layout --------------------------------------------------------
  std::vector<uint32_t> l2c;
  if (U == 1) {
    dp_rows = c.dp_cut;
    flex_rows = c.flex_cut - c.dp_cut;
    rw_rows = c.n_rows - c.flex_cut;
    local_rows = c.n_rows;
  } else {
    const uint64_t n = c.n_rows;
    h_dest.assign(tier_dest, tier_dest + n);
    h_local.assign(n, 0);
    ShardRows sr;
    try {
      shard_layout(n, c.dp_cut, c.flex_cut, tier_dest, N, W, g, h_local.data(), &sr);
    } catch (const LayoutError& e) {
      fail(e.status, e.what());
    }
    dp_rows = sr.dp;
    flex_rows = sr.flex;
    rw_rows = sr.rw;
    local_rows = dp_rows + flex_rows + rw_rows;
    l2c.resize(local_rows);
    for (uint64_t i = 0; i < c.dp_cut; ++i) l2c[i] = static_cast<uint32_t>(i);
    for (uint64_t i = c.dp_cut; i < c.flex_cut; ++i) {
      if (tier_dest[i] == slot) l2c[h_local[i]] = static_cast<uint32_t>(i);
    }
    for (uint64_t i = c.flex_cut; i < n; ++i) {
      if (tier_dest[i] == g) l2c[h_local[i]] = static_cast<uint32_t>(i);
    }
    TSD_CUDA(dev_alloc(&d_dest, n));
    TSD_CUDA(dev_alloc(&d_local, sizeof(uint32_t) * n));
    TSD_CUDA(cudaMemcpyAsync(d_dest, tier_dest, n, cudaMemcpyHostToDevice, stream));
    TSD_CUDA(cudaMemcpyAsync(d_local, h_local.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice,
                             stream));
  }

  {  // fail before allocating when the shard and its step buffers cannot fit
    const ts_table_footprint fp = table_footprint(c, dp_rows, flex_rows, rw_rows, false);
    size_t free_b = 0, total_b = 0;
    TSD_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (fp.total > free_b) {
      const auto gib = [](uint64_t b) { return std::to_string(static_cast<double>(b) / (1ull << 30)).substr(0, 6); };
      fail(TS_ERR_CONFIG, "table: rank " + std::to_string(g) + " needs " + gib(fp.total) + " GiB of HBM (weights " +
                              gib(fp.weights) + ", remap " + gib(fp.remap) + ", step buffers " +
                              gib(fp.step_buffers) + ", exchange " + gib(fp.exchange) + ") but " + gib(free_b) +
                              " GiB are free; shard over more GPUs or lower max_occurrences / recv_rows_hint");
    }
  }
  TSD_CUDA(dev_alloc(&d_w, sizeof(float) * std::max<uint64_t>(local_rows, 1) * c.dim));
  if (c.optimizer == TS_OPT_ROWWISE_ADAGRAD) {
    TSD_CUDA(dev_alloc(&d_state, sizeof(float) * std::max<uint64_t>(local_rows, 1)));
    TSD_CUDA(cudaMemsetAsync(d_state, 0, sizeof(float) * std::max<uint64_t>(local_rows, 1), stream));
  }
  {
    DevBuf<uint32_t> d_l2c;
    if (!l2c.empty()) {
      d_l2c.ensure(l2c.size());
      TSD_CUDA(cudaMemcpyAsync(d_l2c.ptr, l2c.data(), sizeof(uint32_t) * l2c.size(),
                               cudaMemcpyHostToDevice, stream));
    }
    launch_init_weights(d_w, local_rows, c.dim, c.weight_seed, l2c.empty() ? nullptr : d_l2c.ptr,
                        stream);
    TSD_CUDA(cudaStreamSynchronize(stream));
    d_l2c.release();
  }

  // TIERSHARD_L2_HOT_MB=X (default 16): an L2 persisting
  // access-policy window over the first X MB of the shard -- the hottest
  // rows, canonical order being probability order -- on the compute and aux
  // streams, so the output writes and the host path's H2D copies do not
  // evict them.  Measured at C2, N=1 (3 interleaved runs each, samples/s
  // device / e2e): 0 MB 3.336 / 3.117 M, 8 3.354 / 3.131, 12 3.350 / 3.131,
  // 16 3.369 / 3.151, 20 3.373 / 3.149, 24 3.312 / 3.102; 32 and 64 MB
  // slower still (the rest of the L2 shrinks).
  {
    const char* he = std::getenv("TIERSHARD_L2_HOT_MB");
    // at U > 1 the shard starts with the DP rows, the hottest too: N=2 2.24 -> 2.21 ms
    const uint64_t want = static_cast<uint64_t>(std::max(0, he ? std::atoi(he) : 16)) << 20;
    if (want) {
      int max_persist = 0, max_window = 0;
      TSD_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c.device));
      TSD_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, c.device));
      const uint64_t bytes = std::min<uint64_t>({want, static_cast<uint64_t>(max_persist),
                                                 static_cast<uint64_t>(max_window),
                                                 sizeof(float) * local_rows * c.dim});
      TSD_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes));
      cudaStreamAttrValue attr{};
      attr.accessPolicyWindow.base_ptr = d_w;
      attr.accessPolicyWindow.num_bytes = bytes;
      attr.accessPolicyWindow.hitRatio = 1.0f;
      attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      for (cudaStream_t st : {stream, aux}) {
        if (st) TSD_CUDA(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &attr));
      }
    }
  }

  // ---- step buffers ----------------------------------------------------------
  gather_grid = tsd::gather_grid(c.max_occurrences);
  fwd_gather_grid = gather_grid;
  {
    // forward gather variant (TIERSHARD_GATHER=bulk|reg): at U = 1 the
    // bulk-copy gather, whose rows never pass through registers, so it
    // holds few warps and the dedup sort beside it gets the rest of each SM.
    // Measured at C2, N=1 (step ms / gather / sort, tools/gather_ab.sh):
    // register 6 blocks/SM 1.304 / 0.56 / 0.66; bulk 5 blocks x 2 stages
    // 1.230 / 0.63 / 0.53; bulk 6 x 2 1.297 (gather alone 0.53 ms, the
    // fastest); bulk 3 x 3 1.252; bulk 2 x 3 1.385 (sort 0.30, gather 0.79)
    // -- the two kernels trade shared memory, the step follows the slower.
    const char* ge = std::getenv("TIERSHARD_GATHER");
    const bool bulk = ge ? std::string(ge) == "bulk" : U == 1;
    if (const char* se = std::getenv("TIERSHARD_BULK_STAGES")) gather_bulk_stages = std::max(2, std::atoi(se));
    if (!bulk) gather_bulk_stages = 0;
  }
  if (aux) {
    const char* e = std::getenv("TIERSHARD_GATHER_BLOCKS");
    // register gather: 6 blocks per SM leave the dedup sort room beside the
    // gather (C2, N=1: 8 -> 1.318 ms/step, 6 -> 1.307, 4 -> 1.328; aux at
    // high priority).  At U > 1 without the SM partition 8 (N=2: 2.33 ms
    // against 2.35-2.36 with 6; a high-priority aux there costs 0.1 ms: the
    // sort then delays serve and push); with it 4 and a high-priority aux
    // (N=2 medians 2.21 / 2.17 / 2.24 / 2.42 ms with 8 / 4 / 3 / 2, 6: 2.26;
    // tools/mg_env_ab.sh).  Bulk gather: 5 (above).
    const unsigned per_sm = e ? static_cast<unsigned>(std::max(1, std::atoi(e)))
                              : (gather_bulk_stages ? 5u : (U == 1 ? 6u : (smp.active() ? 4u : 8u)));
    fwd_gather_grid = std::min(gather_grid, static_cast<unsigned>(tsd::sm_count()) * per_sm);
    // with the dedup moved beside the previous step's segment update
    // (lookahead), the gather runs alone: its fastest grid (bulk 6 x 2:
    // 0.53 ms per C2 forward; register 8)
    {
      const char* le = std::getenv("TIERSHARD_LA_GATHER_BLOCKS");
      const unsigned la = le ? static_cast<unsigned>(std::max(1, std::atoi(le))) : (gather_bulk_stages ? 6u : 8u);
      la_gather_grid = std::min(gather_grid, static_cast<unsigned>(tsd::sm_count()) * la);
    }
    // TIERSHARD_GATHER_GRID: total blocks (fractional blocks per SM, A/B)
    if (const char* ge2 = std::getenv("TIERSHARD_GATHER_GRID")) {
      fwd_gather_grid = std::min(gather_grid, static_cast<unsigned>(std::max(1, std::atoi(ge2))));
    }
  }
  // [local gather partials | remote partials: staged scatter (gather_grid) or
  //  peer servers' slots (U x kServeGrid)]; zeroed once — slots a server
  //  never writes (our own) must read 0.
  remote_loss_slots = static_cast<uint64_t>(U) * kServeGrid;
  loss_partials.ensure(gather_grid + std::max<uint64_t>(gather_grid, remote_loss_slots));
  TSD_CUDA(cudaMemsetAsync(loss_partials.ptr, 0, sizeof(double) * loss_partials.cap, stream));
  d_loss.ensure(1);
  tier_counts.ensure(4);
  nseg.ensure(4);
  seg_split.ensure(4);
  long_count.ensure(4);
  // dedup / sort sized once for the largest entry count a step can have
  // (the batch, plus what this rank serves at U > 1): a DevBuf that grows
  // mid-run frees and re-allocates, which synchronises the device
  const uint64_t max_entries = c.max_occurrences + (U > 1 ? recv_capacity_rows(c) : 0);
  ensure_sort_capacity(max_entries);
  if (U > 1) {
    entry_keys.ensure(max_entries);
    entry_vals.ensure(max_entries);
    bucket.ensure(c.max_occurrences);
    route_hist.ensure(tsd::route_hist_elems(c.max_occurrences, nb()));
    order.ensure(c.max_occurrences);
    send_ids.ensure(c.max_occurrences);
    // received gradient rows: peers store into this buffer (P2P push), so
    // it is mapped by every peer and only moves through regrow_recv().
    // Sized from the caller's hint (the plan's expected remote occurrences
    // with a margin), else for the worst case, every peer's whole batch
    // (send_rows, the staged path's buffer, is allocated on first use)
    recv_rows.ensure(tsd::recv_capacity_rows(c) * c.dim);
    bucket_start.ensure(nb() + 2);
    all_counts.ensure(static_cast<uint64_t>(U) * (nb() + 1));
    // replicated-row gradients: [U][per_dp][D] receive slots (P2P push
    // mode; the staged path uses the first dp_rows x D as a dense buffer)
    per_dp = static_cast<uint32_t>((dp_rows + U - 1) / U);
    {
      const char* re = std::getenv("TIERSHARD_REPLICA");
      replica_deferred = re && std::string(re) == "deferred";
    }
    const uint64_t sets = replica_deferred ? 2 : 1;
    dp_set_elems = std::max<uint64_t>(uint64_t{U} * per_dp, 1);
    dense_dp.ensure(sets * dp_set_elems * c.dim);
    stamp_dp.ensure(sets * dp_set_elems);
    TSD_CUDA(cudaMemsetAsync(stamp_dp.ptr, 0, sizeof(uint32_t) * stamp_dp.cap, stream));
    if (N > 1) {
      per_flex = static_cast<uint32_t>((flex_rows + N - 1) / N);
      flex_set_elems = std::max<uint64_t>(uint64_t{N} * per_flex, 1);
      dense_flex.ensure(sets * flex_set_elems * c.dim);
      stamp_flex.ensure(sets * flex_set_elems);
      TSD_CUDA(cudaMemsetAsync(stamp_flex.ptr, 0, sizeof(uint32_t) * stamp_flex.cap, stream));
    }
    TSD_CUDA(cudaStreamSynchronize(stream));
    // communicators: world, intra (color = node), cross (color = slot)
    // the exchange / replica stream gets the highest priority: its kernels
    // are short, sit on the critical path, and would otherwise queue behind
    // the persistent compute grids they overlap with
    int lo_prio = 0, hi_prio = 0;
    TSD_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    comm = make_stream(0, hi_prio);
    for (cudaEvent_t* e : {&ev_ids, &ev_fwd, &ev_bwd0, &ev_grads, &ev_dense, &ev_ar}) {
      TSD_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    if (c.group) {
      grp = c.group;
      group_attach(grp, g, c.device);
      attached = true;
    } else {
      ncclUniqueId id;
      std::memcpy(&id, c.nccl_unique_id, sizeof(id));
      TSD_NCCL(ncclCommInitRank(&world, static_cast<int>(U), id, static_cast<int>(g)));
      TSD_NCCL(ncclCommSplit(world, static_cast<int>(node), static_cast<int>(g), &intra, nullptr));
      TSD_NCCL(ncclCommSplit(world, static_cast<int>(slot), static_cast<int>(g), &cross, nullptr));
    }
    setup_p2p();
  }
}

// All ranks contribute `bytes` bytes; returns the U x bytes concatenation.
// Collective on the comm stream; synchronises it.
std::vector<uint8_t> ts_table::allgather_bytes(const void* mine, size_t bytes) {
  using namespace tsd;
  std::vector<uint8_t> all(bytes * U);
  if (grp) {
    group_allgather(grp, g, mine, bytes, all.data());
    return all;
  }
  xfer.ensure(bytes * U);
  export_in_slot = false;  // the step payload's slot may live in xfer
  cudaStream_t ns = nccl_st ? nccl_st : comm;
  if (nccl_st) TSD_CUDA(cudaStreamSynchronize(comm));  // whatever comm had queued, first
  TSD_CUDA(cudaMemcpyAsync(xfer.ptr + bytes * g, mine, bytes, cudaMemcpyHostToDevice, ns));
  TSD_NCCL(ncclAllGather(xfer.ptr + bytes * g, xfer.ptr, bytes, ncclUint8, world, ns));
  TSD_CUDA(cudaMemcpyAsync(all.data(), xfer.ptr, bytes * U, cudaMemcpyDeviceToHost, ns));
  TSD_CUDA(cudaStreamSynchronize(ns));
  return all;
}

// Device-side rendezvous of all ranks on the comm stream (a 1-int all-reduce):
// work queued before it on every rank completes before work queued after it.
void ts_table::barrier_on_comm() {
  using namespace tsd;
  if (grp) {
    group_barrier(grp, g, comm);
    return;
  }
  if (flag_barriers) {
    launch_flag_barrier(flag_barrier, 0, ++barrier_seq, comm);
    return;
  }
  TSD_NCCL(ncclAllReduce(barrier_buf.ptr, barrier_buf.ptr, 1, ncclInt32, ncclSum, world, comm));
}

// Peer mode needs every pair of ranks to be NVLink/P2P reachable (one node)
// and U <= 8; TIERSHARD_EXCHANGE=nccl forces the staged NCCL path.  The
// decision is collective (min over ranks).
void ts_table::setup_p2p() {
  using namespace tsd;
  barrier_buf.ensure(1);
  TSD_CUDA(cudaMemsetAsync(barrier_buf.ptr, 0, sizeof(int32_t), comm));
  int32_t ok = U <= kMaxPeerRanks && U <= kMaxGradPeers + 1 ? 1 : 0;
  if (const char* env = std::getenv("TIERSHARD_EXCHANGE")) {
    if (std::string(env) == "nccl") ok = 0;
  }
  if (grp) {
    // in-process ranks: the peer-memory path is the only one (no NCCL);
    // ranks on other GPUs of this process are reached by UVA pointers
    if (U > kMaxPeerRanks) fail(TS_ERR_CONFIG, "table: the in-process group supports U <= 8");
    int32_t dev = cfg.device;
    const std::vector<uint8_t> devs = allgather_bytes(&dev, sizeof(dev));
    for (uint32_t p = 0; p < U; ++p) {
      int32_t pd;
      std::memcpy(&pd, devs.data() + sizeof(pd) * p, sizeof(pd));
      if (pd == cfg.device) continue;
      int can = 0;
      TSD_CUDA(cudaDeviceCanAccessPeer(&can, cfg.device, pd));
      if (!can) fail(TS_ERR_CONFIG, "table: in-process group ranks on GPUs without peer access");
      const cudaError_t e = cudaDeviceEnablePeerAccess(pd, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else {
        TSD_CUDA(e);
      }
    }
    peers.set_direct(true);
    if (!ok) {  // TIERSHARD_EXCHANGE=nccl: the staged path, its collectives over the group
      p2p = false;
      return;
    }
  }
  char bus[32] = {};
  TSD_CUDA(cudaDeviceGetPCIBusId(bus, sizeof(bus), cfg.device));
  const std::vector<uint8_t> buses = allgather_bytes(bus, sizeof(bus));
  for (uint32_t p = 0; p < U && ok && !grp; ++p) {
    if (p == g) continue;
    int dev = -1, can = 0;
    if (cudaDeviceGetByPCIBusId(&dev, reinterpret_cast<const char*>(buses.data() + sizeof(bus) * p)) !=
        cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    TSD_CUDA(cudaDeviceCanAccessPeer(&can, cfg.device, dev));
    if (!can) ok = 0;
  }
  const std::vector<uint8_t> votes = allgather_bytes(&ok, sizeof(ok));
  for (uint32_t p = 0; p < U; ++p) {
    int32_t v;
    std::memcpy(&v, votes.data() + sizeof(v) * p, sizeof(v));
    if (!v) ok = 0;
  }
  p2p = ok != 0;
  if (!p2p && smp.active()) {
    fail(TS_ERR_CONFIG, "table: the SM partition needs the peer-memory exchange (set TIERSHARD_SM_SPLIT=0)");
  }
  if (!p2p) return;
  if (const char* env = std::getenv("TIERSHARD_REPLICA")) replica_concurrent = std::string(env) != "serial";
  if (const char* env = std::getenv("TIERSHARD_GRADS")) grads_push = std::string(env) != "pull";
  if (const char* env = std::getenv("TIERSHARD_PUSH_ORDER")) push_first = std::string(env) == "first";
  // export the table-owned buffers peers read or write
  auto exp_or_none = [this](const void* p) {
    IpcExport e;
    std::memset(&e, 0, sizeof(e));
    return p ? (grp ? direct_export(p) : export_pointer(p)) : e;
  };
  flag_box.ensure(kFlagChannels * kMaxPeerRanks);
  TSD_CUDA(cudaMemsetAsync(flag_box.ptr, 0, sizeof(uint64_t) * kFlagChannels * kMaxPeerRanks, comm));
  mbox.ensure(step_payload_bytes() * U);
  TSD_CUDA(cudaStreamSynchronize(comm));
  constexpr int kExports = 12;
  IpcExport mine[kExports] = {export_ptr(send_ids.ptr), export_ptr(order.ptr),
                              export_ptr(loss_partials.ptr + gather_grid), exp_or_none(dense_dp.ptr),
                              export_ptr(d_w), exp_or_none(d_state), exp_or_none(dense_flex.ptr),
                              exp_or_none(stamp_dp.ptr), exp_or_none(stamp_flex.ptr),
                              export_ptr(recv_rows.ptr), export_ptr(flag_box.ptr), export_ptr(mbox.ptr)};
  const std::vector<uint8_t> all = allgather_bytes(mine, sizeof(mine));
  peer_ids.assign(U, nullptr);
  peer_pos.assign(U, nullptr);
  peer_loss.assign(U, nullptr);
  peer_dense_dp.assign(U, nullptr);
  peer_dense_flex.assign(U, nullptr);
  peer_w.assign(U, d_w);
  peer_state.assign(U, d_state);
  peer_dense_dp[g] = dense_dp.ptr;
  peer_dense_flex[g] = dense_flex.ptr;
  peer_stamp_dp.assign(U, nullptr);
  peer_stamp_flex.assign(U, nullptr);
  peer_recv_rows.assign(U, nullptr);
  peer_stamp_dp[g] = stamp_dp.ptr;
  peer_stamp_flex[g] = stamp_flex.ptr;
  for (uint32_t p = 0; p < U; ++p) {
    if (p == g) continue;
    IpcExport e[kExports];
    std::memcpy(e, all.data() + sizeof(mine) * p, sizeof(mine));
    const int pp = static_cast<int>(p);
    auto open_opt = [&](const IpcExport& x) { return x.base_id ? peers.open(pp, x) : nullptr; };
    peer_ids[p] = static_cast<const uint32_t*>(peers.open(pp, e[0]));
    peer_pos[p] = static_cast<const uint32_t*>(peers.open(pp, e[1]));
    peer_loss[p] = static_cast<double*>(peers.open(pp, e[2]));
    peer_dense_dp[p] = static_cast<float*>(open_opt(e[3]));
    peer_w[p] = static_cast<float*>(peers.open(pp, e[4]));
    peer_state[p] = static_cast<float*>(open_opt(e[5]));
    peer_dense_flex[p] = static_cast<float*>(open_opt(e[6]));
    peer_stamp_dp[p] = static_cast<uint32_t*>(open_opt(e[7]));
    peer_stamp_flex[p] = static_cast<uint32_t*>(open_opt(e[8]));
    peer_recv_rows[p] = static_cast<float*>(peers.open(pp, e[9]));
    flag_barrier.peer_flags[p] = static_cast<uint64_t*>(peers.open(pp, e[10]));
    mbox_put.peer_box[p] = static_cast<uint8_t*>(peers.open(pp, e[11]));
  }
  mbox_put.peer_box[g] = mbox.ptr;
  mbox_put.n = static_cast<int>(U);
  mbox_put.me = static_cast<int>(g);
  flag_barrier.peer_flags[g] = flag_box.ptr;
  flag_barrier.n = static_cast<int>(U);
  flag_barrier.me = static_cast<int>(g);
  if (!grp) {  // in-process ranks may share a GPU: a spinning block could starve a peer
    const char* be = std::getenv("TIERSHARD_BARRIER");
    flag_barriers = !(be && std::string(be) == "nccl") || smp.active();
    const char* ce = std::getenv("TIERSHARD_FWD_COUNTS");
    // with an SM partition the step keeps NCCL off the (green) comm stream
    mailbox_counts = flag_barriers && ((ce && std::string(ce) == "mailbox") || smp.active());
  }
  replica_deferred = replica_deferred && (flag_barriers || grp);
  if (replica_deferred) {
    int lo_prio = 0, hi_prio = 0;
    TSD_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    rep = make_stream(0, hi_prio);
    TSD_CUDA(cudaEventCreateWithFlags(&ev_rv, cudaEventDisableTiming));
    TSD_CUDA(cudaEventCreateWithFlags(&ev_rep, cudaEventDisableTiming));
  }
  {
    if (const char* oe = std::getenv("TIERSHARD_REPLICA_OWNER")) replica_interleave = std::string(oe) != "block";
    if (const char* pr = std::getenv("TIERSHARD_PUSH_ROTATE")) push_rotate = std::string(pr) != "0";
    const char* re = std::getenv("TIERSHARD_ROUTE");
    route_sort = re && std::string(re) == "sort";
    const char* fe = std::getenv("TIERSHARD_FWD");
    pull_forward = fe && std::string(fe) == "pull" && (flag_barriers || grp) && U <= kMaxGradPeers;
  }
  exchange_recv_exports();
  peer_grad.assign(U, nullptr);
  xfer.ensure(step_payload_bytes() * U);
}

// ---------------------------------------------------------------------------
// NCCL all-to-allv: per-peer offsets/counts in elements of elem_bytes.
// RW traffic rides `world`; Flex traffic rides `intra` (peer = node slot).
// The per-peer buffers are laid out [peer p: RW part | Flex part].
// ---------------------------------------------------------------------------

// Every rank's receive-buffer export and capacity (collective); (re)maps the
// peers' buffers, closing a peer's previous mapping when it moved.
void ts_table::exchange_recv_exports() {
  using namespace tsd;
  struct Rec {
    IpcExport e;
    uint64_t cap_rows;
  } mine{export_ptr(recv_rows.ptr), recv_rows.cap / cfg.dim};
  const std::vector<uint8_t> all = allgather_bytes(&mine, sizeof(mine));
  peer_recv_cap.assign(U, 0);
  peer_recv_export.resize(U);
  for (uint32_t p = 0; p < U; ++p) {
    Rec r;
    std::memcpy(&r, all.data() + sizeof(Rec) * p, sizeof(Rec));
    peer_recv_cap[p] = r.cap_rows;
    if (p == g) continue;
    const IpcExport& old = peer_recv_export[p];
    if (old.base_id && (old.base_id != r.e.base_id || std::memcmp(&old.handle, &r.e.handle, sizeof(old.handle)))) {
      peers.close(static_cast<int>(p), old);
    }
    peer_recv_export[p] = r.e;
    peer_recv_rows[p] = static_cast<float*>(peers.open(static_cast<int>(p), r.e));
  }
}

// The checked overflow path of the bounded receive buffers: `need[p]` =
// rows rank p receives this step (every rank derives the same vector from
// the all-gathered bucket starts, so all ranks take this path together).  A
// rank whose capacity is short re-allocates with 25 % headroom; then every
// rank re-exchanges the exports.  Called after the forward's rendezvous:
// every peer's previous gradient push into the old buffers has completed
// (it precedes the previous step's barrier), and our own readers of it are
// drained here.
void ts_table::regrow_recv(const std::vector<uint64_t>& need) {
  using namespace tsd;
  bool any = false;
  for (uint32_t p = 0; p < U; ++p) any = any || need[p] > peer_recv_cap[p];
  if (!any) return;
  ++recv_regrows;
  TSD_CUDA(cudaStreamSynchronize(stream));
  if (aux) TSD_CUDA(cudaStreamSynchronize(aux));
  TSD_CUDA(cudaStreamSynchronize(comm));
  if (need[g] > peer_recv_cap[g]) {
    recv_rows.release();
    recv_rows.ensure((need[g] + need[g] / 4 + 1) * cfg.dim);
  }
  exchange_recv_exports();
}

void ts_table::group_allreduce(float* buf, uint64_t count, const std::vector<uint32_t>& members,
                               cudaStream_t on) {
  using namespace tsd;
  const uint64_t mine = reinterpret_cast<uint64_t>(buf);
  std::vector<uint64_t> all(U);
  group_allgather(grp, g, &mine, sizeof(mine), all.data());
  ar_tmp.ensure(count);
  SumSources ss{};
  for (uint32_t p : members) ss.src[ss.n++] = reinterpret_cast<const float*>(all[p]);
  group_barrier(grp, g, on);  // every member's partial sums are complete
  if (count) {
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((count + 255) / 256, 4u * sm_count()));
    sum_sources_kernel<<<grid, 256, 0, on>>>(ar_tmp.ptr, ss, count);
    TSD_LAUNCH_CHECK();
  }
  group_barrier(grp, g, on);  // every member has read every buffer
  if (count) TSD_CUDA(cudaMemcpyAsync(buf, ar_tmp.ptr, sizeof(float) * count, cudaMemcpyDeviceToDevice, on));
}

void ts_table::exchange(const void* send, const std::vector<uint64_t>& s_off,
                        const std::vector<uint64_t>& s_cnt, void* recv,
                        const std::vector<uint64_t>& r_off, const std::vector<uint64_t>& r_cnt,
                        size_t elem_bytes, cudaStream_t on) {
  // s_off/s_cnt/r_off/r_cnt have 2*U entries: [p*2 + 0] RW, [p*2 + 1] Flex.
  auto* sb = static_cast<const char*>(send);
  auto* rb = static_cast<char*>(recv);
  if (grp) {
    // in-process: every rank's send base + offsets, a device rendezvous (the
    // send data is complete everywhere), each receiver copies its runs out
    // of the senders' buffers, a rendezvous (the senders may reuse them)
    std::vector<uint64_t> mine(2 * U + 1);
    mine[0] = reinterpret_cast<uint64_t>(sb);
    std::copy(s_off.begin(), s_off.begin() + 2 * U, mine.begin() + 1);
    std::vector<uint64_t> all(mine.size() * U);
    tsd::group_allgather(grp, g, mine.data(), sizeof(uint64_t) * mine.size(), all.data());
    tsd::group_barrier(grp, g, on);
    for (uint32_t p = 0; p < U; ++p) {
      if (p == g) continue;
      const uint64_t* theirs = all.data() + mine.size() * p;
      const char* base = reinterpret_cast<const char*>(theirs[0]);
      for (int part = 0; part < 2; ++part) {
        const uint64_t cnt = r_cnt[2 * p + part];
        if (!cnt) continue;
        TSD_CUDA(cudaMemcpyAsync(rb + r_off[2 * p + part] * elem_bytes,
                                 base + theirs[1 + 2 * g + part] * elem_bytes, cnt * elem_bytes,
                                 cudaMemcpyDefault, on));
      }
    }
    tsd::group_barrier(grp, g, on);
    return;
  }
  TSD_NCCL(ncclGroupStart());
  for (uint32_t p = 0; p < U; ++p) {
    if (p == g) continue;
    const size_t s0 = s_cnt[2 * p] * elem_bytes, r0 = r_cnt[2 * p] * elem_bytes;
    if (s0) TSD_NCCL(ncclSend(sb + s_off[2 * p] * elem_bytes, s0, ncclChar, static_cast<int>(p), world, on));
    if (r0) TSD_NCCL(ncclRecv(rb + r_off[2 * p] * elem_bytes, r0, ncclChar, static_cast<int>(p), world, on));
  }
  for (uint32_t p = node * W; p < (node + 1) * W; ++p) {
    if (p == g) continue;
    const int peer = static_cast<int>(p % W);  // rank inside the intra comm
    const size_t s1 = s_cnt[2 * p + 1] * elem_bytes, r1 = r_cnt[2 * p + 1] * elem_bytes;
    if (s1) TSD_NCCL(ncclSend(sb + s_off[2 * p + 1] * elem_bytes, s1, ncclChar, peer, intra, on));
    if (r1) TSD_NCCL(ncclRecv(rb + r_off[2 * p + 1] * elem_bytes, r1, ncclChar, peer, intra, on));
  }
  TSD_NCCL(ncclGroupEnd());
}

// U = 1 dedup: stable sort of the forward's row ids (key = canonical row,
// value = position) and segment heads, on stream `on`.
void ts_table::dedup_local(cudaStream_t on) { dedup_rows(on, last_rows, last_occ); }

void ts_table::dedup_rows(cudaStream_t on, const uint32_t* rows, uint64_t occ) {
  using namespace tsd;
  RadixBuffers rb{keys_a.ptr, vals_a.ptr, keys_b.ptr, vals_b.ptr, ghist.ptr, goff.ptr,
                  sort_status.ptr, sort_counters.ptr};
  const int key_bits = bits_for(local_rows ? local_rows - 1 : 0);
  int t = phase_begin(kPhaseSort, on);
  radix_sort_pairs(rows, nullptr, occ, key_bits, rb, &dd_keys, &dd_vals, on);
  phase_end(t);
  t = phase_begin(kPhaseSegments, on);
  segment_starts(dd_keys, occ, starts.ptr, seg_keys.ptr, nseg.ptr, seg_scratch.ptr, on);
  TSD_CUDA(cudaMemsetAsync(seg_split.ptr, 0, sizeof(uint32_t), on));  // range [0, nseg)
  phase_end(t);
}

void ts_table::swap_dedup() {
  std::swap(keys_a, alt.keys_a);
  std::swap(vals_a, alt.vals_a);
  std::swap(keys_b, alt.keys_b);
  std::swap(vals_b, alt.vals_b);
  std::swap(ghist, alt.ghist);
  std::swap(goff, alt.goff);
  std::swap(sort_counters, alt.sort_counters);
  std::swap(sort_status, alt.sort_status);
  std::swap(starts, alt.starts);
  std::swap(seg_keys, alt.seg_keys);
  std::swap(seg_scratch, alt.seg_scratch);
  std::swap(nseg, alt.nseg);
  std::swap(seg_split, alt.seg_split);
  std::swap(long_list, alt.long_list);
  std::swap(long_count, alt.long_count);
  std::swap(piece_off, alt.piece_off);
  std::swap(dd_keys, alt.dd_keys);
  std::swap(dd_vals, alt.dd_vals);
}

void ts_table::train_steps_lookahead(uint32_t* const* buf, const uint32_t* const* h_rows, const uint64_t* occ,
                                     uint32_t steps) {
  using namespace tsd;
  if (!alt_ready) {  // the second dedup set, sized like the first
    swap_dedup();
    ensure_sort_capacity(cfg.max_occurrences);
    nseg.ensure(4);
    seg_split.ensure(4);
    long_count.ensure(4);
    swap_dedup();
    alt_ready = true;
  }
  const auto stage = [&](uint32_t s) {
    const int b = static_cast<int>(s & 1u);
    TSD_CUDA(cudaStreamWaitEvent(copy, ev_consumed[b], 0));
    if (occ[s]) {
      TSD_CUDA(cudaMemcpyAsync(buf[b], h_rows[s], sizeof(uint32_t) * occ[s], cudaMemcpyHostToDevice, copy));
    }
    TSD_CUDA(cudaEventRecord(ev_copied[b], copy));
  };
  const auto prefetch = [&](uint32_t s) {  // dedup of step s into the active set, on `pre`
    const int b = static_cast<int>(s & 1u);
    TSD_CUDA(cudaStreamWaitEvent(pre, ev_copied[b], 0));
    dedup_rows(pre, buf[b], occ[s]);
    if (long_concurrent) launch_long_segments(starts.ptr, seg_split.ptr, nseg.ptr, occ[s], seg_scratch_view(), pre);
    TSD_CUDA(cudaEventRecord(ev_pre[b], pre));
  };
  if (dedup_ready) {  // a plain forward left its dedup running
    TSD_CUDA(cudaStreamWaitEvent(stream, ev_dedup, 0));
    dedup_ready = false;
  }
  stage(0);
  prefetch(0);
  const unsigned saved_grid = fwd_gather_grid;
  for (uint32_t s = 0; s < steps; ++s) {
    const int b = static_cast<int>(s & 1u);
    if (s + 1 < steps) stage(s + 1);
    TSD_CUDA(cudaStreamWaitEvent(stream, ev_copied[b], 0));
    skip_fwd_dedup = true;
    fwd_gather_grid = la_gather_grid;
    loss_mirror = h_loss_dev + s;  // the loss kernel writes the host slot itself
    forward(buf[b], occ[s], host_out.ptr);
    fwd_gather_grid = saved_grid;
    skip_fwd_dedup = false;
    if (s + 1 < steps) {  // step s+1's dedup beside this step's segment update
      TSD_CUDA(cudaEventRecord(ev_gather_done, stream));
      swap_dedup();
      TSD_CUDA(cudaStreamWaitEvent(pre, ev_gather_done, 0));
      prefetch(s + 1);
      swap_dedup();
    }
    dedup_ready = true;
    ev_dedup_cur = ev_pre[b];
    backward(host_out.ptr);
    ev_dedup_cur = nullptr;
    TSD_CUDA(cudaEventRecord(ev_consumed[b], stream));
    loss_mirror = nullptr;
    swap_dedup();  // the next step's set becomes the table's
  }
  // the table's members hold the set of step `steps` (unused); fine either
  // way, a later step re-runs its own dedup into whichever set is current
}

// U > 1 (peer path) dedup: (local row, source) entries of the local
// occurrences and of the requests this rank serves, stable sort, segment
// heads, and the replicated / rest split -- on stream `on`.  Needs the
// forward's request lists (recv_ids), not the gradients.
void ts_table::dedup_p2p(cudaStream_t on) {
  using namespace tsd;
  const uint64_t m = n_local_occ + recv_total;
  entry_keys.ensure(m);
  entry_vals.ensure(m);
  ensure_sort_capacity(m);
  launch_build_entries(last_rows, order.ptr + n_remote, n_local_occ, remap_view(), recv_ids.ptr, recv_before,
                       recv_total, static_cast<uint32_t>(last_occ), entry_keys.ptr, entry_vals.ptr, on);
  RadixBuffers rb{keys_a.ptr, vals_a.ptr, keys_b.ptr, vals_b.ptr, ghist.ptr, goff.ptr,
                  sort_status.ptr, sort_counters.ptr};
  int t = phase_begin(kPhaseSort, on);
  radix_sort_pairs(entry_keys.ptr, entry_vals.ptr, m, bits_for(local_rows ? local_rows - 1 : 0), rb, &dd_keys,
                   &dd_vals, on);
  phase_end(t);
  t = phase_begin(kPhaseSegments, on);
  segment_starts(dd_keys, m, starts.ptr, seg_keys.ptr, nseg.ptr, seg_scratch.ptr, on);
  const uint32_t dense_hi = static_cast<uint32_t>(dp_rows + (N > 1 ? flex_rows : 0));
  launch_segment_split(dd_keys, starts.ptr, nseg.ptr, dense_hi, seg_split.ptr, on);
  // several nodes: the DP segments end inside the replicated range, at
  // seg_split[3] (their entries are all local, see backward_p2p)
  if (N > 1 && flex_rows) {
    launch_segment_split(dd_keys, starts.ptr, nseg.ptr, static_cast<uint32_t>(dp_rows), seg_split.ptr + 2, on);
  }
  phase_end(t);
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------

void ts_table::forward(const uint32_t* d_rows, uint64_t occ, float* d_out) {
  using namespace tsd;
  if (occ > cfg.max_occurrences) fail(TS_ERR_VALIDATION, "table: batch exceeds max_occurrences");
  // a forward not followed by a backward (eval, or forward twice) leaves
  // the prefetched dedup running on aux over the shared sort buffers and
  // request lists: this forward's route must not touch them before it ends
  if (dedup_ready) {
    TSD_CUDA(cudaStreamWaitEvent(stream, ev_dedup, 0));
    dedup_ready = false;
  }
  last_rows = d_rows;
  last_occ = occ;
  last_out = d_out;
  const RemapView rv = remap_view();
  TSD_CUDA(cudaMemsetAsync(tier_counts.ptr, 0, sizeof(unsigned long long) * 4, stream));

  if (U == 1) {
    if (aux) TSD_CUDA(cudaEventRecord(ev_fwd0, stream));  // the ids are in place
    int t = phase_begin(kPhaseGather);
    launch_gather_local(d_rows, occ, d_w, d_out, rv, cfg.dim, loss_partials.ptr, fwd_gather_grid, stream,
                        gather_bulk_stages);
    phase_end(t);
    launch_loss_finalize(loss_partials.ptr, gather_grid, d_loss.ptr, stream, loss_mirror);
    n_local_occ = occ;
    n_remote = 0;
    if (aux && !skip_fwd_dedup) {  // the backward's dedup, overlapping the gather
      cudaStream_t ds = dedup_stream();
      TSD_CUDA(cudaStreamWaitEvent(ds, ev_fwd0, 0));
      dedup_local(ds);
      TSD_CUDA(cudaEventRecord(ev_dedup, ds));
      // the long-segment list is needed only by the backward's aux work: it
      // stays off the chain the short-segment kernel waits for
      if (ds != aux) TSD_CUDA(cudaStreamWaitEvent(aux, ev_dedup, 0));
      if (long_concurrent) launch_long_segments(starts.ptr, seg_split.ptr, nseg.ptr, occ, seg_scratch_view(), aux);
      dedup_ready = true;
    }
    return;
  }

  if (p2p) {
    if (pull_forward) {
      forward_p2p_pull(d_rows, occ, d_out);
    } else {
      forward_p2p(d_rows, occ, d_out);
    }
    return;
  }

  // ---- staged NCCL path (no peer access): route, bucket, compaction -------
  int t = phase_begin(kPhaseRoute);
  BucketView bv;
  bv.dest = d_dest;
  bv.dp_cut = cfg.dp_cut;
  bv.flex_cut = cfg.flex_cut;
  bv.u = U;
  bv.w = W;
  bv.rank = g;
  bv.slot = slot;
  launch_bucket_keys(d_rows, occ, bv, bucket.ptr, tier_counts.ptr, stream);
  RadixBuffers rb{keys_a.ptr, vals_a.ptr, keys_b.ptr, vals_b.ptr, ghist.ptr, goff.ptr,
                  sort_status.ptr, sort_counters.ptr};
  uint32_t* sorted_b = nullptr;
  uint32_t* sorted_i = nullptr;
  radix_sort_pairs(bucket.ptr, nullptr, occ, bits_for(nb() - 1), rb, &sorted_b, &sorted_i, stream);
  // keep the occurrence order for backward (sort buffers are reused)
  TSD_CUDA(cudaMemcpyAsync(order.ptr, sorted_i, sizeof(uint32_t) * occ, cudaMemcpyDeviceToDevice, stream));
  phase_end(t);

  // ---- counts: every rank's bucket starts, all-gathered, one D2H sync -----
  {
    const int passes = (bits_for(nb() - 1) + 7) / 8;
    if (passes != 1) fail(TS_ERR_CONFIG, "table: U + W + 1 must be <= 256 buckets");
    // single counting pass: its global digit offsets ARE the bucket starts
    launch_bucket_starts(goff.ptr, 1, nb(), static_cast<uint32_t>(occ),
                         bucket_start.ptr, stream);
    // every NCCL call of this table is issued on the comm stream
    TSD_CUDA(cudaEventRecord(ev_ids, stream));
    TSD_CUDA(cudaStreamWaitEvent(comm, ev_ids, 0));
    h_counts.resize(static_cast<size_t>(U) * (nb() + 1));
    if (grp) {
      std::vector<uint32_t> mine(nb() + 1);
      TSD_CUDA(cudaMemcpyAsync(mine.data(), bucket_start.ptr, sizeof(uint32_t) * (nb() + 1),
                               cudaMemcpyDeviceToHost, comm));
      TSD_CUDA(cudaStreamSynchronize(comm));
      group_allgather(grp, g, mine.data(), sizeof(uint32_t) * (nb() + 1), h_counts.data());
    } else {
      TSD_NCCL(ncclAllGather(bucket_start.ptr, all_counts.ptr, nb() + 1, ncclUint32, world, comm));
      TSD_CUDA(cudaMemcpyAsync(h_counts.data(), all_counts.ptr, sizeof(uint32_t) * U * (nb() + 1),
                               cudaMemcpyDeviceToHost, comm));
      TSD_CUDA(cudaStreamSynchronize(comm));
    }
  }
  // Send layout: my remote buckets are contiguous in bucket order (RW by
  // server, then Flex by slot); receive layout is ordered by source rank
  // [p: RW from p | Flex from p] so server entries keep global occurrence
  // order.  layout.cpp computes both (unit-tested on the CPU).
  ExchangePlan xp;
  exchange_plan(N, W, g, h_counts.data(), &xp);
  send_off = xp.send_off;
  send_cnt = xp.send_cnt;
  recv_off = xp.recv_off;
  recv_cnt = xp.recv_cnt;
  recv_before = xp.recv_before;
  recv_total = xp.recv_total;
  n_remote = xp.n_remote;
  n_local_occ = occ - n_remote;
  recv_ids.ensure(recv_total);
  recv_rows.ensure(recv_total * cfg.dim);
  send_rows.ensure(std::max<uint64_t>(n_remote, 1) * cfg.dim);

  // ---- exchange chain on the comm stream, local gather on the compute
  // stream: the NVLink all-to-allv overlaps the HBM-bound local gather ------
  launch_remote_ids(d_rows, order.ptr, n_remote, d_local, send_ids.ptr, stream);
  TSD_CUDA(cudaEventRecord(ev_ids, stream));
  TSD_CUDA(cudaStreamWaitEvent(comm, ev_ids, 0));
  t = phase_begin(kPhaseExchangeFwd, comm);
  exchange(send_ids.ptr, send_off, send_cnt, recv_ids.ptr, recv_off, recv_cnt, sizeof(uint32_t), comm);
  // server side: rows requested by peers, in received order
  launch_copy_rows(d_w, recv_ids.ptr, recv_rows.ptr, nullptr, recv_total, cfg.dim, comm);
  exchange(recv_rows.ptr, recv_off, recv_cnt, send_rows.ptr, send_off, send_cnt,
           sizeof(float) * cfg.dim, comm);
  phase_end(t);
  t = phase_begin(kPhaseScatter, comm);
  launch_scatter_rows_loss(send_rows.ptr, d_out, order.ptr, n_remote, cfg.dim,
                           loss_partials.ptr + gather_grid, gather_grid, comm);
  phase_end(t);
  TSD_CUDA(cudaEventRecord(ev_fwd, comm));

  t = phase_begin(kPhaseGather);
  launch_gather_local(d_rows, occ, d_w, d_out, rv, cfg.dim, loss_partials.ptr, gather_grid, stream,
                      gather_bulk_stages);
  phase_end(t);
  TSD_CUDA(cudaStreamWaitEvent(stream, ev_fwd, 0));
  // loss = local-gather partials + scatter partials, fixed order
  launch_loss_finalize(loss_partials.ptr, 2 * gather_grid, d_loss.ptr, stream, loss_mirror);
}

// ---------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------

void ts_table::backward(const float* d_grad) {
  using namespace tsd;
  if (!last_rows && last_occ) fail(TS_ERR_VALIDATION, "table: backward without forward");
  const uint64_t occ = last_occ;
  const RemapView rv = remap_view();
  OptParams opt;
  opt.optimizer = cfg.optimizer;
  opt.lr = cfg.lr;
  opt.eps = cfg.eps;
  DenseRange d0, d1;
  GradSource gs;
  gs.local = d_grad;
  gs.n_local = static_cast<uint32_t>(occ);
  SegmentScratch sc;
  sc.long_list = long_list.ptr;
  sc.long_count = long_count.ptr;
  sc.piece_off = piece_off.ptr;
  sc.partials = partials.ptr;
  sc.short_max = seg_short_max;
  RadixBuffers rb{keys_a.ptr, vals_a.ptr, keys_b.ptr, vals_b.ptr, ghist.ptr, goff.ptr,
                  sort_status.ptr, sort_counters.ptr};
  uint32_t* sk = nullptr;
  uint32_t* sv = nullptr;
  const int key_bits = bits_for(local_rows ? local_rows - 1 : 0);

  if (U == 1) {
    // local id == canonical index: sort the forward's rows directly
    last_entries = occ;
    if (dedup_ready) {
      TSD_CUDA(cudaStreamWaitEvent(stream, ev_dedup_cur ? ev_dedup_cur : ev_dedup, 0));
      dedup_ready = false;
    } else {
      dedup_local(stream);
      if (long_concurrent) launch_long_segments(starts.ptr, seg_split.ptr, nseg.ptr, occ, seg_scratch_view(), stream);
    }
    sk = dd_keys;
    sv = dd_vals;
    if (long_concurrent) {
      // long segments (listed with the dedup) on aux, short ones here: they
      // update disjoint rows, and each kernel's tail fills the other's
      TSD_CUDA(cudaEventRecord(ev_seg0, stream));  // gradients + dedup ready
      TSD_CUDA(cudaStreamWaitEvent(aux, ev_seg0, 0));
      SegmentScratch lsc = sc;
      lsc.prefixed = true;
      int t = phase_begin(kPhaseSegmentLong, aux);
      launch_segment_long(sk, sv, starts.ptr, occ, cfg.dim, gs, d_w, d_state, opt, d0, d1, lsc, aux);
      phase_end(t);
      TSD_CUDA(cudaEventRecord(ev_long, aux));
      SegmentScratch ssc = sc;
      ssc.long_list = nullptr;  // listed already: skip, list nothing
      t = phase_begin(kPhaseSegmentUpdate);
      launch_segment_update(sk, sv, starts.ptr, seg_keys.ptr, seg_split.ptr, nseg.ptr, occ, cfg.dim, gs, d_w,
                            d_state, opt, d0, d1, ssc, stream);
      phase_end(t);
      TSD_CUDA(cudaStreamWaitEvent(stream, ev_long, 0));
      return;
    }
    int t = phase_begin(kPhaseSegmentUpdate);
    launch_segment_update(sk, sv, starts.ptr, seg_keys.ptr, seg_split.ptr, nseg.ptr, occ, cfg.dim, gs, d_w, d_state,
                          opt, d0, d1, sc, stream);
    phase_end(t);
    t = phase_begin(kPhaseSegmentLong);
    launch_segment_long(sk, sv, starts.ptr, occ, cfg.dim, gs, d_w, d_state, opt, d0, d1, sc, stream);
    phase_end(t);
    return;
  }

  if (p2p) {
    backward_p2p(d_grad);
    return;
  }

  // ---- comm stream: grads of remote occurrences -> their servers ------------
  TSD_CUDA(cudaEventRecord(ev_bwd0, stream));
  TSD_CUDA(cudaStreamWaitEvent(comm, ev_bwd0, 0));
  int t = phase_begin(kPhaseExchangeBwd, comm);
  launch_copy_rows(d_grad, order.ptr, send_rows.ptr, nullptr, n_remote, cfg.dim, comm);
  exchange(send_rows.ptr, send_off, send_cnt, recv_rows.ptr, recv_off, recv_cnt,
           sizeof(float) * cfg.dim, comm);
  phase_end(t);
  TSD_CUDA(cudaEventRecord(ev_grads, comm));

  // ---- compute stream, overlapped: keys/values need only ids, not grads ----
  gs.remote = recv_rows.ptr;
  const uint64_t m = n_local_occ + recv_total;
  last_entries = m;
  entry_keys.ensure(m);
  entry_vals.ensure(m);
  ensure_sort_capacity(m);
  rb = RadixBuffers{keys_a.ptr, vals_a.ptr, keys_b.ptr, vals_b.ptr, ghist.ptr, goff.ptr,
                    sort_status.ptr, sort_counters.ptr};
  sc.long_list = long_list.ptr;
  sc.piece_off = piece_off.ptr;
  sc.partials = partials.ptr;
  sc.short_max = seg_short_max;
  launch_build_entries(last_rows, order.ptr + n_remote, n_local_occ, rv, recv_ids.ptr, recv_before,
                       recv_total, static_cast<uint32_t>(occ), entry_keys.ptr, entry_vals.ptr, stream);
  // replicated tiers reduce into dense buffers: DP always, Flex across nodes
  if (dp_rows) {
    d0 = DenseRange{0, static_cast<uint32_t>(dp_rows), dense_dp.ptr};
    TSD_CUDA(cudaMemsetAsync(dense_dp.ptr, 0, sizeof(float) * dp_rows * cfg.dim, stream));
  }
  if (N > 1 && flex_rows) {
    d1 = DenseRange{static_cast<uint32_t>(dp_rows), static_cast<uint32_t>(dp_rows + flex_rows),
                    dense_flex.ptr};
    TSD_CUDA(cudaMemsetAsync(dense_flex.ptr, 0, sizeof(float) * flex_rows * cfg.dim, stream));
  }
  t = phase_begin(kPhaseSort);
  radix_sort_pairs(entry_keys.ptr, entry_vals.ptr, m, key_bits, rb, &sk, &sv, stream);
  phase_end(t);
  t = phase_begin(kPhaseSegments);
  segment_starts(sk, m, starts.ptr, seg_keys.ptr, nseg.ptr, seg_scratch.ptr, stream);
  // dense-reduced rows are the lowest local ids: split the segments there
  const uint32_t dense_hi = static_cast<uint32_t>(dp_rows + (N > 1 ? flex_rows : 0));
  launch_segment_split(sk, starts.ptr, nseg.ptr, dense_hi, seg_split.ptr, stream);
  phase_end(t);
  TSD_CUDA(cudaStreamWaitEvent(stream, ev_grads, 0));

  // ---- replicated rows first; their all-reduce overlaps the RW updates ----
  t = phase_begin(kPhaseSegmentUpdate);
  launch_segment_update(sk, sv, starts.ptr, seg_keys.ptr, seg_split.ptr, seg_split.ptr + 1, m, cfg.dim, gs, d_w,
                        d_state, opt, d0, d1, sc, stream);
  phase_end(t);
  t = phase_begin(kPhaseSegmentLong);
  launch_segment_long(sk, sv, starts.ptr, m, cfg.dim, gs, d_w, d_state, opt, d0, d1, sc, stream);
  phase_end(t);
  TSD_CUDA(cudaEventRecord(ev_dense, stream));
  TSD_CUDA(cudaStreamWaitEvent(comm, ev_dense, 0));
  t = phase_begin(kPhaseAllReduce, comm);
  if (grp) {
    // every rank calls both (collective), in the NCCL path's order
    std::vector<uint32_t> world_ranks(U), cross_ranks(N);
    for (uint32_t p = 0; p < U; ++p) world_ranks[p] = p;
    for (uint32_t k = 0; k < N; ++k) cross_ranks[k] = k * W + slot;
    group_allreduce(dense_dp.ptr, dp_rows * cfg.dim, world_ranks, comm);
    if (N > 1) group_allreduce(dense_flex.ptr, flex_rows * cfg.dim, cross_ranks, comm);
  } else {
    TSD_NCCL(ncclGroupStart());
    if (dp_rows) {
      TSD_NCCL(ncclAllReduce(dense_dp.ptr, dense_dp.ptr, dp_rows * cfg.dim, ncclFloat32, ncclSum, world, comm));
    }
    if (N > 1 && flex_rows) {
      TSD_NCCL(ncclAllReduce(dense_flex.ptr, dense_flex.ptr, flex_rows * cfg.dim, ncclFloat32, ncclSum,
                             cross, comm));
    }
    TSD_NCCL(ncclGroupEnd());
  }
  phase_end(t);
  TSD_CUDA(cudaEventRecord(ev_ar, comm));

  t = phase_begin(kPhaseSegmentUpdate);
  launch_segment_update(sk, sv, starts.ptr, seg_keys.ptr, seg_split.ptr + 1, nseg.ptr, m, cfg.dim, gs, d_w, d_state,
                        opt, d0, d1, sc, stream);
  phase_end(t);
  t = phase_begin(kPhaseSegmentLong);
  launch_segment_long(sk, sv, starts.ptr, m, cfg.dim, gs, d_w, d_state, opt, d0, d1, sc, stream);
  phase_end(t);
  TSD_CUDA(cudaStreamWaitEvent(stream, ev_ar, 0));
  t = phase_begin(kPhaseDenseUpdate);
  if (dp_rows) {
    launch_dense_update(dense_dp.ptr, static_cast<uint32_t>(dp_rows), 0, cfg.dim, d_w, d_state, opt, stream);
  }
  if (N > 1 && flex_rows) {
    launch_dense_update(dense_flex.ptr, static_cast<uint32_t>(flex_rows), static_cast<uint32_t>(dp_rows),
                        cfg.dim, d_w, d_state, opt, stream);
  }
  phase_end(t);
}

// ---------------------------------------------------------------------------
// peer-memory forward / backward (U > 1, one node)
// ---------------------------------------------------------------------------

void ts_table::forward_p2p_pull(const uint32_t* d_rows, uint64_t occ, float* d_out) {
  using namespace tsd;
  const RemapView rv = remap_view();
  const size_t P = step_payload_bytes();
  uint8_t* my_slot = (flag_barriers ? mbox.ptr : xfer.ptr) + P * g;

  // ---- route (compute stream): request lists for the backward ------------
  int t = phase_begin(kPhaseRoute);
  BucketView bv;
  bv.dest = d_dest;
  bv.dp_cut = cfg.dp_cut;
  bv.flex_cut = cfg.flex_cut;
  bv.u = U;
  bv.w = W;
  bv.rank = g;
  bv.slot = slot;
  launch_bucket_keys(d_rows, occ, bv, bucket.ptr, tier_counts.ptr, stream);
  RadixBuffers rb{keys_a.ptr, vals_a.ptr, keys_b.ptr, vals_b.ptr, ghist.ptr, goff.ptr,
                  sort_status.ptr, sort_counters.ptr};
  uint32_t* sorted_b = nullptr;
  uint32_t* sorted_i = nullptr;
  radix_sort_pairs(bucket.ptr, nullptr, occ, bits_for(nb() - 1), rb, &sorted_b, &sorted_i, stream);
  TSD_CUDA(cudaMemcpyAsync(order.ptr, sorted_i, sizeof(uint32_t) * occ, cudaMemcpyDeviceToDevice, stream));
  uint32_t* my_starts = reinterpret_cast<uint32_t*>(my_slot);
  launch_bucket_starts(goff.ptr, 1, nb(), static_cast<uint32_t>(occ), my_starts, stream);
  launch_remote_ids_upto(d_rows, order.ptr, occ, my_starts + (U + W), d_local, send_ids.ptr, stream);
  phase_end(t);
  TSD_CUDA(cudaEventRecord(ev_ids, stream));

  // ---- every rank's previous update done, then the rows: local ones on
  // the compute stream, remote ones pulled over NVLink on aux -------------
  if (grp) {
    group_barrier(grp, g, stream);
  } else {
    launch_flag_barrier(flag_barrier, 1, ++step_barrier_seq, stream);
  }
  if (rep_pending) {
    TSD_CUDA(cudaStreamWaitEvent(stream, ev_rep, 0));
    rep_pending = false;
  }
  TSD_CUDA(cudaEventRecord(ev_fwd0, stream));  // shards final everywhere
  PeerWeights pw;
  for (uint32_t p = 0; p < U; ++p) pw.w[p] = peer_w[p];
  pw.node_base = node * W;
  t = phase_begin(kPhaseGather);
  launch_gather_local(d_rows, occ, d_w, d_out, rv, cfg.dim, loss_partials.ptr, fwd_gather_grid, stream,
                      gather_bulk_stages);
  phase_end(t);
  cudaStream_t rs = aux ? aux : comm;
  TSD_CUDA(cudaStreamWaitEvent(rs, ev_fwd0, 0));
  t = phase_begin(kPhaseExchangeFwd, rs);
  {
    static const unsigned per_sm = [] {
      const char* e = std::getenv("TIERSHARD_PULL_BLOCKS");
      return e ? static_cast<unsigned>(std::max(1, std::atoi(e))) : 2u;
    }();
    const unsigned grid = static_cast<unsigned>(
        std::min<uint64_t>(per_sm * static_cast<uint64_t>(sm_count()), remote_loss_slots));
    launch_pull_rows(sorted_b, order.ptr, send_ids.ptr, my_starts + (U + W), occ, pw, U, d_out, cfg.dim,
                     loss_partials.ptr + gather_grid, grid, rs);
  }
  phase_end(t);
  TSD_CUDA(cudaEventRecord(ev_fwd, rs));
  TSD_CUDA(cudaStreamWaitEvent(stream, ev_fwd, 0));
  launch_loss_finalize(loss_partials.ptr, static_cast<unsigned>(gather_grid + remote_loss_slots), d_loss.ptr,
                       stream, loss_mirror);

  // ---- comm stream, beside the gather: counts, then the request lists -----
  TSD_CUDA(cudaStreamWaitEvent(comm, ev_ids, 0));
  h_xfer.resize(P * U);
  if (grp) {
    std::vector<uint8_t> mine(P);
    TSD_CUDA(cudaMemcpyAsync(mine.data(), my_slot, P, cudaMemcpyDeviceToHost, comm));
    TSD_CUDA(cudaStreamSynchronize(comm));
    group_allgather(grp, g, mine.data(), P, h_xfer.data());
  } else {
    launch_mailbox_put(mbox_put, my_slot, P, P * g, comm);
    barrier_on_comm();
    TSD_CUDA(cudaMemcpyAsync(h_xfer.data(), mbox.ptr, P * U, cudaMemcpyDeviceToHost, comm));
    TSD_CUDA(cudaStreamSynchronize(comm));
  }
  h_counts.resize(static_cast<size_t>(U) * (nb() + 1));
  for (uint32_t p = 0; p < U; ++p) {
    std::memcpy(h_counts.data() + size_t{p} * (nb() + 1), h_xfer.data() + P * p, (nb() + 1) * 4);
  }
  ExchangePlan xp;
  exchange_plan(N, W, g, h_counts.data(), &xp);
  send_off = xp.send_off;
  send_cnt = xp.send_cnt;
  recv_off = xp.recv_off;
  recv_cnt = xp.recv_cnt;
  recv_before = xp.recv_before;
  recv_total = xp.recv_total;
  n_remote = xp.n_remote;
  n_local_occ = occ - n_remote;
  {
    std::vector<uint64_t> need(U);
    for (uint32_t p = 0; p < U; ++p) {
      ExchangePlan pp;
      exchange_plan(N, W, p, h_counts.data(), &pp);
      need[p] = pp.recv_total;
    }
    regrow_recv(need);
  }
  recv_ids.ensure(recv_total);
  recv_pos.ensure(recv_total);
  PullTable pt{};
  const auto start_of = [&](uint32_t p, uint32_t b) -> uint64_t { return h_counts[size_t{p} * (nb() + 1) + b]; };
  for (uint32_t p = 0; p < U; ++p) {
    if (p == g) continue;
    if (recv_cnt[2 * p]) {
      pt.seg[pt.nseg++] = PullSeg{peer_ids[p], peer_pos[p], start_of(p, g), recv_off[2 * p], recv_cnt[2 * p]};
    }
    if (recv_cnt[2 * p + 1]) {
      pt.seg[pt.nseg++] = PullSeg{peer_ids[p], peer_pos[p], start_of(p, U + slot), recv_off[2 * p + 1],
                                  recv_cnt[2 * p + 1]};
    }
  }
  pt.total = recv_total;
  if (aux) {
    const uint64_t m = n_local_occ + recv_total;
    entry_keys.ensure(m);
    entry_vals.ensure(m);
    ensure_sort_capacity(m);
  }
  t = phase_begin(kPhaseExchangeFwd, comm);
  launch_pull_requests(pt, recv_ids.ptr, recv_pos.ptr, comm);
  phase_end(t);
  if (aux) {  // the backward's dedup needs only the ids
    TSD_CUDA(cudaEventRecord(ev_fwd0, comm));
    TSD_CUDA(cudaStreamWaitEvent(dedup_stream(), ev_fwd0, 0));
    dedup_p2p(dedup_stream());
    TSD_CUDA(cudaEventRecord(ev_dedup, dedup_stream()));
    dedup_ready = true;
  }
}

void ts_table::forward_p2p(const uint32_t* d_rows, uint64_t occ, float* d_out) {
  using namespace tsd;
  const RemapView rv = remap_view();
  const size_t P = step_payload_bytes();
  const size_t starts_bytes = P - sizeof(IpcExport);
  // mailbox mode: the payload goes through the peers' mailboxes, so the
  // local gather is queued before the exchange of counts (no NCCL kernel
  // for it to starve of SMs) and runs while the host waits for them
  uint8_t* my_slot = (mailbox_counts ? mbox.ptr : xfer.ptr) + P * g;

  // ---- route: bucket + one stable counting pass; request lists in HBM -----
  int t = phase_begin(kPhaseRoute);
  BucketView bv;
  bv.dest = d_dest;
  bv.dp_cut = cfg.dp_cut;
  bv.flex_cut = cfg.flex_cut;
  bv.u = U;
  bv.w = W;
  bv.rank = g;
  bv.slot = slot;
  uint32_t* my_starts = reinterpret_cast<uint32_t*>(my_slot);
  if (route_sort) {  // TIERSHARD_ROUTE=sort: bucket keys + the radix sort (round 1)
    launch_bucket_keys(d_rows, occ, bv, bucket.ptr, tier_counts.ptr, stream);
    RadixBuffers rb{keys_a.ptr, vals_a.ptr, keys_b.ptr, vals_b.ptr, ghist.ptr, goff.ptr,
                    sort_status.ptr, sort_counters.ptr};
    uint32_t* sorted_b = nullptr;
    uint32_t* sorted_i = nullptr;
    radix_sort_pairs(bucket.ptr, nullptr, occ, bits_for(nb() - 1), rb, &sorted_b, &sorted_i, stream);
    TSD_CUDA(cudaMemcpyAsync(order.ptr, sorted_i, sizeof(uint32_t) * occ, cudaMemcpyDeviceToDevice, stream));
    launch_bucket_starts(goff.ptr, 1, nb(), static_cast<uint32_t>(occ), my_starts, stream);
    // ids of the remote prefix (the local bucket is last; its count is on the device)
    launch_remote_ids_upto(d_rows, order.ptr, occ, my_starts + (U + W), d_local, send_ids.ptr, stream);
  } else {  // histogram, scan, stable scatter with the remote ids fused
    launch_route_buckets(d_rows, occ, bv, nb(), route_hist.ptr, order.ptr, my_starts, d_local, send_ids.ptr,
                         tier_counts.ptr, stream);
  }
  {  // the slot keeps the export between steps: rewrite it only when the
     // output moves (a copy-engine op between the route kernels otherwise)
    const IpcExport e = export_ptr(d_out);
    if (!export_in_slot || std::memcmp(&e, &my_export, sizeof(e)) != 0) {
      my_export = e;
      TSD_CUDA(cudaMemcpyAsync(my_slot + starts_bytes, &my_export, sizeof(IpcExport), cudaMemcpyHostToDevice,
                               stream));
      export_in_slot = true;
    }
  }
  phase_end(t);

  // ---- one all-gather: every rank's bucket starts + output export --------
  // (also the rendezvous after which peers may read our request lists)
  TSD_CUDA(cudaEventRecord(ev_ids, stream));
  TSD_CUDA(cudaStreamWaitEvent(comm, ev_ids, 0));
  h_xfer.resize(P * U);
  const bool rep_wait = rep_pending;  // the previous step's deferred replica broadcasts
  if (rep_pending) {
    TSD_CUDA(cudaStreamWaitEvent(stream, ev_rep, 0));
    rep_pending = false;
  }
  if (mailbox_counts) {
    t = phase_begin(kPhaseGather);
    launch_gather_local(d_rows, occ, d_w, d_out, rv, cfg.dim, loss_partials.ptr, fwd_gather_grid, stream,
                        gather_bulk_stages);
    phase_end(t);
    launch_mailbox_put(mbox_put, my_slot, P, P * g, comm);
    barrier_on_comm();
    TSD_CUDA(cudaMemcpyAsync(h_xfer.data(), mbox.ptr, P * U, cudaMemcpyDeviceToHost, comm));
    TSD_CUDA(cudaStreamSynchronize(comm));
  } else if (grp) {
    // in-process: this rank's slot to the host, then a host all-gather.
    // Every rank synchronised its comm stream (which waited for the route)
    // before the gather, so the request lists are complete before any pull
    // -- at least the ordering the NCCL all-gather gives
    std::vector<uint8_t> mine(P);
    TSD_CUDA(cudaMemcpyAsync(mine.data(), my_slot, P, cudaMemcpyDeviceToHost, comm));
    TSD_CUDA(cudaStreamSynchronize(comm));
    group_allgather(grp, g, mine.data(), P, h_xfer.data());
  } else {
    TSD_NCCL(ncclAllGather(my_slot, xfer.ptr, P, ncclUint8, world, comm));
    TSD_CUDA(cudaMemcpyAsync(h_xfer.data(), xfer.ptr, P * U, cudaMemcpyDeviceToHost, comm));
    TSD_CUDA(cudaStreamSynchronize(comm));
  }
  h_counts.resize(static_cast<size_t>(U) * (nb() + 1));
  std::vector<float*> peer_out(U, nullptr);
  for (uint32_t p = 0; p < U; ++p) {
    std::memcpy(h_counts.data() + size_t{p} * (nb() + 1), h_xfer.data() + P * p, (nb() + 1) * 4);
    if (p == g) continue;
    IpcExport e;
    std::memcpy(&e, h_xfer.data() + P * p + starts_bytes, sizeof(e));
    peer_out[p] = static_cast<float*>(peers.open(static_cast<int>(p), e));
  }
  ExchangePlan xp;
  exchange_plan(N, W, g, h_counts.data(), &xp);
  send_off = xp.send_off;
  send_cnt = xp.send_cnt;
  recv_off = xp.recv_off;
  recv_cnt = xp.recv_cnt;
  recv_before = xp.recv_before;
  recv_total = xp.recv_total;
  n_remote = xp.n_remote;
  n_local_occ = occ - n_remote;
  {  // bounded receive buffers: grow (collectively) where this step needs it
    std::vector<uint64_t> need(U);
    for (uint32_t p = 0; p < U; ++p) {
      ExchangePlan pp;
      exchange_plan(N, W, p, h_counts.data(), &pp);
      need[p] = pp.recv_total;
    }
    regrow_recv(need);
  }
  recv_ids.ensure(recv_total);
  recv_pos.ensure(recv_total);

  // ---- comm stream: pull request lists, serve rows into peers' outputs ----
  PullTable pt{};
  ServeTable st{};
  const auto start_of = [&](uint32_t p, uint32_t b) -> uint64_t { return h_counts[size_t{p} * (nb() + 1) + b]; };
  for (uint32_t p = 0; p < U; ++p) {
    if (p == g) continue;
    if (recv_cnt[2 * p]) {
      pt.seg[pt.nseg++] = PullSeg{peer_ids[p], peer_pos[p], start_of(p, g), recv_off[2 * p], recv_cnt[2 * p]};
    }
    if (recv_cnt[2 * p + 1]) {
      pt.seg[pt.nseg++] = PullSeg{peer_ids[p], peer_pos[p], start_of(p, U + slot), recv_off[2 * p + 1],
                                  recv_cnt[2 * p + 1]};
    }
    ServeTarget& tg = st.t[st.n++];
    tg.out = peer_out[p];
    tg.loss_slots = peer_loss[p] + static_cast<uint64_t>(g) * kServeGrid;
    tg.r_begin = recv_off[2 * p];
    tg.r_end = recv_off[2 * p] + recv_cnt[2 * p] + recv_cnt[2 * p + 1];
  }
  pt.total = recv_total;
  if (aux) {  // buffers the aux dedup needs, sized before any of it is queued
    const uint64_t m = n_local_occ + recv_total;
    entry_keys.ensure(m);
    entry_vals.ensure(m);
    ensure_sort_capacity(m);
  }
  t = phase_begin(kPhaseExchangeFwd, comm);
  launch_pull_requests(pt, recv_ids.ptr, recv_pos.ptr, comm);
  if (aux) {  // the backward's dedup needs only the ids: overlap it with the gather / serve
    TSD_CUDA(cudaEventRecord(ev_fwd0, comm));
    TSD_CUDA(cudaStreamWaitEvent(dedup_stream(), ev_fwd0, 0));
    dedup_p2p(dedup_stream());
    TSD_CUDA(cudaEventRecord(ev_dedup, dedup_stream()));
    dedup_ready = true;
  }
  // served Flex rows replicated across nodes are written by the deferred
  // replica update: the serve waits for it (DP rows are never served)
  if (rep_wait && N > 1 && flex_rows) TSD_CUDA(cudaStreamWaitEvent(comm, ev_rep, 0));
  launch_serve_rows(d_w, recv_ids.ptr, recv_pos.ptr, st, cfg.dim, comm);
  barrier_on_comm();  // every server has finished storing into every output
  phase_end(t);
  TSD_CUDA(cudaEventRecord(ev_fwd, comm));

  if (!mailbox_counts) {
    t = phase_begin(kPhaseGather);
    launch_gather_local(d_rows, occ, d_w, d_out, rv, cfg.dim, loss_partials.ptr, fwd_gather_grid, stream,
                        gather_bulk_stages);
    phase_end(t);
  }
  TSD_CUDA(cudaStreamWaitEvent(stream, ev_fwd, 0));
  launch_loss_finalize(loss_partials.ptr, static_cast<unsigned>(gather_grid + remote_loss_slots), d_loss.ptr,
                       stream, loss_mirror);
}

// Segments [*d_lo, *d_hi): short ones on the compute stream, long ones listed
// and reduced on aux beside them (disjoint rows); the compute stream joins.
void ts_table::segment_range_concurrent(const uint32_t* sk, const uint32_t* sv, const uint32_t* d_lo,
                                        const uint32_t* d_hi, uint64_t m, const tsd::GradSource& gs,
                                        const tsd::OptParams& opt, const tsd::DenseRange& d0,
                                        const tsd::DenseRange& d1) {
  using namespace tsd;
  const SegmentScratch sc = seg_scratch_view();
  TSD_CUDA(cudaEventRecord(ev_seg0, stream));  // gradients + segments ready
  TSD_CUDA(cudaStreamWaitEvent(aux, ev_seg0, 0));
  int t = phase_begin(kPhaseSegmentLong, aux);
  launch_long_segments(starts.ptr, d_lo, d_hi, m, sc, aux);
  SegmentScratch lsc = sc;
  lsc.prefixed = true;
  launch_segment_long(sk, sv, starts.ptr, m, cfg.dim, gs, d_w, d_state, opt, d0, d1, lsc, aux);
  phase_end(t);
  TSD_CUDA(cudaEventRecord(ev_long, aux));
  SegmentScratch ssc = sc;
  ssc.long_list = nullptr;
  t = phase_begin(kPhaseSegmentUpdate);
  launch_segment_update(sk, sv, starts.ptr, seg_keys.ptr, d_lo, d_hi, m, cfg.dim, gs, d_w, d_state, opt, d0, d1,
                        ssc, stream);
  phase_end(t);
  TSD_CUDA(cudaStreamWaitEvent(stream, ev_long, 0));
}

void ts_table::backward_p2p(const float* d_grad) {
  using namespace tsd;
  const uint64_t occ = last_occ;
  const RemapView rv = remap_view();
  OptParams opt;
  opt.optimizer = cfg.optimizer;
  opt.lr = cfg.lr;
  opt.eps = cfg.eps;
  DenseRange d0, d1;
  const uint64_t m = n_local_occ + recv_total;
  last_entries = m;
  SegmentScratch sc;
  sc.long_list = long_list.ptr;
  sc.long_count = long_count.ptr;
  sc.piece_off = piece_off.ptr;
  sc.partials = partials.ptr;
  sc.short_max = seg_short_max;

  // ---- entries, sort, segments (no gradient needed): done by the forward on
  // the aux stream when prefetched, else here on the compute stream -------
  TSD_CUDA(cudaEventRecord(ev_bwd0, stream));  // our gradient is complete here
  const bool prefetched = dedup_ready;
  // replicated rows' partials are pushed to their owners' receive slots and
  // stamped with the step's epoch (no clears; untouched slots are ignored)
  if (++epoch == 0) epoch = 1;  // (2^32 steps) 0 is the initial stamp
  if (dp_rows) {
    d0.lo = 0;
    d0.hi = static_cast<uint32_t>(dp_rows);
    d0.epoch = epoch;
    d0.push_n = U;
    d0.per = per_dp;
    d0.interleave = replica_interleave;
    d0.me = g;
    const uint64_t set = replica_deferred ? (epoch & 1u) : 0;
    for (uint32_t p = 0; p < U; ++p) {
      d0.push_grad[p] = peer_dense_dp[p] + set * dp_set_elems * cfg.dim;
      d0.push_stamp[p] = peer_stamp_dp[p] + set * dp_set_elems;
    }
  }
  if (N > 1 && flex_rows) {  // group: the same slot in every node, node order
    d1.lo = static_cast<uint32_t>(dp_rows);
    d1.hi = static_cast<uint32_t>(dp_rows + flex_rows);
    d1.epoch = epoch;
    d1.push_n = N;
    d1.per = per_flex;
    d1.interleave = replica_interleave;
    d1.me = node;
    const uint64_t set = replica_deferred ? (epoch & 1u) : 0;
    for (uint32_t k = 0; k < N; ++k) {
      d1.push_grad[k] = peer_dense_flex[k * W + slot] + set * flex_set_elems * cfg.dim;
      d1.push_stamp[k] = peer_stamp_flex[k * W + slot] + set * flex_set_elems;
    }
  }
  // ---- remote gradient rows -> their servers -------------------------------
  // push (default): after one all-gather of the servers' receive buffers
  // (the rendezvous after which every rank's gradient is complete), each
  // rank STORES the gradients of its remote occurrences into its servers'
  // receive slots (the order the servers pulled our request lists in), then
  // a barrier; pull (TIERSHARD_GRADS=pull): each server gathers them from
  // the requesters' gradient buffers with peer loads.  Either way the remote
  // rows end up in local HBM, recv_rows[r] for received entry r.  The
  // transfer kernel runs on `xs`: the comm stream (overlapping the sort) or,
  // with TIERSHARD_PUSH_ORDER=first, the compute stream ahead of the sort.
  const auto exchange_grads = [&](cudaStream_t xs) {
    TSD_CUDA(cudaStreamWaitEvent(comm, ev_bwd0, 0));
    int tx = phase_begin(kPhaseExchangeBwd, xs);
    if (recv_total * cfg.dim > recv_rows.cap) fail(TS_ERR_INTERNAL, "table: receive buffer overflow");
    if (grads_push) {
      // the receive buffers never move (mapped at setup), and the forward's
      // all-gather already ordered every server's previous reads of them
      // before this step: no rendezvous, no host sync before the push
      PushTable pt{};
      // the grid strides through the runs in table order, so every rank
      // starts with a different server (g+1, g+2, ...): in rank order all
      // of them would store into rank 0 first, then rank 1, ... (incast)
      for (uint32_t i = 1; i < U; ++i) {
        const uint32_t p = push_rotate ? (g + i) % U : (i <= g ? i - 1 : i);
        float* server_recv = peer_recv_rows[p];
        ExchangePlan sp;  // server p's receive layout: which slots hold our entries
        exchange_plan(N, W, p, h_counts.data(), &sp);
        for (int part = 0; part < 2; ++part) {
          const uint64_t cnt = send_cnt[2 * p + part];
          if (!cnt) continue;
          pt.run_start[pt.n] = pt.n ? pt.run_start[pt.n - 1] + pt.run[pt.n - 1].count : 0;
          pt.run[pt.n++] = PushRun{send_off[2 * p + part], cnt, server_recv + sp.recv_off[2 * g + part] * cfg.dim};
        }
      }
      pt.run_start[pt.n] = pt.n ? pt.run_start[pt.n - 1] + pt.run[pt.n - 1].count : 0;
      launch_push_grads(pt, order.ptr, d_grad, cfg.dim, xs);
      if (xs != comm) {
        TSD_CUDA(cudaEventRecord(ev_dense, xs));
        TSD_CUDA(cudaStreamWaitEvent(comm, ev_dense, 0));
      }
      barrier_on_comm();  // every requester's rows have landed in every server
    } else {
      const IpcExport mine = export_ptr(d_grad);
      const std::vector<uint8_t> all = allgather_bytes(&mine, sizeof(mine));
      PullGrads pg{};
      for (uint32_t p = 0; p < U; ++p) {
        if (p == g) continue;
        IpcExport e;
        std::memcpy(&e, all.data() + sizeof(e) * p, sizeof(e));
        pg.src_start[pg.nsrc] = static_cast<uint32_t>(recv_off[2 * p]);
        pg.src[pg.nsrc++] = static_cast<const float*>(peers.open(static_cast<int>(p), e));
      }
      pg.src_start[pg.nsrc] = static_cast<uint32_t>(recv_total);
      launch_pull_grads(pg, recv_pos.ptr, recv_total, recv_rows.ptr, cfg.dim, xs);
      if (xs != comm) {
        TSD_CUDA(cudaEventRecord(ev_dense, xs));
        TSD_CUDA(cudaStreamWaitEvent(comm, ev_dense, 0));
      }
    }
    phase_end(tx);
    TSD_CUDA(cudaEventRecord(ev_grads, comm));
  };
  if (push_first) exchange_grads(stream);
  if (prefetched) {
    TSD_CUDA(cudaStreamWaitEvent(stream, ev_dedup, 0));
    dedup_ready = false;
  } else {
    dedup_p2p(stream);
  }
  uint32_t* sk = dd_keys;
  uint32_t* sv = dd_vals;
  int t = -1;

  if (!push_first) exchange_grads(comm);
  GradSource gs;
  gs.local = d_grad;
  gs.n_local = static_cast<uint32_t>(occ);
  gs.remote = recv_rows.ptr;

  // ---- replicated rows first; their reduction overlaps the RW updates.  The
  // DP segments hold local entries only (a DP row is served by its
  // requester), so they start without the remote rows, beside the gradient
  // push; Flex rows replicated across nodes (N > 1) need them.
  const auto seg_range = [&](const uint32_t* d_lo, const uint32_t* d_hi) {
    if (long_concurrent) {
      segment_range_concurrent(sk, sv, d_lo, d_hi, m, gs, opt, d0, d1);
      return;
    }
    int tt = phase_begin(kPhaseSegmentUpdate);
    launch_segment_update(sk, sv, starts.ptr, seg_keys.ptr, d_lo, d_hi, m, cfg.dim, gs, d_w, d_state, opt, d0, d1,
                          sc, stream);
    phase_end(tt);
    tt = phase_begin(kPhaseSegmentLong);
    launch_segment_long(sk, sv, starts.ptr, m, cfg.dim, gs, d_w, d_state, opt, d0, d1, sc, stream);
    phase_end(tt);
  };
  if (N > 1 && flex_rows) {
    seg_range(seg_split.ptr + 2, seg_split.ptr + 3);  // DP: [0, split at dp_rows)
    TSD_CUDA(cudaStreamWaitEvent(stream, ev_grads, 0));
    seg_range(seg_split.ptr + 3, seg_split.ptr + 1);  // Flex: up to the replicated bound
  } else {
    seg_range(seg_split.ptr, seg_split.ptr + 1);
    TSD_CUDA(cudaStreamWaitEvent(stream, ev_grads, 0));
  }
  // ---- replicated tiers over peer memory: after a rendezvous (all ranks'
  // partials written), each rank reduces its slice of the replicated rows in
  // group-rank order, updates it and broadcasts it to every replica --------
  TSD_CUDA(cudaEventRecord(ev_dense, stream));
  TSD_CUDA(cudaStreamWaitEvent(comm, ev_dense, 0));
  cudaStream_t rs = replica_deferred ? rep : (replica_concurrent ? comm : stream);
  t = phase_begin(kPhaseRendezvous, comm);
  barrier_on_comm();
  phase_end(t);
  if (replica_deferred) {
    TSD_CUDA(cudaEventRecord(ev_rv, comm));
    TSD_CUDA(cudaStreamWaitEvent(rep, ev_rv, 0));
  }
  const uint64_t rset = replica_deferred ? (epoch & 1u) : 0;
  if (!replica_concurrent && !replica_deferred) {
    TSD_CUDA(cudaEventRecord(ev_ar, comm));
    TSD_CUDA(cudaStreamWaitEvent(stream, ev_ar, 0));
  }
  t = phase_begin(kPhaseReplicaUpdate, rs);
  if (dp_rows) {
    ReplicaGroup grp;
    grp.size = static_cast<int>(U);
    grp.me = static_cast<int>(g);
    grp.rows = static_cast<uint32_t>(dp_rows);
    grp.row_lo = 0;
    grp.recv = dense_dp.ptr + rset * dp_set_elems * cfg.dim;
    grp.recv_stamp = stamp_dp.ptr + rset * dp_set_elems;
    grp.per = per_dp;
    grp.interleave = replica_interleave;
    grp.epoch = epoch;
    for (uint32_t p = 0; p < U; ++p) {
      grp.weights[p] = peer_w[p];
      grp.state[p] = peer_state[p];
    }
    launch_replica_update(grp, cfg.dim, opt, rs);
  }
  if (N > 1 && flex_rows) {
    ReplicaGroup grp;  // same slot in every node, node order
    grp.size = static_cast<int>(N);
    grp.me = static_cast<int>(node);
    grp.rows = static_cast<uint32_t>(flex_rows);
    grp.row_lo = static_cast<uint32_t>(dp_rows);
    for (uint32_t k = 0; k < N; ++k) {
      const uint32_t p = k * W + slot;
      grp.weights[k] = peer_w[p] + dp_rows * cfg.dim;
      grp.state[k] = peer_state[p] ? peer_state[p] + dp_rows : nullptr;
    }
    grp.recv = dense_flex.ptr + rset * flex_set_elems * cfg.dim;
    grp.recv_stamp = stamp_flex.ptr + rset * flex_set_elems;
    grp.per = per_flex;
    grp.interleave = replica_interleave;
    grp.epoch = epoch;
    launch_replica_update(grp, cfg.dim, opt, rs);
  }
  phase_end(t);
  if (replica_deferred) {
    // every owner's broadcast has landed everywhere once this completes
    if (grp) {
      group_barrier(this->grp, g, rep);
    } else {
      launch_flag_barrier(flag_barrier, 2, ++rep_barrier_seq, rep);
    }
    TSD_CUDA(cudaEventRecord(ev_rep, rep));
    rep_pending = true;
  } else if (replica_concurrent) {
    TSD_CUDA(cudaEventRecord(ev_ar, comm));
  }
  if (long_concurrent) {
    segment_range_concurrent(sk, sv, seg_split.ptr + 1, nseg.ptr, m, gs, opt, d0, d1);
  } else {
    t = phase_begin(kPhaseSegmentUpdate);
    launch_segment_update(sk, sv, starts.ptr, seg_keys.ptr, seg_split.ptr + 1, nseg.ptr, m, cfg.dim, gs, d_w,
                          d_state, opt, d0, d1, sc, stream);
    phase_end(t);
    t = phase_begin(kPhaseSegmentLong);
    launch_segment_long(sk, sv, starts.ptr, m, cfg.dim, gs, d_w, d_state, opt, d0, d1, sc, stream);
    phase_end(t);
  }
  if (replica_concurrent && !replica_deferred) TSD_CUDA(cudaStreamWaitEvent(stream, ev_ar, 0));
  // peers store into our replicated rows: the next step's rendezvous (its
  // all-gather on the comm stream, after this stream's work) orders those
  // stores before any of our reads
  TSD_CUDA(cudaEventRecord(ev_ar, stream));
  TSD_CUDA(cudaStreamWaitEvent(comm, ev_ar, 0));
}

void ts_table::train_step(const uint32_t* d_rows, uint64_t occ, float* d_out) {
  using namespace tsd;
  if (!step_graph || timing) {
    forward(d_rows, occ, d_out);
    backward(d_out);  // loss = 0.5*|out|^2  =>  d loss / d out = out
    return;
  }
  // a previous forward without backward left its prefetched dedup running:
  // wait for it here (a capture may not wait on an event recorded outside it)
  if (dedup_ready) {
    TSD_CUDA(cudaStreamWaitEvent(stream, ev_dedup, 0));
    dedup_ready = false;
  }
  cudaGraph_t graph = nullptr;
  TSD_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
  try {
    forward(d_rows, occ, d_out);
    backward(d_out);
  } catch (...) {
    cudaStreamEndCapture(stream, &graph);  // leave capture mode before reporting
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    throw;
  }
  TSD_CUDA(cudaStreamEndCapture(stream, &graph));
  bool updated = false;
  if (step_exec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(step_exec, graph, &info) == cudaSuccess) {
      updated = true;
      ++graph_updates;
    } else {
      cudaGetLastError();
      cudaGraphExecDestroy(step_exec);
      step_exec = nullptr;
    }
  }
  if (!updated) {
    const cudaError_t e = cudaGraphInstantiate(&step_exec, graph, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(graph);
      TSD_CUDA(e);
    }
    ++graph_instantiations;
  }
  cudaGraphDestroy(graph);
  TSD_CUDA(cudaGraphLaunch(step_exec, stream));
}

void ts_table::destroy() {
  cudaSetDevice(cfg.device);
  if (step_exec) cudaGraphExecDestroy(step_exec);
  step_exec = nullptr;
  if (stream) cudaStreamSynchronize(stream);
  if (aux) cudaStreamSynchronize(aux);
  if (rep) cudaStreamSynchronize(rep);
  if (pre) cudaStreamSynchronize(pre);
  if (dd) cudaStreamSynchronize(dd);
  if (ready && p2p) {
    // peers may still be storing into our exported buffers (replica rows,
    // gradient receive slots): a rendezvous before anything is freed
    try {
      barrier_on_comm();
    } catch (const tsd::Failure&) {
    }
  }
  if (comm) cudaStreamSynchronize(comm);
  if (grp && attached) {
    try {
      if (ready) tsd::group_wait(grp);  // every rank is past its last rendezvous
    } catch (const tsd::Failure&) {
    }
    tsd::group_detach(grp, g);
    attached = false;
  }
  if (world) ncclCommDestroy(world);
  if (intra) ncclCommDestroy(intra);
  if (cross) ncclCommDestroy(cross);
  cudaFree(d_w);
  cudaFree(d_state);
  cudaFree(d_dest);
  cudaFree(d_local);
  for (auto* b : {&loss_partials}) b->release();
  d_loss.release();
  tier_counts.release();
  rows_dev.release();
  host_out.release();
  sort_status.release();
  seg_split.release();
  seg_keys.release();
  for (auto* b : {&keys_a, &vals_a, &keys_b, &vals_b, &ghist, &goff, &sort_counters, &starts,
                  &seg_scratch, &nseg, &long_list, &long_count, &piece_off, &entry_keys,
                  &entry_vals, &bucket, &order, &send_ids, &recv_ids, &bucket_start, &all_counts}) {
    b->release();
  }
  for (auto* b : {&partials, &send_rows, &recv_rows, &dense_dp, &dense_flex, &ar_tmp}) b->release();
  flag_box.release();
  mbox.release();
  stamp_dp.release();
  stamp_flex.release();
  for (auto& [a, b] : ev_pool) {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  for (cudaEvent_t e : {ev_ids, ev_fwd, ev_bwd0, ev_grads, ev_dense, ev_ar, ev_fwd0, ev_dedup, ev_seg0, ev_long}) {
    if (e) cudaEventDestroy(e);
  }
  if (aux) {
    cudaStreamSynchronize(aux);
    cudaStreamDestroy(aux);
  }
  if (copy) {
    cudaStreamSynchronize(copy);
    cudaStreamDestroy(copy);
  }
  for (cudaEvent_t e : {ev_copied[0], ev_copied[1], ev_consumed[0], ev_consumed[1]}) {
    if (e) cudaEventDestroy(e);
  }
  rows_dev2.release();
  if (h_loss_pinned) cudaFreeHost(h_loss_pinned);
  if (comm) cudaStreamDestroy(comm);
  if (rep) cudaStreamDestroy(rep);
  if (pre) cudaStreamDestroy(pre);
  for (cudaEvent_t e : {ev_pre[0], ev_pre[1], ev_gather_done}) {
    if (e) cudaEventDestroy(e);
  }
  for (auto* b : {&alt.keys_a, &alt.vals_a, &alt.keys_b, &alt.vals_b, &alt.ghist, &alt.goff, &alt.sort_counters,
                  &alt.starts, &alt.seg_keys, &alt.seg_scratch, &alt.nseg, &alt.seg_split, &alt.long_list,
                  &alt.long_count, &alt.piece_off}) {
    b->release();
  }
  alt.sort_status.release();
  for (cudaEvent_t e : {ev_rv, ev_rep}) {
    if (e) cudaEventDestroy(e);
  }
  if (stream) cudaStreamDestroy(stream);
  if (nccl_st) cudaStreamDestroy(nccl_st);
  if (dd) cudaStreamDestroy(dd);
  tsd::destroy_partition(smp);
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------

namespace {
// guarded() for the entry points of a table that may sit in an in-process
// group: a failure poisons the group, so the other ranks' collectives fail
// at once instead of waiting out the rendezvous timeout.
template <typename Body>
ts_status table_guarded(ts_table* t, Body&& body) {
  const ts_status st = tsd::guarded(std::forward<Body>(body));
  if (st != TS_OK && t && t->grp) tsd::group_poison(t->grp);
  return st;
}
}  // namespace

extern "C" {

ts_status ts_table_create(ts_table** out, const ts_table_config* cfg, const uint8_t* tier_dest) {
  return tsd::guarded([&] {
    if (!out || !cfg) tsd::fail(TS_ERR_CONFIG, "ts_table_create: null argument");
    *out = nullptr;
    auto t = std::make_unique<ts_table>();
    try {
      t->create(*cfg, tier_dest);
      t->ready = true;
    } catch (...) {
      if (cfg->group) tsd::group_poison(cfg->group);  // the other ranks' creation fails fast
      t->destroy();
      throw;
    }
    *out = t.release();
  });
}

ts_status ts_table_destroy(ts_table* t) {
  return tsd::guarded([&] {
    if (!t) return;
    t->destroy();
    delete t;
  });
}

ts_status ts_table_recv_capacity(ts_table* t, uint64_t* rows, uint64_t* regrows) {
  return tsd::guarded([&] {
    if (!t) tsd::fail(TS_ERR_CONFIG, "ts_table_recv_capacity: null table");
    if (rows) *rows = t->U > 1 ? t->recv_rows.cap / t->cfg.dim : 0;
    if (regrows) *regrows = t->recv_regrows;
  });
}

ts_status ts_table_shard_rows(ts_table* t, uint64_t* dp_rows, uint64_t* flex_rows, uint64_t* rw_rows) {
  return tsd::guarded([&] {
    if (!t) tsd::fail(TS_ERR_CONFIG, "ts_table_shard_rows: null table");
    if (dp_rows) *dp_rows = t->dp_rows;
    if (flex_rows) *flex_rows = t->flex_rows;
    if (rw_rows) *rw_rows = t->rw_rows;
  });
}

ts_status ts_table_stream(ts_table* t, void** stream) {
  return tsd::guarded([&] {
    if (!t || !stream) tsd::fail(TS_ERR_CONFIG, "ts_table_stream: null argument");
    *stream = static_cast<void*>(t->stream);
  });
}

ts_status ts_table_forward(ts_table* t, const uint32_t* d_rows, uint64_t occ, float* d_out) {
  return table_guarded(t, [&] {
    if (!t || (occ && (!d_rows || !d_out))) tsd::fail(TS_ERR_CONFIG, "ts_table_forward: null argument");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    t->forward(d_rows, occ, d_out);
  });
}

ts_status ts_table_backward(ts_table* t, const float* d_grad) {
  return table_guarded(t, [&] {
    if (!t || (t->last_occ && !d_grad)) tsd::fail(TS_ERR_CONFIG, "ts_table_backward: null argument");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    t->backward(d_grad);
  });
}

ts_status ts_table_train_step(ts_table* t, const uint32_t* d_rows, uint64_t occ, float* d_out) {
  return table_guarded(t, [&] {
    if (!t || (occ && (!d_rows || !d_out))) tsd::fail(TS_ERR_CONFIG, "ts_table_train_step: null argument");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    t->train_step(d_rows, occ, d_out);
  });
}

ts_status ts_table_train_step_host(ts_table* t, const uint32_t* h_rows, uint64_t occ, double* h_loss) {
  return table_guarded(t, [&] {
    if (!t || (occ && !h_rows)) tsd::fail(TS_ERR_CONFIG, "ts_table_train_step_host: null argument");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    if (occ > t->cfg.max_occurrences) {
      tsd::fail(TS_ERR_VALIDATION, "ts_table_train_step_host: occurrences exceed max_occurrences");
    }
    // sized once for the step cap: the output is peer-mapped by the other
    // ranks, so it must not move between steps
    t->rows_dev.ensure(t->cfg.max_occurrences);
    t->host_out.ensure(t->cfg.max_occurrences * t->cfg.dim);
    if (occ) {
      TSD_CUDA(cudaMemcpyAsync(t->rows_dev.ptr, h_rows, sizeof(uint32_t) * occ, cudaMemcpyHostToDevice,
                               t->stream));
    }
    t->train_step(t->rows_dev.ptr, occ, t->host_out.ptr);
    double loss = 0.0;
    TSD_CUDA(cudaMemcpyAsync(&loss, t->d_loss.ptr, sizeof(double), cudaMemcpyDeviceToHost, t->stream));
    TSD_CUDA(cudaStreamSynchronize(t->stream));
    if (h_loss) *h_loss = loss;
  });
}

ts_status ts_table_train_steps_host(ts_table* t, const uint32_t* const* h_rows, const uint64_t* occ,
                                   uint32_t steps, double* h_losses) {
  return table_guarded(t, [&] {
    using namespace tsd;
    if (!t || (steps && (!h_rows || !occ))) tsd::fail(TS_ERR_CONFIG, "ts_table_train_steps_host: null argument");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    for (uint32_t s = 0; s < steps; ++s) {
      if (occ[s] > t->cfg.max_occurrences) {
        tsd::fail(TS_ERR_VALIDATION, "ts_table_train_steps_host: occurrences exceed max_occurrences");
      }
      if (occ[s] && !h_rows[s]) tsd::fail(TS_ERR_CONFIG, "ts_table_train_steps_host: null batch");
    }
    if (steps == 0) return;
    // buffers that never move (peers map the output), created once
    t->rows_dev.ensure(t->cfg.max_occurrences);
    t->rows_dev2.ensure(t->cfg.max_occurrences);
    t->host_out.ensure(t->cfg.max_occurrences * t->cfg.dim);
    if (!t->copy) {
      TSD_CUDA(cudaStreamCreateWithFlags(&t->copy, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b) {
        TSD_CUDA(cudaEventCreateWithFlags(&t->ev_copied[b], cudaEventDisableTiming));
        TSD_CUDA(cudaEventCreateWithFlags(&t->ev_consumed[b], cudaEventDisableTiming));
        TSD_CUDA(cudaEventRecord(t->ev_consumed[b], t->stream));
      }
    }
    if (steps > t->h_loss_cap) {  // pinning synchronises the device: grow rarely
      if (t->h_loss_pinned) TSD_CUDA(cudaFreeHost(t->h_loss_pinned));
      t->h_loss_pinned = nullptr;
      t->h_loss_cap = 0;
      const uint32_t cap = std::max<uint32_t>(steps, 4096);
      TSD_CUDA(cudaHostAlloc(&t->h_loss_pinned, sizeof(double) * cap, cudaHostAllocMapped));
      TSD_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&t->h_loss_dev), t->h_loss_pinned, 0));
      t->h_loss_cap = cap;
    }
    uint32_t* buf[2] = {t->rows_dev.ptr, t->rows_dev2.ptr};
    if (t->lookahead && t->U == 1) {
      t->train_steps_lookahead(buf, h_rows, occ, steps);
      TSD_CUDA(cudaStreamSynchronize(t->stream));
      if (h_losses) std::memcpy(h_losses, t->h_loss_pinned, sizeof(double) * steps);
      return;
    }
    // step s's ids go to buffer s % 2 on the copy stream once step s-2 (the
    // buffer's last reader) has finished; the copy of step s+1 is queued
    // before step s's compute, so it overlaps it
    const auto stage = [&](uint32_t s) {
      const int b = static_cast<int>(s & 1u);
      TSD_CUDA(cudaStreamWaitEvent(t->copy, t->ev_consumed[b], 0));
      if (occ[s]) {
        TSD_CUDA(cudaMemcpyAsync(buf[b], h_rows[s], sizeof(uint32_t) * occ[s], cudaMemcpyHostToDevice, t->copy));
      }
      TSD_CUDA(cudaEventRecord(t->ev_copied[b], t->copy));
    };
    stage(0);
    for (uint32_t s = 0; s < steps; ++s) {
      if (s + 1 < steps) stage(s + 1);
      const int b = static_cast<int>(s & 1u);
      TSD_CUDA(cudaStreamWaitEvent(t->stream, t->ev_copied[b], 0));
      t->loss_mirror = t->h_loss_dev + s;  // the loss kernel writes the host slot itself
      t->train_step(buf[b], occ[s], t->host_out.ptr);
      t->loss_mirror = nullptr;
      TSD_CUDA(cudaEventRecord(t->ev_consumed[b], t->stream));
    }
    TSD_CUDA(cudaStreamSynchronize(t->stream));
    if (h_losses) std::memcpy(h_losses, t->h_loss_pinned, sizeof(double) * steps);
  });
}

ts_status ts_table_loss(ts_table* t, double* loss) {
  return tsd::guarded([&] {
    if (!t || !loss) tsd::fail(TS_ERR_CONFIG, "ts_table_loss: null argument");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    TSD_CUDA(cudaMemcpyAsync(loss, t->d_loss.ptr, sizeof(double), cudaMemcpyDeviceToHost, t->stream));
    TSD_CUDA(cudaStreamSynchronize(t->stream));
  });
}

ts_status ts_table_counters(ts_table* t, uint64_t* counters) {
  return tsd::guarded([&] {
    if (!t || !counters) tsd::fail(TS_ERR_CONFIG, "ts_table_counters: null argument");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    const uint32_t U = t->U, g = t->g;
    std::memset(counters, 0, sizeof(uint64_t) * TS_NUM_COUNTERS * U);
    unsigned long long tiers[3] = {0, 0, 0};
    uint32_t nseg = 0;
    if (U == 1 && t->last_occ) {
      // tiers are not bucketed at U == 1 (every occurrence is local): count
      // them from the placement cuts over the last batch, on the device
      const unsigned grid = static_cast<unsigned>(
          std::min<uint64_t>((t->last_occ + 255) / 256, 4u * tsd::sm_count()));
      TSD_CUDA(cudaMemsetAsync(t->tier_counts.ptr, 0, sizeof(unsigned long long) * 3, t->stream));
      tsd::count_tiers_kernel<<<grid, 256, 0, t->stream>>>(t->last_rows, t->last_occ, t->cfg.dp_cut,
                                                      t->cfg.flex_cut, t->tier_counts.ptr);
      TSD_LAUNCH_CHECK();
    }
    TSD_CUDA(cudaMemcpyAsync(tiers, t->tier_counts.ptr, sizeof(tiers), cudaMemcpyDeviceToHost, t->stream));
    TSD_CUDA(cudaMemcpyAsync(&nseg, t->nseg.ptr, sizeof(uint32_t), cudaMemcpyDeviceToHost, t->stream));
    TSD_CUDA(cudaStreamSynchronize(t->stream));
    // requester column g
    counters[TS_CTR_RECV_GLOBAL * U + g] = tiers[0];
    counters[TS_CTR_RECV_INTRA * U + g] = tiers[1];
    counters[TS_CTR_DP_LOCAL * U + g] = tiers[2];
    // server column g: every entry served here, by tier
    uint64_t rw_served = 0, flex_served = 0;
    if (U == 1) {
      rw_served = tiers[0];
      flex_served = tiers[1];
    } else {
      // local own-shard occurrences (RW owned by g / Flex in my slot) plus received ones
      const uint32_t nb = t->nb();
      auto start_of = [&](uint32_t p, uint32_t b) -> uint64_t {
        return t->h_counts[size_t{p} * (nb + 1) + b];
      };
      for (uint32_t p = 0; p < U; ++p) {
        if (p == g) continue;
        rw_served += start_of(p, g + 1) - start_of(p, g);
        if (p / t->W == t->node) flex_served += start_of(p, U + t->slot + 1) - start_of(p, U + t->slot);
      }
      // own RW/Flex occurrences served locally = my tiers minus what I sent
      uint64_t rw_sent = 0, flex_sent = 0;
      for (uint32_t b = 0; b < U; ++b) rw_sent += start_of(g, b + 1) - start_of(g, b);
      for (uint32_t b = U; b < U + t->W; ++b) flex_sent += start_of(g, b + 1) - start_of(g, b);
      rw_served += tiers[0] - rw_sent;
      flex_served += tiers[1] - flex_sent;
    }
    counters[TS_CTR_SEND_GLOBAL * U + g] = rw_served;
    counters[TS_CTR_SEND_INTRA * U + g] = flex_served;
    counters[TS_CTR_SERVED * U + g] = t->last_entries;
    counters[TS_CTR_DISTINCT * U + g] = nseg;
  });
}

ts_status ts_table_read_rows(ts_table* t, const uint32_t* rows, uint64_t count, float* h_weights,
                             float* h_state) {
  return tsd::guarded([&] {
    using namespace tsd;
    if (!t || (count && (!rows || !h_weights))) tsd::fail(TS_ERR_CONFIG, "ts_table_read_rows: null argument");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    const uint32_t dim = t->cfg.dim;
    // local ids resolved on the host (all rejected before any copy), then per
    // chunk: one upload, a row gather (+ state gather) into staging, one D2H
    std::vector<uint32_t> lids(count);
    for (uint64_t k = 0; k < count; ++k) {
      const uint32_t c = rows[k];
      if (c >= t->cfg.n_rows) tsd::fail(TS_ERR_VALIDATION, "read_rows: row outside the plan");
      uint32_t lid = c;
      if (t->U > 1 && c >= t->cfg.dp_cut) {
        const uint8_t d = t->h_dest[c];
        const bool mine = c < t->cfg.flex_cut ? d == t->slot : d == t->g;
        if (!mine) tsd::fail(TS_ERR_VALIDATION, "read_rows: row is not stored on this rank");
        lid = t->h_local[c];
      }
      lids[k] = lid;
    }
    if (count == 0) return;
    TSD_CUDA(cudaStreamSynchronize(t->stream));
    const uint64_t chunk = std::min<uint64_t>(count, std::max<uint64_t>(1, (uint64_t{64} << 20) / dim));
    DevBuf<uint32_t> d_ids;
    DevBuf<float> d_rows, d_st;
    d_ids.ensure(chunk);
    d_rows.ensure(chunk * dim);
    const bool with_state = h_state && t->d_state;
    if (with_state) d_st.ensure(chunk);
    for (uint64_t k0 = 0; k0 < count; k0 += chunk) {
      const uint64_t m = std::min(chunk, count - k0);
      TSD_CUDA(cudaMemcpyAsync(d_ids.ptr, lids.data() + k0, sizeof(uint32_t) * m, cudaMemcpyHostToDevice,
                               t->stream));
      launch_copy_rows(t->d_w, d_ids.ptr, d_rows.ptr, nullptr, m, dim, t->stream);
      TSD_CUDA(cudaMemcpyAsync(h_weights + k0 * dim, d_rows.ptr, sizeof(float) * m * dim, cudaMemcpyDeviceToHost,
                               t->stream));
      if (with_state) {
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((m + 255) / 256, 4u * sm_count()));
        tsd::gather_scalars_kernel<<<grid, 256, 0, t->stream>>>(t->d_state, d_ids.ptr, d_st.ptr, m);
        TSD_LAUNCH_CHECK();
        TSD_CUDA(cudaMemcpyAsync(h_state + k0, d_st.ptr, sizeof(float) * m, cudaMemcpyDeviceToHost, t->stream));
      }
      TSD_CUDA(cudaStreamSynchronize(t->stream));  // staging reused by the next chunk
    }
  });
}

ts_status ts_table_synchronize(ts_table* t) {
  return table_guarded(t, [&] {
    if (!t) tsd::fail(TS_ERR_CONFIG, "ts_table_synchronize: null table");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    if (t->p2p) {
      // collective: peers store into our replicated rows and receive
      // buffers, so "our step is done" means every rank's step is done --
      // a rendezvous behind all of this rank's streams, then wait for it
      for (cudaStream_t s : {t->stream, t->aux, t->rep, t->dd}) {
        if (!s) continue;
        TSD_CUDA(cudaEventRecord(t->ev_ar, s));
        TSD_CUDA(cudaStreamWaitEvent(t->comm, t->ev_ar, 0));
      }
      t->barrier_on_comm();
    }
    TSD_CUDA(cudaStreamSynchronize(t->stream));
    if (t->aux) TSD_CUDA(cudaStreamSynchronize(t->aux));
    if (t->comm) TSD_CUDA(cudaStreamSynchronize(t->comm));
    if (t->rep) TSD_CUDA(cudaStreamSynchronize(t->rep));
    if (t->pre) TSD_CUDA(cudaStreamSynchronize(t->pre));
    if (t->dd) TSD_CUDA(cudaStreamSynchronize(t->dd));
  });
}

ts_status ts_table_enable_timing(ts_table* t, int enable) {
  return tsd::guarded([&] {
    if (!t) tsd::fail(TS_ERR_CONFIG, "ts_table_enable_timing: null table");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    t->collect_timing();
    t->timing = enable != 0;
    std::fill(std::begin(t->phase_ms), std::end(t->phase_ms), 0.0);
    std::fill(std::begin(t->phase_launches), std::end(t->phase_launches), 0);
  });
}

ts_status ts_table_phase_times(ts_table* t, double* ms, uint64_t* launches, int capacity, int* count) {
  return tsd::guarded([&] {
    if (!t) tsd::fail(TS_ERR_CONFIG, "ts_table_phase_times: null table");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    t->collect_timing();
    const int n = std::min<int>(capacity, tsd::kNumPhases);
    for (int i = 0; i < n; ++i) {
      if (ms) ms[i] = t->phase_ms[i];
      if (launches) launches[i] = t->phase_launches[i];
    }
    if (count) *count = tsd::kNumPhases;
  });
}

ts_status ts_table_phase_trace(ts_table* t, int* phase, int* stream_id, double* t0_ms, double* t1_ms,
                               int capacity, int* count) {
  return tsd::guarded([&] {
    if (!t) tsd::fail(TS_ERR_CONFIG, "ts_table_phase_trace: null table");
    TSD_CUDA(cudaSetDevice(t->cfg.device));
    t->collect_timing();
    const int n = std::min<int>(capacity, static_cast<int>(t->trace.size()));
    for (int i = 0; i < n; ++i) {
      if (phase) phase[i] = t->trace[i].phase;
      if (stream_id) stream_id[i] = t->trace[i].stream_id;
      if (t0_ms) t0_ms[i] = t->trace[i].t0;
      if (t1_ms) t1_ms[i] = t->trace[i].t1;
    }
    if (count) *count = static_cast<int>(t->trace.size());
  });
}

const char* ts_table_phase_name(int phase) {
  return phase >= 0 && phase < tsd::kNumPhases ? tsd::kPhaseNames[phase] : "?";
}

}  // extern "C"
