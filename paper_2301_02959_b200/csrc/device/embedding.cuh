// Value-path kernels of the tiered sequence embedding: unpooled gather,
// deterministic segment reduction of gradients and the fused row-wise
// optimizer.  Contract (bit-for-bit on one GPU): oracle/restate.h.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tsd {

// Pieces of a long segment: ORC_PIECE in the oracle.
constexpr uint32_t kPiece = 256;
// Segments longer than this (<= kPiece) take the warp-per-piece path
// (default for a job of `gpus` GPUs, or TIERSHARD_SHORT_MAX).
uint32_t short_max(uint32_t gpus);

// How a requester finds the local shard row of a canonical row (or learns it
// is served remotely).  identity: U == 1, local id == canonical index.
struct RemapView {
  const uint8_t* dest = nullptr;    // [n] RW owner / Flex slot
  const uint32_t* local = nullptr;  // [n] local id at the serving rank
  uint64_t dp_cut = 0, flex_cut = 0;
  uint32_t rank = 0;   // g
  uint32_t slot = 0;   // g % W
  bool identity = true;
};

struct OptParams {
  int optimizer = 0;  // TS_OPT_*
  float lr = 0.01f;
  float eps = 1e-8f;
};

// Rows in [dense_lo, dense_hi) are not updated in place: their reduced
// gradient is written to dense_grad[row - dense_lo] (all-reduced later).
// With `stamp`, the row's stamp[row - dense_lo] is set to `epoch` as well:
// the replica update then reads only rows stamped this step, so the dense
// buffer never needs clearing and untouched rows cost no NVLink traffic.
constexpr int kMaxGradPeers = 8;

// Push mode (U > 1 over peer memory): the range is the replicated rows of a
// replica group of push_n members; relative row r belongs to member
// o = r / per, which receives every member's partial in its [push_n][per]
// buffer: the row's gradient is STORED (NVLink) to push_grad[o] at slot
// me * per + r % per, and its stamp to push_stamp[o] at the same slot.
struct DenseRange {
  uint32_t lo = 0, hi = 0;
  float* grad = nullptr;
  uint32_t* stamp = nullptr;
  uint32_t epoch = 0;
  uint32_t push_n = 0, per = 0, me = 0;
  // owner of tier row r: r % push_n, its slot r / push_n (interleaved: the
  // hot rows, first in canonical order, spread over every owner); else
  // blocks of `per` rows, r / per
  bool interleave = false;
  float* push_grad[kMaxGradPeers] = {};
  uint32_t* push_stamp[kMaxGradPeers] = {};
};

// Gradient source of sorted entry value v: v < n_local -> local grads
// [n_local x dim]; else r = v - n_local is a received entry, remote[r x dim]
// (received rows staged in local HBM by the exchange).
struct GradSource {
  const float* local = nullptr;
  const float* remote = nullptr;
  uint32_t n_local = 0;
};

// out[i] = W[local(rows[i])] for every occurrence served locally; remote
// occurrences are skipped (filled by the exchange).  Writes per-block
// partial sums of out^2 (double) into loss_partials[gridDim.x].
// bulk_stages > 0: the bulk-copy variant (gather_bulk_kernel: 4-warp blocks,
// bulk_stages x 4 KB shared-memory stages per warp), else the register one.
void launch_gather_local(const uint32_t* rows, uint64_t occ, const float* weights, float* out,
                         const RemapView& remap, uint32_t dim, double* loss_partials,
                         unsigned grid, cudaStream_t stream, int bulk_stages = 0);
unsigned gather_grid(uint64_t occ);

// Requester-pull forward (U > 1, peer memory): out[i] = the row of
// occurrence i read where it lives -- this rank's shard, or a peer's shard
// over NVLink (weights[s] = rank s's shard, mapped; node_base = g/W*W for
// the Flex server).  Needs no request lists and no count exchange.
struct PeerWeights {
  const float* w[kMaxGradPeers];
  uint32_t node_base = 0;
};
void launch_gather_all(const uint32_t* rows, uint64_t occ, const PeerWeights& pw, float* out,
                       const RemapView& remap, uint32_t dim, double* loss_partials, unsigned grid,
                       cudaStream_t stream);
// The remote half of the requester-pull forward: for the first *d_count
// occurrences of the route's destination order (sorted bucket b, server
// b < u ? b : node_base + b - u, local id ids[j], output row order[j]) load
// the row from its server's shard over NVLink into out; per-block loss
// partials into loss_partials[grid].
void launch_pull_rows(const uint32_t* sorted_bucket, const uint32_t* order, const uint32_t* ids,
                      const uint32_t* d_count, uint64_t max_count, const PeerWeights& pw, uint32_t u,
                      float* out, uint32_t dim, double* loss_partials, unsigned grid, cudaStream_t stream);
// Blocks per SM of the compute-stream persistent grids (8 = whole SM; the
// table sets 6 when U > 1 so comm-stream kernels keep two slots per SM).
void set_compute_blocks_per_sm(unsigned per_sm);

// Final fixed-order reduction of the loss partials: *loss = 0.5 * sum.
// mirror (nullable): a second destination, e.g. a host-mapped pinned slot,
// written by the same kernel (no copy-engine operation per step).
void launch_loss_finalize(const double* partials, unsigned count, double* loss,
                          cudaStream_t stream, double* mirror = nullptr);

// Segment reduction + optimizer over sorted (keys, vals) with segment starts.
// Short segments (<= kPiece entries) are reduced and applied by one warp;
// longer ones are split into kPiece pieces reduced in parallel and combined
// in piece order.  long_list / piece_off / partials are scratch sized by
// max_long (segments) and max_pieces (pieces) — see DESIGN.md.
struct SegmentScratch {
  uint32_t* long_list = nullptr;   // max_long
  uint32_t* long_count = nullptr;  // 1 (+ pad)
  uint32_t* piece_off = nullptr;   // max_long + 1
  float* partials = nullptr;       // max_pieces * dim
  uint32_t max_long = 0;
  uint32_t max_pieces = 0;
  uint32_t short_max = kPiece;     // longer segments take the piece path
  bool prefixed = false;           // piece_off already built (launch_long_segments)
};

// Segments [*d_lo, *d_hi) (device scalars, so ranges can be chosen on the
// device without a host sync).
void launch_segment_update(const uint32_t* keys, const uint32_t* vals, const uint32_t* starts,
                           const uint32_t* seg_keys, const uint32_t* d_lo, const uint32_t* d_hi,
                           uint64_t n_entries, uint32_t dim, const GradSource& grads, float* weights,
                           float* state, const OptParams& opt, const DenseRange& dense0,
                           const DenseRange& dense1, const SegmentScratch& scratch,
                           cudaStream_t stream);
// Second half of the segment update: segments longer than kPiece entries
// that launch_segment_update listed (piece sums, then one combine per row).
void launch_segment_long(const uint32_t* keys, const uint32_t* vals, const uint32_t* starts,
                         uint64_t n_entries, uint32_t dim, const GradSource& grads, float* weights,
                         float* state, const OptParams& opt, const DenseRange& dense0,
                         const DenseRange& dense1, const SegmentScratch& scratch,
                         cudaStream_t stream);

// Lists the segments of [*d_lo, *d_hi) longer than scratch.short_max and
// builds piece_off, ahead of the segment update: then launch_segment_update
// runs with scratch.long_list == nullptr (skip long segments, list nothing)
// and launch_segment_long with scratch.prefixed, on another stream.
void launch_long_segments(const uint32_t* starts, const uint32_t* d_lo, const uint32_t* d_hi,
                          uint64_t n_entries, const SegmentScratch& scratch, cudaStream_t stream);

// out[0] = 0, out[1] = number of segments whose key < split_key.
void launch_segment_split(const uint32_t* keys, const uint32_t* starts, const uint32_t* d_nseg,
                          uint32_t split_key, uint32_t* out, cudaStream_t stream);

// Dense optimizer over rows [row_lo, row_lo + rows) with gradients g[rows x dim].
void launch_dense_update(const float* grad, uint32_t rows, uint32_t row_lo, uint32_t dim,
                         float* weights, float* state, const OptParams& opt, cudaStream_t stream);

// Replicated-tier update over peer memory (replaces all-reduce + dense
// update): member `me` of a replica group owns the group's rows
// r = i * size + me (interleave) or [me * per, (me + 1) * per); i is the
// row's slot.  Every member has already pushed its partial
// gradient of those rows into the owner's local receive buffer
// recv[size][per][dim] (slot k = member k; DenseRange push mode), stamped
// with `epoch` where it touched the row.  The owner sums the stamped
// partials IN GROUP-RANK ORDER (an untouched member's partial is zero:
// skipping it changes nothing), applies the optimizer to its replica and
// stores the updated row (and Adagrad state) into every member's replica
// (peer stores).  Rows no member touched have a zero gradient, which leaves
// SGD and row-wise Adagrad rows unchanged, so they are skipped.  All loads
// are local; deterministic and identical on all replicas by construction.
struct ReplicaGroup {
  int size = 0;
  int me = 0;                          // my index in the group
  const float* recv = nullptr;         // [size][per][dim], local
  const uint32_t* recv_stamp = nullptr;  // [size][per], local
  uint32_t epoch = 0;
  uint32_t per = 0;                    // rows owned per member
  float* weights[kMaxGradPeers] = {};  // replicas: weights + row_lo * dim
  float* state[kMaxGradPeers] = {};    // Adagrad state + row_lo (may be null)
  uint32_t rows = 0;                   // replicated rows of the tier
  uint32_t row_lo = 0;                 // local id of replicated row 0
  bool interleave = false;             // ownership, as DenseRange::interleave
};

void launch_replica_update(const ReplicaGroup& grp, uint32_t dim, const OptParams& opt,
                           cudaStream_t stream);

// weights[l, d] = init_weight(seed, canon(l), d); canon = l when l2c == nullptr.
void launch_init_weights(float* weights, uint64_t local_rows, uint32_t dim, uint64_t seed,
                         const uint32_t* l2c, cudaStream_t stream);

}  // namespace tsd
