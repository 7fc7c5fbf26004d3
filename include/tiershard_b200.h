/*
 * tiershard_b200.h — C-ABI of the B200 device path (libtiershard_b200.so).
 *
 * The reference (tiershard 0.1.0, /root/reference/proj) is a C++ library with
 * no device code and no C-ABI.  Its hot path is the per-iteration routing loop
 * inside simulate() (/root/reference/proj/src/simulator.cpp:215-257), which
 * only COUNTS traffic; the lookup/update entry points the north star asks for
 * (gather, exchange, dedup, optimizer) have no reference counterpart
 * (SURVEY.md §8a rows a16-a20).  This header is the thin layer the host C++
 * API (include/tiershard/ *.hpp) crosses to reach CUDA; INTEGRATION.md shows
 * how a reference user binds it (C++ relink, or the ctypes stub).
 *
 * Conventions
 *   - plain C types only; no CUDA, NCCL or torch types cross this boundary
 *     (streams are exposed as opaque void*);
 *   - every entry point returns a ts_status; on failure ts_last_error()
 *     returns the message for the calling thread.  The C++ shim rethrows
 *     TS_ERR_CONFIG / TS_ERR_VALIDATION / TS_ERR_INTERNAL as
 *     tiershard::ConfigError / ValidationError / Error with the same text,
 *     and every device/NCCL failure as tiershard::Error;
 *   - "rows" are canonical row indices (the u32 index space of
 *     RowDistribution's canonical order, distribution.hpp:26-30);
 *   - `tier_dest[i]` is the per-canonical-row placement byte emitted by the
 *     host planner: the RW owner GPU (h % U, simulator.cpp:103-104) for
 *     i >= flex_cut, the Flex slot (h % W, simulator.cpp:99-101) for
 *     dp_cut <= i < flex_cut, ignored for DP rows (i < dp_cut);
 *   - a handle is not reentrant: one host thread drives one handle.
 *   - there is no CPU fallback: without a CUDA device every call that needs
 *     one returns TS_ERR_NO_DEVICE.
 */
#ifndef TIERSHARD_B200_H_
#define TIERSHARD_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 2

typedef enum ts_status {
  TS_OK = 0,
  TS_ERR_CONFIG = 1,     /* -> tiershard::ConfigError     (error.hpp:18-21)  */
  TS_ERR_VALIDATION = 2, /* -> tiershard::ValidationError (error.hpp:25-28)  */
  TS_ERR_INTERNAL = 3,   /* -> tiershard::Error           (error.hpp:12-15)  */
  TS_ERR_CUDA = 4,       /* CUDA runtime / launch failure -> tiershard::Error */
  TS_ERR_NCCL = 5,       /* NCCL failure -> tiershard::Error                  */
  TS_ERR_NO_DEVICE = 6   /* no usable sm_100 device -> tiershard::Error       */
} ts_status;

/* Counter block layout returned by the routing entry points: 7 vectors of
 * U uint64 each, [counter][gpu], in this order.  The first six are the
 * reference's GpuCounters (simulator.cpp:112-119), the seventh its distinct
 * served-row count (simulator.cpp:250-255). */
enum {
  TS_CTR_SEND_GLOBAL = 0,
  TS_CTR_RECV_GLOBAL = 1,
  TS_CTR_SEND_INTRA = 2,
  TS_CTR_RECV_INTRA = 3,
  TS_CTR_DP_LOCAL = 4,
  TS_CTR_SERVED = 5,
  TS_CTR_DISTINCT = 6,
  TS_NUM_COUNTERS = 7
};

enum { TS_OPT_SGD = 0, TS_OPT_ROWWISE_ADAGRAD = 1 };

/* Thread-local message of the last failing call on this thread. */
const char* ts_last_error(void);
/* ABI version, build flags, CUDA/NCCL versions. */
const char* ts_build_info(void);
int ts_abi_version(void);
/* Number of CUDA devices visible (0 when no driver/device). */
ts_status ts_device_count(int* count);
/* A fresh 128-byte ncclUniqueId (rank 0 creates it and broadcasts it to the
 * other ranks through any host channel before ts_table_create). */
ts_status ts_nccl_unique_id(void* out128);
/* Number of device kernels this library has launched in this process (the
 * bench's gpu_launches evidence). */
uint64_t ts_kernel_launches(void);

/* ------------------------------------------------------------------------
 * Router: the reference's routing + traffic-accounting loop on one GPU for a
 * LOGICAL cluster of U = N*W GPUs (every requester's samples of one
 * iteration are routed in one launch).  Replaces the per-occurrence loop of
 * simulate() (simulator.cpp:215-257); the host shim derives
 * IterationMetrics from the counters with the reference formulas
 * (simulator.cpp:259-331).
 * ---------------------------------------------------------------------- */
typedef struct ts_router ts_router;

/* Uploads the remap table (tier from the cuts, tier_dest byte per row).
 * Requires 1 <= U <= 256 and n_rows < 2^32. */
ts_status ts_router_create(ts_router** out, int device, uint64_t n_rows,
                           uint64_t dp_cut, uint64_t flex_cut,
                           const uint8_t* tier_dest, uint32_t num_nodes,
                           uint32_t gpus_per_node);

/* One iteration: host CSR (sample_offsets has U*local_batch+1 entries,
 * GPU-major), copied to HBM, routed, 7*U counters copied back to host. */
ts_status ts_router_iteration(ts_router* r, uint32_t local_batch,
                              const uint64_t* sample_offsets,
                              const uint32_t* rows, uint64_t occurrences,
                              uint64_t* counters);

/* Same, with device-resident inputs (no copies); counters to host. */
ts_status ts_router_iteration_device(ts_router* r, const uint64_t* d_requester_begin,
                                     const uint32_t* d_rows, uint64_t occurrences,
                                     uint64_t* counters);

/* Device time of the last iteration (CUDA events on the router's stream):
 * the routing kernel alone, and the whole iteration including the counter /
 * distinct-bitmap clears (U x n_rows bits). */
ts_status ts_router_last_timing(ts_router* r, double* kernel_ms, double* total_ms);

ts_status ts_router_destroy(ts_router* r);

/* ------------------------------------------------------------------------
 * Key map: raw (table_id, row_id) keys -> canonical row index (the u32 the
 * router and the table consume), for inputs that arrive as raw ids: the
 * reference names rows by (table_id, row_id) in RowRecord
 * (distribution.hpp:31-38), in the plan document's dp_rows / flex_rows and
 * in the assignment CSV (json_io.cpp:235-244, 380-394).
 * ---------------------------------------------------------------------- */
typedef struct ts_keymap ts_keymap;

/* Uploads the canonical order: row i of the plan is (table_ids[i],
 * row_ids[i]).  ValidationError on duplicate keys; ConfigError when table
 * ids reach 2^24, row ids reach 2^40 or are too sparse for the dense map. */
ts_status ts_keymap_create(ts_keymap** out, int device, uint64_t n_rows,
                           const uint32_t* table_ids, const uint64_t* row_ids);

/* d_canon[i] = canonical index of (d_table_ids[i], d_row_ids[i]), or
 * 0xFFFFFFFF for keys absent from the plan (all device pointers; stream NULL
 * = the map's own stream).  With misses != NULL the call synchronises and
 * stores the number of absent keys. */
ts_status ts_keymap_lookup(ts_keymap* m, const uint32_t* d_table_ids,
                           const uint64_t* d_row_ids, uint64_t n, uint32_t* d_canon,
                           void* stream, uint64_t* misses);

ts_status ts_keymap_destroy(ts_keymap* m);

/* ------------------------------------------------------------------------
 * GPU workload sampler, for throughput runs.  Every
 * sample follows the reference's per-sample procedure (Workload::
 * materialize_iteration, simulator.cpp:54-71: a Poisson(L) length, then L
 * alias draws; rng.cpp:15-115) on its own SplitMix64 stream seeded from
 * (seed, iteration, sample), over the reference's alias table (built on the
 * host, uploaded).  Same distribution as the host Workload, not the same
 * stream: the host path stays the bit-exact one.
 * ---------------------------------------------------------------------- */
typedef struct ts_sampler ts_sampler;

/* alias_prob / alias_index: the AliasTable of the canonical probabilities
 * (tiershard::AliasTable::probabilities() / aliases()). */
ts_status ts_sampler_create(ts_sampler** out, int device, uint64_t n_rows,
                            const double* alias_prob, const uint32_t* alias_index,
                            double expected_length, uint64_t seed);

/* Samples [sample_begin, sample_begin + samples) of `iteration` (GPU g of a
 * U-GPU job passes sample_begin = g * local_batch): canonical rows into
 * d_rows (device), CSR offsets into d_offsets (device, samples + 1 entries,
 * may be NULL), the occurrence count into *occurrences (host; the call
 * synchronises once).  ValidationError when the rows exceed rows_capacity. */
ts_status ts_sampler_iteration(ts_sampler* s, uint32_t iteration, uint64_t sample_begin,
                               uint32_t samples, uint32_t* d_rows, uint64_t rows_capacity,
                               uint64_t* d_offsets, uint64_t* occurrences, void* stream);

ts_status ts_sampler_destroy(ts_sampler* s);

/* ------------------------------------------------------------------------
 * Planner preview: frontier landmarks and 2- / 3-tier
 * cuts for many what-if cost models over one canonical distribution, from
 * one GPU prefix scan (planner.cpp build_frontier / find_points /
 * plan_2tier / plan_3tier restated on mem(k) = k*mem_a + mem_b*P(k)).  The
 * host planner stays authoritative: the scan's summation order can move a
 * cut by a row where the frontier crosses zero within rounding.
 * ---------------------------------------------------------------------- */
typedef struct ts_frontier_query {
  double mem_a;        /* DP memory marginal of a row: mem_a + mem_b * p (bytes) */
  double mem_b;
  double p_comm_dp;    /* DP communication breakpoint (landmark c) */
  double flex_price;   /* Flex memory price per row (3-tier) */
  double p_comm_flex;  /* Flex communication breakpoint; < 0: no Flex tier (2-tier only) */
} ts_frontier_query;

typedef struct ts_frontier_answer {
  uint64_t a, b, c;          /* find_points landmarks (d = n) */
  uint64_t dp_cut_3tier;     /* 3-tier cuts (== b, b without a Flex tier) */
  uint64_t flex_cut_3tier;
  double reduction_2tier;    /* predicted global-a2a reduction = covered expected length share */
  double reduction_3tier;
} ts_frontier_answer;

/* probabilities: n canonical (non-increasing) probabilities, host memory. */
ts_status ts_frontier_preview(int device, uint64_t n, const double* probabilities, uint32_t nq,
                              const ts_frontier_query* queries, ts_frontier_answer* answers);

/* ------------------------------------------------------------------------
 * Host-only planning helpers of the U > 1 path (no device needed).
 * ---------------------------------------------------------------------- */

/* Shard layout of rank g: local_id[i] for every canonical row i (the row's
 * position inside the shard of the rank that serves it: DP rows keep i, Flex
 * rows follow as [dp_cut + rank among rows of the same slot], RW rows as
 * [dp_cut + flex rows of the owner's slot + rank among rows of the same
 * owner]).  *dp_rows / *flex_rows / *rw_rows describe rank g's shard.
 * local_id may be NULL. */
ts_status ts_shard_layout(uint64_t n_rows, uint64_t dp_cut, uint64_t flex_cut,
                          const uint8_t* tier_dest, uint32_t num_nodes,
                          uint32_t gpus_per_node, uint32_t rank, uint32_t* local_id,
                          uint64_t* dp_rows, uint64_t* flex_rows, uint64_t* rw_rows);

/* All-to-allv plan of rank g from every rank's bucket starts (the counts the
 * table all-gathers each step): all_starts is [U][U+W+2] u32 where rank p's
 * bucket b (RW to server b for b < U, Flex to slot b-U for U <= b < U+W,
 * local b = U+W) spans [all_starts[p][b], all_starts[p][b+1]).  Outputs
 * 2*U entries each ([2p] RW part, [2p+1] Flex part), in elements: send
 * offsets/counts into this rank's bucket-ordered buffer, receive
 * offsets/counts into a buffer ordered by source rank; *recv_before = the
 * number of received entries from ranks < g, *recv_total the sum. */
ts_status ts_exchange_plan(uint32_t num_nodes, uint32_t gpus_per_node, uint32_t rank,
                           const uint32_t* all_starts, uint64_t* send_off,
                           uint64_t* send_cnt, uint64_t* recv_off, uint64_t* recv_cnt,
                           uint64_t* recv_before, uint64_t* recv_total);

/* ------------------------------------------------------------------------
 * Sharded sequence-embedding table: lookup (forward) and update (backward)
 * for one rank of a U = N*W GPU job.  Rank g stores, in one contiguous fp32
 * [local_rows x dim] shard: the dp_cut DP rows, the Flex rows of slot g % W,
 * and the RW rows it owns.  With U > 1 the ranks
 * exchange ids/rows with NCCL (world communicator for RW, intra-node
 * communicator g / W for Flex) and all-reduce DP (world) and Flex (cross
 * communicator g % W) gradients.
 * ---------------------------------------------------------------------- */
typedef struct ts_table ts_table;

/* In-process rank group: all U ranks of a job are host threads of ONE process
 * (any mix of GPUs, including several ranks on one GPU, which NCCL cannot
 * do).  Passed as ts_table_config.group instead of an NCCL id, it carries the
 * table's collectives (host all-gather, device rendezvous by cross-stream
 * events) and maps peer buffers by plain device pointers; the exchange is
 * the peer-memory path.  Each rank's table must be created, stepped and
 * destroyed by its own thread, collectively (a rendezvous that does not
 * complete within TIERSHARD_GROUP_TIMEOUT seconds, default 300, fails the
 * call and poisons the group).  Destroy the group after its tables. */
typedef struct ts_group ts_group;
ts_status ts_group_create(ts_group** out, uint32_t ranks);
/* Marks the group failed (a rank's host thread failed outside the library):
 * every pending and later collective of its tables returns an error at once. */
ts_status ts_group_abort(ts_group* g);
ts_status ts_group_destroy(ts_group* g);

typedef struct ts_table_config {
  uint32_t num_nodes;      /* N */
  uint32_t gpus_per_node;  /* W */
  uint32_t rank;           /* g in [0, N*W) */
  int32_t device;          /* CUDA ordinal */
  uint32_t dim;            /* D: multiple of 32, <= 1024 */
  uint64_t n_rows;         /* canonical rows (< 2^32) */
  uint64_t dp_cut;
  uint64_t flex_cut;
  uint64_t weight_seed;    /* orc_init_weight contract, oracle/restate.h */
  int32_t optimizer;       /* TS_OPT_* */
  float lr;
  float eps;               /* Adagrad epsilon */
  uint64_t max_occurrences;      /* capacity: occurrences per step, this rank */
  const void* nccl_unique_id;    /* 128-byte ncclUniqueId (one process per rank) */
  struct ts_group* group;        /* in-process rank group (ts_group_create), or NULL;
                                    U > 1 needs exactly one of nccl_unique_id / group */
  uint64_t recv_rows_hint;       /* U > 1: initial capacity (rows) of the buffer peers
                                    push this rank's remote gradients into -- e.g. the
                                    plan's expected remote occurrences plus a margin;
                                    0 = the worst case, (U-1) x max_occurrences.  A step
                                    that needs more grows it (collectively, with 25 %
                                    headroom) instead of failing. */
} ts_table_config;

/* Device bytes one rank allocates, itemised (ts_table_plan_footprint). */
typedef struct ts_table_footprint {
  uint64_t weights;          /* [local_rows x dim] fp32 shard */
  uint64_t optimizer_state;  /* row-wise Adagrad state */
  uint64_t remap;            /* U > 1: placement byte + local id per canonical row */
  uint64_t step_buffers;     /* dedup sort, segments, piece partials */
  uint64_t exchange;         /* U > 1: request lists, gradient receive buffer */
  uint64_t replicated;       /* U > 1: replicated-row receive slots + stamps */
  uint64_t host_api;         /* ts_table_train_step(s)_host staging + output */
  uint64_t total;
} ts_table_footprint;

/* Host-only: what ts_table_create (and, with host_api, the host-buffer
 * entry points) will allocate on a rank whose shard holds dp_rows /
 * flex_rows / rw_rows rows (ts_shard_layout's counts).  ts_table_create
 * checks the same sum against the device's free memory and fails with
 * TS_ERR_CONFIG before allocating when it does not fit. */
ts_status ts_table_plan_footprint(const ts_table_config* cfg, uint64_t dp_rows, uint64_t flex_rows,
                                  uint64_t rw_rows, int host_api, ts_table_footprint* out);

/* Collective over all U ranks when U > 1 (NCCL communicator creation). */
ts_status ts_table_create(ts_table** out, const ts_table_config* cfg,
                          const uint8_t* tier_dest);
ts_status ts_table_destroy(ts_table* t);

/* U > 1: current gradient receive-buffer capacity (rows) and how many times
 * a step has grown it (the bounded-buffer overflow path). */
ts_status ts_table_recv_capacity(ts_table* t, uint64_t* rows, uint64_t* regrows);

/* Rows of this rank's shard by tier. */
ts_status ts_table_shard_rows(ts_table* t, uint64_t* dp_rows,
                              uint64_t* flex_rows, uint64_t* rw_rows);

/* The table's CUDA stream (cudaStream_t as void*). */
ts_status ts_table_stream(ts_table* t, void** stream);

/* Forward: d_rows are this rank's occurrences (device memory, canonical
 * indices); writes the unpooled [occ x dim] fp32 embeddings to d_out. */
ts_status ts_table_forward(ts_table* t, const uint32_t* d_rows, uint64_t occ,
                           float* d_out);

/* Backward + update for the last forward: d_grad is [occ x dim] (may alias
 * that forward's d_out).  Dedup, segment-reduce, all-reduce of replicated
 * tiers, fused optimizer. */
ts_status ts_table_backward(ts_table* t, const float* d_grad);

/* One synthetic training step: forward, loss = 0.5*sum(out^2) (device),
 * backward with grad = out.  Device inputs; no host synchronisation. */
ts_status ts_table_train_step(ts_table* t, const uint32_t* d_rows,
                              uint64_t occ, float* d_out);

/* End-to-end step through host memory: copies h_rows (pinned or pageable)
 * to HBM, runs ts_table_train_step, and reads the loss back to *h_loss. */
ts_status ts_table_train_step_host(ts_table* t, const uint32_t* h_rows,
                                   uint64_t occ, double* h_loss);

/* Loss of the last train step (synchronises the table stream). */
/* `steps` host-buffer steps in one call (h_rows[s] / occ[s] = step s's batch
 * in pinned host memory; h_losses[s] receives its loss, may be NULL).  Same
 * math as calling ts_table_train_step_host once per step, pipelined: step
 * s+1's host-to-device copy runs on a copy stream while step s computes. */
ts_status ts_table_train_steps_host(ts_table* t, const uint32_t* const* h_rows, const uint64_t* occ,
                                   uint32_t steps, double* h_losses);

ts_status ts_table_loss(ts_table* t, double* loss);

/* This rank's counter contribution for the last forward/backward: for the
 * requester side its own column, for the server side the occurrences and
 * distinct rows it served (filled in by backward). 7*U host uint64. */
ts_status ts_table_counters(ts_table* t, uint64_t* counters);

/* Copies rows (canonical indices stored on this rank) and, for Adagrad,
 * their state back to host.  ValidationError for rows not on this rank. */
ts_status ts_table_read_rows(ts_table* t, const uint32_t* rows, uint64_t count,
                             float* h_weights, float* h_state);

/* Waits for this rank's queued work.  With U > 1 on the peer-memory path it
 * is COLLECTIVE (every rank calls it): peers store into this rank's
 * replicated rows and receive buffers, so it first rendezvous with them and
 * returns once every rank's queued steps are complete -- after it,
 * ts_table_read_rows sees the final replicated rows. */
ts_status ts_table_synchronize(ts_table* t);

/* Per-phase device time accumulated since the last reset (CUDA events on the
 * table stream), in ms: see ts_table_phase_name for the index meaning. */
ts_status ts_table_enable_timing(ts_table* t, int enable);
ts_status ts_table_phase_times(ts_table* t, double* ms, uint64_t* launches,
                               int capacity, int* count);
const char* ts_table_phase_name(int phase);
/* Timeline of the phases recorded since the last collection (timing must be
 * enabled): phase index, stream (0 compute, 1 exchange), start / end in ms
 * from the first recorded event.  Synchronises the table's streams. */
ts_status ts_table_phase_trace(ts_table* t, int* phase, int* stream_id, double* t0_ms,
                               double* t1_ms, int capacity, int* count);

/* ts_table_forward with raw (table_id, row_id) keys (ts_keymap above): the
 * lookup runs on the table's stream into a scratch the map keeps per table
 * (valid until that table's next call, so the following ts_table_backward
 * sees the same ids; several tables may share one map), then the forward.
 * Synchronises once to reject absent keys (ValidationError) before any row
 * is read. */
ts_status ts_table_forward_keys(ts_table* t, ts_keymap* m, const uint32_t* d_table_ids,
                                const uint64_t* d_row_ids, uint64_t occurrences, float* d_out);

#ifdef __cplusplus
}
#endif
#endif /* TIERSHARD_B200_H_ */
