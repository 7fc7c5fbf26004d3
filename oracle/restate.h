/*
 * oracle/restate.h — plain-C restatement of the reference's per-iteration
 * routing/accounting loop and of the value-path contract (gather, dedup,
 * row-wise optimizer) that the reference leaves undefined.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so, and
 * only as the checker.  The product library never links or calls it.
 *
 * Parity status
 *   routing / counters / distinct / metrics: PINNED — checked bit-exactly
 *     against the compiled reference (oracle/_ref/ref_driver) in
 *     tests/test_oracle.py and against tests/golden/ fixtures.
 *   gather / segment sum / SGD / row-wise Adagrad: the reference has no
 *     implementation (SURVEY.md §8c "parity unpinned"); this file DEFINES the
 *     contract the CUDA path must meet bit-for-bit on one GPU.
 */
#ifndef TIERSHARD_ORACLE_RESTATE_H_
#define TIERSHARD_ORACLE_RESTATE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* hashing.hpp:14-22, 26-30, 37-39 */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_row_key_hash(uint32_t table_id, uint64_t row_id, uint64_t seed);
uint64_t orc_derive_seed(uint64_t seed, uint64_t index);

/* simulator.cpp:82-108 — placements for canonical rows [0, n). */
void orc_assign_rows(uint64_t n, const uint32_t* table_id, const uint64_t* row_id,
                     uint64_t dp_cut, uint64_t flex_cut, uint32_t num_gpus,
                     uint32_t gpus_per_node, uint64_t hash_seed,
                     uint8_t* tier, uint32_t* owner, uint32_t* slot);

/* Counter block layout, each a uint64_t[U] vector, in this order. */
enum {
  ORC_SEND_GLOBAL = 0,
  ORC_RECV_GLOBAL = 1,
  ORC_SEND_INTRA = 2,
  ORC_RECV_INTRA = 3,
  ORC_DP_LOCAL = 4,
  ORC_SERVED = 5,
  ORC_DISTINCT = 6,
  ORC_NUM_COUNTERS = 7
};

/* simulator.cpp:215-257 — one iteration's routing loop.  `counters` receives
 * 7*U uint64 values laid out [counter][gpu].  Returns 0, or -1 when a row
 * index is out of range. */
int orc_route_counts(uint32_t num_gpus, uint32_t gpus_per_node,
                     uint32_t local_batch, const uint64_t* sample_offsets,
                     const uint32_t* rows, uint64_t n_rows, const uint8_t* tier,
                     const uint32_t* owner, const uint32_t* slot,
                     uint64_t* counters);

/* simulator.cpp:259-331 — IterationMetrics from the counters, 26 doubles in
 * the declaration order of simulator.hpp:91-122.  Returns -1 on a
 * conservation violation (simulator.cpp:267-269). */
int orc_iteration_metrics(uint32_t num_gpus, uint32_t embedding_dim,
                          uint32_t scalar_bytes, uint32_t dyn_passes,
                          uint32_t stat_passes, int include_id_bytes,
                          double bytes_per_id, double a2a_global,
                          double a2a_intra, double ar_global, double ar_cross,
                          double ar_global_bytes, double ar_cross_max,
                          double ar_cross_mean, const uint64_t* counters,
                          double* metrics26);

/* ---------------------------------------------------------------------------
 * Value path contract (builder-defined).
 * ------------------------------------------------------------------------- */

/* Seeded initial weight of canonical row c, column d:
 *   u = mix64(seed ^ mix64(c * D + d));  v = (int32)(u >> 40) - 2^23;
 *   w = (float)v * 2^-23 * 0.01   (exact in fp32, |w| <= 0.01)            */
float orc_init_weight(uint64_t seed, uint64_t c, uint32_t d, uint32_t dim);
void orc_init_table(uint64_t seed, uint64_t n, uint32_t dim, float* w, int threads);
/* w[k,:] = initial weights of canonical row canon[k] (compact tables). */
void orc_init_rows(uint64_t seed, const uint32_t* canon, uint64_t count, uint32_t dim,
                   float* w, int threads);

/* Unpooled sequence gather: out[i,:] = w[rows[i],:]. */
void orc_gather(const float* w, uint32_t dim, const uint32_t* rows, uint64_t occ,
                float* out, int threads);

/* Synthetic loss 0.5*sum(out^2) in double (a reported scalar only). */
double orc_half_sq_sum(const float* x, uint64_t count);

enum { ORC_OPT_SGD = 0, ORC_OPT_ROWWISE_ADAGRAD = 1 };

/* Pieces of a segment are PIECE consecutive entries (segment-relative). */
#define ORC_PIECE 256u

/* Dedup + segment sum + fused row-wise update over all occurrences of one
 * batch, in canonical row space:
 *   - occurrences are grouped by row; inside a group entries keep ascending
 *     occurrence index (stable sort);
 *   - a group is cut into pieces of ORC_PIECE entries; each piece is summed
 *     left to right in fp32 starting from its first entry; the piece sums are
 *     then added left to right;
 *   - SGD:      w[d] = fmaf(-lr, g[d], w[d])
 *   - row-wise Adagrad: lane partials q_l = sum_{d in lane l} fmaf(g,g,q)
 *     (lane l owns d in [l*V, (l+1)*V), V = dim/32), butterfly
 *     q_l += q_{l^m} for m = 16,8,4,2,1;  G += q / dim;
 *     w[d] = fmaf(-lr, g[d] / (sqrtf(G) + eps), w[d]).
 * grads is [occ x dim]; w is [n x dim]; state is [n] (Adagrad only).
 * Returns the number of distinct rows updated. */
uint64_t orc_backward_update(float* w, float* state, uint64_t n, uint32_t dim,
                             const uint32_t* rows, uint64_t occ,
                             const float* grads, int optimizer, float lr,
                             float eps, int threads);

#ifdef __cplusplus
}
#endif
#endif /* TIERSHARD_ORACLE_RESTATE_H_ */
