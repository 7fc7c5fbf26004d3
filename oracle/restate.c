/*
 * oracle/restate.c — CPU restatement (test infrastructure only; see
 * restate.h for the contract and who may load this).
 *
 * Reference anchors (paths under /root/reference/proj):
 *   orc_mix64 / orc_row_key_hash / orc_derive_seed  include/tiershard/hashing.hpp:14-39
 *   orc_assign_rows                                 src/simulator.cpp:82-108
 *   orc_route_counts                                src/simulator.cpp:215-257
 *                                                   (+ stamps, :158-166, :250-255)
 *   orc_iteration_metrics                           src/simulator.cpp:259-331
 * The value-path functions have no reference counterpart.
 */
#include "restate.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* hashing                                                                  */
/* ------------------------------------------------------------------------ */

uint64_t orc_mix64(uint64_t x) {
  /* golden-ratio increment + Stafford mix13, hashing.hpp:14-22 */
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t orc_row_key_hash(uint32_t table_id, uint64_t row_id, uint64_t seed) {
  /* hashing.hpp:26-30 */
  return orc_mix64(orc_mix64(seed ^ ((uint64_t)table_id * 0x9E3779B97F4A7C15ull)) ^ row_id);
}

uint64_t orc_derive_seed(uint64_t seed, uint64_t index) {
  /* hashing.hpp:37-39 */
  return orc_mix64(seed ^ orc_mix64(index + 1));
}

/* ------------------------------------------------------------------------ */
/* placement                                                                */
/* ------------------------------------------------------------------------ */

void orc_assign_rows(uint64_t n, const uint32_t* table_id, const uint64_t* row_id,
                     uint64_t dp_cut, uint64_t flex_cut, uint32_t num_gpus,
                     uint32_t gpus_per_node, uint64_t hash_seed, uint8_t* tier,
                     uint32_t* owner, uint32_t* slot) {
  /* simulator.cpp:93-107: tier by canonical index against the two cuts;
   * RW owner = h % U, Flex slot = h % W (the other field stays 0). */
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t h = orc_row_key_hash(table_id[i], row_id[i], hash_seed);
    owner[i] = 0;
    slot[i] = 0;
    if (i < dp_cut) {
      tier[i] = 0;
    } else if (i < flex_cut) {
      tier[i] = 1;
      slot[i] = (uint32_t)(h % gpus_per_node);
    } else {
      tier[i] = 2;
      owner[i] = (uint32_t)(h % num_gpus);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* routing loop                                                             */
/* ------------------------------------------------------------------------ */

int orc_route_counts(uint32_t u, uint32_t w, uint32_t local_batch,
                     const uint64_t* off, const uint32_t* rows, uint64_t n,
                     const uint8_t* tier, const uint32_t* owner,
                     const uint32_t* slot, uint64_t* c) {
  memset(c, 0, sizeof(uint64_t) * ORC_NUM_COUNTERS * u);
  uint64_t* sg = c + (size_t)ORC_SEND_GLOBAL * u;
  uint64_t* rg = c + (size_t)ORC_RECV_GLOBAL * u;
  uint64_t* si = c + (size_t)ORC_SEND_INTRA * u;
  uint64_t* ri = c + (size_t)ORC_RECV_INTRA * u;
  uint64_t* dl = c + (size_t)ORC_DP_LOCAL * u;
  uint64_t* sv = c + (size_t)ORC_SERVED * u;
  uint64_t* ds = c + (size_t)ORC_DISTINCT * u;
  /* A (server,row) "seen" bitmap stands in for the reference's iteration
   * stamps (simulator.cpp:158-166): both count first touches. */
  const uint64_t words = (n + 63) / 64;
  uint64_t* seen = (uint64_t*)calloc((size_t)u * words, sizeof(uint64_t));
  if (!seen) return -2;
  int rc = 0;
  for (uint32_t g = 0; g < u && rc == 0; ++g) {
    const uint64_t begin = off[(uint64_t)g * local_batch];
    const uint64_t end = off[(uint64_t)(g + 1) * local_batch];
    const uint32_t node_base = (g / w) * w;
    for (uint64_t k = begin; k < end; ++k) {
      const uint32_t r = rows[k];
      if (r >= n) { rc = -1; break; }
      uint32_t server;
      if (tier[r] == 2) {          /* Tier::kRowWise */
        server = owner[r];
        sg[server]++;
        rg[g]++;
      } else if (tier[r] == 1) {   /* Tier::kFlex */
        server = node_base + slot[r];
        si[server]++;
        ri[g]++;
      } else {                     /* Tier::kDataParallel */
        server = g;
        dl[g]++;
      }
      sv[server]++;
      uint64_t* word = &seen[(size_t)server * words + (r >> 6)];
      const uint64_t bit = 1ull << (r & 63);
      if (!(*word & bit)) {
        *word |= bit;
        ds[server]++;
      }
    }
  }
  free(seen);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* metric derivation                                                        */
/* ------------------------------------------------------------------------ */

static void mmm(const uint64_t* v, uint32_t u, double* mn, double* mx, double* mean) {
  uint64_t lo = v[0], hi = v[0], tot = 0;
  for (uint32_t i = 0; i < u; ++i) {
    if (v[i] < lo) lo = v[i];
    if (v[i] > hi) hi = v[i];
    tot += v[i];
  }
  *mn = (double)lo;
  *mx = (double)hi;
  *mean = (double)tot / (double)u;
}

int orc_iteration_metrics(uint32_t u, uint32_t dim, uint32_t scalar_bytes,
                          uint32_t dyn_p, uint32_t stat_p, int include_id,
                          double bytes_per_id, double a2a_global, double a2a_intra,
                          double ar_global, double ar_cross, double ar_global_bytes,
                          double ar_cross_max, double ar_cross_mean,
                          const uint64_t* c, double* m) {
  const uint64_t* sg = c + (size_t)ORC_SEND_GLOBAL * u;
  const uint64_t* rg = c + (size_t)ORC_RECV_GLOBAL * u;
  const uint64_t* si = c + (size_t)ORC_SEND_INTRA * u;
  const uint64_t* ri = c + (size_t)ORC_RECV_INTRA * u;
  const uint64_t* dl = c + (size_t)ORC_DP_LOCAL * u;
  const double row_bytes = (double)dim * scalar_bytes;
  const double dyn = dyn_p, stat = stat_p;
  const double id_bytes = include_id ? bytes_per_id : 0.0;
  uint64_t tsg = 0, trg = 0, tsi = 0, tri = 0;
  uint64_t msg = 0, mrg = 0, msi = 0, mri = 0, peak = 0;
  for (uint32_t g = 0; g < u; ++g) {
    tsg += sg[g]; trg += rg[g]; tsi += si[g]; tri += ri[g];
    if (sg[g] > msg) msg = sg[g];
    if (rg[g] > mrg) mrg = rg[g];
    if (si[g] > msi) msi = si[g];
    if (ri[g] > mri) mri = ri[g];
    const uint64_t units = sg[g] + rg[g] + si[g] + ri[g] + dl[g];
    if (units > peak) peak = units;
  }
  if (tsg != trg || tsi != tri) return -1;
  /* field order = simulator.hpp:91-122 */
  m[0] = (double)msg * row_bytes;              /* global_a2a_send_max */
  m[1] = (double)mrg * row_bytes;              /* global_a2a_recv_max */
  m[3] = (double)tsg * row_bytes;              /* global_a2a_total */
  m[2] = m[3] / u;                             /* global_a2a_bytes_mean */
  m[4] = (double)msi * row_bytes;              /* intra_a2a_send_max */
  m[5] = (double)mri * row_bytes;              /* intra_a2a_recv_max */
  m[7] = (double)tsi * row_bytes;              /* intra_a2a_total */
  m[6] = m[7] / u;                             /* intra_a2a_bytes_mean */
  m[8] = ar_global_bytes;
  m[9] = ar_cross_max;
  m[10] = ar_cross_mean;
  const uint64_t gmax = msg > mrg ? msg : mrg;
  const uint64_t imax = msi > mri ? msi : mri;
  m[11] = dyn * ((double)gmax * row_bytes) / a2a_global;
  m[12] = dyn * ((double)imax * row_bytes) / a2a_intra;
  if (id_bytes > 0.0) {
    m[11] += (double)gmax * id_bytes / a2a_global;
    m[12] += (double)imax * id_bytes / a2a_intra;
  }
  m[13] = stat * ar_global_bytes / ar_global;
  m[14] = stat * ar_cross_max / ar_cross;
  m[15] = m[11] + m[12] + m[13] + m[14];
  m[16] = m[11] + m[13];
  m[17] = (double)peak * row_bytes;
  double mn, mx, mean;
  mmm(c + (size_t)ORC_SERVED * u, u, &mn, &mx, &mean);
  m[18] = mn * dim;
  m[19] = mx * dim;
  m[20] = mean * dim;
  m[21] = mean > 0.0 ? mx / mean : 1.0;
  mmm(c + (size_t)ORC_DISTINCT * u, u, &mn, &mx, &mean);
  m[22] = mn;
  m[23] = mx;
  m[24] = mean;
  m[25] = mean > 0.0 ? mx / mean : 1.0;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* value path                                                               */
/* ------------------------------------------------------------------------ */

float orc_init_weight(uint64_t seed, uint64_t c, uint32_t d, uint32_t dim) {
  const uint64_t u = orc_mix64(seed ^ orc_mix64(c * (uint64_t)dim + d));
  const int32_t v = (int32_t)(u >> 40) - (1 << 23);
  return (float)v * (0.01f / 8388608.0f);
}

typedef struct {
  int tid, nthreads;
  void* a;
} job_t;

typedef void (*job_fn)(int tid, int nthreads, void* arg);

typedef struct {
  job_fn fn;
  int tid, nthreads;
  void* arg;
} thr_t;

static void* thr_main(void* p) {
  thr_t* t = (thr_t*)p;
  t->fn(t->tid, t->nthreads, t->arg);
  return NULL;
}

static void run_par(job_fn fn, void* arg, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  thr_t ctx[256];
  for (int i = 0; i < threads; ++i) {
    ctx[i].fn = fn;
    ctx[i].tid = i;
    ctx[i].nthreads = threads;
    ctx[i].arg = arg;
    if (i > 0) pthread_create(&th[i], NULL, thr_main, &ctx[i]);
  }
  fn(0, threads, arg);
  for (int i = 1; i < threads; ++i) pthread_join(th[i], NULL);
}

typedef struct {
  uint64_t seed, n;
  uint32_t dim;
  float* w;
} init_args;

static void init_job(int tid, int nt, void* p) {
  init_args* a = (init_args*)p;
  const uint64_t lo = a->n * tid / nt, hi = a->n * (tid + 1) / nt;
  for (uint64_t c = lo; c < hi; ++c)
    for (uint32_t d = 0; d < a->dim; ++d)
      a->w[c * a->dim + d] = orc_init_weight(a->seed, c, d, a->dim);
}

void orc_init_table(uint64_t seed, uint64_t n, uint32_t dim, float* w, int threads) {
  init_args a = {seed, n, dim, w};
  run_par(init_job, &a, threads);
}

typedef struct {
  uint64_t seed, count;
  uint32_t dim;
  const uint32_t* canon;
  float* w;
} init_rows_args;

static void init_rows_job(int tid, int nt, void* p) {
  init_rows_args* a = (init_rows_args*)p;
  const uint64_t lo = a->count * tid / nt, hi = a->count * (tid + 1) / nt;
  for (uint64_t k = lo; k < hi; ++k)
    for (uint32_t d = 0; d < a->dim; ++d)
      a->w[k * a->dim + d] = orc_init_weight(a->seed, a->canon[k], d, a->dim);
}

void orc_init_rows(uint64_t seed, const uint32_t* canon, uint64_t count, uint32_t dim,
                   float* w, int threads) {
  init_rows_args a = {seed, count, dim, canon, w};
  run_par(init_rows_job, &a, threads);
}

typedef struct {
  const float* w;
  uint32_t dim;
  const uint32_t* rows;
  uint64_t occ;
  float* out;
} gather_args;

static void gather_job(int tid, int nt, void* p) {
  gather_args* a = (gather_args*)p;
  const uint64_t lo = a->occ * tid / nt, hi = a->occ * (tid + 1) / nt;
  for (uint64_t i = lo; i < hi; ++i)
    memcpy(a->out + i * a->dim, a->w + (uint64_t)a->rows[i] * a->dim,
           sizeof(float) * a->dim);
}

void orc_gather(const float* w, uint32_t dim, const uint32_t* rows, uint64_t occ,
                float* out, int threads) {
  gather_args a = {w, dim, rows, occ, out};
  run_par(gather_job, &a, threads);
}

double orc_half_sq_sum(const float* x, uint64_t count) {
  double s = 0.0;
  for (uint64_t i = 0; i < count; ++i) s += (double)x[i] * (double)x[i];
  return 0.5 * s;
}

/* LSD radix sort of (row << 32 | occurrence) keys: a stable group-by-row. */
static void radix_sort_u64(uint64_t* a, uint64_t* tmp, uint64_t n, int key_bits) {
  for (int shift = 0; shift < key_bits; shift += 8) {
    uint64_t cnt[257];
    memset(cnt, 0, sizeof(cnt));
    for (uint64_t i = 0; i < n; ++i) cnt[((a[i] >> shift) & 255) + 1]++;
    for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
    for (uint64_t i = 0; i < n; ++i) tmp[cnt[(a[i] >> shift) & 255]++] = a[i];
    memcpy(a, tmp, n * sizeof(uint64_t));
  }
}

typedef struct {
  float* w;
  float* state;
  uint32_t dim;
  const uint64_t* sorted;
  const uint64_t* seg_begin; /* nseg + 1 entries */
  uint64_t nseg;
  const float* grads;
  int opt;
  float lr, eps;
} bwd_args;

static void bwd_job(int tid, int nt, void* p) {
  bwd_args* a = (bwd_args*)p;
  const uint32_t dim = a->dim;
  float* g = (float*)malloc(sizeof(float) * dim);
  float* piece = (float*)malloc(sizeof(float) * dim);
  const uint64_t lo = a->nseg * tid / nt, hi = a->nseg * (tid + 1) / nt;
  for (uint64_t s = lo; s < hi; ++s) {
    const uint64_t b = a->seg_begin[s], e = a->seg_begin[s + 1];
    const uint32_t row = (uint32_t)(a->sorted[b] >> 32);
    for (uint64_t pb = b; pb < e; pb += ORC_PIECE) {
      const uint64_t pe = (pb + ORC_PIECE < e) ? pb + ORC_PIECE : e;
      const float* first = a->grads + (a->sorted[pb] & 0xffffffffull) * dim;
      for (uint32_t d = 0; d < dim; ++d) piece[d] = first[d];
      for (uint64_t k = pb + 1; k < pe; ++k) {
        const float* src = a->grads + (a->sorted[k] & 0xffffffffull) * dim;
        for (uint32_t d = 0; d < dim; ++d) piece[d] = piece[d] + src[d];
      }
      if (pb == b) {
        memcpy(g, piece, sizeof(float) * dim);
      } else {
        for (uint32_t d = 0; d < dim; ++d) g[d] = g[d] + piece[d];
      }
    }
    float* wr = a->w + (uint64_t)row * dim;
    if (a->opt == ORC_OPT_SGD) {
      for (uint32_t d = 0; d < dim; ++d) wr[d] = fmaf(-a->lr, g[d], wr[d]);
    } else {
      const uint32_t v = dim / 32;
      float q[32];
      for (uint32_t l = 0; l < 32; ++l) {
        float acc = 0.0f;
        for (uint32_t j = 0; j < v; ++j) {
          const float x = g[l * v + j];
          acc = fmaf(x, x, acc);
        }
        q[l] = acc;
      }
      for (uint32_t m = 16; m >= 1; m >>= 1) {
        float nq[32];
        for (uint32_t l = 0; l < 32; ++l) nq[l] = q[l] + q[l ^ m];
        memcpy(q, nq, sizeof(q));
      }
      const float gs = a->state[row] + q[0] / (float)dim;
      a->state[row] = gs;
      const float denom = sqrtf(gs) + a->eps;
      for (uint32_t d = 0; d < dim; ++d) wr[d] = fmaf(-a->lr, g[d] / denom, wr[d]);
    }
  }
  free(g);
  free(piece);
}

uint64_t orc_backward_update(float* w, float* state, uint64_t n, uint32_t dim,
                             const uint32_t* rows, uint64_t occ,
                             const float* grads, int optimizer, float lr,
                             float eps, int threads) {
  if (occ == 0) return 0;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * occ);
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (occ + 1));
  for (uint64_t i = 0; i < occ; ++i) keys[i] = ((uint64_t)rows[i] << 32) | i;
  int row_bits = 1;
  while (row_bits < 32 && (1ull << row_bits) < n) ++row_bits;
  /* low 32 bits already ascending within equal rows: sorting the row bits
   * stably keeps that order */
  for (uint64_t i = 0; i < occ; ++i) keys[i] = (keys[i] >> 32) | (keys[i] << 32);
  radix_sort_u64(keys, tmp, occ, (row_bits + 7) & ~7);
  for (uint64_t i = 0; i < occ; ++i) keys[i] = (keys[i] >> 32) | (keys[i] << 32);
  uint64_t nseg = 0;
  for (uint64_t i = 0; i < occ; ++i)
    if (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) tmp[nseg++] = i;
  tmp[nseg] = occ;
  bwd_args a = {w, state, dim, keys, tmp, nseg, grads, optimizer, lr, eps};
  run_par(bwd_job, &a, threads);
  free(keys);
  free(tmp);
  return nseg;
}
