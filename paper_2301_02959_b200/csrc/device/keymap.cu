// ts_keymap_*: raw (table_id, row_id) keys -> canonical row index on the
// device.  The reference identifies rows by (table_id, row_id) everywhere
// outside the canonical order (RowRecord, distribution.hpp:31-38; the plan
// document's dp_rows / flex_rows and the assignment CSV, json_io.cpp:235-244,
// 380-394); an input pipeline sends those raw ids, the table consumes
// canonical indices.  SURVEY.md §8(f) row 1.
//
// Layout: one dense u32 slot per (table, row id) in [0, span_t) where span_t
// = 1 + the table's largest row id (row ids of a table are dense in
// practice: synthesize_zipf / histograms number rows 0..E-1), tables
// concatenated; a small per-table-id directory {base, span} (table ids are
// small integers).  A lookup is one coalesced 12 B key read, one 16 B
// directory read (L1/L2-resident) and one random 4 B slot read, 4 B write:
// HBM-bound.  Absent keys map to kAbsent and are counted.
#include <cuda_runtime.h>

#include <map>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace tsd {
namespace {

constexpr uint32_t kAbsent = 0xFFFFFFFFu;
constexpr int kThreads = 256;
constexpr uint32_t kMaxTableId = 1u << 24;

struct TableDir {
  uint64_t base;
  uint64_t span;  // 0: table absent
};

__global__ void __launch_bounds__(kThreads)
keymap_fill_kernel(const uint32_t* __restrict__ table_ids, const uint64_t* __restrict__ row_ids,
                   uint64_t n, const TableDir* __restrict__ dir, uint32_t* __restrict__ slots,
                   unsigned long long* __restrict__ dups) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) {
    const TableDir d = dir[table_ids[i]];
    const uint32_t prev = atomicExch(slots + d.base + row_ids[i], static_cast<uint32_t>(i));
    if (prev != kAbsent) atomicAdd(dups, 1ull);
  }
}

__global__ void __launch_bounds__(kThreads)
keymap_lookup_kernel(const uint32_t* __restrict__ table_ids, const uint64_t* __restrict__ row_ids,
                     uint64_t n, const TableDir* __restrict__ dir, uint32_t n_dir,
                     const uint32_t* __restrict__ slots, uint32_t* __restrict__ canon,
                     unsigned long long* __restrict__ misses) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  unsigned miss = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) {
    const uint32_t t = __ldg(table_ids + i);
    const uint64_t r = __ldg(row_ids + i);
    uint32_t c = kAbsent;
    if (t < n_dir) {
      const TableDir d = dir[t];
      if (r < d.span) c = __ldg(slots + d.base + r);
    }
    canon[i] = c;
    miss += c == kAbsent;
  }
  // one atomic per warp
  for (int m = 16; m >= 1; m >>= 1) miss += __shfl_xor_sync(0xFFFFFFFFu, miss, m);
  if ((threadIdx.x & 31u) == 0 && miss) atomicAdd(misses, static_cast<unsigned long long>(miss));
}

}  // namespace
}  // namespace tsd

struct ts_keymap {
  int device = 0;
  uint64_t n_rows = 0;
  uint32_t n_dir = 0;
  tsd::TableDir* d_dir = nullptr;
  uint32_t* d_slots = nullptr;
  unsigned long long* d_count = nullptr;
  cudaStream_t stream = nullptr;
  // ts_table_forward_keys scratch, one per table: the table's backward reads
  // its forward's ids again, so a second table sharing this map must not
  // overwrite them (kept until that table's next call or the map's destroy)
  struct Canon {
    uint32_t* ptr = nullptr;
    uint64_t cap = 0;
  };
  std::map<const ts_table*, Canon> canon;

  void destroy() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& kv : canon) cudaFree(kv.second.ptr);
    canon.clear();
    cudaFree(d_dir);
    cudaFree(d_slots);
    cudaFree(d_count);
    if (stream) cudaStreamDestroy(stream);
  }
};

extern "C" {

ts_status ts_keymap_create(ts_keymap** out, int device, uint64_t n_rows, const uint32_t* table_ids,
                           const uint64_t* row_ids) {
  return tsd::guarded([&] {
    using namespace tsd;
    if (!out || (n_rows && (!table_ids || !row_ids))) fail(TS_ERR_CONFIG, "ts_keymap_create: null argument");
    *out = nullptr;
    if (n_rows >= kAbsent) fail(TS_ERR_VALIDATION, "keymap: need rows < 2^32 - 1");
    // directory over table ids (host; validation before any device work)
    uint32_t max_t = 0;
    for (uint64_t i = 0; i < n_rows; ++i) max_t = std::max(max_t, table_ids[i]);
    if (n_rows && max_t >= kMaxTableId) {
      fail(TS_ERR_CONFIG, "keymap: table_id " + std::to_string(max_t) + " exceeds the directory limit 2^24");
    }
    const uint32_t n_dir = n_rows ? max_t + 1 : 0;
    std::vector<uint64_t> span(n_dir, 0);
    // row ids far beyond the dense map's reach are rejected here (row_id + 1
    // must not wrap, and the span check below needs the true extent)
    constexpr uint64_t kMaxRowId = uint64_t{1} << 40;
    for (uint64_t i = 0; i < n_rows; ++i) {
      if (row_ids[i] >= kMaxRowId) {
        fail(TS_ERR_CONFIG, "keymap: row id " + std::to_string(row_ids[i]) + " too large for the dense map (< 2^40)");
      }
      span[table_ids[i]] = std::max(span[table_ids[i]], row_ids[i] + 1);
    }
    std::vector<TableDir> dir(n_dir);
    uint64_t total = 0;
    for (uint32_t t = 0; t < n_dir; ++t) {
      dir[t] = TableDir{total, span[t]};
      total += span[t];
    }
    if (total > 4 * n_rows + (uint64_t{1} << 24)) {
      fail(TS_ERR_CONFIG, "keymap: row ids too sparse for the dense map (" + std::to_string(total) +
                              " slots for " + std::to_string(n_rows) + " rows)");
    }
    use_device(device);
    auto m = std::make_unique<ts_keymap>();
    m->device = device;
    m->n_rows = n_rows;
    m->n_dir = n_dir;
    try {
      TSD_CUDA(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
      TSD_CUDA(dev_alloc(&m->d_dir, sizeof(TableDir) * std::max<uint32_t>(n_dir, 1)));
      TSD_CUDA(dev_alloc(&m->d_slots, sizeof(uint32_t) * std::max<uint64_t>(total, 1)));
      TSD_CUDA(dev_alloc(&m->d_count, sizeof(unsigned long long)));
      TSD_CUDA(cudaMemsetAsync(m->d_slots, 0xFF, sizeof(uint32_t) * std::max<uint64_t>(total, 1), m->stream));
      TSD_CUDA(cudaMemsetAsync(m->d_count, 0, sizeof(unsigned long long), m->stream));
      if (n_rows) {
        TSD_CUDA(cudaMemcpyAsync(m->d_dir, dir.data(), sizeof(TableDir) * n_dir, cudaMemcpyHostToDevice,
                                 m->stream));
        uint32_t* d_t = nullptr;
        uint64_t* d_r = nullptr;
        TSD_CUDA(dev_alloc(&d_t, sizeof(uint32_t) * n_rows));
        TSD_CUDA(dev_alloc(&d_r, sizeof(uint64_t) * n_rows));
        TSD_CUDA(cudaMemcpyAsync(d_t, table_ids, sizeof(uint32_t) * n_rows, cudaMemcpyHostToDevice, m->stream));
        TSD_CUDA(cudaMemcpyAsync(d_r, row_ids, sizeof(uint64_t) * n_rows, cudaMemcpyHostToDevice, m->stream));
        const unsigned grid = std::max(1u, std::min<unsigned>(ceil_div(n_rows, kThreads), 8 * sm_count()));
        keymap_fill_kernel<<<grid, kThreads, 0, m->stream>>>(d_t, d_r, n_rows, m->d_dir, m->d_slots, m->d_count);
        TSD_LAUNCH_CHECK();
        unsigned long long dups = 0;
        TSD_CUDA(cudaMemcpyAsync(&dups, m->d_count, sizeof(dups), cudaMemcpyDeviceToHost, m->stream));
        TSD_CUDA(cudaStreamSynchronize(m->stream));
        cudaFree(d_t);
        cudaFree(d_r);
        if (dups) {
          fail(TS_ERR_VALIDATION, "keymap: " + std::to_string(dups) + " duplicate (table_id, row_id) keys");
        }
      }
    } catch (...) {
      m->destroy();
      throw;
    }
    *out = m.release();
  });
}

ts_status ts_keymap_lookup(ts_keymap* m, const uint32_t* d_table_ids, const uint64_t* d_row_ids,
                           uint64_t n, uint32_t* d_canon, void* stream, uint64_t* misses) {
  return tsd::guarded([&] {
    using namespace tsd;
    if (!m || (n && (!d_table_ids || !d_row_ids || !d_canon))) {
      fail(TS_ERR_CONFIG, "ts_keymap_lookup: null argument");
    }
    TSD_CUDA(cudaSetDevice(m->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : m->stream;
    TSD_CUDA(cudaMemsetAsync(m->d_count, 0, sizeof(unsigned long long), s));
    if (n) {
      const unsigned grid = std::max(1u, std::min<unsigned>(ceil_div(n, kThreads), 8 * sm_count()));
      keymap_lookup_kernel<<<grid, kThreads, 0, s>>>(d_table_ids, d_row_ids, n, m->d_dir, m->n_dir,
                                                     m->d_slots, d_canon, m->d_count);
      TSD_LAUNCH_CHECK();
    }
    if (misses) {
      unsigned long long c = 0;
      TSD_CUDA(cudaMemcpyAsync(&c, m->d_count, sizeof(c), cudaMemcpyDeviceToHost, s));
      TSD_CUDA(cudaStreamSynchronize(s));
      *misses = c;
    }
  });
}

ts_status ts_table_forward_keys(ts_table* t, ts_keymap* m, const uint32_t* d_table_ids,
                                const uint64_t* d_row_ids, uint64_t occ, float* d_out) {
  uint32_t* canon_out = nullptr;
  const ts_status st = tsd::guarded([&] {
    using namespace tsd;
    if (!t || !m) fail(TS_ERR_CONFIG, "ts_table_forward_keys: null argument");
    void* s = nullptr;
    const ts_status ss = ts_table_stream(t, &s);
    if (ss != TS_OK) fail(ss, ts_last_error());
    TSD_CUDA(cudaSetDevice(m->device));
    ts_keymap::Canon& cb = m->canon[t];
    if (occ > cb.cap) {
      // the table reads these ids again in backward: grow only between steps
      TSD_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(s)));
      cudaFree(cb.ptr);
      cb.ptr = nullptr;
      cb.cap = 0;
      TSD_CUDA(dev_alloc(&cb.ptr, sizeof(uint32_t) * std::max<uint64_t>(occ, 1)));
      cb.cap = occ;
    }
    canon_out = cb.ptr;
    uint64_t misses = 0;
    const ts_status ls = ts_keymap_lookup(m, d_table_ids, d_row_ids, occ, cb.ptr, s, &misses);
    if (ls != TS_OK) fail(ls, ts_last_error());
    if (misses) {
      fail(TS_ERR_VALIDATION, "forward_keys: " + std::to_string(misses) +
                                  " (table_id, row_id) keys are absent from the plan");
    }
  });
  if (st != TS_OK) return st;
  return ts_table_forward(t, canon_out, occ, d_out);
}

ts_status ts_keymap_destroy(ts_keymap* m) {
  return tsd::guarded([&] {
    if (!m) return;
    m->destroy();
    delete m;
  });
}

}  // extern "C"
