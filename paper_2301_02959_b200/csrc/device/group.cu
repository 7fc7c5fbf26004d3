// In-process rank group (group.cuh): host barrier / all-gather and the
// event-based device rendezvous the U > 1 peer-memory path uses when all of
// its ranks are threads of one process.
#include <array>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "group.cuh"

struct ts_group {
  uint32_t size = 0;
  std::mutex mu;
  std::condition_variable cv;
  uint32_t arrived = 0;
  uint64_t generation = 0;
  bool broken = false;
  std::vector<uint8_t> staging;               // all-gather buffer [size x bytes]
  std::vector<uint8_t> attached;              // rank slot taken
  std::vector<std::array<cudaEvent_t, 2>> ev;  // per rank: rendezvous events (its device)
  std::vector<uint64_t> seq;                  // per rank: rendezvous issued
  std::chrono::seconds timeout{300};
};

namespace tsd {

namespace {

// Host barrier; caller holds `lk`.
void wait_locked(ts_group* g, std::unique_lock<std::mutex>& lk) {
  if (g->broken) fail(TS_ERR_INTERNAL, "group: a rank failed; the group is unusable");
  const uint64_t gen = g->generation;
  if (++g->arrived == g->size) {
    g->arrived = 0;
    ++g->generation;
    g->cv.notify_all();
    return;
  }
  if (!g->cv.wait_for(lk, g->timeout, [&] { return g->generation != gen || g->broken; })) {
    g->broken = true;
    g->cv.notify_all();
    fail(TS_ERR_INTERNAL, "group: rendezvous timed out (TIERSHARD_GROUP_TIMEOUT); a rank did not arrive");
  }
  if (g->broken && g->generation == gen) fail(TS_ERR_INTERNAL, "group: a rank failed; the group is unusable");
}

}  // namespace

void group_attach(ts_group* g, uint32_t rank, int device) {
  if (!g) fail(TS_ERR_CONFIG, "group: null group");
  std::lock_guard<std::mutex> lk(g->mu);
  if (rank >= g->size) fail(TS_ERR_CONFIG, "group: rank out of range");
  if (g->attached[rank]) fail(TS_ERR_CONFIG, "group: rank " + std::to_string(rank) + " is already attached");
  TSD_CUDA(cudaSetDevice(device));
  for (auto& e : g->ev[rank]) TSD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  g->seq[rank] = 0;
  g->attached[rank] = 1;
}

void group_detach(ts_group* g, uint32_t rank) {
  if (!g || rank >= g->size) return;
  std::lock_guard<std::mutex> lk(g->mu);
  if (!g->attached[rank]) return;
  for (auto& e : g->ev[rank]) {
    if (e) cudaEventDestroy(e);
    e = nullptr;
  }
  g->attached[rank] = 0;
}

uint32_t group_size(const ts_group* g) { return g ? g->size : 0; }

void group_wait(ts_group* g) {
  std::unique_lock<std::mutex> lk(g->mu);
  wait_locked(g, lk);
}

void group_allgather(ts_group* g, uint32_t rank, const void* mine, size_t bytes, void* all) {
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->staging.size() < bytes * g->size) g->staging.resize(bytes * g->size);
  if (bytes) std::memcpy(g->staging.data() + bytes * rank, mine, bytes);
  wait_locked(g, lk);  // every slot written
  if (bytes) std::memcpy(all, g->staging.data(), bytes * g->size);
  wait_locked(g, lk);  // every rank has read: the buffer may be reused
}

void group_poison(ts_group* g) {
  if (!g) return;
  std::lock_guard<std::mutex> lk(g->mu);
  g->broken = true;
  g->cv.notify_all();
}

void group_barrier(ts_group* g, uint32_t rank, cudaStream_t stream) {
  std::unique_lock<std::mutex> lk(g->mu);
  const uint64_t k = g->seq[rank]++;
  TSD_CUDA(cudaEventRecord(g->ev[rank][k & 1], stream));
  wait_locked(g, lk);  // every rank has recorded its event k
  for (uint32_t p = 0; p < g->size; ++p) {
    if (p != rank) TSD_CUDA(cudaStreamWaitEvent(stream, g->ev[p][k & 1], 0));
  }
}

}  // namespace tsd

extern "C" {

ts_status ts_group_create(ts_group** out, uint32_t ranks) {
  return tsd::guarded([&] {
    if (!out) tsd::fail(TS_ERR_CONFIG, "ts_group_create: null argument");
    *out = nullptr;
    if (ranks == 0 || ranks > 256) tsd::fail(TS_ERR_CONFIG, "ts_group_create: need 1 <= ranks <= 256");
    auto* g = new ts_group;
    g->size = ranks;
    g->attached.assign(ranks, 0);
    g->ev.assign(ranks, {nullptr, nullptr});
    g->seq.assign(ranks, 0);
    if (const char* e = std::getenv("TIERSHARD_GROUP_TIMEOUT")) {
      g->timeout = std::chrono::seconds(std::max(1, std::atoi(e)));
    }
    *out = g;
  });
}

ts_status ts_group_abort(ts_group* g) {
  return tsd::guarded([&] {
    if (!g) tsd::fail(TS_ERR_CONFIG, "ts_group_abort: null group");
    tsd::group_poison(g);
  });
}

ts_status ts_group_destroy(ts_group* g) {
  return tsd::guarded([&] {
    if (!g) return;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      for (uint8_t a : g->attached) {
        if (a) tsd::fail(TS_ERR_CONFIG, "ts_group_destroy: a table of the group is still alive");
      }
    }
    delete g;
  });
}

}  // extern "C"
