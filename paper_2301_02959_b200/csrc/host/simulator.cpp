// Workloads, placement and the device-routed simulation (simulator.hpp).
//
// Host parts are bit-identical to /root/reference/proj/src/simulator.cpp:
//   Workload / materialize_iteration  :29-71   (same RNG consumption order)
//   assign_rows                       :82-108  (parallel; pure per row)
//   static all-reduce payloads        :196-210
//   metric derivation                 :271-331 (same formulas and order)
//   mean / compare_to_baseline / compare :374-494
// The per-occurrence routing loop (:223-257) runs on the GPU through
// ts_router_iteration (csrc/device/router.cu); there is no CPU fallback.
#include "tiershard/simulator.hpp"

#include <mutex>
#include <condition_variable>
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <exception>
#include <limits>
#include <thread>

#include "capi_check.hpp"
#include "parallel.hpp"
#include "tiershard/error.hpp"
#include "tiershard_b200.h"

namespace tiershard {

const char* tier_name(Tier t) {
  switch (t) {
    case Tier::kDataParallel: return "dp";
    case Tier::kFlex: return "flex";
    case Tier::kRowWise: return "rw";
  }
  return "?";
}

Workload::Workload(std::shared_ptr<const RowDistribution> dist, uint32_t local_batch,
                   uint32_t num_gpus, uint64_t seed, uint32_t num_iterations)
    : dist_(std::move(dist)), local_batch_(local_batch), num_gpus_(num_gpus), seed_(seed),
      num_iterations_(num_iterations) {
  if (!dist_ || dist_->rows().empty()) {
    throw ValidationError("workload: distribution has no materialized rows");
  }
  expected_length_ = dist_->expected_length();
  if (!(expected_length_ > 0.0)) {
    throw ValidationError("workload: total expected length must be positive");
  }
  if (local_batch_ == 0 || num_gpus_ == 0 || num_iterations_ == 0) {
    throw ValidationError("workload: batch, GPU and iteration counts must be >= 1");
  }
  const auto& rows = dist_->rows();
  std::vector<double> p(rows.size());
  detail::parallel_for(rows.size(), [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) p[i] = rows[i].probability;
  });
  alias_ = AliasTable(p);
}

void Workload::materialize_iteration(uint32_t iteration, IterationBatch& out) const {
  // One stream per iteration; per sample: Poisson(L) length, then that many
  // alias draws, GPU-major sample order.
  SplitMix64 rng(derive_seed(seed_, iteration));
  const uint64_t samples = uint64_t{local_batch_} * num_gpus_;
  out.local_batch = local_batch_;
  out.num_gpus = num_gpus_;
  out.rows.clear();
  out.sample_offsets.assign(1, 0);
  out.sample_offsets.reserve(samples + 1);
  for (uint64_t s = 0; s < samples; ++s) {
    for (uint32_t left = poisson(rng, expected_length_); left > 0; --left) {
      out.rows.push_back(alias_.sample(rng));
    }
    out.sample_offsets.push_back(out.rows.size());
  }
}

Workload sample_workload(std::shared_ptr<const RowDistribution> dist,
                         const CostModelConfig& cfg, const Topology& topo, uint64_t seed,
                         uint32_t num_iterations) {
  cfg.validate();
  topo.validate();
  return Workload(std::move(dist), cfg.local_batch, topo.total_gpus(), seed, num_iterations);
}

std::vector<RowPlacement> assign_rows(const ShardingPlan& plan, const RowDistribution& dist,
                                      const Topology& topo, uint64_t hash_seed) {
  const auto& rows = dist.rows();
  if (plan.total_rows != rows.size() || plan.dp_cut > plan.flex_cut ||
      plan.flex_cut > plan.total_rows) {
    throw ValidationError("assign_rows: plan does not cover the distribution");
  }
  const uint64_t u = topo.total_gpus();
  const uint64_t w = topo.gpus_per_node;
  std::vector<RowPlacement> out(rows.size());
  detail::parallel_for(rows.size(), [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      RowPlacement& pl = out[i];
      if (i < plan.dp_cut) {
        pl.tier = Tier::kDataParallel;
        continue;
      }
      const uint64_t h = row_key_hash(rows[i].table_id, rows[i].row_id, hash_seed);
      if (i < plan.flex_cut) {
        pl.tier = Tier::kFlex;
        pl.flex_slot = static_cast<uint32_t>(h % w);
      } else {
        pl.tier = Tier::kRowWise;
        pl.owner_gpu = static_cast<uint32_t>(h % u);
      }
    }
  });
  return out;
}

namespace {

constexpr std::array<double IterationMetrics::*, 26> kMetricFields = {
    &IterationMetrics::global_a2a_send_max,       &IterationMetrics::global_a2a_recv_max,
    &IterationMetrics::global_a2a_bytes_mean,     &IterationMetrics::global_a2a_total,
    &IterationMetrics::intra_a2a_send_max,        &IterationMetrics::intra_a2a_recv_max,
    &IterationMetrics::intra_a2a_bytes_mean,      &IterationMetrics::intra_a2a_total,
    &IterationMetrics::ar_global_bytes,           &IterationMetrics::ar_cross_bytes_max,
    &IterationMetrics::ar_cross_bytes_mean,       &IterationMetrics::global_a2a_seconds,
    &IterationMetrics::intra_a2a_seconds,         &IterationMetrics::ar_global_seconds,
    &IterationMetrics::ar_cross_seconds,          &IterationMetrics::total_seconds,
    &IterationMetrics::total_seconds_critical,    &IterationMetrics::peak_dynamic_memory_bytes,
    &IterationMetrics::rows_accessed_scalars_min, &IterationMetrics::rows_accessed_scalars_max,
    &IterationMetrics::rows_accessed_scalars_mean, &IterationMetrics::load_imbalance,
    &IterationMetrics::distinct_rows_min,         &IterationMetrics::distinct_rows_max,
    &IterationMetrics::distinct_rows_mean,        &IterationMetrics::distinct_row_imbalance};

struct Spread {
  double lo, hi, avg;
};

Spread spread(const uint64_t* v, uint32_t u) {
  const auto [mn, mx] = std::minmax_element(v, v + u);
  uint64_t sum = 0;
  for (uint32_t i = 0; i < u; ++i) sum += v[i];
  return Spread{static_cast<double>(*mn), static_cast<double>(*mx),
                static_cast<double>(sum) / static_cast<double>(u)};
}

// Static (plan-only) collective payloads of one iteration.
struct StaticPayload {
  double ar_global = 0.0, ar_cross_max = 0.0, ar_cross_mean = 0.0;
};

// Counters (7 x U, ts_router layout) -> IterationMetrics, reference formulas.
IterationMetrics derive_metrics(const uint64_t* c, uint32_t u, const CostModelConfig& cfg,
                                const Topology& topo, const StaticPayload& sp) {
  const uint64_t* send_g = c + TS_CTR_SEND_GLOBAL * u;
  const uint64_t* recv_g = c + TS_CTR_RECV_GLOBAL * u;
  const uint64_t* send_i = c + TS_CTR_SEND_INTRA * u;
  const uint64_t* recv_i = c + TS_CTR_RECV_INTRA * u;
  const uint64_t* dp_loc = c + TS_CTR_DP_LOCAL * u;
  const double row_bytes = static_cast<double>(cfg.embedding_dim) * cfg.scalar_bytes;
  const double dyn = cfg.dynamic_pass_count;
  const double stat = cfg.static_pass_count;
  const double id_bytes = cfg.include_id_bytes ? cfg.bytes_per_id : 0.0;

  uint64_t tot_sg = 0, tot_rg = 0, tot_si = 0, tot_ri = 0;
  uint64_t max_sg = 0, max_rg = 0, max_si = 0, max_ri = 0, peak = 0;
  for (uint32_t g = 0; g < u; ++g) {
    tot_sg += send_g[g];
    tot_rg += recv_g[g];
    tot_si += send_i[g];
    tot_ri += recv_i[g];
    max_sg = std::max(max_sg, send_g[g]);
    max_rg = std::max(max_rg, recv_g[g]);
    max_si = std::max(max_si, send_i[g]);
    max_ri = std::max(max_ri, recv_i[g]);
    peak = std::max(peak, send_g[g] + recv_g[g] + send_i[g] + recv_i[g] + dp_loc[g]);
  }
  if (tot_sg != tot_rg || tot_si != tot_ri) throw Error("simulate: byte conservation violated");

  IterationMetrics m;
  m.global_a2a_send_max = static_cast<double>(max_sg) * row_bytes;
  m.global_a2a_recv_max = static_cast<double>(max_rg) * row_bytes;
  m.global_a2a_total = static_cast<double>(tot_sg) * row_bytes;
  m.global_a2a_bytes_mean = m.global_a2a_total / u;
  m.intra_a2a_send_max = static_cast<double>(max_si) * row_bytes;
  m.intra_a2a_recv_max = static_cast<double>(max_ri) * row_bytes;
  m.intra_a2a_total = static_cast<double>(tot_si) * row_bytes;
  m.intra_a2a_bytes_mean = m.intra_a2a_total / u;
  m.ar_global_bytes = sp.ar_global;
  m.ar_cross_bytes_max = sp.ar_cross_max;
  m.ar_cross_bytes_mean = sp.ar_cross_mean;

  const uint64_t g_units = std::max(max_sg, max_rg);
  const uint64_t i_units = std::max(max_si, max_ri);
  m.global_a2a_seconds = dyn * (static_cast<double>(g_units) * row_bytes) / topo.a2a_global;
  m.intra_a2a_seconds = dyn * (static_cast<double>(i_units) * row_bytes) / topo.a2a_intra;
  if (id_bytes > 0.0) {
    m.global_a2a_seconds += static_cast<double>(g_units) * id_bytes / topo.a2a_global;
    m.intra_a2a_seconds += static_cast<double>(i_units) * id_bytes / topo.a2a_intra;
  }
  m.ar_global_seconds = stat * sp.ar_global / topo.ar_global;
  m.ar_cross_seconds = stat * sp.ar_cross_max / topo.ar_cross;
  m.total_seconds =
      m.global_a2a_seconds + m.intra_a2a_seconds + m.ar_global_seconds + m.ar_cross_seconds;
  m.total_seconds_critical = m.global_a2a_seconds + m.ar_global_seconds;
  m.peak_dynamic_memory_bytes = static_cast<double>(peak) * row_bytes;

  const double d = cfg.embedding_dim;
  const Spread served = spread(c + TS_CTR_SERVED * u, u);
  m.rows_accessed_scalars_min = served.lo * d;
  m.rows_accessed_scalars_max = served.hi * d;
  m.rows_accessed_scalars_mean = served.avg * d;
  m.load_imbalance = served.avg > 0.0 ? served.hi / served.avg : 1.0;
  const Spread distinct = spread(c + TS_CTR_DISTINCT * u, u);
  m.distinct_rows_min = distinct.lo;
  m.distinct_rows_max = distinct.hi;
  m.distinct_rows_mean = distinct.avg;
  m.distinct_row_imbalance = distinct.avg > 0.0 ? distinct.hi / distinct.avg : 1.0;
  return m;
}

// RAII over the C-ABI router handle.
class DeviceRouter {
 public:
  DeviceRouter(const ShardingPlan& plan, const std::vector<RowPlacement>& placements,
               const Topology& topo) {
    std::vector<uint8_t> dest(placements.size(), 0);
    detail::parallel_for(placements.size(), [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) {
        const RowPlacement& p = placements[i];
        dest[i] = static_cast<uint8_t>(p.tier == Tier::kFlex ? p.flex_slot : p.owner_gpu);
      }
    });
    int device = 0;
    if (const char* env = std::getenv("TIERSHARD_DEVICE")) device = std::atoi(env);
    detail::check(ts_router_create(&handle_, device, placements.size(), plan.dp_cut,
                                   plan.flex_cut, dest.data(), topo.num_nodes,
                                   topo.gpus_per_node));
  }
  ~DeviceRouter() {
    if (handle_) ts_router_destroy(handle_);
  }
  DeviceRouter(const DeviceRouter&) = delete;
  DeviceRouter& operator=(const DeviceRouter&) = delete;

  void route(const IterationBatch& b, uint64_t* counters) {
    detail::check(ts_router_iteration(handle_, b.local_batch, b.sample_offsets.data(),
                                      b.rows.data(), b.rows.size(), counters));
  }

 private:
  ts_router* handle_ = nullptr;
};

}  // namespace

SimReport simulate(const ShardingPlan& plan, const Workload& workload,
                   const CostModelConfig& cfg, const Topology& topo, uint64_t hash_seed,
                   unsigned threads) {
  cfg.validate();
  topo.validate();
  const RowDistribution& dist = workload.distribution();
  if (plan.total_rows != dist.rows().size()) {
    throw ValidationError("simulate: workload rows are absent from the plan (row count mismatch)");
  }
  if (workload.local_batch() != cfg.local_batch || workload.num_gpus() != topo.total_gpus()) {
    throw ValidationError("simulate: workload was sampled for a different shape");
  }
  const std::vector<RowPlacement> placements = assign_rows(plan, dist, topo, hash_seed);
  const uint32_t u = topo.total_gpus();
  const uint32_t w = topo.gpus_per_node;
  if (u > 256) throw Error("simulate: the device router supports at most 256 GPUs");

  const double row_bytes = static_cast<double>(cfg.embedding_dim) * cfg.scalar_bytes;
  StaticPayload sp;
  sp.ar_global = static_cast<double>(plan.dp_cut) * row_bytes;
  {
    std::vector<uint64_t> per_slot(w, 0);
    for (size_t i = plan.dp_cut; i < plan.flex_cut; ++i) ++per_slot[placements[i].flex_slot];
    uint64_t most = 0, all = 0;
    for (const uint64_t c : per_slot) {
      most = std::max(most, c);
      all += c;
    }
    sp.ar_cross_max = static_cast<double>(most) * row_bytes;
    sp.ar_cross_mean = static_cast<double>(all) / w * row_bytes;
  }

  DeviceRouter router(plan, placements, topo);
  const uint32_t iterations = workload.num_iterations();
  std::vector<IterationMetrics> results(iterations);
  const unsigned workers = std::max(1u, std::min(threads, iterations));
  std::vector<uint64_t> counters(size_t{TS_NUM_COUNTERS} * u);

  // Pipeline: `workers` host threads materialize iterations (in index order
  // of claim) into a ring of workers + 2 batch slots while this thread routes
  // them on the device in iteration order, so host sampling overlaps device
  // routing.  Iteration i uses slot i % K, which iteration i - K (routed
  // already) has freed.  Each result depends only on its index.
  const uint32_t K = workers + 2;
  std::vector<IterationBatch> slots(K);
  std::vector<uint8_t> ready(iterations, 0);
  std::mutex mu;
  std::condition_variable cv;
  uint32_t next = 0, routed = 0;
  std::exception_ptr error;
  bool stop = false;
  std::vector<std::thread> pool;
  for (unsigned k = 0; k < workers; ++k) {
    pool.emplace_back([&] {
      for (;;) {
        uint32_t it;
        {
          std::unique_lock<std::mutex> lk(mu);
          if (stop || next >= iterations) return;
          it = next++;
          // slot it % K is free once iteration it - K has been routed
          cv.wait(lk, [&] { return stop || it < routed + K; });
          if (stop) return;
        }
        try {
          workload.materialize_iteration(it, slots[it % K]);
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          if (!error) error = std::current_exception();
          stop = true;
          cv.notify_all();
          return;
        }
        std::lock_guard<std::mutex> lk(mu);
        ready[it] = 1;
        cv.notify_all();
      }
    });
  }
  std::exception_ptr route_error;
  for (uint32_t it = 0; it < iterations && !route_error; ++it) {
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return stop || ready[it]; });
      if (!ready[it]) break;  // a worker failed
    }
    try {
      router.route(slots[it % K], counters.data());
      results[it] = derive_metrics(counters.data(), u, cfg, topo, sp);
    } catch (...) {
      route_error = std::current_exception();
    }
    std::lock_guard<std::mutex> lk(mu);
    routed = it + 1;
    if (route_error) stop = true;
    cv.notify_all();
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    stop = true;
    cv.notify_all();
  }
  for (auto& t : pool) t.join();
  if (route_error) std::rethrow_exception(route_error);
  if (error) std::rethrow_exception(error);

  SimReport report;
  report.seed = workload.seed();
  report.hash_seed = hash_seed;
  report.num_iterations = iterations;
  report.iterations = std::move(results);
  const double inv = 1.0 / iterations;
  for (const IterationMetrics& m : report.iterations) {
    for (auto field : kMetricFields) report.mean.*field += m.*field * inv;
  }
  return report;
}

SimComparison compare_to_baseline(const SimReport& baseline, const SimReport& plan) {
  if (baseline.num_iterations != plan.num_iterations || baseline.seed != plan.seed) {
    throw ValidationError("compare_to_baseline: reports come from different workloads");
  }
  SimComparison out;
  out.baseline_global_a2a_bytes = baseline.mean.global_a2a_total;
  out.plan_global_a2a_bytes = plan.mean.global_a2a_total;
  out.global_a2a_reduction = out.baseline_global_a2a_bytes > 0.0
                                 ? 1.0 - out.plan_global_a2a_bytes / out.baseline_global_a2a_bytes
                                 : 0.0;
  out.baseline_total_seconds = baseline.mean.total_seconds;
  out.plan_total_seconds = plan.mean.total_seconds;
  out.plan_total_seconds_critical = plan.mean.total_seconds_critical;
  out.latency_improvement =
      out.plan_total_seconds > 0.0 ? out.baseline_total_seconds / out.plan_total_seconds : 1.0;
  out.latency_improvement_critical =
      out.plan_total_seconds_critical > 0.0
          ? out.baseline_total_seconds / out.plan_total_seconds_critical
          : 1.0;
  out.baseline_peak_dynamic_memory_bytes = baseline.mean.peak_dynamic_memory_bytes;
  out.plan_peak_dynamic_memory_bytes = plan.mean.peak_dynamic_memory_bytes;
  return out;
}

std::vector<MetricDiscrepancy> compare(const CostReport& predicted, const SimReport& simulated,
                                       double tolerance) {
  const IterationMetrics& s = simulated.mean;
  const std::pair<const char*, std::pair<double, double>> rows[] = {
      {"global_a2a_bytes_per_gpu", {predicted.global_a2a_bytes, s.global_a2a_bytes_mean}},
      {"intra_a2a_bytes_per_gpu", {predicted.intra_a2a_bytes, s.intra_a2a_bytes_mean}},
      {"ar_global_bytes_per_gpu", {predicted.ar_global_bytes, s.ar_global_bytes}},
      {"ar_cross_bytes_per_gpu", {predicted.ar_cross_bytes, s.ar_cross_bytes_mean}},
      {"global_a2a_seconds", {predicted.global_a2a_seconds, s.global_a2a_seconds}},
      {"intra_a2a_seconds", {predicted.intra_a2a_seconds, s.intra_a2a_seconds}},
      {"ar_global_seconds", {predicted.ar_global_seconds, s.ar_global_seconds}},
      {"ar_cross_seconds", {predicted.ar_cross_seconds, s.ar_cross_seconds}},
      {"peak_dynamic_memory_bytes",
       {predicted.peak_dynamic_memory_bytes, s.peak_dynamic_memory_bytes}},
      {"rows_accessed_scalars", {predicted.rows_accessed_scalars, s.rows_accessed_scalars_mean}},
  };
  std::vector<MetricDiscrepancy> out;
  for (const auto& [name, values] : rows) {
    MetricDiscrepancy d;
    d.metric = name;
    d.predicted = values.first;
    d.simulated = values.second;
    if (d.predicted == 0.0) {
      d.relative_error = d.simulated == 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
    } else {
      d.relative_error = (d.simulated - d.predicted) / d.predicted;
    }
    d.flagged = std::abs(d.relative_error) > tolerance;
    out.push_back(std::move(d));
  }
  return out;
}

}  // namespace tiershard
