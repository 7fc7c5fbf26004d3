// Small host-side parallel helpers for the planner's O(n) / O(n log n) passes
// over up to 1.6e9 canonical rows (C5).  Parallelism never changes a result:
// sorts are by a strict total order and every floating-point reduction that a
// threshold is compared against stays sequential.
#pragma once

#include <algorithm>
#include <cstddef>
#include <thread>
#include <vector>

namespace tiershard::detail {

inline unsigned host_threads() {
  const unsigned hc = std::thread::hardware_concurrency();
  return hc == 0 ? 1u : std::min(hc, 64u);
}

// fn(begin, end) over [0, n) split into contiguous chunks.
template <typename Fn>
void parallel_for(size_t n, Fn&& fn, size_t min_chunk = size_t{1} << 16) {
  unsigned t = host_threads();
  if (n < min_chunk * 2 || t == 1) {
    fn(size_t{0}, n);
    return;
  }
  t = static_cast<unsigned>(std::min<size_t>(t, n / min_chunk));
  std::vector<std::thread> pool;
  pool.reserve(t);
  for (unsigned i = 1; i < t; ++i) {
    pool.emplace_back([&, i] { fn(n * i / t, n * (i + 1) / t); });
  }
  fn(size_t{0}, n / t);
  for (auto& th : pool) th.join();
}

// Chunked std::sort followed by a parallel bottom-up merge tree.
template <typename T, typename Less>
void parallel_sort(std::vector<T>& v, Less less) {
  const size_t n = v.size();
  if (std::is_sorted(v.begin(), v.end(), less)) return;
  unsigned t = host_threads();
  if (n < (size_t{1} << 18) || t == 1) {
    std::sort(v.begin(), v.end(), less);
    return;
  }
  std::vector<size_t> bounds(t + 1);
  for (unsigned i = 0; i <= t; ++i) bounds[i] = n * i / t;
  {
    std::vector<std::thread> pool;
    for (unsigned i = 0; i < t; ++i) {
      pool.emplace_back([&, i] {
        std::sort(v.begin() + bounds[i], v.begin() + bounds[i + 1], less);
      });
    }
    for (auto& th : pool) th.join();
  }
  std::vector<T> buf(n);
  std::vector<T>* src = &v;
  std::vector<T>* dst = &buf;
  while (bounds.size() > 2) {
    std::vector<size_t> next;
    std::vector<std::thread> pool;
    for (size_t i = 0; i + 1 < bounds.size(); i += 2) {
      const size_t lo = bounds[i];
      const size_t mid = bounds[i + 1];
      const size_t hi = i + 2 < bounds.size() ? bounds[i + 2] : mid;
      next.push_back(lo);
      pool.emplace_back([=, &less] {
        std::merge(src->begin() + lo, src->begin() + mid, src->begin() + mid,
                   src->begin() + hi, dst->begin() + lo, less);
      });
    }
    next.push_back(n);
    for (auto& th : pool) th.join();
    bounds.swap(next);
    std::swap(src, dst);
  }
  if (src != &v) v.swap(*src);
}

}  // namespace tiershard::detail
