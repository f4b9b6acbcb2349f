// lbbsp/batch_sizer.hpp -- B200 drop-in for the reference solver API
// (core/include/lbbsp/batch_sizer.hpp:10-46). cpu_allocate / gpu_allocate run
// the single-block device kernels K1 / K2 through the C-ABI (bit-exact against
// batch_sizer.cpp:54-99 / 101-199) and throw the reference's exception types
// with its messages. The exhaustive oracles and makespans are CPU test
// utilities (out of scope for the device) written out here so
// that the reference's own tests compile against this header unchanged.
#pragma once
#include <algorithm>
#include <functional>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbbsp_c.h"

namespace lbbsp {

struct GpuProfile {
  double sec_per_sample = 0.0;  // Gamma slope above the saturation point
  double base_time_s = 0.0;     // Gamma intercept
  int saturation_point = 1;
  int oom_point = 1;
};

struct BatchAssignment {
  std::vector<int> sizes;
  int total_budget = 0;
};

// lbbsp_c.h status -> the reference's exception types
inline void throw_status(int rc) {
  if (rc == LBBSP_OK) return;
  const std::string msg = lbbsp_last_error();
  switch (rc) {
    case LBBSP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LBBSP_OUT_OF_RANGE: throw std::out_of_range(msg);
    case LBBSP_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

namespace b200_detail {
inline std::vector<lbbsp_gpu_profile> to_c(std::span<const GpuProfile> p) {
  std::vector<lbbsp_gpu_profile> out(p.size());
  for (std::size_t i = 0; i < p.size(); ++i)
    out[i] = lbbsp_gpu_profile{p[i].sec_per_sample, p[i].base_time_s, p[i].saturation_point, p[i].oom_point};
  return out;
}
inline double gamma_time(const GpuProfile& p, int x, double comm) {
  return p.sec_per_sample * static_cast<double>(std::max(x, p.saturation_point)) + p.base_time_s + comm;
}
// exhaustive search over x_i in [lo_i, hi_i] with sum = budget, minimising
// the largest per-worker cost (first minimum in lexicographic order)
inline std::vector<int> exhaustive(int n, int budget, const std::vector<int>& lo, const std::vector<int>& hi,
                                   const std::function<double(int, int)>& cost) {
  std::vector<int> cur(static_cast<std::size_t>(n)), best;
  double best_val = std::numeric_limits<double>::infinity();
  std::function<void(int, int, double)> rec = [&](int i, int left, double worst) {
    if (i == n - 1) {
      if (left < lo[i] || left > hi[i]) return;
      cur[i] = left;
      const double w = std::max(worst, cost(i, left));
      if (w < best_val) {
        best_val = w;
        best = cur;
      }
      return;
    }
    for (int x = lo[i]; x <= std::min(hi[i], left); ++x) {
      cur[i] = x;
      rec(i + 1, left - x, std::max(worst, cost(i, x)));
    }
  };
  if (n > 0) rec(0, budget, 0.0);
  return best;
}
inline void oracle_size_guard(std::size_t n, int budget) {
  if (n > 4 || budget > 200)
    throw std::invalid_argument("allocate oracle: instance too large (n <= 4, budget <= 200)");
}
}  // namespace b200_detail

// batch_sizer.hpp:24 -- device kernel K1
inline BatchAssignment cpu_allocate(std::span<const double> speeds, int total_budget) {
  BatchAssignment a;
  a.total_budget = total_budget;
  a.sizes.resize(speeds.size());
  throw_status(lbbsp_cpu_allocate(speeds.data(), static_cast<int>(speeds.size()), total_budget, a.sizes.data()));
  return a;
}

// batch_sizer.hpp:30 -- device kernel K2
inline BatchAssignment gpu_allocate(std::span<const GpuProfile> profiles, std::span<const double> comm_s,
                                    int total_budget) {
  if (profiles.size() != comm_s.size())
    throw std::invalid_argument("gpu_allocate: profiles and comm_s differ in length");
  const auto p = b200_detail::to_c(profiles);
  BatchAssignment a;
  a.total_budget = total_budget;
  a.sizes.resize(profiles.size());
  throw_status(lbbsp_gpu_allocate(p.data(), comm_s.data(), static_cast<int>(p.size()), total_budget,
                                  a.sizes.data()));
  return a;
}

inline BatchAssignment oracle_cpu_allocate(std::span<const double> speeds, int total_budget) {
  b200_detail::oracle_size_guard(speeds.size(), total_budget);
  const int n = static_cast<int>(speeds.size());
  if (n == 0) throw std::invalid_argument("oracle_cpu_allocate: no workers");
  if (total_budget < n) throw std::invalid_argument("oracle_cpu_allocate: budget below worker count");
  for (double v : speeds)
    if (!(v > 0.0)) throw std::invalid_argument("oracle_cpu_allocate: speeds must be > 0");
  const std::vector<int> lo(static_cast<std::size_t>(n), 1), hi(static_cast<std::size_t>(n), total_budget);
  return {b200_detail::exhaustive(n, total_budget, lo, hi,
                                  [&](int i, int x) { return static_cast<double>(x) / speeds[i]; }),
          total_budget};
}

inline BatchAssignment oracle_gpu_allocate(std::span<const GpuProfile> profiles, std::span<const double> comm_s,
                                           int total_budget) {
  b200_detail::oracle_size_guard(profiles.size(), total_budget);
  const int n = static_cast<int>(profiles.size());
  if (n == 0 || comm_s.size() != profiles.size())
    throw std::invalid_argument("oracle_gpu_allocate: bad instance");
  std::vector<int> lo, hi;
  for (const auto& p : profiles) {
    lo.push_back(p.saturation_point);
    hi.push_back(p.oom_point);
  }
  auto best = b200_detail::exhaustive(n, total_budget, lo, hi, [&](int i, int x) {
    return b200_detail::gamma_time(profiles[i], x, comm_s[i]);
  });
  if (best.empty()) throw std::invalid_argument("oracle_gpu_allocate: no assignment within the bounds");
  return {best, total_budget};
}

inline double cpu_makespan(std::span<const double> speeds, const BatchAssignment& a) {
  double worst = 0.0;
  for (std::size_t i = 0; i < speeds.size(); ++i) worst = std::max(worst, a.sizes[i] / speeds[i]);
  return worst;
}

inline double gpu_makespan(std::span<const GpuProfile> profiles, std::span<const double> comm_s,
                           const BatchAssignment& a) {
  double worst = 0.0;
  for (std::size_t i = 0; i < profiles.size(); ++i)
    worst = std::max(worst, b200_detail::gamma_time(profiles[i], a.sizes[i], comm_s[i]));
  return worst;
}

// batch_sizer.hpp:45 (batch_sizer.cpp:12-14)
inline double clamp_speed_floor(double speed, double floor = 1e-3) { return speed > floor ? speed : floor; }

}  // namespace lbbsp
