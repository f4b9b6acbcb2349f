// lbbsp_b200.hpp -- header-only C++ shim that re-exposes the reference's
// hot-path signatures (core/include/lbbsp/batch_sizer.hpp:24-46,
// predictor.hpp:29-37,82-96, coordination.hpp:32,43) on top of the B200 C-ABI
// (lbbsp_c.h), throwing the same exception types with the same messages.
// A reference-side caller swaps `lbbsp::` for `lbbsp::b200::` (or adds
// `using namespace lbbsp::b200;`) and links liblbbsp_b200.so. See
// INTEGRATION.md.
#pragma once
#include <array>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbbsp_c.h"

namespace lbbsp::b200 {

using GpuProfile = lbbsp_gpu_profile;  // same field order as lbbsp::GpuProfile

struct BatchAssignment {
  std::vector<int> sizes;
  int total_budget = 0;
};

// lbbsp::ConfigError (scenario.hpp:13-15)
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// status -> reference exception type
inline void throw_if(int rc) {
  if (rc == LBBSP_OK) return;
  const std::string msg = lbbsp_last_error();
  switch (rc) {
    case LBBSP_CONFIG: throw ConfigError(msg);
    case LBBSP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LBBSP_OUT_OF_RANGE: throw std::out_of_range(msg);
    case LBBSP_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// batch_sizer.hpp:24 -- K1 single-block kernel
inline BatchAssignment cpu_allocate(std::span<const double> speeds, int total_budget) {
  BatchAssignment a;
  a.total_budget = total_budget;
  a.sizes.resize(speeds.size());
  throw_if(lbbsp_cpu_allocate(speeds.data(), static_cast<int>(speeds.size()), total_budget,
                              a.sizes.data()));
  return a;
}

// batch_sizer.hpp:30 -- K2 single-block kernel
inline BatchAssignment gpu_allocate(std::span<const GpuProfile> profiles,
                                    std::span<const double> comm_s, int total_budget) {
  if (profiles.size() != comm_s.size())
    throw std::invalid_argument("gpu_allocate: profiles/comm size mismatch");
  BatchAssignment a;
  a.total_budget = total_budget;
  a.sizes.resize(profiles.size());
  throw_if(lbbsp_gpu_allocate(profiles.data(), comm_s.data(), static_cast<int>(profiles.size()),
                              total_budget, a.sizes.data()));
  return a;
}

// batch_sizer.hpp:45
inline double clamp_speed_floor(double speed, double floor = 1e-3) {
  return speed > floor ? speed : floor;
}

// predictor.hpp:32 -- K3
inline double ema(std::span<const double> series, double alpha) {
  double out = 0.0;
  throw_if(lbbsp_ema(series.data(), static_cast<int>(series.size()), alpha, &out));
  return out;
}

using NarxModel = lbbsp_narx_model;
using NarxTrainConfig = lbbsp_narx_train_cfg;
using NarxTrainReport = lbbsp_narx_report;

inline NarxTrainConfig default_train_config() { return NarxTrainConfig{0.05, 500, 1e-4, 4, 500}; }

inline NarxModel narx_init(std::uint64_t seed) {
  NarxModel m{};
  throw_if(lbbsp_narx_init(seed, &m));
  return m;
}

// predictor.hpp:82 -- K4
inline double narx_predict(const NarxModel& model, const std::array<double, 2>& recent_speeds,
                           const std::array<double, 3>& cpu_window,
                           const std::array<double, 3>& mem_window, double floor = 1e-3) {
  double out = 0.0;
  throw_if(lbbsp_narx_predict(&model, recent_speeds.data(), cpu_window.data(), mem_window.data(),
                              floor, &out));
  return out;
}

// predictor.hpp:95 -- K5 (bit-exact fp64 trainer), history as three series
inline NarxTrainReport narx_train_online(NarxModel& model, std::span<const double> speed,
                                         std::span<const double> cpu,
                                         std::span<const double> mem,
                                         const NarxTrainConfig& cfg = default_train_config(),
                                         std::vector<double>* training_loss = nullptr) {
  NarxTrainReport r{};
  std::vector<double> log(static_cast<std::size_t>(cfg.max_epochs > 0 ? cfg.max_epochs : 1));
  throw_if(lbbsp_narx_train_online(&model, speed.data(), cpu.data(), mem.data(),
                                   static_cast<int>(speed.size()), &cfg, &r, log.data()));
  if (training_loss) training_loss->insert(training_loss->end(), log.begin(), log.begin() + r.epochs);
  return r;
}

// coordination.hpp:32/43 -- K8 (values row-major [n][dim])
inline std::vector<double> aggregate(std::span<const double> grads, std::span<const int> sizes,
                                     int dim, bool weighted) {
  std::vector<double> out(static_cast<std::size_t>(dim));
  throw_if(lbbsp_aggregate(grads.data(), sizes.data(), static_cast<int>(sizes.size()), dim,
                           weighted ? 1 : 0, out.data()));
  return out;
}

// scenario.hpp:82-90 -- CLI entry points over the device driver (exit status)
inline int cmd_run(const std::string& config, const std::string& out_dir,
                   std::optional<std::uint64_t> seed_override = std::nullopt) {
  return lbbsp_cmd_run(config.c_str(), out_dir.c_str(), seed_override ? 1 : 0,
                       seed_override.value_or(0));
}

// predictor.cpp:215-243
inline lbbsp_narx_model load_narx_csv(const std::string& path) {
  lbbsp_narx_model m{};
  throw_if(lbbsp_narx_load_csv(path.c_str(), &m));
  return m;
}

}  // namespace lbbsp::b200
