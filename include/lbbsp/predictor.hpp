// lbbsp/predictor.hpp -- B200 drop-in for the reference speed-predictor API
// (core/include/lbbsp/predictor.hpp:15-136). EMA (K3), narx_predict (K4) and
// narx_train_online (K5: scaler refit, backtracking GD, early stop) run as the
// bit-exact fp64 device kernels behind the C-ABI; the reference types
// (SpeedHistory, NarxModel with its training_loss log, PredictorConfig,
// SpeedPredictor) are kept so callers compile unchanged.
#pragma once
#include <array>
#include <cstdint>
#include <filesystem>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "lbbsp/batch_sizer.hpp"  // throw_status
#include "lbbsp_c.h"

namespace lbbsp {

struct SpeedHistory {
  std::vector<double> speed;
  std::vector<double> cpu_avail;
  std::vector<double> mem_avail;
  void push(double v, double c, double m) {
    speed.push_back(v);
    cpu_avail.push_back(c);
    mem_avail.push_back(m);
  }
  std::size_t size() const { return speed.size(); }
};

struct SeriesScaler {
  double mean = 0.0;
  double stddev = 1.0;
  double norm(double x) const { return (x - mean) / stddev; }
  double denorm(double z) const { return mean + stddev * z; }
};

struct NarxModel {
  static constexpr int kSpeedLags = 2;
  static constexpr int kCpuWindow = 3;
  static constexpr int kMemWindow = 3;
  static constexpr int kInputs = kSpeedLags + kCpuWindow + kMemWindow;
  std::array<double, kInputs> input_weights{};
  double hidden_bias = 0.0;
  double output_weight = 1.0;
  double output_bias = 0.0;
  SeriesScaler speed_scaler{};
  SeriesScaler cpu_scaler{};
  SeriesScaler mem_scaler{};
  std::vector<double> training_loss;
  static constexpr int parameter_count() { return kInputs + 3; }
};

struct NarxTrainConfig {
  double step = 0.05;
  int max_epochs = 500;
  double early_stop_delta = 1e-4;
  int early_stop_patience = 4;
  int min_history = 500;
};

struct NarxTrainReport {
  bool ran = false;
  int epochs = 0;
  double final_loss = 0.0;
};

namespace b200_detail {
inline lbbsp_narx_model to_c(const NarxModel& m) {
  lbbsp_narx_model c{};
  for (int j = 0; j < NarxModel::kInputs; ++j) c.input_weights[j] = m.input_weights[static_cast<std::size_t>(j)];
  c.hidden_bias = m.hidden_bias;
  c.output_weight = m.output_weight;
  c.output_bias = m.output_bias;
  c.speed_mean = m.speed_scaler.mean;
  c.speed_stddev = m.speed_scaler.stddev;
  c.cpu_mean = m.cpu_scaler.mean;
  c.cpu_stddev = m.cpu_scaler.stddev;
  c.mem_mean = m.mem_scaler.mean;
  c.mem_stddev = m.mem_scaler.stddev;
  return c;
}
inline void from_c(const lbbsp_narx_model& c, NarxModel& m) {  // keeps m.training_loss
  for (int j = 0; j < NarxModel::kInputs; ++j) m.input_weights[static_cast<std::size_t>(j)] = c.input_weights[j];
  m.hidden_bias = c.hidden_bias;
  m.output_weight = c.output_weight;
  m.output_bias = c.output_bias;
  m.speed_scaler = {c.speed_mean, c.speed_stddev};
  m.cpu_scaler = {c.cpu_mean, c.cpu_stddev};
  m.mem_scaler = {c.mem_mean, c.mem_stddev};
}
inline lbbsp_narx_train_cfg to_c(const NarxTrainConfig& t) {
  return lbbsp_narx_train_cfg{t.step, t.max_epochs, t.early_stop_delta, t.early_stop_patience, t.min_history};
}
}  // namespace b200_detail

inline double predict_memoryless(const SpeedHistory& history) {
  if (history.size() == 0) throw std::invalid_argument("predict_memoryless: empty history");
  return history.speed.back();
}

// predictor.cpp:18-25, device K3 (same left fold)
inline double ema(std::span<const double> series, double alpha) {
  double out = 0.0;
  throw_status(lbbsp_ema(series.data(), static_cast<int>(series.size()), alpha, &out));
  return out;
}
inline double predict_ema(const SpeedHistory& history, double alpha) { return ema(history.speed, alpha); }
inline double predict_comm_ema(std::span<const double> comm_s, double alpha) { return ema(comm_s, alpha); }

inline NarxModel narx_init(std::uint64_t seed) {
  lbbsp_narx_model c{};
  throw_status(lbbsp_narx_init(seed, &c));
  NarxModel m;
  b200_detail::from_c(c, m);
  return m;
}

// predictor.cpp:147-153, device K4
inline double narx_predict(const NarxModel& model, const std::array<double, 2>& recent_speeds,
                           const std::array<double, 3>& cpu_window, const std::array<double, 3>& mem_window,
                           double floor = 1e-3) {
  const lbbsp_narx_model c = b200_detail::to_c(model);
  double out = 0.0;
  throw_status(lbbsp_narx_predict(&c, recent_speeds.data(), cpu_window.data(), mem_window.data(), floor, &out));
  return out;
}

// predictor.cpp:155-196, device K5 (bit-exact); appends the accepted epochs'
// losses to model.training_loss as the reference does
inline NarxTrainReport narx_train_online(NarxModel& model, const SpeedHistory& history,
                                         const NarxTrainConfig& cfg = {}) {
  lbbsp_narx_model c = b200_detail::to_c(model);
  const lbbsp_narx_train_cfg tc = b200_detail::to_c(cfg);
  lbbsp_narx_report r{};
  std::vector<double> log(static_cast<std::size_t>(cfg.max_epochs > 0 ? cfg.max_epochs : 1));
  throw_status(lbbsp_narx_train_online(&c, history.speed.data(), history.cpu_avail.data(),
                                       history.mem_avail.data(), static_cast<int>(history.size()), &tc, &r,
                                       log.data()));
  b200_detail::from_c(c, model);
  model.training_loss.insert(model.training_loss.end(), log.begin(), log.begin() + r.epochs);
  return NarxTrainReport{r.ran != 0, r.epochs, r.final_loss};
}

inline void save_narx_csv(const NarxModel& model, const std::filesystem::path& path) {
  const lbbsp_narx_model c = b200_detail::to_c(model);
  throw_status(lbbsp_narx_save_csv(&c, path.string().c_str()));
}
inline NarxModel load_narx_csv(const std::filesystem::path& path) {
  lbbsp_narx_model c{};
  throw_status(lbbsp_narx_load_csv(path.string().c_str(), &c));
  NarxModel m;
  b200_detail::from_c(c, m);
  return m;
}

enum class PredictorKind { Memoryless, Ema, Narx, Perfect };

inline const char* to_string(PredictorKind kind) {
  switch (kind) {
    case PredictorKind::Memoryless: return "memoryless";
    case PredictorKind::Ema: return "ema";
    case PredictorKind::Narx: return "narx";
    case PredictorKind::Perfect: return "perfect";
  }
  return "?";
}

inline PredictorKind predictor_from_string(std::string_view name) {
  for (PredictorKind k : {PredictorKind::Memoryless, PredictorKind::Ema, PredictorKind::Narx, PredictorKind::Perfect})
    if (name == to_string(k)) return k;
  throw std::invalid_argument("unknown predictor: " + std::string(name));
}

struct PredictorConfig {
  PredictorKind kind = PredictorKind::Ema;
  double alpha = 0.2;
  int warmup_iterations = 500;
  double speed_floor = 1e-3;
  NarxTrainConfig train{};
  std::filesystem::path initial_weights;
};

// predictor.hpp:118-136 (predictor.cpp:255-297)
class SpeedPredictor {
 public:
  SpeedPredictor() = default;
  SpeedPredictor(const PredictorConfig& cfg, std::uint64_t seed) : cfg_(cfg) {
    cfg_.train.min_history = cfg_.warmup_iterations;  // the warm-up gates training
    model_ = cfg_.initial_weights.empty() ? narx_init(seed) : load_narx_csv(cfg_.initial_weights);
  }

  double predict(const SpeedHistory& history, double cpu_now, double mem_now) const {
    switch (cfg_.kind) {
      case PredictorKind::Memoryless:
        return predict_memoryless(history);
      case PredictorKind::Ema:
      case PredictorKind::Perfect:
        return predict_ema(history, cfg_.alpha);
      case PredictorKind::Narx: {
        const std::size_t k = history.size();
        if (static_cast<long long>(k) < cfg_.warmup_iterations || k < 2) return predict_ema(history, cfg_.alpha);
        return narx_predict(model_, {history.speed[k - 1], history.speed[k - 2]},
                            {cpu_now, history.cpu_avail[k - 1], history.cpu_avail[k - 2]},
                            {mem_now, history.mem_avail[k - 1], history.mem_avail[k - 2]}, cfg_.speed_floor);
      }
    }
    throw std::logic_error("SpeedPredictor::predict: unknown predictor kind");
  }

  NarxTrainReport train(const SpeedHistory& history) {
    if (cfg_.kind != PredictorKind::Narx) return {};
    return narx_train_online(model_, history, cfg_.train);
  }

  const NarxModel& model() const { return model_; }
  const PredictorConfig& config() const { return cfg_; }

 private:
  PredictorConfig cfg_{};
  NarxModel model_{};
};

}  // namespace lbbsp
