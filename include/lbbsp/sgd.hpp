// lbbsp/sgd.hpp -- B200 drop-in for the reference worker API
// (core/include/lbbsp/sgd.hpp:10-52). The per-worker gradient (K7), the loss
// (K10) and the update (K9) run as device kernels through the C-ABI on a
// device copy of the caller's dataset (uploaded per call: the reference's
// value semantics -- the AoS Dataset stays the caller's), with the
// reference's exceptions and messages. generate_dataset is the setup-time
// host generator (sgd.cpp:32-57).
#pragma once
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

#include "lbbsp/batch_sizer.hpp"  // throw_status
#include "lbbsp_c.h"

namespace lbbsp {

struct Sample {
  std::vector<double> features;
  double label = 0.0;
};

struct Dataset {
  std::vector<Sample> samples;
  int dim = 0;
  std::uint64_t seed = 0;
  std::size_t size() const { return samples.size(); }
};

struct ModelState {
  std::vector<double> params;
  double learning_rate = 0.1;
  std::int64_t clock = 0;
};

struct Gradient {
  std::vector<double> values;
  int batch_size = 0;
};

namespace b200_detail {
struct LrData {
  lbbsp_lr_data* p = nullptr;
  ~LrData() {
    if (p) lbbsp_lr_data_destroy(p);
  }
};
// SoA device copy of an AoS dataset (dimension = the model's)
inline std::unique_ptr<LrData> upload(const Dataset& data, std::size_t dim) {
  const std::size_t n = data.samples.size();
  std::vector<double> feat(n * dim), lab(n);
  for (std::size_t i = 0; i < n; ++i) {
    const auto& f = data.samples[i].features;
    if (f.size() != dim) throw std::invalid_argument("dataset: feature dimension mismatch");
    std::copy(f.begin(), f.end(), feat.begin() + static_cast<std::ptrdiff_t>(i * dim));
    lab[i] = data.samples[i].label;
  }
  auto d = std::make_unique<LrData>();
  throw_status(lbbsp_lr_data_upload(feat.data(), lab.data(), static_cast<int>(n), static_cast<int>(dim), &d->p));
  return d;
}
}  // namespace b200_detail

inline std::vector<double> separator_params(std::uint64_t seed, int dim) {
  std::vector<double> w(static_cast<std::size_t>(dim > 0 ? dim : 0));
  throw_status(lbbsp_separator_params(seed, dim, w.data()));
  return w;
}

inline Dataset generate_dataset(std::uint64_t seed, int n, int d, double noise_amplitude = 0.2) {
  if (n < 1) throw std::invalid_argument("generate_dataset: n must be >= 1");
  if (d < 1) throw std::invalid_argument("generate_dataset: d must be >= 1");
  std::vector<double> feat(static_cast<std::size_t>(n) * d), lab(static_cast<std::size_t>(n));
  throw_status(lbbsp_generate_dataset(seed, n, d, noise_amplitude, feat.data(), lab.data()));
  Dataset out;
  out.dim = d;
  out.seed = seed;
  out.samples.resize(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    auto& s = out.samples[static_cast<std::size_t>(i)];
    s.features.assign(feat.begin() + static_cast<std::ptrdiff_t>(i) * d,
                      feat.begin() + static_cast<std::ptrdiff_t>(i + 1) * d);
    s.label = lab[static_cast<std::size_t>(i)];
  }
  return out;
}

// loss (sgd.cpp:65-70), device K10
inline double loss(const ModelState& model, const Dataset& data) {
  if (data.samples.empty()) throw std::invalid_argument("loss: empty dataset");
  auto d = b200_detail::upload(data, model.params.size());
  double out = 0.0;
  throw_status(lbbsp_loss(d->p, model.params.data(), &out));
  return out;
}

// sample_loss (sgd.cpp:59-63): the K10 kernel over a one-sample dataset
inline double sample_loss(const std::vector<double>& params, const Sample& s) {
  Dataset one;
  one.samples.push_back(s);
  ModelState m;
  m.params = params;
  return loss(m, one);
}

// batch_gradient (sgd.cpp:72-90), device K7
inline Gradient batch_gradient(const ModelState& model, const Dataset& data, std::span<const int> indices) {
  if (indices.empty()) throw std::invalid_argument("batch_gradient: empty index set");
  auto d = b200_detail::upload(data, model.params.size());
  Gradient g;
  g.values.resize(model.params.size());
  throw_status(lbbsp_batch_gradient(d->p, model.params.data(), indices.data(), static_cast<int>(indices.size()),
                                    g.values.data()));
  g.batch_size = static_cast<int>(indices.size());
  return g;
}

// apply_update (sgd.cpp:92-99), device K9
inline ModelState apply_update(ModelState model, const Gradient& g) {
  if (g.values.size() != model.params.size())
    throw std::invalid_argument("apply_update: gradient dimension mismatch");
  throw_status(lbbsp_apply_update(model.params.data(), static_cast<int>(model.params.size()), g.values.data(),
                                  model.learning_rate));
  model.clock += 1;
  return model;
}

}  // namespace lbbsp
