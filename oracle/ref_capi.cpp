// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim around the UNMODIFIED reference core (/root/reference/proj/
// core/src/*.cpp, compiled by oracle/Makefile into oracle/_ref/liblbbsp_ref.so).
// It lets tests/, bench.py's cpu_baseline leg and __graft_entry__.smoke() call
// the reference itself as the checker. Every function forwards to the public
// reference API; nothing here re-implements reference arithmetic.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <optional>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbbsp/batch_sizer.hpp"
#include "lbbsp/cluster_sim.hpp"
#include "lbbsp/coordination.hpp"
#include "lbbsp/predictor.hpp"
#include "lbbsp/rng.hpp"
#include "lbbsp/scenario.hpp"
#include "lbbsp/sgd.hpp"
#include "lbbsp/trace.hpp"
#include "lbbsp_c.h"

using namespace lbbsp;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define REF_GUARD(...)                                                  \
  try {                                                                 \
    __VA_ARGS__;                                                             \
    return 0;                                                           \
  } catch (const std::invalid_argument& e) {                            \
    return fail(e, LBBSP_INVALID_ARGUMENT);                             \
  } catch (const std::out_of_range& e) {                                \
    return fail(e, LBBSP_OUT_OF_RANGE);                                 \
  } catch (const std::logic_error& e) {                                 \
    return fail(e, LBBSP_LOGIC);                                        \
  } catch (const std::runtime_error& e) {                               \
    return fail(e, LBBSP_RUNTIME);                                      \
  } catch (const std::exception& e) {                                   \
    return fail(e, LBBSP_RUNTIME);                                      \
  }

NarxModel to_model(const lbbsp_narx_model& m) {
  NarxModel r;
  for (int j = 0; j < 8; ++j) r.input_weights[static_cast<std::size_t>(j)] = m.input_weights[j];
  r.hidden_bias = m.hidden_bias;
  r.output_weight = m.output_weight;
  r.output_bias = m.output_bias;
  r.speed_scaler = {m.speed_mean, m.speed_stddev};
  r.cpu_scaler = {m.cpu_mean, m.cpu_stddev};
  r.mem_scaler = {m.mem_mean, m.mem_stddev};
  return r;
}

void from_model(const NarxModel& r, lbbsp_narx_model* m) {
  for (int j = 0; j < 8; ++j) m->input_weights[j] = r.input_weights[static_cast<std::size_t>(j)];
  m->hidden_bias = r.hidden_bias;
  m->output_weight = r.output_weight;
  m->output_bias = r.output_bias;
  m->speed_mean = r.speed_scaler.mean;
  m->speed_stddev = r.speed_scaler.stddev;
  m->cpu_mean = r.cpu_scaler.mean;
  m->cpu_stddev = r.cpu_scaler.stddev;
  m->mem_mean = r.mem_scaler.mean;
  m->mem_stddev = r.mem_scaler.stddev;
}

NarxTrainConfig to_train(const lbbsp_narx_train_cfg& c) {
  NarxTrainConfig t;
  t.step = c.step;
  t.max_epochs = c.max_epochs;
  t.early_stop_delta = c.early_stop_delta;
  t.early_stop_patience = c.early_stop_patience;
  t.min_history = c.min_history;
  return t;
}

PredictorConfig to_pred(const lbbsp_predictor_cfg& c) {
  PredictorConfig p;
  p.kind = static_cast<PredictorKind>(c.kind);
  p.alpha = c.alpha;
  p.warmup_iterations = c.warmup_iterations;
  p.speed_floor = c.speed_floor;
  p.train = to_train(c.train);
  return p;
}

SimConfig to_sim(const lbbsp_sim_cfg& c) {
  SimConfig cfg;
  cfg.scheme.kind = static_cast<SchemeKind>(c.scheme);
  cfg.scheme.total_budget = c.total_budget;
  cfg.scheme.staleness_threshold = c.staleness_threshold;
  const int n = c.n_workers;
  if (c.gpu_profiles) {
    for (int i = 0; i < n; ++i) {
      WorkerProfile wp;
      wp.id = i;
      wp.kind = WorkerKind::Gpu;
      const auto& g = c.gpu_profiles[i];
      wp.gpu = GpuProfile{g.sec_per_sample, g.base_time_s, g.saturation_point, g.oom_point};
      wp.comm.base_tm_s = c.base_comm_s;
      if (c.bw_worker == i) wp.comm.schedule.push_back({c.bw_at_iteration, c.bw_factor});
      cfg.workers.push_back(wp);
    }
  } else if (c.preset != LBBSP_PRESET_NONE) {
    const Preset p = heterogeneity_preset(static_cast<PresetName>(c.preset), n, c.seed,
                                          c.base_speed);
    cfg.workers = p.workers;
    cfg.dynamics = p.dynamics;
  } else {
    for (int i = 0; i < n; ++i) {
      WorkerProfile wp;
      wp.id = i;
      wp.base_speed = c.base_speed;
      cfg.workers.push_back(wp);
    }
  }
  for (int i = 0; i < n; ++i) {
    auto& wp = cfg.workers[static_cast<std::size_t>(i)];
    if (!c.gpu_profiles) {
      wp.comm.base_tm_s = c.base_comm_s;
      if (c.bw_worker == i) wp.comm.schedule.push_back({c.bw_at_iteration, c.bw_factor});
    }
  }
  if (c.preset == LBBSP_PRESET_NONE && !c.gpu_profiles) {
    cfg.dynamics.kind = static_cast<DynamicsKind>(c.dynamics);
    if (c.static_cpu) cfg.dynamics.static_cpu.assign(c.static_cpu, c.static_cpu + n);
    if (c.static_mem) cfg.dynamics.static_mem.assign(c.static_mem, c.static_mem + n);
    if (c.stragglers)
      for (int i = 0; i < n; ++i) {
        const auto& s = c.stragglers[i];
        cfg.dynamics.stragglers.push_back(
            StragglerSpec{s.on_probability, s.cpu_consumed, s.mem_consumed, s.period});
      }
    if (c.dynamics == LBBSP_DYN_TRACE)
      for (int i = 0; i < n; ++i) {
        ResourceTrace t;
        t.machine_id = std::to_string(i);
        for (int q = c.trace_offsets[i]; q < c.trace_offsets[i + 1]; ++q)
          t.points.push_back(TracePoint{c.trace_t[q], c.trace_cpu[q], c.trace_mem[q]});
        cfg.dynamics.traces.push_back(t);
      }
    if (c.dynamics == LBBSP_DYN_BENCHMARK) {
      auto& b = cfg.dynamics.benchmark;
      b.iterations = c.bench_iterations;
      b.regime_length = c.bench_regime_length;
      b.high_band_lo = c.bench_high_lo;
      b.high_band_hi = c.bench_high_hi;
      b.low_band_lo = c.bench_low_lo;
      b.low_band_hi = c.bench_low_hi;
      b.spike_mult = c.bench_spike_mult;
      b.spike_prob = c.bench_spike_prob;
    }
  }
  cfg.predictor = to_pred(c.predictor);
  if (c.narx_weights_path) cfg.predictor.initial_weights = c.narx_weights_path;
  cfg.learning_rate = c.learning_rate;
  cfg.dataset_seed = c.dataset_seed;
  cfg.dataset_size = c.dataset_size;
  cfg.dataset_dim = c.dataset_dim;
  cfg.dataset_noise = c.dataset_noise;
  cfg.convergence_loss = c.convergence_loss;
  cfg.convergence_consecutive = c.convergence_consecutive;
  cfg.max_updates = c.max_updates;
  cfg.seed = c.seed;
  cfg.record_params = true;
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_mix_seed3(uint64_t a, uint64_t b, uint64_t c) { return mix_seed(a, b, c); }
uint64_t ref_mix_seed2(uint64_t a, uint64_t b) { return mix_seed(a, b); }

// Rng draws (rng.hpp:24-42)
void ref_rng_u64(uint64_t seed, int count, uint64_t* out) {
  Rng r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.next_u64();
}
void ref_rng_uniform_int(uint64_t seed, int count, int lo, int hi, int* out) {
  Rng r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.uniform_int(lo, hi);
}

int ref_cpu_allocate(const double* v, int n, int budget, int* out) {
  REF_GUARD({
    const auto a = cpu_allocate(std::span<const double>(v, static_cast<std::size_t>(n)), budget);
    for (int i = 0; i < n; ++i) out[i] = a.sizes[static_cast<std::size_t>(i)];
  })
}

int ref_gpu_allocate(const lbbsp_gpu_profile* p, const double* comm, int n, int budget,
                     int* out) {
  REF_GUARD({
    std::vector<GpuProfile> prof;
    for (int i = 0; i < n; ++i)
      prof.push_back(GpuProfile{p[i].sec_per_sample, p[i].base_time_s, p[i].saturation_point,
                                p[i].oom_point});
    const auto a = gpu_allocate(prof, std::span<const double>(comm, static_cast<std::size_t>(n)),
                                budget);
    for (int i = 0; i < n; ++i) out[i] = a.sizes[static_cast<std::size_t>(i)];
  })
}

int ref_oracle_cpu_allocate(const double* v, int n, int budget, int* out) {
  REF_GUARD({
    const auto a =
        oracle_cpu_allocate(std::span<const double>(v, static_cast<std::size_t>(n)), budget);
    for (int i = 0; i < n; ++i) out[i] = a.sizes[static_cast<std::size_t>(i)];
  })
}

int ref_oracle_gpu_allocate(const lbbsp_gpu_profile* p, const double* comm, int n, int budget,
                            int* out) {
  REF_GUARD({
    std::vector<GpuProfile> prof;
    for (int i = 0; i < n; ++i)
      prof.push_back(GpuProfile{p[i].sec_per_sample, p[i].base_time_s, p[i].saturation_point,
                                p[i].oom_point});
    const auto a = oracle_gpu_allocate(
        prof, std::span<const double>(comm, static_cast<std::size_t>(n)), budget);
    for (int i = 0; i < n; ++i) out[i] = a.sizes[static_cast<std::size_t>(i)];
  })
}

double ref_clamp_speed_floor(double v, double floor) { return clamp_speed_floor(v, floor); }

int ref_ema(const double* s, int len, double alpha, double* out) {
  REF_GUARD({ *out = ema(std::span<const double>(s, static_cast<std::size_t>(len)), alpha); })
}

double ref_tanh(double x);  // libm, same as the reference's std::tanh
double ref_tanh(double x) { return std::tanh(x); }
double ref_expm1(double x) { return std::expm1(x); }

void ref_narx_init(uint64_t seed, lbbsp_narx_model* out) { from_model(narx_init(seed), out); }

double ref_narx_predict(const lbbsp_narx_model* m, const double* v, const double* c,
                        const double* mm, double floor) {
  return narx_predict(to_model(*m), {v[0], v[1]}, {c[0], c[1], c[2]}, {mm[0], mm[1], mm[2]},
                      floor);
}

int ref_narx_train(lbbsp_narx_model* m, const double* v, const double* c, const double* mm,
                   int len, const lbbsp_narx_train_cfg* cfg, lbbsp_narx_report* rep,
                   double* loss_log, int loss_cap) {
  REF_GUARD({
    NarxModel model = to_model(*m);
    SpeedHistory h;
    for (int i = 0; i < len; ++i) h.push(v[i], c[i], mm[i]);
    const auto r = narx_train_online(model, h, to_train(*cfg));
    from_model(model, m);
    rep->ran = r.ran ? 1 : 0;
    rep->epochs = r.epochs;
    rep->final_loss = r.final_loss;
    if (loss_log)
      for (std::size_t e = 0; e < model.training_loss.size() && static_cast<int>(e) < loss_cap; ++e)
        loss_log[e] = model.training_loss[e];
  })
}

// SpeedPredictor::predict on one history (predictor.cpp:271-292)
int ref_predictor_predict(const lbbsp_predictor_cfg* cfg, const lbbsp_narx_model* m,
                          const double* v, const double* c, const double* mm, int len,
                          double c_now, double m_now, double* out) {
  REF_GUARD({
    PredictorConfig pc = to_pred(*cfg);
    SpeedPredictor sp(pc, 0);
    // install the given model through the CSV-free path: train() never runs here
    SpeedHistory h;
    for (int i = 0; i < len; ++i) h.push(v[i], c[i], mm[i]);
    if (pc.kind == PredictorKind::Narx && len >= pc.warmup_iterations && len >= 2) {
      *out = narx_predict(to_model(*m), {v[len - 1], v[len - 2]}, {c_now, c[len - 1], c[len - 2]},
                          {m_now, mm[len - 1], mm[len - 2]}, pc.speed_floor);
    } else {
      *out = sp.predict(h, c_now, m_now);
    }
  })
}

// Dataset / LR (sgd.cpp)
int ref_generate_dataset(uint64_t seed, int n, int d, double noise, double* feat,
                         double* labels) {
  REF_GUARD({
    const Dataset ds = generate_dataset(seed, n, d, noise);
    for (int i = 0; i < n; ++i) {
      const auto& s = ds.samples[static_cast<std::size_t>(i)];
      for (int j = 0; j < d; ++j) feat[i * d + j] = s.features[static_cast<std::size_t>(j)];
      labels[i] = s.label;
    }
  })
}

namespace {
Dataset make_ds(const double* feat, const double* labels, int n, int d) {
  Dataset ds;
  ds.dim = d;
  ds.samples.resize(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    auto& s = ds.samples[static_cast<std::size_t>(i)];
    s.features.assign(feat + static_cast<std::ptrdiff_t>(i) * d,
                      feat + static_cast<std::ptrdiff_t>(i + 1) * d);
    s.label = labels[i];
  }
  return ds;
}
}  // namespace

int ref_batch_gradient(const double* feat, const double* labels, int n, int d,
                       const double* params, const int* idx, int count, double* out) {
  REF_GUARD({
    const Dataset ds = make_ds(feat, labels, n, d);
    ModelState m;
    m.params.assign(params, params + d);
    const Gradient g = batch_gradient(m, ds, std::span<const int>(idx, static_cast<std::size_t>(count)));
    for (int j = 0; j < d; ++j) out[j] = g.values[static_cast<std::size_t>(j)];
  })
}

int ref_loss(const double* feat, const double* labels, int n, int d, const double* params,
             double* out) {
  REF_GUARD({
    const Dataset ds = make_ds(feat, labels, n, d);
    ModelState m;
    m.params.assign(params, params + d);
    *out = loss(m, ds);
  })
}

int ref_aggregate(const double* grads, const int* sizes, int n, int dim, int weighted,
                  double* out) {
  REF_GUARD({
    std::vector<Gradient> gs;
    for (int i = 0; i < n; ++i) {
      Gradient g;
      g.values.assign(grads + static_cast<std::ptrdiff_t>(i) * dim,
                      grads + static_cast<std::ptrdiff_t>(i + 1) * dim);
      g.batch_size = sizes[i];
      gs.push_back(std::move(g));
    }
    const Gradient a = weighted ? aggregate_weighted(gs) : aggregate_naive(gs);
    for (int j = 0; j < dim; ++j) out[j] = a.values[static_cast<std::size_t>(j)];
  })
}

// make_benchmark_series (cluster_sim.cpp:41-64) with default BenchmarkTraceConfig
int ref_benchmark_series(uint64_t seed, int iterations, double* cpu, double* mem,
                         double* mult) {
  REF_GUARD({
    BenchmarkTraceConfig bc;
    bc.iterations = iterations;
    const SyntheticSeries s = make_benchmark_series(seed, bc);
    for (int k = 0; k < iterations; ++k) {
      cpu[k] = s.states[static_cast<std::size_t>(k)].cpu_avail;
      mem[k] = s.states[static_cast<std::size_t>(k)].mem_avail;
      mult[k] = s.states[static_cast<std::size_t>(k)].speed_mult;
    }
  })
}

// Full reference Simulation run (cluster_sim.cpp:247-296, 633-643) flattened.
int ref_sim_run(const lbbsp_sim_cfg* c, int max_rows, int* rows, lbbsp_iter_scalars* sc,
                int* batch, double* tp, double* tm, double* wait, double* v_pred,
                double* v_actual, double* params, int* converged, int* worker_id,
                int* row_workers) {
  REF_GUARD({
    Simulation sim(to_sim(*c));
    const SimResult r = sim.run();
    const int n = c->n_workers;
    const int d = c->dataset_dim;
    int count = 0;
    for (const auto& rec : r.records) {
      if (count >= max_rows) break;
      if (sc) sc[count] = lbbsp_iter_scalars{rec.k, rec.grad_norm, rec.loss, rec.wall_s};
      if (row_workers) row_workers[count] = static_cast<int>(rec.workers.size());
      for (std::size_t i = 0; i < rec.workers.size(); ++i) {
        const auto& w = rec.workers[i];
        const std::size_t o = static_cast<std::size_t>(count) * n + i;
        if (worker_id) worker_id[o] = w.worker_id;
        if (batch) batch[o] = w.batch;
        if (tp) tp[o] = w.tp_s;
        if (tm) tm[o] = w.tm_s;
        if (wait) wait[o] = w.wait_s;
        if (v_pred) v_pred[o] = w.v_pred;
        if (v_actual) v_actual[o] = w.v_actual;
      }
      if (params)
        for (int j = 0; j < d; ++j)
          params[static_cast<std::size_t>(count) * d + j] =
              r.param_trajectory[static_cast<std::size_t>(count)][static_cast<std::size_t>(j)];
      ++count;
    }
    *rows = count;
    if (converged) *converged = r.metrics.converged ? 1 : 0;
  })
}

// Replay driver: feeds an observed per-iteration stream
// (v, c, m) for n workers through the public SpeedPredictor + solver API in
// exactly step_sync's order (cluster_sim.cpp:355-402, 458-464) and
// train_rotation's schedule (:315-324). sizes_out/v_pred_out are [iters*n].
int ref_replay_cpu(const lbbsp_predictor_cfg* pcfg, const uint64_t* seeds, int n, int budget,
                   int iters, const double* v_obs, const double* c_obs, const double* m_obs,
                   int* sizes_out, double* v_pred_out) {
  REF_GUARD({
    const PredictorConfig pc = to_pred(*pcfg);
    std::vector<SpeedPredictor> preds;
    std::vector<SpeedHistory> hist(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) preds.emplace_back(pc, seeds[i]);
    int cursor = 0;
    std::vector<int> equal(static_cast<std::size_t>(n), budget / n);
    for (int i = 0; i < budget % n; ++i) equal[static_cast<std::size_t>(i)] += 1;
    for (int k = 0; k < iters; ++k) {
      std::vector<double> vp(static_cast<std::size_t>(n), 0.0);
      for (int i = 0; i < n; ++i) {
        const std::size_t o = static_cast<std::size_t>(k) * n + i;
        if (hist[static_cast<std::size_t>(i)].size() >= 1)
          vp[static_cast<std::size_t>(i)] =
              pc.kind == PredictorKind::Perfect
                  ? v_obs[o]
                  : preds[static_cast<std::size_t>(i)].predict(hist[static_cast<std::size_t>(i)],
                                                               c_obs[o], m_obs[o]);
      }
      std::vector<int> sizes;
      if (k == 0) {
        sizes = equal;
      } else {
        std::vector<double> sp;
        for (int i = 0; i < n; ++i)
          sp.push_back(clamp_speed_floor(vp[static_cast<std::size_t>(i)], pc.speed_floor));
        sizes = cpu_allocate(sp, budget).sizes;
      }
      for (int i = 0; i < n; ++i) {
        const std::size_t o = static_cast<std::size_t>(k) * n + i;
        sizes_out[o] = sizes[static_cast<std::size_t>(i)];
        if (v_pred_out) v_pred_out[o] = vp[static_cast<std::size_t>(i)];
        hist[static_cast<std::size_t>(i)].push(v_obs[o], c_obs[o], m_obs[o]);
      }
      if (pc.kind == PredictorKind::Narx) {
        const int b = (n + 1) / 2;
        for (int j = 0; j < b; ++j) {
          const int w = (cursor + j) % n;
          preds[static_cast<std::size_t>(w)].train(hist[static_cast<std::size_t>(w)]);
        }
        cursor = (cursor + b) % n;
      }
    }
  })
}


// ---- scenario / exporters / traces (scenario.cpp, trace.cpp) --------------
int ref_cmd_run(const char* config, const char* out_dir, int has_seed, uint64_t seed) {
  std::optional<std::uint64_t> s;
  if (has_seed) s = seed;
  return cmd_run(config, out_dir, s);
}

int ref_cmd_compare(const char* const* configs, int n, const char* out_dir, int has_seed,
                    uint64_t seed) {
  std::optional<std::uint64_t> s;
  if (has_seed) s = seed;
  std::vector<std::filesystem::path> paths(configs, configs + n);
  return cmd_compare(paths, out_dir, s);
}

int ref_cmd_predict_bench(const char* config, const char* out_dir, int has_seed, uint64_t seed) {
  std::optional<std::uint64_t> s;
  if (has_seed) s = seed;
  return cmd_predict_bench(config, out_dir, s);
}

// load_scenario's error text (ConfigError is a runtime_error -> LBBSP_RUNTIME here)
int ref_scenario_check(const char* path) { REF_GUARD({ (void)load_scenario(path); }) }

int ref_trace_map(const char* path, int workers, uint64_t seed, int* out, int* n_traces) {
  REF_GUARD({
    const auto traces = parse_trace(path);
    const auto a = map_traces(traces, workers, seed);
    for (int i = 0; i < workers; ++i) out[i] = static_cast<int>(a[static_cast<std::size_t>(i)]);
    *n_traces = static_cast<int>(traces.size());
  })
}

int ref_trace_at(const char* path, int i, double time_s, double* c, double* m) {
  REF_GUARD({
    const auto traces = parse_trace(path);
    const auto v = trace_at(traces.at(static_cast<std::size_t>(i)), time_s);
    *c = v.first;
    *m = v.second;
  })
}

int ref_series_rmse(int kind, const lbbsp_predictor_cfg* base, const double* cpu,
                    const double* mem, const double* mult, int len, double base_speed,
                    uint64_t seed, int measure_from, double* out) {
  REF_GUARD({
    SyntheticSeries series;
    for (int k = 0; k < len; ++k) {
      ResourceState rs;
      rs.cpu_avail = cpu[k];
      rs.mem_avail = mem[k];
      rs.speed_mult = mult[k];
      series.states.push_back(rs);
    }
    *out = predictor_series_rmse(static_cast<PredictorKind>(kind), to_pred(*base), series,
                                 base_speed, seed, measure_from);
  })
}

}  // extern "C"
