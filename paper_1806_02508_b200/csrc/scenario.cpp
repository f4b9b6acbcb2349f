// scenario.cpp -- host side of SURVEY 8(f): recorded resource traces, the
// scenario JSON loader, record/metric exporters and the CLI entry points.
//
// This is host glue around the device driver (lbbsp_sim_*): it parses and
// validates inputs once, hands the device a flat lbbsp_sim_cfg, and formats
// what the device recorded. Every function names the reference function it
// mirrors (paths relative to /root/reference/proj). Output files are
// byte-identical to the reference's (tests/test_scenario*.py).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <numeric>
#include <optional>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "lbbsp_c.h"

namespace lbbsp {
int set_error(int code, const char* fmt, ...);
}

namespace {

namespace fs = std::filesystem;
using nlohmann::json;
using lbbsp::set_error;

// rng.hpp:9-42 (mix_seed + Rng::uniform) on the host
uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
uint64_t mix_seed(uint64_t a, uint64_t b) { return mix64(a ^ mix64(b)); }
struct Rng {
  std::mt19937_64 g;
  explicit Rng(uint64_t s) : g(s) {}
  double uniform() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
};

// Exceptions carry the status code to the C-ABI edge.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& m) { throw Error(code, m); }
// ConfigError (scenario.hpp:13-15)
[[noreturn]] void config_error(const std::string& m) { throw Error(LBBSP_CONFIG, m); }

// Runs fn, mapping exceptions to a status + lbbsp_last_error().
template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return LBBSP_OK;
  } catch (const Error& e) {
    return set_error(e.code, "%s", e.what());
  } catch (const std::exception& e) {
    return set_error(LBBSP_RUNTIME, "%s", e.what());
  }
}
// Re-raises a failed C-ABI status as an exception carrying lbbsp_last_error().
void check(int rc) {
  if (rc != LBBSP_OK) fail(rc, lbbsp_last_error());
}

// ---------------------------------------------------------------------------
// Number formatting (scenario.cpp:60-72)
// ---------------------------------------------------------------------------
void format_real(std::string& out, double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.9g", v);
  out += buf;
}
double round9(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.9g", v);
  return std::strtod(buf, nullptr);
}

// ---------------------------------------------------------------------------
// Traces (trace.cpp)
// ---------------------------------------------------------------------------
struct TracePoint {
  double t, cpu, mem;
};
struct Trace {
  std::string machine_id;
  std::vector<TracePoint> points;
  // ResourceTrace::mean_cpu (trace.cpp:14-19): sequential sum
  double mean_cpu() const {
    if (points.empty()) return 0.0;
    double s = 0.0;
    for (const auto& p : points) s += p.cpu;
    return s / static_cast<double>(points.size());
  }
};

std::vector<std::string> split_csv(const std::string& line) {  // trace.cpp:23-30
  std::vector<std::string> out;
  size_t start = 0;
  while (start <= line.size()) {
    const size_t comma = line.find(',', start);
    if (comma == std::string::npos) {
      if (start < line.size()) out.push_back(line.substr(start));
      break;
    }
    out.push_back(line.substr(start, comma - start));
    start = comma + 1;
  }
  if (!line.empty() && line.back() == ',') out.emplace_back();
  return out;
}

double parse_real(const std::string& s, const char* what, int line_no) {  // :32-43
  bool ok = true;
  double v = 0.0;
  try {
    size_t used = 0;
    v = std::stod(s, &used);
    ok = used == s.size();
  } catch (const std::exception&) {
    ok = false;
  }
  if (!ok)
    fail(LBBSP_RUNTIME, "trace line " + std::to_string(line_no) + ": bad " + what + " '" + s + "'");
  return v;
}

double parse_fraction(const std::string& s, const char* what, int line_no) {  // :45-51
  const double v = parse_real(s, what, line_no);
  if (v < 0.0 || v > 1.0)
    fail(LBBSP_RUNTIME, "trace line " + std::to_string(line_no) + ": " + what + " " + s +
                            " outside [0,1]");
  return v;
}

std::vector<Trace> parse_trace(const std::string& path) {  // trace.cpp:54-97
  std::ifstream in(path);
  if (!in) fail(LBBSP_RUNTIME, "parse_trace: cannot open " + path);
  std::string header;
  if (!std::getline(in, header)) fail(LBBSP_RUNTIME, "parse_trace: empty file " + path);
  if (!header.empty() && header.back() == '\r') header.pop_back();
  const std::vector<std::string> cols = split_csv(header);
  const std::vector<std::string> want = {"machine_id", "t_offset_s", "cpu_avail", "mem_avail"};
  for (const auto& name : want)
    if (std::find(cols.begin(), cols.end(), name) == cols.end())
      fail(LBBSP_RUNTIME, "parse_trace: missing column '" + name + "'");
  if (cols != want)
    fail(LBBSP_RUNTIME,
         "parse_trace: unexpected column order, want machine_id,t_offset_s,cpu_avail,mem_avail");
  std::vector<Trace> traces;
  std::map<std::string, size_t> index;
  std::string line;
  int line_no = 1;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    const auto f = split_csv(line);
    if (f.size() != 4)
      fail(LBBSP_RUNTIME, "trace line " + std::to_string(line_no) + ": expected 4 fields, got " +
                              std::to_string(f.size()));
    TracePoint p;
    p.t = parse_real(f[1], "t_offset_s", line_no);
    p.cpu = parse_fraction(f[2], "cpu_avail", line_no);
    p.mem = parse_fraction(f[3], "mem_avail", line_no);
    auto it = index.find(f[0]);
    if (it == index.end()) {
      it = index.emplace(f[0], traces.size()).first;
      traces.push_back(Trace{f[0], {}});
    }
    Trace& t = traces[it->second];
    if (!t.points.empty() && p.t < t.points.back().t)
      fail(LBBSP_RUNTIME, "trace line " + std::to_string(line_no) +
                              ": time offsets not sorted for machine " + f[0]);
    t.points.push_back(p);
  }
  return traces;
}

// map_traces (trace.cpp:109-135): stratified by mean cpu, one seeded draw per worker.
std::vector<int> map_traces(const std::vector<Trace>& traces, int workers, uint64_t seed) {
  if (traces.empty()) fail(LBBSP_INVALID_ARGUMENT, "map_traces: no traces");
  if (workers < 1) fail(LBBSP_INVALID_ARGUMENT, "map_traces: workers must be >= 1");
  std::vector<double> mean(traces.size());
  for (size_t i = 0; i < traces.size(); ++i) mean[i] = traces[i].mean_cpu();
  std::vector<size_t> order(traces.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t a, size_t b) { return mean[a] < mean[b]; });
  Rng rng(mix_seed(seed, 0x7ace5ull));
  std::vector<int> out(static_cast<size_t>(workers));
  const double stride = static_cast<double>(traces.size()) / static_cast<double>(workers);
  for (int w = 0; w < workers; ++w) {
    const size_t lo = static_cast<size_t>(std::floor(stride * w));
    size_t hi = static_cast<size_t>(std::floor(stride * (w + 1)));
    if (hi <= lo) hi = lo + 1;
    if (hi > traces.size()) hi = traces.size();
    const size_t pick = lo + static_cast<size_t>(rng.uniform() * static_cast<double>(hi - lo));
    out[static_cast<size_t>(w)] = static_cast<int>(order[std::min(pick, traces.size() - 1)]);
  }
  return out;
}

// ---------------------------------------------------------------------------
// NARX weights CSV (predictor.cpp:198-243)
// ---------------------------------------------------------------------------
lbbsp_narx_model load_narx_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(LBBSP_RUNTIME, "load_narx_csv: cannot open " + path);
  std::map<std::string, double> values;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    const auto comma = line.find(',');
    if (comma == std::string::npos) fail(LBBSP_RUNTIME, "load_narx_csv: malformed row '" + line + "'");
    values[line.substr(0, comma)] = std::stod(line.substr(comma + 1));
  }
  auto get = [&](const std::string& name) {
    const auto it = values.find(name);
    if (it == values.end()) fail(LBBSP_RUNTIME, "load_narx_csv: missing parameter '" + name + "'");
    return it->second;
  };
  lbbsp_narx_model m{};
  for (int j = 0; j < 8; ++j) m.input_weights[j] = get("input_weight_" + std::to_string(j));
  m.hidden_bias = get("hidden_bias");
  m.output_weight = get("output_weight");
  m.output_bias = get("output_bias");
  m.speed_mean = get("speed_mean");
  m.speed_stddev = get("speed_stddev");
  m.cpu_mean = get("cpu_mean");
  m.cpu_stddev = get("cpu_stddev");
  m.mem_mean = get("mem_mean");
  m.mem_stddev = get("mem_stddev");
  return m;
}

// ---------------------------------------------------------------------------
// Scenario (scenario.cpp:31-294)
// ---------------------------------------------------------------------------
const std::set<std::string> kKnownKeys = {
    "scheme", "staleness_threshold", "workers", "total_budget", "preset", "trace_path",
    "gpu_profiles", "bandwidth_drop", "base_speed", "base_comm_s", "predictor", "alpha",
    "warmup_iterations", "speed_floor", "narx_weights_path", "learning_rate",
    "dataset_seed", "dataset_size", "dataset_dim", "dataset_noise", "convergence_loss",
    "convergence_consecutive", "max_iterations", "seed", "benchmark_iterations",
    "benchmark_regime_length", "benchmark_spike_mult", "benchmark_spike_prob",
    "benchmark_high_band", "benchmark_low_band", "paired_sim"};

template <typename T>
T require(const json& j, const std::string& key) {
  if (!j.contains(key)) config_error("config: missing field '" + key + "'");
  try {
    return j.at(key).get<T>();
  } catch (const json::exception&) {
    config_error("config: bad value for field '" + key + "'");
  }
}

template <typename T>
T get_or(const json& j, const std::string& key, T fallback) {
  if (!j.contains(key)) return fallback;
  try {
    return j.at(key).get<T>();
  } catch (const json::exception&) {
    config_error("config: bad value for field '" + key + "'");
  }
}

int scheme_from_string(const std::string& s) {  // coordination.cpp:19-25
  if (s == "bsp") return LBBSP_SCHEME_BSP;
  if (s == "asp") return LBBSP_SCHEME_ASP;
  if (s == "ssp") return LBBSP_SCHEME_SSP;
  if (s == "lb-bsp" || s == "lbbsp") return LBBSP_SCHEME_LBBSP;
  throw std::invalid_argument("unknown scheme: " + s);
}
const char* scheme_name(int k) {  // coordination.cpp:9-17
  switch (k) {
    case LBBSP_SCHEME_BSP: return "bsp";
    case LBBSP_SCHEME_ASP: return "asp";
    case LBBSP_SCHEME_SSP: return "ssp";
    case LBBSP_SCHEME_LBBSP: return "lb-bsp";
  }
  return "?";
}
int predictor_from_string(const std::string& s) {  // predictor.cpp:255-261
  if (s == "memoryless") return LBBSP_PRED_MEMORYLESS;
  if (s == "ema") return LBBSP_PRED_EMA;
  if (s == "narx") return LBBSP_PRED_NARX;
  if (s == "perfect") return LBBSP_PRED_PERFECT;
  throw std::invalid_argument("unknown predictor: " + s);
}
const char* predictor_name(int k) {  // predictor.cpp:245-253
  switch (k) {
    case LBBSP_PRED_MEMORYLESS: return "memoryless";
    case LBBSP_PRED_EMA: return "ema";
    case LBBSP_PRED_NARX: return "narx";
    case LBBSP_PRED_PERFECT: return "perfect";
  }
  return "?";
}
int preset_from_string(const std::string& s) {  // cluster_sim.cpp:131-138
  if (s == "homo") return LBBSP_PRESET_HOMO;
  if (s == "hetero-l2") return LBBSP_PRESET_HETERO_L2;
  if (s == "hetero-l3") return LBBSP_PRESET_HETERO_L3;
  if (s == "hetero-l2-static") return LBBSP_PRESET_HETERO_L2_STATIC;
  if (s == "hetero-l3-static") return LBBSP_PRESET_HETERO_L3_STATIC;
  throw std::invalid_argument("unknown preset: " + s);
}

struct GpuGroup {
  lbbsp_gpu_profile profile;
  int count;
};
struct BandwidthDrop {
  int worker;
  int64_t at_iteration;
  double comm_factor;
};
struct Bench {  // BenchmarkTraceConfig defaults (cluster_sim.hpp:76-83)
  int iterations = 1200, regime_length = 50;
  double high_lo = 0.75, high_hi = 1.0, low_lo = 0.30, low_hi = 0.55;
  double spike_mult = 3.0, spike_prob = 0.02;
};

struct Scenario {  // ScenarioConfig (scenario.hpp:33-64)
  std::string name;
  int scheme = LBBSP_SCHEME_BSP;
  int staleness_threshold = 0;
  int workers = 0;
  int total_budget = 0;
  std::string preset = "homo";
  std::string trace_path;
  std::vector<GpuGroup> gpu_profiles;
  std::optional<BandwidthDrop> bandwidth_drop;
  double base_speed = 10.0;
  double base_comm_s = 0.0;
  int predictor = LBBSP_PRED_EMA;
  double alpha = 0.2;
  int warmup_iterations = 500;
  double speed_floor = 1e-3;
  std::string narx_weights_path;
  double learning_rate = 0.5;
  uint64_t dataset_seed = 7;
  int dataset_size = 1000;
  int dataset_dim = 10;
  double dataset_noise = 0.1;
  double convergence_loss = 0.40;
  int convergence_consecutive = 10;
  int64_t max_iterations = 500;
  uint64_t seed = 1;
  Bench benchmark;
  bool paired_sim = true;
};

void validate_scenario(const Scenario& c) {  // scenario.cpp:183-217
  if (c.workers < 1) config_error("config: field 'workers' must be >= 1");
  if (c.total_budget < c.workers) config_error("config: field 'total_budget' must be >= workers");
  if (c.staleness_threshold < 0) config_error("config: field 'staleness_threshold' must be >= 0");
  if (!(c.alpha > 0.0 && c.alpha <= 1.0)) config_error("config: field 'alpha' must be in (0, 1]");
  if (c.learning_rate <= 0.0) config_error("config: field 'learning_rate' must be > 0");
  if (c.dataset_size < 1) config_error("config: field 'dataset_size' must be >= 1");
  if (c.dataset_dim < 1) config_error("config: field 'dataset_dim' must be >= 1");
  if (c.convergence_loss <= 0.0) config_error("config: field 'convergence_loss' must be > 0");
  if (c.convergence_consecutive < 1)
    config_error("config: field 'convergence_consecutive' must be >= 1");
  if (c.max_iterations < 1) config_error("config: field 'max_iterations' must be >= 1");
  if (!c.trace_path.empty() && !fs::exists(c.trace_path))
    config_error("config: trace file not found: " + c.trace_path);
  if (!c.narx_weights_path.empty() && !fs::exists(c.narx_weights_path))
    config_error("config: narx weights file not found: " + c.narx_weights_path);
  if (!c.gpu_profiles.empty()) {
    int total = 0;
    for (const auto& g : c.gpu_profiles) total += g.count;
    if (total != c.workers)
      config_error("config: gpu_profiles counts sum to " + std::to_string(total) +
                   ", field 'workers' says " + std::to_string(c.workers));
    if (!c.trace_path.empty()) config_error("config: gpu_profiles and trace_path cannot be combined");
  }
  if (c.bandwidth_drop &&
      (c.bandwidth_drop->worker < 0 || c.bandwidth_drop->worker >= c.workers))
    config_error("config: bandwidth_drop worker out of range");
}

Scenario load_scenario(const std::string& path_str) {  // scenario.cpp:92-181
  const fs::path path(path_str);
  std::ifstream in(path);
  if (!in) config_error("config: cannot open " + path.string());
  json j;
  try {
    in >> j;
  } catch (const json::exception& e) {
    config_error("config: invalid JSON in " + path.string() + ": " + e.what());
  }
  if (!j.is_object()) config_error("config: top level must be a JSON object");
  for (const auto& [key, value] : j.items())
    if (!kKnownKeys.count(key)) config_error("config: unknown field '" + key + "'");
  Scenario c;
  c.name = path.stem().string();
  try {
    c.scheme = scheme_from_string(require<std::string>(j, "scheme"));
  } catch (const std::invalid_argument& e) {
    config_error(std::string("config: field 'scheme': ") + e.what());
  }
  c.workers = require<int>(j, "workers");
  c.staleness_threshold = get_or(j, "staleness_threshold", 0);
  c.total_budget = get_or(j, "total_budget", 128 * c.workers);
  c.preset = get_or<std::string>(j, "preset", "homo");
  c.trace_path = get_or<std::string>(j, "trace_path", "");
  c.base_speed = get_or(j, "base_speed", 10.0);
  c.base_comm_s = get_or(j, "base_comm_s", 0.0);
  try {
    c.predictor = predictor_from_string(get_or<std::string>(j, "predictor", "ema"));
  } catch (const std::invalid_argument& e) {
    config_error(std::string("config: field 'predictor': ") + e.what());
  }
  c.alpha = get_or(j, "alpha", 0.2);
  c.warmup_iterations = get_or(j, "warmup_iterations", 500);
  c.speed_floor = get_or(j, "speed_floor", 1e-3);
  c.narx_weights_path = get_or<std::string>(j, "narx_weights_path", "");
  c.learning_rate = get_or(j, "learning_rate", 0.5);
  c.dataset_seed = get_or<uint64_t>(j, "dataset_seed", 7);
  c.dataset_size = get_or(j, "dataset_size", 1000);
  c.dataset_dim = get_or(j, "dataset_dim", 10);
  c.dataset_noise = get_or(j, "dataset_noise", 0.1);
  c.convergence_loss = get_or(j, "convergence_loss", 0.40);
  c.convergence_consecutive = get_or(j, "convergence_consecutive", 10);
  c.max_iterations = get_or<int64_t>(j, "max_iterations", 500);
  c.seed = get_or<uint64_t>(j, "seed", 1);
  c.paired_sim = get_or(j, "paired_sim", true);
  c.benchmark.iterations = get_or(j, "benchmark_iterations", c.benchmark.iterations);
  c.benchmark.regime_length = get_or(j, "benchmark_regime_length", c.benchmark.regime_length);
  c.benchmark.spike_mult = get_or(j, "benchmark_spike_mult", c.benchmark.spike_mult);
  c.benchmark.spike_prob = get_or(j, "benchmark_spike_prob", c.benchmark.spike_prob);
  if (j.contains("benchmark_high_band")) {
    const auto band = require<std::vector<double>>(j, "benchmark_high_band");
    if (band.size() != 2) config_error("config: field 'benchmark_high_band' needs [lo, hi]");
    c.benchmark.high_lo = band[0];
    c.benchmark.high_hi = band[1];
  }
  if (j.contains("benchmark_low_band")) {
    const auto band = require<std::vector<double>>(j, "benchmark_low_band");
    if (band.size() != 2) config_error("config: field 'benchmark_low_band' needs [lo, hi]");
    c.benchmark.low_lo = band[0];
    c.benchmark.low_hi = band[1];
  }
  if (j.contains("gpu_profiles")) {
    const json& groups = j.at("gpu_profiles");
    if (!groups.is_array()) config_error("config: field 'gpu_profiles' must be an array");
    for (const json& g : groups) {
      GpuGroup grp{};
      grp.profile.sec_per_sample = require<double>(g, "sec_per_sample");
      grp.profile.base_time_s = require<double>(g, "base_time_s");
      grp.profile.saturation_point = require<int>(g, "saturation_point");
      grp.profile.oom_point = require<int>(g, "oom_point");
      grp.count = get_or(g, "count", 1);
      c.gpu_profiles.push_back(grp);
    }
  }
  if (j.contains("bandwidth_drop")) {
    const json& d = j.at("bandwidth_drop");
    BandwidthDrop drop{};
    drop.worker = require<int>(d, "worker");
    drop.at_iteration = require<int64_t>(d, "at_iteration");
    drop.comm_factor = require<double>(d, "comm_factor");
    c.bandwidth_drop = drop;
  }
  validate_scenario(c);
  return c;
}

// A resolved simulation config plus the arrays it points into.
struct BuiltSim {
  lbbsp_sim_cfg cfg{};
  std::vector<lbbsp_gpu_profile> profiles;
  std::vector<int> trace_offsets;
  std::vector<double> trace_t, trace_cpu, trace_mem;
  std::string narx_path;
};

lbbsp_narx_train_cfg default_train_cfg(int min_history) {  // NarxTrainConfig (predictor.hpp:69-75)
  return lbbsp_narx_train_cfg{0.05, 500, 1e-4, 4, min_history};
}

// build_sim_config (scenario.cpp:219-294)
void build_sim_config(const Scenario& c, BuiltSim& b) {
  lbbsp_sim_cfg& s = b.cfg;
  s = lbbsp_sim_cfg{};
  s.scheme = c.scheme;
  s.staleness_threshold = c.staleness_threshold;
  s.n_workers = c.workers;
  s.total_budget = c.total_budget;
  s.preset = LBBSP_PRESET_NONE;
  s.base_speed = c.base_speed;
  s.dynamics = LBBSP_DYN_STATIC;
  s.bench_iterations = c.benchmark.iterations;
  s.bench_regime_length = c.benchmark.regime_length;
  s.bench_high_lo = c.benchmark.high_lo;
  s.bench_high_hi = c.benchmark.high_hi;
  s.bench_low_lo = c.benchmark.low_lo;
  s.bench_low_hi = c.benchmark.low_hi;
  s.bench_spike_mult = c.benchmark.spike_mult;
  s.bench_spike_prob = c.benchmark.spike_prob;
  s.predictor.kind = c.predictor;
  s.predictor.alpha = c.alpha;
  s.predictor.warmup_iterations = c.warmup_iterations;
  s.predictor.speed_floor = c.speed_floor;
  s.predictor.train = default_train_cfg(c.warmup_iterations);
  b.narx_path = c.narx_weights_path;
  s.narx_weights_path = b.narx_path.empty() ? nullptr : b.narx_path.c_str();
  s.learning_rate = c.learning_rate;
  s.dataset_seed = c.dataset_seed;
  s.dataset_size = c.dataset_size;
  s.dataset_dim = c.dataset_dim;
  s.dataset_noise = c.dataset_noise;
  s.convergence_loss = c.convergence_loss;
  s.convergence_consecutive = c.convergence_consecutive;
  s.max_updates = c.max_iterations;
  s.seed = c.seed;
  s.base_comm_s = c.base_comm_s;
  s.bw_worker = -1;
  b.profiles.clear();
  b.trace_offsets.clear();
  b.trace_t.clear();
  b.trace_cpu.clear();
  b.trace_mem.clear();
  if (!c.gpu_profiles.empty()) {
    for (const auto& g : c.gpu_profiles)
      for (int i = 0; i < g.count; ++i) b.profiles.push_back(g.profile);
    s.gpu_profiles = b.profiles.data();
  } else if (!c.trace_path.empty()) {
    const std::vector<Trace> traces = parse_trace(c.trace_path);
    const std::vector<int> mapping = map_traces(traces, c.workers, c.seed);
    s.dynamics = LBBSP_DYN_TRACE;
    b.trace_offsets.push_back(0);
    for (int w = 0; w < c.workers; ++w) {
      const Trace& t = traces[static_cast<size_t>(mapping[static_cast<size_t>(w)])];
      if (t.points.empty()) fail(LBBSP_INVALID_ARGUMENT, "trace_at: empty trace");
      for (const auto& p : t.points) {
        b.trace_t.push_back(p.t);
        b.trace_cpu.push_back(p.cpu);
        b.trace_mem.push_back(p.mem);
      }
      b.trace_offsets.push_back(static_cast<int>(b.trace_t.size()));
    }
    s.trace_offsets = b.trace_offsets.data();
    s.trace_t = b.trace_t.data();
    s.trace_cpu = b.trace_cpu.data();
    s.trace_mem = b.trace_mem.data();
  } else if (c.preset == "benchmark") {
    s.dynamics = LBBSP_DYN_BENCHMARK;
  } else {
    try {
      s.preset = preset_from_string(c.preset);
    } catch (const std::invalid_argument& e) {
      config_error(std::string("config: field 'preset': ") + e.what());
    }
  }
  if (c.bandwidth_drop) {
    s.bw_worker = c.bandwidth_drop->worker;
    s.bw_at_iteration = c.bandwidth_drop->at_iteration;
    s.bw_factor = c.bandwidth_drop->comm_factor;
  }
}

// ---------------------------------------------------------------------------
// Records and metrics
// ---------------------------------------------------------------------------
struct Records {  // a host copy of a device record stream
  int rows = 0, n = 0;
  std::vector<lbbsp_iter_scalars> sc;
  std::vector<int> batch, worker_id, row_workers;
  std::vector<double> tp, tm, wait, v_pred, v_actual;
  lbbsp_records_view view() const {
    return lbbsp_records_view{rows,          n,           sc.data(),        batch.data(),
                              tp.data(),     tm.data(),   wait.data(),      v_pred.data(),
                              v_actual.data(), worker_id.data(), row_workers.data()};
  }
};

int row_stats(const lbbsp_records_view& r, int i) { return r.row_workers ? r.row_workers[i] : r.n; }
int slot_worker(const lbbsp_records_view& r, size_t o, int w) { return r.worker_id ? r.worker_id[o] : w; }

// compute_metrics (cluster_sim.cpp:217-245) -- sequential folds in record order.
lbbsp_metrics compute_metrics(const lbbsp_records_view& r, bool converged, int rmse_from,
                              bool rounded) {
  auto rd = [&](double v) { return rounded ? round9(v) : v; };
  lbbsp_metrics m{};
  m.converged = converged ? 1 : 0;
  m.updates_to_convergence = r.rows;
  if (r.rows == 0) return m;
  double time_total = 0.0, wait_fraction_sum = 0.0, sse = 0.0;
  int64_t row_count = 0, sse_count = 0;
  for (int i = 0; i < r.rows; ++i) {
    const double wall = rd(r.scalars[i].wall_s);
    time_total += wall;
    for (int w = 0; w < row_stats(r, i); ++w) {
      const size_t o = static_cast<size_t>(i) * r.n + w;
      wait_fraction_sum += wall > 0.0 ? rd(r.wait[o]) / wall : 0.0;
      ++row_count;
      const double vp = rd(r.v_pred[o]);
      if (vp > 0.0 && r.scalars[i].k >= rmse_from) {
        const double e = vp - rd(r.v_actual[o]);
        sse += e * e;
        ++sse_count;
      }
    }
  }
  m.mean_per_update_time = time_total / static_cast<double>(r.rows);
  m.wastage = row_count > 0 ? wait_fraction_sum / static_cast<double>(row_count) : 0.0;
  m.predictor_rmse = sse_count > 0 ? std::sqrt(sse / static_cast<double>(sse_count)) : 0.0;
  return m;
}

// write_records_csv (scenario.cpp:306-342). %.9g of a value and of its
// round9() image are the same string, so the raw records can be written.
void write_records_csv(const lbbsp_records_view& r, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(LBBSP_RUNTIME, "cannot open " + path);
  std::string buf;
  buf.reserve(1 << 16);
  buf += "k,worker_id,x,tp_s,tm_s,wait_s,v_pred,v_actual,loss,iter_wall_s\n";
  for (int i = 0; i < r.rows; ++i) {
    for (int w = 0; w < row_stats(r, i); ++w) {
      const size_t o = static_cast<size_t>(i) * r.n + w;
      buf += std::to_string(r.scalars[i].k);
      buf += ',';
      buf += std::to_string(slot_worker(r, o, w));
      buf += ',';
      buf += std::to_string(r.batch[o]);
      for (const double v : {r.tp[o], r.tm[o], r.wait[o], r.v_pred[o], r.v_actual[o],
                             r.scalars[i].loss, r.scalars[i].wall_s}) {
        buf += ',';
        format_real(buf, v);
      }
      buf += '\n';
      if (buf.size() > (1 << 15)) {
        out << buf;
        buf.clear();
      }
    }
  }
  out << buf;
}

void write_metrics_json(const lbbsp_metrics& m, double conv_loss, int conv_consec, int warmup,
                        const std::string& path) {  // scenario.cpp:344-358
  json j;
  j["updates_to_convergence"] = static_cast<std::int64_t>(m.updates_to_convergence);
  j["mean_per_update_time"] = m.mean_per_update_time;
  j["wastage"] = m.wastage;
  j["predictor_rmse"] = m.predictor_rmse;
  j["converged"] = m.converged != 0;
  j["convergence_loss"] = conv_loss;
  j["convergence_consecutive"] = conv_consec;
  j["warmup_iterations"] = warmup;
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(LBBSP_RUNTIME, "cannot open " + path);
  out << j.dump(2) << "\n";
}

// ---------------------------------------------------------------------------
// Running a scenario on the device driver (run_scenario, scenario.cpp:296-304)
// ---------------------------------------------------------------------------
struct SimRun {
  Records rec;
  bool converged = false;
  lbbsp_metrics metrics{};  // Simulation::run's metrics, computed on device
};

struct SimHandle {
  lbbsp_sim* p = nullptr;
  ~SimHandle() {
    if (p) lbbsp_sim_destroy(p);
  }
};

SimRun run_sim(const lbbsp_sim_cfg& cfg) {
  SimHandle h;
  check(lbbsp_sim_create(&cfg, &h.p));
  check(lbbsp_sim_run(h.p, static_cast<int>(cfg.max_updates), nullptr));
  SimRun out;
  Records& r = out.rec;
  const size_t cap = static_cast<size_t>(cfg.max_updates), n = static_cast<size_t>(cfg.n_workers);
  r.n = cfg.n_workers;
  r.sc.resize(cap);
  r.batch.resize(cap * n);
  for (auto* v : {&r.tp, &r.tm, &r.wait, &r.v_pred, &r.v_actual}) v->resize(cap * n);
  r.worker_id.resize(cap * n);
  r.row_workers.resize(cap);
  int done = 0, conv = 0;
  check(lbbsp_sim_status(h.p, &done, &conv));
  check(lbbsp_sim_records(h.p, static_cast<int>(cap), &r.rows, r.sc.data(), r.batch.data(),
                          r.tp.data(), r.tm.data(), r.wait.data(), r.v_pred.data(),
                          r.v_actual.data(), nullptr));
  check(lbbsp_sim_record_workers(h.p, static_cast<int>(cap), r.worker_id.data(), r.row_workers.data()));
  out.converged = conv != 0;
  check(lbbsp_sim_metrics(h.p, cfg.predictor.warmup_iterations, &out.metrics));
  return out;
}

bool log_enabled() {  // scenario.cpp:18-23
  const char* v = std::getenv("LBBSP_LOG");
  if (!v) return false;
  const std::string s(v);
  return !s.empty() && s != "0" && s != "off";
}

SimRun run_scenario(const Scenario& c) {
  BuiltSim b;
  build_sim_config(c, b);
  SimRun r = run_sim(b.cfg);
  if (log_enabled())
    std::cerr << "[lbbsp] run '" << c.name << "' scheme=" << scheme_name(c.scheme)
              << " updates=" << std::to_string(r.metrics.updates_to_convergence)
              << " per_update=" << std::to_string(r.metrics.mean_per_update_time)
              << (r.metrics.converged ? " converged" : " capped") << "\n";
  return r;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
struct lbbsp_traces {
  std::vector<Trace> traces;
};

struct lbbsp_scenario {
  Scenario cfg;
  BuiltSim built;
  bool built_ok = false;
};

extern "C" int lbbsp_compute_metrics(const lbbsp_records_view* rec, int converged,
                                     int rmse_from_iteration, int round9_flag, lbbsp_metrics* out) {
  return guarded([&] {
    if (!rec || !out) fail(LBBSP_INVALID_ARGUMENT, "compute_metrics: null argument");
    *out = compute_metrics(*rec, converged != 0, rmse_from_iteration, round9_flag != 0);
  });
}

extern "C" int lbbsp_write_records_csv(const lbbsp_records_view* rec, const char* path) {
  return guarded([&] { write_records_csv(*rec, path); });
}

extern "C" int lbbsp_write_metrics_json(const lbbsp_metrics* m, double convergence_loss,
                                        int convergence_consecutive, int warmup_iterations,
                                        const char* path) {
  return guarded([&] {
    write_metrics_json(*m, convergence_loss, convergence_consecutive, warmup_iterations, path);
  });
}

extern "C" int lbbsp_trace_parse(const char* path, lbbsp_traces** out) {
  return guarded([&] {
    auto t = std::make_unique<lbbsp_traces>();
    t->traces = parse_trace(path);
    *out = t.release();
  });
}

extern "C" int lbbsp_trace_create(int n_traces, const char* const* ids, const int* offsets,
                                  const double* t, const double* cpu, const double* mem,
                                  lbbsp_traces** out) {
  return guarded([&] {
    if (n_traces < 0) fail(LBBSP_INVALID_ARGUMENT, "trace_create: n_traces must be >= 0");
    auto tr = std::make_unique<lbbsp_traces>();
    for (int i = 0; i < n_traces; ++i) {
      Trace x;
      x.machine_id = ids ? ids[i] : std::to_string(i);
      for (int p = offsets[i]; p < offsets[i + 1]; ++p) x.points.push_back({t[p], cpu[p], mem[p]});
      tr->traces.push_back(std::move(x));
    }
    *out = tr.release();
  });
}

extern "C" int lbbsp_trace_destroy(lbbsp_traces* tr) {
  delete tr;
  return LBBSP_OK;
}

extern "C" int lbbsp_trace_count(const lbbsp_traces* tr, int* n) {
  *n = static_cast<int>(tr->traces.size());
  return LBBSP_OK;
}

static int trace_index_ok(const lbbsp_traces* tr, int i) {
  if (i < 0 || i >= static_cast<int>(tr->traces.size()))
    return set_error(LBBSP_OUT_OF_RANGE, "trace index %d out of range", i);
  return LBBSP_OK;
}

extern "C" int lbbsp_trace_info(const lbbsp_traces* tr, int i, const char** machine_id,
                                int* points, double* mean_cpu) {
  if (int rc = trace_index_ok(tr, i)) return rc;
  const Trace& t = tr->traces[static_cast<size_t>(i)];
  if (machine_id) *machine_id = t.machine_id.c_str();
  if (points) *points = static_cast<int>(t.points.size());
  if (mean_cpu) *mean_cpu = t.mean_cpu();
  return LBBSP_OK;
}

extern "C" int lbbsp_trace_points(const lbbsp_traces* tr, int i, double* t, double* cpu,
                                  double* mem) {
  if (int rc = trace_index_ok(tr, i)) return rc;
  const Trace& x = tr->traces[static_cast<size_t>(i)];
  for (size_t p = 0; p < x.points.size(); ++p) {
    if (t) t[p] = x.points[p].t;
    if (cpu) cpu[p] = x.points[p].cpu;
    if (mem) mem[p] = x.points[p].mem;
  }
  return LBBSP_OK;
}

extern "C" int lbbsp_trace_write(const lbbsp_traces* tr, const char* path) {  // trace.cpp:99-107
  return guarded([&] {
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(LBBSP_RUNTIME, std::string("write_trace: cannot open ") + path);
    out.precision(17);
    out << "machine_id,t_offset_s,cpu_avail,mem_avail\n";
    for (const auto& t : tr->traces)
      for (const auto& p : t.points)
        out << t.machine_id << "," << p.t << "," << p.cpu << "," << p.mem << "\n";
  });
}

extern "C" int lbbsp_trace_map(const lbbsp_traces* tr, int workers, uint64_t seed,
                               int* assignment) {
  return guarded([&] {
    const std::vector<int> a = map_traces(tr->traces, workers, seed);
    std::copy(a.begin(), a.end(), assignment);
  });
}

extern "C" int lbbsp_trace_at(const lbbsp_traces* tr, int i, double time_s, double* cpu,
                              double* mem) {  // trace.cpp:137-143
  if (int rc = trace_index_ok(tr, i)) return rc;
  const auto& pts = tr->traces[static_cast<size_t>(i)].points;
  if (pts.empty()) return set_error(LBBSP_INVALID_ARGUMENT, "trace_at: empty trace");
  auto it = std::upper_bound(pts.begin(), pts.end(), time_s,
                             [](double t, const TracePoint& p) { return t < p.t; });
  if (it != pts.begin()) --it;
  *cpu = it->cpu;
  *mem = it->mem;
  return LBBSP_OK;
}

extern "C" int lbbsp_narx_load_csv(const char* path, lbbsp_narx_model* out) {
  return guarded([&] { *out = load_narx_csv(path); });
}

extern "C" int lbbsp_narx_save_csv(const lbbsp_narx_model* m, const char* path) {
  return guarded([&] {  // predictor.cpp:198-213
    std::ofstream out(path);
    if (!out) fail(LBBSP_RUNTIME, std::string("save_narx_csv: cannot open ") + path);
    out.precision(17);
    for (int j = 0; j < 8; ++j) out << "input_weight_" << j << "," << m->input_weights[j] << "\n";
    out << "hidden_bias," << m->hidden_bias << "\n";
    out << "output_weight," << m->output_weight << "\n";
    out << "output_bias," << m->output_bias << "\n";
    out << "speed_mean," << m->speed_mean << "\n";
    out << "speed_stddev," << m->speed_stddev << "\n";
    out << "cpu_mean," << m->cpu_mean << "\n";
    out << "cpu_stddev," << m->cpu_stddev << "\n";
    out << "mem_mean," << m->mem_mean << "\n";
    out << "mem_stddev," << m->mem_stddev << "\n";
  });
}

extern "C" int lbbsp_scenario_load(const char* path, lbbsp_scenario** out) {
  return guarded([&] {
    auto s = std::make_unique<lbbsp_scenario>();
    s->cfg = load_scenario(path);
    *out = s.release();
  });
}

extern "C" int lbbsp_scenario_destroy(lbbsp_scenario* s) {
  delete s;
  return LBBSP_OK;
}

extern "C" int lbbsp_scenario_set_seed(lbbsp_scenario* s, uint64_t seed) {
  s->cfg.seed = seed;
  s->built_ok = false;
  return LBBSP_OK;
}

extern "C" int lbbsp_scenario_get_info(const lbbsp_scenario* s, lbbsp_scenario_info* info) {
  const Scenario& c = s->cfg;
  *info = lbbsp_scenario_info{};
  std::snprintf(info->name, sizeof info->name, "%s", c.name.c_str());
  info->scheme = c.scheme;
  info->staleness_threshold = c.staleness_threshold;
  info->workers = c.workers;
  info->total_budget = c.total_budget;
  info->predictor = c.predictor;
  info->alpha = c.alpha;
  info->warmup_iterations = c.warmup_iterations;
  info->speed_floor = c.speed_floor;
  info->base_speed = c.base_speed;
  info->base_comm_s = c.base_comm_s;
  info->learning_rate = c.learning_rate;
  info->convergence_loss = c.convergence_loss;
  info->convergence_consecutive = c.convergence_consecutive;
  info->max_iterations = c.max_iterations;
  info->seed = c.seed;
  info->paired_sim = c.paired_sim ? 1 : 0;
  return LBBSP_OK;
}

extern "C" int lbbsp_scenario_sim_cfg(lbbsp_scenario* s, const lbbsp_sim_cfg** cfg) {
  return guarded([&] {
    if (!s->built_ok) {
      build_sim_config(s->cfg, s->built);
      s->built_ok = true;
    }
    *cfg = &s->built.cfg;
  });
}

// cmd_run / cmd_compare / cmd_predict_bench (scenario.cpp:369-481)
template <class F>
static int cli(const char* prefix, F&& fn) {
  const int rc = guarded(fn);
  if (rc == LBBSP_OK) return 0;
  std::cerr << prefix << lbbsp_last_error() << "\n";
  return 1;
}

extern "C" int lbbsp_cmd_run(const char* config, const char* out_dir, int has_seed,
                             uint64_t seed) {
  return cli("lbbsp run: ", [&] {
    Scenario c = load_scenario(config);
    if (has_seed) c.seed = seed;
    fs::create_directories(out_dir);
    const SimRun r = run_scenario(c);
    const lbbsp_records_view v = r.rec.view();
    write_records_csv(v, (fs::path(out_dir) / "records.csv").string());
    const lbbsp_metrics exported = compute_metrics(v, r.converged, c.warmup_iterations, true);
    write_metrics_json(exported, c.convergence_loss, c.convergence_consecutive,
                       c.warmup_iterations, (fs::path(out_dir) / "metrics.json").string());
  });
}

extern "C" int lbbsp_cmd_compare(const char* const* configs, int n_configs, const char* out_dir,
                                 int has_seed, uint64_t seed) {
  return cli("lbbsp compare: ", [&] {
    fs::create_directories(out_dir);
    const std::string path = (fs::path(out_dir) / "comparison.csv").string();
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(LBBSP_RUNTIME, "cannot open " + path);
    out << "scenario,metric,value\n";
    for (int i = 0; i < n_configs; ++i) {
      Scenario c = load_scenario(configs[i]);
      if (has_seed) c.seed = seed;
      const SimRun r = run_scenario(c);
      std::string row;
      auto emit = [&](const char* metric, double value) {
        row.clear();
        row += c.name;
        row += ',';
        row += metric;
        row += ',';
        format_real(row, value);
        row += '\n';
        out << row;
      };
      emit("updates_to_convergence", static_cast<double>(r.metrics.updates_to_convergence));
      emit("mean_per_update_time", r.metrics.mean_per_update_time);
      emit("wastage", r.metrics.wastage);
      emit("predictor_rmse", r.metrics.predictor_rmse);
      emit("converged", r.metrics.converged ? 1.0 : 0.0);
    }
  });
}

extern "C" int lbbsp_cmd_predict_bench(const char* config, const char* out_dir, int has_seed,
                                       uint64_t seed) {
  return cli("lbbsp predict-bench: ", [&] {
    Scenario c = load_scenario(config);
    if (has_seed) c.seed = seed;
    fs::create_directories(out_dir);
    const Bench& bc = c.benchmark;
    if (bc.iterations < 1 || bc.regime_length < 1)
      fail(LBBSP_INVALID_ARGUMENT, "benchmark series: need iterations, regime >= 1");
    std::vector<double> cpu(bc.iterations), mem(bc.iterations), mult(bc.iterations);
    check(lbbsp_benchmark_series(c.seed, bc.iterations, bc.regime_length, bc.high_lo, bc.high_hi,
                                 bc.low_lo, bc.low_hi, bc.spike_mult, bc.spike_prob, cpu.data(),
                                 mem.data(), mult.data()));
    lbbsp_predictor_cfg base{};
    base.alpha = c.alpha;
    base.warmup_iterations = c.warmup_iterations;
    base.speed_floor = c.speed_floor;
    base.train = default_train_cfg(c.warmup_iterations);
    // paired runs always use the benchmark dynamics on a CPU cluster
    Scenario paired_base = c;
    paired_base.preset = "benchmark";
    paired_base.trace_path.clear();
    paired_base.gpu_profiles.clear();
    paired_base.bandwidth_drop.reset();
    double bsp_per_update = 0.0;
    if (c.paired_sim) {
      Scenario bsp = paired_base;
      bsp.scheme = LBBSP_SCHEME_BSP;
      bsp_per_update = run_scenario(bsp).metrics.mean_per_update_time;
    }
    const std::string path = (fs::path(out_dir) / "predict_bench.csv").string();
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(LBBSP_RUNTIME, "cannot open " + path);
    out << "predictor,rmse,normalized_per_update_time\n";
    for (const int kind : {LBBSP_PRED_MEMORYLESS, LBBSP_PRED_EMA, LBBSP_PRED_NARX}) {
      double rmse = 0.0;
      check(lbbsp_predictor_series_rmse(kind, &base, cpu.data(), mem.data(), mult.data(),
                                        bc.iterations, c.base_speed, mix_seed(c.seed, 0xbe11c4ull),
                                        c.warmup_iterations, &rmse));
      std::string row(predictor_name(kind));
      row += ',';
      format_real(row, rmse);
      row += ',';
      if (c.paired_sim) {
        Scenario paired = paired_base;
        paired.scheme = LBBSP_SCHEME_LBBSP;
        paired.predictor = kind;
        const double per_update = run_scenario(paired).metrics.mean_per_update_time;
        format_real(row, per_update / bsp_per_update);
      }
      row += '\n';
      out << row;
    }
  });
}
