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
#include <cerrno>
#include <cctype>
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
// Traces (trace.cpp): CSV `machine_id,t_offset_s,cpu_avail,mem_avail`, one
// series per machine in first-appearance order, times non-decreasing.
// ---------------------------------------------------------------------------
struct TracePoint {
  double t, cpu, mem;
};
struct Trace {
  std::string machine_id;
  std::vector<TracePoint> points;
  // ResourceTrace::mean_cpu (trace.cpp:14-19): sequential sum over the points
  double mean_cpu() const {
    double s = 0.0;
    for (const auto& p : points) s += p.cpu;
    return points.empty() ? 0.0 : s / static_cast<double>(points.size());
  }
};

// Comma-separated fields; a trailing comma ends with an empty field.
std::vector<std::string> csv_fields(const std::string& line) {
  std::vector<std::string> f;
  std::string cur;
  for (char ch : line) {
    if (ch == ',') {
      f.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(ch);
    }
  }
  if (!cur.empty() || (!line.empty() && line.back() == ',')) f.push_back(cur);
  return f;
}

// Reads a trace file; every diagnostic names the 1-based line it concerns
// (the wording of trace.cpp:32-97, which tests and callers match on).
class TraceReader {
 public:
  explicit TraceReader(const std::string& path) : path_(path) {}

  std::vector<Trace> read() {
    std::ifstream in(path_);
    if (!in) fail(LBBSP_RUNTIME, "parse_trace: cannot open " + path_);
    std::string text;
    if (!std::getline(in, text)) fail(LBBSP_RUNTIME, "parse_trace: empty file " + path_);
    check_header(csv_fields(strip_cr(text)));
    int line_no = 1;
    while (std::getline(in, text)) {
      ++line_no;
      const std::string row = strip_cr(text);
      if (!row.empty()) add_row(csv_fields(row), line_no);
    }
    return std::move(out_);
  }

 private:
  static std::string strip_cr(std::string s) {
    if (!s.empty() && s.back() == '\r') s.pop_back();
    return s;
  }
  [[noreturn]] static void at_line(int line_no, const std::string& msg) {
    fail(LBBSP_RUNTIME, "trace line " + std::to_string(line_no) + ": " + msg);
  }
  static void check_header(const std::vector<std::string>& cols) {
    static const char* const kCols[4] = {"machine_id", "t_offset_s", "cpu_avail", "mem_avail"};
    for (const char* name : kCols)
      if (std::find(cols.begin(), cols.end(), name) == cols.end())
        fail(LBBSP_RUNTIME, std::string("parse_trace: missing column '") + name + "'");
    const bool in_order = cols.size() == 4 && std::equal(cols.begin(), cols.end(), kCols);
    if (!in_order)
      fail(LBBSP_RUNTIME, "parse_trace: unexpected column order, want machine_id,t_offset_s,cpu_avail,mem_avail");
  }
  // the whole field must convert (std::stod semantics: leading blanks are
  // skipped, out-of-range values are errors)
  static double number(const std::string& s, const char* what, int line_no) {
    char* end = nullptr;
    errno = 0;
    const double v = std::strtod(s.c_str(), &end);
    if (end == s.c_str() || end != s.c_str() + s.size() || errno == ERANGE)
      at_line(line_no, std::string("bad ") + what + " '" + s + "'");
    return v;
  }
  static double share(const std::string& s, const char* what, int line_no) {
    const double v = number(s, what, line_no);
    if (!(v >= 0.0 && v <= 1.0)) at_line(line_no, std::string(what) + " " + s + " outside [0,1]");
    return v;
  }
  void add_row(const std::vector<std::string>& f, int line_no) {
    if (f.size() != 4) at_line(line_no, "expected 4 fields, got " + std::to_string(f.size()));
    const TracePoint p{number(f[1], "t_offset_s", line_no), share(f[2], "cpu_avail", line_no),
                       share(f[3], "mem_avail", line_no)};
    auto [it, fresh] = slot_.try_emplace(f[0], out_.size());
    if (fresh) out_.push_back(Trace{f[0], {}});
    std::vector<TracePoint>& pts = out_[it->second].points;
    if (!pts.empty() && p.t < pts.back().t)
      at_line(line_no, "time offsets not sorted for machine " + f[0]);
    pts.push_back(p);
  }

  std::string path_;
  std::vector<Trace> out_;
  std::map<std::string, size_t> slot_;
};

std::vector<Trace> parse_trace(const std::string& path) { return TraceReader(path).read(); }

// map_traces (trace.cpp:109-135): the traces ranked by mean cpu availability
// (stable), cut into `workers` equal strata; worker w draws one trace of its
// stratum with the seeded generator.
std::vector<int> map_traces(const std::vector<Trace>& traces, int workers, uint64_t seed) {
  if (traces.empty()) fail(LBBSP_INVALID_ARGUMENT, "map_traces: no traces");
  if (workers < 1) fail(LBBSP_INVALID_ARGUMENT, "map_traces: workers must be >= 1");
  const size_t T = traces.size();
  std::vector<std::pair<double, size_t>> ranked;
  for (size_t i = 0; i < T; ++i) ranked.emplace_back(traces[i].mean_cpu(), i);
  std::stable_sort(ranked.begin(), ranked.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  Rng draw(mix_seed(seed, 0x7ace5ull));
  const double width = static_cast<double>(T) / static_cast<double>(workers);
  std::vector<int> pick(static_cast<size_t>(workers));
  for (int w = 0; w < workers; ++w) {
    const size_t first = static_cast<size_t>(std::floor(width * w));
    const size_t end = std::min(T, std::max(first + 1, static_cast<size_t>(std::floor(width * (w + 1)))));
    const size_t at = first + static_cast<size_t>(draw.uniform() * static_cast<double>(end - first));
    pick[static_cast<size_t>(w)] = static_cast<int>(ranked[std::min(at, T - 1)].second);
  }
  return pick;
}

// ---------------------------------------------------------------------------
// NARX weights CSV (predictor.cpp:198-243): `name,value` rows
// ---------------------------------------------------------------------------
struct NarxField {
  std::string name;
  double lbbsp_narx_model::*member;
  int index;  // input_weights[index] when member is null
};
const std::vector<NarxField>& narx_fields() {
  static const std::vector<NarxField> f = [] {
    std::vector<NarxField> v;
    for (int j = 0; j < 8; ++j) v.push_back({"input_weight_" + std::to_string(j), nullptr, j});
    v.push_back({"hidden_bias", &lbbsp_narx_model::hidden_bias, -1});
    v.push_back({"output_weight", &lbbsp_narx_model::output_weight, -1});
    v.push_back({"output_bias", &lbbsp_narx_model::output_bias, -1});
    v.push_back({"speed_mean", &lbbsp_narx_model::speed_mean, -1});
    v.push_back({"speed_stddev", &lbbsp_narx_model::speed_stddev, -1});
    v.push_back({"cpu_mean", &lbbsp_narx_model::cpu_mean, -1});
    v.push_back({"cpu_stddev", &lbbsp_narx_model::cpu_stddev, -1});
    v.push_back({"mem_mean", &lbbsp_narx_model::mem_mean, -1});
    v.push_back({"mem_stddev", &lbbsp_narx_model::mem_stddev, -1});
    return v;
  }();
  return f;
}
double& narx_ref(lbbsp_narx_model& m, const NarxField& f) {
  return f.member ? m.*(f.member) : m.input_weights[f.index];
}

lbbsp_narx_model load_narx_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(LBBSP_RUNTIME, "load_narx_csv: cannot open " + path);
  std::map<std::string, double> kv;
  for (std::string row; std::getline(in, row);) {
    if (row.empty()) continue;
    const size_t cut = row.find(',');
    if (cut == std::string::npos) fail(LBBSP_RUNTIME, "load_narx_csv: malformed row '" + row + "'");
    kv[row.substr(0, cut)] = std::stod(row.substr(cut + 1));
  }
  lbbsp_narx_model m{};
  for (const NarxField& f : narx_fields()) {
    const auto hit = kv.find(f.name);
    if (hit == kv.end()) fail(LBBSP_RUNTIME, "load_narx_csv: missing parameter '" + f.name + "'");
    narx_ref(m, f) = hit->second;
  }
  return m;
}

void save_narx_csv(lbbsp_narx_model m, const std::string& path) {
  std::ofstream out(path);
  if (!out) fail(LBBSP_RUNTIME, "save_narx_csv: cannot open " + path);
  out.precision(17);
  for (const NarxField& f : narx_fields()) out << f.name << "," << narx_ref(m, f) << "\n";
}

// ---------------------------------------------------------------------------
// Names (coordination.cpp:9-25, predictor.cpp:245-261, cluster_sim.cpp:131-138)
// ---------------------------------------------------------------------------
struct Named {
  const char* name;
  int value;
};
constexpr Named kSchemes[] = {{"bsp", LBBSP_SCHEME_BSP}, {"asp", LBBSP_SCHEME_ASP},
                              {"ssp", LBBSP_SCHEME_SSP}, {"lb-bsp", LBBSP_SCHEME_LBBSP},
                              {"lbbsp", LBBSP_SCHEME_LBBSP}};
constexpr Named kPredictors[] = {{"memoryless", LBBSP_PRED_MEMORYLESS}, {"ema", LBBSP_PRED_EMA},
                                 {"narx", LBBSP_PRED_NARX}, {"perfect", LBBSP_PRED_PERFECT}};
constexpr Named kPresets[] = {{"homo", LBBSP_PRESET_HOMO},
                              {"hetero-l2", LBBSP_PRESET_HETERO_L2},
                              {"hetero-l3", LBBSP_PRESET_HETERO_L3},
                              {"hetero-l2-static", LBBSP_PRESET_HETERO_L2_STATIC},
                              {"hetero-l3-static", LBBSP_PRESET_HETERO_L3_STATIC}};
template <size_t N>
int lookup(const Named (&table)[N], const std::string& s, const char* what) {
  for (const Named& e : table)
    if (s == e.name) return e.value;
  throw std::invalid_argument(std::string("unknown ") + what + ": " + s);
}
template <size_t N>
const char* name_of(const Named (&table)[N], int v) {
  for (const Named& e : table)
    if (e.value == v) return e.name;
  return "?";
}
const char* scheme_name(int k) { return name_of(kSchemes, k); }
const char* predictor_name(int k) { return name_of(kPredictors, k); }

// ---------------------------------------------------------------------------
// Scenario JSON (ScenarioConfig, scenario.hpp:33-64; loader scenario.cpp:31-217)
// ---------------------------------------------------------------------------
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

struct Scenario {
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

// A typed read of one JSON member: absent -> nullopt; present but of the
// wrong type -> "config: bad value for field '<key>'".
template <typename T>
std::optional<T> member(const json& obj, const char* key) {
  const auto it = obj.find(key);
  if (it == obj.end()) return std::nullopt;
  try {
    return it->template get<T>();
  } catch (const json::exception&) {
    config_error(std::string("config: bad value for field '") + key + "'");
  }
}
template <typename T>
T needed(const json& obj, const char* key) {
  if (auto v = member<T>(obj, key)) return *v;
  config_error(std::string("config: missing field '") + key + "'");
}
template <typename T>
void optional_into(const json& obj, const char* key, T& dst) {
  if (auto v = member<T>(obj, key)) dst = *v;
}

// One entry per accepted key, in the order the fields are read (which is the
// order their errors take precedence in). total_budget defaults to 128 per
// worker, so it follows workers.
struct FieldRule {
  const char* key;
  void (*read)(const json& j, Scenario& c);
};
void read_band(const json& j, const char* key, double& lo, double& hi) {
  if (!j.contains(key)) return;
  const auto band = needed<std::vector<double>>(j, key);
  if (band.size() != 2) config_error(std::string("config: field '") + key + "' needs [lo, hi]");
  lo = band[0];
  hi = band[1];
}
const std::vector<FieldRule>& field_rules() {
  static const std::vector<FieldRule> rules = {
      {"scheme",
       [](const json& j, Scenario& c) {
         const std::string s = needed<std::string>(j, "scheme");
         try {
           c.scheme = lookup(kSchemes, s, "scheme");
         } catch (const std::invalid_argument& e) {
           config_error(std::string("config: field 'scheme': ") + e.what());
         }
       }},
      {"workers", [](const json& j, Scenario& c) { c.workers = needed<int>(j, "workers"); }},
      {"staleness_threshold", [](const json& j, Scenario& c) { optional_into(j, "staleness_threshold", c.staleness_threshold); }},
      {"total_budget",
       [](const json& j, Scenario& c) {
         c.total_budget = 128 * c.workers;
         optional_into(j, "total_budget", c.total_budget);
       }},
      {"preset", [](const json& j, Scenario& c) { optional_into(j, "preset", c.preset); }},
      {"trace_path", [](const json& j, Scenario& c) { optional_into(j, "trace_path", c.trace_path); }},
      {"base_speed", [](const json& j, Scenario& c) { optional_into(j, "base_speed", c.base_speed); }},
      {"base_comm_s", [](const json& j, Scenario& c) { optional_into(j, "base_comm_s", c.base_comm_s); }},
      {"predictor",
       [](const json& j, Scenario& c) {
         std::string s = "ema";
         optional_into(j, "predictor", s);
         try {
           c.predictor = lookup(kPredictors, s, "predictor");
         } catch (const std::invalid_argument& e) {
           config_error(std::string("config: field 'predictor': ") + e.what());
         }
       }},
      {"alpha", [](const json& j, Scenario& c) { optional_into(j, "alpha", c.alpha); }},
      {"warmup_iterations", [](const json& j, Scenario& c) { optional_into(j, "warmup_iterations", c.warmup_iterations); }},
      {"speed_floor", [](const json& j, Scenario& c) { optional_into(j, "speed_floor", c.speed_floor); }},
      {"narx_weights_path", [](const json& j, Scenario& c) { optional_into(j, "narx_weights_path", c.narx_weights_path); }},
      {"learning_rate", [](const json& j, Scenario& c) { optional_into(j, "learning_rate", c.learning_rate); }},
      {"dataset_seed", [](const json& j, Scenario& c) { optional_into(j, "dataset_seed", c.dataset_seed); }},
      {"dataset_size", [](const json& j, Scenario& c) { optional_into(j, "dataset_size", c.dataset_size); }},
      {"dataset_dim", [](const json& j, Scenario& c) { optional_into(j, "dataset_dim", c.dataset_dim); }},
      {"dataset_noise", [](const json& j, Scenario& c) { optional_into(j, "dataset_noise", c.dataset_noise); }},
      {"convergence_loss", [](const json& j, Scenario& c) { optional_into(j, "convergence_loss", c.convergence_loss); }},
      {"convergence_consecutive",
       [](const json& j, Scenario& c) { optional_into(j, "convergence_consecutive", c.convergence_consecutive); }},
      {"max_iterations", [](const json& j, Scenario& c) { optional_into(j, "max_iterations", c.max_iterations); }},
      {"seed", [](const json& j, Scenario& c) { optional_into(j, "seed", c.seed); }},
      {"paired_sim", [](const json& j, Scenario& c) { optional_into(j, "paired_sim", c.paired_sim); }},
      {"benchmark_iterations",
       [](const json& j, Scenario& c) { optional_into(j, "benchmark_iterations", c.benchmark.iterations); }},
      {"benchmark_regime_length",
       [](const json& j, Scenario& c) { optional_into(j, "benchmark_regime_length", c.benchmark.regime_length); }},
      {"benchmark_spike_mult",
       [](const json& j, Scenario& c) { optional_into(j, "benchmark_spike_mult", c.benchmark.spike_mult); }},
      {"benchmark_spike_prob",
       [](const json& j, Scenario& c) { optional_into(j, "benchmark_spike_prob", c.benchmark.spike_prob); }},
      {"benchmark_high_band",
       [](const json& j, Scenario& c) { read_band(j, "benchmark_high_band", c.benchmark.high_lo, c.benchmark.high_hi); }},
      {"benchmark_low_band",
       [](const json& j, Scenario& c) { read_band(j, "benchmark_low_band", c.benchmark.low_lo, c.benchmark.low_hi); }},
      {"gpu_profiles",
       [](const json& j, Scenario& c) {
         const auto it = j.find("gpu_profiles");
         if (it == j.end()) return;
         if (!it->is_array()) config_error("config: field 'gpu_profiles' must be an array");
         for (const json& e : *it) {
           GpuGroup grp{};
           grp.profile = lbbsp_gpu_profile{needed<double>(e, "sec_per_sample"), needed<double>(e, "base_time_s"),
                                           needed<int>(e, "saturation_point"), needed<int>(e, "oom_point")};
           grp.count = 1;
           optional_into(e, "count", grp.count);
           c.gpu_profiles.push_back(grp);
         }
       }},
      {"bandwidth_drop",
       [](const json& j, Scenario& c) {
         const auto it = j.find("bandwidth_drop");
         if (it == j.end()) return;
         c.bandwidth_drop = BandwidthDrop{needed<int>(*it, "worker"), needed<int64_t>(*it, "at_iteration"),
                                          needed<double>(*it, "comm_factor")};
       }},
  };
  return rules;
}

// validate_scenario (scenario.cpp:183-217): the first violated rule wins.
struct CheckRule {
  bool (*bad)(const Scenario& c);
  std::string (*message)(const Scenario& c);
};
int gpu_count(const Scenario& c) {
  int total = 0;
  for (const auto& g : c.gpu_profiles) total += g.count;
  return total;
}
const std::vector<CheckRule>& check_rules() {
  using S = const Scenario&;
  static const std::vector<CheckRule> rules = {
      {[](S c) { return c.workers < 1; }, [](S) { return std::string("field 'workers' must be >= 1"); }},
      {[](S c) { return c.total_budget < c.workers; },
       [](S) { return std::string("field 'total_budget' must be >= workers"); }},
      {[](S c) { return c.staleness_threshold < 0; },
       [](S) { return std::string("field 'staleness_threshold' must be >= 0"); }},
      {[](S c) { return !(c.alpha > 0.0 && c.alpha <= 1.0); },
       [](S) { return std::string("field 'alpha' must be in (0, 1]"); }},
      {[](S c) { return c.learning_rate <= 0.0; }, [](S) { return std::string("field 'learning_rate' must be > 0"); }},
      {[](S c) { return c.dataset_size < 1; }, [](S) { return std::string("field 'dataset_size' must be >= 1"); }},
      {[](S c) { return c.dataset_dim < 1; }, [](S) { return std::string("field 'dataset_dim' must be >= 1"); }},
      {[](S c) { return c.convergence_loss <= 0.0; },
       [](S) { return std::string("field 'convergence_loss' must be > 0"); }},
      {[](S c) { return c.convergence_consecutive < 1; },
       [](S) { return std::string("field 'convergence_consecutive' must be >= 1"); }},
      {[](S c) { return c.max_iterations < 1; }, [](S) { return std::string("field 'max_iterations' must be >= 1"); }},
      {[](S c) { return !c.trace_path.empty() && !fs::exists(c.trace_path); },
       [](S c) { return "trace file not found: " + c.trace_path; }},
      {[](S c) { return !c.narx_weights_path.empty() && !fs::exists(c.narx_weights_path); },
       [](S c) { return "narx weights file not found: " + c.narx_weights_path; }},
      {[](S c) { return !c.gpu_profiles.empty() && gpu_count(c) != c.workers; },
       [](S c) {
         return "gpu_profiles counts sum to " + std::to_string(gpu_count(c)) + ", field 'workers' says " +
                std::to_string(c.workers);
       }},
      {[](S c) { return !c.gpu_profiles.empty() && !c.trace_path.empty(); },
       [](S) { return std::string("gpu_profiles and trace_path cannot be combined"); }},
      {[](S c) {
         return c.bandwidth_drop && (c.bandwidth_drop->worker < 0 || c.bandwidth_drop->worker >= c.workers);
       },
       [](S) { return std::string("bandwidth_drop worker out of range"); }},
  };
  return rules;
}

void validate_scenario(const Scenario& c) {
  for (const CheckRule& r : check_rules())
    if (r.bad(c)) config_error("config: " + r.message(c));
}

Scenario load_scenario(const std::string& path_str) {
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
  const auto& rules = field_rules();
  for (const auto& item : j.items()) {  // strict keys (object keys iterate sorted)
    const bool known = std::any_of(rules.begin(), rules.end(),
                                   [&](const FieldRule& r) { return item.key() == r.key; });
    if (!known) config_error("config: unknown field '" + item.key() + "'");
  }
  Scenario c;
  c.name = path.stem().string();
  for (const FieldRule& r : rules) r.read(j, c);
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
      s.preset = lookup(kPresets, c.preset, "preset");
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
  return guarded([&] { save_narx_csv(*m, path); });
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

// cmd_run (scenario.cpp:369-386): the records/metrics exporters over one scenario
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
