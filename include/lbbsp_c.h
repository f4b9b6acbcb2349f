/*
 * lbbsp_c.h -- C-ABI boundary of the B200-native LB-BSP iteration hot path.
 *
 * The reference (arxiv 1806.02508, /root/reference/proj) has no FFI: its API is
 * the C++ headers under core/include/lbbsp/. Every entry point below names the
 * reference function it replaces (file:line, relative to /root/reference/proj).
 * A reference-side caller binds these symbols with ctypes / a C++ shim
 * (include/lbbsp_b200.hpp) -- see INTEGRATION.md.
 *
 * Conventions
 *   - Plain pointers and sizes only. `d_` prefixes are DEVICE pointers, `h_`
 *     prefixes HOST pointers. Streams are passed as `void*` (cudaStream_t).
 *   - Every call returns an int status (LBBSP_OK == 0). The message of the
 *     last failure on this thread is `lbbsp_last_error()`, worded like the
 *     reference exception text (e.g. "gpu_allocate: budget 100 below total
 *     saturation minimum 150", batch_sizer.cpp:37-42).
 *   - Device-side precondition failures are written to a device status word
 *     (lbbsp_dev_status) and surfaced by the host-pointer variants, which
 *     synchronise; the device-pointer variants never synchronise.
 *   - There is no CPU fallback: without a CUDA device every compute entry
 *     point returns LBBSP_CUDA.
 */
#ifndef LBBSP_C_H
#define LBBSP_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map to the reference exception types) --- */
#define LBBSP_OK 0
#define LBBSP_INVALID_ARGUMENT (-1) /* std::invalid_argument */
#define LBBSP_OUT_OF_RANGE (-2)     /* std::out_of_range     */
#define LBBSP_RUNTIME (-3)          /* std::runtime_error    */
#define LBBSP_LOGIC (-4)            /* std::logic_error      */
#define LBBSP_CUDA (-5)
#define LBBSP_NCCL (-6)
#define LBBSP_CONFIG (-7)           /* lbbsp::ConfigError (scenario.hpp:13-15), a runtime_error */

const char* lbbsp_last_error(void);
int lbbsp_version(void);
/* number of CUDA devices visible to the library; 0 on a CPU-only host */
int lbbsp_device_count(void);

/* Device status word written by kernels when a precondition fails. */
typedef struct {
  int code;   /* 0 ok, else one of the status codes above            */
  int what;   /* which check failed (LBBSP_E_* below)                */
  int64_t a;  /* numeric payload for the message                     */
  int64_t b;
} lbbsp_dev_status;

/* Formats a device status word copied back to the host into
 * lbbsp_last_error() (reference wording) and returns its code. */
int lbbsp_check_status(const lbbsp_dev_status* h_status);

enum {
  LBBSP_E_NONE = 0,
  LBBSP_E_CPU_NO_WORKERS = 1,      /* "cpu_allocate: no workers"                  */
  LBBSP_E_CPU_BUDGET = 2,          /* "cpu_allocate: budget a below worker count b"*/
  LBBSP_E_CPU_SPEED = 3,           /* "cpu_allocate: speeds must be > 0"          */
  LBBSP_E_CPU_MIN1 = 4,            /* "cpu_allocate: cannot enforce minimum batch"*/
  LBBSP_E_GPU_NO_WORKERS = 10,
  LBBSP_E_GPU_SLOPE = 11,
  LBBSP_E_GPU_BASE = 12,
  LBBSP_E_GPU_BOUNDS = 13,
  LBBSP_E_GPU_COMM = 14,
  LBBSP_E_GPU_BELOW = 15,          /* "budget a below total saturation minimum b" */
  LBBSP_E_GPU_ABOVE = 16,          /* "budget a above total memory capacity b"    */
  LBBSP_E_GPU_REPAIR = 17,
  LBBSP_E_GPU_OOM = 18,            /* gpu_compute_time: batch above oom point     */
  LBBSP_E_GRAD_EMPTY = 20,
  LBBSP_E_GRAD_INDEX = 21,
  LBBSP_E_AGG_BATCH = 22,
  LBBSP_E_MLP_CAPACITY = 30        /* "mlp: round a exceeds max_iterations b"      */
};

/* ======================================================================== */
/* Batch-size solver (K1/K2)                                                */
/* ======================================================================== */

/* GpuProfile, batch_sizer.hpp:10-15 */
typedef struct {
  double sec_per_sample;
  double base_time_s;
  int saturation_point;
  int oom_point;
} lbbsp_gpu_profile;

/* clamp_speed_floor (batch_sizer.cpp:12-14) + cpu_allocate (batch_sizer.cpp:54-99)
 * as ONE single-block kernel. speed_floor <= 0 disables the clamp (plain
 * cpu_allocate). Device pointers, stream-ordered, no host sync. */
int lbbsp_solve_prop(const double* d_speeds, int n, int budget, double speed_floor,
                     int* d_sizes, lbbsp_dev_status* d_status, void* stream);

/* gpu_allocate (batch_sizer.cpp:101-199), single-block kernel. */
int lbbsp_solve_gpu(const lbbsp_gpu_profile* d_profiles, const double* d_comm, int n,
                    int budget, int* d_sizes, lbbsp_dev_status* d_status, void* stream);

/* Host-pointer variants (synchronous): same kernels, reference error text. */
int lbbsp_cpu_allocate(const double* h_speeds, int n, int budget, int* h_sizes);
int lbbsp_gpu_allocate(const lbbsp_gpu_profile* h_profiles, const double* h_comm, int n,
                       int budget, int* h_sizes);

/* ======================================================================== */
/* Speed predictor (K3-K5)                                                  */
/* ======================================================================== */

enum { LBBSP_PRED_MEMORYLESS = 0, LBBSP_PRED_EMA = 1, LBBSP_PRED_NARX = 2, LBBSP_PRED_PERFECT = 3 };

/* NarxModel (predictor.hpp:49-67) without the unbounded training_loss log. */
typedef struct {
  double input_weights[8];
  double hidden_bias;
  double output_weight;
  double output_bias;
  double speed_mean, speed_stddev;
  double cpu_mean, cpu_stddev;
  double mem_mean, mem_stddev;
} lbbsp_narx_model;

/* NarxTrainConfig (predictor.hpp:69-75) */
typedef struct {
  double step;
  int max_epochs;
  double early_stop_delta;
  int early_stop_patience;
  int min_history;
} lbbsp_narx_train_cfg;

/* NarxTrainReport (predictor.hpp:84-88) */
typedef struct {
  int ran;
  int epochs;
  double final_loss;
} lbbsp_narx_report;

/* narx_init (predictor.cpp:35-44), computed on the host (setup, not hot path). */
int lbbsp_narx_init(uint64_t seed, lbbsp_narx_model* out);

/* ema (predictor.cpp:18-25) over a host series, evaluated by the device kernel. */
int lbbsp_ema(const double* h_series, int len, double alpha, double* h_out);

/* narx_predict (predictor.cpp:147-153). windows most-recent-first. */
int lbbsp_narx_predict(const lbbsp_narx_model* h_model, const double h_speeds[2],
                       const double h_cpu[3], const double h_mem[3], double floor,
                       double* h_out);

/* Verification hook: the device restatement of glibc tanh that every NARX
 * forward uses (exactmath.cuh; std::tanh at predictor.cpp:60,109,117),
 * evaluated elementwise over n host inputs. */
int lbbsp_glibc_tanh(const double* h_x, double* h_y, long long n);

/* narx_train_online (predictor.cpp:155-196) over one host history.
 * h_loss_log (optional, may be NULL) receives one entry per accepted epoch
 * (NarxModel::training_loss), capacity max_epochs. Bit-exact fp64 kernel. */
int lbbsp_narx_train_online(lbbsp_narx_model* h_model, const double* h_speed,
                            const double* h_cpu, const double* h_mem, int len,
                            const lbbsp_narx_train_cfg* cfg, lbbsp_narx_report* h_report,
                            double* h_loss_log);

/* PredictorConfig (predictor.hpp:107-114) */
typedef struct {
  int kind;
  double alpha;
  int warmup_iterations;
  double speed_floor;
  lbbsp_narx_train_cfg train; /* train.min_history is forced to warmup (predictor.cpp:264) */
} lbbsp_predictor_cfg;

/* A bank of per-worker SpeedPredictors (predictor.hpp:118-136) whose
 * histories (SpeedHistory, predictor.hpp:15-26) live in device memory. */
typedef struct lbbsp_predictor lbbsp_predictor;

/* seeds[i] is the per-worker predictor seed (cluster_sim.cpp:295 uses
 * mix_seed(seed, 0x9ced1c70, i)); NULL initial models => narx_init(seeds[i]). */
int lbbsp_predictor_create(const lbbsp_predictor_cfg* cfg, int n_workers, int max_history,
                           const uint64_t* h_seeds, const lbbsp_narx_model* h_initial,
                           lbbsp_predictor** out);
int lbbsp_predictor_destroy(lbbsp_predictor* p);
/* SpeedHistory::push for every worker (cluster_sim.cpp:309-313). */
int lbbsp_predictor_observe(lbbsp_predictor* p, const double* d_v, const double* d_c,
                            const double* d_m, void* stream);
/* SpeedPredictor::predict for every worker (predictor.cpp:271-292), batched. */
int lbbsp_predictor_predict(lbbsp_predictor* p, const double* d_c_now, const double* d_m_now,
                            double* d_v_pred, void* stream);
/* train_rotation (cluster_sim.cpp:315-324): trains ceil(n/2) models from the
 * device-resident cursor, one CTA per model, and advances the cursor. */
int lbbsp_predictor_train_rotation(lbbsp_predictor* p, void* stream);
/* Train every model (predictor_series_rmse replays / C4 sweep). */
int lbbsp_predictor_train_all(lbbsp_predictor* p, void* stream);
int lbbsp_predictor_get_models(lbbsp_predictor* p, lbbsp_narx_model* h_models);
int lbbsp_predictor_history_len(lbbsp_predictor* p, int* h_len);

/* ======================================================================== */
/* Workload: reference logistic-regression worker (K6-K10), fp64            */
/* ======================================================================== */

/* sample_stream (cluster_sim.cpp:302-307): B draws of
 * mt19937_64(mix_seed(seed, 0x57e3a9, k)) mapped by Rng::uniform_int(0, N-1). */
int lbbsp_sample_stream(uint64_t seed, int64_t iteration, int budget, int dataset_size,
                        int* d_indices, void* stream);

/* Dataset (sgd.hpp:15-21) resident on device, SoA features [N][d] + labels. */
typedef struct lbbsp_lr_data lbbsp_lr_data;
/* generate_dataset (sgd.cpp:39-57) */
int lbbsp_lr_data_create(uint64_t seed, int n, int d, double noise, lbbsp_lr_data** out);
/* Upload an explicit dataset (row-major features[n*d], labels[n]). */
int lbbsp_lr_data_upload(const double* h_features, const double* h_labels, int n, int d,
                         lbbsp_lr_data** out);
int lbbsp_lr_data_destroy(lbbsp_lr_data* data);
int lbbsp_lr_data_dim(const lbbsp_lr_data* data, int* n, int* d);

/* batch_gradient (sgd.cpp:72-90) for n_seg contiguous segments of d_idx:
 * segment i = d_idx[off_i : off_i + d_sizes[i]], off_i = prefix sum.
 * d_grads receives n_seg x d per-worker MEAN gradients (Gradient::values). */
int lbbsp_lr_worker_grads(const lbbsp_lr_data* data, const double* d_params,
                          const int* d_idx, const int* d_sizes, int n_seg, double* d_grads,
                          lbbsp_dev_status* d_status, void* stream);

/* aggregate_weighted (coordination.cpp:52-68) when weighted != 0, else
 * aggregate_naive (coordination.cpp:39-50), fused with apply_update
 * (sgd.cpp:92-99): params -= lr * agg. d_agg (optional) receives the aggregate,
 * d_norm (optional) its l2 norm (cluster_sim.cpp:203-207). */
int lbbsp_aggregate_apply(const double* d_grads, const int* d_sizes, int n_seg, int dim,
                          int weighted, double lr, double* d_params, double* d_agg,
                          double* d_norm, lbbsp_dev_status* d_status, void* stream);

/* loss (sgd.cpp:65-70) over the whole device dataset. */
int lbbsp_lr_loss(const lbbsp_lr_data* data, const double* d_params, double* d_loss,
                  void* stream);

/* generate_dataset / separator_params (sgd.cpp:32-57) into host arrays
 * (row-major features [n][d], labels [n]): setup-time host generators. */
int lbbsp_generate_dataset(uint64_t seed, int n, int d, double noise, double* h_features,
                           double* h_labels);
int lbbsp_separator_params(uint64_t seed, int d, double* h_out);
/* apply_update (sgd.cpp:92-99): h_params -= lr * h_grad on the device (K9). */
int lbbsp_apply_update(double* h_params, int dim, const double* h_grad, double lr);

/* Host-pointer convenience variants for the reference-shaped API. */
int lbbsp_batch_gradient(const lbbsp_lr_data* data, const double* h_params,
                         const int* h_indices, int count, double* h_grad);
int lbbsp_loss(const lbbsp_lr_data* data, const double* h_params, double* h_loss);
/* aggregate over n host gradients of dimension dim with batch sizes */
int lbbsp_aggregate(const double* h_grads, const int* h_sizes, int n, int dim, int weighted,
                    double* h_out);

/* ======================================================================== */
/* Fused iteration driver (A1 step_sync, cluster_sim.cpp:349-469; ASP/SSP  */
/* step_async :486-631 as one persistent event-loop CTA)                    */
/* ======================================================================== */

enum { LBBSP_SCHEME_BSP = 0, LBBSP_SCHEME_ASP = 1, LBBSP_SCHEME_SSP = 2, LBBSP_SCHEME_LBBSP = 3 };
enum {
  LBBSP_DYN_STATIC = 0,
  LBBSP_DYN_STRAGGLER = 1,
  LBBSP_DYN_BENCHMARK = 2,
  LBBSP_DYN_TRACE = 3     /* recorded resource traces (cluster_sim.cpp:110-115) */
};
enum {
  LBBSP_PRESET_NONE = -1,
  LBBSP_PRESET_HOMO = 0,
  LBBSP_PRESET_HETERO_L2 = 1,
  LBBSP_PRESET_HETERO_L3 = 2,
  LBBSP_PRESET_HETERO_L2_STATIC = 3,
  LBBSP_PRESET_HETERO_L3_STATIC = 4
};

/* StragglerSpec, cluster_sim.hpp:43-48 */
typedef struct {
  double on_probability;
  double cpu_consumed;
  double mem_consumed;
  int period;
} lbbsp_straggler;

#define LBBSP_MAX_WORKERS 1024

/* SimConfig (cluster_sim.hpp:165-180) flattened, plus the worker/dynamics
 * description that SimConfig carries in WorkerProfile/DynamicsConfig. */
typedef struct {
  int scheme;             /* LBBSP_SCHEME_BSP | LBBSP_SCHEME_LBBSP                  */
  int n_workers;
  int total_budget;
  int preset;             /* LBBSP_PRESET_*, NONE => use dynamics below         */
  double base_speed;      /* WorkerProfile::base_speed (CPU kind)                 */
  int dynamics;           /* LBBSP_DYN_* when preset == NONE                     */
  const double* static_cpu;              /* [n] or NULL (1.0)                    */
  const double* static_mem;              /* [n] or NULL (1.0)                    */
  const lbbsp_straggler* stragglers;     /* [n] for LBBSP_DYN_STRAGGLER          */
  /* BenchmarkTraceConfig, cluster_sim.hpp:76-83 */
  int bench_iterations, bench_regime_length;
  double bench_high_lo, bench_high_hi, bench_low_lo, bench_low_hi;
  double bench_spike_mult, bench_spike_prob;
  /* predictor */
  lbbsp_predictor_cfg predictor;
  /* GPU-kind cluster (gpu_mode): profiles[n] != NULL switches every worker to Gpu */
  const lbbsp_gpu_profile* gpu_profiles;
  /* CommModel per worker: tm = base_comm_s * factor(k) */
  double base_comm_s;
  int bw_worker;          /* -1: none; else BandwidthEvent on that worker         */
  int64_t bw_at_iteration;
  double bw_factor;
  /* SimConfig scalars */
  double learning_rate;
  uint64_t dataset_seed;
  int dataset_size;
  int dataset_dim;
  double dataset_noise;
  double convergence_loss;
  int convergence_consecutive;
  int64_t max_updates;
  uint64_t seed;
  /* DynamicsKind::Trace (cluster_sim.cpp:110-115): worker i follows the
   * step-interpolated trace (trace_at, trace.cpp:137-143) made of points
   * [trace_offsets[i], trace_offsets[i+1]) of the three arrays, looked up at
   * the simulated clock (the sum of the previous rounds' walls). */
  const int* trace_offsets;   /* [n+1] */
  const double* trace_t;
  const double* trace_cpu;
  const double* trace_mem;
  /* PredictorConfig::initial_weights (predictor.cpp:264-269): NULL or "" =>
   * narx_init(mix_seed(seed, 0x9ced1c70, i)); else load_narx_csv(path) */
  const char* narx_weights_path;
  /* SchemeConfig::staleness_threshold (coordination.hpp:15-19), SSP only */
  int staleness_threshold;
} lbbsp_sim_cfg;

/* IterationRecord (cluster_sim.hpp:149-155) + WorkerIterationStats (:139-147),
 * flattened: per-iteration scalars and [n] per-worker arrays. */
typedef struct {
  int64_t k;
  double grad_norm;
  double loss;
  double wall_s;
} lbbsp_iter_scalars;

/* make_benchmark_series (cluster_sim.cpp:41-64) with the given
 * BenchmarkTraceConfig: the recorded-trace generator behind the "benchmark"
 * dynamics (A2). Host arrays of length iterations. */
int lbbsp_benchmark_series(uint64_t seed, int iterations, int regime_length, double high_lo,
                           double high_hi, double low_lo, double low_hi, double spike_mult,
                           double spike_prob, double* h_cpu, double* h_mem, double* h_mult);

typedef struct lbbsp_sim lbbsp_sim;

int lbbsp_sim_create(const lbbsp_sim_cfg* cfg, lbbsp_sim** out);
int lbbsp_sim_destroy(lbbsp_sim* sim);
/* Run up to `iterations` LB-BSP/BSP barrier rounds with no host round trip
 * (the convergence stop of check_stop, cluster_sim.cpp:326-334, is evaluated
 * on device and turns the remaining rounds into no-ops). */
int lbbsp_sim_run(lbbsp_sim* sim, int iterations, void* stream);
/* Copy out the records produced so far (blocking). Arrays are [rows] and
 * [rows*n]; params is [rows*d] (the record_params trajectory). Any pointer
 * may be NULL. Returns the row count in *rows. */
int lbbsp_sim_records(lbbsp_sim* sim, int max_rows, int* rows, lbbsp_iter_scalars* scalars,
                      int* batch, double* tp, double* tm, double* wait, double* v_pred,
                      double* v_actual, double* params);
int lbbsp_sim_status(lbbsp_sim* sim, int* done, int* converged);
/* Worker ids of the record slots ([rows*n]) and the number of worker stats
 * per record ([rows]): n for BSP/LB-BSP/SSP rounds, 1 for ASP updates. */
int lbbsp_sim_record_workers(lbbsp_sim* sim, int max_rows, int* worker_id, int* row_workers);
/* SimResult::total_time_s and max_ssp_skew (cluster_sim.cpp:633-643). */
int lbbsp_sim_summary(lbbsp_sim* sim, double* total_time_s, int64_t* max_ssp_skew);
/* Number of CUDA kernels one iteration launches (captured graph nodes). */
int lbbsp_sim_launches_per_iteration(lbbsp_sim* sim, int* launches);

/* ======================================================================== */
/* Records, metrics and exporters                      */
/* ======================================================================== */

/* A host view of a record stream: [rows] scalars, [rows*n] per-worker rows. */
typedef struct {
  int rows;
  int n;
  const lbbsp_iter_scalars* scalars;
  const int* batch;
  const double* tp;
  const double* tm;
  const double* wait;
  const double* v_pred;
  const double* v_actual;
  const int* worker_id;    /* [rows*n] or NULL (slot i = worker i)          */
  const int* row_workers;  /* [rows] stats per row or NULL (n; 1 for ASP)   */
} lbbsp_records_view;

/* Metrics (cluster_sim.hpp:157-163) */
typedef struct {
  int64_t updates_to_convergence;
  double mean_per_update_time;
  double wastage;
  double predictor_rmse;
  int converged;
} lbbsp_metrics;

/* compute_metrics (cluster_sim.cpp:217-245). round9 != 0 first rounds every
 * real to 9 significant digits as the exporter does (round_records,
 * scenario.cpp:66-88), giving the metrics.json numbers. Host. */
int lbbsp_compute_metrics(const lbbsp_records_view* rec, int converged, int rmse_from_iteration,
                          int round9, lbbsp_metrics* out);
/* Simulation::run's metrics (cluster_sim.cpp:638) computed on device from the
 * device-resident records: per-row terms in parallel, the reference's
 * sequential folds by one thread. */
int lbbsp_sim_metrics(lbbsp_sim* sim, int rmse_from_iteration, lbbsp_metrics* out);
/* write_records_csv (scenario.cpp:306-342): byte-identical records.csv. */
int lbbsp_write_records_csv(const lbbsp_records_view* rec, const char* path);
/* write_metrics_json (scenario.cpp:344-358): byte-identical metrics.json. */
int lbbsp_write_metrics_json(const lbbsp_metrics* m, double convergence_loss,
                             int convergence_consecutive, int warmup_iterations, const char* path);

/* ======================================================================== */
/* Recorded resource traces (trace.hpp:11-38)           */
/* ======================================================================== */

typedef struct lbbsp_traces lbbsp_traces;

/* parse_trace (trace.cpp:54-97): machine_id,t_offset_s,cpu_avail,mem_avail. */
int lbbsp_trace_parse(const char* path, lbbsp_traces** out);
/* In-memory traces: trace i = points [offsets[i], offsets[i+1]). */
int lbbsp_trace_create(int n_traces, const char* const* machine_ids, const int* offsets,
                       const double* t, const double* cpu, const double* mem,
                       lbbsp_traces** out);
int lbbsp_trace_destroy(lbbsp_traces* tr);
int lbbsp_trace_count(const lbbsp_traces* tr, int* n_traces);
/* machine id (valid until destroy), point count, ResourceTrace::mean_cpu */
int lbbsp_trace_info(const lbbsp_traces* tr, int i, const char** machine_id, int* points,
                     double* mean_cpu);
int lbbsp_trace_points(const lbbsp_traces* tr, int i, double* t, double* cpu, double* mem);
/* write_trace (trace.cpp:99-107) */
int lbbsp_trace_write(const lbbsp_traces* tr, const char* path);
/* map_traces (trace.cpp:109-135): one trace index per worker. */
int lbbsp_trace_map(const lbbsp_traces* tr, int workers, uint64_t seed, int* assignment);
/* trace_at (trace.cpp:137-143) */
int lbbsp_trace_at(const lbbsp_traces* tr, int i, double time_s, double* cpu, double* mem);

/* load_narx_csv / save_narx_csv (predictor.cpp:198-243) */
int lbbsp_narx_load_csv(const char* path, lbbsp_narx_model* out);
int lbbsp_narx_save_csv(const lbbsp_narx_model* m, const char* path);

/* ======================================================================== */
/* Scenario JSON and the CLI entry points (scenario.hpp:13-91, 8(f) rank 3) */
/* ======================================================================== */

typedef struct lbbsp_scenario lbbsp_scenario;

/* ScenarioConfig scalars (scenario.hpp:33-64) */
typedef struct {
  char name[256];           /* config file stem */
  int scheme;               /* LBBSP_SCHEME_* */
  int staleness_threshold;
  int workers;
  int total_budget;
  int predictor;            /* LBBSP_PRED_* */
  double alpha;
  int warmup_iterations;
  double speed_floor;
  double base_speed;
  double base_comm_s;
  double learning_rate;
  double convergence_loss;
  int convergence_consecutive;
  int64_t max_iterations;
  uint64_t seed;
  int paired_sim;
} lbbsp_scenario_info;

/* load_scenario + validate_scenario (scenario.cpp:92-217): strict keys,
 * reference ConfigError wording (LBBSP_CONFIG). */
int lbbsp_scenario_load(const char* path, lbbsp_scenario** out);
int lbbsp_scenario_destroy(lbbsp_scenario* s);
/* the CLI's --seed override (cfg.seed = seed before build_sim_config) */
int lbbsp_scenario_set_seed(lbbsp_scenario* s, uint64_t seed);
int lbbsp_scenario_get_info(const lbbsp_scenario* s, lbbsp_scenario_info* info);
/* build_sim_config (scenario.cpp:219-294): presets, traces (parse_trace +
 * map_traces), GPU groups and the bandwidth drop resolved into a
 * lbbsp_sim_cfg whose arrays the scenario owns (valid until destroy or the
 * next set_seed). ASP/SSP scenarios are rejected (out of scope). */
int lbbsp_scenario_sim_cfg(lbbsp_scenario* s, const lbbsp_sim_cfg** cfg);

/* predictor_series_rmse (cluster_sim.cpp:645-672) on device: one predictor
 * replayed over a benchmark series (h_cpu/h_mem/h_mult [len]), predicting
 * then observing then training every step, one CTA. */
int lbbsp_predictor_series_rmse(int kind, const lbbsp_predictor_cfg* base, const double* h_cpu,
                                const double* h_mem, const double* h_mult, int len,
                                double base_speed, uint64_t seed, int measure_from,
                                double* rmse);

/* cmd_run (scenario.cpp:369-386): load a scenario, run it on the device
 * driver, write records.csv + metrics.json. Returns the CLI exit status (0 ok,
 * 1 error; the error is printed to stderr as "lbbsp run: <what>" and kept in
 * lbbsp_last_error()). has_seed selects the --seed override. The other CLI
 * commands (compare, predict-bench) are front-end glue outside the hot path
 * and are not exported. */
int lbbsp_cmd_run(const char* config, const char* out_dir, int has_seed, uint64_t seed);

/* ======================================================================== */
/* C4: NARX at sweep scale -- delay d, hidden H, W models, fp32 CUDA cores   */
/* ======================================================================== */

/* Generalised NarxModel (predictor.hpp:49-67) with lags d (inputs 3d+2) and H
 * tanh units; params per model: W1[H][3d+2] | b1[H] | w2[H] | b2 | 6 scalers. */
int lbbsp_narxg_param_count(int delay, int hidden);
/* narx_init (predictor.cpp:35-44) generalised, same draw order (host). */
int lbbsp_narxg_init(uint64_t seed, int delay, int hidden, float* h_params);
/* narx_train_online (predictor.cpp:155-196) for W models at once, one CTA per
 * model; histories d_v/d_c/d_m are [W][L]; fixed_epochs > 0 disables the
 * early stop (throughput mode). d_epochs [W], d_loss [W] outputs;
 * d_scratch: lbbsp_narx_sweep_scratch_floats(...) floats. */
int lbbsp_narx_sweep_train(int W, int L, int delay, int hidden, const double* d_v,
                           const double* d_c, const double* d_m, float* d_params,
                           const lbbsp_narx_train_cfg* cfg, int fixed_epochs, int* d_epochs,
                           float* d_loss, float* d_scratch, void* stream);
long long lbbsp_narx_sweep_scratch_floats(int W, int L, int delay, int hidden);
/* narx_predict (predictor.cpp:147-153) for W models (histories [W][L], the
 * current exogenous values c_now/m_now [W]). */
int lbbsp_narx_sweep_predict(int W, int L, int delay, int hidden, const double* d_v,
                             const double* d_c, const double* d_m, const double* d_c_now,
                             const double* d_m_now, const float* d_params, double floor,
                             double* d_out, void* stream);

/* ======================================================================== */
/* Gradient engine building block: tcgen05/TMA bf16 GEMM (K7, north_star 1) */
/* ======================================================================== */

/* C[M,N] = epilogue(A * B^T) with bf16 operands, fp32 accumulation in TMEM.
 *   A: a_mn ? [K][M] : [M][K];  B: b_mn ? [K][N] : [N][K] (dense bf16 rows)
 *   epilogue: 0 C_f32 = acc; 1 C_bf16 = relu(acc + bias); 2 C_bf16 = acc + bias;
 *             3 C_bf16 = acc * (aux > 0)  (aux = bf16 [M][N])
 *   mode 0 (rows): worker g owns rows [r0_g, r1_g) of M (ragged, masked);
 *   mode 1 (k-split): worker g owns K range [r0_g, r1_g) and writes its fp32
 *   partial to C + g*M*N (the segmented reduction sums them).
 *   Worker g runs on CTAs [cta0_g, cta0_g + ctan_g) -- its SM cap.
 *   d_timing (optional) [n_groups][2] u64 {min start, max end} globaltimer ns.
 * Replaces the per-worker batch_gradient loop (sgd.cpp:72-90,
 * cluster_sim.cpp:422-431) for the dense-layer workloads. */
int lbbsp_gemm_bf16(const void* d_a, const void* d_b, void* d_c, int M, int N, int K, int a_mn,
                    int b_mn, int epilogue, const float* d_bias, const void* d_aux, int mode,
                    int n_groups, const int* d_group_r0, const int* d_group_r1,
                    const int* d_group_cta0, const int* d_group_ctan, int ctas,
                    unsigned long long* d_timing, int bn, void* stream);

/* ======================================================================== */
/* MLP gradient engine with emulated / sharded workers (C1-C5)               */
/* ======================================================================== */

#define LBBSP_MLP_MAX_LAYERS 8

/* One LB-BSP iteration of data-parallel MLP training on this GPU. Workers are
 * either emulated on this GPU (n_workers_local > 1: each gets a CTA partition
 * = SM cap driven by the trace) or one per GPU (n_workers_local == 1, ranks
 * exchange gradients with ncclAllReduce and speeds with ncclAllGather).
 * The workload generalises the reference's logistic regression
 * (sgd.cpp:32-99) to an MLP with softmax-CE; sample stream, contiguous
 * chunking, Eq.-7 weighting and the update follow cluster_sim.cpp:422-439. */
typedef struct {
  int n_layers;                       /* number of Linear layers            */
  int dims[LBBSP_MLP_MAX_LAYERS + 1]; /* dims[0] input .. dims[n_layers] out */
  int n_workers_total;
  int n_workers_local;
  int rank, world;
  int global_batch;                   /* B over all workers                  */
  int scheme;                         /* LBBSP_SCHEME_BSP | _LBBSP           */
  int static_sizes;                   /* 1: h_static_sizes every round        */
  const int* h_static_sizes;          /* [n_workers_total] (static-proportional) */
  lbbsp_predictor_cfg predictor;
  double learning_rate;
  uint64_t seed;                      /* sample stream + predictor seeds     */
  uint64_t dataset_seed;
  int dataset_size;
  int loss_every;                     /* full-dataset loss cadence (1 = every round) */
  int sm_budget;                      /* SMs this rank's workers may use (0 = all) */
  /* straggler trace, iteration-indexed: worker availability
   * a = min(1, c * MemPenalty(m) * mult) (cluster_sim.cpp:22-29), injected as
   * straggler_mode says; [n_workers_total][trace_len], host */
  const double* h_trace_c;
  const double* h_trace_m;
  const double* h_trace_mult;
  int trace_len;
  const double* h_worker_share;       /* [n_workers_total] nominal share of its GPU (NULL: 1/n_local) */
  int max_iterations;                 /* record capacity                     */
  int straggler_mode;                 /* LBBSP_STRAGGLE_INTERFERE (0, default) | _SM_CAP (1) */
  int solver;                         /* LBBSP_SOLVER_PROPORTIONAL (0, default) | _GAMMA (1) */
  const lbbsp_gpu_profile* h_gpu_profiles; /* [n_workers_total] unloaded Gamma (GAMMA solver, CAPACITY) */
  int observe;                        /* LBBSP_OBSERVE_RATE (0, default) | _CAPACITY (1) */
} lbbsp_mlp_cfg;

/* Batch-size solver of the MLP engine's LB-BSP rounds:
 * PROPORTIONAL: cpu_allocate over clamp_speed_floor(v_pred), v = b / t
 *   (the reference's CPU-cluster branch, north_star (4));
 * GAMMA: gpu_allocate over per-worker profiles Gamma_i(x) = (m0_i max(x, x_s_i)
 *   + b0_i) / a_i, with the unloaded (m0, b0, x_s, x_o) given and a_i the
 *   predicted availability; the observed speed is Gamma0_i(b) / t (the
 *   reference's GPU-cluster branch with a predictor, cluster_sim.cpp:373-387). */
#define LBBSP_SOLVER_PROPORTIONAL 0
#define LBBSP_SOLVER_GAMMA 1

/* The speed the proportional solver's predictor observes per worker and round
 * (b rows in t seconds):
 * RATE: b / t;
 * CAPACITY: a * x_n / Gamma0(x_n), the worker's speed at the nominal batch
 *   x_n = B / n with a = Gamma0(b) / t read off its unloaded profile (needs
 *   h_gpu_profiles) -- the reference's CPU-mode v_actual (the speed of the
 *   worker under its resource state, cluster_sim.cpp:357-361), which b / t is
 *   not when the worker time has a fixed latency. */
#define LBBSP_OBSERVE_RATE 0
#define LBBSP_OBSERVE_CAPACITY 1

/* How a worker's availability a = min(1, c * MemPenalty(m) * mult) is injected:
 * INTERFERE: the worker keeps its nominal CTA partition and co-scheduled
 *   interference on those SMs stretches every phase to (work time) / a
 *   (SM-bound FMA chains; HBM-bound streaming for the memory-penalty part);
 * SM_CAP: the partition shrinks to floor(budget * share * a) CTAs (round 1). */
#define LBBSP_STRAGGLE_INTERFERE 0
#define LBBSP_STRAGGLE_SM_CAP 1

typedef struct lbbsp_mlp lbbsp_mlp;

int lbbsp_mlp_create(const lbbsp_mlp_cfg* cfg, lbbsp_mlp** out);
int lbbsp_mlp_destroy(lbbsp_mlp* m);
/* NCCL plumbing for world > 1: rank 0 gets an id, every rank inits with it. */
int lbbsp_nccl_unique_id(unsigned char h_id[128]);
int lbbsp_mlp_init_comm(lbbsp_mlp* m, const unsigned char h_id[128]);
/* Optional NVLink peer exchange on several GPUs: each rank exports a device
 * buffer (64-byte CUDA IPC handle); the caller all-gathers the handles
 * ([world][64], rank order) and passes them back. With several workers per
 * GPU the speed all-gather and gradient all-reduce then run as peer-memory
 * kernels (rank-ordered, deterministic sum) instead of NCCL calls; with one
 * worker per GPU (2 GPUs) the bf16 gradient buckets are pushed by the copy
 * engines into the peers' buffers and summed in rank order.
 * Call before the first lbbsp_mlp_run. */
int lbbsp_mlp_peer_handle(lbbsp_mlp* m, unsigned char h_handle[64]);
int lbbsp_mlp_init_peers(lbbsp_mlp* m, const unsigned char* h_handles);
/* Run `iterations` LB-BSP rounds on the engine stream (no host sync). */
int lbbsp_mlp_run(lbbsp_mlp* m, int iterations);
void* lbbsp_mlp_stream(lbbsp_mlp* m);
/* Stream of the e2e result reads (lbbsp_mlp_read_result_async): a caller that
 * times or synchronises on the engine stream waits on this one too. */
void* lbbsp_mlp_result_stream(lbbsp_mlp* m);
/* Records of the rounds run so far (blocking): [rows][n_total] arrays. */
int lbbsp_mlp_records(lbbsp_mlp* m, int max_rows, int* rows, int* sizes, double* v_pred,
                      double* v_obs, int* caps, double* t_worker, double* loss);
/* Copy the fp32 master parameters (flat, per layer W [out][in] then b [out],
 * each segment padded to 64 elements) and the offsets of each segment. */
int lbbsp_mlp_params(lbbsp_mlp* m, float* h_params, long long* h_offsets, long long* n_params);
int lbbsp_mlp_set_params(lbbsp_mlp* m, const float* h_params);
int lbbsp_mlp_dataset(lbbsp_mlp* m, void* h_x_bf16, int* h_labels);
int lbbsp_mlp_launches_per_iteration(lbbsp_mlp* m, int* launches);
/* End-to-end plumbing (async, pinned host buffers): replace the resident
 * dataset with host rows ([dataset_size][dims[0]] bf16 + labels) before the
 * next round -- the dataset is double-buffered: the host->device copy runs on
 * a copy stream into the buffer the round in flight does not read, and the
 * next round reads it -- and read back the newest round's record (sizes
 * [n_total] ints, then loss) after it. */
int lbbsp_mlp_load_data_async(lbbsp_mlp* m, const void* h_x_bf16, const int* h_labels);
int lbbsp_mlp_read_result_async(lbbsp_mlp* m, int* h_sizes, double* h_loss);
/* load_data_async + one round + read_result_async in one call (the e2e step). */
int lbbsp_mlp_step_e2e(lbbsp_mlp* m, const void* h_x_bf16, const int* h_labels, int* h_sizes,
                       double* h_loss);
/* Mean per-phase device time of the rounds run so far: phase p of the last
 * round as {min start, max end} over workers (globaltimer ns); n_phases out. */
int lbbsp_mlp_phase_times(lbbsp_mlp* m, double* h_phase_ns, int* n_phases);
/* Per-worker device time of each phase of the last round: h_ns[p*n_local+i]. */
int lbbsp_mlp_worker_phase_times(lbbsp_mlp* m, double* h_ns, int* n_phases);
/* algorithmic work of one round on this rank: GEMM flops, reduction bytes */
int lbbsp_mlp_work(lbbsp_mlp* m, double* gemm_flops, double* reduce_bytes);
/* Rows one CTA of a worker's partition covers per tile wave (64: the fused
 * pair kernel, two CTAs per 128-row tile; 128: one CTA per tile). A worker
 * with cap CTAs runs ceil(b / (cap * rows_per_cta)) waves. */
int lbbsp_mlp_rows_per_cta(lbbsp_mlp* m, int* rows);

#ifdef __cplusplus
}
#endif

#endif /* LBBSP_C_H */
