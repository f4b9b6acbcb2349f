// kernels.cuh -- kernel launchers shared between the C-ABI (capi.cu) and the
// fused iteration driver (sim.cu).
#pragma once
#include "common.cuh"

namespace lbbsp {

// Simulation device state (Simulation, cluster_sim.hpp:197-258), all
// pointers device-resident. Passed by value to every iteration kernel.
struct SimDev {
  // SimConfig scalars
  int n, B, N, d;
  int scheme, gpu_mode, dyn_kind;
  double base_speed, lr, conv_loss;
  int conv_consec;
  long long max_updates;
  unsigned long long seed;
  // dynamics
  const double* static_cpu;  // [n]
  const double* static_mem;  // [n]
  const lbbsp_straggler* strag;
  const double* phase;       // [n]
  int bench_len;
  const double* bcpu;        // [n][bench_len]
  const double* bmem;
  const double* bmult;
  const int* trace_off;      // [n+1] (Trace dynamics)
  const double* trace_t;
  const double* trace_c;
  const double* trace_m;
  // comm model
  double base_comm;
  int bw_worker;
  long long bw_at;
  double bw_factor;
  const lbbsp_gpu_profile* prof;  // [n] or null
  const int* equal;               // [n] equal_split
  // iteration state
  long long* k;
  int* done;
  int* active;
  int* converged;
  int* below;
  int* rows;
  int* train_first;
  // per-iteration scratch
  double* c_now;
  double* m_now;
  double* vact;
  double* vpred;
  double* tp;
  double* tm;
  int* sizes;
  int* offsets;
  double* wall;
  double* now;  // simulated clock (Simulation::now_, cluster_sim.cpp:466)
  // workload (reference logistic regression, fp64)
  const double* feat;  // [N][d]
  const double* lab;   // [N]
  double* params;      // [d]
  double* grads;       // [n][d]
  double* agg;         // [d]
  const int* streams;  // [max_updates][B] pre-generated sample streams
  // records
  lbbsp_iter_scalars* rec_sc;
  int* rec_batch;
  double *rec_tp, *rec_tm, *rec_wait, *rec_vpred, *rec_vact, *rec_params;
  lbbsp_dev_status* status;
  PredDev pred;
};

// Event-driven ASP/SSP state (Simulation::step_async, cluster_sim.cpp:486-631):
// per-worker runtime (WorkerRuntime async fields, cluster_sim.hpp:209-224),
// the SSP round buffers and the per-row worker lists of the records.
struct AsyncDev {
  int ssp;           // 0: ASP, 1: SSP
  long long stale;   // staleness_threshold
  int ring;          // SSP round-buffer slots
  int n_streams;     // pre-generated local-iteration streams
  int* started;      // device flag: workers launched at t = 0
  long long* completed;
  int* running;
  int* blocked;
  int* hist_len;     // per-worker SpeedHistory length
  double* block_start;
  double* pending_wait;
  double* finish;
  double* inflight_grad;  // [n][d]
  double* inflight;       // [n][8]: x, tp, tm, wait, v_pred, v_act, c, m
  double* ring_grads;     // [ring][n][d]
  double* ring_stats;     // [ring][n][6]
  int* ring_count;        // [ring]
  double* last_update;
  long long* clock;       // ModelState::clock
  long long* max_skew;
  int* rec_worker;        // [rows][n] worker id of each record slot
  int* rec_nw;            // [rows] stats per record (1 for ASP, n for SSP)
};

// ---- launchers (return cudaError_t) -----------------------------------------
cudaError_t launch_solve_prop(const double* d_speeds, int n, int budget, double speed_floor,
                              int* d_sizes, lbbsp_dev_status* d_status, cudaStream_t s);
cudaError_t launch_solve_gpu(const lbbsp_gpu_profile* d_prof, const double* d_comm, int n,
                             int budget, int* d_sizes, lbbsp_dev_status* d_status,
                             cudaStream_t s);
cudaError_t launch_ema(const double* d_series, int len, double alpha, double* d_out,
                       cudaStream_t s);
cudaError_t launch_narx_predict(const lbbsp_narx_model* d_model, const double* d_in /*8*/,
                                double floor, double* d_out, cudaStream_t s);
cudaError_t launch_narx_train_one(lbbsp_narx_model* d_model, const double* d_v, const double* d_c,
                                  const double* d_m, int len, lbbsp_narx_train_cfg cfg,
                                  lbbsp_narx_report* d_rep, double* d_loss_log, int loss_cap,
                                  double* d_scratch, cudaStream_t s);
cudaError_t launch_pred_observe(const PredDev& P, const double* d_v, const double* d_c,
                                const double* d_m, const double* d_tm, cudaStream_t s);
cudaError_t launch_pred_predict(const PredDev& P, const double* d_c, const double* d_m,
                                double* d_out, cudaStream_t s);
cudaError_t launch_pred_train(const PredDev& P, int rotation, cudaStream_t s);
cudaError_t launch_sample_streams(unsigned long long seed, long long k0, int iters, int budget,
                                  int dataset_size, int* d_out, cudaStream_t s);
cudaError_t launch_lr_worker_grads(const double* feat, const double* lab, int N, int d,
                                   const double* params, const int* idx, const int* sizes,
                                   int n_seg, double* grads, lbbsp_dev_status* st,
                                   cudaStream_t s);
cudaError_t launch_aggregate_apply(const double* grads, const int* sizes, int n, int d,
                                   int weighted, double lr, double* params, double* agg,
                                   double* norm, lbbsp_dev_status* st, cudaStream_t s);
cudaError_t launch_lr_loss(const double* feat, const double* lab, int N, int d,
                           const double* params, double* out, cudaStream_t s);
cudaError_t launch_sim_iteration(const SimDev& S, cudaStream_t s, int* launches);
// ASP/SSP: up to `updates` records in one persistent CTA (no host round trip).
cudaError_t launch_async_sim(const SimDev& S, const AsyncDev& A, int updates, cudaStream_t s);
size_t async_smem_bytes(int max_hist);
// compute_metrics (cluster_sim.cpp:217-245) over the device-resident records;
// out = {time_total.., see kernels.cu}; scratch: 2*rows*n doubles.
cudaError_t launch_sim_metrics(const SimDev& S, const int* rec_nw, int rmse_from, double* scratch,
                               lbbsp_metrics* out, cudaStream_t s);
// predictor_series_rmse (cluster_sim.cpp:645-672): P has n == 1 and history
// capacity >= len; writes {sse, count} to out2.
cudaError_t launch_series_rmse(const PredDev& P, const double* cpu, const double* mem,
                               const double* mult, int len, double base_speed, int measure_from,
                               double* out2, cudaStream_t s);

size_t train_smem_bytes(int max_hist);

}  // namespace lbbsp
