// kernels.cu -- sm_100a kernels of the LB-BSP hot path (K1-K10 of SURVEY 2.3)
// and the fused iteration (A1 step_sync, cluster_sim.cpp:349-469).
//
// These kernels are latency-bound by construction (n <= 1024 workers, fp64
// sequential reductions pinned by the reference); their measure is us/call
// and zero host synchronisations. The bandwidth/tensor-bound
// work of the hot path lives in mlp.cu / gemm_tc.cuh.
#include <algorithm>

#include "exactmath.cuh"
#include "kernels.cuh"
#include "predictor.cuh"
#include "solver.cuh"

namespace lbbsp {

constexpr int kSolverThreads = 256;
constexpr int kMaxSolverN = 4096;

// ---------------------------------------------------------------------------
// K1 / K2 standalone
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSolverThreads) solve_prop_kernel(
    const double* __restrict__ speeds, int n, int budget, double speed_floor, int* sizes,
    lbbsp_dev_status* st) {
  extern __shared__ double sm_d[];
  __shared__ SolverSmem sm;
  __shared__ int sz[kMaxSolverN];
  block_cpu_allocate(speeds, n, budget, speed_floor, sz, sm_d, &sm, st);
  for (int i = threadIdx.x; i < n; i += blockDim.x) sizes[i] = sz[i];
}

__global__ void __launch_bounds__(kSolverThreads) solve_gpu_kernel(
    const lbbsp_gpu_profile* __restrict__ prof_g, const double* __restrict__ comm_g, int n,
    int budget, int* sizes, lbbsp_dev_status* st) {
  extern __shared__ double sm_d[];
  __shared__ SolverSmem sm;
  lbbsp_gpu_profile* prof = reinterpret_cast<lbbsp_gpu_profile*>(sm_d);
  double* comm = reinterpret_cast<double*>(prof + n);
  double* bp = comm + n;
  double* tmp = bp + 2 * n;
  int* sz = reinterpret_cast<int*>(tmp + 2 * n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    prof[i] = prof_g[i];
    comm[i] = comm_g[i];
  }
  __syncthreads();
  block_gpu_allocate(prof, comm, n, budget, sz, bp, tmp, &sm, st);
  for (int i = threadIdx.x; i < n; i += blockDim.x) sizes[i] = sz[i];
}

static size_t gpu_solver_smem(int n) {
  return static_cast<size_t>(n) * sizeof(lbbsp_gpu_profile) + static_cast<size_t>(n) * 8 * 5 +
         static_cast<size_t>(n) * 4 + 64;
}

cudaError_t launch_solve_prop(const double* d_speeds, int n, int budget, double speed_floor,
                              int* d_sizes, lbbsp_dev_status* d_status, cudaStream_t s) {
  if (n > kMaxSolverN) return cudaErrorInvalidValue;
  solve_prop_kernel<<<1, kSolverThreads, sizeof(double) * std::max(n, 1), s>>>(
      d_speeds, n, budget, speed_floor, d_sizes, d_status);
  return cudaGetLastError();
}

cudaError_t launch_solve_gpu(const lbbsp_gpu_profile* d_prof, const double* d_comm, int n,
                             int budget, int* d_sizes, lbbsp_dev_status* d_status,
                             cudaStream_t s) {
  const size_t smem = gpu_solver_smem(std::max(n, 1));
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(solve_gpu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  }
  solve_gpu_kernel<<<1, kSolverThreads, smem, s>>>(d_prof, d_comm, n, budget, d_sizes, d_status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K3/K4/K5 standalone (reference free functions)
// ---------------------------------------------------------------------------
__global__ void ema_kernel(const double* __restrict__ s, int len, double alpha, double* out) {
  if (threadIdx.x == 0) {  // predictor.cpp:18-25, left-to-right fold
    double v = s[0];
    const double oma = dsub(1.0, alpha);
    for (int k = 1; k < len; ++k) v = dadd(dmul(alpha, s[k]), dmul(oma, v));
    *out = v;
  }
}

cudaError_t launch_ema(const double* d_series, int len, double alpha, double* d_out,
                       cudaStream_t s) {
  ema_kernel<<<1, 32, 0, s>>>(d_series, len, alpha, d_out);
  return cudaGetLastError();
}

__global__ void narx_predict_kernel(const lbbsp_narx_model* m, const double* in, double floor_,
                                    double* out) {
  if (threadIdx.x == 0)
    *out = narx_predict_d(*m, in[0], in[1], in[2], in[3], in[4], in[5], in[6], in[7], floor_);
}

cudaError_t launch_narx_predict(const lbbsp_narx_model* d_model, const double* d_in, double floor,
                                double* d_out, cudaStream_t s) {
  narx_predict_kernel<<<1, 32, 0, s>>>(d_model, d_in, floor, d_out);
  return cudaGetLastError();
}

constexpr size_t kTrainSmemCap = 200 * 1024;

size_t train_smem_bytes(int max_hist) {
  return std::min(narx_train_scratch_bytes(max_hist), kTrainSmemCap);
}

__global__ void __launch_bounds__(kTrainThreads) narx_train_one_kernel(
    lbbsp_narx_model* m, const double* v, const double* c, const double* mm, int len,
    lbbsp_narx_train_cfg cfg, lbbsp_narx_report* rep, double* loss_log, int loss_cap,
    double* gscratch, size_t smem_bytes) {
  extern __shared__ double sm_d[];
  __shared__ NarxTrainSmem s;
  size_t nd = 0;
  double* buf = narx_train_buf(len, sm_d, smem_bytes, gscratch,
                               narx_train_scratch_bytes(len) / sizeof(double), &nd);
  narx_train_block(m, v, c, mm, len, cfg, rep, loss_log, loss_cap, buf, nd, &s);
}

cudaError_t launch_narx_train_one(lbbsp_narx_model* d_model, const double* d_v, const double* d_c,
                                  const double* d_m, int len, lbbsp_narx_train_cfg cfg,
                                  lbbsp_narx_report* d_rep, double* d_loss_log, int loss_cap,
                                  double* d_scratch, cudaStream_t s) {
  const size_t smem = train_smem_bytes(len);
  cudaFuncSetAttribute(narx_train_one_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kTrainSmemCap));
  narx_train_one_kernel<<<1, kTrainThreads, smem, s>>>(d_model, d_v, d_c, d_m, len, cfg, d_rep,
                                                        d_loss_log, loss_cap, d_scratch, smem);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Predictor bank (SpeedPredictor x n, device-resident histories)
// ---------------------------------------------------------------------------
__global__ void pred_observe_kernel(PredDev P, const double* v, const double* c, const double* m,
                                    const double* tm) {
  const int len = *P.len;
  for (int w = threadIdx.x + blockIdx.x * blockDim.x; w < P.n; w += blockDim.x * gridDim.x)
    observe_d(P, w, len, v[w], c[w], m[w], tm ? tm[w] : 0.0);
}

__global__ void pred_len_bump_kernel(PredDev P) {
  if (threadIdx.x == 0) *P.len += 1;
}

cudaError_t launch_pred_observe(const PredDev& P, const double* d_v, const double* d_c,
                                const double* d_m, const double* d_tm, cudaStream_t s) {
  const int blocks = (P.n + 255) / 256;
  pred_observe_kernel<<<blocks, 256, 0, s>>>(P, d_v, d_c, d_m, d_tm);
  pred_len_bump_kernel<<<1, 32, 0, s>>>(P);
  return cudaGetLastError();
}

__global__ void pred_predict_kernel(PredDev P, const double* c, const double* m, double* out) {
  const int len = *P.len;
  for (int w = threadIdx.x + blockIdx.x * blockDim.x; w < P.n; w += blockDim.x * gridDim.x)
    out[w] = len >= 1 ? predictor_predict_d(P, w, len, c[w], m[w]) : 0.0;
}

cudaError_t launch_pred_predict(const PredDev& P, const double* d_c, const double* d_m,
                                double* d_out, cudaStream_t s) {
  pred_predict_kernel<<<(P.n + 255) / 256, 256, 0, s>>>(P, d_c, d_m, d_out);
  return cudaGetLastError();
}

// rotation != 0: train_rotation (cluster_sim.cpp:315-324), ceil(n/2) models
// from the cursor; rotation == 0: every model.
__global__ void __launch_bounds__(kTrainThreads) pred_train_kernel(PredDev P, int rotation,
                                                                   const int* active,
                                                                   const int* first_slot,
                                                                   size_t smem_bytes) {
  if (active && !*active) return;
  extern __shared__ double sm_d[];
  __shared__ NarxTrainSmem s;
  const int first = rotation ? (first_slot ? *first_slot : *P.cursor) : 0;
  const int w = (first + blockIdx.x) % P.n;
  const int len = *P.len;
  const int L = len < P.max_hist ? len : P.max_hist;
  const size_t slot = narx_train_scratch_bytes(P.max_hist) / sizeof(double);
  size_t nd = 0;
  double* buf = narx_train_buf(L, sm_d, smem_bytes, P.scratch + blockIdx.x * slot, slot, &nd);
  lbbsp_narx_train_cfg cfg = P.train;
  cfg.min_history = P.warmup;
  const size_t o = static_cast<size_t>(w) * P.max_hist;
  narx_train_block(&P.models[w], P.hv + o, P.hc + o, P.hm + o, L, cfg, &P.reports[w], nullptr, 0,
                   buf, nd, &s);
}

cudaError_t launch_pred_train_from(const PredDev& P, const int* first_slot, cudaStream_t s) {
  if (P.kind != LBBSP_PRED_NARX) return cudaSuccess;
  const size_t smem = train_smem_bytes(P.max_hist);
  cudaFuncSetAttribute(pred_train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kTrainSmemCap));
  pred_train_kernel<<<(P.n + 1) / 2, kTrainThreads, smem, s>>>(P, 1, nullptr, first_slot, smem);
  return cudaGetLastError();
}

__global__ void pred_cursor_kernel(PredDev P) {
  if (threadIdx.x == 0) *P.cursor = (*P.cursor + (P.n + 1) / 2) % P.n;
}

cudaError_t launch_pred_train(const PredDev& P, int rotation, cudaStream_t s) {
  if (P.kind != LBBSP_PRED_NARX) return cudaSuccess;
  const size_t smem = train_smem_bytes(P.max_hist);
  cudaFuncSetAttribute(pred_train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kTrainSmemCap));
  const int blocks = rotation ? (P.n + 1) / 2 : P.n;
  pred_train_kernel<<<blocks, kTrainThreads, smem, s>>>(P, rotation, nullptr, nullptr, smem);
  if (rotation) pred_cursor_kernel<<<1, 32, 0, s>>>(P);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K6 sample streams: one CTA per iteration regenerates
// mt19937_64(mix_seed(seed, 0x57e3a9, k)) with the twist split into its three
// data-parallel phases; every (seed, k) stream is independent, so the whole
// run's streams are produced ahead of time, off the iteration's critical path.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(320) sample_stream_kernel(unsigned long long seed, long long k0,
                                                            int budget, int dataset_size,
                                                            int* out) {
  __shared__ uint64_t mt[312];
  const int tid = threadIdx.x;
  const long long k = k0 + blockIdx.x;
  if (tid == 0) {
    uint64_t x = mix_seed(seed, 0x57e3a9ull, static_cast<uint64_t>(k));
    mt[0] = x;
    for (int i = 1; i < 312; ++i) {
      x = 6364136223846793005ull * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
      mt[i] = x;
    }
  }
  __syncthreads();
  int* dst = out + static_cast<size_t>(blockIdx.x) * budget;
  for (int base = 0; base < budget; base += 312) {
    uint64_t nv = 0;
    if (tid < 156) nv = mt64_twist_one(mt[tid], mt[tid + 1], mt[tid + 156]);
    __syncthreads();
    if (tid < 156) mt[tid] = nv;
    __syncthreads();
    if (tid >= 156 && tid < 311) nv = mt64_twist_one(mt[tid], mt[tid + 1], mt[tid - 156]);
    __syncthreads();
    if (tid >= 156 && tid < 311) mt[tid] = nv;
    __syncthreads();
    if (tid == 311) mt[311] = mt64_twist_one(mt[311], mt[0], mt[155]);
    __syncthreads();
    if (tid < 312 && base + tid < budget)
      dst[base + tid] = uniform_int_from(mt64_temper(mt[tid]), 0, dataset_size);
    __syncthreads();
  }
}

cudaError_t launch_sample_streams(unsigned long long seed, long long k0, int iters, int budget,
                                  int dataset_size, int* d_out, cudaStream_t s) {
  if (iters <= 0) return cudaSuccess;
  sample_stream_kernel<<<iters, 320, 0, s>>>(seed, k0, budget, dataset_size, d_out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K7 logistic-regression worker gradients (sgd.cpp:72-90), fp64, with the
// reference's per-dimension left-to-right accumulation over each segment.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double sigmoid_d(double z) {  // sgd.cpp:26-30
  if (z >= 0) return ddiv(1.0, dadd(1.0, exp(-z)));
  const double e = exp(z);
  return ddiv(e, dadd(1.0, e));
}

constexpr int kGradChunk = 1024;

__device__ void lr_segment_grad(const double* __restrict__ feat, const double* __restrict__ lab,
                                int N, int d, const double* __restrict__ params,
                                const int* __restrict__ idx, int count, double* g,
                                lbbsp_dev_status* st, double* coeff /*smem kGradChunk*/) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  if (count <= 0) {
    if (threadIdx.x == 0) set_status(st, LBBSP_INVALID_ARGUMENT, LBBSP_E_GRAD_EMPTY, 0, 0);
    return;
  }
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // thread j accumulates dims j, j+nt, ... (d <= 4*nt)
  for (int base = 0; base < count; base += kGradChunk) {
    const int m = min(kGradChunk, count - base);
    for (int t = threadIdx.x; t < m; t += blockDim.x) {
      const int i = idx[base + t];
      if (i < 0 || i >= N) {
        bad = 1;
        coeff[t] = 0.0;
        continue;
      }
      const double* x = feat + static_cast<size_t>(i) * d;
      double z = 0.0;
      for (int j = 0; j < d; ++j) z = dadd(z, dmul(params[j], x[j]));  // dot, sgd.cpp:14-18
      coeff[t] = dsub(sigmoid_d(z), lab[i]);
    }
    __syncthreads();
    if (bad) break;
    for (int r = 0; r < 4; ++r) {
      const int j = threadIdx.x + r * blockDim.x;
      if (j >= d) break;
      double a = acc[r];
      for (int t = 0; t < m; ++t)
        a = dadd(a, dmul(coeff[t], feat[static_cast<size_t>(idx[base + t]) * d + j]));
      acc[r] = a;
    }
    __syncthreads();
  }
  if (bad) {
    if (threadIdx.x == 0) set_status(st, LBBSP_OUT_OF_RANGE, LBBSP_E_GRAD_INDEX, 0, 0);
    return;
  }
  const double inv = ddiv(1.0, static_cast<double>(count));
  for (int r = 0; r < 4; ++r) {
    const int j = threadIdx.x + r * blockDim.x;
    if (j < d) g[j] = dmul(acc[r], inv);
  }
}

__global__ void __launch_bounds__(256) lr_worker_grads_kernel(
    const double* __restrict__ feat, const double* __restrict__ lab, int N, int d,
    const double* __restrict__ params, const int* __restrict__ idx, const int* __restrict__ sizes,
    double* grads, lbbsp_dev_status* st) {
  __shared__ double coeff[kGradChunk];
  __shared__ int off;
  const int w = blockIdx.x;
  if (threadIdx.x == 0) {
    int o = 0;
    for (int i = 0; i < w; ++i) o += sizes[i];
    off = o;
  }
  __syncthreads();
  lr_segment_grad(feat, lab, N, d, params, idx + off, sizes[w], grads + static_cast<size_t>(w) * d,
                  st, coeff);
}

cudaError_t launch_lr_worker_grads(const double* feat, const double* lab, int N, int d,
                                   const double* params, const int* idx, const int* sizes,
                                   int n_seg, double* grads, lbbsp_dev_status* st,
                                   cudaStream_t s) {
  if (d > 4 * 256) return cudaErrorInvalidValue;
  lr_worker_grads_kernel<<<n_seg, 256, 0, s>>>(feat, lab, N, d, params, idx, sizes, grads, st);
  return cudaGetLastError();
}

// K8/K9: aggregate_weighted | aggregate_naive (coordination.cpp:39-68) fused
// with apply_update (sgd.cpp:92-99) and l2_norm (cluster_sim.cpp:203-207).
__device__ void block_aggregate_apply(const double* __restrict__ grads, const int* __restrict__ sizes,
                                      int n, int d, int weighted, double lr, double* params,
                                      double* agg, double* norm, lbbsp_dev_status* st) {
  __shared__ double total;
  __shared__ int badb;
  if (threadIdx.x == 0) {
    double t = 0.0;
    int b = 0;
    for (int i = 0; i < n; ++i) {
      if (sizes[i] < 1) b = 1;
      t = dadd(t, static_cast<double>(sizes[i]));
    }
    total = t;
    badb = b;
    if (b && weighted) set_status(st, LBBSP_INVALID_ARGUMENT, LBBSP_E_AGG_BATCH, 0, 0);
  }
  __syncthreads();
  if (badb && weighted) return;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double out = 0.0;
    if (weighted) {
      for (int i = 0; i < n; ++i)
        out = dadd(out, dmul(ddiv(static_cast<double>(sizes[i]), total),
                             grads[static_cast<size_t>(i) * d + j]));
    } else {
      for (int i = 0; i < n; ++i) out = dadd(out, grads[static_cast<size_t>(i) * d + j]);
      out = dmul(out, ddiv(1.0, static_cast<double>(n)));
    }
    if (agg) agg[j] = out;
    if (params) params[j] = dsub(params[j], dmul(lr, out));
  }
  __syncthreads();
  if (norm && threadIdx.x == 0) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s = dadd(s, dmul(agg[j], agg[j]));
    *norm = __dsqrt_rn(s);
  }
  __syncthreads();
}

__global__ void aggregate_apply_kernel(const double* grads, const int* sizes, int n, int d,
                                       int weighted, double lr, double* params, double* agg,
                                       double* norm, lbbsp_dev_status* st) {
  block_aggregate_apply(grads, sizes, n, d, weighted, lr, params, agg, norm, st);
}

cudaError_t launch_aggregate_apply(const double* grads, const int* sizes, int n, int d,
                                   int weighted, double lr, double* params, double* agg,
                                   double* norm, lbbsp_dev_status* st, cudaStream_t s) {
  aggregate_apply_kernel<<<1, 256, 0, s>>>(grads, sizes, n, d, weighted, lr, params, agg, norm, st);
  return cudaGetLastError();
}

// K10: loss (sgd.cpp:65-70) -- per-sample terms in parallel, the reference's
// left-to-right total by one thread.
__device__ __forceinline__ double log1p_exp_d(double z) {  // sgd.cpp:20-24
  if (z > 0) return dadd(z, log1p(exp(-z)));
  return log1p(exp(z));
}

constexpr int kLossChunk = 2048;

__device__ double block_lr_loss(const double* __restrict__ feat, const double* __restrict__ lab,
                                int N, int d, const double* __restrict__ params, double* terms) {
  __shared__ double total;
  if (threadIdx.x == 0) total = 0.0;
  __syncthreads();
  for (int base = 0; base < N; base += kLossChunk) {
    const int m = min(kLossChunk, N - base);
    for (int t = threadIdx.x; t < m; t += blockDim.x) {
      const double* x = feat + static_cast<size_t>(base + t) * d;
      double z = 0.0;
      for (int j = 0; j < d; ++j) z = dadd(z, dmul(params[j], x[j]));
      terms[t] = dsub(log1p_exp_d(z), dmul(lab[base + t], z));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = total;
      for (int t = 0; t < m; ++t) s = dadd(s, terms[t]);
      total = s;
    }
    __syncthreads();
  }
  return ddiv(total, static_cast<double>(N));
}

__global__ void __launch_bounds__(512) lr_loss_kernel(const double* feat, const double* lab, int N,
                                                      int d, const double* params, double* out) {
  __shared__ double terms[kLossChunk];
  const double l = block_lr_loss(feat, lab, N, d, params, terms);
  if (threadIdx.x == 0) *out = l;
}

cudaError_t launch_lr_loss(const double* feat, const double* lab, int N, int d,
                           const double* params, double* out, cudaStream_t s) {
  lr_loss_kernel<<<1, 512, 0, s>>>(feat, lab, N, d, params, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// A1: the fused iteration. Four kernels per round, no host round trip:
//   sim_plan    P1-P5   dynamics, prediction, batch sizes, timing, record
//   sim_grad    P7      per-worker gradients over the pre-generated stream
//   sim_update  P8-P10  aggregate+apply, norm, loss, check_stop, observe
//   pred_train  P10     NARX train_rotation, one CTA per model
// ---------------------------------------------------------------------------
__device__ void dyn_at_d(const SimDev& S, int w, long long k, double now, double* c, double* m,
                         double* mult) {
  *c = 1.0;
  *m = 1.0;
  *mult = 1.0;
  switch (S.dyn_kind) {  // Dynamics::at, cluster_sim.cpp:77-118
    case LBBSP_DYN_STATIC:
      if (S.static_cpu) *c = S.static_cpu[w];
      if (S.static_mem) *m = S.static_mem[w];
      return;
    case LBBSP_DYN_STRAGGLER: {
      if (!S.strag) return;
      const lbbsp_straggler sp = S.strag[w];
      if (sp.on_probability <= 0.0) return;
      const double q = static_cast<double>(k / (sp.period > 1 ? sp.period : 1));
      const double ph = S.phase[w];
      const bool on = floor(dmul(dadd(dadd(q, 1.0), ph), sp.on_probability)) >
                      floor(dmul(dadd(q, ph), sp.on_probability));
      if (on) {
        *c = dsub(1.0, sp.cpu_consumed);
        *m = dsub(1.0, sp.mem_consumed);
      }
      return;
    }
    case LBBSP_DYN_BENCHMARK: {
      const long long idx = k < S.bench_len - 1 ? k : S.bench_len - 1;
      const size_t o = static_cast<size_t>(w) * S.bench_len + idx;
      *c = S.bcpu[o];
      *m = S.bmem[o];
      *mult = S.bmult[o];
      return;
    }
    case LBBSP_DYN_TRACE: {  // trace_at (trace.cpp:137-143): last point at or before now
      int lo = S.trace_off[w], hi = S.trace_off[w + 1];  // upper_bound over [lo, hi)
      const int first = lo;
      while (lo < hi) {
        const int mid = lo + (hi - lo) / 2;
        if (now < S.trace_t[mid])
          hi = mid;
        else
          lo = mid + 1;
      }
      const int p = lo > first ? lo - 1 : first;
      *c = S.trace_c[p];
      *m = S.trace_m[p];
      return;
    }
  }
}

__global__ void __launch_bounds__(kSolverThreads) sim_plan_kernel(SimDev S) {
  extern __shared__ double sm_d[];
  __shared__ SolverSmem sm;
  __shared__ int active;
  if (threadIdx.x == 0) {
    active = !*S.done;
    *S.active = active;
  }
  __syncthreads();
  if (!active) return;
  const int n = S.n, tid = threadIdx.x;
  const long long k = *S.k;
  const int len = *S.pred.len;
  const double now = *S.now;
  // P1-P3 (cluster_sim.cpp:355-367)
  for (int i = tid; i < n; i += blockDim.x) {
    double c, m, mult;
    dyn_at_d(S, i, k, now, &c, &m, &mult);
    S.c_now[i] = c;
    S.m_now[i] = m;
    double va = 0.0, vp = 0.0;
    if (!S.gpu_mode) {
      const double pen = m >= 0.5 ? 1.0 : dadd(0.25, dmul(0.75, ddiv(m, 0.5)));  // :22-29
      va = dmul(dmul(dmul(S.base_speed, c), pen), mult);
      if (len >= 1)
        vp = S.pred.kind == LBBSP_PRED_PERFECT ? va : predictor_predict_d(S.pred, i, len, c, m);
    }
    S.vact[i] = va;
    S.vpred[i] = vp;
  }
  __syncthreads();
  // P4 sizes (:371-402)
  int code = 0;
  lbbsp_gpu_profile* prof = reinterpret_cast<lbbsp_gpu_profile*>(sm_d);
  double* comm = reinterpret_cast<double*>(prof + n);
  double* bp = comm + n;
  double* tmp = bp + 2 * n;
  if (S.scheme == LBBSP_SCHEME_LBBSP) {
    if (S.gpu_mode) {
      for (int i = tid; i < n; i += blockDim.x) {
        prof[i] = S.prof[i];
        comm[i] = k < 2 ? 0.0 : S.pred.comm_ema_lag[i];
        S.sizes[i] = S.equal[i];
      }
      __shared__ int feasible;
      if (tid == 0) feasible = 1;
      __syncthreads();
      if (k < 2) {  // initial_gpu_sizes (:471-484)
        for (int i = tid; i < n; i += blockDim.x)
          if (S.equal[i] < prof[i].saturation_point || S.equal[i] > prof[i].oom_point) feasible = 0;
        __syncthreads();
      }
      if (k >= 2 || !feasible)
        code = block_gpu_allocate(prof, comm, n, S.B, S.sizes, bp, tmp, &sm, S.status);
    } else if (k == 0) {
      for (int i = tid; i < n; i += blockDim.x) S.sizes[i] = S.equal[i];
    } else {
      code = block_cpu_allocate(S.vpred, n, S.B, S.pred.floor, S.sizes, bp, &sm, S.status);
    }
  } else {
    for (int i = tid; i < n; i += blockDim.x) S.sizes[i] = S.equal[i];
  }
  __syncthreads();
  if (code) {
    if (tid == 0) {
      *S.done = 1;
      *S.active = 0;
    }
    return;
  }
  // P5 timing (:404-420)
  __shared__ int bad_oom;
  if (tid == 0) bad_oom = 0;
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) {
    const int x = S.sizes[i];
    double tp;
    if (S.gpu_mode) {
      const lbbsp_gpu_profile p = S.prof[i];
      if (x < 1 || x > p.oom_point) {
        bad_oom = 1;
        set_status(S.status, LBBSP_RUNTIME, LBBSP_E_GPU_OOM, x, p.oom_point);
      }
      tp = dadd(dmul(p.sec_per_sample, static_cast<double>(x > p.saturation_point ? x : p.saturation_point)),
                p.base_time_s);
      S.vact[i] = ddiv(static_cast<double>(x), tp);
    } else {
      tp = ddiv(static_cast<double>(x), S.vact[i]);
    }
    const double f = (S.bw_worker == i && S.bw_at <= k) ? S.bw_factor : 1.0;  // tm_at :13-20
    S.tp[i] = tp;
    S.tm[i] = dmul(S.base_comm, f);
  }
  __syncthreads();
  if (bad_oom) {
    if (tid == 0) {
      *S.done = 1;
      *S.active = 0;
    }
    return;
  }
  if (tid == 0) {
    double wall = 0.0;
    int o = 0;
    for (int i = 0; i < n; ++i) {
      const double t = dadd(S.tp[i], S.tm[i]);
      wall = wall > t ? wall : t;
      S.offsets[i] = o;
      o += S.sizes[i];
    }
    *S.wall = wall;
    const int row = *S.rows;
    S.rec_sc[row].k = k;
    S.rec_sc[row].wall_s = wall;
  }
  __syncthreads();
  const int row = *S.rows;
  const double wall = *S.wall;
  for (int i = tid; i < n; i += blockDim.x) {
    const size_t o = static_cast<size_t>(row) * n + i;
    S.rec_batch[o] = S.sizes[i];
    S.rec_tp[o] = S.tp[i];
    S.rec_tm[o] = S.tm[i];
    S.rec_wait[o] = dsub(dsub(wall, S.tp[i]), S.tm[i]);
    S.rec_vpred[o] = S.vpred[i];
    S.rec_vact[o] = S.vact[i];
  }
}

__global__ void __launch_bounds__(256) sim_grad_kernel(SimDev S) {
  if (!*S.active) return;
  __shared__ double coeff[kGradChunk];
  const int w = blockIdx.x;
  const long long k = *S.k;
  const int* idx = S.streams + static_cast<size_t>(*S.rows) * S.B + S.offsets[w];
  lr_segment_grad(S.feat, S.lab, S.N, S.d, S.params, idx, S.sizes[w],
                  S.grads + static_cast<size_t>(w) * S.d, S.status, coeff);
  (void)k;
}

__global__ void __launch_bounds__(512) sim_update_kernel(SimDev S) {
  if (!*S.active) return;
  __shared__ double terms[kLossChunk];
  __shared__ double nrm;
  if (S.status->code != 0) {  // a worker reported a bad index / empty batch
    if (threadIdx.x == 0) {
      *S.done = 1;
      *S.active = 0;
    }
    return;
  }
  block_aggregate_apply(S.grads, S.sizes, S.n, S.d, S.scheme == LBBSP_SCHEME_LBBSP, S.lr, S.params,
                        S.agg, &nrm, S.status);
  const double loss = block_lr_loss(S.feat, S.lab, S.N, S.d, S.params, terms);
  const int row = *S.rows;
  for (int j = threadIdx.x; j < S.d; j += blockDim.x)
    S.rec_params[static_cast<size_t>(row) * S.d + j] = S.params[j];
  const int len = *S.pred.len;
  for (int i = threadIdx.x; i < S.n; i += blockDim.x)
    observe_d(S.pred, i, len, S.vact[i], S.c_now[i], S.m_now[i], S.tm[i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    S.rec_sc[row].grad_norm = nrm;
    S.rec_sc[row].loss = loss;
    *S.pred.len = len + 1;
    *S.train_first = *S.pred.cursor;
    *S.pred.cursor = (*S.pred.cursor + (S.n + 1) / 2) % S.n;
    *S.rows = row + 1;
    *S.k += 1;
    *S.now = dadd(*S.now, *S.wall);  // now_ += wall (cluster_sim.cpp:466)
    // check_stop (cluster_sim.cpp:326-334)
    const int below = loss < S.conv_loss ? *S.below + 1 : 0;
    *S.below = below;
    if (below >= S.conv_consec) {
      *S.converged = 1;
      *S.done = 1;
    }
    if (row + 1 >= S.max_updates) *S.done = 1;
  }
}

cudaError_t launch_sim_iteration(const SimDev& S, cudaStream_t s, int* launches) {
  const size_t plan_smem = gpu_solver_smem(std::max(S.n, 1));
  if (plan_smem > 48 * 1024)
    cudaFuncSetAttribute(sim_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(plan_smem));
  sim_plan_kernel<<<1, kSolverThreads, plan_smem, s>>>(S);
  sim_grad_kernel<<<S.n, 256, 0, s>>>(S);
  sim_update_kernel<<<1, 512, 0, s>>>(S);
  int nl = 3;
  if (S.pred.kind == LBBSP_PRED_NARX) {
    const size_t smem = train_smem_bytes(S.pred.max_hist);
    cudaFuncSetAttribute(pred_train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kTrainSmemCap));
    pred_train_kernel<<<(S.n + 1) / 2, kTrainThreads, smem, s>>>(S.pred, 1, S.active,
                                                                  S.train_first, smem);
    ++nl;
  }
  if (launches) *launches = nl;
  return cudaGetLastError();
}

// compute_metrics (cluster_sim.cpp:217-245) on the device-resident records:
// per-row terms in parallel, then the reference's three sequential folds by
// three threads of warp 0 (time_total, wait fractions, squared errors).
__global__ void __launch_bounds__(256) sim_metrics_kernel(SimDev S, const int* rec_nw, int rmse_from,
                                                          double* wf, double* se, lbbsp_metrics* out) {
  const int rows = *S.rows, n = S.n;
  const size_t total = static_cast<size_t>(rows) * n;
  for (size_t o = threadIdx.x; o < total; o += blockDim.x) {
    const size_t r = o / n;
    const double wall = S.rec_sc[r].wall_s;
    if (rec_nw && static_cast<int>(o % n) >= rec_nw[r]) {  // ASP rows carry one worker
      wf[o] = 0.0;
      se[o] = -2.0;
      continue;
    }
    wf[o] = wall > 0.0 ? ddiv(S.rec_wait[o], wall) : 0.0;
    const double vp = S.rec_vpred[o];
    se[o] = -1.0;  // marks "not counted"
    if (vp > 0.0 && S.rec_sc[r].k >= rmse_from) {
      const double e = dsub(vp, S.rec_vact[o]);
      se[o] = dmul(e, e);
    }
  }
  __syncthreads();
  __shared__ double time_total, wsum, sse;
  __shared__ long long sse_count, row_count;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int r = 0; r < rows; ++r) t = dadd(t, S.rec_sc[r].wall_s);
    time_total = t;
  } else if (threadIdx.x == 1) {
    double a = 0.0;
    long long c = 0;
    for (size_t o = 0; o < total; ++o)
      if (se[o] != -2.0) {
        a = dadd(a, wf[o]);
        ++c;
      }
    wsum = a;
    row_count = c;
  } else if (threadIdx.x == 2) {
    double a = 0.0;
    long long c = 0;
    for (size_t o = 0; o < total; ++o)
      if (se[o] >= 0.0) {
        a = dadd(a, se[o]);
        ++c;
      }
    sse = a;
    sse_count = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    lbbsp_metrics m{};
    m.converged = *S.converged;
    m.updates_to_convergence = rows;
    if (rows > 0) {
      m.mean_per_update_time = ddiv(time_total, static_cast<double>(rows));
      m.wastage = row_count > 0 ? ddiv(wsum, static_cast<double>(row_count)) : 0.0;
      m.predictor_rmse = sse_count > 0 ? __dsqrt_rn(ddiv(sse, static_cast<double>(sse_count))) : 0.0;
    }
    *out = m;
  }
}

cudaError_t launch_sim_metrics(const SimDev& S, const int* rec_nw, int rmse_from, double* scratch,
                               lbbsp_metrics* out, cudaStream_t s) {
  const size_t cap = static_cast<size_t>(S.max_updates) * S.n;
  sim_metrics_kernel<<<1, 256, 0, s>>>(S, rec_nw, rmse_from, scratch, scratch + cap, out);
  return cudaGetLastError();
}

// predictor_series_rmse (cluster_sim.cpp:645-672): one CTA replays the whole
// series -- predict (k >= 1 and k >= measure_from), push, train -- with the
// history, EMA state and NARX model resident; no launch per step.
__global__ void __launch_bounds__(kTrainThreads) series_rmse_kernel(PredDev P, const double* cpu,
                                                                    const double* mem,
                                                                    const double* mult, int len,
                                                                    double base_speed,
                                                                    int measure_from, double* out2,
                                                                    size_t smem_bytes) {
  extern __shared__ double sm_d[];
  __shared__ NarxTrainSmem s;
  __shared__ double sse;
  __shared__ long long count;
  if (threadIdx.x == 0) {
    sse = 0.0;
    count = 0;
  }
  lbbsp_narx_train_cfg cfg = P.train;
  cfg.min_history = P.warmup;
  for (int k = 0; k < len; ++k) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const double c = cpu[k], m = mem[k];
      const double pen = m >= 0.5 ? 1.0 : dadd(0.25, dmul(0.75, ddiv(m, 0.5)));  // :22-29
      const double va = dmul(dmul(dmul(base_speed, c), pen), mult[k]);
      if (k >= 1 && k >= measure_from) {
        const double vp = predictor_predict_d(P, 0, k, c, m);
        const double e = dsub(vp, va);
        sse = dadd(sse, dmul(e, e));
        ++count;
      }
      observe_d(P, 0, k, va, c, m, 0.0);
    }
    __syncthreads();
    if (P.kind == LBBSP_PRED_NARX) {
      const int L = k + 1;
      size_t nd = 0;
      double* buf = narx_train_buf(L, sm_d, smem_bytes, P.scratch,
                                   narx_train_scratch_bytes(P.max_hist) / sizeof(double), &nd);
      narx_train_block(&P.models[0], P.hv, P.hc, P.hm, L, cfg, &P.reports[0], nullptr, 0, buf, nd,
                       &s);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out2[0] = sse;
    out2[1] = static_cast<double>(count);
    *P.len = len;
  }
}

cudaError_t launch_series_rmse(const PredDev& P, const double* cpu, const double* mem,
                               const double* mult, int len, double base_speed, int measure_from,
                               double* out2, cudaStream_t s) {
  const size_t smem = train_smem_bytes(P.max_hist);
  cudaFuncSetAttribute(series_rmse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kTrainSmemCap));
  series_rmse_kernel<<<1, kTrainThreads, smem, s>>>(P, cpu, mem, mult, len, base_speed,
                                                    measure_from, out2, smem);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// ASP / SSP (Simulation::step_async, cluster_sim.cpp:486-631). The event loop
// is inherently sequential -- one worker finishes at a time -- so one
// persistent CTA runs it end to end: earliest-finish selection, observe + NARX
// train of the finisher, the parameter-server update (ASP) or round assembly
// (SSP), the full-dataset loss, the record, and start_worker's gradient for
// the restarted workers. Every value is computed with the reference's
// operations in the reference's order (bit-exact records).
// ---------------------------------------------------------------------------
constexpr int kAsyncThreads = 512;
constexpr size_t kAsyncTrainSmemCap = 180 * 1024;

size_t async_smem_bytes(int max_hist) {
  return std::min(narx_train_scratch_bytes(max_hist), kAsyncTrainSmemCap);
}

// start_worker (cluster_sim.cpp:504-536) for worker w at time now; CTA-wide.
__device__ void async_start_worker(const SimDev& S, const AsyncDev& A, int w, double now,
                                   double* coeff) {
  __shared__ int x_s, off_s;
  __shared__ long long j_s;
  if (threadIdx.x == 0) {
    const long long j = A.completed[w];
    double c, m, mult;
    dyn_at_d(S, w, j, now, &c, &m, &mult);
    const int x = S.equal[w];
    double tp, va, vp = 0.0;
    if (S.gpu_mode) {
      const lbbsp_gpu_profile p = S.prof[w];
      if (x < 1 || x > p.oom_point) set_status(S.status, LBBSP_RUNTIME, LBBSP_E_GPU_OOM, x, p.oom_point);
      tp = dadd(dmul(p.sec_per_sample, static_cast<double>(x > p.saturation_point ? x : p.saturation_point)),
                p.base_time_s);
      va = ddiv(static_cast<double>(x), tp);
    } else {
      const double pen = m >= 0.5 ? 1.0 : dadd(0.25, dmul(0.75, ddiv(m, 0.5)));
      va = dmul(dmul(dmul(S.base_speed, c), pen), mult);
      tp = ddiv(static_cast<double>(x), va);
      if (A.hist_len[w] >= 1)
        vp = S.pred.kind == LBBSP_PRED_PERFECT ? va : predictor_predict_d(S.pred, w, A.hist_len[w], c, m);
    }
    const double f = (S.bw_worker == w && S.bw_at <= j) ? S.bw_factor : 1.0;  // tm_at (:13-20)
    const double tm = dmul(S.base_comm, f);
    double* inf = A.inflight + static_cast<size_t>(w) * 8;
    inf[0] = x;
    inf[1] = tp;
    inf[2] = tm;
    inf[3] = A.pending_wait[w];
    inf[4] = vp;
    inf[5] = va;
    inf[6] = c;
    inf[7] = m;
    A.pending_wait[w] = 0.0;
    A.running[w] = 1;
    A.finish[w] = dadd(dadd(now, tp), tm);
    int off = 0;
    for (int i = 0; i < w; ++i) off += S.equal[i];
    x_s = x;
    off_s = off;
    j_s = j < A.n_streams - 1 ? j : A.n_streams - 1;
  }
  __syncthreads();
  // gradient against the parameters pulled now, over stream(j)[off, off + x)
  const int* idx = S.streams + static_cast<size_t>(j_s) * S.B + off_s;
  lr_segment_grad(S.feat, S.lab, S.N, S.d, S.params, idx, x_s,
                  A.inflight_grad + static_cast<size_t>(w) * S.d, S.status, coeff);
  __syncthreads();
}

__device__ __forceinline__ bool ssp_gate_d(long long clock, long long min_clock, long long s) {
  return clock - min_clock <= s;  // coordination.cpp:70-73
}

__global__ void __launch_bounds__(kAsyncThreads) async_sim_kernel(SimDev S, AsyncDev A, int updates,
                                                                  size_t smem_bytes) {
  extern __shared__ double sm_d[];
  __shared__ double coeff[kGradChunk];
  __shared__ double terms[kLossChunk];
  __shared__ NarxTrainSmem ts;
  __shared__ int next_s, rec_s, stop_s, restart_s;
  __shared__ double nrm;
  const int n = S.n, d = S.d, tid = threadIdx.x;
  if (*S.done) return;
  if (!*A.started) {  // the constructor starts every worker at t = 0 (:293-294)
    for (int w = 0; w < n; ++w) async_start_worker(S, A, w, 0.0, coeff);
    if (tid == 0) *A.started = 1;
    __syncthreads();
  }
  lbbsp_narx_train_cfg tcfg = S.pred.train;
  tcfg.min_history = S.pred.warmup;
  int produced = 0;
  while (produced < updates) {
    if (tid == 0) {
      stop_s = 0;
      rec_s = 0;
      int next = -1;  // earliest finish, ties to the lowest id (:541-548)
      for (int i = 0; i < n; ++i) {
        if (!A.running[i]) continue;
        if (next < 0 || A.finish[i] < A.finish[next]) next = i;
      }
      if (next < 0 || S.status->code) {
        *S.done = 1;
        stop_s = 1;
      } else {
        *S.now = A.finish[next];
        A.running[next] = 0;
        A.completed[next] += 1;
        const double* inf = A.inflight + static_cast<size_t>(next) * 8;
        observe_d(S.pred, next, A.hist_len[next], inf[5], inf[6], inf[7], inf[2]);  // (:309-313)
        A.hist_len[next] += 1;
      }
      next_s = next;
    }
    __syncthreads();
    if (stop_s) break;
    const int w = next_s;
    const double now = *S.now;
    // rt.predictor.train(rt.history) (:558)
    if (S.pred.kind == LBBSP_PRED_NARX) {
      const int L = A.hist_len[w] < S.pred.max_hist ? A.hist_len[w] : S.pred.max_hist;
      const size_t o = static_cast<size_t>(w) * S.pred.max_hist;
      size_t nd = 0;
      double* buf = narx_train_buf(L, sm_d, smem_bytes, S.pred.scratch,
                                   narx_train_scratch_bytes(S.pred.max_hist) / sizeof(double), &nd);
      narx_train_block(&S.pred.models[w], S.pred.hv + o, S.pred.hc + o, S.pred.hm + o, L, tcfg,
                       &S.pred.reports[w], nullptr, 0, buf, nd, &ts);
    }
    __syncthreads();
    const double* inf = A.inflight + static_cast<size_t>(w) * 8;
    if (!A.ssp) {  // ASP: one update, one record (:563-575)
      __shared__ int one;
      if (tid == 0) one = static_cast<int>(inf[0]);
      __syncthreads();
      block_aggregate_apply(A.inflight_grad + static_cast<size_t>(w) * d, &one, 1, d, 0, S.lr,
                            S.params, S.agg, &nrm, S.status);
      const double loss = block_lr_loss(S.feat, S.lab, S.N, d, S.params, terms);
      if (tid == 0) {
        *A.clock += 1;
        const int row = *S.rows;
        S.rec_sc[row].k = *A.clock - 1;
        S.rec_sc[row].grad_norm = nrm;
        S.rec_sc[row].loss = loss;
        S.rec_sc[row].wall_s = dsub(now, *A.last_update);
        *A.last_update = now;
        const size_t o = static_cast<size_t>(row) * n;
        A.rec_worker[o] = w;
        A.rec_nw[row] = 1;
        S.rec_batch[o] = static_cast<int>(inf[0]);
        S.rec_tp[o] = inf[1];
        S.rec_tm[o] = inf[2];
        S.rec_wait[o] = inf[3];
        S.rec_vpred[o] = inf[4];
        S.rec_vact[o] = inf[5];
        rec_s = 1;
      }
    } else {  // SSP: buffer until the round has every worker's update (:577-606)
      __shared__ int slot, full;
      if (tid == 0) {
        const long long round = A.completed[w] - 1;
        slot = static_cast<int>(round % A.ring);
        double* st = A.ring_stats + (static_cast<size_t>(slot) * n + w) * 6;
        for (int q = 0; q < 6; ++q) st[q] = inf[q];
        full = ++A.ring_count[slot] == n;
      }
      __syncthreads();
      double* rg = A.ring_grads + static_cast<size_t>(slot) * n * d;
      for (int j = tid; j < d; j += blockDim.x)
        rg[static_cast<size_t>(w) * d + j] = A.inflight_grad[static_cast<size_t>(w) * d + j];
      __syncthreads();
      if (full) {
        block_aggregate_apply(rg, S.equal, n, d, 0, S.lr, S.params, S.agg, &nrm, S.status);
        const double loss = block_lr_loss(S.feat, S.lab, S.N, d, S.params, terms);
        if (tid == 0) {
          *A.clock += 1;
          const int row = *S.rows;
          S.rec_sc[row].k = *A.clock - 1;
          S.rec_sc[row].grad_norm = nrm;
          S.rec_sc[row].loss = loss;
          S.rec_sc[row].wall_s = dsub(now, *A.last_update);
          *A.last_update = now;
          A.rec_nw[row] = n;
          for (int i = 0; i < n; ++i) {
            const size_t o = static_cast<size_t>(row) * n + i;
            const double* st = A.ring_stats + (static_cast<size_t>(slot) * n + i) * 6;
            A.rec_worker[o] = i;
            S.rec_batch[o] = static_cast<int>(st[0]);
            S.rec_tp[o] = st[1];
            S.rec_tm[o] = st[2];
            S.rec_wait[o] = st[3];
            S.rec_vpred[o] = st[4];
            S.rec_vact[o] = st[5];
          }
          A.ring_count[slot] = 0;
          rec_s = 1;
        }
      }
    }
    __syncthreads();
    // restart or park the finisher, then re-check the blocked workers (:609-626)
    if (!A.ssp) {
      async_start_worker(S, A, w, now, coeff);
    } else {
      for (int i = -1; i < n; ++i) {  // i = -1: the finisher
        if (tid == 0) {
          long long lo = LLONG_MAX;
          for (int q = 0; q < n; ++q) lo = A.completed[q] < lo ? A.completed[q] : lo;
          restart_s = 0;
          if (i < 0) {
            if (ssp_gate_d(A.completed[w], lo, A.stale)) {
              restart_s = 1;
            } else {
              A.blocked[w] = 1;
              A.block_start[w] = now;
            }
          } else if (A.blocked[i] && ssp_gate_d(A.completed[i], lo, A.stale)) {
            A.blocked[i] = 0;
            A.pending_wait[i] = dsub(now, A.block_start[i]);
            restart_s = 1;
          }
        }
        __syncthreads();
        if (restart_s) async_start_worker(S, A, i < 0 ? w : i, now, coeff);
        __syncthreads();
      }
      if (tid == 0) {  // track_skew (:492-502)
        long long hi = LLONG_MIN, lo = LLONG_MAX;
        for (int q = 0; q < n; ++q) {
          const long long c = A.running[q] ? A.completed[q] + 1 : A.completed[q];
          hi = c > hi ? c : hi;
          lo = c < lo ? c : lo;
        }
        *A.max_skew = hi - lo > *A.max_skew ? hi - lo : *A.max_skew;
      }
    }
    __syncthreads();
    if (rec_s) {
      if (tid == 0) {  // records_.push_back + check_stop (:336-347, :326-334)
        const int row = *S.rows;
        for (int j = 0; j < d; ++j) S.rec_params[static_cast<size_t>(row) * d + j] = S.params[j];
        *S.rows = row + 1;
        const double loss = S.rec_sc[row].loss;
        const int below = loss < S.conv_loss ? *S.below + 1 : 0;
        *S.below = below;
        if (below >= S.conv_consec) {
          *S.converged = 1;
          *S.done = 1;
        }
        if (row + 1 >= S.max_updates) *S.done = 1;
        stop_s = *S.done;
      }
      __syncthreads();
      ++produced;
      if (stop_s) break;
    }
  }
}

cudaError_t launch_async_sim(const SimDev& S, const AsyncDev& A, int updates, cudaStream_t s) {
  const size_t smem = async_smem_bytes(S.pred.max_hist);
  cudaFuncSetAttribute(async_sim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kAsyncTrainSmemCap));
  async_sim_kernel<<<1, kAsyncThreads, smem, s>>>(S, A, updates, smem);
  return cudaGetLastError();
}

}  // namespace lbbsp
