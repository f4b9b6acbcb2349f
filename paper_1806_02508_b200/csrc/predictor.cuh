// predictor.cuh -- K3/K4/K5: the speed predictor on device.
//
//   ema state update            : ema / predict_ema / predict_comm_ema
//                                 (predictor.cpp:18-33), incremental but with
//                                 the same operation sequence as the refold
//   narx_predict_d              : standardize + forward + denorm + floor
//                                 (predictor.cpp:52-69, 147-153)
//   predictor_predict_d         : SpeedPredictor::predict (predictor.cpp:271-292)
//   narx_train_block            : narx_train_online (predictor.cpp:155-196),
//                                 one CTA per model, fp64, bit-exact
#pragma once
#include "common.cuh"
#include "exactmath.cuh"

namespace lbbsp {

__device__ __forceinline__ double narx_forward_d(const double* w /*11*/, const double* z) {
  double a = w[8];  // hidden_bias
  for (int j = 0; j < 8; ++j) a = dadd(a, dmul(w[j], z[j]));
  const double h = glibc_tanh(a);
  return dadd(dmul(w[9], h), w[10]);
}

__device__ __forceinline__ void model_weights(const lbbsp_narx_model& m, double* w) {
  for (int j = 0; j < 8; ++j) w[j] = m.input_weights[j];
  w[8] = m.hidden_bias;
  w[9] = m.output_weight;
  w[10] = m.output_bias;
}

// narx_predict, predictor.cpp:147-153
__device__ inline double narx_predict_d(const lbbsp_narx_model& m, double v0, double v1, double c0,
                                 double c1, double c2, double m0, double m1, double m2,
                                 double floor_) {
  double z[8], w[11];
  z[0] = ddiv_std(dsub(v0, m.speed_mean), m.speed_stddev);
  z[1] = ddiv_std(dsub(v1, m.speed_mean), m.speed_stddev);
  z[2] = ddiv_std(dsub(c0, m.cpu_mean), m.cpu_stddev);
  z[3] = ddiv_std(dsub(c1, m.cpu_mean), m.cpu_stddev);
  z[4] = ddiv_std(dsub(c2, m.cpu_mean), m.cpu_stddev);
  z[5] = ddiv_std(dsub(m0, m.mem_mean), m.mem_stddev);
  z[6] = ddiv_std(dsub(m1, m.mem_mean), m.mem_stddev);
  z[7] = ddiv_std(dsub(m2, m.mem_mean), m.mem_stddev);
  model_weights(m, w);
  const double v = dadd(m.speed_mean, dmul(m.speed_stddev, narx_forward_d(w, z)));
  return v > floor_ ? v : floor_;
}

// SpeedPredictor::predict (predictor.cpp:271-292) for worker w; requires len >= 1.
__device__ inline double predictor_predict_d(const PredDev& P, int w, int len, double c_now,
                                      double m_now) {
  const double* v = P.hv + static_cast<size_t>(w) * P.max_hist;
  switch (P.kind) {
    case LBBSP_PRED_MEMORYLESS:
      return v[len - 1];
    case LBBSP_PRED_NARX:
      if (len >= P.warmup && len >= 2) {
        const double* c = P.hc + static_cast<size_t>(w) * P.max_hist;
        const double* m = P.hm + static_cast<size_t>(w) * P.max_hist;
        return narx_predict_d(P.models[w], v[len - 1], v[len - 2], c_now, c[len - 1], c[len - 2],
                              m_now, m[len - 1], m[len - 2], P.floor);
      }
      return P.ema[w];
    default:  // Ema, Perfect
      return P.ema[w];
  }
}

// SpeedHistory::push + comm_obs push (cluster_sim.cpp:309-313) with the
// incremental EMA states. `len` is the length BEFORE the push.
__device__ inline void observe_d(const PredDev& P, int w, int len, double v, double c, double m,
                          double tm) {
  const size_t o = static_cast<size_t>(w) * P.max_hist + len;
  if (len < P.max_hist) {
    P.hv[o] = v;
    P.hc[o] = c;
    P.hm[o] = m;
  }
  const double a = P.alpha, oma = dsub(1.0, P.alpha);
  // ema_0 = x_0, ema_k = alpha*x_k + (1-alpha)*ema_{k-1}  (predictor.cpp:22-23)
  P.ema[w] = len == 0 ? v : dadd(dmul(a, v), dmul(oma, P.ema[w]));
  // lagged comm EMA covers comm_obs[0..len-1] after this push
  if (len == 1)
    P.comm_ema_lag[w] = P.comm_last[w];
  else if (len > 1)
    P.comm_ema_lag[w] = dadd(dmul(a, P.comm_last[w]), dmul(oma, P.comm_ema_lag[w]));
  P.comm_last[w] = tm;
}

// Training scratch: per-sample arrays of stride narx_train_stride(len)
// doubles -- a multiple of 16 plus 17 (= 1 mod 16), so the arrays start in distinct
// shared-memory bank pairs and the 12 fold lanes (E, G[0..10]) read
// conflict-free; the stride also covers the zero padding of the folds to a
// multiple of 16 terms and 16 doubles of prefetch slack. Layout: Z[8], T, then one or two evaluation buffers
// {E, G[11]} (the second one holds the speculative halved-step evaluation).
constexpr int kNarxArraysMin = 21;   // Z[8], T, E, G[11]
constexpr int kNarxArrays = 33;      // + a second {E, G[11]}
__host__ __device__ __forceinline__ int narx_train_stride(int len) {
  const int cnt = len > 2 ? len - 2 : 1;
  return (cnt + 15) / 16 * 16 + 17;  // + 16 doubles of prefetch slack
}
// bytes for the full (two-buffer) layout; allocations are sized with this
__host__ __device__ __forceinline__ size_t narx_train_scratch_bytes(int len) {
  return static_cast<size_t>(narx_train_stride(len)) * kNarxArrays * sizeof(double);
}
// bytes for the one-buffer layout (no speculative halving)
__host__ __device__ __forceinline__ size_t narx_train_min_bytes(int len) {
  return static_cast<size_t>(narx_train_stride(len)) * kNarxArraysMin * sizeof(double);
}

// Training scratch for one call: shared memory when at least the one-buffer
// layout fits there, else the caller's global slot (sized for the full layout).
__device__ __forceinline__ double* narx_train_buf(int L, double* smem, size_t smem_bytes,
                                                  double* gslot, size_t gslot_doubles,
                                                  size_t* doubles) {
  if (narx_train_min_bytes(L) <= smem_bytes) {
    *doubles = smem_bytes / sizeof(double);
    return smem;
  }
  *doubles = gslot_doubles;
  return gslot;
}

#ifdef LBBSP_NARX_PROF
// probe builds only: per-CTA %globaltimer stamps of one training
// [0] entry [1] history copied [2] scalers [3] training set built
// [4] first evaluation [5] end; [6] evaluations, [7] epochs, [8] L
__device__ unsigned long long g_narx_prof[64][16];
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define NARX_PROF(i, v) \
  if (threadIdx.x == 0 && blockIdx.x < 64) g_narx_prof[blockIdx.x][i] = (v)
#else
#define NARX_PROF(i, v)
#endif
struct NarxTrainSmem {
  double w[11], g[11], gs[11], trial[11], sc[6];
  double val;
  int stall, epochs, stop;
};

// Per-sample pass of one evaluation (predictor.cpp:102-134) over samples
// first, first + stride, ...: the squared error E_i (mse, :104-107) and the 11
// gradient terms G_k,i (loss_gradient, :121-132: dz*z_k, dz, dy*h, dy -- each
// the same single product the reference forms).
__device__ __forceinline__ void narx_eval_terms(const double* wt, const double* Z, const double* T,
                                                double* E, double* G, int S, int cnt, double scale,
                                                int first, int stride) {
  for (int i = first; i < cnt; i += stride) {
    double z[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) z[j] = Z[static_cast<size_t>(j) * S + i];
    double a = wt[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a = dadd(a, dmul(wt[j], z[j]));
    const double h = glibc_tanh(a);
    const double y = dadd(dmul(wt[9], h), wt[10]);
    const double e = dsub(y, T[i]);
    E[i] = dmul(e, e);
    const double dy = dmul(scale, e);
    const double dz = dmul(dmul(dy, wt[9]), dsub(1.0, dmul(h, h)));
#pragma unroll
    for (int j = 0; j < 8; ++j) G[static_cast<size_t>(j) * S + i] = dmul(dz, z[j]);
    G[static_cast<size_t>(8) * S + i] = dz;
    G[static_cast<size_t>(9) * S + i] = dmul(dy, h);
    G[static_cast<size_t>(10) * S + i] = dy;
  }
}

// One evaluation of the training objective fused with the gradient. If fwd_w
// is given, all threads first form the per-sample terms of fwd_w in buffer
// (E, G); otherwise they are already there (a speculative pass). Then lanes
// 0..11 of warp 1 fold E and G_0..10 left to right, one array per lane, 8 terms
// ahead in registers so only the dependent DADD chain is exposed (the folds are
// zero padded to a multiple of 16; adding +0.0 to a sum that starts at +0.0 is
// the identity). Meanwhile, if spec_step > 0, every other thread forms the
// terms of the halved trial w - spec_step * g in (Es, Gs): it is exactly the
// next evaluation whenever this trial is rejected (apply_step :136-143 with
// the halved step, same operations), and is discarded otherwise. The gradient
// folded here is likewise the next epoch's loss_gradient(model) whenever the
// trial is accepted.
__device__ inline double block_eval(const double* fwd_w, const double* Z, const double* T,
                                    double* E, double* G, double* Es, double* Gs, int S, int cnt,
                                    double scale, double spec_step, double* gout, NarxTrainSmem* s) {
#ifdef LBBSP_NARX_PROF
  const unsigned long long pt0 = clock64();
#endif
  if (fwd_w) {
    narx_eval_terms(fwd_w, Z, T, E, G, S, cnt, scale, threadIdx.x, blockDim.x);
    __syncthreads();
  }
#ifdef LBBSP_NARX_PROF
  const unsigned long long pt1 = clock64();
#endif
  if (threadIdx.x >= 32 && threadIdx.x < 44) {
    const int k = threadIdx.x - 32;
    const double* src = k < 11 ? G + static_cast<size_t>(k) * S : E;
    // two 8-term register blocks alternate (no register moves); the block
    // after the last one is read from the stride's slack and never added
    const int n16 = (cnt + 15) / 16 * 16;
    double acc = 0.0, a[8], b[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = src[q];
    for (int i = 0; i < n16; i += 16) {
#pragma unroll
      for (int q = 0; q < 8; ++q) b[q] = src[i + 8 + q];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc = dadd(acc, a[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = src[i + 16 + q];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc = dadd(acc, b[q]);
    }
    if (k < 11) gout[k] = acc;
    else s->val = ddiv(acc, static_cast<double>(cnt));
  } else if (spec_step > 0.0 && (threadIdx.x < 32 || threadIdx.x >= 64)) {
    double sw[11];
#pragma unroll
    for (int t = 0; t < 11; ++t) sw[t] = dsub(s->w[t], dmul(spec_step, s->g[t]));
    const int idx = threadIdx.x < 32 ? threadIdx.x : threadIdx.x - 32;
    narx_eval_terms(sw, Z, T, Es, Gs, S, cnt, scale, idx, blockDim.x - 32);
  }
#ifdef LBBSP_NARX_PROF
  if (threadIdx.x == 32 && blockIdx.x < 64) {  // the E-fold lane: its fold end
    g_narx_prof[blockIdx.x][11] += clock64() - pt1;
  }
#endif
  __syncthreads();
#ifdef LBBSP_NARX_PROF
  if (threadIdx.x == 0 && blockIdx.x < 64) {
    g_narx_prof[blockIdx.x][9] += pt1 - pt0;            // terms + barrier
    g_narx_prof[blockIdx.x][10] += clock64() - pt1;   // fold + barrier
  }
#endif
  return s->val;
}

// narx_train_online (predictor.cpp:155-196) for one model with history
// (v, c, m)[0..L). buf: buf_doubles doubles of scratch (shared or global), at
// least narx_train_min_bytes(L); with narx_train_scratch_bytes(L) the halved
// trial step is evaluated speculatively beside each fold. Bit-exact: every
// value the reference computes is computed with the same operations in the
// same order; only independent work is overlapped.
// staged > 0: the caller already copied history [0, staged) into the
// scratch's history region (narx_history_region); pre_sums: the three scaler
// sums' left folds over [0, pre_n), continued here in the same order (the
// caller folds the earlier rounds before the newest observation exists).
__host__ __device__ __forceinline__ double* narx_history_region(double* buf, int L) {
  return buf + 9 * static_cast<size_t>(narx_train_stride(L));
}
__device__ inline void narx_train_block(lbbsp_narx_model* gm, const double* v, const double* c,
                                        const double* m, int L, const lbbsp_narx_train_cfg cfg,
                                        lbbsp_narx_report* rep, double* loss_log, int loss_cap,
                                        double* buf, size_t buf_doubles, NarxTrainSmem* s,
                                        int staged = 0, const double* pre_sums = nullptr,
                                        int pre_n = 0) {
  const int tid = threadIdx.x;
  const int minh = cfg.min_history > 3 ? cfg.min_history : 3;
  if (L < minh) {
    if (tid == 0 && rep) *rep = lbbsp_narx_report{0, 0, 0.0};
    return;
  }
  NARX_PROF(0, gtimer_ns());
  NARX_PROF(8, L);
  NARX_PROF(9, 0);
  NARX_PROF(10, 0);
  NARX_PROF(11, 0);
  NARX_PROF(12, 0);
  NARX_PROF(15, 0);
  const int S = narx_train_stride(L);
  // the history into the scratch's E/G region first (written only once the
  // evaluations start): one parallel round trip, instead of the sequential
  // scaler folds below waiting on each cache line of v, c, m in turn
  double* hv = narx_history_region(buf, L);
  double* hc = hv + L;
  double* hm = hc + L;
  for (int i = staged + tid; i < L; i += blockDim.x) {
    hv[i] = v[i];
    hc[i] = c[i];
    hm[i] = m[i];
  }
  v = hv;
  c = hc;
  m = hm;
  __syncthreads();
  NARX_PROF(1, gtimer_ns());
  // fit_scaler x3 (predictor.cpp:71-82), one sequential thread per series
  if (tid == 0 || tid == 32 || tid == 64) {
    const int which = tid / 32;
    const double* xs = which == 0 ? v : (which == 1 ? c : m);
    double sum = pre_sums ? pre_sums[which] : 0.0;
    for (int i = pre_sums ? pre_n : 0; i < L; ++i) sum = dadd(sum, xs[i]);
    const double mean = ddiv(sum, static_cast<double>(L));
    double var = 0.0;
    for (int i = 0; i < L; ++i) {
      const double d = dsub(xs[i], mean);
      var = dadd(var, dmul(d, d));
    }
    var = ddiv(var, static_cast<double>(L));
    s->sc[2 * which] = mean;
    s->sc[2 * which + 1] = var > 1e-18 ? __dsqrt_rn(var) : 1.0;
  }
  if (tid == 96) {
    model_weights(*gm, s->w);
    s->stall = 0;
    s->epochs = 0;
    s->stop = 0;
  }
  __syncthreads();
  NARX_PROF(2, gtimer_ns());
  const int cnt = L - 2;
  double* Z = buf;                             // [8][S]
  double* T = Z + static_cast<size_t>(8) * S;  // [S]
  // {E [S], G [11][S]} x 2 at T + S and T + 13 S. Addressed arithmetically,
  // not through a pointer array: a runtime-indexed local array would hold
  // the pointers in local memory and turn every access through them into a
  // generic load/store instead of LDS/STS
  double* const EG0 = T + S;
  const size_t EGs = 12 * static_cast<size_t>(S);
  const bool spec = buf_doubles >= static_cast<size_t>(kNarxArrays) * S &&
                    cnt <= static_cast<int>(blockDim.x) - 32;
  const double mv = s->sc[0], sv = s->sc[1], mc = s->sc[2], scd = s->sc[3], mm = s->sc[4],
               sm = s->sc[5];
  // build_training_set (predictor.cpp:89-100): the 9 standardised columns
  // (Z[0..7], T = row 8 of the same layout) one element per thread -- each
  // element the reference's single (x - mean) / stddev, 9x fewer dependent
  // divisions per thread than one sample per thread
  for (int e = tid; e < 9 * cnt; e += blockDim.x) {
    const int f = e / cnt, i = e - f * cnt, t = i + 2;
    // feature f: series (v, v, c, c, c, m, m, m, v) at lag (1, 2, 0, 1, 2, 0, 1, 2, 0)
    const int ser = f < 2 ? 0 : (f < 5 ? 1 : (f < 8 ? 2 : 0));
    const int lag = f == 8 ? 0 : (f < 2 ? f + 1 : (f - (f < 5 ? 2 : 5)));
    const double* xs = ser == 0 ? v : (ser == 1 ? c : m);
    const double mu = ser == 0 ? mv : (ser == 1 ? mc : mm);
    const double sd = ser == 0 ? sv : (ser == 1 ? scd : sm);
    Z[static_cast<size_t>(f) * S + i] = ddiv_std(dsub(xs[t - lag], mu), sd);
  }
  __syncthreads();
  NARX_PROF(14, gtimer_ns());
  // zero padding of the folds (never written by the evaluations; after the
  // build, which read the history copy in the same region)
  for (int i = cnt + tid; i < (cnt + 15) / 16 * 16; i += blockDim.x)
    for (int b = 0; b < (spec ? 2 : 1); ++b)
      for (int k = 0; k < 12; ++k) EG0[b * EGs + static_cast<size_t>(k) * S + i] = 0.0;
  __syncthreads();
  NARX_PROF(3, gtimer_ns());
  const double scale = ddiv(2.0, static_cast<double>(cnt));
  auto E_ = [&](int b) { return EG0 + b * EGs; };
  auto G_ = [&](int b) { return EG0 + b * EGs + S; };
  // current = mse(model) (:165), and loss_gradient(model) of epoch 0
  double current = block_eval(s->w, Z, T, E_(0), G_(0), nullptr, nullptr, S, cnt, scale, 0.0,
                              s->g, s);
  NARX_PROF(4, gtimer_ns());
#ifdef LBBSP_NARX_PROF
  int n_eval = 1;
#define NARX_EVAL_COUNT ++n_eval
#else
#define NARX_EVAL_COUNT
#endif
  for (int epoch = 0; epoch < cfg.max_epochs; ++epoch) {
    double step = cfg.step;
    if (tid < 11) s->trial[tid] = dsub(s->w[tid], dmul(step, s->g[tid]));  // apply_step :136-143
    __syncthreads();
    // The epoch's first trial is evaluated alone: it is accepted ~3 times in
    // 4 (0.27 halvings per epoch on the bench histories), and a speculative
    // halved trial beside its fold would lengthen it (the halved terms'
    // tanh chains outlast the fold). After a rejection halvings cluster, so
    // from then on each fold runs beside the next halved trial's terms.
    int b = 0;
    double next = block_eval(s->trial, Z, T, E_(b), G_(b), nullptr, nullptr, S, cnt, scale, 0.0,
                             s->gs, s);
    NARX_EVAL_COUNT;
    int halvings = 0;
    bool have_spec = false;
    while (next > current && halvings < 20) {
      step = dmul(step, 0.5);
      if (tid < 11) s->trial[tid] = dsub(s->w[tid], dmul(step, s->g[tid]));
      __syncthreads();
      if (spec && have_spec) {  // this trial's terms were formed beside the previous fold
        b ^= 1;
        next = block_eval(nullptr, Z, T, E_(b), G_(b), E_(b ^ 1), G_(b ^ 1), S, cnt, scale,
                          dmul(step, 0.5), s->gs, s);
      } else if (spec) {  // first halving: its own terms, the next halving's beside its fold
        next = block_eval(s->trial, Z, T, E_(b), G_(b), E_(b ^ 1), G_(b ^ 1), S, cnt, scale,
                          dmul(step, 0.5), s->gs, s);
        have_spec = true;
      } else {
        next = block_eval(s->trial, Z, T, E_(0), G_(0), nullptr, nullptr, S, cnt, scale, 0.0,
                          s->gs, s);
      }
      ++halvings;
      NARX_EVAL_COUNT;
    }
    if (next > current) break;  // no descent direction left (:182)
    if (tid < 11) {
      s->w[tid] = s->trial[tid];
      s->g[tid] = s->gs[tid];  // loss_gradient at the accepted weights
    }
    if (tid == 0) {
      if (loss_log && s->epochs < loss_cap) loss_log[s->epochs] = next;
      s->epochs += 1;
      s->stall = dsub(current, next) < cfg.early_stop_delta ? s->stall + 1 : 0;
    }
    __syncthreads();
    current = next;
    if (s->stall >= cfg.early_stop_patience) break;
  }
  NARX_PROF(5, gtimer_ns());
#ifdef LBBSP_NARX_PROF
  NARX_PROF(6, n_eval);
  NARX_PROF(7, s->epochs);
#endif
  if (tid == 0) {
    if (rep) *rep = lbbsp_narx_report{1, s->epochs, current};
    for (int j = 0; j < 8; ++j) gm->input_weights[j] = s->w[j];
    gm->hidden_bias = s->w[8];
    gm->output_weight = s->w[9];
    gm->output_bias = s->w[10];
    gm->speed_mean = mv;
    gm->speed_stddev = sv;
    gm->cpu_mean = mc;
    gm->cpu_stddev = scd;
    gm->mem_mean = mm;
    gm->mem_stddev = sm;
  }
  __syncthreads();
}

}  // namespace lbbsp
