// narx_sweep.cu -- C4: the NARX predictor at sweep scale (BASELINE configs[3]):
// W worker histories, delay d (inputs I = 3d+2), hidden width H, batched
// inference and training in fp32 on CUDA cores, one CTA per model.
//
// Same algorithm as narx_train_online (predictor.cpp:155-196) generalised to
// (d, H) exactly as the fp64 oracle oracle/lbbsp_oracle.c:orc_narxg_train:
// scaler refit, windowed training set, full-batch GD with <= 20 halvings of the
// trial step, stop on no descent or 4 epochs with improvement < 1e-4.
// Per epoch the trial weights are evaluated once: a sample-parallel pass
// (forward, squared error, dy, dz, hidden activations) and a parameter-
// parallel pass (dW1 = dz^T Z, db1, dw2, db2, mse) -- the gradient at the trial
// is speculative and becomes the next epoch's gradient when accepted.
// Tolerance-based parity vs the fp64 oracle (tests/test_gpu_narx_sweep.py).
#include <cmath>
#include <random>
#include <vector>

#include "common.cuh"
#include "exactmath.cuh"

namespace lbbsp {
namespace sweep {

constexpr int kThreads = 256;
constexpr int kMaxI = 32;   // 3d+2 <= 32  (d <= 10)
constexpr int kMaxH = 64;

__host__ __device__ constexpr int param_count(int d, int h) { return h * (3 * d + 2) + 2 * h + 1 + 6; }

struct SweepArgs {
  int W, L, d, h;
  const double* v;  // [W][L]
  const double* c;
  const double* m;
  float* params;    // [W][P]
  lbbsp_narx_train_cfg cfg;
  int fixed_epochs;
  int* epochs_out;        // [W]
  float* loss_out;        // [W]
  float* scratch;         // [W][cnt][2H + 2] global (h, dz, dy, E)
  int smem_z;             // 1: Z/T in shared memory
};

__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  if (threadIdx.x < 32) {
    s = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  return red[0];
}

__device__ __forceinline__ double block_sum_d(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < static_cast<int>(blockDim.x / 32); ++i) s += red[i];
    red[0] = s;
  }
  __syncthreads();
  return red[0];
}

// Evaluate weights wt (shared): returns the mse and writes the gradient at wt
// to g (shared). Samples are processed in chunks of 64 through shared memory:
//   phase A: 4 threads per sample, each owning ceil(H/4) hidden units --
//            forward, tanh, output (quad shuffle), error, dy, dz;
//   phase B: each thread folds its <= 8 W1 entries and its b1/w2 entry over
//            the chunk into registers.
constexpr int kChunk = 64;
constexpr int kQuad = 4;
constexpr int kUnits = kMaxH / kQuad;  // 16
constexpr int kW1PerThread = kMaxH * kMaxI / kThreads;  // 8

__device__ float eval_and_grad(const float* wt, const float* W1p, float* g, const float* Z,
                               const float* T, int cnt, int I, int H, float scale, float* hc,
                               float* dzc, float* dyc, float* red) {
  // W1p: W1 with row stride I+1 and Z: rows of stride I+1 (bank-conflict-free)
  const int ldz = I + 1;
  const float* b1 = wt + H * I;
  const float* w2 = b1 + H;
  const float b2 = w2[H];
  const int tid = threadIdx.x;
  const int s_in = tid / kQuad, part = tid % kQuad;
  const int upt = (H + kQuad - 1) / kQuad;  // hidden units per thread
  const int j0 = part * upt;
  float gw1[kW1PerThread];
#pragma unroll
  for (int r = 0; r < kW1PerThread; ++r) gw1[r] = 0.f;
  float gb1 = 0.f, gw2 = 0.f, esum = 0.f, dysum = 0.f;
  const int nW1 = H * I;
  for (int base = 0; base < cnt; base += kChunk) {
    const int ns = min(kChunk, cnt - base);
    // ---- phase A (every lane runs the quad shuffles; only valid samples store) ----
    {
      const bool valid = s_in < ns;
      const int i = base + (valid ? s_in : 0);
      const float* x = Z + static_cast<size_t>(i) * ldz;
      float xr[kMaxI];
#pragma unroll
      for (int q = 0; q < kMaxI; ++q) xr[q] = q < I ? x[q] : 0.f;
      float hloc[kUnits];
      float yp = 0.f;
#pragma unroll
      for (int u = 0; u < kUnits; ++u) {
        const int j = j0 + u;
        hloc[u] = 0.f;
        if (u < upt && j < H) {
          float a = b1[j];
          const float* wr = W1p + j * ldz;
#pragma unroll
          for (int q = 0; q < kMaxI; ++q)
            if (q < I) a = fmaf(wr[q], xr[q], a);
          const float hj = tanhf(a);
          hloc[u] = hj;
          yp = fmaf(w2[j], hj, yp);
        }
      }
      yp += __shfl_xor_sync(0xffffffffu, yp, 1);
      yp += __shfl_xor_sync(0xffffffffu, yp, 2);
      const float e = yp + b2 - T[i];
      const float dy = scale * e;
      if (valid) {
        if (part == 0) {
          esum = fmaf(e, e, esum);
          dysum += dy;
          dyc[s_in] = dy;
        }
#pragma unroll
        for (int u = 0; u < kUnits; ++u) {
          const int j = j0 + u;
          if (u < upt && j < H) {
            hc[s_in * H + j] = hloc[u];
            dzc[s_in * H + j] = dy * w2[j] * (1.f - hloc[u] * hloc[u]);
          }
        }
      }
    }
    __syncthreads();
    // ---- phase B ----
#pragma unroll
    for (int r = 0; r < kW1PerThread; ++r) {
      const int e = tid + r * kThreads;
      if (e < nW1) {
        const int j = e / I, q = e % I;
        float a = gw1[r];
        for (int s2 = 0; s2 < ns; ++s2) a = fmaf(dzc[s2 * H + j], Z[static_cast<size_t>(base + s2) * ldz + q], a);
        gw1[r] = a;
      }
    }
    if (tid < H) {
      for (int s2 = 0; s2 < ns; ++s2) gb1 += dzc[s2 * H + tid];
    } else if (tid >= 128 && tid < 128 + H) {
      const int j = tid - 128;
      for (int s2 = 0; s2 < ns; ++s2) gw2 = fmaf(dyc[s2], hc[s2 * H + j], gw2);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < kW1PerThread; ++r) {
    const int e = tid + r * kThreads;
    if (e < nW1) g[e] = gw1[r];
  }
  if (tid < H) g[nW1 + tid] = gb1;
  if (tid >= 128 && tid < 128 + H) g[nW1 + H + (tid - 128)] = gw2;
  const float mse = block_sum(esum, red) / static_cast<float>(cnt);
  const float db2 = block_sum(dysum, red);
  if (tid == 0) g[nW1 + 2 * H] = db2;
  __syncthreads();
  return mse;
}

__global__ void __launch_bounds__(kThreads) narxg_train_kernel(SweepArgs A) {
  extern __shared__ float sm[];
  __shared__ float red[32];
  __shared__ double redd[32];
  __shared__ int s_stall, s_epochs;
  __shared__ float s_sc[6];
  const int w = blockIdx.x;
  const int d = A.d, H = A.h, I = 3 * d + 2, L = A.L;
  const int P = H * I + 2 * H + 1;
  const int cnt = L - d;
  float* params = A.params + static_cast<size_t>(w) * (P + 6);
  const double* v = A.v + static_cast<size_t>(w) * L;
  const double* c = A.c + static_cast<size_t>(w) * L;
  const double* m = A.m + static_cast<size_t>(w) * L;
  const int minh = A.cfg.min_history > d + 1 ? A.cfg.min_history : d + 1;
  if (L < minh) {
    if (threadIdx.x == 0) {
      A.epochs_out[w] = 0;
      A.loss_out[w] = 0.f;
    }
    return;
  }
  // shared layout: wcur[P] | wtrial[P] | g[P] | gs[P] | (Z[cnt*I] | T[cnt])?
  float* wcur = sm;
  float* wtr = wcur + P;
  float* g = wtr + P;
  float* gs = g + P;
  float* zt = gs + P;
  float* w1c = zt;                         // [H][I+1] padded W1 of wcur
  float* w1t = w1c + H * (I + 1);           // [H][I+1] padded W1 of wtr
  float* hc = w1t + H * (I + 1);            // [kChunk][H]
  float* dzc = hc + kChunk * H;             // [kChunk][H]
  float* dyc = dzc + kChunk * H;            // [kChunk]
  float* zsm = dyc + kChunk;
  float* Z = A.smem_z ? zsm : A.scratch + static_cast<size_t>(w) * cnt * (I + 2);
  float* T = Z + static_cast<size_t>(cnt) * (I + 1);
  // scalers (fp64 mean / population std, predictor.cpp:71-82)
  for (int which = 0; which < 3; ++which) {
    const double* xs = which == 0 ? v : (which == 1 ? c : m);
    double sacc = 0.0;
    for (int i = threadIdx.x; i < L; i += blockDim.x) sacc += xs[i];
    const double mean = block_sum_d(sacc, redd) / L;
    double vacc = 0.0;
    for (int i = threadIdx.x; i < L; i += blockDim.x) vacc += (xs[i] - mean) * (xs[i] - mean);
    const double var = block_sum_d(vacc, redd) / L;
    if (threadIdx.x == 0) {
      s_sc[2 * which] = static_cast<float>(mean);
      s_sc[2 * which + 1] = static_cast<float>(var > 1e-18 ? sqrt(var) : 1.0);
    }
  }
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    wcur[i] = params[i];
    if (i < H * I) w1c[(i / I) * (I + 1) + i % I] = params[i];
  }
  if (threadIdx.x == 0) {
    s_stall = 0;
    s_epochs = 0;
  }
  __syncthreads();
  const float mv = s_sc[0], sv = s_sc[1], mc = s_sc[2], scd = s_sc[3], mm = s_sc[4], smm = s_sc[5];
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int t = i + d;
    float* z = Z + static_cast<size_t>(i) * (I + 1);
    for (int l = 0; l < d; ++l) z[l] = static_cast<float>((v[t - 1 - l] - mv) / sv);
    for (int l = 0; l <= d; ++l) z[d + l] = static_cast<float>((c[t - l] - mc) / scd);
    for (int l = 0; l <= d; ++l) z[2 * d + 1 + l] = static_cast<float>((m[t - l] - mm) / smm);
    T[i] = static_cast<float>((v[t] - mv) / sv);
  }
  __syncthreads();
  const float scale = 2.f / static_cast<float>(cnt);
  float current = eval_and_grad(wcur, w1c, g, Z, T, cnt, I, H, scale, hc, dzc, dyc, red);
  const int max_ep = A.fixed_epochs > 0 ? A.fixed_epochs : A.cfg.max_epochs;
  for (int epoch = 0; epoch < max_ep; ++epoch) {
    float step = static_cast<float>(A.cfg.step);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      wtr[i] = wcur[i] - step * g[i];
      if (i < H * I) w1t[(i / I) * (I + 1) + i % I] = wtr[i];
    }
    __syncthreads();
    float next = eval_and_grad(wtr, w1t, gs, Z, T, cnt, I, H, scale, hc, dzc, dyc, red);
    int halvings = 0;
    while (next > current && halvings < 20) {
      step *= 0.5f;
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        wtr[i] = wcur[i] - step * g[i];
        if (i < H * I) w1t[(i / I) * (I + 1) + i % I] = wtr[i];
      }
      __syncthreads();
      next = eval_and_grad(wtr, w1t, gs, Z, T, cnt, I, H, scale, hc, dzc, dyc, red);
      ++halvings;
    }
    if (next > current) break;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      wcur[i] = wtr[i];
      g[i] = gs[i];
      if (i < H * I) w1c[(i / I) * (I + 1) + i % I] = wtr[i];
    }
    if (threadIdx.x == 0) {
      s_epochs += 1;
      s_stall = (current - next < static_cast<float>(A.cfg.early_stop_delta)) ? s_stall + 1 : 0;
    }
    __syncthreads();
    current = next;
    if (A.fixed_epochs <= 0 && s_stall >= A.cfg.early_stop_patience) break;
  }
  for (int i = threadIdx.x; i < P; i += blockDim.x) params[i] = wcur[i];
  if (threadIdx.x < 6) params[P + threadIdx.x] = s_sc[threadIdx.x];
  if (threadIdx.x == 0) {
    A.epochs_out[w] = s_epochs;
    A.loss_out[w] = current;
  }
}

// batched narx_predict (predictor.cpp:147-153) for W models, one warp each
__global__ void narxg_predict_kernel(int W, int L, int d, int H, const double* v, const double* c,
                                     const double* m, const double* c_now, const double* m_now,
                                     const float* params, double floor_, double* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= W) return;
  const int I = 3 * d + 2, P = H * I + 2 * H + 1;
  const float* p = params + static_cast<size_t>(warp) * (P + 6);
  const float* sc = p + P;
  const double* vv = v + static_cast<size_t>(warp) * L;
  const double* cc = c + static_cast<size_t>(warp) * L;
  const double* mm = m + static_cast<size_t>(warp) * L;
  float x = 0.f;  // lane q holds input q
  if (lane < d) x = static_cast<float>((vv[L - 1 - lane] - sc[0]) / sc[1]);
  else if (lane < 2 * d + 1) {
    const int l = lane - d;
    const double cv = l == 0 ? c_now[warp] : cc[L - l];
    x = static_cast<float>((cv - sc[2]) / sc[3]);
  } else if (lane < I) {
    const int l = lane - 2 * d - 1;
    const double mv = l == 0 ? m_now[warp] : mm[L - l];
    x = static_cast<float>((mv - sc[4]) / sc[5]);
  }
  float y = 0.f;
  for (int j = 0; j < H; ++j) {
    float a = lane < I ? p[j * I + lane] * x : 0.f;
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    y += p[H * I + H + j] * tanhf(a + p[H * I + j]);
  }
  y += p[H * I + 2 * H];
  if (lane == 0) {
    const double o = static_cast<double>(sc[0]) + static_cast<double>(sc[1]) * y;
    out[warp] = o > floor_ ? o : floor_;
  }
}

}  // namespace sweep
}  // namespace lbbsp

using namespace lbbsp;

extern "C" int lbbsp_narxg_param_count(int delay, int hidden) {
  return sweep::param_count(delay, hidden);
}

// generalised narx_init (predictor.cpp:35-44) in fp32, same draw order as
// oracle orc_narxg_init (host, setup-time)
extern "C" int lbbsp_narxg_init(uint64_t seed, int delay, int hidden, float* h_params) {
  const int I = 3 * delay + 2;
  std::mt19937_64 gen(mix_seed(seed, 0x9a4c0ull));
  auto uni = [&](double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(gen() >> 11) * 0x1.0p-53);
  };
  for (int j = 0; j < hidden * I; ++j) h_params[j] = static_cast<float>(uni(-0.3, 0.3));
  for (int j = 0; j < hidden; ++j) h_params[hidden * I + j] = static_cast<float>(uni(-0.1, 0.1));
  for (int j = 0; j < hidden; ++j) h_params[hidden * I + hidden + j] = static_cast<float>(uni(-0.3, 0.3));
  h_params[hidden * I + 2 * hidden] = 0.f;
  float* sc = h_params + hidden * I + 2 * hidden + 1;
  sc[0] = 0.f; sc[1] = 1.f; sc[2] = 0.f; sc[3] = 1.f; sc[4] = 0.f; sc[5] = 1.f;
  return LBBSP_OK;
}

extern "C" int lbbsp_narx_sweep_train(int W, int L, int delay, int hidden, const double* d_v,
                                      const double* d_c, const double* d_m, float* d_params,
                                      const lbbsp_narx_train_cfg* cfg, int fixed_epochs,
                                      int* d_epochs, float* d_loss, float* d_scratch,
                                      void* stream) {
  const int I = 3 * delay + 2;
  if (delay < 1 || I > sweep::kMaxI || hidden < 1 || hidden > sweep::kMaxH || W < 1 || L < 2)
    return set_error(LBBSP_INVALID_ARGUMENT, "narx sweep: need 1 <= delay <= 10, 1 <= hidden <= 64");
  const int P = hidden * I + 2 * hidden + 1;
  const int cnt = L - delay;
  const size_t base = static_cast<size_t>(4 * P + 2 * hidden * (I + 1) + 2 * sweep::kChunk * hidden +
                                          sweep::kChunk) * sizeof(float);
  const size_t zbytes = static_cast<size_t>(cnt) * (I + 2) * sizeof(float);
  const bool smem_z = base + zbytes <= 200 * 1024;
  const size_t smem = base + (smem_z ? zbytes : 0);
  sweep::SweepArgs a{};
  a.W = W;
  a.L = L;
  a.d = delay;
  a.h = hidden;
  a.v = d_v;
  a.c = d_c;
  a.m = d_m;
  a.params = d_params;
  a.cfg = *cfg;
  a.fixed_epochs = fixed_epochs;
  a.epochs_out = d_epochs;
  a.loss_out = d_loss;
  a.scratch = d_scratch;
  a.smem_z = smem_z ? 1 : 0;
  LBBSP_CUDA_CHECK(cudaFuncSetAttribute(sweep::narxg_train_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
  sweep::narxg_train_kernel<<<W, sweep::kThreads, smem, static_cast<cudaStream_t>(stream)>>>(a);
  LBBSP_CUDA_CHECK(cudaGetLastError());
  return LBBSP_OK;
}

// scratch floats needed by lbbsp_narx_sweep_train
extern "C" long long lbbsp_narx_sweep_scratch_floats(int W, int L, int delay, int hidden) {
  const int I = 3 * delay + 2;
  const long long cnt = L - delay;
  return static_cast<long long>(W) * cnt * (I + 2);
}

extern "C" int lbbsp_narx_sweep_predict(int W, int L, int delay, int hidden, const double* d_v,
                                        const double* d_c, const double* d_m, const double* d_c_now,
                                        const double* d_m_now, const float* d_params, double floor,
                                        double* d_out, void* stream) {
  if (3 * delay + 2 > 32 || hidden > sweep::kMaxH)
    return set_error(LBBSP_INVALID_ARGUMENT, "narx sweep: need 3*delay+2 <= 32, hidden <= 64");
  const int threads = 256, warps_per_block = threads / 32;
  const int blocks = (W + warps_per_block - 1) / warps_per_block;
  sweep::narxg_predict_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      W, L, delay, hidden, d_v, d_c, d_m, d_c_now, d_m_now, d_params, floor, d_out);
  LBBSP_CUDA_CHECK(cudaGetLastError());
  return LBBSP_OK;
}
