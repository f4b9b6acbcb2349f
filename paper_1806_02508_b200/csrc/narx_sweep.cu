// narx_sweep.cu -- C4: the NARX predictor at sweep scale (BASELINE configs[3]):
// W worker histories, delay d (inputs I = 3d+2), hidden width H, batched
// inference and training, one CTA per model. Training runs on warp tensor-core
// MMA with split-bf16 (hi + lo) operands whenever the training set fits shared
// memory (history <= ~1150 at delay 10 / hidden 64; narxg_train_tc_kernel),
// else on fp32 CUDA cores with the training set in global scratch
// (narxg_train_kernel).
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
#include <cstdlib>
#include <random>
#include <vector>

#include <cuda_bf16.h>

#include "common.cuh"
#include "exactmath.cuh"
#include "tc_ptx.cuh"

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

// ---------------------------------------------------------------------------
// Tensor-core trainer (the default whenever the history fits shared memory).
// Same epochs / step halvings / stopping rule as narxg_train_kernel; each
// evaluation runs on warp MMA (mma.sync m16n8k16, bf16 operands, fp32
// accumulate) with every operand split into bf16 hi + lo and the product taken
// as hi*hi + hi*lo + lo*hi (~2^-16 relative, well inside the fp32 tolerance).
// Per 16-sample tile, one warp:
//   A   = Z W1^T + b1          48 MMAs (A = Z via ldmatrix, B = W1 via ldmatrix)
//   h   = tanh(A); y = h w2 + b2; e; dy; dz = dy w2 (1 - h^2)   (on fragments)
//   dW1 += dz^T Z              48 MMAs (A = dz^T by movmatrix.trans from the
//                                       accumulator fragments, B = Z via .trans)
//   db1 += col sums of dz, dw2 += dy^T h, mse, db2        (registers)
// Warps own disjoint tiles; their dW1 partials are combined in a fixed tree
// order (deterministic). Z is stored once per model as bf16 hi/lo rows of 64 B
// (32 inputs, zero padded) with a 16-B chunk XOR swizzle, so every ldmatrix
// phase is bank-conflict free.
namespace tcs {

constexpr int kTcThreads = 512;
constexpr int kPairs = kTcThreads / 64;  // warp pairs; each pair splits the hidden units
constexpr int kRedFloats = 8 * 1024;   // dW1 tree scratch: 4 pairs x 2 halves x 32x32

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t r[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t r[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ uint32_t movt(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ void mma(float c[4], const uint32_t a[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// x ~= hi + lo, both bf16; two elements per 32-bit word (lower index low)
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
// tanh(x) = 1 - 2 / (1 + e^{2x}) on the SFU (ex2 + rcp, both ~2^-22 relative):
// absolute error < 3e-7 over the whole range, saturating to +-1 -- 5
// instructions against ~20 for tanhf's two-branch form.
__device__ __forceinline__ float tanh_sfu(float x) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * 2.8853900817779268f));  // 2 / ln 2
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + e));
  return fmaf(-2.f, r, 1.f);
}
// byte offset of (row, 16-B chunk) in a [rows][64 B] swizzled array
__device__ __forceinline__ int zsw(int row, int chunk) { return row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4); }

struct Smem {
  unsigned char* zh;  // [cntp][64 B]
  unsigned char* zl;
  unsigned char* wh;  // [64 hidden][64 B]
  unsigned char* wl;
  float* red;         // [kRedFloats]
  float* T;           // [cntp]
  float* bw;          // [2][64]: b1 | w2 of the staged weights (zero padded)
  float* colred;      // [kPairs][128]
  float* ypart;       // [kPairs][2 parity][2 halves][16]
  float* scal;        // [1] mse broadcast
};

__host__ __device__ inline size_t smem_bytes(int cnt, int P) {
  const size_t cntp = (cnt + 15) / 16 * 16;
  return 2 * cntp * 64 + 2 * 4096 + kRedFloats * 4 +
         4 * (cntp + 4 * static_cast<size_t>(P) + 128 + kPairs * 128 + kPairs * 64 + 4) + 64;
}

// write parameter i (value x) of the staged weight set
__device__ __forceinline__ void stage_param(const Smem& S, int i, float x, int I, int H) {
  if (i < H * I) {
    const int j = i / I, q = i - j * I;
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
    const int off = zsw(j, q >> 3) + (q & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(S.wh + off) = h;
    *reinterpret_cast<__nv_bfloat16*>(S.wl + off) = l;
  } else if (i < H * I + 2 * H) {
    const int k = i - H * I;
    S.bw[k < H ? k : 64 + (k - H)] = x;
  }
}

// mse of the staged weights; gradient at them -> gout[P].
// Warp w = 2p + hh: pair p owns tiles p, p + 8, ...; half hh owns hidden units
// [32 hh, 32 hh + 32) -- forward n-tiles 4hh..4hh+3 and dW1 rows of that half.
// The two halves of y = h w2 are exchanged through shared memory under a
// pair-wide named barrier and summed in a fixed order.
__device__ float eval_tc(const Smem& S, float b2, float* gout, int cnt, int I, int H, float scale,
                         float* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int pr = warp >> 1, hh = warp & 1;
  const uint32_t zh = saddr(S.zh), zl = saddr(S.zl), wh = saddr(S.wh), wl = saddr(S.wl);
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lch = lane >> 4;
  const int ntiles = (cnt + 15) / 16;
  const float* b1h = S.bw + 32 * hh;
  const float* w2h = S.bw + 64 + 32 * hh;
  float dw[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int r = 0; r < 4; ++r) dw[a][b][r] = 0.f;
  float db1[8], dw2[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) db1[k] = dw2[k] = 0.f;
  float esum = 0.f, dysum = 0.f;
  int it = 0;
  for (int tile = pr; tile < ntiles; tile += kPairs, ++it) {
    const int r0 = tile * 16;
    float acc[4][4];
    {
      uint32_t ah[2][4], al[2][4];
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        ldsm_x4(zh + zsw(r0 + lrow, 2 * ks + lch), ah[ks]);
        ldsm_x4(zl + zsw(r0 + lrow, 2 * ks + lch), al[ks]);
      }
      // the small cross products (lo*hi, hi*lo) in their own accumulator:
      // two independent MMA chains per n-tile instead of one of six
      float accx[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const float2 b = *reinterpret_cast<const float2*>(b1h + 8 * nt + 2 * t);
        acc[nt][0] = b.x; acc[nt][1] = b.y; acc[nt][2] = b.x; acc[nt][3] = b.y;
        accx[nt][0] = accx[nt][1] = accx[nt][2] = accx[nt][3] = 0.f;
        uint32_t bh[4], bl[4];
        const int wrow = 32 * hh + 8 * nt + (lane & 7);
        ldsm_x4(wh + zsw(wrow, lane >> 3), bh);
        ldsm_x4(wl + zsw(wrow, lane >> 3), bl);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          mma(accx[nt], al[ks], bh[2 * ks], bh[2 * ks + 1]);
          mma(acc[nt], ah[ks], bh[2 * ks], bh[2 * ks + 1]);
          mma(accx[nt], ah[ks], bl[2 * ks], bl[2 * ks + 1]);
        }
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[nt][r] += accx[nt][r];
    }
    float y0 = 0.f, y1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const float2 w = *reinterpret_cast<const float2*>(w2h + 8 * nt + 2 * t);
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[nt][r] = tanh_sfu(acc[nt][r]);
      y0 = fmaf(w.x, acc[nt][0], fmaf(w.y, acc[nt][1], y0));
      y1 = fmaf(w.x, acc[nt][2], fmaf(w.y, acc[nt][3], y1));
    }
    y0 += __shfl_xor_sync(0xffffffffu, y0, 1);
    y0 += __shfl_xor_sync(0xffffffffu, y0, 2);
    y1 += __shfl_xor_sync(0xffffffffu, y1, 1);
    y1 += __shfl_xor_sync(0xffffffffu, y1, 2);
    float* yb = S.ypart + ((pr * 2 + (it & 1)) * 2) * 16;  // [half][16 rows]
    if (t == 0) {
      yb[hh * 16 + g] = y0;
      yb[hh * 16 + g + 8] = y1;
    }
    asm volatile("bar.sync %0, 64;" ::"r"(1 + pr) : "memory");
    y0 = yb[g] + yb[16 + g];
    y1 = yb[g + 8] + yb[16 + g + 8];
    const int s0 = r0 + g, s1 = s0 + 8;
    const float e0 = s0 < cnt ? y0 + b2 - S.T[s0] : 0.f;
    const float e1 = s1 < cnt ? y1 + b2 - S.T[s1] : 0.f;
    const float dy0 = scale * e0, dy1 = scale * e1;
    if (t == 0 && hh == 0) {
      esum = fmaf(e0, e0, fmaf(e1, e1, esum));
      dysum += dy0 + dy1;
    }
    uint32_t th[4], tl[4], bh8[4], bl8[4];  // dz blocks: rows 0-7 / 8-15 of each n-tile
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const float2 w = *reinterpret_cast<const float2*>(w2h + 8 * nt + 2 * t);
      const float h0 = acc[nt][0], h1 = acc[nt][1], h2 = acc[nt][2], h3 = acc[nt][3];
      const float z0 = dy0 * w.x * (1.f - h0 * h0), z1 = dy0 * w.y * (1.f - h1 * h1);
      const float z2 = dy1 * w.x * (1.f - h2 * h2), z3 = dy1 * w.y * (1.f - h3 * h3);
      db1[2 * nt] += z0 + z2;
      db1[2 * nt + 1] += z1 + z3;
      dw2[2 * nt] = fmaf(dy0, h0, fmaf(dy1, h2, dw2[2 * nt]));
      dw2[2 * nt + 1] = fmaf(dy0, h1, fmaf(dy1, h3, dw2[2 * nt + 1]));
      split2(z0, z1, th[nt], tl[nt]);
      split2(z2, z3, bh8[nt], bl8[nt]);
    }
    uint32_t zb[2][4], zbl[2][4];  // Z as B (k = samples, n = inputs), two n-tiles per load
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      ldsm_x4_t(zh + zsw(r0 + lrow, 2 * p + lch), zb[p]);
      ldsm_x4_t(zl + zsw(r0 + lrow, 2 * p + lch), zbl[p]);
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const uint32_t a_h[4] = {movt(th[2 * mt]), movt(th[2 * mt + 1]), movt(bh8[2 * mt]),
                               movt(bh8[2 * mt + 1])};
      const uint32_t a_l[4] = {movt(tl[2 * mt]), movt(tl[2 * mt + 1]), movt(bl8[2 * mt]),
                               movt(bl8[2 * mt + 1])};
#pragma unroll
      for (int nq = 0; nq < 4; ++nq) {
        const uint32_t b0 = zb[nq >> 1][(nq & 1) * 2], b1 = zb[nq >> 1][(nq & 1) * 2 + 1];
        const uint32_t c0 = zbl[nq >> 1][(nq & 1) * 2], c1 = zbl[nq >> 1][(nq & 1) * 2 + 1];
        mma(dw[mt][nq], a_l, b0, b1);
        mma(dw[mt][nq], a_h, c0, c1);
        mma(dw[mt][nq], a_h, b0, b1);
      }
    }
  }
  // bias / output-weight columns: sum over the 8 row groups, then over pairs
#pragma unroll
  for (int k = 0; k < 8; ++k) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      db1[k] += __shfl_xor_sync(0xffffffffu, db1[k], o);
      dw2[k] += __shfl_xor_sync(0xffffffffu, dw2[k], o);
    }
  }
  if (lane < 4) {
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      float* cr = S.colred + pr * 128 + 32 * hh + 8 * nt + 2 * t;
      cr[0] = db1[2 * nt];
      cr[1] = db1[2 * nt + 1];
      cr[64] = dw2[2 * nt];
      cr[65] = dw2[2 * nt + 1];
    }
  }
  // dW1: fixed tree over pairs (p + 4, then + 2, then + 1), both halves at once
  auto ridx = [&](int mt, int nq, int r) { return ((mt * 4 + nq) * 4 + r) * 32 + lane; };
#pragma unroll 1
  for (int half = 4; half >= 1; half >>= 1) {
    __syncthreads();
    if (pr >= half && pr < 2 * half) {
      float* dst = S.red + (hh * 4 + (pr - half)) * 1024;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nq = 0; nq < 4; ++nq)
#pragma unroll
          for (int r = 0; r < 4; ++r) dst[ridx(mt, nq, r)] = dw[mt][nq][r];
    }
    __syncthreads();
    if (pr < half) {
      const float* src = S.red + (hh * 4 + pr) * 1024;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nq = 0; nq < 4; ++nq)
#pragma unroll
          for (int r = 0; r < 4; ++r) dw[mt][nq][r] += src[ridx(mt, nq, r)];
    }
  }
  if (pr == 0) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nq = 0; nq < 4; ++nq)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int j = 32 * hh + 16 * mt + g + (r >= 2 ? 8 : 0), q = 8 * nq + 2 * t + (r & 1);
          if (j < H && q < I) gout[j * I + q] = dw[mt][nq][r];
        }
  }
  if (threadIdx.x < 128) {
    const int col = threadIdx.x & 63, which = threadIdx.x >> 6;
    float s = 0.f;
    for (int p = 0; p < kPairs; ++p) s += S.colred[p * 128 + which * 64 + col];
    if (col < H) gout[H * I + which * H + col] = s;
  }
  // mse and db2 in one block reduction (warp sums -> red[w], red[16 + w])
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    esum += __shfl_xor_sync(0xffffffffu, esum, o);
    dysum += __shfl_xor_sync(0xffffffffu, dysum, o);
  }
  if (lane == 0) {
    red[warp] = esum;
    red[16 + warp] = dysum;
  }
  __syncthreads();
  if (warp == 0) {
    float a = lane < 16 ? red[lane] : 0.f, b = lane < 16 ? red[16 + lane] : 0.f;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) {
      S.scal[0] = a / static_cast<float>(cnt);
      gout[H * I + 2 * H] = b;
    }
  }
  __syncthreads();
  return S.scal[0];
}

}  // namespace tcs

__global__ void __launch_bounds__(tcs::kTcThreads, 1) narxg_train_tc_kernel(SweepArgs A) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ float red[32];
  __shared__ double redd[32];
  __shared__ int s_stall, s_epochs;
  __shared__ float s_sc[6];
  const int w = blockIdx.x;
  const int d = A.d, H = A.h, I = 3 * d + 2, L = A.L;
  const int P = H * I + 2 * H + 1;
  const int cnt = L - d;
  const int cntp = (cnt + 15) / 16 * 16;
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
  tcs::Smem S;
  S.zh = smraw;
  S.zl = S.zh + static_cast<size_t>(cntp) * 64;
  S.wh = S.zl + static_cast<size_t>(cntp) * 64;
  S.wl = S.wh + 4096;
  S.red = reinterpret_cast<float*>(S.wl + 4096);
  S.T = S.red + tcs::kRedFloats;
  float* wcur = S.T + cntp;
  float* wtr = wcur + P;
  float* g = wtr + P;
  float* gs = g + P;
  S.bw = gs + P;
  S.colred = S.bw + 128;
  S.ypart = S.colred + tcs::kPairs * 128;
  S.scal = S.ypart + tcs::kPairs * 64;
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
  for (int i = threadIdx.x; i < 2 * 4096 / 4; i += blockDim.x) reinterpret_cast<float*>(S.wh)[i] = 0.f;
  for (int i = threadIdx.x; i < 128; i += blockDim.x) S.bw[i] = 0.f;
  if (threadIdx.x == 0) {
    s_stall = 0;
    s_epochs = 0;
  }
  __syncthreads();
  // (x - mean) * (1 / std) in fp64: the reciprocal once instead of a
  // division per element (the prologue was ~3x longer)
  const double mv = s_sc[0], mc = s_sc[2], mm = s_sc[4];
  const double isv = 1.0 / s_sc[1], iscd = 1.0 / s_sc[3], ismm = 1.0 / s_sc[5];
  // Z rows as bf16 hi/lo, one (row, 8-input chunk) per work item
  for (int it = threadIdx.x; it < cntp * 4; it += blockDim.x) {
    const int i = it >> 2, ch = it & 3;
    float x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = ch * 8 + u;
      float val = 0.f;
      if (i < cnt && q < I) {
        const int tt = i + d;
        if (q < d) val = static_cast<float>((v[tt - 1 - q] - mv) * isv);
        else if (q <= 2 * d) val = static_cast<float>((c[tt - (q - d)] - mc) * iscd);
        else val = static_cast<float>((m[tt - (q - 2 * d - 1)] - mm) * ismm);
      }
      x[u] = val;
    }
    uint4 hv, lv;
    tcs::split2(x[0], x[1], hv.x, lv.x);
    tcs::split2(x[2], x[3], hv.y, lv.y);
    tcs::split2(x[4], x[5], hv.z, lv.z);
    tcs::split2(x[6], x[7], hv.w, lv.w);
    *reinterpret_cast<uint4*>(S.zh + tcs::zsw(i, ch)) = hv;
    *reinterpret_cast<uint4*>(S.zl + tcs::zsw(i, ch)) = lv;
    if (ch == 0) S.T[i] = i < cnt ? static_cast<float>((v[i + d] - mv) * isv) : 0.f;
  }
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    const float x = params[i];
    wcur[i] = x;
    tcs::stage_param(S, i, x, I, H);
  }
  __syncthreads();
  const float scale = 2.f / static_cast<float>(cnt);
  float current = tcs::eval_tc(S, wcur[P - 1], g, cnt, I, H, scale, red);
  const int max_ep = A.fixed_epochs > 0 ? A.fixed_epochs : A.cfg.max_epochs;
  for (int epoch = 0; epoch < max_ep; ++epoch) {
    float step = static_cast<float>(A.cfg.step);
    float next = 0.f;
    for (int halvings = 0;; ++halvings) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const float x = wcur[i] - step * g[i];
        wtr[i] = x;
        tcs::stage_param(S, i, x, I, H);
      }
      __syncthreads();
      next = tcs::eval_tc(S, wtr[P - 1], gs, cnt, I, H, scale, red);
      if (!(next > current) || halvings >= 20) break;
      step *= 0.5f;
    }
    if (next > current) break;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      wcur[i] = wtr[i];
      g[i] = gs[i];
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

#include "narx_umma.cuh"

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
  const size_t um_smem = sweep::ums::smem_bytes(cnt, P);
  if (um_smem <= 227 * 1024 && getenv("LBBSP_C4_UMMA")) {
    // tcgen05 trainer (narx_umma.cuh), opt-in: per evaluation it runs at the
    // warp-MMA trainer's speed (~16 us at L = 1000, W = 148) -- the
    // evaluation is bound by the per-tile epilogue chain (tanh, the y
    // exchange, dz), not by the MMAs (profiles/r02_c4_umma.txt)
    sweep::SweepArgs a{};
    a.W = W; a.L = L; a.d = delay; a.h = hidden; a.v = d_v; a.c = d_c; a.m = d_m;
    a.params = d_params; a.cfg = *cfg; a.fixed_epochs = fixed_epochs;
    a.epochs_out = d_epochs; a.loss_out = d_loss; a.scratch = d_scratch; a.smem_z = 1;
    LBBSP_CUDA_CHECK(cudaFuncSetAttribute(sweep::narxg_train_umma_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(um_smem)));
    sweep::narxg_train_umma_kernel<<<W, sweep::ums::kThreads, um_smem, static_cast<cudaStream_t>(stream)>>>(a);
    LBBSP_CUDA_CHECK(cudaGetLastError());
    return LBBSP_OK;
  }
  const size_t tc_smem = sweep::tcs::smem_bytes(cnt, P);
  if (tc_smem <= 227 * 1024) {
    sweep::SweepArgs a{};
    a.W = W; a.L = L; a.d = delay; a.h = hidden; a.v = d_v; a.c = d_c; a.m = d_m;
    a.params = d_params; a.cfg = *cfg; a.fixed_epochs = fixed_epochs;
    a.epochs_out = d_epochs; a.loss_out = d_loss; a.scratch = d_scratch; a.smem_z = 1;
    LBBSP_CUDA_CHECK(cudaFuncSetAttribute(sweep::narxg_train_tc_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(tc_smem)));
    sweep::narxg_train_tc_kernel<<<W, sweep::tcs::kTcThreads, tc_smem, static_cast<cudaStream_t>(stream)>>>(a);
    LBBSP_CUDA_CHECK(cudaGetLastError());
    return LBBSP_OK;
  }
  // long histories: CUDA-core trainer with Z streamed from global scratch
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
  if (sweep::tcs::smem_bytes(static_cast<int>(cnt), hidden * I + 2 * hidden + 1) <= 227 * 1024 ||
      sweep::ums::smem_bytes(static_cast<int>(cnt), hidden * I + 2 * hidden + 1) <= 227 * 1024)
    return 0;  // tensor-core trainers keep the training set in shared memory
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
