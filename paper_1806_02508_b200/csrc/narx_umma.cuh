// narx_umma.cuh -- the C4 NARX sweep trainer on tcgen05 (included by
// narx_sweep.cu after the warp-MMA trainer; same algorithm, same split-bf16
// numerics: every operand x = hi + lo, every product hi*hi + hi*lo + lo*hi).
//
// One CTA per model, 288 threads: warp 0 allocates TMEM and issues the MMAs,
// warps 1-8 are the epilogue (TMEM lane quarter w % 4, hidden-unit half
// (w - 1) / 4). Per evaluation, over 128-sample tiles of the training set:
//   forward   A[s][j] = sum_q Z[s][q] W1[j][q]       tcgen05 M=128 N=64 K=64
//             with Z rows stored as [Zh(32) | Zl(32)] bf16 (one 128-B SW128
//             row per sample) against B1 rows [W1h_j | W1h_j] (K = 0..63:
//             Zh W1h + Zl W1h) and B2 rows [W1l_j | 0] (K = 0..31: Zh W1l);
//             two accumulators in TMEM, tile t+1's forward beside tile t's
//             epilogue
//   epilogue  h = tanh(A + b1), y = h w2 + b2 (the two halves' partial sums
//             added in half order), e, dy, dz = dy w2 (1 - h^2); dz -> smem
//             as the backward's A operand [dz_h ; dz_l] (M = 128, MN-major);
//             db1, dw2, mse, db2 accumulated per thread
//   backward  D += [dz_h ; dz_l]^T-by-sample x [Zh | Zl]   tcgen05 M=128 N=64,
//             K = the tile's 128 samples, both operands MN-major -- the Z rows
//             of the forward are the backward's B operand as they lie; D's
//             quadrants give dz_h Zh, dz_h Zl and dz_l Zh, and
//             dW1 = (dz_h Zh + dz_h Zl) + dz_l Zh in that order
// The per-thread db1 / dw2 partials are reduced across lanes by a transpose
// reduction (31 shuffles per 32 values) and across quarters in quarter order:
// every reduction has a fixed order, so training is deterministic.
// Inputs pad to 32 (I = 3d + 2 <= 32) and hidden units to 64 with zeros.
#pragma once

namespace ums {

using namespace lbbsp::tc;

constexpr int kThreads = 544;  // warp 0: MMA; warps 1-16: epilogue (lane quarter x 16-unit column group)
constexpr int kTile = 128;
constexpr int kMaxTiles = 8;       // training sets up to 1024 samples
constexpr int kZRow = 128;         // bytes per sample row: Zh (64 B) | Zl (64 B)
constexpr int kDzTile = 32768;     // [2 K-blocks][2 chunks (hi, lo)][64 samples][128 B]

struct Smem {
  uint8_t* z;      // [ntiles * 128][128 B] SW128
  uint8_t* b1;     // [64][128 B] SW128: W1h | W1h
  uint8_t* b2;     // [64][128 B] SW128: W1l | 0
  uint8_t* dz;     // kDzTile
  float* T;        // [ntiles * 128]
  float* bw;       // [2][64]: b1 | w2 of the staged weights
  float* ypart;    // [2 parity][2 halves][128]
  float* red;      // [8] x 4 scratch
  uint64_t* bars;  // tfull[2], tempty[2], dzfull, dzempty, bwfull
  uint32_t* tmem_slot;
  float* scal;
};

__host__ __device__ inline size_t smem_bytes(int cnt, int P) {
  const size_t tiles = (cnt + kTile - 1) / kTile;
  return 1024 /*align*/ + tiles * kTile * kZRow + 2 * 8192 + kDzTile + 4 * tiles * kTile +
         4 * (128 + 1024 + 32 + 4 * static_cast<size_t>(P)) + 128;
}

// byte offset of element (row, col) of a 128-B-row SW128 array (bf16 cols)
__device__ __forceinline__ int sw128(int row, int col) {
  return row * 128 + ((((col >> 3) ^ (row & 7))) << 4) + (col & 7) * 2;
}

// write parameter i (value x) of the staged weight set: W1 [H][I] -> B1 / B2
__device__ __forceinline__ void stage_param(const Smem& S, int i, float x, int I, int H) {
  if (i < H * I) {
    const int j = i / I, q = i - j * I;
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
    *reinterpret_cast<__nv_bfloat16*>(S.b1 + sw128(j, q)) = h;
    *reinterpret_cast<__nv_bfloat16*>(S.b1 + sw128(j, 32 + q)) = h;
    *reinterpret_cast<__nv_bfloat16*>(S.b2 + sw128(j, q)) = l;
  } else if (i < H * I + 2 * H) {
    const int k = i - H * I;
    S.bw[k < H ? k : 64 + (k - H)] = x;
  }
}

// lane l ends with the sum over the warp's lanes of v[l & 15] (fixed
// butterfly order: four halving steps, then the two lane halves)
__device__ __forceinline__ void transpose_reduce16(float v[16], int lane) {
#pragma unroll
  for (int step = 0; step < 4; ++step) {
    const int off = 8 >> step, n = 16 >> step;
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < n / 2; ++k) {
      const float send = up ? v[k] : v[k + n / 2];
      const float keep = up ? v[k + n / 2] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 16);
}
// 32 lanes x 16 consecutive 32-bit TMEM columns
__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

// mbarrier wait with a watchdog (50 ms): on timeout records `code` in *err
// and returns (the evaluation is then garbage, the kernel still terminates)
__device__ __forceinline__ void wait_wd(uint64_t* bar, uint32_t parity, int* err, int code) {
  const unsigned long long t0 = globaltimer();
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 100000;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (!ok && globaltimer() - t0 > 50000000ull) {
      if (*err == 0) *err = code;
      return;
    }
  }
}

// mse of the staged weights; gradient at them -> gout[P]
__device__ float eval_umma(const Smem& S, float b2, float* gout, int cnt, int I, int H, float scale, int* err) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (cnt + kTile - 1) / kTile;
  uint64_t* tfull = S.bars;
  uint64_t* tempty = S.bars + 2;
  uint64_t* dzfull = S.bars + 4;
  uint64_t* dzempty = S.bars + 5;
  uint64_t* bwfull = S.bars + 6;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 16);
    }
    mbar_init(dzfull, 16);
    mbar_init(dzempty, 1);
    mbar_init(bwfull, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();  // the staged weights -> the tensor cores
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *S.tmem_slot;
  float mse = 0.f, db2 = 0.f;
  if (warp == 0) {
    // ================= MMA issuer =================
    if (lane == 0) {
      constexpr uint32_t kIdF = idesc_bf16_f32(128, 64, false, false);
      constexpr uint32_t kIdB = idesc_bf16_f32(128, 64, true, true);
      const uint32_t z0 = smem_u32(S.z), b1 = smem_u32(S.b1), b2s = smem_u32(S.b2), dz = smem_u32(S.dz);
      auto fwd = [&](int t) {
        wait_wd(&tempty[t & 1], ((t >> 1) & 1) ^ 1, err, 100 + t);
        tc_fence_after();
        const uint32_t a = z0 + t * kTile * kZRow, d = tmem + (t & 1) * 64;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(d, umma_desc_sw128(a + k * 32, 16, 1024), umma_desc_sw128(b1 + k * 32, 16, 1024), kIdF,
                    k > 0 ? 1u : 0u);
#pragma unroll
        for (int k = 0; k < 2; ++k)
          umma_bf16(d, umma_desc_sw128(a + k * 32, 16, 1024), umma_desc_sw128(b2s + k * 32, 16, 1024), kIdF, 1u);
        umma_commit(&tfull[t & 1]);
      };
      fwd(0);
      for (int t = 0; t < ntiles; ++t) {
        if (t + 1 < ntiles) fwd(t + 1);
        wait_wd(dzfull, t & 1, err, 200 + t);
        tc_fence_after();
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t a = dz + kb * 16384 + k * 2048;
            const uint32_t bz = z0 + (t * kTile + kb * 64) * kZRow + k * 2048;
            umma_bf16(tmem + 128, umma_desc_sw128(a, 8192, 1024), umma_desc_sw128(bz, 8192, 1024), kIdB,
                      (t > 0 || kb > 0 || k > 0) ? 1u : 0u);
          }
        umma_commit(dzempty);
      }
      umma_commit(bwfull);
    }
    __syncwarp();
  } else {
    // ================= epilogue (warps 1-16) =================
    const int q = warp & 3, cg = (warp - 1) >> 2;  // TMEM lane quarter, 16-unit column group
    const int r = 32 * q + lane;  // sample row within the tile / TMEM lane
    const float* b1v = S.bw + 16 * cg;
    const float* w2v = S.bw + 64 + 16 * cg;
    float db1[16], dw2[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) db1[j] = dw2[j] = 0.f;
    for (int t = 0; t < ntiles; ++t) {
      wait_wd(&tfull[t & 1], (t >> 1) & 1, err, 300 + t);
      tc_fence_after();
      uint32_t v[16];
      tmem_ld_x16(tmem + (static_cast<uint32_t>(32 * q) << 16) + (t & 1) * 64 + 16 * cg, v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[t & 1]);
      float h[16];
      float yp = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        h[j] = tcs::tanh_sfu(__uint_as_float(v[j]) + b1v[j]);
        yp = fmaf(w2v[j], h[j], yp);
      }
      float* yb = S.ypart + (t & 1) * 512;
      yb[cg * 128 + r] = yp;
      epi_sync();
      const float y = ((yb[r] + yb[128 + r]) + yb[256 + r]) + yb[384 + r] + b2;
      const int s = t * kTile + r;
      const float e = s < cnt ? y - S.T[s] : 0.f;
      const float dy = scale * e;
      if (cg == 0) {
        mse = fmaf(e, e, mse);
        db2 += dy;
      }
      // the backward of tile t - 1 must have read the dz buffer
      if (t > 0) wait_wd(dzempty, (t - 1) & 1, err, 400 + t);
      const int kb = r >> 6, rr = r & 63;
      uint8_t* rowh = S.dz + kb * 16384 + rr * 128;
      uint8_t* rowl = rowh + 8192;
#pragma unroll
      for (int c = 0; c < 2; ++c) {  // 8 hidden units per 16-B chunk
        uint4 hv, lv;
        uint32_t* hp = reinterpret_cast<uint32_t*>(&hv);
        uint32_t* lp = reinterpret_cast<uint32_t*>(&lv);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j0 = 8 * c + 2 * u;
          const float z0 = dy * w2v[j0] * (1.f - h[j0] * h[j0]);
          const float z1 = dy * w2v[j0 + 1] * (1.f - h[j0 + 1] * h[j0 + 1]);
          db1[j0] += z0;
          db1[j0 + 1] += z1;
          dw2[j0] = fmaf(dy, h[j0], dw2[j0]);
          dw2[j0 + 1] = fmaf(dy, h[j0 + 1], dw2[j0 + 1]);
          tcs::split2(z0, z1, hp[u], lp[u]);
        }
        const int chunk = 2 * cg + c;  // hidden units 8 chunk .. 8 chunk + 7
        *reinterpret_cast<uint4*>(rowh + ((chunk ^ (rr & 7)) << 4)) = hv;
        *reinterpret_cast<uint4*>(rowl + ((chunk ^ (rr & 7)) << 4)) = lv;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(dzfull);
    }
    // ---- dW1 from the backward accumulator's quadrants ----
    // (the last tile's dz-free arrival too: the barriers are re-initialised at
    // the next evaluation, and a commit landing after that would shift its
    // phases by one -- a wait for a phase that never completes)
    wait_wd(dzempty, (ntiles - 1) & 1, err, 500);
    wait_wd(bwfull, 0, err, 600);
    tc_fence_after();
    // the dz buffer is free now: 3 x [64 hidden][33] floats of quadrants
    float* quad = reinterpret_cast<float*>(S.dz);
    {
      uint32_t v[16];
      tmem_ld_x16(tmem + (static_cast<uint32_t>(32 * q) << 16) + 128 + 16 * cg, v);
      tmem_ld_wait();
      // quarters 0-1: rows j = dz_h (cols 0-31 x Zh, 32-63 x Zl); quarters 2-3: dz_l (cols 0-31 x Zh)
      const int which = q < 2 ? (cg < 2 ? 0 : 1) : (cg < 2 ? 2 : -1);
      const int j = r & 63, c0 = (16 * cg) & 31;
      if (which >= 0)
#pragma unroll
        for (int c = 0; c < 16; ++c) quad[(which * 64 + j) * 33 + c0 + c] = __uint_as_float(v[c]);
    }
    // ---- db1 / dw2: lanes (samples) then quarters, in order ----
    transpose_reduce16(db1, lane);
    transpose_reduce16(dw2, lane);
    float* colred = quad + 3 * 64 * 33;  // [2 arrays][4 quarters][64 cols]
    if (lane < 16) {
      colred[(0 * 4 + q) * 64 + 16 * cg + lane] = db1[0];
      colred[(1 * 4 + q) * 64 + 16 * cg + lane] = dw2[0];
    }
    // ---- mse, db2: warp sums (column-group-0 warps hold them) ----
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mse += __shfl_xor_sync(0xffffffffu, mse, o);
      db2 += __shfl_xor_sync(0xffffffffu, db2, o);
    }
    if (lane == 0) {
      S.red[warp - 1] = mse;
      S.red[16 + warp - 1] = db2;
    }
    epi_sync();
    const int et = threadIdx.x - 32;  // 0..511
    for (int idx = et; idx < 64 * 32; idx += 512) {
      const int j = idx >> 5, c = idx & 31;
      const float g = (quad[j * 33 + c] + quad[(64 + j) * 33 + c]) + quad[(128 + j) * 33 + c];
      if (j < H && c < I) gout[j * I + c] = g;
    }
    if (et < 128) {
      const int which = et >> 6, col = et & 63;
      const float* cr = colred + which * 256;
      const float sum = ((cr[col] + cr[64 + col]) + cr[128 + col]) + cr[192 + col];
      if (col < H) gout[H * I + which * H + col] = sum;
    }
    if (et == 0) {
      float a = 0.f, b = 0.f;
      for (int w = 0; w < 16; ++w) {
        a += S.red[w];
        b += S.red[16 + w];
      }
      S.scal[0] = a / static_cast<float>(cnt);
      gout[H * I + 2 * H] = b;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  return S.scal[0];
}

}  // namespace ums

__global__ void __launch_bounds__(ums::kThreads, 1) narxg_train_umma_kernel(SweepArgs A) {
  using namespace lbbsp::tc;
  extern __shared__ __align__(1024) unsigned char smraw_u[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw_u) + 1023) & ~uintptr_t(1023));
  __shared__ double redd[32];
  __shared__ int s_stall, s_epochs;
  __shared__ float s_sc[6];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t tmem_slot;
  __shared__ int s_err;
  const int w = blockIdx.x;
  const int d = A.d, H = A.h, I = 3 * d + 2, L = A.L;
  const int P = H * I + 2 * H + 1;
  const int cnt = L - d;
  const int ntiles = (cnt + ums::kTile - 1) / ums::kTile;
  const int cntp = ntiles * ums::kTile;
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
  ums::Smem S;
  S.z = base;
  S.b1 = S.z + static_cast<size_t>(cntp) * ums::kZRow;
  S.b2 = S.b1 + 8192;
  S.dz = S.b2 + 8192;
  S.T = reinterpret_cast<float*>(S.dz + ums::kDzTile);
  S.bw = S.T + cntp;
  S.ypart = S.bw + 128;
  S.red = S.ypart + 1024;
  float* wcur = S.red + 32;
  float* wtr = wcur + P;
  float* g = wtr + P;
  float* gs = g + P;
  S.scal = gs + P;
  S.bars = bars;
  S.tmem_slot = &tmem_slot;
  if (threadIdx.x == 0) s_err = 0;
  if (threadIdx.x < 32) tmem_alloc<256>(&tmem_slot);
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
  for (int i = threadIdx.x; i < 2 * 8192 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(S.b1)[i] = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < 128; i += blockDim.x) S.bw[i] = 0.f;
  if (threadIdx.x == 0) {
    s_stall = 0;
    s_epochs = 0;
  }
  __syncthreads();
  const double mv = s_sc[0], mc = s_sc[2], mm = s_sc[4];
  const double isv = 1.0 / s_sc[1], iscd = 1.0 / s_sc[3], ismm = 1.0 / s_sc[5];
  // Z rows as [Zh | Zl] bf16 (SW128), one (row, 8-input chunk) per work item
  for (int it = threadIdx.x; it < cntp * 4; it += blockDim.x) {
    const int i = it >> 2, ch = it & 3;
    float x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int qq = ch * 8 + u;
      float val = 0.f;
      if (i < cnt && qq < I) {
        const int tt = i + d;
        if (qq < d) val = static_cast<float>((v[tt - 1 - qq] - mv) * isv);
        else if (qq <= 2 * d) val = static_cast<float>((c[tt - (qq - d)] - mc) * iscd);
        else val = static_cast<float>((m[tt - (qq - 2 * d - 1)] - mm) * ismm);
      }
      x[u] = val;
    }
    uint4 hv, lv;
    tcs::split2(x[0], x[1], hv.x, lv.x);
    tcs::split2(x[2], x[3], hv.y, lv.y);
    tcs::split2(x[4], x[5], hv.z, lv.z);
    tcs::split2(x[6], x[7], hv.w, lv.w);
    *reinterpret_cast<uint4*>(S.z + i * 128 + ((ch ^ (i & 7)) << 4)) = hv;
    *reinterpret_cast<uint4*>(S.z + i * 128 + (((4 + ch) ^ (i & 7)) << 4)) = lv;
    if (ch == 0) S.T[i] = i < cnt ? static_cast<float>((v[i + d] - mv) * isv) : 0.f;
  }
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    const float x = params[i];
    wcur[i] = x;
    ums::stage_param(S, i, x, I, H);
  }
  __syncthreads();
  const float scale = 2.f / static_cast<float>(cnt);
  float current = ums::eval_umma(S, wcur[P - 1], g, cnt, I, H, scale, &s_err);
  const int max_ep = A.fixed_epochs > 0 ? A.fixed_epochs : A.cfg.max_epochs;
  for (int epoch = 0; epoch < max_ep; ++epoch) {
    float step = static_cast<float>(A.cfg.step);
    float next = 0.f;
    for (int halvings = 0;; ++halvings) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const float x = wcur[i] - step * g[i];
        wtr[i] = x;
        ums::stage_param(S, i, x, I, H);
      }
      __syncthreads();
      next = ums::eval_umma(S, wtr[P - 1], gs, cnt, I, H, scale, &s_err);
      if (s_err) break;
      if (!(next > current) || halvings >= 20) break;
      step *= 0.5f;
    }
    if (next > current || s_err) break;
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
    A.epochs_out[w] = s_err ? -s_err : s_epochs;
    A.loss_out[w] = current;
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<256>(tmem_slot);
}
