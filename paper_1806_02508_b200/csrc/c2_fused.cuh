// c2_fused.cuh -- one persistent kernel for every emulated worker's whole
// gradient on the small-head MLP (784 -> 256 -> 10, BASELINE configs[0..1]):
//
//   phase F  (per 128-row M-tile of the worker's batch rows)
//     H   = relu(X W0^T + b0)          tcgen05 M=128 N=256 K=784, TMEM acc
//     head: logits, softmax-CE, dl, dW1 += dl^T H, dH = (dl W1) (H > 0),
//           db1, db0 (column sums)     warp MMA on the H tile in smem
//     dZ0 = dH  -> global (the dW0 operand)
//   worker barrier (the worker's head CTAs have published dZ0 and partials)
//   phase W  (per 128 x 128 tile of dW0 = dZ0^T X, K = the worker's rows)
//     tcgen05 M=128 N=128, MN-major operands, ragged K tail zeroed in smem
//   combine: the worker's CTAs sum the head CTA partials in CTA order
//
// Replaces the three launches per round (forward GEMM, head, dW GEMM) whose
// kernel boundaries synchronised every worker with every other worker at
// every phase; here a worker's CTAs advance on their own (the reference's
// workers are independent until the barrier, cluster_sim.cpp:422-431), and a
// worker's time is one window: its first CTA's start to its last CTA's end.
// Numerics are those of the separate kernels (same K order in every
// accumulation, same head code, same CTA-ordered combine), so the weights are
// bitwise those of the unfused path (tests/test_gpu_fused.py).
//
// Warp roles (320 threads): warps 0-7 epilogue + head (TMEM lane quarter w%4,
// column half w/4; head tile w), warp 8 TMA producer, warp 9 TMEM allocator +
// MMA issuer. Shared memory: 4 x 48 KB TMA stages; the phase-F H tile (8 x 8
// KB head tiles) and the end-of-phase reductions reuse the stage region while
// no TMA load is in flight (the producer waits for the head before it loads
// again); W1 fragments and dl tiles live beside it.
#pragma once
#include <cuda_bf16.h>

#include "head_mma.cuh"
#include "interfere.cuh"
#include "mlp_kernels.cuh"
#include "tc_ptx.cuh"

namespace lbbsp {
namespace mlp {

constexpr int kFzThreads = 320;
constexpr int kFzStages = 4;
constexpr int kFzStage = 48 * 1024;               // A 128x64 + B 256x64 bf16 (phase F)
constexpr int kFzD0 = 784;                        // input width
constexpr int kFzBNW = 128;                       // dW0 tile width
constexpr int kFzNTW = (kFzD0 + kFzBNW - 1) / kFzBNW;  // 7 dW0 column tiles
constexpr int kFzWTiles = 2 * kFzNTW;             // 14 dW0 tiles per worker
// dynamic smem layout (after 1024 alignment)
constexpr int kFzOffWl = kFzStages * kFzStage;    // head B fragments (logits)  8 KB
constexpr int kFzOffWd = kFzOffWl + 8192;         // head B fragments (dH)      8 KB
constexpr int kFzOffDl = kFzOffWd + 8192;         // dl tiles [8][16][16] bf16  4 KB
constexpr int kFzOffB0 = kFzOffDl + 4096;         // b0 [256] fp32              1 KB
constexpr int kFzOffBar = kFzOffB0 + 1024;        // mbarriers + slots
constexpr size_t kFzSmem = kFzOffBar + 256 + 1024;

struct FusedArgs {
  Groups G;
  __nv_bfloat16* dZ0;       // [B][256] dH of the batch rows (phase W operand)
  const float* W1;          // [10][256] fp32 master
  const float* b0;          // [256]
  const float* b1;          // [10]
  const int* y;             // [B] labels of the batch rows
  const float* row_scale;   // [B] Eq. 6/7 row scales
  float* slab;              // [n_local][P] worker gradient slabs
  long long slab_stride;
  long long off_w0, off_w1, off_b1, off_b0;
  float* head_part;         // [grid][kHeadPartVals] CTA partials
  unsigned* done;           // [n_local] head CTAs finished (zeroed by the round's plan)
  unsigned long long* timing;  // [n_local][2] worker window
  lbbsp_dev_status* status;
  unsigned long long* dbg;  // optional [grid][8] per-CTA stage stamps (globaltimer)
  // in-kernel row gather (c2_pair_worker_kernel, gather != 0): the batch rows
  // are read straight from the resident dataset by sample index -- X / y of
  // local row r are data_x / data_y [streams[k * B_total + *stream_off + r]]
  int gather;
  const int* streams;       // [max_rows][B_total] sample streams
  const long long* kptr;    // the round index (written by the observe branch)
  const int* stream_off;    // this rank's offset in the round's stream (plan)
  const int* data_y;        // [N_data] dataset labels
  int B_total, max_rows;
};

__device__ __forceinline__ void named_sync_epi() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__global__ void __launch_bounds__(kFzThreads, 1)
    c2_fused_worker_kernel(const __grid_constant__ CUtensorMap tmX,    // X [B][784], box {64,128}
                           const __grid_constant__ CUtensorMap tmW0,   // W0 [256][784], box {64,256}
                           const __grid_constant__ CUtensorMap tmDz,   // dZ0 [B][256] as [K][M], box {64,64}
                           const __grid_constant__ CUtensorMap tmXn,   // X [B][784] as [K][N], box {64,64}
                           FusedArgs A) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t fz_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fz_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kFzOffBar);
  uint64_t* empty = full + kFzStages;
  uint64_t* tfull = empty + kFzStages;   // [3]: phase F acc, phase W acc 0/1
  uint64_t* tempty = tfull + 3;          // [3]
  uint64_t* hdone = tempty + 3;          // head of an M-tile done: stage smem free again
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hdone + 1);
  int* grp = reinterpret_cast<int*>(tmem_slot + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const Groups& G = A.G;

  if (warp == 8 && lane == 0) {
    for (int s = 0; s < kFzStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 3; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);  // one arrive per epilogue warp
    }
    mbar_init(hdone, 1);
    fence_barrier_init();
    tma_prefetch(&tmX);
    tma_prefetch(&tmW0);
    tma_prefetch(&tmDz);
    tma_prefetch(&tmXn);
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  // W1 (fp32 master, final before the previous kernel started) -> bf16 head
  // B fragments, staged through the stage region (no TMA in flight yet)
  if (warp < 8) {
    const float* wraw = reinterpret_cast<const float*>(smem);
    for (int i = threadIdx.x; i < kHeadNC * kHeadDH / 4; i += 256)
      cp_async16(smem_addr(smem + 16 * i), A.W1 + 4 * i, 16);
    cp_async_commit();
    cp_async_wait<0>();
    named_sync_epi();
    uint2* wl = reinterpret_cast<uint2*>(smem + kFzOffWl);
    uint2* wd = reinterpret_cast<uint2*>(smem + kFzOffWd);
    auto wv = [&](int c, int j) { return c < kHeadNC ? wraw[c * kHeadDH + j] : 0.f; };
    for (int i = threadIdx.x; i < 16 * 2 * 32; i += 256) {
      const int l = i & 31, nt = (i >> 5) & 1, s = i >> 6;
      const int c = 8 * nt + (l >> 2), k = 16 * s + 2 * (l & 3);
      wl[i] = make_uint2(pack_bf16(wv(c, k), wv(c, k + 1)), pack_bf16(wv(c, k + 8), wv(c, k + 9)));
    }
    for (int i = threadIdx.x; i < 32 * 32; i += 256) {
      const int l = i & 31, j = i >> 5;
      const int n = 8 * j + (l >> 2), c = 2 * (l & 3);
      wd[i] = make_uint2(pack_bf16(wv(c, n), wv(c + 1, n)), pack_bf16(wv(c + 8, n), wv(c + 9, n)));
    }
    float* b0s = reinterpret_cast<float*>(smem + kFzOffB0);
    for (int i = threadIdx.x; i < kHeadDH; i += 256) b0s[i] = A.b0[i];
    fence_proxy_async_smem();  // the stage region is next written by TMA
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // X, labels, row scales, groups: written by the plan / gather
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    int g = -1, cta_in = 0, cnt = 1;
    for (int i = 0; i < G.n; ++i) {
      const int c0 = G.cta0[i], cn = G.ctan[i];
      if (static_cast<int>(blockIdx.x) >= c0 && static_cast<int>(blockIdx.x) < c0 + cn) {
        g = i;
        cta_in = blockIdx.x - c0;
        cnt = cn;
        break;
      }
    }
    grp[0] = g;
    grp[1] = cta_in;
    grp[2] = cnt;
  }
  __syncthreads();
  const uint32_t tmem = *tmem_slot;
  const int g = grp[0], cta_in = grp[1], cnt = grp[2];
  const unsigned long long t_cta0 = globaltimer();
  if (g >= 0 && A.timing && threadIdx.x == 0) atomicMin(&A.timing[2 * g], t_cta0);
  unsigned long long* dbg = A.dbg ? A.dbg + 16ull * blockIdx.x : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = t_cta0;
  const int r0 = g >= 0 ? G.r0[g] : 0, r1 = g >= 0 ? G.r1[g] : 0;
  const int rows = r1 - r0;
  const int n_mt = rows > 0 ? (rows + 127) / 128 : 0;
  const int head_ctas = n_mt < cnt ? n_mt : cnt;
  const int my_mt = g >= 0 && cta_in < n_mt ? (n_mt - cta_in + cnt - 1) / cnt : 0;
  const int k_blocks_w = rows > 0 ? (rows + 63) / 64 : 0;
  const int w_tiles = rows > 0 ? kFzWTiles : 0;  // an empty worker contributes dW0 = 0
  unsigned* done = A.done;

  if (warp == 8) {
    // ============================ TMA producer ============================
    if (lane == 0 && g >= 0) {
      int stage = 0;
      uint32_t ph = 0, hph = 0;
      for (int it = 0; it < my_mt; ++it) {
        const int m0 = r0 + (cta_in + it * cnt) * 128;
        if (it > 0) {  // the previous tile's head used the stage region
          mbar_wait(hdone, hph);
          hph ^= 1;
        }
        for (int kb = 0; kb < (kFzD0 + 63) / 64; ++kb) {
          mbar_wait(&empty[stage], ph ^ 1);
          uint8_t* sa = smem + stage * kFzStage;
          mbar_arrive_expect_tx(&full[stage], kFzStage);
          tma_load_2d(sa, &tmX, &full[stage], kb * 64, m0);
          tma_load_2d(sa + 16384, &tmW0, &full[stage], kb * 64, 0);
          if (++stage == kFzStages) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
      if (my_mt > 0) {
        mbar_wait(hdone, hph);
        hph ^= 1;
      }
      // worker barrier: every head CTA of this worker published dZ0
      const unsigned long long t0 = globaltimer();
      unsigned seen;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(done + g) : "memory");
        if (globaltimer() - t0 > 2000000000ull) {  // 2 s: never (a bug) -- fail, do not hang
          set_status(A.status, LBBSP_RUNTIME, 3, seen, head_ctas);
          break;
        }
      } while (seen < static_cast<unsigned>(head_ctas));
      fence_proxy_async_global();  // dZ0 (generic stores of other CTAs) -> TMA reads
      if (dbg) dbg[3] = globaltimer();
      for (int t = cta_in; t < w_tiles; t += cnt) {
        const int mt = t % 2, nt = t / 2;
        for (int kb = 0; kb < k_blocks_w; ++kb) {
          const int k0 = r0 + kb * 64;
          mbar_wait(&empty[stage], ph ^ 1);
          uint8_t* sa = smem + stage * kFzStage;
          mbar_arrive_expect_tx(&full[stage], 32768);
          tma_load_2d(sa, &tmDz, &full[stage], mt * 128, k0);
          tma_load_2d(sa + 8192, &tmDz, &full[stage], mt * 128 + 64, k0);
          tma_load_2d(sa + 16384, &tmXn, &full[stage], nt * 128, k0);
          tma_load_2d(sa + 24576, &tmXn, &full[stage], nt * 128 + 64, k0);
          if (++stage == kFzStages) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 9) {
    // ============================ MMA issuer ==============================
    if (g >= 0) {
      int stage = 0;
      uint32_t ph = 0, fph = 0;
      constexpr uint32_t kIdF = idesc_bf16_f32(128, 256, false, false);
      constexpr uint32_t kIdW = idesc_bf16_f32(128, 128, true, true);
      for (int it = 0; it < my_mt; ++it) {
        mbar_wait(&tempty[0], fph ^ 1);  // the previous tile's epilogue read the accumulator
        fph ^= 1;
        tc_fence_after();
        for (int kb = 0; kb < (kFzD0 + 63) / 64; ++kb) {
          mbar_wait(&full[stage], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a = smem_u32(smem + stage * kFzStage), b = a + 16384;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tmem, umma_desc_sw128(a + k * 32, 16, 1024), umma_desc_sw128(b + k * 32, 16, 1024),
                        kIdF, (kb > 0 || k > 0) ? 1u : 0u);
            umma_commit(&empty[stage]);
            if (kb == (kFzD0 + 63) / 64 - 1) umma_commit(&tfull[0]);
          }
          __syncwarp();
          if (++stage == kFzStages) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
      int acc = 0;
      uint32_t aph[2] = {0u, 0u};
      for (int t = cta_in; t < w_tiles; t += cnt) {
        mbar_wait(&tempty[1 + acc], aph[acc] ^ 1);
        aph[acc] ^= 1;
        tc_fence_after();
        const uint32_t d = tmem + 256 + acc * 128;
        for (int kb = 0; kb < k_blocks_w; ++kb) {
          mbar_wait(&full[stage], ph);
          tc_fence_after();
          uint8_t* sa = smem + stage * kFzStage;
          const int valid_k = rows - kb * 64;
          if (valid_k < 64) {  // ragged K tail: zero the A rows past the worker's end
            for (int box = 0; box < 2; ++box) {
              uint4* p = reinterpret_cast<uint4*>(sa + box * 8192 + valid_k * 128);
              const int n16 = (64 - valid_k) * 8;
              for (int i = lane; i < n16; i += 32) p[i] = make_uint4(0, 0, 0, 0);
            }
            fence_proxy_async_smem();
            __syncwarp();
          }
          if (lane == 0) {
            const uint32_t a = smem_u32(sa), b = a + 16384;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(d, umma_desc_sw128(a + k * 2048, 8192, 1024), umma_desc_sw128(b + k * 2048, 8192, 1024),
                        kIdW, (kb > 0 || k > 0) ? 1u : 0u);
            umma_commit(&empty[stage]);
            if (kb == k_blocks_w - 1) umma_commit(&tfull[1 + acc]);
          }
          __syncwarp();
          if (++stage == kFzStages) {
            stage = 0;
            ph ^= 1;
          }
        }
        acc ^= 1;
      }
    }
  } else if (g >= 0) {
    // ====================== epilogue + head (warps 0-7) =====================
    const int q = warp & 3, half = warp >> 2;
    const int gq = lane >> 2, tq = lane & 3;
    const uint2* wl = reinterpret_cast<const uint2*>(smem + kFzOffWl);
    const uint2* wd = reinterpret_cast<const uint2*>(smem + kFzOffWd);
    const float* b0s = reinterpret_cast<const float*>(smem + kFzOffB0);
    uint8_t* dls = smem + kFzOffDl + warp * 512;
    const float b_lo0 = A.b1[2 * tq], b_lo1 = A.b1[2 * tq + 1];
    const float b_hi0 = tq == 0 ? A.b1[8] : 0.f, b_hi1 = tq == 0 ? A.b1[9] : 0.f;
    float dw[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) dw[j][0] = dw[j][1] = dw[j][2] = dw[j][3] = 0.f;
    float dbh[4] = {0.f, 0.f, 0.f, 0.f};
    float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint32_t fph = 0;
    for (int it = 0; it < my_mt; ++it) {
      const int m0 = r0 + (cta_in + it * cnt) * 128;
      // labels and row scales of this warp's head rows: independent of the
      // forward, loaded while the tensor core runs it
      const int tile = warp;
      const int row0 = m0 + tile * 16;
      const bool have = row0 < r1;
      const int ra = row0 + gq, rb = row0 + gq + 8;
      const bool va = ra < r1, vb = rb < r1;
      const int ya = have && va ? A.y[ra] : -1, yb = have && vb ? A.y[rb] : -1;
      const float rsa = have && va ? A.row_scale[ra] : 0.f;
      const float rsb = have && vb ? A.row_scale[rb] : 0.f;
      // ---- H = bf16(relu(acc + b0)) -> the head's swizzled 16-row tiles ----
      mbar_wait(&tfull[0], fph);
      fph ^= 1;
      tc_fence_after();
      if (dbg && threadIdx.x == 0 && it == 0) dbg[1] = globaltimer();
      const int r = 32 * q + lane;  // row of the M-tile this thread reads
      uint8_t* htile = smem + (r >> 4) * 8192;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int col0 = half * 128 + c * 32;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(32 * q) << 16) + col0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 pk;
          uint32_t* p = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float a0 = fmaxf(__uint_as_float(v[j + 2 * u]) + b0s[col0 + j + 2 * u], 0.f);
            const float a1 = fmaxf(__uint_as_float(v[j + 2 * u + 1]) + b0s[col0 + j + 2 * u + 1], 0.f);
            p[u] = pack_bf16(a0, a1);
          }
          *reinterpret_cast<uint4*>(htile + hsw(r & 15, (col0 + j) >> 3)) = pk;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[0]);
      named_sync_epi();  // the whole H tile is in smem
      if (dbg && threadIdx.x == 0 && it == 0) dbg[6] = globaltimer();
      // ---- head on tile `warp` (rows m0 + 16 warp ..): head_mma.cuh, one iteration ----
      const uint32_t hb = smem_addr(smem + tile * 8192);
      uint8_t* hp = smem + tile * 8192;
      uint32_t ad[4] = {0u, 0u, 0u, 0u};
      const int mi = lane >> 3, lr = (lane & 7) + (mi & 1) * 8;
      if (have) {
        float lo[4] = {0.f, 0.f, 0.f, 0.f}, hi[4] = {0.f, 0.f, 0.f, 0.f};
        float lo2[4] = {0.f, 0.f, 0.f, 0.f}, hi2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int s = 0; s < 16; s += 2) {
          uint32_t a[4], a2[4];
          ldsm_x4(hb + hsw(lr, 2 * s + (mi >> 1)), a);
          ldsm_x4(hb + hsw(lr, 2 * s + 2 + (mi >> 1)), a2);
          const uint2 w0 = wl[(s * 2 + 0) * 32 + lane], w1 = wl[(s * 2 + 1) * 32 + lane];
          const uint2 w2 = wl[(s * 2 + 2) * 32 + lane], w3 = wl[(s * 2 + 3) * 32 + lane];
          mma16816(lo, a, w0.x, w0.y);
          mma16816(hi, a, w1.x, w1.y);
          mma16816(lo2, a2, w2.x, w2.y);
          mma16816(hi2, a2, w3.x, w3.y);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          lo[e] += lo2[e];
          hi[e] += hi2[e];
        }
        lo[0] += b_lo0; lo[1] += b_lo1; lo[2] += b_lo0; lo[3] += b_lo1;
        hi[0] += b_hi0; hi[1] += b_hi1; hi[2] += b_hi0; hi[3] += b_hi1;
        const bool hv = tq == 0;
        float ma = fmaxf(lo[0], lo[1]), mb = fmaxf(lo[2], lo[3]);
        if (hv) {
          ma = fmaxf(ma, fmaxf(hi[0], hi[1]));
          mb = fmaxf(mb, fmaxf(hi[2], hi[3]));
        }
        ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, 1));
        ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, 2));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 1));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 2));
        float pl[4], ph[4];
        pl[0] = __expf(lo[0] - ma); pl[1] = __expf(lo[1] - ma);
        pl[2] = __expf(lo[2] - mb); pl[3] = __expf(lo[3] - mb);
        ph[0] = hv ? __expf(hi[0] - ma) : 0.f; ph[1] = hv ? __expf(hi[1] - ma) : 0.f;
        ph[2] = hv ? __expf(hi[2] - mb) : 0.f; ph[3] = hv ? __expf(hi[3] - mb) : 0.f;
        float sa = pl[0] + pl[1] + ph[0] + ph[1], sb = pl[2] + pl[3] + ph[2] + ph[3];
        sa += __shfl_xor_sync(0xffffffffu, sa, 1);
        sa += __shfl_xor_sync(0xffffffffu, sa, 2);
        sb += __shfl_xor_sync(0xffffffffu, sb, 1);
        sb += __shfl_xor_sync(0xffffffffu, sb, 2);
        const int c0 = 2 * tq, c1 = 2 * tq + 1, c2 = 8 + 2 * tq, c3 = 9 + 2 * tq;
        const float sca = rsa / sa, scb = rsb / sb;
        float dlo[4], dhi[4];
        dlo[0] = pl[0] * sca - (c0 == ya ? rsa : 0.f);
        dlo[1] = pl[1] * sca - (c1 == ya ? rsa : 0.f);
        dlo[2] = pl[2] * scb - (c0 == yb ? rsb : 0.f);
        dlo[3] = pl[3] * scb - (c1 == yb ? rsb : 0.f);
        dhi[0] = hv ? ph[0] * sca - (c2 == ya ? rsa : 0.f) : 0.f;
        dhi[1] = hv ? ph[1] * sca - (c3 == ya ? rsa : 0.f) : 0.f;
        dhi[2] = hv ? ph[2] * scb - (c2 == yb ? rsb : 0.f) : 0.f;
        dhi[3] = hv ? ph[3] * scb - (c3 == yb ? rsb : 0.f) : 0.f;
        dbh[0] += dlo[0] + dlo[2];
        dbh[1] += dlo[1] + dlo[3];
        dbh[2] += dhi[0] + dhi[2];
        dbh[3] += dhi[1] + dhi[3];
        ad[0] = pack_bf16(dlo[0], dlo[1]);
        ad[1] = pack_bf16(dlo[2], dlo[3]);
        ad[2] = pack_bf16(dhi[0], dhi[1]);
        ad[3] = pack_bf16(dhi[2], dhi[3]);
        *reinterpret_cast<uint32_t*>(dls + gq * 32 + 4 * tq) = ad[0];
        *reinterpret_cast<uint32_t*>(dls + (gq + 8) * 32 + 4 * tq) = ad[1];
        *reinterpret_cast<uint32_t*>(dls + gq * 32 + 16 + 4 * tq) = ad[2];
        *reinterpret_cast<uint32_t*>(dls + (gq + 8) * 32 + 16 + 4 * tq) = ad[3];
      }
      named_sync_epi();  // every tile's dl and H are in smem
      // ---- dW1[:, 32 warp .. +32) += dl_t^T H_t over the tile's 8 row groups ----
#pragma unroll 1
      for (int t = 0; t < 8; ++t) {
        if (m0 + 16 * t >= r1) break;
        uint32_t at[4];
        ldsm_x4_t(smem_addr(smem + kFzOffDl + t * 512) + ((lane & 7) + (mi >> 1) * 8) * 32 + (mi & 1) * 16, at);
        const uint32_t ht = smem_addr(smem + t * 8192);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          uint32_t b[4];
          ldsm_x4_t(ht + hsw(lr, 2 * (2 * warp + p) + (mi >> 1)), b);
          mma16816(dw[2 * p], at, b[0], b[1]);
          mma16816(dw[2 * p + 1], at, b[2], b[3]);
        }
      }
      named_sync_epi();  // H tiles may now be overwritten by dH
      if (have) {
        // ---- dH = (dl W1) * (H > 0), in place over the H tile ----
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float d[4] = {0.f, 0.f, 0.f, 0.f};
          const uint2 wj = wd[j * 32 + lane];
          mma16816(d, ad, wj.x, wj.y);
          uint32_t* pa = reinterpret_cast<uint32_t*>(hp + hsw(gq, j) + 4 * tq);
          uint32_t* pb = reinterpret_cast<uint32_t*>(hp + hsw(gq + 8, j) + 4 * tq);
          const __nv_bfloat162 ha = *reinterpret_cast<const __nv_bfloat162*>(pa);
          const __nv_bfloat162 hbv = *reinterpret_cast<const __nv_bfloat162*>(pb);
          *pa = pack_bf16(__low2float(ha) > 0.f ? d[0] : 0.f, __high2float(ha) > 0.f ? d[1] : 0.f);
          *pb = pack_bf16(__low2float(hbv) > 0.f ? d[2] : 0.f, __high2float(hbv) > 0.f ? d[3] : 0.f);
        }
        __syncwarp();
        // ---- dZ0 rows (coalesced) + db0 column sums ----
#pragma unroll 4
        for (int qq = 0; qq < 16; ++qq) {
          const int rr = row0 + qq;
          if (rr >= r1) break;
          const uint4 v = *reinterpret_cast<const uint4*>(hp + hsw(qq, lane));
          *reinterpret_cast<uint4*>(A.dZ0 + static_cast<long long>(rr) * kHeadDH + lane * 8) = v;
          const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            cs[2 * u] += __low2float(e[u]);
            cs[2 * u + 1] += __high2float(e[u]);
          }
        }
      }
      __syncwarp();
      // the producer may refill the stage region once every warp is done with it
      fence_proxy_async_smem();
      named_sync_epi();
      if (dbg && threadIdx.x == 0 && it == 0) dbg[7] = globaltimer();
      if (threadIdx.x == 0) mbar_arrive(hdone);
    }
    if (my_mt > 0) {
      // ---- CTA partials (head_mma.cuh layout) -> head_part[blockIdx.x] ----
      constexpr int kSmallVals = kHeadPartVals - kHeadFrag;
      float* part = A.head_part + static_cast<long long>(blockIdx.x) * kHeadPartVals;
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int e = 0; e < 4; ++e) part[((4 * warp + p) * 4 + e) * 32 + lane] = dw[p][e];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float v = dbh[u];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        dbh[u] = v;
      }
      // the stage region is free until the producer passes the worker barrier,
      // which needs this CTA's partials first
      float* red = reinterpret_cast<float*>(smem);
      float* mine = red + warp * kSmallVals;
#pragma unroll
      for (int u = 0; u < 4; ++u) mine[u * 32 + lane] = dbh[u];
#pragma unroll
      for (int u = 0; u < 8; ++u) mine[128 + u * 32 + lane] = cs[u];
      named_sync_epi();
      for (int k = threadIdx.x; k < kSmallVals; k += 256) {
        float v = red[k];
#pragma unroll
        for (int w = 1; w < 8; ++w) v += red[w * kSmallVals + k];
        part[kHeadFrag + k] = v;
      }
      fence_proxy_async_smem();
      __threadfence();
      named_sync_epi();
      if (threadIdx.x == 0) atomicAdd(done + g, 1u);  // release: dZ0 rows + partials
      if (dbg && threadIdx.x == 0) dbg[2] = globaltimer();
    }
    // ---- phase W epilogue: dW0 tiles -> the worker's fp32 slab ----
    float* dst = A.slab + static_cast<long long>(g) * A.slab_stride + A.off_w0;
    int acc = 0;
    uint32_t aph[2] = {0u, 0u};
    if (rows == 0 && cta_in == 0)
      for (int i = threadIdx.x; i < kHeadDH * kFzD0; i += 256) dst[i] = 0.f;
    for (int t = cta_in; t < w_tiles; t += cnt) {
      const int mt = t % 2, nt = t / 2;
      mbar_wait(&tfull[1 + acc], aph[acc]);
      aph[acc] ^= 1;
      tc_fence_after();
      const int row = mt * 128 + 32 * q + lane;  // dW0 row (hidden unit)
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int cl = half * 64 + c * 32;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(32 * q) << 16) + 256 + acc * 128 + cl, v);
        tmem_ld_wait();
        const int col0 = nt * 128 + cl;
        if (col0 >= kFzD0) continue;
        float* o = dst + static_cast<long long>(row) * kFzD0 + col0;
        if (col0 + 32 <= kFzD0) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(o + j) = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                                            __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
        } else {
          for (int j = 0; j < 32 && col0 + j < kFzD0; ++j) o[j] = __uint_as_float(v[j]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[1 + acc]);
      acc ^= 1;
    }
  }
  if (dbg && threadIdx.x == 0) dbg[4] = globaltimer();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc<512>(tmem);
  // ---- combine: the head CTA partials summed in CTA order (head_combine's
  // order), the worker's CTAs splitting the values between them; every head
  // partial was published before this CTA's producer passed the barrier ----
  if (g >= 0) {
    const int cbase = blockIdx.x - cta_in;
    const int per = (kHeadPartVals + cnt - 1) / cnt;
    const int k0 = cta_in * per, k1 = min(kHeadPartVals, k0 + per);
    float* gs = A.slab + static_cast<long long>(g) * A.slab_stride;
    for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      float x[4];
      float v = 0.f;
      for (int c4 = 0; c4 < head_ctas; c4 += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          x[u] = c4 + u < head_ctas ? __ldcg(&A.head_part[static_cast<long long>(cbase + c4 + u) * kHeadPartVals + k]) : 0.f;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c4 + u < head_ctas) v += x[u];
      }
      const int i = head_frag_to_natural(k);
      if (i < 0) continue;
      const long long o = i < kHeadNC * kHeadDH ? A.off_w1 + i
                          : i < kHeadNC * kHeadDH + kHeadNC ? A.off_b1 + (i - kHeadNC * kHeadDH)
                                                            : A.off_b0 + (i - kHeadNC * kHeadDH - kHeadNC);
      gs[o] = v;
    }
    if (dbg && threadIdx.x == 0) dbg[5] = globaltimer();
    interfere(G.intf, g, A.timing ? &A.timing[2 * g] : nullptr, t_cta0);
    if (A.timing && threadIdx.x == 0) atomicMax(&A.timing[2 * g + 1], static_cast<unsigned long long>(globaltimer()));
  }
}

}  // namespace mlp
}  // namespace lbbsp
