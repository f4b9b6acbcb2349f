// gemm_tc.cuh -- the dense-layer GEMM of the per-worker gradient engine
// (north_star (1)): bf16 operands staged by TMA into 128B-swizzled shared
// memory, tcgen05.mma (M=128, N=BN, K=16) issued by one thread, fp32
// accumulators double-buffered in TMEM, fused epilogues read back with
// tcgen05.ld. Persistent and warp-specialised:
//   warp 0       TMA producer (one elected lane)
//   warp 1       TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5   epilogue (TMEM lanes 32*(w%4) .. +31)
//
// Emulated workers (one GPU hosting n workers): the launch's
// CTAs are partitioned per worker (a per-worker SM cap); a worker's tiles are
// processed only by its own CTAs. Ragged per-worker batches are masked, not
// padded to max b_i:
//   kRows   (forward / dX): worker g owns batch rows [r0_g, r1_g) of M; rows
//           past r1_g are dropped in the epilogue.
//   kKSplit (dW = dY^T X): worker g owns the K range [r0_g, r1_g); the rows of
//           the last K block past r1_g are zeroed in shared memory before the
//           MMA, and worker g's partial goes to its own fp32 slab (the
//           segmented reduction sums the slabs).
#pragma once
#include <cuda_bf16.h>

#include "interfere.cuh"
#include "tc_ptx.cuh"

namespace lbbsp {
namespace tc {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kGemmThreads = 192;

enum GemmMode { kRows = 0, kKSplit = 1 };
enum Epilogue {
  kEpiF32 = 0,          // C_f32 = acc
  kEpiBiasReluBf16 = 1, // C_bf16 = relu(acc + bias)
  kEpiBiasBf16 = 2,     // C_bf16 = acc + bias
  kEpiDReluBf16 = 3,    // C_bf16 = acc * (aux > 0)   (dX through ReLU)
  kEpiBiasReluBoth = 4, // C_bf16 = relu(acc + bias) and C_f32 = same (testing)
  kEpiBf16 = 5          // C_bf16 = acc (bf16 gradient buckets for the all-reduce)
};

struct GemmArgs {
  int M, N, K;
  int mode;
  // worker partition (device arrays, n_groups entries); n_groups == 0 means
  // one group covering the whole problem with every CTA.
  int n_groups;
  const int* g_r0;
  const int* g_r1;
  const int* g_cta0;
  const int* g_ctan;
  // epilogue
  float* c_f32;
  __nv_bfloat16* c_bf16;
  long long ldc;
  long long group_stride;  // kKSplit: elements between per-worker partial slabs
  const float* bias;
  const __nv_bfloat16* aux;
  long long ld_aux;
  // per-group phase timing (globaltimer ns): [n_groups][2] = {min start, max end}
  unsigned long long* timing;
  // straggler injection on the worker's own CTAs after its tiles (interfere.cuh)
  Interference intf;
};

template <int BN>
struct GemmSmem {
  static constexpr int kABytes = kBM * kBK * 2;  // 16 KB
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
};

template <int BN, int STAGES>
constexpr size_t gemm_smem_bytes() {
  return static_cast<size_t>(STAGES) * GemmSmem<BN>::kStageBytes + 1024 /*align*/ + 256;
}

__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }

template <int BN, bool A_MN, bool B_MN, int EPI, int STAGES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
  static_assert(BN % 64 == 0 && BN >= 64 && BN <= 256, "BN");
  constexpr int kStage = GemmSmem<BN>::kStageBytes;
  constexpr int kA = GemmSmem<BN>::kABytes;
  constexpr uint32_t kIdesc = idesc_bf16_f32(kBM, BN, A_MN, B_MN);
  constexpr int kTmemCols = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* grp_slot = reinterpret_cast<int*>(tmem_base_slot + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_base_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // the prologue above overlaps the previous kernel (programmatic launch);
  // everything below may read its outputs (A operand, groups from the plan)
  pdl_wait();
  pdl_launch_dependents();
  // ---- which worker (group) does this CTA serve? --------------------------------
  if (threadIdx.x == 0) {
    int g = -1, cta_in = 0, cta_cnt = gridDim.x;
    if (args.n_groups == 0) {
      g = 0;
      cta_in = blockIdx.x;
    } else {
      for (int i = 0; i < args.n_groups; ++i) {
        const int c0 = args.g_cta0[i], cn = args.g_ctan[i];
        if (static_cast<int>(blockIdx.x) >= c0 && static_cast<int>(blockIdx.x) < c0 + cn) {
          g = i;
          cta_in = blockIdx.x - c0;
          cta_cnt = cn;
          break;
        }
      }
    }
    grp_slot[0] = g;
    grp_slot[1] = cta_in;
    grp_slot[2] = cta_cnt;
  }
  __syncthreads();
  const uint32_t tmem_base = *tmem_base_slot;
  const int g = grp_slot[0], cta_in = grp_slot[1], cta_cnt = grp_slot[2];

  int r0 = 0, r1 = args.mode == kRows ? args.M : args.K;
  if (g >= 0 && args.n_groups > 0) {
    r0 = args.g_r0[g];
    r1 = args.g_r1[g];
  }
  // tile space of this group
  int m_begin, m_len, k_begin, k_len;
  if (args.mode == kRows) {
    m_begin = r0; m_len = r1 - r0; k_begin = 0; k_len = args.K;
  } else {
    m_begin = 0; m_len = args.M; k_begin = r0; k_len = r1 - r0;
  }
  const int m_tiles = m_len > 0 ? (m_len + kBM - 1) / kBM : 0;
  const int n_tiles = (args.N + BN - 1) / BN;
  const int num_tiles = g >= 0 ? m_tiles * n_tiles : 0;
  const int k_blocks = k_len > 0 ? (k_len + kBK - 1) / kBK : 0;

  const unsigned long long t_cta0 = globaltimer();
  if (g >= 0 && args.timing && threadIdx.x == 0) atomicMin(&args.timing[2 * g], t_cta0);

  if (warp == 0) {
    // =========================== TMA producer =============================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cta_in; t < num_tiles; t += cta_cnt) {
        const int mt = t % m_tiles, nt = t / m_tiles;
        const int m0 = m_begin + mt * kBM, n0 = nt * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          const int k0 = k_begin + kb * kBK;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStage;
          uint8_t* sb = sa + kA;
          mbar_arrive_expect_tx(&full[stage], kStage);
          if (A_MN) {  // global [K][M], boxes {64 (M), 64 (K)}
            tma_load_2d(sa, &tmA, &full[stage], m0, k0);
            tma_load_2d(sa + 8192, &tmA, &full[stage], m0 + 64, k0);
          } else {     // global [M][K], box {64 (K), 128 (M)}
            tma_load_2d(sa, &tmA, &full[stage], k0, m0);
          }
          if (B_MN) {  // global [K][N], boxes {64 (N), 64 (K)}
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0);
          } else {     // global [N][K], box {64 (K), BN (N)}
            tma_load_2d(sb, &tmB, &full[stage], k0, n0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // =========================== MMA issuer ===============================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cta_in; t < num_tiles; t += cta_cnt) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        uint8_t* sa = smem + stage * kStage;
        uint8_t* sb = sa + kA;
        // ragged K tail of this worker (kKSplit): zero the A rows past r1
        const int valid_k = k_len - kb * kBK;
        if (A_MN && args.mode == kKSplit && valid_k < kBK) {
          // A tile = 2 boxes x 64 K-rows x 128 B; a K row is one 128-B line
          for (int box = 0; box < 2; ++box) {
            uint4* p = reinterpret_cast<uint4*>(sa + box * 8192 + valid_k * 128);
            const int n16 = (kBK - valid_k) * 8;
            for (int i = lane; i < n16; i += 32) p[i] = make_uint4(0, 0, 0, 0);
          }
          fence_proxy_async_smem();
          __syncwarp();
        }
        if (lane == 0) {
          const uint32_t a_base = smem_u32(sa), b_base = smem_u32(sb);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            uint64_t adesc, bdesc;
            if (A_MN)  // K rows of 128 B; 8-row groups at 1024 B; 64-wide M blocks at 8 KB
              adesc = umma_desc_sw128(a_base + k * 2048, 8192, 1024);
            else       // 128-B rows (64 K); 8-row atoms at 1024 B; +32 B per K=16
              adesc = umma_desc_sw128(a_base + k * 32, 16, 1024);
            if (B_MN)
              bdesc = umma_desc_sw128(b_base + k * 2048, 8192, 1024);
            else
              bdesc = umma_desc_sw128(b_base + k * 32, 16, 1024);
            umma_bf16(d_tmem, adesc, bdesc, kIdesc, (kb > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);                   // smem slot free once MMAs read it
          if (kb == k_blocks - 1) umma_commit(&tfull[acc]);  // accumulator ready
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else {
    // =========================== epilogue =================================
    const int ew = warp % 4;           // TMEM lane quarter this warp may access
    const int row_in_tile = ew * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cta_in; t < num_tiles; t += cta_cnt) {
      const int mt = t % m_tiles, nt = t / m_tiles;
      const int row = m_begin + mt * kBM + row_in_tile;
      const int row_end = m_begin + m_len;
      const int n0 = nt * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const bool row_ok = row < row_end;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + c, v);
        tmem_ld_wait();
        const int col0 = n0 + c;
        if (!row_ok || col0 >= args.N) continue;
        const bool full_cols = col0 + 32 <= args.N;
        if (EPI == kEpiF32) {
          float* dst = args.c_f32 + (args.mode == kKSplit && args.n_groups > 0 ? g * args.group_stride : 0) +
                       static_cast<long long>(row) * args.ldc + col0;
          if (full_cols && (args.ldc % 4 == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(dst + j) =
                  make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                              __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
          } else {
            for (int j = 0; j < 32 && col0 + j < args.N; ++j) dst[j] = __uint_as_float(v[j]);
          }
        } else {
          float f[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
          if (EPI == kEpiBiasReluBf16 || EPI == kEpiBiasBf16 || EPI == kEpiBiasReluBoth) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float b = (col0 + j < args.N) ? args.bias[col0 + j] : 0.f;
              f[j] += b;
              if (EPI != kEpiBiasBf16) f[j] = fmaxf(f[j], 0.f);
            }
          } else if (EPI == kEpiDReluBf16) {
            const __nv_bfloat16* h = args.aux + static_cast<long long>(row) * args.ld_aux + col0;
            if (full_cols && (args.ld_aux % 8 == 0)) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                const uint4 hv = *reinterpret_cast<const uint4*>(h + j);
                const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&hv);
#pragma unroll
                for (int q = 0; q < 8; ++q) f[j + q] = bf2f(hb[q]) > 0.f ? f[j + q] : 0.f;
              }
            } else {
              for (int j = 0; j < 32; ++j) f[j] = (col0 + j < args.N && bf2f(h[j]) > 0.f) ? f[j] : 0.f;
            }
          }
          __nv_bfloat16* dst = args.c_bf16 + static_cast<long long>(row) * args.ldc + col0;
          if (full_cols && (args.ldc % 8 == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              uint4 pk;
              __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
              for (int q = 0; q < 4; ++q) p2[q] = __floats2bfloat162_rn(f[j + 2 * q], f[j + 2 * q + 1]);
              *reinterpret_cast<uint4*>(dst + j) = pk;
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < args.N; ++j) dst[j] = __float2bfloat16_rn(f[j]);
          }
          if (EPI == kEpiBiasReluBoth) {
            float* d32 = args.c_f32 + static_cast<long long>(row) * args.ldc + col0;
            for (int j = 0; j < 32 && col0 + j < args.N; ++j) d32[j] = f[j];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem_base);
  if (g >= 0 && args.n_groups > 0)
    interfere(args.intf, g, args.timing ? &args.timing[2 * g] : nullptr, t_cta0);
  if (g >= 0 && args.timing && threadIdx.x == 0)
    atomicMax(&args.timing[2 * g + 1], static_cast<unsigned long long>(globaltimer()));
}

}  // namespace tc
}  // namespace lbbsp
