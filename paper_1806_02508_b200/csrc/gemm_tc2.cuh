// gemm_tc2.cuh -- CTA-pair variant of the gradient-engine GEMM for the large,
// ungrouped layers (C3: 4096-wide, one worker per GPU).
//
// Two CTAs of a (2,1,1) cluster compute one 256 x BN tile with
// tcgen05.mma.cta_group::2 (UMMA M=256): each CTA stages its 128 rows of A and
// its BN/2 rows of B per k-block (so a pair moves 1.5x fewer bytes from L2 per
// flop than a 128 x BN single-CTA tile), the leader CTA issues the MMAs, and
// each CTA drains its own 128 TMEM lanes. Barriers:
//   full[s]   leader only; both CTAs' TMA complete_tx on it (peer-bit masked)
//   empty[s]  per CTA; the leader's tcgen05.commit multicasts to both
//   tfull[a]  per CTA; multicast commit when the accumulator is final
//   tempty[a] leader only; 4 local + 4 remote epilogue-warp arrivals
#pragma once
#include "gemm_tc.cuh"

namespace lbbsp {
namespace tc {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA into this CTA's smem, transaction bytes counted on the LEADER's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* tm, uint64_t* bar,
                                                 int c0, int c1) {
  const uint32_t bar_leader = smem_u32(bar) & 0xFEFFFFFFu;  // peer bit cleared -> CTA 0
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar_leader), "r"(c0), "r"(c1)
      : "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
               : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(0x3))
      : "memory");
}

template <int BN>
struct Gemm2Smem {
  static constexpr int kABytes = kBM * kBK * 2;         // 128 rows of A per CTA
  static constexpr int kBBytes = (BN / 2) * kBK * 2;    // BN/2 rows of B per CTA
  static constexpr int kStageBytes = kABytes + kBBytes;
};

template <int BN, int STAGES>
constexpr size_t gemm2_smem_bytes() {
  return static_cast<size_t>(STAGES) * Gemm2Smem<BN>::kStageBytes + 1024 + 256;
}

template <int BN, bool A_MN, bool B_MN, int EPI, int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tc2_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
  static_assert(BN == 256 || BN == 128, "BN");
  constexpr int kStage = Gemm2Smem<BN>::kStageBytes;
  constexpr int kA = Gemm2Smem<BN>::kABytes;
  constexpr int kHalfN = BN / 2;
  constexpr uint32_t kIdesc = idesc_bf16_f32(2 * kBM, BN, A_MN, B_MN);
  constexpr int kTmemCols = 2 * BN <= 256 ? 256 : 512;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);  // 4 epilogue warps in each CTA of the pair
    }
    fence_barrier_init();
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) tmem_alloc_pair<kTmemCols>(tmem_base_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  pdl_wait();  // prologue above overlaps the previous kernel (programmatic launch)
  pdl_launch_dependents();
  // One worker per GPU (n_groups <= 1): its rows (kRows) or K range (kKSplit)
  // and its SM cap come from device memory, set by the round's plan kernel.
  // A k-split worker's K range is rounded up to the 64-row block; the rows
  // past its end are kept zero in the A operand by the producer of dZ.
  int cta_lo = 0, cta_n = gridDim.x, r0 = 0, r1 = args.mode == kRows ? args.M : args.K;
  if (args.n_groups == 1) {
    cta_lo = args.g_cta0[0];
    cta_n = args.g_ctan[0];
    r0 = args.g_r0[0];
    r1 = args.g_r1[0];
  }
  cta_lo &= ~1;
  cta_n &= ~1;
  if (cta_n < 2) cta_n = 2;
  const bool idle = static_cast<int>(blockIdx.x) < cta_lo || static_cast<int>(blockIdx.x) >= cta_lo + cta_n;
  const int pair = (static_cast<int>(blockIdx.x) - cta_lo) / 2, n_pairs = cta_n / 2;


  int m_begin, m_len, k_begin, k_len;
  if (args.mode == kRows) {
    m_begin = r0; m_len = r1 - r0; k_begin = 0; k_len = args.K;
  } else {
    m_begin = 0; m_len = args.M; k_begin = r0; k_len = r1 - r0;
  }
  const int m_tiles = m_len > 0 ? (m_len + 2 * kBM - 1) / (2 * kBM) : 0;
  const int n_tiles = (args.N + BN - 1) / BN;
  const int num_tiles = idle ? 0 : m_tiles * n_tiles;
  const int k_blocks = k_len > 0 ? (k_len + kBK - 1) / kBK : 0;
  const unsigned long long t_cta0 = globaltimer();
  if (!idle && args.timing && threadIdx.x == 0) atomicMin(&args.timing[0], t_cta0);

  if (warp == 0) {
    // ==================== TMA producer (both CTAs) ====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < num_tiles; t += n_pairs) {
        const int mt = t % m_tiles, nt = t / m_tiles;
        const int m0 = m_begin + mt * 2 * kBM + static_cast<int>(rank) * kBM;  // this CTA's 128 rows
        const int n0 = nt * BN + static_cast<int>(rank) * kHalfN;      // this CTA's BN/2 rows of B
        for (int kb = 0; kb < k_blocks; ++kb) {
          const int k0 = k_begin + kb * kBK;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStage;
          uint8_t* sb = sa + kA;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kStage);
          if (A_MN) {
            tma_load_2d_pair(sa, &tmA, &full[stage], m0, k0);
            tma_load_2d_pair(sa + 8192, &tmA, &full[stage], m0 + 64, k0);
          } else {
            tma_load_2d_pair(sa, &tmA, &full[stage], k0, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < kHalfN / 64; ++j)
              tma_load_2d_pair(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0);
          } else {
            tma_load_2d_pair(sb, &tmB, &full[stage], k0, n0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ==================== MMA issuer (leader CTA) ======================
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = pair; t < num_tiles; t += n_pairs) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_base = smem_u32(smem + stage * kStage), b_base = a_base + kA;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t adesc = A_MN ? umma_desc_sw128(a_base + k * 2048, 8192, 1024)
                                          : umma_desc_sw128(a_base + k * 32, 16, 1024);
              const uint64_t bdesc = B_MN ? umma_desc_sw128(b_base + k * 2048, 8192, 1024)
                                          : umma_desc_sw128(b_base + k * 32, 16, 1024);
              umma_bf16_pair(d_tmem, adesc, bdesc, kIdesc, (kb > 0 || k > 0) ? 1u : 0u);
            }
            umma_commit_pair_mc(&empty[stage]);
            if (kb == k_blocks - 1) umma_commit_pair_mc(&tfull[acc]);
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
    }
  } else {
    // ==================== epilogue (both CTAs) ==========================
    const int ew = warp % 4;
    const int row_in_tile = static_cast<int>(rank) * kBM + ew * 32 + lane;
    const uint32_t tempty_leader = mapa_shared(&tempty[0], 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = pair; t < num_tiles; t += n_pairs) {
      const int mt = t % m_tiles, nt = t / m_tiles;
      const int row = m_begin + mt * 2 * kBM + row_in_tile;
      const int n0 = nt * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const bool row_ok = row < m_begin + m_len;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + c, v);
        tmem_ld_wait();
        const int col0 = n0 + c;
        if (!row_ok || col0 >= args.N) continue;
        const bool full_cols = col0 + 32 <= args.N;
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
        if (EPI == kEpiF32) {
          float* dst = args.c_f32 + static_cast<long long>(row) * args.ldc + col0;
          if (full_cols && (args.ldc % 4 == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
          } else {
            for (int j = 0; j < 32 && col0 + j < args.N; ++j) dst[j] = f[j];
          }
          continue;
        }
        if (EPI == kEpiBiasReluBf16 || EPI == kEpiBiasBf16) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            f[j] += (col0 + j < args.N) ? args.bias[col0 + j] : 0.f;
            if (EPI == kEpiBiasReluBf16) f[j] = fmaxf(f[j], 0.f);
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
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty_leader + static_cast<uint32_t>(acc) * 8u);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<kTmemCols>(tmem_base);
  if (!idle && args.n_groups > 0) interfere(args.intf, 0, args.timing ? &args.timing[0] : nullptr, t_cta0);
  if (!idle && args.timing && threadIdx.x == 0)
    atomicMax(&args.timing[1], static_cast<unsigned long long>(globaltimer()));
}

}  // namespace tc
}  // namespace lbbsp
