// c2_fused_pair.cuh -- the fused worker kernel (c2_fused.cuh) with each
// 128-row tile's forward and head split across a (2,1,1) CTA cluster by
// hidden columns: CTA r of the pair computes H[:, 128r .. 128r+128) (tcgen05
// M=128 N=128 K=784 -- half the MMA work and half the W0 bytes of the
// single-CTA tile), its partial logits over those columns, and exchanges them
// with the peer through distributed shared memory; both CTAs add the two
// partials (p0 + p1, the same bits on both) and run softmax-CE on identical
// logits, then each forms dW1, dH = (dl W1) (H > 0), dZ0 and db0 for its own
// columns (db1 by CTA 0 only). Phase W (dW0 = dZ0^T X) and the ordered head
// combine are as in c2_fused.cuh. The worker's latency -- the quantity a
// straggler's 1/a multiplies -- drops with the halved per-CTA tile work.
//
// Worker CTA partitions must be cluster-aligned (even first CTA, even count);
// the plan rounds the caps down to even when this kernel is selected.
#pragma once
#include <cuda_bf16.h>

#include "c2_fused.cuh"
#include "gemm_tc2.cuh"

namespace lbbsp {
namespace mlp {

constexpr int kFpThreads = 320;
constexpr int kFpStages = 4;                       // phase W ring (stage region)
constexpr int kFpStagesF = 6;                      // phase F ring: + 2 stages in the (idle) W staging region
constexpr int kFpStage = 32 * 1024;                // A 128x64 + B 128x64 bf16
constexpr int kFpPartVals = 2048 + 128 + 128;      // dW1 frag | db1 frag | db0 (own 128 cols)
// dynamic smem layout (after 1024 alignment)
constexpr int kFpOffWl = kFpStages * kFpStage;     // logits B fragments (own cols)   4 KB
constexpr int kFpOffWd = kFpOffWl + 4096;          // dH B fragments (own cols)       4 KB
constexpr int kFpOffDl = kFpOffWd + 4096;          // dl tiles [8][16][16] bf16       4 KB
constexpr int kFpOffB0 = kFpOffDl + 4096;          // b0 (own 128 cols) fp32          512 B
constexpr int kFpOffXl = kFpOffB0 + 512;           // peer partial logits [2][8][32][8] f32  16 KB
constexpr int kFpOffFlag = kFpOffXl + 16384;       // [8] peer arrival sequence numbers
constexpr int kFpOffEpi = (kFpOffFlag + 64 + 1023) / 1024 * 1024;  // phase-W tile staging [4][128][32] f32 SW128, 64 KB
constexpr int kFpOffBar = kFpOffEpi + 65536;      // mbarriers + slots
constexpr size_t kFpSmem = kFpOffBar + 256 + 1024;
static_assert(kFpOffEpi % 1024 == 0, "SW128 staging must be 1 KB aligned");
static_assert(kFpSmem <= 232448, "pair kernel exceeds the 227 KB dynamic smem limit");

// byte offset of (row, 16-B chunk) in a swizzled 16 x 256 B tile (128 bf16 columns)
__device__ __forceinline__ int hsw2(int row, int chunk) { return row * 256 + ((chunk ^ (row & 7)) << 4); }

// fragment-order partial index -> natural index for column half r (dW1
// [class][col] | db1 [class] | db0 [col]), -1 for padded / not-owned entries
__device__ __forceinline__ int pair_frag_to_natural(int k, int r) {
  if (k < 2048) {
    const int w = k >> 8, p = (k >> 7) & 1, e = (k >> 5) & 3, l = k & 31;
    const int cls = (l >> 2) + (e >= 2 ? 8 : 0), col = 128 * r + 16 * w + 8 * p + 2 * (l & 3) + (e & 1);
    return cls < kHeadNC ? cls * kHeadDH + col : -1;
  }
  if (k < 2048 + 128) {
    if (r != 0) return -1;
    const int u = (k - 2048) >> 5, l = k & 31;
    const int cls = (u < 2 ? 2 * l + u : 8 + 2 * l + (u - 2));
    return ((l >> 2) == 0 && (u < 2 || l == 0)) ? kHeadNC * kHeadDH + cls : -1;
  }
  const int j = k - 2048 - 128, u = j >> 4, c = j & 15;
  return kHeadNC * kHeadDH + kHeadNC + 128 * r + 8 * c + u;
}

// TMA store of a {32, 128, 1} fp32 box from 128B-swizzled smem (bulk group)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tm)),
               "r"(tc::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_release_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cluster_u32(const void* p) {
  uint32_t v;
  asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(tc::smem_u32(p)) : "memory");
  return v;
}

// phase F stage s: the four W stages, then two 32 KB blocks of the W staging
// region (idle until phase W, which starts after this CTA's last head)
__device__ __forceinline__ uint8_t* fp_stage_f(uint8_t* smem, int s) {
  return s < kFpStages ? smem + s * kFpStage : smem + kFpOffEpi + (s - kFpStages) * kFpStage;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFpThreads, 1)
    c2_pair_worker_kernel(const __grid_constant__ CUtensorMap tmX,    // X [B][784], box {64,128}; gather: dataset, box {64,1}
                          const __grid_constant__ CUtensorMap tmW0h,  // W0 [256][784], box {64,128}
                          const __grid_constant__ CUtensorMap tmDz,   // dZ0 [B][256] as [K][M], box {64,64}
                          const __grid_constant__ CUtensorMap tmXn,   // X [B][784] as [K][N], box {64,64}; gather: = tmX
                          const __grid_constant__ CUtensorMap tmOut,  // slabs [n_local][256][784] f32, box {32,128,1}
                          FusedArgs A) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t fp_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fp_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kFpOffBar);
  uint64_t* empty = full + kFpStages;
  uint64_t* tfull = empty + kFpStages;  // [3]: phase F acc, phase W acc 0/1
  uint64_t* tempty = tfull + 3;         // [3]
  uint64_t* hdone = tempty + 3;
  uint64_t* fullF = hdone + 1;           // [kFpStagesF] phase F ring
  uint64_t* emptyF = fullF + kFpStagesF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(emptyF + kFpStagesF);
  int* grp = reinterpret_cast<int*>(tmem_slot + 1);
  uint32_t* flag = reinterpret_cast<uint32_t*>(smem + kFpOffFlag);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank(), peer = rank ^ 1u;
  const Groups& G = A.G;

  if (warp == 8 && lane == 0) {
    for (int s = 0; s < kFpStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 3; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);
    }
    mbar_init(hdone, 1);
    for (int s = 0; s < kFpStagesF; ++s) {
      mbar_init(&fullF[s], 1);
      mbar_init(&emptyF[s], 1);
    }
    fence_barrier_init();
    tma_prefetch(&tmX);
    tma_prefetch(&tmW0h);
    tma_prefetch(&tmDz);
    tma_prefetch(&tmXn);
    tma_prefetch(&tmOut);
  }
  if (warp < 8 && lane == 0) flag[warp] = 0u;
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  // W1 (fp32 master) -> bf16 B fragments of this CTA's 128 columns, staged
  // through the stage region (no TMA in flight yet); b0 of its columns
  if (warp < 8) {
    const float* wraw = reinterpret_cast<const float*>(smem);
    for (int i = threadIdx.x; i < kHeadNC * kHeadDH / 4; i += 256)
      cp_async16(smem_addr(smem + 16 * i), A.W1 + 4 * i, 16);
    cp_async_commit();
    cp_async_wait<0>();
    named_sync_epi();
    uint2* wl = reinterpret_cast<uint2*>(smem + kFpOffWl);
    uint2* wd = reinterpret_cast<uint2*>(smem + kFpOffWd);
    const int cb = 128 * static_cast<int>(rank);
    auto wv = [&](int c, int j) { return c < kHeadNC ? wraw[c * kHeadDH + cb + j] : 0.f; };
    for (int i = threadIdx.x; i < 8 * 2 * 32; i += 256) {  // [8 k-steps][2 class tiles][32 lanes]
      const int l = i & 31, nt = (i >> 5) & 1, s = i >> 6;
      const int c = 8 * nt + (l >> 2), k = 16 * s + 2 * (l & 3);
      wl[i] = make_uint2(pack_bf16(wv(c, k), wv(c, k + 1)), pack_bf16(wv(c, k + 8), wv(c, k + 9)));
    }
    for (int i = threadIdx.x; i < 16 * 32; i += 256) {  // [16 n8 tiles][32 lanes]
      const int l = i & 31, j = i >> 5;
      const int n = 8 * j + (l >> 2), c = 2 * (l & 3);
      wd[i] = make_uint2(pack_bf16(wv(c, n), wv(c + 1, n)), pack_bf16(wv(c + 8, n), wv(c + 9, n)));
    }
    float* b0s = reinterpret_cast<float*>(smem + kFpOffB0);
    for (int i = threadIdx.x; i < 128; i += 256) b0s[i] = A.b0[cb + i];
    fence_proxy_async_smem();
  }
  tc_fence_before();
  cluster_sync_all();  // barriers and flags of both CTAs initialised before any remote access
  tc_fence_after();
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    int g = -1, cta_in = 0, cnt = 2;
    for (int i = 0; i < G.n; ++i) {
      const int c0 = G.cta0[i], cn = G.ctan[i] & ~1;
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
  const int pair = cta_in >> 1, n_pairs = cnt >> 1;
  const unsigned long long t_cta0 = globaltimer();
  if (g >= 0 && A.timing && threadIdx.x == 0) atomicMin(&A.timing[2 * g], t_cta0);
  unsigned long long* dbg = A.dbg ? A.dbg + 16ull * blockIdx.x : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = t_cta0;
  const int r0 = g >= 0 ? G.r0[g] : 0, r1 = g >= 0 ? G.r1[g] : 0;
  const int rows = r1 - r0;
  const int n_mt = rows > 0 ? (rows + 127) / 128 : 0;
  const int head_ctas = 2 * (n_mt < n_pairs ? n_mt : n_pairs);
  const int my_mt = g >= 0 && pair < n_mt ? (n_mt - pair + n_pairs - 1) / n_pairs : 0;
  const int k_blocks_w = rows > 0 ? (rows + 63) / 64 : 0;
  const int w_tiles = rows > 0 ? kFzWTiles : 0;
  unsigned* done = A.done;
  // in-kernel row gather: local row r of this rank's batch is dataset row
  // gidx[r] (rows past the round's stream read row 0; they are masked)
  const int* gidx = nullptr;
  int gmax = 0;
  if (A.gather && g >= 0 && warp != 9) {
    long long k = *A.kptr;
    k = k < A.max_rows - 1 ? k : A.max_rows - 1;
    const int off = *A.stream_off;
    gidx = A.streams + k * A.B_total + off;
    gmax = A.B_total - off;
  }

  if (warp == 8) {
    // ============================ TMA producer ============================
    // Lane 0 issues the W0 / dZ0 tiles; with the in-kernel gather every lane
    // issues one tile::gather4 of four batch rows per stage (X straight from
    // the resident dataset -- no gathered copy of the batch in HBM).
    if (g >= 0) {
      int stage = 0, fs = 0;
      uint32_t ph = 0, hph = 0, fph = 0;
      if (dbg && lane == 0) dbg[13] = globaltimer();
      for (int it = 0; it < my_mt; ++it) {
        const int m0 = r0 + (pair + it * n_pairs) * 128;
        int gr[4] = {0, 0, 0, 0};
        if (gidx) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int rr = m0 + 4 * lane + u;
            gr[u] = rr < gmax ? __ldg(gidx + rr) : 0;
          }
        }
        if (it > 0) {
          mbar_wait(hdone, hph);
          hph ^= 1;
        }
        for (int kb = 0; kb < (kFzD0 + 63) / 64; ++kb) {
          mbar_wait(&emptyF[fs], fph ^ 1);
          uint8_t* sa = fp_stage_f(smem, fs);
          if (lane == 0) {
            mbar_arrive_expect_tx(&fullF[fs], kFpStage);
            tma_load_2d(sa + 16384, &tmW0h, &fullF[fs], kb * 64, 128 * static_cast<int>(rank));
            if (!gidx) tma_load_2d(sa, &tmX, &fullF[fs], kb * 64, m0);
          }
          __syncwarp();
          if (gidx) tma_gather4(sa + 512 * lane, &tmX, &fullF[fs], kb * 64, gr[0], gr[1], gr[2], gr[3]);
          if (++fs == kFpStagesF) {
            fs = 0;
            fph ^= 1;
          }
        }
      }
      if (my_mt > 0) {
        mbar_wait(hdone, hph);
        hph ^= 1;
      }
      // phase W's X operand does not depend on the worker barrier: the first
      // ring stages get their X halves now, their dZ0 halves after it (the
      // stage region is idle once the last head is done; the head partials'
      // reduction below uses only its first 8 KB, the X halves start at 16 KB)
      const int my_w = w_tiles > cta_in ? ((w_tiles - cta_in + cnt - 1) / cnt) * k_blocks_w : 0;
      const int n_pre = gidx ? 0 : (my_w < kFpStages ? my_w : kFpStages);
      if (lane == 0) {
        for (int i = 0; i < n_pre; ++i) {
          const int t = cta_in + (i / k_blocks_w) * cnt, kb = i % k_blocks_w;
          uint8_t* sa = smem + i * kFpStage;
          mbar_arrive_expect_tx(&full[i], 32768);
          tma_load_2d(sa + 16384, &tmXn, &full[i], (t / 2) * 128, r0 + kb * 64);
          tma_load_2d(sa + 24576, &tmXn, &full[i], (t / 2) * 128 + 64, r0 + kb * 64);
        }
      }
      if (lane == 0) {
        const unsigned long long t0 = globaltimer();
        unsigned seen;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(done + g) : "memory");
          if (globaltimer() - t0 > 2000000000ull) {
            set_status(A.status, LBBSP_RUNTIME, 3, seen, head_ctas);
            break;
          }
        } while (seen < static_cast<unsigned>(head_ctas));
        fence_proxy_async_global();
        if (dbg) dbg[3] = globaltimer();
      }
      // the worker's row indices -> the (now idle) peer-logit region; every
      // head CTA of the worker, the peer included, has finished writing it
      int* sidx = reinterpret_cast<int*>(smem + kFpOffXl);
      const bool sidx_ok = gidx && k_blocks_w * 64 <= (kFpOffFlag - kFpOffXl) / 4;
      if (w_tiles > 0 && sidx_ok) {
        for (int i = lane; i < k_blocks_w * 64; i += 32) {
          const int rr = r0 + i;
          sidx[i] = rr < gmax ? __ldg(gidx + rr) : 0;
        }
      }
      __syncwarp();
      int wi = 0;
      for (int t = cta_in; t < w_tiles; t += cnt) {
        const int mt = t % 2, nt = t / 2;
        for (int kb = 0; kb < k_blocks_w; ++kb, ++wi) {
          const int k0 = r0 + kb * 64;
          uint8_t* sa = smem + stage * kFpStage;
          if (wi < n_pre) {  // X already in flight
            if (lane == 0) {
              tma_load_2d(sa, &tmDz, &full[stage], mt * 128, k0);
              tma_load_2d(sa + 8192, &tmDz, &full[stage], mt * 128 + 64, k0);
            }
            if (++stage == kFpStages) {
              stage = 0;
              ph ^= 1;
            }
            continue;
          }
          mbar_wait(&empty[stage], ph ^ 1);
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[stage], 32768);
            tma_load_2d(sa, &tmDz, &full[stage], mt * 128, k0);
            tma_load_2d(sa + 8192, &tmDz, &full[stage], mt * 128 + 64, k0);
            if (!gidx) {
              tma_load_2d(sa + 16384, &tmXn, &full[stage], nt * 128, k0);
              tma_load_2d(sa + 24576, &tmXn, &full[stage], nt * 128 + 64, k0);
            }
          }
          __syncwarp();
          if (gidx) {
            const int box = lane >> 4, q4 = lane & 15;
            int rr[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = kb * 64 + 4 * q4 + u;
              rr[u] = sidx_ok ? sidx[i] : (r0 + i < gmax ? __ldg(gidx + r0 + i) : 0);
            }
            tma_gather4(sa + 16384 + box * 8192 + q4 * 512, &tmXn, &full[stage], nt * 128 + 64 * box, rr[0],
                        rr[1], rr[2], rr[3]);
          }
          if (++stage == kFpStages) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 9) {
    // ============================ MMA issuer ==============================
    if (g >= 0) {
      int stage = 0, fs = 0;
      uint32_t ph = 0, fph = 0, sph = 0;
      constexpr uint32_t kIdF = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t kIdW = idesc_bf16_f32(128, 128, true, true);
      for (int it = 0; it < my_mt; ++it) {
        mbar_wait(&tempty[0], fph ^ 1);
        fph ^= 1;
        tc_fence_after();
        for (int kb = 0; kb < (kFzD0 + 63) / 64; ++kb) {
          mbar_wait(&fullF[fs], sph);
          tc_fence_after();
          if (dbg && lane == 0 && it == 0 && kb == 0) dbg[11] = globaltimer();
          if (dbg && lane == 0 && it == 0 && kb == (kFzD0 + 63) / 64 - 1) dbg[12] = globaltimer();
          if (lane == 0) {
            const uint32_t a = smem_u32(fp_stage_f(smem, fs)), b = a + 16384;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tmem, umma_desc_sw128(a + k * 32, 16, 1024), umma_desc_sw128(b + k * 32, 16, 1024), kIdF,
                        (kb > 0 || k > 0) ? 1u : 0u);
            umma_commit(&emptyF[fs]);
            if (kb == (kFzD0 + 63) / 64 - 1) umma_commit(&tfull[0]);
          }
          __syncwarp();
          if (++fs == kFpStagesF) {
            fs = 0;
            sph ^= 1;
          }
        }
      }
      int acc = 0;
      uint32_t aph[2] = {0u, 0u};
      for (int t = cta_in; t < w_tiles; t += cnt) {
        mbar_wait(&tempty[1 + acc], aph[acc] ^ 1);
        aph[acc] ^= 1;
        tc_fence_after();
        const uint32_t d = tmem + 128 + acc * 128;
        for (int kb = 0; kb < k_blocks_w; ++kb) {
          mbar_wait(&full[stage], ph);
          tc_fence_after();
          if (dbg && lane == 0 && t == cta_in && kb == 0) dbg[8] = globaltimer();
          if (dbg && lane == 0 && t == cta_in && kb == k_blocks_w - 1) dbg[9] = globaltimer();
          uint8_t* sa = smem + stage * kFpStage;
          const int valid_k = rows - kb * 64;
          if (valid_k < 64) {
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
          if (++stage == kFpStages) {
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
    const uint2* wl = reinterpret_cast<const uint2*>(smem + kFpOffWl);
    const uint2* wd = reinterpret_cast<const uint2*>(smem + kFpOffWd);
    const float* b0s = reinterpret_cast<const float*>(smem + kFpOffB0);
    uint8_t* dls = smem + kFpOffDl + warp * 512;
    const float b_lo0 = A.b1[2 * tq], b_lo1 = A.b1[2 * tq + 1];
    const float b_hi0 = tq == 0 ? A.b1[8] : 0.f, b_hi1 = tq == 0 ? A.b1[9] : 0.f;
    // the peer's copy of my partial-logit slot and arrival flag
    const uint32_t xl_peer = mapa_shared(smem + kFpOffXl, peer);
    const uint32_t flag_peer = mapa_shared(flag + warp, peer);
    float dw[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j) dw[j][0] = dw[j][1] = dw[j][2] = dw[j][3] = 0.f;
    float dbh[4] = {0.f, 0.f, 0.f, 0.f};
    float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint32_t fph = 0;
    for (int it = 0; it < my_mt; ++it) {
      const int m0 = r0 + (pair + it * n_pairs) * 128;
      const int tile = warp;
      const int row0 = m0 + tile * 16;
      const bool have = row0 < r1;
      const int ra = row0 + gq, rb = row0 + gq + 8;
      const bool va = ra < r1, vb = rb < r1;
      const int ya = have && va ? (gidx ? A.data_y[gidx[ra]] : A.y[ra]) : -1;
      const int yb = have && vb ? (gidx ? A.data_y[gidx[rb]] : A.y[rb]) : -1;
      const float rsa = have && va ? A.row_scale[ra] : 0.f;
      const float rsb = have && vb ? A.row_scale[rb] : 0.f;
      // ---- H[:, own 128 columns] = bf16(relu(acc + b0)) -> 16 x 256 B head tiles ----
      mbar_wait(&tfull[0], fph);
      fph ^= 1;
      tc_fence_after();
      if (dbg && threadIdx.x == 0 && it == 0) dbg[1] = globaltimer();
      const int r = 32 * q + lane;
      uint8_t* htile = smem + (r >> 4) * 4096;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int col0 = half * 64 + c * 32;
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
          *reinterpret_cast<uint4*>(htile + hsw2(r & 15, (col0 + j) >> 3)) = pk;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[0]);
      named_sync_epi();
      if (dbg && threadIdx.x == 0 && it == 0) dbg[6] = globaltimer();
      const uint32_t hb = smem_addr(smem + tile * 4096);
      uint8_t* hp = smem + tile * 4096;
      uint32_t ad[4] = {0u, 0u, 0u, 0u};
      const int mi = lane >> 3, lr = (lane & 7) + (mi & 1) * 8;
      // ---- partial logits over the own 128 columns, exchanged with the peer ----
      float lo[4] = {0.f, 0.f, 0.f, 0.f}, hi[4] = {0.f, 0.f, 0.f, 0.f};
      if (have) {
        float lo2[4] = {0.f, 0.f, 0.f, 0.f}, hi2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int s = 0; s < 8; s += 2) {
          uint32_t a[4], a2[4];
          ldsm_x4(hb + hsw2(lr, 2 * s + (mi >> 1)), a);
          ldsm_x4(hb + hsw2(lr, 2 * s + 2 + (mi >> 1)), a2);
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
      }
      {
        const int buf = it & 1;
        const uint32_t slot = xl_peer + static_cast<uint32_t>(((buf * 8 + warp) * 32 + lane) * 32);
        st_cluster_v4(slot, make_float4(lo[0], lo[1], lo[2], lo[3]));
        st_cluster_v4(slot + 16, make_float4(hi[0], hi[1], hi[2], hi[3]));
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        __syncwarp();
        if (lane == 0) st_release_cluster_u32(flag_peer, static_cast<uint32_t>(it + 1));
        const unsigned long long tw = globaltimer();
        while (ld_acquire_cluster_u32(flag + warp) < static_cast<uint32_t>(it + 1)) {
          if (globaltimer() - tw > 2000000000ull) {  // 2 s: the peer never arrived -- fail, do not hang
            if (lane == 0) set_status(A.status, LBBSP_RUNTIME, 4, it, warp);
            break;
          }
        }
        const float* mine = reinterpret_cast<const float*>(smem + kFpOffXl) + ((buf * 8 + warp) * 32 + lane) * 8;
        // p0 + p1: fp addition commutes, so both CTAs hold the same bits
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          lo[e] += mine[e];
          hi[e] += mine[4 + e];
        }
      }
      if (have) {
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
        if (rank == 0) {  // db1 once per pair
          dbh[0] += dlo[0] + dlo[2];
          dbh[1] += dlo[1] + dlo[3];
          dbh[2] += dhi[0] + dhi[2];
          dbh[3] += dhi[1] + dhi[3];
        }
        ad[0] = pack_bf16(dlo[0], dlo[1]);
        ad[1] = pack_bf16(dlo[2], dlo[3]);
        ad[2] = pack_bf16(dhi[0], dhi[1]);
        ad[3] = pack_bf16(dhi[2], dhi[3]);
        *reinterpret_cast<uint32_t*>(dls + gq * 32 + 4 * tq) = ad[0];
        *reinterpret_cast<uint32_t*>(dls + (gq + 8) * 32 + 4 * tq) = ad[1];
        *reinterpret_cast<uint32_t*>(dls + gq * 32 + 16 + 4 * tq) = ad[2];
        *reinterpret_cast<uint32_t*>(dls + (gq + 8) * 32 + 16 + 4 * tq) = ad[3];
      }
      named_sync_epi();
      // ---- dW1[:, own cols 16 warp .. +16) += dl_t^T H_t over the 8 row groups ----
#pragma unroll 1
      for (int t = 0; t < 8; ++t) {
        if (m0 + 16 * t >= r1) break;
        uint32_t at[4];
        ldsm_x4_t(smem_addr(smem + kFpOffDl + t * 512) + ((lane & 7) + (mi >> 1) * 8) * 32 + (mi & 1) * 16, at);
        const uint32_t ht = smem_addr(smem + t * 4096);
        uint32_t b[4];
        ldsm_x4_t(ht + hsw2(lr, 2 * warp + (mi >> 1)), b);
        mma16816(dw[0], at, b[0], b[1]);
        mma16816(dw[1], at, b[2], b[3]);
      }
      named_sync_epi();
      if (have) {
        // ---- dH[:, own cols] = (dl W1) * (H > 0), in place over the H tile ----
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float d[4] = {0.f, 0.f, 0.f, 0.f};
          const uint2 wj = wd[j * 32 + lane];
          mma16816(d, ad, wj.x, wj.y);
          uint32_t* pa = reinterpret_cast<uint32_t*>(hp + hsw2(gq, j) + 4 * tq);
          uint32_t* pb = reinterpret_cast<uint32_t*>(hp + hsw2(gq + 8, j) + 4 * tq);
          const __nv_bfloat162 ha = *reinterpret_cast<const __nv_bfloat162*>(pa);
          const __nv_bfloat162 hbv = *reinterpret_cast<const __nv_bfloat162*>(pb);
          *pa = pack_bf16(__low2float(ha) > 0.f ? d[0] : 0.f, __high2float(ha) > 0.f ? d[1] : 0.f);
          *pb = pack_bf16(__low2float(hbv) > 0.f ? d[2] : 0.f, __high2float(hbv) > 0.f ? d[3] : 0.f);
        }
        __syncwarp();
        // ---- dZ0 rows (own 256 B per row, two rows per instruction) + db0 sums ----
        const int hq = lane >> 4, ch = lane & 15;
#pragma unroll 4
        for (int qq = 0; qq < 16; qq += 2) {
          const int rr = row0 + qq + hq;
          if (rr < r1) {
            const uint4 v = *reinterpret_cast<const uint4*>(hp + hsw2(qq + hq, ch));
            *reinterpret_cast<uint4*>(A.dZ0 + static_cast<long long>(rr) * kHeadDH + 128 * rank + ch * 8) = v;
            const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              cs[2 * u] += __low2float(e[u]);
              cs[2 * u + 1] += __high2float(e[u]);
            }
          }
        }
      }
      __syncwarp();
      fence_proxy_async_smem();
      named_sync_epi();
      if (dbg && threadIdx.x == 0 && it == 0) dbg[7] = globaltimer();
      if (threadIdx.x == 0) mbar_arrive(hdone);
    }
    if (my_mt > 0) {
      // ---- CTA partials -> head_part[blockIdx.x] (pair_frag_to_natural layout) ----
      float* part = A.head_part + static_cast<long long>(blockIdx.x) * kFpPartVals;
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int e = 0; e < 4; ++e) part[((2 * warp + p) * 4 + e) * 32 + lane] = dw[p][e];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float v = dbh[u];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        dbh[u] = v;
      }
      // db0: lanes l and l + 16 hold the same 8 columns (rows of opposite parity)
#pragma unroll
      for (int u = 0; u < 8; ++u) cs[u] += __shfl_xor_sync(0xffffffffu, cs[u], 16);
      float* red = reinterpret_cast<float*>(smem);  // stage region: free until the barrier
      float* mine = red + warp * 256;
#pragma unroll
      for (int u = 0; u < 4; ++u) mine[u * 32 + lane] = dbh[u];
      if (lane < 16)
#pragma unroll
        for (int u = 0; u < 8; ++u) mine[128 + u * 16 + lane] = cs[u];
      named_sync_epi();
      for (int k = threadIdx.x; k < 256; k += 256) {
        float v = red[k];
#pragma unroll
        for (int w = 1; w < 8; ++w) v += red[w * 256 + k];
        part[2048 + k] = v;
      }
      fence_proxy_async_smem();
      __threadfence();
      named_sync_epi();
      if (threadIdx.x == 0) atomicAdd(done + g, 1u);
      if (dbg && threadIdx.x == 0) dbg[2] = globaltimer();
    }
    // ---- phase W epilogue: dW0 tiles -> the worker's fp32 slab by TMA store
    // (the accumulator goes through 128B-swizzled smem boxes of 32 columns;
    // per-thread row stores would write 16 B into a different line per lane) ----
    float* dst = A.slab + static_cast<long long>(g) * A.slab_stride + A.off_w0;
    uint8_t* epi = smem + kFpOffEpi;
    int acc = 0;
    uint32_t aph[2] = {0u, 0u};
    if (rows == 0 && cta_in == 0)
      for (int i = threadIdx.x; i < kHeadDH * kFzD0; i += 256) dst[i] = 0.f;
    for (int t = cta_in; t < w_tiles; t += cnt) {
      const int mt = t % 2, nt = t / 2;
      mbar_wait(&tfull[1 + acc], aph[acc]);
      aph[acc] ^= 1;
      tc_fence_after();
      if (dbg && threadIdx.x == 0 && t == cta_in) dbg[10] = globaltimer();
      const int r = 32 * q + lane;  // row of the 128-row output tile
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int cc = half * 2 + c;  // 32-column box of the tile
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(32 * q) << 16) + 128 + acc * 128 + cc * 32, v);
        tmem_ld_wait();
        uint8_t* box = epi + cc * 16384 + r * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(box + ((j ^ (r & 7)) << 4)) =
              make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[1 + acc]);
      fence_proxy_async_smem();
      named_sync_epi();
      if (threadIdx.x == 0) {
        for (int cc = 0; cc < 4; ++cc) {
          const int col = nt * 128 + cc * 32;
          if (col < kFzD0) tma_store_3d(&tmOut, epi + cc * 16384, col, mt * 128, g);
        }
        bulk_commit();
        bulk_wait_read0();  // the staging boxes may be rewritten by the next tile
      }
      named_sync_epi();
      acc ^= 1;
    }
    // the staging smem must outlive the stores' reads; their global writes are
    // complete by the grid's end, before any dependent launch reads the slab
    if (threadIdx.x == 0) bulk_wait_read0();
  }
  if (dbg && threadIdx.x == 0) dbg[4] = globaltimer();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc<512>(tmem);
  // ---- combine: head partials summed per column half in pair order ----
  if (g >= 0) {
    const int cbase = blockIdx.x - cta_in;
    const int per = (2 * kFpPartVals + cnt - 1) / cnt;  // (half, k) pairs split over the worker's CTAs
    const int j0 = cta_in * per, j1 = min(2 * kFpPartVals, j0 + per);
    float* gs = A.slab + static_cast<long long>(g) * A.slab_stride;
    for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      const int rr = j / kFpPartVals, k = j % kFpPartVals;
      const int i = pair_frag_to_natural(k, rr);
      if (i < 0) continue;
      float v = 0.f;
      for (int p4 = 0; p4 < head_ctas / 2; p4 += 4) {
        float x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          x[u] = p4 + u < head_ctas / 2
                     ? __ldcg(&A.head_part[static_cast<long long>(cbase + 2 * (p4 + u) + rr) * kFpPartVals + k])
                     : 0.f;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (p4 + u < head_ctas / 2) v += x[u];
      }
      const long long o = i < kHeadNC * kHeadDH ? A.off_w1 + i
                          : i < kHeadNC * kHeadDH + kHeadNC ? A.off_b1 + (i - kHeadNC * kHeadDH)
                                                            : A.off_b0 + (i - kHeadNC * kHeadDH - kHeadNC);
      gs[o] = v;
    }
    if (dbg && threadIdx.x == 0) dbg[5] = globaltimer();
    interfere(G.intf, g, A.timing ? &A.timing[2 * g] : nullptr, t_cta0);
    if (A.timing && threadIdx.x == 0) atomicMax(&A.timing[2 * g + 1], static_cast<unsigned long long>(globaltimer()));
  }
  cluster_sync_all();  // the peer may still write into this CTA's smem until here
}

}  // namespace mlp
}  // namespace lbbsp
