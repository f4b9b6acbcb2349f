// head_mma.cuh -- the small classifier head (256 -> 10, softmax-CE) of the
// MLP workload on warp-level tensor-core MMA (mma.sync m16n8k16, bf16 in,
// fp32 accumulate). One warp owns a 16-row tile at a time:
//
//   logits = H W^T + b          32 MMAs  (A = H via ldmatrix, B = W frags in smem)
//   dl     = (softmax - onehot) * row_scale        (on the accumulator fragments)
//   dW    += dl^T H             32 MMAs  (A = dl^T via ldmatrix.trans, B = H via .trans)
//   dH     = (dl W) * (H > 0)   32 MMAs  (A = dl straight from the logits fragments)
//   db    += column sums of dl and of dH (the previous layer's bias gradient)
//
// H tiles are staged with cp.async (double-buffered, XOR-swizzled 16-B chunks
// so every ldmatrix phase is bank-conflict free) and dH is written back through
// the same buffer with 16-B coalesced stores. Per-CTA partials are combined by
// the last CTA of each worker in CTA order (deterministic).
//
// Replaces the per-sample gradient of the reference's logistic regression
// (sgd.cpp:72-90) for the MLP's last layer; see mlp.cu for the round.
#pragma once
#include <cuda_bf16.h>

#include "mlp_kernels.cuh"
#include "tc_ptx.cuh"

namespace lbbsp {
namespace mlp {

using hbf16 = __nv_bfloat16;

constexpr int kHeadDH = 256;                  // hidden width
constexpr int kHeadNC = 10;                   // classes
constexpr int kHeadVals = kHeadNC * kHeadDH + kHeadNC + kHeadDH;  // dW | db | prev db
// dynamic shared memory layout (bytes)
constexpr int kHmWl = 0;                                // logits B frags [16 s][2 nt][32] uint2
constexpr int kHmWd = kHmWl + 16 * 2 * 32 * 8;         // dH B frags [32 nt][32] uint2
constexpr int kHmH = kHmWd + 32 * 32 * 8;              // H tiles [8 warps][2][16 rows][512 B]
constexpr int kHmDl = kHmH + 8 * 2 * 16 * 512;         // dl [8 warps][16][16] bf16
constexpr int kHmBp = kHmDl + 8 * 512;                 // prev-layer db [8 warps][256] f32
constexpr int kHmLoss = kHmBp + 8 * 256 * 4;           // [8] f64
constexpr int kHmWraw = kHmLoss + 8 * 8 + 64;          // W fp32 staging [10][256]
constexpr int kHeadMmaSmem = kHmWraw + kHeadNC * kHeadDH * 4;
constexpr int kHeadFrag = 32 * 4 * 32;                 // dW accumulator entries per warp
// CTA partials are kept in the warps' fragment order (coalesced writes):
// [kHeadFrag dW | 4x32 db | 8x32 prev db]; padded classes are carried and dropped
// when the worker's last CTA maps the sums to natural order
constexpr int kHeadPartVals = kHeadFrag + 4 * 32 + 8 * 32;

// fragment-order partial index -> natural index (dW [class][col] | db [class] |
// prev db [col]), -1 for the padded classes
__device__ __forceinline__ int head_frag_to_natural(int k) {
  if (k < kHeadFrag) {
    const int j = k >> 7, e = (k >> 5) & 3, l = k & 31;
    const int cls = (l >> 2) + (e >= 2 ? 8 : 0), col = 8 * j + 2 * (l & 3) + (e & 1);
    return cls < kHeadNC ? cls * kHeadDH + col : -1;
  }
  if (k < kHeadFrag + 128) {
    const int u = (k - kHeadFrag) >> 5, l = k & 31;
    const int cls = (u < 2 ? 2 * l + u : 8 + 2 * l + (u - 2));
    return ((l >> 2) == 0 && (u < 2 || l == 0)) ? kHeadNC * kHeadDH + cls : -1;
  }
  const int u = (k - kHeadFrag - 128) >> 5, l = k & 31;
  return kHeadNC * kHeadDH + kHeadNC + 8 * l + u;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
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
__device__ __forceinline__ void mma16816(float c[4], const uint32_t a[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}
// byte offset of (row, 16-B chunk) in a swizzled 16 x 512 B tile
__device__ __forceinline__ int hsw(int row, int chunk) { return row * 512 + ((chunk ^ (row & 7)) << 4); }

// stage rows [row0, row0+16) (clipped to row_end) of H into a tile buffer
__device__ __forceinline__ void stage_tile(uint32_t buf, const hbf16* H, int row0, int row_end,
                                           int lane) {
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int r = row0 + q;
    const bool ok = r < row_end;
    const hbf16* src = H + static_cast<long long>(ok ? r : row0) * kHeadDH + lane * 8;
    cp_async16(buf + hsw(q, lane), src, ok ? 16 : 0);
  }
  cp_async_commit();
}

template <bool TRAIN>
__global__ void __launch_bounds__(256, 1) head_mma_kernel(
    Groups G, int rows_total, const hbf16* __restrict__ H, const float* __restrict__ W,
    const float* __restrict__ bias, const int* __restrict__ y, const float* __restrict__ row_scale,
    hbf16* dH, float* slab, long long slab_stride, long long off_w, long long off_b,
    long long off_b_prev, double* loss_acc, float* cta_part, double* cta_loss, unsigned* counters,
    unsigned long long* timing, double* loss_rec, const long long* round_k, int max_rows) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ int last;
  int g, cta_in, cta_cnt;
  if (!my_group(G, &g, &cta_in, &cta_cnt)) return;
  const int r0 = G.n ? G.r0[g] : 0, r1 = G.n ? G.r1[g] : rows_total;
  const int n_tiles = (r1 - r0 + 15) / 16;
  // a worker uses at most one CTA per 8 tiles of its SM cap: the head is
  // latency-bound, and fewer CTA partials keep the final combine short
  cta_cnt = min(cta_cnt, max(1, (n_tiles + 7) / 8));
  if (cta_in >= cta_cnt) return;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int gq = lane >> 2, tq = lane & 3;
  const int wstride = cta_cnt * 8;
  int tile = cta_in * 8 + warp;
  const uint32_t hbuf0 = smem_addr(sm + kHmH + warp * 2 * 8192);

  // W (fp32 master): one cp.async round into smem, then bf16 B fragments
  // (zero for classes >= 10). W and the worker groups were final before the
  // previous kernel started, so this overlaps it (programmatic launch).
  const float* wraw = reinterpret_cast<const float*>(sm + kHmWraw);
  for (int i = threadIdx.x; i < kHeadNC * kHeadDH / 4; i += blockDim.x)
    cp_async16(smem_addr(sm + kHmWraw + 16 * i), W + 4 * i, 16);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  uint2* wl = reinterpret_cast<uint2*>(sm + kHmWl);
  uint2* wd = reinterpret_cast<uint2*>(sm + kHmWd);
  auto wv = [&](int c, int j) { return c < kHeadNC ? wraw[c * kHeadDH + j] : 0.f; };
  for (int i = threadIdx.x; i < 16 * 2 * 32; i += blockDim.x) {
    const int l = i & 31, nt = (i >> 5) & 1, s = i >> 6;
    const int c = 8 * nt + (l >> 2), k = 16 * s + 2 * (l & 3);
    wl[i] = make_uint2(pack_bf16(wv(c, k), wv(c, k + 1)), pack_bf16(wv(c, k + 8), wv(c, k + 9)));
  }
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
    const int l = i & 31, j = i >> 5;
    const int n = 8 * j + (l >> 2), c = 2 * (l & 3);
    wd[i] = make_uint2(pack_bf16(wv(c, n), wv(c + 1, n)), pack_bf16(wv(c + 8, n), wv(c + 9, n)));
  }
  __syncthreads();
  tc::pdl_wait();  // H, labels and row scales come from the kernels before
  tc::pdl_launch_dependents();
  const unsigned long long t_cta0 = gtimer();
  if (timing && threadIdx.x == 0) atomicMin(&timing[2 * g], t_cta0);
  if (tile < n_tiles) stage_tile(hbuf0, H, r0 + tile * 16, r1, lane);

  const float b_lo0 = bias[2 * tq], b_lo1 = bias[2 * tq + 1];
  const float b_hi0 = tq == 0 ? bias[8] : 0.f, b_hi1 = tq == 0 ? bias[9] : 0.f;
  // dW is column-sliced: warp w accumulates dW[:, 32w .. 32w+32) over every
  // tile of the CTA (A = dl^T of tile t, B = H of tile t), so no cross-warp
  // reduction of dW is needed; the tiles' dl and H are shared through smem
  float dw[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) dw[j][0] = dw[j][1] = dw[j][2] = dw[j][3] = 0.f;
  float dbh[4] = {0.f, 0.f, 0.f, 0.f};
  float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // prev db, cols 8*lane..+7
  double lsum = 0.0;
  uint8_t* dls = sm + kHmDl + warp * 512;
  int buf = 0;
  const int first_tile = cta_in * 8;
  const int n_iter = n_tiles > first_tile ? (n_tiles - first_tile + wstride - 1) / wstride : 0;
  for (int it = 0; it < n_iter; ++it, tile += wstride) {
    const bool have = tile < n_tiles;
    const int row0 = r0 + tile * 16;
    const uint32_t hb = hbuf0 + buf * 8192;
    uint8_t* hp = sm + kHmH + warp * 2 * 8192 + buf * 8192;
    const int next = tile + wstride;
    const int ra = row0 + gq, rb = row0 + gq + 8;
    const bool va = ra < r1, vb = rb < r1;
    const int ya = have && va ? y[ra] : -1, yb = have && vb ? y[rb] : -1;
    const float rsa = TRAIN && have && va ? row_scale[ra] : 0.f;
    const float rsb = TRAIN && have && vb ? row_scale[rb] : 0.f;
    if (next < n_tiles) {
      stage_tile(hbuf0 + (buf ^ 1) * 8192, H, r0 + next * 16, r1, lane);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    uint32_t ad[4] = {0u, 0u, 0u, 0u};  // dl as the m16k16 A operand of dH = dl W
    const int mi = lane >> 3, lr = (lane & 7) + (mi & 1) * 8;
    if (have) {
    // ---- logits: 16 k-steps x 2 class tiles, two independent chains each ----
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
    // ---- softmax-CE on the fragments: rows gq (c0,c1) and gq+8 (c2,c3) ----
    lo[0] += b_lo0; lo[1] += b_lo1; lo[2] += b_lo0; lo[3] += b_lo1;
    hi[0] += b_hi0; hi[1] += b_hi1; hi[2] += b_hi0; hi[3] += b_hi1;
    const bool hv = tq == 0;  // this lane's classes 8+2tq, 9+2tq exist
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
    float la = (c0 == ya ? lo[0] : 0.f) + (c1 == ya ? lo[1] : 0.f) + (hv && c2 == ya ? hi[0] : 0.f) +
               (hv && c3 == ya ? hi[1] : 0.f);
    float lb = (c0 == yb ? lo[2] : 0.f) + (c1 == yb ? lo[3] : 0.f) + (hv && c2 == yb ? hi[2] : 0.f) +
               (hv && c3 == yb ? hi[3] : 0.f);
    la += __shfl_xor_sync(0xffffffffu, la, 1);
    la += __shfl_xor_sync(0xffffffffu, la, 2);
    lb += __shfl_xor_sync(0xffffffffu, lb, 1);
    lb += __shfl_xor_sync(0xffffffffu, lb, 2);
    if (tq == 0) {
      if (va) lsum += static_cast<double>(logf(sa) + ma - la);
      if (vb) lsum += static_cast<double>(logf(sb) + mb - lb);
    }
    if (TRAIN) {
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
      // dl as the A operand of dH = dl W (the m16n8 accumulator layout is the
      // m16k16 A layout), and as [row][class] bf16 for dl^T via ldmatrix.trans
      ad[0] = pack_bf16(dlo[0], dlo[1]);
      ad[1] = pack_bf16(dlo[2], dlo[3]);
      ad[2] = pack_bf16(dhi[0], dhi[1]);
      ad[3] = pack_bf16(dhi[2], dhi[3]);
      *reinterpret_cast<uint32_t*>(dls + gq * 32 + 4 * tq) = ad[0];
      *reinterpret_cast<uint32_t*>(dls + (gq + 8) * 32 + 4 * tq) = ad[1];
      *reinterpret_cast<uint32_t*>(dls + gq * 32 + 16 + 4 * tq) = ad[2];
      *reinterpret_cast<uint32_t*>(dls + (gq + 8) * 32 + 16 + 4 * tq) = ad[3];
    }
    }  // have
    if (TRAIN) {
      __syncthreads();  // every tile's dl and H of this iteration are in smem
      // ---- dW[:, 32 warp .. +32) += dl_t^T H_t over the CTA's tiles t ----
#pragma unroll 1
      for (int t = 0; t < 8; ++t) {
        if (first_tile + t + it * wstride >= n_tiles) break;
        uint32_t at[4];
        ldsm_x4_t(smem_addr(sm + kHmDl + t * 512) + ((lane & 7) + (mi >> 1) * 8) * 32 + (mi & 1) * 16,
                  at);
        const uint32_t ht = smem_addr(sm + kHmH + t * 2 * 8192) + buf * 8192;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          uint32_t b[4];
          ldsm_x4_t(ht + hsw(lr, 2 * (2 * warp + p) + (mi >> 1)), b);
          mma16816(dw[2 * p], at, b[0], b[1]);
          mma16816(dw[2 * p + 1], at, b[2], b[3]);
        }
      }
      __syncthreads();  // H tiles may now be overwritten by dH
    }
    if (TRAIN && have) {
      // ---- dH = (dl W) * (H > 0), written in place over the H tile ----
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
      // ---- coalesced dH rows + the previous layer's bias (column sums) ----
#pragma unroll 4
      for (int q = 0; q < 16; ++q) {
        const int r = row0 + q;
        if (r >= r1) break;
        const uint4 v = *reinterpret_cast<const uint4*>(hp + hsw(q, lane));
        *reinterpret_cast<uint4*>(dH + static_cast<long long>(r) * kHeadDH + lane * 8) = v;
        const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          cs[2 * u] += __low2float(e[u]);
          cs[2 * u + 1] += __high2float(e[u]);
        }
      }
    }
    __syncwarp();
    buf ^= 1;
  }
  // ---- CTA partials: warps -> smem (over the H tiles) -> summed in warp order ----
  double* wl_loss = reinterpret_cast<double*>(sm + kHmLoss);
  lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
  lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
  lsum += __shfl_xor_sync(0xffffffffu, lsum, 4);
  lsum += __shfl_xor_sync(0xffffffffu, lsum, 8);
  lsum += __shfl_xor_sync(0xffffffffu, lsum, 16);
  if (lane == 0) wl_loss[warp] = lsum;
  // per-warp partials in fragment order (lane-contiguous, conflict-free):
  // [kHeadFrag dW | 4x32 db | 8x32 prev db]
  // dW: each warp's column slice goes straight to the CTA partial, in the
  // fragment order of head_frag_to_natural (n-tile j = 4 warp + p);
  // db / prev db: per-warp values summed over the 8 warps in warp order
  constexpr int kSmallVals = kHeadPartVals - kHeadFrag;  // 4x32 db | 8x32 prev db
  float* red = reinterpret_cast<float*>(sm + kHmH);     // [8][kSmallVals] over the H tiles
  float* part = cta_part + static_cast<long long>(blockIdx.x) * kHeadPartVals;
  if (TRAIN) {
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
  }
  __syncthreads();  // every warp is done with its H tiles
  if (TRAIN) {
    float* mine = red + warp * kSmallVals;
#pragma unroll
    for (int u = 0; u < 4; ++u) mine[u * 32 + lane] = dbh[u];
#pragma unroll
    for (int u = 0; u < 8; ++u) mine[128 + u * 32 + lane] = cs[u];
  }
  __syncthreads();
  if (TRAIN)
    for (int k = threadIdx.x; k < kSmallVals; k += blockDim.x) {
      float v = red[k];
#pragma unroll
      for (int w = 1; w < 8; ++w) v += red[w * kSmallVals + k];
      part[kHeadFrag + k] = v;
    }
  if (threadIdx.x == 0) {
    double l = 0.0;
    for (int w = 0; w < 8; ++w) l += wl_loss[w];
    cta_loss[blockIdx.x] = l;
  }
  // Training: the CTA partials are combined by head_combine_kernel, launched
  // beside the next backward GEMM (off the worker-phase chain). Dataset loss:
  // the last CTA sums the CTA losses in CTA order.
  if (!TRAIN) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&counters[g], 1u) == static_cast<unsigned>(cta_cnt - 1);
    __syncthreads();
    if (last && threadIdx.x == 0) {
      __threadfence();
      const int c0 = blockIdx.x - cta_in;
      if (loss_acc) {
        double l = 0.0;
        for (int c = 0; c < cta_cnt; ++c) l += __ldcg(&cta_loss[c0 + c]);
        *loss_acc = l;
        // the round's record too (the same value the next plan writes), so a
        // host read of this round's result need not wait for that plan
        if (loss_rec) {
          const long long r = *round_k;
          if (r >= 0 && r < max_rows) loss_rec[r] = l / static_cast<double>(rows_total);
        }
      }
      counters[g] = 0u;
    }
  }
  if (TRAIN && G.n > 0) interfere(G.intf, g, timing ? &timing[2 * g] : nullptr, t_cta0);
  if (timing && threadIdx.x == 0) atomicMax(&timing[2 * g + 1], static_cast<unsigned long long>(gtimer()));
}

// Sums each worker's head CTA partials in CTA order (the same CTAs and order
// head_mma_kernel<true> used) and writes dW | db | prev db into the worker's
// gradient slab. Grid: n_local x kCombineSlices CTAs of 256 threads.
constexpr int kCombineSlices = 6;
__global__ void __launch_bounds__(256) head_combine_kernel(Groups G, const float* __restrict__ cta_part,
                                                           float* slab, long long slab_stride,
                                                           long long off_w, long long off_b,
                                                           long long off_b_prev) {
  const int g = blockIdx.x / kCombineSlices, slice = blockIdx.x % kCombineSlices;
  if (g >= G.n) return;
  const int n_tiles = (G.r1[g] - G.r0[g] + 15) / 16;
  const int c0 = G.cta0[g];
  const int cnt = min(G.ctan[g], max(1, (n_tiles + 7) / 8));
  const int k = slice * 256 * 3 + threadIdx.x;  // 3 values per thread, 6 x 768 >= kHeadPartVals
  float v[3] = {0.f, 0.f, 0.f};
  for (int c4 = 0; c4 < cnt; c4 += 4) {  // 4 CTAs' loads in flight per round trip
    float x[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int i = k + 256 * u;
        x[q][u] = c4 + q < cnt && i < kHeadPartVals
                      ? __ldcg(&cta_part[static_cast<long long>(c0 + c4 + q) * kHeadPartVals + i])
                      : 0.f;
      }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int u = 0; u < 3; ++u)
        if (c4 + q < cnt) v[u] += x[q][u];
  }
  float* gs = slab + static_cast<long long>(g) * slab_stride;
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int kk = k + 256 * u;
    const int i = kk < kHeadPartVals ? head_frag_to_natural(kk) : -1;
    if (i < 0) continue;
    const long long o = i < kHeadNC * kHeadDH ? off_w + i
                        : i < kHeadNC * kHeadDH + kHeadNC ? off_b + (i - kHeadNC * kHeadDH)
                                                          : off_b_prev + (i - kHeadNC * kHeadDH - kHeadNC);
    gs[o] = v[u];
  }
}
static_assert(kCombineSlices * 768 >= kHeadPartVals, "combine slices do not cover the partials");

}  // namespace mlp
}  // namespace lbbsp
