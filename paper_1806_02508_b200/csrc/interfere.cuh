// interfere.cuh -- straggler injection on real hardware (north_star: "capping
// per-worker SM counts and co-scheduled interference kernels driven from a
// recorded trace", the Dynamics/effective_speed row).
//
// The reference's straggler model scales a worker's speed by its availability
//   a = c * MemPenalty(m) * speed_mult          (cluster_sim.cpp:22-29, 77-118)
// where c is the CPU share a co-located job leaves it and m the memory share.
// On the B200 each emulated worker owns a fixed CTA partition of the GPU (its
// SM cap, sized by its nominal share). Its availability is realised by an
// interference job co-scheduled on that partition: once a CTA of worker g has
// finished the phase's real work, the same SMs run interference until the
// phase has lasted (phase work time) / a. The injected time is split the way
// the model splits the slowdown:
//   * memory-pressure part (1/a - 1/a_sm of the work time, a_sm = min(1, c*mult)):
//     HBM-bound -- the CTA streams a buffer larger than L2 (real DRAM traffic
//     that co-resident workers also feel, as a memory-hungry neighbour would);
//   * the rest: SM-bound -- dependent FMA chains on every warp of the CTA.
// A worker at availability a therefore runs 1/a slower than at a = 1 by
// construction, whatever the phase's latency structure (an SM-count cap alone
// is not proportional: a latency-bound phase barely slows when it loses SMs).
//
// Why inside the worker's kernels and not a separate launch: CUDA has no SM
// affinity for a kernel, so a separate interference kernel cannot be placed on
// worker g's SMs; green contexts (cuDevSmResourceSplitByCount) partition in
// static groups of 8 SMs on sm_90+, too coarse for 8 workers on 148 SMs and
// fixed for the context's lifetime, while the trace changes a every round.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace lbbsp {

// Per-round straggler state of this rank's workers, written by the plan.
struct Interference {
  const float2* w;   // [n_local] {availability a in (0, 1], HBM share of the injected time}
  const uint4* buf;  // HBM-bound interference source (> L2)
  long long nvec;    // uint4 elements in buf
};

__device__ __forceinline__ unsigned long long intf_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Every thread of a CTA of worker g calls this once its share of the phase's
// real work is done. phase_t0 = the worker's phase start (the min CTA start,
// globaltimer ns; null: this CTA's own start t_cta0). Stretches the phase so
// it ends at t0 + (now - t0) / a.
static __device__ __noinline__ void interfere(const Interference I, int g, const unsigned long long* phase_t0,
                                       unsigned long long t_cta0) {
  if (!I.w || g < 0) return;
  const float2 p = I.w[g];
  if (!(p.x < 1.f) || !(p.x > 0.f)) return;
  __shared__ unsigned long long t_hbm, t_end;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t0 = t_cta0;
    if (phase_t0) {
      const unsigned long long s = *reinterpret_cast<const volatile unsigned long long*>(phase_t0);
      if (s < t0) t0 = s;
    }
    const unsigned long long now = intf_gtimer();
    const double work = static_cast<double>(now > t0 ? now - t0 : 0ull);
    const double extra = work * (1.0 / static_cast<double>(p.x) - 1.0);
    t_hbm = now + static_cast<unsigned long long>(extra * static_cast<double>(p.y));
    t_end = now + static_cast<unsigned long long>(extra);
  }
  __syncthreads();
  const unsigned long long th = t_hbm, te = t_end;
  // HBM-bound part: 4 independent 16-B streaming loads in flight per thread
  unsigned acc = 0u;
  if (I.buf && I.nvec > 0) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x +
                   static_cast<long long>(intf_gtimer() & 0xfffff) * 4096) % I.nvec;
    while (intf_gtimer() < th) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        q[u] = __ldcs(I.buf + i);
        i += stride;
        if (i >= I.nvec) i -= I.nvec;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc ^= q[u].x ^ q[u].w;
    }
  }
  // SM-bound part: four dependent FMA chains per thread
  float x0 = __uint_as_float(0x3f800000u | (acc & 0xffu)), x1 = x0 + 1.f, x2 = x0 + 2.f, x3 = x0 + 3.f;
  while (intf_gtimer() < te) {
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      x0 = fmaf(x0, 0.999f, 0.001f);
      x1 = fmaf(x1, 0.999f, 0.001f);
      x2 = fmaf(x2, 0.999f, 0.001f);
      x3 = fmaf(x3, 0.999f, 0.001f);
    }
  }
  asm volatile("" ::"f"(x0), "f"(x1), "f"(x2), "f"(x3), "r"(acc));
}

}  // namespace lbbsp
