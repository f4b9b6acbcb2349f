// mlp_kernels.cuh -- the non-GEMM kernels of the MLP gradient engine
// (north_star (1)/(2)): row gather with the Eq.-6/7 row scale, warp-shuffle
// softmax-CE heads, per-worker bias-gradient column sums, and the HBM-bound
// segmented reduction + SGD apply.
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

#include "interfere.cuh"

namespace lbbsp {
namespace mlp {

// Per-worker CTA partition + batch rows for one iteration, device-resident.
struct Groups {
  int n;            // local workers
  const int* r0;    // [n] first local batch row
  const int* r1;    // [n] one past last
  const int* cta0;  // [n]
  const int* ctan;  // [n]
  Interference intf;  // straggler injection after each worker phase (interfere.cuh)
};

__device__ __forceinline__ bool my_group(const Groups& G, int* g, int* cta_in, int* cta_cnt) {
  if (G.n == 0) {
    *g = 0;
    *cta_in = blockIdx.x;
    *cta_cnt = gridDim.x;
    return true;
  }
  for (int i = 0; i < G.n; ++i) {
    const int c0 = G.cta0[i], cn = G.ctan[i];
    if (static_cast<int>(blockIdx.x) >= c0 && static_cast<int>(blockIdx.x) < c0 + cn) {
      *g = i;
      *cta_in = blockIdx.x - c0;
      *cta_cnt = cn;
      return true;
    }
  }
  return false;
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// splitmix64-based counter hash -> uniform [lo, hi) (setup-time data / init)
__host__ __device__ __forceinline__ uint64_t hash64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ float hash_uniform(uint64_t seed, uint64_t i, float lo, float hi) {
  const uint64_t h = hash64(seed * 0x100000001b3ull ^ hash64(i));
  return lo + (hi - lo) * static_cast<float>((h >> 40) * 0x1.0p-24);
}

}  // namespace mlp
}  // namespace lbbsp
