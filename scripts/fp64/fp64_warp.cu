// Microbenchmark (GPU): fp64 dependent-chain latency vs active lanes per warp
// and warps per SM (clock64 per warp; every active lane runs its own chain).
// Build like fp64_lat.cu.
#include <cstdio>
#include "exactmath.cuh"
__global__ void chain(int lanes, int ops, double x0, long long* out, double* sink) {
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  if (lane >= lanes) return;
  double x = x0 + lane, y = 0.5;
  long long t0 = clock64();
  if (ops == 0)
    for (int i = 0; i < 256; ++i) x = lbbsp::dadd(x, y);
  else
    for (int i = 0; i < 16; ++i) x = lbbsp::glibc_tanh(x) + 0.5;
  long long t1 = clock64();
  if (lane == 0) out[warp] = t1 - t0;
  if (x == 12345.0) *sink = x;
}
int main() {
  long long* d; double* s; long long h[32];
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&s, 8);
  for (int ops = 0; ops < 2; ++ops)
    for (int warps : {1, 4, 8})
      for (int lanes : {1, 12, 16, 32}) {
        chain<<<1, 32 * warps>>>(lanes, ops, 1.0, d, s);
        chain<<<1, 32 * warps>>>(lanes, ops, 1.0, d, s);
        cudaMemcpy(h, d, sizeof(long long) * warps, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
        printf("%s warps %d lanes %2d: %.1f cycles per op\n", ops ? "tanh" : "dadd", warps, lanes,
               mx / (ops ? 16.0 : 256.0));
      }
  return 0;
}
