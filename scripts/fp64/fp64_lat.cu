// Microbenchmark (GPU): dependent-chain latency of the fp64 operations the
// bit-exact NARX trainer is built from (clock64 around 512-long chains, one
// thread), plus one glibc_tanh and the smem left fold of 112 terms as
// block_eval runs it. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   -I paper_1806_02508_b200/csrc -I include scripts/fp64/fp64_lat.cu -o scripts/fp64/fp64_lat
#include <cstdio>
#include "exactmath.cuh"

__global__ void lat(double x0, long long* out, double* sink) {
  __shared__ double src[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) src[i] = 1e-3 * i;
  __syncthreads();
  if (threadIdx.x) return;
  double x = x0, y = x0 * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < 512; ++i) x = lbbsp::dadd(x, y);
  long long t1 = clock64();
  for (int i = 0; i < 512; ++i) x = lbbsp::dmul(x, 0.999999);
  long long t2 = clock64();
  for (int i = 0; i < 64; ++i) x = lbbsp::ddiv(x, 1.0000001);
  long long t3 = clock64();
  for (int i = 0; i < 64; ++i) x = lbbsp::glibc_tanh(x) + 0.5;
  long long t4 = clock64();
  double acc = 0.0, a[8], b[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = src[q];
  for (int i = 0; i < 112; i += 16) {
#pragma unroll
    for (int q = 0; q < 8; ++q) b[q] = src[i + 8 + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = lbbsp::dadd(acc, a[q]);
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = src[i + 16 + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = lbbsp::dadd(acc, b[q]);
  }
  long long t5 = clock64();
  __syncthreads();
  long long t6 = clock64();
  out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4;
  *sink = x + acc;
}
__global__ void bar_lat(long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < 64; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[5] = t1 - t0;
}
int main() {
  long long* d; double* s;
  cudaMalloc(&d, 8 * sizeof(long long)); cudaMalloc(&s, 8);
  for (int rep = 0; rep < 3; ++rep) {
    lat<<<1, 32>>>(1.0, d, s);
    bar_lat<<<1, 544>>>(d);
    long long h[8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("cycles: dadd %.1f  dmul %.1f  ddiv %.1f  tanh+add %.1f  fold112 %lld (%.1f per term)  syncthreads(544) %.1f\n",
           h[0] / 512.0, h[1] / 512.0, h[2] / 64.0, h[3] / 64.0, h[4], h[4] / 112.0, h[5] / 64.0);
  }
  return 0;
}
