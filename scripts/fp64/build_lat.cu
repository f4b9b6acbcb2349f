// Microbenchmark (GPU): the NARX training-set build loop in isolation (256
// threads, 9 x 118 standardised elements, one __ddiv_rn each, shared memory),
// cycles per CTA; with and without zero numerators (constant series).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1806_02508_b200/csrc -I include
//   scripts/fp64/build_lat.cu -o scripts/fp64/build_lat
#include <cstdio>
#include "exactmath.cuh"
__global__ void build(int L, int zero_m, long long* out, double* sink) {
  __shared__ double h[3 * 256];
  __shared__ double Z[9 * 256];
  const int tid = threadIdx.x;
  for (int i = tid; i < L; i += blockDim.x) {
    h[i] = 1000.0 + 37.0 * (i % 7);
    h[L + i] = 0.5 + 0.01 * (i % 5);
    h[2 * L + i] = zero_m ? 1.0 : 0.9 + 0.001 * i;
  }
  __syncthreads();
  const double* v = h; const double* c = h + L; const double* m = h + 2 * L;
  const double mv = 1100.0, sv = 70.0, mc = 0.52, scd = 0.014, mm = zero_m ? 1.0 : 0.95, sm = zero_m ? 1.0 : 0.05;
  const int cnt = L - 2, S = 256;
  long long t0 = clock64();
  for (int e = tid; e < 9 * cnt; e += blockDim.x) {
    const int f = e / cnt, i = e - f * cnt, t = i + 2;
    const int ser = f < 2 ? 0 : (f < 5 ? 1 : (f < 8 ? 2 : 0));
    const int lag = f == 8 ? 0 : (f < 2 ? f + 1 : (f - (f < 5 ? 2 : 5)));
    const double* xs = ser == 0 ? v : (ser == 1 ? c : m);
    const double mu = ser == 0 ? mv : (ser == 1 ? mc : mm);
    const double sd = ser == 0 ? sv : (ser == 1 ? scd : sm);
    Z[f * S + i] = lbbsp::ddiv(lbbsp::dsub(xs[t - lag], mu), sd);
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) { out[0] = t1 - t0; *sink = Z[5]; }
}
int main() {
  long long* d; double* s; long long h;
  cudaMalloc(&d, 64); cudaMalloc(&s, 8);
  for (int zero_m = 0; zero_m < 2; ++zero_m)
    for (int rep = 0; rep < 3; ++rep) {
      build<<<1, 256>>>(120, zero_m, d, s);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("build loop L=120 %s: %lld cycles (%.2f us at 1.9 GHz)\n", zero_m ? "constant m series" : "varying series", h, h / 1900.0);
    }
  return 0;
}
