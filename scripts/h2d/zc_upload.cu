// Probe (GPU): the C2 e2e upload (1.57 MB) by the copy engine (cudaMemcpyAsync
// from page-locked memory) vs by SMs reading the mapped page-locked buffer
// directly (zero-copy over PCIe, 16-B loads, CTAs x threads in flight).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/h2d/zc_upload.cu -o scripts/h2d/zc_upload
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <sys/mman.h>
#include <cstring>
#include <algorithm>
#include <vector>
__global__ void zc_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  constexpr int kU = 4;
  size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + (kU - 1) * stride < n16; i += kU * stride) {
    uint4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < kU; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}
int main() {
  const size_t nbytes = 1000 * 784 * 2 + 1000 * 4, n16 = (nbytes + 15) / 16;
  const size_t size = 2 << 20;
  void* raw = mmap(nullptr, size * 2, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  char* h = (char*)(((uintptr_t)raw + size - 1) & ~(uintptr_t)(size - 1));
  madvise(h, size, MADV_HUGEPAGE);
  memset(h, 1, size);
  cudaHostRegister(h, size, cudaHostRegisterMapped);
  void* hd = nullptr;
  cudaHostGetDevicePointer(&hd, h, 0);
  void* d = nullptr;
  cudaMalloc(&d, size);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto bench = [&](const char* name, auto fn) {
    std::vector<float> t;
    for (int r = 0; r < 1500; ++r) {
      cudaEventRecord(e0, s); fn(); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 500) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    printf("%-28s median %6.1f us (%5.1f GB/s) p10 %6.1f p90 %6.1f\n", name, t[t.size() / 2],
           nbytes / t[t.size() / 2] / 1e3, t[t.size() / 10], t[9 * t.size() / 10]);
  };
  for (int pass = 0; pass < 2; ++pass) {
    bench("copy engine", [&] { cudaMemcpyAsync(d, h, nbytes, cudaMemcpyHostToDevice, s); });
    for (int ctas : {16, 32, 64, 148})
      for (int thr : {256, 512}) {
        char name[64];
        snprintf(name, sizeof name, "zero-copy %3d x %3d", ctas, thr);
        bench(name, [&] { zc_copy<<<ctas, thr, 0, s>>>((const uint4*)hd, (uint4*)d, n16); });
      }
  }
  return 0;
}
