// NVLink P2P probe (one process, two GPUs): the access patterns of the
// engine's peer exchange (csrc/mlp.cu peer_grad_push_kernel: uint4 stores of
// this rank's gradient slab into every peer's slot; peer_grad_apply: local
// reads) -- here GPU 0 pushes n bytes into GPU 1's buffer with the same
// grid-stride uint4 stores, then pulls them back with uint4 loads, and a
// cudaMemcpyPeerAsync (copy engine) moves the same bytes. Run under ncu with
// nvltx__bytes.sum / nvlrx__bytes.sum for the bus counters; without ncu it
// prints the event-timed GB/s.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__global__ void push_kernel(const uint4* __restrict__ src, uint4* dst, long long n) {
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) dst[i] = src[i];
}
__global__ void pull_kernel(const uint4* src, uint4* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) dst[i] = src[i];
}

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                   \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

int main(int argc, char** argv) {
  const long long bytes = argc > 1 ? atoll(argv[1]) : (64ll << 20);
  const long long n = bytes / 16;
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  if (!can) {
    printf("{\"error\": \"no peer access 0->1\"}\n");
    return 0;
  }
  uint4 *a0, *b0, *b1;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 1, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float t_push = 1e30f, t_pull = 1e30f, t_ce = 1e30f, ms;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(e0));
    push_kernel<<<sms * 4, 256>>>(a0, b1, n);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    t_push = ms < t_push ? ms : t_push;
    CK(cudaEventRecord(e0));
    pull_kernel<<<sms * 4, 256>>>(b1, b0, n);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    t_pull = ms < t_pull ? ms : t_pull;
    CK(cudaEventRecord(e0));
    CK(cudaMemcpyPeerAsync(b1, 1, a0, 0, bytes));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    t_ce = ms < t_ce ? ms : t_ce;
  }
  printf("{\"bytes\": %lld, \"push_stores_GBps\": %.1f, \"pull_loads_GBps\": %.1f, \"copy_engine_GBps\": %.1f}\n",
         bytes, bytes / (t_push * 1e-3) / 1e9, bytes / (t_pull * 1e-3) / 1e9, bytes / (t_ce * 1e-3) / 1e9);
  return 0;
}
