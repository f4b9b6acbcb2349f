// host.cuh -- host-side owner types shared by capi.cu and mlp.cu.
#pragma once
#include <vector>

#include "common.cuh"

// A bank of per-worker SpeedPredictors with device-resident histories.
struct lbbsp_predictor {
  lbbsp::PredDev dev{};
  std::vector<void*> allocs;
  ~lbbsp_predictor() {
    for (void* p : allocs) cudaFree(p);
  }
  template <typename T>
  cudaError_t alloc(T** p, size_t count) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1));
    if (e == cudaSuccess) {
      allocs.push_back(*p);
      cudaMemset(*p, 0, sizeof(T) * (count ? count : 1));
    }
    return e;
  }
};
