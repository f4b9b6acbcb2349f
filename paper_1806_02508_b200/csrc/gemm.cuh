// gemm.cuh -- host-side plan for the tcgen05 GEMM (gemm_tc.cuh).
#pragma once
#include <utility>
#include <cuda.h>

#include "gemm_tc.cuh"
#include "gemm_tc2.cuh"

namespace lbbsp {

struct GemmPlan {
  CUtensorMap ta, tb;
  tc::GemmArgs args;
  bool a_mn = false, b_mn = false;
  int bn = 256;
  int args_epi = 0;
  int ctas = 148;
  bool pair = false;  // CTA-pair (cta_group::2) kernel: 256 x bn tiles, ungrouped only
  bool pdl = false;   // programmatic dependent launch (prologue overlaps the previous kernel)
};

// Launches `kern` with the programmatic-stream-serialization attribute when
// pdl is set (the kernel must call pdl_wait() before reading its inputs).
template <typename... KArgs, typename... Args>
cudaError_t launch_maybe_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem,
                             cudaStream_t s, bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

int make_tmap_bf16(CUtensorMap* tm, const void* ptr, long long inner, long long outer, long long ld,
                   int box_outer);
int make_tmap_f32_3d(CUtensorMap* tm, const void* ptr, long long d0, long long d1, long long d2, long long ld1,
                     long long ld2, int box1);
int gemm_plan(GemmPlan* p, const void* A, const void* B, int M, int N, int K, bool a_mn, bool b_mn,
              int bn, int epi, bool pair = false);
int gemm_launch(const GemmPlan& p, cudaStream_t s);
int num_sms();

}  // namespace lbbsp
