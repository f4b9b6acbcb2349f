// gemm.cuh -- host-side plan for the tcgen05 GEMM (gemm_tc.cuh).
#pragma once
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
};

int make_tmap_bf16(CUtensorMap* tm, const void* ptr, long long inner, long long outer, long long ld,
                   int box_outer);
int gemm_plan(GemmPlan* p, const void* A, const void* B, int M, int N, int K, bool a_mn, bool b_mn,
              int bn, int epi, bool pair = false);
int gemm_launch(const GemmPlan& p, cudaStream_t s);
int num_sms();

}  // namespace lbbsp
