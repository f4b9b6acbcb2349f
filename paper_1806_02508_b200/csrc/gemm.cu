// gemm.cu -- host side of the tcgen05 GEMM: TMA tensor maps (driver entry
// point resolved at run time, no -lcuda), template dispatch, C-ABI entry.
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "gemm.cuh"
#include "gemm_tc.cuh"

namespace lbbsp {

using tc::GemmArgs;

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

// bf16 matrix [outer][inner] (inner contiguous, row pitch ld elements),
// 128B swizzle, box {64, box_outer}, OOB -> zero fill.
int make_tmap_bf16(CUtensorMap* tm, const void* ptr, long long inner, long long outer, long long ld,
                   int box_outer) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return set_error(LBBSP_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((ld * 2) % 16 != 0 || (reinterpret_cast<uintptr_t>(ptr) % 16) != 0)
    return set_error(LBBSP_INVALID_ARGUMENT, "tma: rows must be 16-byte aligned (ld=%lld)", ld);
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(LBBSP_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return LBBSP_OK;
}

// fp32 [d2][d1][d0] slabs (d0 contiguous, d1 stride ld1 elements, d2 stride
// ld2 elements), 128B swizzle, box {32, box1, 1}: the TMA-store epilogue of
// the fused worker kernel (per-worker dW0 partials).
int make_tmap_f32_3d(CUtensorMap* tm, const void* ptr, long long d0, long long d1, long long d2, long long ld1,
                     long long ld2, int box1) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return set_error(LBBSP_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((ld1 * 4) % 16 != 0 || (ld2 * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(ptr) % 16) != 0)
    return set_error(LBBSP_INVALID_ARGUMENT, "tma: fp32 slab rows must be 16-byte aligned");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(d0), static_cast<cuuint64_t>(d1), static_cast<cuuint64_t>(d2)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld1 * 4), static_cast<cuuint64_t>(ld2 * 4)};
  cuuint32_t box[3] = {32u, static_cast<cuuint32_t>(box1), 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(LBBSP_CUDA, "cuTensorMapEncodeTiled (f32 3d) failed (%d)", (int)r);
  return LBBSP_OK;
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
static int launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a, int ctas,
                    cudaStream_t s, bool pdl) {
  constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  constexpr size_t smem = tc::gemm_smem_bytes<BN, STAGES>();
  auto kern = tc::gemm_bf16_tc_kernel<BN, A_MN, B_MN, EPI, STAGES>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  LBBSP_CUDA_CHECK(launch_maybe_pdl(kern, ctas, tc::kGemmThreads, smem, s, pdl, ta, tb, a));
  return LBBSP_OK;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
static int launch_t2(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a, int ctas,
                     cudaStream_t s, bool pdl) {
  constexpr int STAGES = BN == 256 ? 7 : 8;
  constexpr size_t smem = tc::gemm2_smem_bytes<BN, STAGES>();
  auto kern = tc::gemm_bf16_tc2_kernel<BN, A_MN, B_MN, EPI, STAGES>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  LBBSP_CUDA_CHECK(launch_maybe_pdl(kern, ctas, tc::kGemmThreads, smem, s, pdl, ta, tb, a));
  return LBBSP_OK;
}

#define LBBSP_GEMM2_CASE(BN_, AMN, BMN, EPI_)                                          \
  if (bn == BN_ && a_mn == AMN && b_mn == BMN && epi == EPI_)                          \
    return launch_t2<BN_, AMN, BMN, EPI_>(p.ta, p.tb, p.args, ctas, s, p.pdl);

#define LBBSP_GEMM_CASE(BN_, AMN, BMN, EPI_)                                           \
  if (bn == BN_ && a_mn == AMN && b_mn == BMN && epi == EPI_)                          \
    return launch_t<BN_, AMN, BMN, EPI_>(p.ta, p.tb, p.args, ctas, s, p.pdl);

int gemm_launch(const GemmPlan& p, cudaStream_t s) {
  const int bn = p.bn, epi = p.args_epi;
  const bool a_mn = p.a_mn, b_mn = p.b_mn;
  int ctas = p.ctas;
  if (p.pair) {
    ctas &= ~1;
    if (ctas < 2) ctas = 2;
    LBBSP_GEMM2_CASE(256, false, false, tc::kEpiBiasReluBf16)
    LBBSP_GEMM2_CASE(256, false, false, tc::kEpiBiasBf16)
    LBBSP_GEMM2_CASE(256, false, false, tc::kEpiF32)
    LBBSP_GEMM2_CASE(256, false, true, tc::kEpiDReluBf16)
    LBBSP_GEMM2_CASE(256, false, true, tc::kEpiF32)
    LBBSP_GEMM2_CASE(256, true, true, tc::kEpiF32)
    LBBSP_GEMM2_CASE(256, true, true, tc::kEpiBf16)
    return set_error(LBBSP_INVALID_ARGUMENT, "gemm: unsupported pair variant bn=%d a_mn=%d b_mn=%d epi=%d",
                     bn, (int)a_mn, (int)b_mn, epi);
  }
  // forward / hidden layers
  LBBSP_GEMM_CASE(256, false, false, tc::kEpiBiasReluBf16)
  LBBSP_GEMM_CASE(128, false, false, tc::kEpiBiasReluBf16)
  LBBSP_GEMM_CASE(64, false, false, tc::kEpiBiasReluBf16)
  LBBSP_GEMM_CASE(256, false, false, tc::kEpiBiasBf16)
  LBBSP_GEMM_CASE(128, false, false, tc::kEpiBiasBf16)
  LBBSP_GEMM_CASE(64, false, false, tc::kEpiBiasBf16)
  LBBSP_GEMM_CASE(256, false, false, tc::kEpiF32)
  LBBSP_GEMM_CASE(128, false, false, tc::kEpiF32)
  LBBSP_GEMM_CASE(64, false, false, tc::kEpiF32)
  // dX through ReLU
  LBBSP_GEMM_CASE(256, false, true, tc::kEpiDReluBf16)
  LBBSP_GEMM_CASE(128, false, true, tc::kEpiDReluBf16)
  LBBSP_GEMM_CASE(64, false, true, tc::kEpiDReluBf16)
  LBBSP_GEMM_CASE(256, false, true, tc::kEpiF32)
  LBBSP_GEMM_CASE(128, false, true, tc::kEpiF32)
  LBBSP_GEMM_CASE(64, false, true, tc::kEpiF32)
  // dW = dY^T X (per-worker K split)
  LBBSP_GEMM_CASE(256, true, true, tc::kEpiF32)
  LBBSP_GEMM_CASE(256, true, true, tc::kEpiBf16)
  LBBSP_GEMM_CASE(128, true, true, tc::kEpiBf16)
  LBBSP_GEMM_CASE(128, true, true, tc::kEpiF32)
  LBBSP_GEMM_CASE(64, true, true, tc::kEpiF32)
  LBBSP_GEMM_CASE(256, true, false, tc::kEpiF32)
  LBBSP_GEMM_CASE(128, true, false, tc::kEpiF32)
  LBBSP_GEMM_CASE(64, true, false, tc::kEpiF32)
  return set_error(LBBSP_INVALID_ARGUMENT, "gemm: unsupported variant bn=%d a_mn=%d b_mn=%d epi=%d",
                   bn, (int)a_mn, (int)b_mn, epi);
}

// A: a_mn ? [K][M] : [M][K];  B: b_mn ? [K][N] : [N][K]  (bf16, dense rows)
int gemm_plan(GemmPlan* p, const void* A, const void* B, int M, int N, int K, bool a_mn, bool b_mn,
              int bn, int epi, bool pair) {
  p->a_mn = a_mn;
  p->b_mn = b_mn;
  p->bn = bn;
  p->args_epi = epi;
  p->pair = pair;
  int rc = a_mn ? make_tmap_bf16(&p->ta, A, M, K, M, 64) : make_tmap_bf16(&p->ta, A, K, M, K, 128);
  if (rc) return rc;
  // a CTA pair stages bn/2 rows of B per CTA
  rc = b_mn ? make_tmap_bf16(&p->tb, B, N, K, N, 64)
            : make_tmap_bf16(&p->tb, B, K, N, K, pair ? bn / 2 : bn);
  if (rc) return rc;
  GemmArgs& a = p->args;
  a = GemmArgs{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.mode = tc::kRows;
  a.ldc = N;
  const int tiles = ((M + tc::kBM - 1) / tc::kBM) * ((N + bn - 1) / bn);
  p->ctas = tiles < num_sms() ? tiles : num_sms();
  if (pair) {  // one 256-row tile per CTA pair
    const int tiles2 = ((M + 2 * tc::kBM - 1) / (2 * tc::kBM)) * ((N + bn - 1) / bn);
    p->ctas = 2 * (tiles2 < num_sms() / 2 ? tiles2 : num_sms() / 2);
  }
  return LBBSP_OK;
}

}  // namespace lbbsp

using namespace lbbsp;

extern "C" int lbbsp_gemm_bf16(const void* d_a, const void* d_b, void* d_c, int M, int N, int K,
                               int a_mn, int b_mn, int epilogue, const float* d_bias,
                               const void* d_aux, int mode, int n_groups, const int* d_group_r0,
                               const int* d_group_r1, const int* d_group_cta0,
                               const int* d_group_ctan, int ctas, unsigned long long* d_timing,
                               int bn, void* stream) {
  GemmPlan p;
  // bn < 0 selects the CTA-pair kernel (256 x |bn| tiles, ungrouped problems)
  const bool pair = bn < 0 && n_groups == 0;
  if (bn < 0) bn = -bn;
  if (bn != 64 && bn != 128 && bn != 256) bn = N > 128 ? 256 : 128;
  int rc = gemm_plan(&p, d_a, d_b, M, N, K, a_mn != 0, b_mn != 0, bn, epilogue, pair);
  if (rc) return rc;
  tc::GemmArgs& a = p.args;
  a.mode = mode;
  a.n_groups = n_groups;
  a.g_r0 = d_group_r0;
  a.g_r1 = d_group_r1;
  a.g_cta0 = d_group_cta0;
  a.g_ctan = d_group_ctan;
  a.timing = d_timing;
  if (epilogue == tc::kEpiF32)
    a.c_f32 = static_cast<float*>(d_c);
  else
    a.c_bf16 = static_cast<__nv_bfloat16*>(d_c);
  a.group_stride = static_cast<long long>(M) * N;
  a.bias = d_bias;
  a.aux = static_cast<const __nv_bfloat16*>(d_aux);
  a.ld_aux = N;
  if (!pair && (n_groups > 0 || ctas > 0)) p.ctas = ctas > 0 ? ctas : num_sms();
  return gemm_launch(p, static_cast<cudaStream_t>(stream));
}
