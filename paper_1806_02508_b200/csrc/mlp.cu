// mlp.cu -- the data-parallel MLP gradient engine of the LB-BSP iteration
// (north_star (1)-(4) on one or more B200s) and its C-ABI.
//
// One round (cluster_sim.cpp:349-469 with the simulated timing replaced by
// measured per-worker compute time under SM caps):
//   plan        P1-P4  trace -> SM caps, predictor -> v_pred, solver -> b_i
//   gather      P6     stream rows -> X, labels, Eq.6/7 row scales
//   fwd GEMMs   P7     per-worker CTA partitions, ragged rows masked
//   head        P7     softmax-CE + dlogits (+ small last layer on CUDA cores)
//   bwd         P7     bias-grad column sums, dW (k-split per worker), dX
//   reduce      P8     segmented reduction of worker partials (+ ncclAllReduce)
//   apply       P8     w -= lr g, bf16 copies
//   loss        P9     full-dataset loss (forward only)
//   observe     P10    measured t_p -> v (+ ncclAllGather), push histories
//   train       P10    NARX train_rotation
#include <cuda_bf16.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "common.cuh"
#include "exactmath.cuh"
#include "gemm.cuh"
#include "host.cuh"
#include "kernels.cuh"
#include "head_mma.cuh"
#include "mlp_kernels.cuh"
#include "predictor.cuh"
#include "solver.cuh"
#include "c2_fused.cuh"
#include "c2_fused_pair.cuh"
#include "c2_fused_quad.cuh"

namespace lbbsp {

cudaError_t launch_pred_train_from(const PredDev& P, const int* first_slot, cudaStream_t s);

// NCCL is resolved at run time (dlopen of libnccl.so.2): inside a PyTorch
// process this binds the NCCL build torch already loaded instead of forcing
// a second, older copy into the process.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
      api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
      api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    }
  }
  return api.AllReduce ? &api : nullptr;
}

namespace mlp {

using bf16 = __nv_bfloat16;
constexpr int kMaxPhases = 3 * LBBSP_MLP_MAX_LAYERS + 4;

// ---------------------------------------------------------------------------
// setup kernels (run once)
// ---------------------------------------------------------------------------
__global__ void init_x_kernel(bf16* x, long long count, uint64_t seed) {
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < count; i += 256ll * gridDim.x)
    x[i] = __float2bfloat16_rn(hash_uniform(seed, static_cast<uint64_t>(i), -1.f, 1.f));
}

// labels = argmax_c(W* x + U[-0.1, 0.1]) with a seeded teacher W* (the
// multi-class generalisation of generate_dataset, sgd.cpp:32-57), so every
// head width has a learnable target. Ties go to the lowest class.
__global__ void teacher_labels_kernel(const bf16* x, int* y, int d, int d_out, uint64_t seed) {
  __shared__ float acc[32];
  const int i = blockIdx.x;
  if (d_out > 32) {
    // wide heads: a thread per class (strided), the sample row in shared memory
    extern __shared__ float xs[];
    for (int j = threadIdx.x; j < d; j += blockDim.x) xs[j] = __bfloat162float(x[static_cast<long long>(i) * d + j]);
    __syncthreads();
    float bv = -1e30f;
    int best = d_out;
    for (int c = threadIdx.x; c < d_out; c += blockDim.x) {
      float s = 0.f;
      for (int j = 0; j < d; ++j)
        s += hash_uniform(seed ^ 0x5e9a7a70ull, static_cast<uint64_t>(c) * d + j, -1.f, 1.f) * xs[j];
      const float v = s + hash_uniform(seed ^ 0xda7a5e7ull, static_cast<uint64_t>(i) * d_out + c, -0.1f, 0.1f);
      if (v > bv) { bv = v; best = c; }
    }
    // block argmax, lowest class on ties
    __shared__ float rv[32];
    __shared__ int rc[32];
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oc = __shfl_xor_sync(0xffffffffu, best, o);
      if (ov > bv || (ov == bv && oc < best)) { bv = ov; best = oc; }
    }
    if ((threadIdx.x & 31) == 0) { rv[threadIdx.x / 32] = bv; rc[threadIdx.x / 32] = best; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < static_cast<int>(blockDim.x / 32); ++w)
        if (rv[w] > bv || (rv[w] == bv && rc[w] < best)) { bv = rv[w]; best = rc[w]; }
      y[i] = best;
    }
    return;
  }
  if (threadIdx.x < 32) acc[threadIdx.x] = 0.f;
  __syncthreads();
  for (int c = 0; c < d_out; ++c) {
    float s = 0.f;
    for (int j = threadIdx.x; j < d; j += blockDim.x)
      s += hash_uniform(seed ^ 0x5e9a7a70ull, static_cast<uint64_t>(c) * d + j, -1.f, 1.f) *
           __bfloat162float(x[static_cast<long long>(i) * d + j]);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) atomicAdd(&acc[c], s);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int best = 0;
    float bv = -1e30f;
    for (int c = 0; c < d_out; ++c) {
      const float v = acc[c] + hash_uniform(seed ^ 0xda7a5e7ull, static_cast<uint64_t>(i) * d_out + c, -0.1f, 0.1f);
      if (v > bv) { bv = v; best = c; }
    }
    y[i] = best;
  }
}

__global__ void init_params_kernel(float* p, bf16* pb, long long off_w, long long off_b, int dout,
                                   int din, uint64_t seed) {
  const float s = rsqrtf(static_cast<float>(din));
  const long long nw = static_cast<long long>(dout) * din;
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < nw; i += 256ll * gridDim.x) {
    const float w = hash_uniform(seed, static_cast<uint64_t>(off_w + i), -s, s);
    p[off_w + i] = w;
    pb[off_w + i] = __float2bfloat16_rn(w);
  }
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < dout; i += 256ll * gridDim.x) {
    p[off_b + i] = 0.f;
    pb[off_b + i] = __float2bfloat16_rn(0.f);
  }
}

// ---------------------------------------------------------------------------
// iteration state (device-resident) shared by the small kernels
// ---------------------------------------------------------------------------
struct PlanDev {
  int n_total, n_local, rank, B_total, scheme, static_sizes, sm_budget, trace_len;
  const int* static_sizes_d;
  const double* trace_c;
  const double* trace_m;
  const double* trace_mult;
  const double* share;  // [n_total]
  PredDev pred;
  long long* k;
  long long* round_k;  // k snapshot taken by the plan (stable for the whole round)
  int* rows;
  int max_rows;
  int* sizes_all;      // [n_total]
  int* r0;             // [n_local]
  int* r1;
  int* cta0;
  int* ctan;
  int* local_rows;     // scalar
  int* stream_off;     // scalar
  double* c_now;       // [n_total]
  double* m_now;
  double* v_pred;
  unsigned long long* timing;  // [kMaxPhases][n_local][2]
  double* v_obs_local;  // [n_local]
  double* v_obs_all;    // [n_total]
  double* loss_acc;
  int N_data;
  int loss_on;
  int* train_first;
  int* rec_sizes;
  double* rec_vpred;
  double* rec_vobs;
  int* rec_caps;
  double* rec_t;
  double* rec_loss;
  lbbsp_dev_status* status;
  unsigned long long* stamps;  // [16] globaltimer at kernel boundaries (last round)
  unsigned long long* gather_done;  // single rank: gather CTAs finished, summed over all rounds
  int straggler_mode;          // LBBSP_STRAGGLE_INTERFERE | LBBSP_STRAGGLE_SM_CAP
  int solver;                  // LBBSP_SOLVER_PROPORTIONAL | LBBSP_SOLVER_GAMMA
  int observe;                 // LBBSP_OBSERVE_RATE | LBBSP_OBSERVE_CAPACITY (proportional solver)
  // next-round predictions made by the observe branch (the models, histories
  // and EMA states are final there, and hot): v_next[w] is what the plan of
  // round *vnext_k would compute for worker w, bit for bit
  double* v_next;              // [n_total]
  double* nx_c;                // [n_total] trace c, m and availability of round *vnext_k
  double* nx_m;
  double* nx_a;
  float2* nx_intf;             // [n_local] interference weights of round *vnext_k
  long long* vnext_k;          // the round v_next is for (-1: none)
  unsigned long long* obs_seq; // rounds whose observe (history push, EMA) is complete
  const lbbsp_gpu_profile* prof0;  // [n_total] unloaded Gamma profiles (GAMMA solver, CAPACITY)
  float2* intf_w;              // [n_local] {availability, HBM share of the injected time}
  unsigned* fz_done;           // [n_local] fused worker kernel: head CTAs done (zeroed here)
  int cap_align;               // worker CTA partitions cluster-aligned: 2 (pair kernel), 4 (quad), else 1
  int plan_fast;               // one rank, n <= 32, proportional solver: plan_fast_body when the look-ahead is there
  int gather_ctas;             // > 0: the plan completes only once they all have
};

__device__ __forceinline__ void stamp(const PlanDev& D, int i) {
  if (threadIdx.x == 0 && blockIdx.x == 0) D.stamps[i] = gtimer();
}

// Single rank: the gather of the whole batch runs beside the plan; the plan
// completes only once every gather CTA of this round has, so the forward GEMM
// depends on the plan alone and keeps its programmatic (overlapped) launch.
// The arrival count only grows: round k waits for (k + 1) * gather_ctas, so a
// late CTA of an earlier round can never satisfy a later round's wait. A wait
// that times out (the gather never ran: kernels serialised by a tool) poisons
// the round -- status set, every worker's row range emptied -- instead of
// computing on a stale X. Tools that serialise kernels get the event join
// instead (LBBSP_GATHER_JOIN / CUDA_INJECTION64_PATH, see enqueue_iteration).
__device__ __forceinline__ bool wait_gather(const PlanDev& D, long long k) {
  __shared__ int ok_s;
  if (threadIdx.x == 0) {
    ok_s = 1;
    if (D.gather_ctas > 0) {
      const unsigned long long want = static_cast<unsigned long long>(k + 1) * D.gather_ctas;
      const unsigned long long t0 = gtimer();
      unsigned long long seen;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(D.gather_done) : "memory");
        if (gtimer() - t0 > 2000000000ull) {  // 2 s: the gather never ran -- fail, do not hang
          set_status(D.status, LBBSP_RUNTIME, 0, static_cast<long long>(seen), static_cast<long long>(want));
          ok_s = 0;
          break;
        }
      } while (seen < want);
    }
  }
  __syncthreads();
  return ok_s != 0;
}

// P1-P4: trace -> caps, predictor -> v_pred, solver -> sizes, local slice,
// plus the Eq. 6/7 row scales of this rank's rows. Everything thread 0 walks
// sequentially lives in shared memory (no dependent global round trips).
// Worker i's straggler state in round kk: trace (c, m), availability
// a = min(1, c * MemPenalty(m) * mult) (effective_speed * speed_mult,
// cluster_sim.cpp:22-29) and, in interference mode, the weights interfere.cuh
// injects (the part of the injected time the memory penalty adds,
// 1/a - 1/a_sm with a_sm = min(1, c mult), is HBM-bound, the rest SM-bound).
struct WorkerRound {
  double c, m, a;
  float2 intf;
};
__device__ inline WorkerRound worker_round(const PlanDev& D, int i, long long kk) {
  const long long ti = kk < D.trace_len - 1 ? kk : D.trace_len - 1;
  const size_t o = static_cast<size_t>(i) * D.trace_len + ti;
  WorkerRound r;
  r.c = D.trace_c[o];
  r.m = D.trace_m[o];
  const double mult = D.trace_mult[o];
  const double pen = r.m >= 0.5 ? 1.0 : dadd(0.25, dmul(0.75, ddiv(r.m, 0.5)));
  const double a = dmul(dmul(r.c, pen), mult);
  r.a = a < 1.0 ? a : 1.0;
  r.intf = make_float2(1.f, 0.f);
  if (D.straggler_mode == LBBSP_STRAGGLE_INTERFERE) {
    const double asm_ = fmin(1.0, r.c * mult), at = r.a;
    const double hbm = at < 1.0 ? fmax(0.0, fmin(1.0, (1.0 / at - 1.0 / asm_) / (1.0 / at - 1.0))) : 0.0;
    r.intf = make_float2(static_cast<float>(at), static_cast<float>(hbm));
  }
  return r;
}

// The observe branch's look-ahead for round kk = k + 1 (history length len
// after this round's push): every worker's straggler state and, for the
// workers in `mine` (all but the ones a training CTA predicts itself), the
// plan's prediction (Perfect: the availability, cluster_sim.cpp:362-367).
__device__ inline void look_ahead(const PlanDev& D, int i, long long kk, int len, bool predict) {
  const WorkerRound r = worker_round(D, i, kk);
  D.nx_c[i] = r.c;
  D.nx_m[i] = r.m;
  D.nx_a[i] = r.a;
  const int li = i - D.rank * D.n_local;
  if (li >= 0 && li < D.n_local) D.nx_intf[li] = r.intf;
  if (predict) D.v_next[i] = D.pred.kind == LBBSP_PRED_PERFECT ? r.a : predictor_predict_d(D.pred, i, len, r.c, r.m);
}

__device__ __forceinline__ void plan_body(const PlanDev& D, float* row_scale) {
  tc::pdl_launch_dependents();  // the forward GEMM's prologue may start now
  __shared__ SolverSmem sm;
  __shared__ double rem[LBBSP_MAX_WORKERS];
  __shared__ double avail[LBBSP_MAX_WORKERS];
  __shared__ double vp_s[LBBSP_MAX_WORKERS];
  __shared__ double share_s[LBBSP_MAX_WORKERS];
  __shared__ int sz[LBBSP_MAX_WORKERS];
  __shared__ int r0_s[LBBSP_MAX_WORKERS + 1];
  const int tid = threadIdx.x, n = D.n_total;
  stamp(D, 0);
  const long long k = *D.k;
  const int len = min(*D.pred.len, D.pred.max_hist);
  const long long vk = *D.vnext_k;
  // scalars needed later, loaded now beside k (no dependent round trips later)
  __shared__ int rows_s;
  __shared__ double loss_prev_s;
  if (tid == 0) {
    rows_s = *D.rows;
    loss_prev_s = D.loss_on ? *D.loss_acc : 0.0;
  }
  if (tid == 0) *D.round_k = k;
  if (k >= D.max_rows && tid == 0)
    set_status(D.status, LBBSP_RUNTIME, LBBSP_E_MLP_CAPACITY, k, D.max_rows);
  // Per worker: trace state, availability, interference weights and the
  // prediction. The observe branch of the last round computed all of them
  // for this round (vk == k: look_ahead, the same calls on the same state),
  // so the usual path only moves them -- a round's first instructions come
  // from DRAM after the L2 flush, and this kernel's latency is mostly fetch.
  for (int i = tid; i < n; i += blockDim.x) {
    share_s[i] = D.share[i];
    double c, m, a, vp;
    float2 iw = make_float2(1.f, 0.f);
    if (vk == k) {
      c = D.nx_c[i];
      m = D.nx_m[i];
      a = D.nx_a[i];
      vp = len >= 1 ? D.v_next[i] : 0.0;
    } else {
      const WorkerRound r = worker_round(D, i, k);
      c = r.c;
      m = r.m;
      a = r.a;
      iw = r.intf;
      // Perfect (step_sync: v_pred = v_actual, cluster_sim.cpp:362-367): the
      // worker's true relative speed this round is its injected availability
      vp = D.pred.kind == LBBSP_PRED_PERFECT ? a : (len >= 1 ? predictor_predict_d(D.pred, i, len, c, m) : 0.0);
    }
    D.c_now[i] = c;
    D.m_now[i] = m;
    avail[i] = a;
    if (D.straggler_mode == LBBSP_STRAGGLE_INTERFERE) {
      const int li = i - D.rank * D.n_local;
      if (li >= 0 && li < D.n_local) D.intf_w[li] = vk == k ? D.nx_intf[li] : iw;
    }
    vp_s[i] = vp;
    D.v_pred[i] = vp;
  }
  __syncthreads();
  stamp(D, 10);
  int code = 0;
  if (D.static_sizes) {
    for (int i = tid; i < n; i += blockDim.x) sz[i] = D.static_sizes_d[i];
  } else if (D.scheme == LBBSP_SCHEME_LBBSP && D.solver == LBBSP_SOLVER_GAMMA) {
    // GPU-cluster branch (cluster_sim.cpp:373-387): gpu_allocate over the
    // workers' Gamma profiles -- the unloaded profile scaled by the predicted
    // availability (clamp_speed_floor of v_pred) -- and the lagged comm EMA;
    // k < 2: initial_gpu_sizes (:471-484) on the unloaded profiles
    extern __shared__ double gsm[];
    lbbsp_gpu_profile* prof = reinterpret_cast<lbbsp_gpu_profile*>(gsm);
    double* comm = reinterpret_cast<double*>(prof + n);
    double* bp = comm + n;
    double* tmp = bp + 2 * n;
    __shared__ int feasible;
    for (int i = tid; i < n; i += blockDim.x) {
      const lbbsp_gpu_profile p0 = D.prof0[i];
      const double a = k < 2 ? 1.0 : (vp_s[i] > D.pred.floor ? vp_s[i] : D.pred.floor);
      prof[i] = lbbsp_gpu_profile{ddiv(p0.sec_per_sample, a), ddiv(p0.base_time_s, a), p0.saturation_point,
                                  p0.oom_point};
      comm[i] = k < 2 ? 0.0 : D.pred.comm_ema_lag[i];
      sz[i] = D.B_total / n + (i < D.B_total % n ? 1 : 0);
    }
    if (tid == 0) feasible = 1;
    __syncthreads();
    if (k < 2)
      for (int i = tid; i < n; i += blockDim.x)
        if (sz[i] < prof[i].saturation_point || sz[i] > prof[i].oom_point) feasible = 0;
    __syncthreads();
    if (k >= 2 || !feasible) code = block_gpu_allocate(prof, comm, n, D.B_total, sz, bp, tmp, &sm, D.status);
  } else if (D.scheme == LBBSP_SCHEME_LBBSP && k > 0) {
    code = block_cpu_allocate(vp_s, n, D.B_total, D.pred.floor, sz, rem, &sm, D.status);
  } else {
    for (int i = tid; i < n; i += blockDim.x)
      sz[i] = D.B_total / n + (i < D.B_total % n ? 1 : 0);  // equal_split
  }
  __syncthreads();
  stamp(D, 11);
  if (code) {
    wait_gather(D, k);
    return;
  }
  const int first = D.rank * D.n_local;
  if (tid == 0) {
    int off = 0;
    for (int i = 0; i < first; ++i) off += sz[i];
    *D.stream_off = off;
    int r = 0, c0 = 0;
    for (int i = 0; i < D.n_local; ++i) {
      const int w = first + i;
      r0_s[i] = r;
      D.r0[i] = r;
      r += sz[w];
      D.r1[i] = r;
      const double share = share_s[w];
      // SM-cap mode: the availability scales the CTA partition; interference
      // mode: the partition is the nominal share, the availability is injected
      const double av = D.straggler_mode == LBBSP_STRAGGLE_SM_CAP ? avail[w] : 1.0;
      int cap = static_cast<int>(floor(static_cast<double>(D.sm_budget) * share * av));
      cap = cap < 1 ? 1 : cap;
      if (D.cap_align > 1) cap = cap < D.cap_align ? D.cap_align : cap - cap % D.cap_align;  // clusters
      if (c0 + cap > D.sm_budget) cap = D.sm_budget - c0 > 0 ? D.sm_budget - c0 : 1;
      D.cta0[i] = c0;
      D.ctan[i] = cap;
      c0 += cap;
    }
    r0_s[D.n_local] = r;
    *D.local_rows = r;
    // the previous round's full-dataset loss (computed beside its observe branch)
    const int prev = rows_s - 1;
    if (prev >= 0 && prev < D.max_rows)
      D.rec_loss[prev] = D.loss_on ? loss_prev_s / static_cast<double>(D.N_data) : -1.0;
    *D.loss_acc = 0.0;
  }
  for (int i = tid; i < kMaxPhases * D.n_local; i += blockDim.x) {
    D.timing[2 * i] = ~0ull;
    D.timing[2 * i + 1] = 0ull;
  }
  if (D.fz_done)
    for (int i = tid; i < D.n_local; i += blockDim.x) D.fz_done[i] = 0u;
  if (tid == 0) {
    D.stamps[6] = ~0ull;  // loss-branch head {first start, last end}
    D.stamps[7] = 0ull;
  }
  for (int i = tid; i < n; i += blockDim.x) D.sizes_all[i] = sz[i];
  __syncthreads();
  stamp(D, 12);
  // row scales: Eq. 7 folds 1/B into every row; Eq. 6 (BSP) 1/(n b_i) per worker
  const int rows = r0_s[D.n_local];
  if (D.scheme == LBBSP_SCHEME_LBBSP) {
    const float s = 1.0f / static_cast<float>(D.B_total);
    for (int r = tid; r < rows; r += blockDim.x) row_scale[r] = s;
  } else {
    for (int g = 0; g < D.n_local; ++g) {
      const float s = 1.0f / (static_cast<float>(D.n_total) * static_cast<float>(sz[first + g]));
      for (int r = r0_s[g] + tid; r < r0_s[g + 1]; r += blockDim.x) row_scale[r] = s;
    }
  }
  const int row = rows_s;
  if (row < D.max_rows) {
    for (int i = tid; i < n; i += blockDim.x) {
      D.rec_sizes[static_cast<size_t>(row) * n + i] = sz[i];
      D.rec_vpred[static_cast<size_t>(row) * n + i] = vp_s[i];
    }
    for (int i = tid; i < D.n_local; i += blockDim.x)
      D.rec_caps[static_cast<size_t>(row) * n + D.rank * D.n_local + i] = D.ctan[i];
  }
  stamp(D, 8);  // plan computed; the wait for the gather follows
  if (!wait_gather(D, k)) {  // poisoned round: no worker computes on a stale batch
    for (int i = tid; i < D.n_local; i += blockDim.x) D.r1[i] = D.r0[i];
    if (tid == 0) *D.local_rows = 0;
  }
  stamp(D, 1);
}

// dynamic shared memory of the plan for the Gamma solver: profiles, comm,
// breakpoints and scratch (block_gpu_allocate)
static size_t gamma_plan_smem(int n) {
  return static_cast<size_t>(n) * sizeof(lbbsp_gpu_profile) + static_cast<size_t>(n) * 8 * 5 + 64;
}

__global__ void __launch_bounds__(256) plan_kernel(const __grid_constant__ PlanDev D, float* row_scale);

// P6: X[r] = data[stream[off + r]], labels, row scale (Eq. 7: 1/B; Eq. 6: 1/(n b_i))
// fixed_rows > 0: a single rank gathers the whole batch [0, B) of stream k,
// which does not depend on the plan, so it runs beside the plan (the blocks
// 1.. of plan_gather_kernel). Block bid of nblk.
__device__ __forceinline__ void gather_body(const PlanDev& D, const int* streams, int B_total, const bf16* data_x,
                                            const int* data_y, int d0, bf16* X, int* y, int fixed_rows,
                                            float* slab, long long slab_stride, const long long* reg_off,
                                            const long long* reg_len, int n_reg, int bid, int nblk) {
  if (threadIdx.x == 0 && bid == 0) D.stamps[2] = gtimer();
  // zero the partial regions accumulated with atomics (biases, small head)
  for (int sl = 0; sl < D.n_local; ++sl)
    for (int rg = 0; rg < n_reg; ++rg) {
      float* p = slab + sl * slab_stride + reg_off[rg];
      for (long long i = bid * 256ll + threadIdx.x; i < reg_len[rg]; i += 256ll * nblk)
        p[i] = 0.f;
    }
  // several ranks: the slice offset and length come from the plan (programmatic
  // launch: the zeroing above overlaps the plan)
  tc::pdl_wait();
  tc::pdl_launch_dependents();
  const long long k = min(*D.k, static_cast<long long>(D.max_rows - 1));  // capacity-guarded
  const int rows = fixed_rows > 0 ? fixed_rows : *D.local_rows;
  const int off = fixed_rows > 0 ? 0 : *D.stream_off;
  const int* idx = streams + static_cast<size_t>(k) * B_total + off;
  const int vec = d0 / 8;  // 16-byte chunks per row
  const int total = rows * vec;
  const int step = 256 * nblk;
  const uint4* src4 = reinterpret_cast<const uint4*>(data_x);
  uint4* dst4 = reinterpret_cast<uint4*>(X);
  // four independent row reads in flight per thread
  for (int t0 = bid * 256 + threadIdx.x; t0 < total; t0 += 4 * step) {
    uint4 v[4];
    int dsti[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * step;
      dsti[u] = -1;
      if (t < total) {
        const int r = t / vec, c = t - r * vec;
        v[u] = __ldg(&src4[static_cast<size_t>(__ldg(&idx[r])) * vec + c]);
        dsti[u] = t;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (dsti[u] >= 0) dst4[dsti[u]] = v[u];
  }
  for (int r = bid * 256 + threadIdx.x; r < rows; r += 256 * nblk) y[r] = data_y[idx[r]];
  if (D.stamps && threadIdx.x == 0) atomicMax(&D.stamps[9], static_cast<unsigned long long>(gtimer()));
  if (fixed_rows > 0 && D.gather_ctas > 0) {  // tell the plan (see plan_kernel)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(D.gather_done, 1ull);
    }
  }
}

__global__ void gather_kernel(PlanDev D, const int* streams, int B_total, const bf16* data_x,
                              const int* data_y, int d0, bf16* X, int* y, int fixed_rows,
                              float* slab, long long slab_stride, const long long* reg_off,
                              const long long* reg_len, int n_reg) {
  gather_body(D, streams, B_total, data_x, data_y, d0, X, y, fixed_rows, slab, slab_stride, reg_off, reg_len,
              n_reg, blockIdx.x, gridDim.x);
}

// The plan of a round whose per-worker state the observe branch computed
// ahead (vk == k): n <= 32 workers in all, the proportional solver. The
// same arithmetic as plan_body, with every per-worker step in one lane of
// warp 0 -- the sizes' and caps' prefix sums by warp scans -- so the round's
// first kernel fetches a few hundred instructions instead of the general
// plan's thousand-odd (cold after the bench's L2 flush, they set its
// latency). Falls back to plan_body otherwise.
__device__ __forceinline__ void plan_fast_body(const PlanDev& D, float* row_scale) {
  const int tid = threadIdx.x, lane = tid & 31, n = D.n_total;
  __shared__ long long k_s, vk_s;
  __shared__ int len_s, rows_s;
  __shared__ double loss_s;
  if (tid == 0) {
    k_s = *D.k;
    vk_s = *D.vnext_k;
    len_s = min(*D.pred.len, D.pred.max_hist);
    rows_s = *D.rows;
    loss_s = D.loss_on ? *D.loss_acc : 0.0;
  }
  __syncthreads();
  const long long k = k_s;
  if (vk_s != k || k >= D.max_rows) {
    __syncthreads();
    plan_body(D, row_scale);
    return;
  }
  tc::pdl_launch_dependents();
  stamp(D, 0);
  __shared__ SolverSmem sm;
  __shared__ double vp_s[32];
  __shared__ int sz[32];
  // warp 0: the workers' state; the other warps reset the round's counters
  double vp = 0.0, share = 0.0, a = 0.0;
  if (tid < 32) {
    if (lane < n) {
      const double c = D.nx_c[lane], m = D.nx_m[lane];
      a = D.nx_a[lane];
      share = D.share[lane];
      vp = D.pred.kind == LBBSP_PRED_PERFECT ? a : (len_s >= 1 ? D.v_next[lane] : 0.0);
      D.c_now[lane] = c;
      D.m_now[lane] = m;
      const int li = lane - D.rank * D.n_local;
      if (D.straggler_mode == LBBSP_STRAGGLE_INTERFERE && li >= 0 && li < D.n_local) D.intf_w[li] = D.nx_intf[li];
      D.v_pred[lane] = vp;
      vp_s[lane] = vp;
      sz[lane] = D.static_sizes ? D.static_sizes_d[lane] : D.B_total / n + (lane < D.B_total % n ? 1 : 0);
    }
    if (tid == 0) *D.round_k = k;
  } else {
    for (int i = tid - 32; i < kMaxPhases * D.n_local; i += blockDim.x - 32) {
      D.timing[2 * i] = ~0ull;
      D.timing[2 * i + 1] = 0ull;
    }
    if (D.fz_done)
      for (int i = tid - 32; i < D.n_local; i += blockDim.x - 32) D.fz_done[i] = 0u;
    if (tid == 32) {
      D.stamps[6] = ~0ull;  // loss-branch head {first start, last end}
      D.stamps[7] = 0ull;
    }
  }
  __syncthreads();
  stamp(D, 10);
  int code = 0;
  if (!D.static_sizes && D.scheme == LBBSP_SCHEME_LBBSP && k > 0)
    code = warp_cpu_allocate(vp_s, n, D.B_total, D.pred.floor, sz, &sm, D.status);  // ends with __syncthreads
  stamp(D, 11);
  if (code) {
    wait_gather(D, k);
    return;
  }
  __shared__ int local_total_s;
  const int first = D.rank * D.n_local, nl = D.n_local;
  if (tid < 32) {
    const int x = lane < n ? sz[lane] : 0;
    const bool local = lane >= first && lane < first + nl;
    const int li = lane - first;
    // the stream offsets: exclusive prefix of the sizes over all workers
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int off = first > 0 ? __shfl_sync(0xffffffffu, incl, first - 1) : 0;  // this rank's first row
    const int r0 = incl - x - off;
    const int total = __shfl_sync(0xffffffffu, incl, first + nl - 1) - off;
    // CTA partitions of the local workers: floor(budget * share * av),
    // aligned; their prefix -- the sequential clamp of plan_body only acts
    // when the caps overrun the budget, then lane 0 runs that loop
    int cap = 0;
    if (local) {
      const double av = D.straggler_mode == LBBSP_STRAGGLE_SM_CAP ? a : 1.0;
      cap = static_cast<int>(floor(static_cast<double>(D.sm_budget) * share * av));
      cap = cap < 1 ? 1 : cap;
      if (D.cap_align > 1) cap = cap < D.cap_align ? D.cap_align : cap - cap % D.cap_align;
    }
    int cincl = cap;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, cincl, o);
      if (lane >= o) cincl += y;
    }
    const bool over = __shfl_sync(0xffffffffu, cincl, 31) > D.sm_budget;
    if (lane < n) D.sizes_all[lane] = x;
    if (local) {
      D.r0[li] = r0;
      D.r1[li] = r0 + x;
      if (!over) {
        D.cta0[li] = cincl - cap;
        D.ctan[li] = cap;
      }
    }
    if (over && lane == 0) {
      int c0 = 0;
      for (int i = 0; i < nl; ++i) {
        const int w = first + i;
        const double av = D.straggler_mode == LBBSP_STRAGGLE_SM_CAP ? D.nx_a[w] : 1.0;
        int cp = static_cast<int>(floor(static_cast<double>(D.sm_budget) * D.share[w] * av));
        cp = cp < 1 ? 1 : cp;
        if (D.cap_align > 1) cp = cp < D.cap_align ? D.cap_align : cp - cp % D.cap_align;
        if (c0 + cp > D.sm_budget) cp = D.sm_budget - c0 > 0 ? D.sm_budget - c0 : 1;
        D.cta0[i] = c0;
        D.ctan[i] = cp;
        c0 += cp;
      }
    }
    __syncwarp();
    const int row = rows_s;
    if (row < D.max_rows && lane < n) {
      D.rec_sizes[static_cast<size_t>(row) * n + lane] = x;
      D.rec_vpred[static_cast<size_t>(row) * n + lane] = vp_s[lane];
      if (local) D.rec_caps[static_cast<size_t>(row) * n + lane] = over ? D.ctan[li] : cap;
    }
    if (lane == 0) {
      *D.stream_off = off;
      *D.local_rows = total;
      local_total_s = total;
      const int prev = row - 1;
      if (prev >= 0 && prev < D.max_rows)
        D.rec_loss[prev] = D.loss_on ? loss_s / static_cast<double>(D.N_data) : -1.0;
      *D.loss_acc = 0.0;
    }
  }
  __syncthreads();
  // row scales: Eq. 7 folds 1/B into every row; Eq. 6 (BSP) 1/(n b_i) per worker
  if (D.scheme == LBBSP_SCHEME_LBBSP) {
    const float sc = 1.0f / static_cast<float>(D.B_total);
    for (int r = tid; r < local_total_s; r += blockDim.x) row_scale[r] = sc;
  } else {
    int r = 0;
    for (int g = 0; g < nl; ++g) {
      const int b = sz[first + g];
      const float sc = 1.0f / (static_cast<float>(D.n_total) * static_cast<float>(b));
      for (int q = r + tid; q < r + b; q += blockDim.x) row_scale[q] = sc;
      r += b;
    }
  }
  stamp(D, 12);
  stamp(D, 8);
  if (!wait_gather(D, k)) {  // poisoned round: no worker computes on a stale batch
    if (tid < nl) D.r1[tid] = D.r0[tid];
    if (tid == 0) *D.local_rows = 0;
  }
  stamp(D, 1);
}

__global__ void __launch_bounds__(256) plan_kernel(const __grid_constant__ PlanDev D, float* row_scale) {
  if (D.plan_fast)
    plan_fast_body(D, row_scale);
  else
    plan_body(D, row_scale);
}

// Single rank: block 0 plans the round, blocks 1.. gather its batch -- one
// launch, so the two run side by side (as two graph roots the plan started
// only once the gather had finished: 6.6 us on the round's critical path).
struct GatherArgs {
  const int* streams;
  int B_total;
  const bf16* data_x;
  const int* data_y;
  int d0;
  bf16* X;
  int* y;
  float* slab;
  long long slab_stride;
  const long long* reg_off;
  const long long* reg_len;
  int n_reg;
};
__global__ void __launch_bounds__(256) plan_gather_kernel(const __grid_constant__ PlanDev D, float* row_scale,
                                                          const __grid_constant__ GatherArgs a) {
  if (blockIdx.x == 0) {
    if (D.plan_fast)
      plan_fast_body(D, row_scale);
    else
      plan_body(D, row_scale);
  } else
    gather_body(D, a.streams, a.B_total, a.data_x, a.data_y, a.d0, a.X, a.y, a.B_total, a.slab, a.slab_stride,
                a.reg_off, a.reg_len, a.n_reg, blockIdx.x - 1, gridDim.x - 1);
}

__device__ __forceinline__ unsigned long long phase_begin(unsigned long long* timing, int g) {
  const unsigned long long t = gtimer();
  if (timing && threadIdx.x == 0) atomicMin(&timing[2 * g], t);
  return t;
}
// end of worker g's share of a phase: the injected interference, then the stamp
__device__ __forceinline__ void phase_finish(const Groups& G, unsigned long long* timing, int g,
                                             unsigned long long t_cta0) {
  if (G.n > 0) interfere(G.intf, g, timing ? &timing[2 * g] : nullptr, t_cta0);
  if (timing && threadIdx.x == 0) atomicMax(&timing[2 * g + 1], static_cast<unsigned long long>(gtimer()));
}

// Large softmax-CE head: one warp per row -- the fallback for other widths over bf16 logits [rows][n_out]
// (n_out % 256 == 0): loss and dZ = (softmax - onehot) * row_scale.
__global__ void __launch_bounds__(256) softmax_ce_kernel(
    Groups G, int rows_total, const bf16* __restrict__ logits, int n_out,
    const int* __restrict__ y, const float* __restrict__ row_scale, bf16* dZ, double* loss_acc,
    unsigned long long* timing) {
  int g, cta_in, cta_cnt;
  if (!my_group(G, &g, &cta_in, &cta_cnt)) return;
  const unsigned long long t_cta0 = phase_begin(timing, g);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const int r0 = G.n ? G.r0[g] : 0, r1 = G.n ? G.r1[g] : rows_total;
  double lsum = 0.0;
  for (int r = r0 + cta_in * nw + warp; r < r1; r += cta_cnt * nw) {
    const uint4* row = reinterpret_cast<const uint4*>(logits + static_cast<long long>(r) * n_out);
    const int nv = n_out / 8;
    float mx = -1e30f;
    for (int v = lane; v < nv; v += 32) {
      const uint4 q = row[v];
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(b2[j]);
        mx = fmaxf(mx, fmaxf(f.x, f.y));
      }
    }
    mx = warp_max(mx);
    float se = 0.f;
    for (int v = lane; v < nv; v += 32) {
      const uint4 q = row[v];
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(b2[j]);
        se += __expf(f.x - mx) + __expf(f.y - mx);
      }
    }
    se = warp_sum(se);
    const int yr = y[r];
    const float ly = __bfloat162float(logits[static_cast<long long>(r) * n_out + yr]);
    if (lane == 0) lsum += static_cast<double>(logf(se) + mx - ly);
    if (dZ) {
      const float inv = 1.f / se, sc = row_scale[r];
      uint4* out = reinterpret_cast<uint4*>(dZ + static_cast<long long>(r) * n_out);
      for (int v = lane; v < nv; v += 32) {
        const uint4 q = row[v];
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&q);
        uint4 o;
        __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(b2[j]);
          const int c = v * 8 + 2 * j;
          const float a = (__expf(f.x - mx) * inv - (c == yr ? 1.f : 0.f)) * sc;
          const float b = (__expf(f.y - mx) * inv - (c + 1 == yr ? 1.f : 0.f)) * sc;
          o2[j] = __floats2bfloat162_rn(a, b);
        }
        out[v] = o;
      }
    }
  }
  if (loss_acc && lane == 0 && lsum != 0.0) atomicAdd(loss_acc, lsum);
  __syncthreads();
  phase_finish(G, timing, g, t_cta0);
}

// Softmax-CE head for n_out = 256 * NV (NV <= 16): one warp per row, the row
// read once into registers (max, sum and dlogits from the same values), and
// the next row's loads issued before this row's math.
template <int NV>
__global__ void __launch_bounds__(256) softmax_ce_reg_kernel(
    Groups G, int rows_total, const bf16* __restrict__ logits, const int* __restrict__ y,
    const float* __restrict__ row_scale, bf16* dZ, double* loss_acc, unsigned long long* timing) {
  constexpr int n_out = 256 * NV;
  int g, cta_in, cta_cnt;
  if (!my_group(G, &g, &cta_in, &cta_cnt)) return;
  tc::pdl_wait();
  tc::pdl_launch_dependents();
  const unsigned long long t_cta0 = phase_begin(timing, g);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const int r0 = G.n ? G.r0[g] : 0, r1 = G.n ? G.r1[g] : rows_total;
  double lsum = 0.0;
  const int stride = cta_cnt * nw;
  int r = r0 + cta_in * nw + warp;
  uint4 nq[NV];
  if (r < r1) {
    const uint4* row = reinterpret_cast<const uint4*>(logits + static_cast<long long>(r) * n_out);
#pragma unroll
    for (int v = 0; v < NV; ++v) nq[v] = __ldg(&row[lane + 32 * v]);
  }
  for (; r < r1; r += stride) {
    uint4 q[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) q[v] = nq[v];
    if (r + stride < r1) {
      const uint4* nrow = reinterpret_cast<const uint4*>(logits + static_cast<long long>(r + stride) * n_out);
#pragma unroll
      for (int v = 0; v < NV; ++v) nq[v] = __ldg(&nrow[lane + 32 * v]);
    }
    float mx = -1e30f;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&q[v]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(b2[j]);
        mx = fmaxf(mx, fmaxf(f.x, f.y));
      }
    }
    mx = warp_max(mx);
    float se = 0.f;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&q[v]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(b2[j]);
        se += __expf(f.x - mx) + __expf(f.y - mx);
      }
    }
    se = warp_sum(se);
    const int yr = y[r];
    const float ly = __bfloat162float(logits[static_cast<long long>(r) * n_out + yr]);
    if (lane == 0) lsum += static_cast<double>(logf(se) + mx - ly);
    if (dZ) {
      const float inv = 1.f / se, sc = row_scale[r];
      uint4* out = reinterpret_cast<uint4*>(dZ + static_cast<long long>(r) * n_out);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&q[v]);
        uint4 o;
        __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(b2[j]);
          const int c = (lane + 32 * v) * 8 + 2 * j;
          const float a = (__expf(f.x - mx) * inv - (c == yr ? 1.f : 0.f)) * sc;
          const float b = (__expf(f.y - mx) * inv - (c + 1 == yr ? 1.f : 0.f)) * sc;
          o2[j] = __floats2bfloat162_rn(a, b);
        }
        out[lane + 32 * v] = o;
      }
    }
  }
  if (loss_acc && lane == 0 && lsum != 0.0) atomicAdd(loss_acc, lsum);
  __syncthreads();
  phase_finish(G, timing, g, t_cta0);
}

static cudaError_t launch_softmax_ce(int sms, cudaStream_t s, bool pdl, Groups G, int rows_total,
                                     const bf16* logits, int n_out, const int* y,
                                     const float* row_scale, bf16* dZ, double* loss_acc,
                                     unsigned long long* timing) {
  switch (n_out) {
#define LBBSP_SMX(NV_)                                                                          \
  case 256 * NV_:                                                                               \
    return launch_maybe_pdl(softmax_ce_reg_kernel<NV_>, sms, 256, 0, s, pdl, G, rows_total, logits, \
                            y, row_scale, dZ, loss_acc, timing);
    LBBSP_SMX(1)
    LBBSP_SMX(2)
    LBBSP_SMX(4)
    LBBSP_SMX(8)
    LBBSP_SMX(16)
#undef LBBSP_SMX
    default:
      softmax_ce_kernel<<<sms, 256, 0, s>>>(G, rows_total, logits, n_out, y, row_scale, dZ,
                                            loss_acc, timing);
      return cudaGetLastError();
  }
}


// db partial of worker g = column sums of dZ over its rows (N % 8 == 0),
// written into the worker's slab (or its bf16 bucket). Work units are
// 256-column strips x row chunks (the worker's CTAs / strips chunks per
// strip, two CTAs per partition slot): a warp reads 512 contiguous bytes of
// a row (16 B = 8 columns per lane), the rows streaming through shared memory
// by cp.async in 4 stages of 4 rows per row lane (64 KB per CTA in flight).
// A unit's 8 row-lane sums are added in lane order in shared memory; with
// several chunks per strip each unit writes its partial row to the scratch
// and the last unit to arrive on the strip's counter (self-resetting) adds
// the chunk partials in chunk order -- deterministic for a given CTA
// partition, one pass over dZ. C3 layer (4096 x 4096 bf16): 8.2 us in the
// round (was 22.5 with 32-column strips and register loads, which ptxas
// interleaved with the adds: one or two loads in flight), 13.6 us cold
// under ncu (profiles/r02_c3_hbm_kernels.txt).
constexpr int kBiasCols = 2048;  // (scratch sizing floor, kept for the C-ABI's allocation)
constexpr int kBiasStrip = 256;
constexpr int kBiasLanes = 256 / (kBiasStrip / 8);  // 8 row lanes
constexpr int kBiasRowsInFlight = 4;  // rows per lane per cp.async batch
constexpr int kBiasStages = 4;
constexpr int kBiasCtasPerSlot = 2;
constexpr int kBiasSmem = kBiasStages * kBiasRowsInFlight * 256 * 16;  // cp.async stages
__host__ __device__ constexpr int bias_strips(int N) { return (N + kBiasStrip - 1) / kBiasStrip; }
template <int kPerSlot>
__global__ void __launch_bounds__(256) bias_grad_kernel(Groups G, const bf16* __restrict__ dZ, int N,
                                                        float* slab, long long slab_stride,
                                                        long long off_b, float* scratch,
                                                        unsigned* counters, bf16* out_b16,
                                                        unsigned long long* timing) {
  // launched with kPerSlot CTAs per partition slot (more rows in
  // flight per SM); slot s = blockIdx.x / kPerSlot keeps the worker's
  // CTA partition
  int g = 0, cta_in = blockIdx.x, cta_cnt = gridDim.x;
  if (G.n > 0) {
    const int slot = blockIdx.x / kPerSlot;
    bool found = false;
    for (int i = 0; i < G.n && !found; ++i) {
      const int c0 = G.cta0[i], cn = G.ctan[i];
      if (slot >= c0 && slot < c0 + cn) {
        g = i;
        cta_in = (slot - c0) * kPerSlot + static_cast<int>(blockIdx.x % kPerSlot);
        cta_cnt = cn * kPerSlot;
        found = true;
      }
    }
    if (!found) return;
  }
  const int n_strips = bias_strips(N);
  const int n_chunks = cta_cnt / n_strips > 1 ? cta_cnt / n_strips : 1;
  const int n_units = n_strips * n_chunks;
  if (cta_in >= n_units) return;
  const unsigned long long t_cta0 = phase_begin(timing, g);
  __shared__ __align__(16) float red[kBiasLanes][kBiasStrip];
  __shared__ int s_last;
  extern __shared__ __align__(16) uint4 stage[];  // [kBiasStages][kBiasRowsInFlight][256]
  const int R0 = G.n ? G.r0[g] : 0, R1 = G.n ? G.r1[g] : 0;
  const long long R = R1 - R0;
  const int cl = threadIdx.x % 32, rl = threadIdx.x / 32;
  float* gs = slab + static_cast<long long>(g) * slab_stride + off_b;
  // worker g's [n_chunks][N] partials: chunk counts are floor(ctan / strips)
  // (>= 1), so these offsets never overlap (scratch: 2 sms * 256 + n_local * N)
  float* part = scratch + static_cast<long long>((G.n ? G.cta0[g] * kPerSlot : 0) / n_strips + g) * N;
  unsigned* cnt = counters + static_cast<long long>(g) * n_strips;
  for (int u = cta_in; u < n_units; u += cta_cnt) {
    const int st = u % n_strips, ch = u / n_strips;
    const int ra = R0 + static_cast<int>(R * ch / n_chunks), rb = R0 + static_cast<int>(R * (ch + 1) / n_chunks);
    const int col = st * kBiasStrip + cl * 8;
    float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (col < N) {
      // rows stream through shared memory by cp.async (16 B per row per
      // thread, kBiasRowsInFlight rows per batch, two batches in flight): the
      // copies need no registers, so every one of them issues before the
      // adds (register loads were interleaved with the adds by ptxas, one
      // or two in flight). Each thread reads back only its own slots. Rows
      // past the chunk are zero-filled (src-size 0; x + 0.0f == x).
      const bf16* base = dZ + col;
      const int step = kBiasLanes * kBiasRowsInFlight;
      auto issue = [&](int buf, int r) {
#pragma unroll
        for (int v = 0; v < kBiasRowsInFlight; ++v) {
          const int rr = r + kBiasLanes * v;
          const bf16* src = base + static_cast<long long>(rr < rb ? rr : ra) * N;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                           tc::smem_u32(&stage[(buf * kBiasRowsInFlight + v) * 256 + threadIdx.x])),
                       "l"(src), "r"(rr < rb ? 16 : 0)
                       : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      // kBiasStages batches in flight: the prologue issues S-1, each step
      // issues one more (or an empty group) and waits for the oldest
#pragma unroll
      for (int b = 0; b < kBiasStages - 1; ++b) {
        if (ra + rl + b * step < rb)
          issue(b, ra + rl + b * step);
        else
          asm volatile("cp.async.commit_group;" ::: "memory");
      }
      int buf = 0;
#pragma unroll 1
      for (int r = ra + rl; r < rb; r += step) {
        const int rn = r + (kBiasStages - 1) * step;
        const int bn = buf == 0 ? kBiasStages - 1 : buf - 1;
        if (rn < rb)
          issue(bn, rn);
        else
          asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(kBiasStages - 1) : "memory");
#pragma unroll
        for (int v = 0; v < kBiasRowsInFlight; ++v) {
          const uint4 q = stage[(buf * kBiasRowsInFlight + v) * 256 + threadIdx.x];
          const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(b2[j]);
            a[2 * j] += f.x;
            a[2 * j + 1] += f.y;
          }
        }
        buf = buf + 1 == kBiasStages ? 0 : buf + 1;
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    reinterpret_cast<float4*>(&red[rl][cl * 8])[0] = make_float4(a[0], a[1], a[2], a[3]);
    reinterpret_cast<float4*>(&red[rl][cl * 8])[1] = make_float4(a[4], a[5], a[6], a[7]);
    __syncthreads();
    const int c = st * kBiasStrip + threadIdx.x;
    float v = 0.f;
#pragma unroll
    for (int q = 0; q < kBiasLanes; ++q) v += red[q][threadIdx.x];
    bool write = n_chunks == 1;
    if (!write) {
      if (c < N) part[static_cast<long long>(ch) * N + c] = v;
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_last = atomicAdd(&cnt[st], 1u) == static_cast<unsigned>(n_chunks - 1);
      __syncthreads();
      write = s_last;
      if (write) {
        __threadfence();
        if (threadIdx.x == 0) cnt[st] = 0u;
        v = 0.f;
        if (c < N) {
          const float* pc = part + c;
          int q = 0;
          for (; q + 8 <= n_chunks; q += 8) {
            float t[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) t[j] = __ldcg(pc + static_cast<long long>(q + j) * N);
#pragma unroll
            for (int j = 0; j < 8; ++j) v += t[j];
          }
          for (; q < n_chunks; ++q) v += __ldcg(pc + static_cast<long long>(q) * N);
        }
      }
    }
    if (write && c < N) {
      if (out_b16)
        out_b16[c] = __float2bfloat16_rn(v);
      else
        gs[c] = v;
    }
    __syncthreads();
  }
  phase_finish(G, timing, g, t_cta0);
}

// Segmented reduction of the worker partial slabs + SGD apply (K8+K9), HBM-
// bound: reads (n+1) P fp32, writes P fp32 + P bf16. `apply` == 0 only
// reduces into grad (the allreduce then runs on grad).
__global__ void __launch_bounds__(256) reduce_apply_kernel(const float* __restrict__ partial, int n,
                                                           long long P, float* grad, float* params,
                                                           bf16* pb, float lr, int apply,
                                                           unsigned long long* stamps) {
  tc::pdl_wait();  // the worker partials come from the backward GEMMs
  tc::pdl_launch_dependents();
  if (stamps && threadIdx.x == 0 && blockIdx.x == 0) stamps[5] = gtimer();
  const long long nv = P / 4;
  for (long long v = blockIdx.x * 256ll + threadIdx.x; v < nv; v += 256ll * gridDim.x) {
    float4 s = reinterpret_cast<const float4*>(partial)[v];
    for (int g = 1; g < n; ++g) {
      const float4 q = reinterpret_cast<const float4*>(partial + g * P)[v];
      s.x += q.x; s.y += q.y; s.z += q.z; s.w += q.w;
    }
    if (!apply) {
      reinterpret_cast<float4*>(grad)[v] = s;
      continue;
    }
    float4 w = reinterpret_cast<float4*>(params)[v];
    w.x -= lr * s.x; w.y -= lr * s.y; w.z -= lr * s.z; w.w -= lr * s.w;
    reinterpret_cast<float4*>(params)[v] = w;
    __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(pb) + 2 * v;
    o[0] = __floats2bfloat162_rn(w.x, w.y);
    o[1] = __floats2bfloat162_rn(w.z, w.w);
  }
}

// SGD apply from an all-reduced bf16 gradient bucket (+ the bf16 weight copy)
__global__ void __launch_bounds__(256) apply_bf16_kernel(const bf16* __restrict__ g, long long n,
                                                         float* params, bf16* pb, float lr) {
  const long long nv = n / 8;
  for (long long v = blockIdx.x * 256ll + threadIdx.x; v < nv; v += 256ll * gridDim.x) {
    const uint4 q = reinterpret_cast<const uint4*>(g)[v];
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&q);
    float4* p4 = reinterpret_cast<float4*>(params) + 2 * v;
    float4 w0 = p4[0], w1 = p4[1];
    const float2 a = __bfloat1622float2(g2[0]), b = __bfloat1622float2(g2[1]);
    const float2 c = __bfloat1622float2(g2[2]), d = __bfloat1622float2(g2[3]);
    w0.x -= lr * a.x; w0.y -= lr * a.y; w0.z -= lr * b.x; w0.w -= lr * b.y;
    w1.x -= lr * c.x; w1.y -= lr * c.y; w1.z -= lr * d.x; w1.w -= lr * d.y;
    p4[0] = w0;
    p4[1] = w1;
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
    o2[0] = __floats2bfloat162_rn(w0.x, w0.y);
    o2[1] = __floats2bfloat162_rn(w0.z, w0.w);
    o2[2] = __floats2bfloat162_rn(w1.x, w1.y);
    o2[3] = __floats2bfloat162_rn(w1.z, w1.w);
    reinterpret_cast<uint4*>(pb)[v] = o;
  }
}

// zero the partial regions that are accumulated with atomics (biases, head)
__global__ void zero_regions_kernel(float* slab, long long slab_stride, int n_slabs,
                                    const long long* reg_off, const long long* reg_len, int n_reg) {
  for (int s = 0; s < n_slabs; ++s)
    for (int r = 0; r < n_reg; ++r) {
      float* p = slab + s * slab_stride + reg_off[r];
      for (long long i = blockIdx.x * 256ll + threadIdx.x; i < reg_len[r]; i += 256ll * gridDim.x) p[i] = 0.f;
    }
}

// One worker per GPU: zero rows [rows, roundup64(rows)) of every dZ buffer so
// the CTA-pair dW GEMM can read whole 64-row K blocks; record the rounded end.
__global__ void zero_dz_tail_kernel(PlanDev D, bf16** dz, const int* widths, int n_layers,
                                    int* dz_end, int cap) {
  const int rows = *D.local_rows;
  int end = (rows + 63) / 64 * 64;
  end = end < cap ? end : cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) *dz_end = end;
  for (int l = 0; l < n_layers; ++l) {
    if (!dz[l]) continue;
    const long long n = static_cast<long long>(end - rows) * widths[l];
    bf16* p = dz[l] + static_cast<long long>(rows) * widths[l];
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x)
      p[i] = __float2bfloat16_rn(0.f);
  }
}

// Worker time of local worker i in the last round: the sum of its phase
// windows (globaltimer ns -> s).
__device__ inline double worker_time(const PlanDev& D, int i, int n_phases) {
  double t = 0.0;
  for (int p = 0; p < n_phases; ++p) {
    const unsigned long long s0 = D.timing[2 * (p * D.n_local + i)], e0 = D.timing[2 * (p * D.n_local + i) + 1];
    if (s0 != ~0ull && e0 > s0) t += static_cast<double>(e0 - s0) * 1e-9;
  }
  return t;
}

// Unloaded Gamma time of worker w for b rows: m0 max(b, x_s) + b0.
__device__ inline double gamma0(const lbbsp_gpu_profile& p, double b) {
  const double xs = static_cast<double>(p.saturation_point);
  return dadd(dmul(p.sec_per_sample, b > xs ? b : xs), p.base_time_s);
}

// The observation pushed into worker w's history for a batch of b rows that
// took t seconds.
//  * RATE: the realised rate b / t (the reference's GPU-mode v_actual = x / tp,
//    cluster_sim.cpp:412-413).
//  * CAPACITY: the worker's sustainable speed at the nominal batch
//    x_n = B / n, a * x_n / Gamma0(x_n) with the availability a = Gamma0(b) / t
//    read off its unloaded profile -- the reference's CPU-mode v_actual, the
//    worker's speed under its current resource state whatever batch it ran
//    (effective_speed * speed_mult, cluster_sim.cpp:357-361). On a worker with
//    a fixed latency b / t is not that: a worker handed few rows looks slow,
//    gets fewer rows, and collapses to the floor (measured, DESIGN 2.3).
//  * Gamma solver: the availability Gamma0(b) / t itself.
__device__ inline double observed_speed(const PlanDev& D, int w, int b, double t) {
  if (D.solver == LBBSP_SOLVER_GAMMA || D.observe == LBBSP_OBSERVE_CAPACITY) {
    const lbbsp_gpu_profile p = D.prof0[w];
    const double a = t > 0.0 ? ddiv(gamma0(p, static_cast<double>(b)), t) : 1.0;
    if (D.solver == LBBSP_SOLVER_GAMMA) return a;
    const double xn = ddiv(static_cast<double>(D.B_total), static_cast<double>(D.n_total));
    return dmul(a, ddiv(xn, gamma0(p, xn)));
  }
  return t > 0.0 ? static_cast<double>(b) / t : static_cast<double>(b);
}

// The plan's prediction for worker w in round kk (history length len >= 1):
// SpeedPredictor::predict (predictor.cpp:271-292) on the trace's (c, m) of
// round kk -- the same call plan_body makes.
__device__ inline double predict_for_round(const PlanDev& D, int w, int len, long long kk) {
  const long long ti = kk < D.trace_len - 1 ? kk : D.trace_len - 1;
  const size_t o = static_cast<size_t>(w) * D.trace_len + ti;
  return predictor_predict_d(D.pred, w, len, D.trace_c[o], D.trace_m[o]);
}

// measured per-worker compute time -> observed speed
__global__ void speed_kernel(PlanDev D, int n_phases) {
  const int i = threadIdx.x;
  if (i >= D.n_local) return;
  const double t = worker_time(D, i, n_phases);
  const int w = D.rank * D.n_local + i;
  D.v_obs_local[i] = observed_speed(D, w, D.sizes_all[w], t);
  const int row = *D.rows;
  if (row < D.max_rows) D.rec_t[static_cast<size_t>(row) * D.n_total + w] = t;
}

// Observed speed of local worker i from its phase times.
__device__ inline double local_speed(const PlanDev& D, int i, int n_phases, double* t_out) {
  const double t = worker_time(D, i, n_phases);
  if (t_out) *t_out = t;
  const int w = D.rank * D.n_local + i;
  return observed_speed(D, w, D.sizes_all[w], t);
}

// P10 fused: observe (cluster_sim.cpp:309-313) + train_rotation (:315-324)
// in one launch. CTA j < nb trains model (cursor + j) % n on the history
// extended by this round's observation (it writes that one sample itself --
// the same bits the observe CTA writes); the last CTA computes every speed,
// pushes every history and EMA state, and advances the round counters once
// all training CTAs have read them (a device-side arrival count; all CTAs
// are co-resident, nb < SM count).
__global__ void __launch_bounds__(kTrainThreads) observe_train_kernel(PlanDev D, int fused_speed_phases,
                                                                     unsigned* arrive,
                                                                     size_t smem_bytes, int early) {
  extern __shared__ double sm_d[];
  __shared__ NarxTrainSmem ts;
  const int nb = gridDim.x - 1;
  const int n = D.n_total, tid = threadIdx.x;
  if (static_cast<int>(blockIdx.x) < nb) {
    __shared__ int len_s, w_s;
    __shared__ long long k_s;
    if (tid == 0) {
      len_s = *D.pred.len;
      w_s = (*D.pred.cursor + static_cast<int>(blockIdx.x)) % n;
      k_s = *D.k;
      __threadfence();
      atomicAdd(arrive, 1u);
    }
    __syncthreads();
    const int len = len_s, w = w_s;
    const size_t o = static_cast<size_t>(w) * D.pred.max_hist;
    if (tid == 0 && blockIdx.x == 0) D.stamps[15] = gtimer();  // kernel entry (debug timeline)
    const int L = len + 1 < D.pred.max_hist ? len + 1 : D.pred.max_hist;
    const bool in_smem = narx_train_min_bytes(L) <= smem_bytes;
    // While the workers still run: the history of earlier rounds into the
    // trainer's shared-memory history region, and its part of the three
    // scaler sums (fit_scaler's left fold, continued by the trainer with the
    // newest observation) -- off the critical path of the round.
    __shared__ double pre_sums[3];
    const int old = len < L ? len : L;
    lbbsp_narx_train_cfg cfg = D.pred.train;
    cfg.min_history = D.pred.warmup;
    if (in_smem) {
      double* hv = narx_history_region(sm_d, L);
      for (int i = tid; i < old; i += blockDim.x) {
        hv[i] = D.pred.hv[o + i];
        hv[L + i] = D.pred.hc[o + i];
        hv[2 * L + i] = D.pred.hm[o + i];
      }
      __syncthreads();
      if (tid == 0 || tid == 32 || tid == 64) {
        const double* xs = hv + (tid / 32) * L;
        double sum = 0.0;
        for (int i = 0; i < old; ++i) sum = dadd(sum, xs[i]);
        pre_sums[tid / 32] = sum;
      }
    }
    if (early) tc::pdl_wait();  // the worker kernel's phase times are final
    if (tid == 0 && len < D.pred.max_hist) {
      const double v = fused_speed_phases > 0 ? local_speed(D, w - D.rank * D.n_local, fused_speed_phases, nullptr)
                                              : D.v_obs_all[w];
      const double cn = D.c_now[w], mn = D.m_now[w];
      D.pred.hv[o + len] = v;
      D.pred.hc[o + len] = cn;
      D.pred.hm[o + len] = mn;
      if (in_smem) {  // and straight into the staged copy (index len = L - 1)
        double* hv = narx_history_region(sm_d, L);
        hv[len] = v;
        hv[L + len] = cn;
        hv[2 * L + len] = mn;
      }
    }
    __syncthreads();
    if (tid == 0 && blockIdx.x == 0) D.stamps[14] = gtimer();  // training starts
    const size_t slot = narx_train_scratch_bytes(D.pred.max_hist) / sizeof(double);
    // the shared-memory scratch passed as sm_d itself (not through a
    // shared-or-global select), so the inlined trainer's loads and stores
    // compile to LDS/STS instead of generic accesses
    if (in_smem)
      narx_train_block(&D.pred.models[w], D.pred.hv + o, D.pred.hc + o, D.pred.hm + o, L, cfg,
                       &D.pred.reports[w], nullptr, 0, sm_d, smem_bytes / sizeof(double), &ts, L,
                       pre_sums, old);
    else
      narx_train_block(&D.pred.models[w], D.pred.hv + o, D.pred.hc + o, D.pred.hm + o, L, cfg,
                       &D.pred.reports[w], nullptr, 0, D.pred.scratch + blockIdx.x * slot, slot, &ts);
    // the next round's prediction with the model just trained (after the
    // observe CTA's EMA / history push, which an EMA fallback reads)
    if (tid == 0) {
      unsigned long long seen;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(D.obs_seq) : "memory");
      } while (seen < static_cast<unsigned long long>(k_s + 1));
      D.v_next[w] = predict_for_round(D, w, L, k_s + 1);
      atomicMax(&D.stamps[13], static_cast<unsigned long long>(gtimer()));  // last training done
    }
    return;
  }
  if (early) tc::pdl_wait();
  if (tid == 0) D.stamps[3] = gtimer();
  const long long k_obs = *D.k;
  const int cursor0 = *D.pred.cursor;
  if (fused_speed_phases > 0) {  // single rank: measured speeds computed here
    for (int i = tid; i < D.n_local; i += blockDim.x) {
      double t;
      D.v_obs_local[i] = local_speed(D, i, fused_speed_phases, &t);
      const int rw = *D.rows;
      if (rw < D.max_rows) D.rec_t[static_cast<size_t>(rw) * D.n_total + D.rank * D.n_local + i] = t;
    }
    __syncthreads();
  }
  const int len = *D.pred.len;
  const int row = *D.rows;
  for (int i = tid; i < n; i += blockDim.x) {
    observe_d(D.pred, i, len, D.v_obs_all[i], D.c_now[i], D.m_now[i], 0.0);
    if (row < D.max_rows) D.rec_vobs[static_cast<size_t>(row) * n + i] = D.v_obs_all[i];
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(D.obs_seq),
                 "l"(static_cast<unsigned long long>(k_obs + 1))
                 : "memory");
  }
  // next-round predictions of the models not trained this round
  const int Ln = len + 1 < D.pred.max_hist ? len + 1 : D.pred.max_hist;
  for (int i = tid; i < n; i += blockDim.x) look_ahead(D, i, k_obs + 1, Ln, (i - cursor0 + n) % n >= nb);
  __syncthreads();
  if (tid == 0) {
    while (atomicAdd(arrive, 0u) < static_cast<unsigned>(nb)) {
    }
    *arrive = 0u;
    *D.vnext_k = k_obs + 1;
    *D.pred.len = len + 1 < D.pred.max_hist ? len + 1 : D.pred.max_hist;
    *D.train_first = *D.pred.cursor;
    *D.pred.cursor = (*D.pred.cursor + (n + 1) / 2) % n;
    *D.rows = row + 1;
    *D.k += 1;
    D.stamps[4] = gtimer();
  }
}

// P10: push every worker's (v, c, m) (cluster_sim.cpp:309-313), advance round
__global__ void observe_kernel(PlanDev D, int fused_speed_phases) {
  stamp(D, 3);
  if (fused_speed_phases > 0) {  // single rank: measured speeds computed here
    const int i = threadIdx.x;
    if (i < D.n_local) {
      double t;
      D.v_obs_local[i] = local_speed(D, i, fused_speed_phases, &t);
      const int w = D.rank * D.n_local + i;
      const int rw = *D.rows;
      if (rw < D.max_rows) D.rec_t[static_cast<size_t>(rw) * D.n_total + w] = t;
    }
    __syncthreads();
  }
  const int len = *D.pred.len;
  const int row = *D.rows;
  const long long k_obs = *D.k;
  // next-round predictions (not for NARX: its rotation trains after this kernel)
  const bool ahead = D.pred.kind != LBBSP_PRED_NARX;
  const int Ln = len + 1 < D.pred.max_hist ? len + 1 : D.pred.max_hist;
  for (int i = threadIdx.x; i < D.n_total; i += blockDim.x) {
    observe_d(D.pred, i, len, D.v_obs_all[i], D.c_now[i], D.m_now[i], 0.0);
    if (row < D.max_rows) D.rec_vobs[static_cast<size_t>(row) * D.n_total + i] = D.v_obs_all[i];
    // (EMA / memoryless read only this worker's state, written just above)
    if (ahead) look_ahead(D, i, k_obs + 1, Ln, true);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (ahead) *D.vnext_k = k_obs + 1;
    *D.pred.len = len + 1 < D.pred.max_hist ? len + 1 : D.pred.max_hist;
    *D.train_first = *D.pred.cursor;
    *D.pred.cursor = (*D.pred.cursor + (D.n_total + 1) / 2) % D.n_total;
    *D.rows = row + 1;
    *D.k += 1;
  }
  stamp(D, 4);
}

// ---------------------------------------------------------------------------
// NVLink peer-memory exchange for several workers per GPU on several GPUs
// (C2 at N > 1): the speed all-gather and the gradient all-reduce as our own
// kernels over CUDA-IPC-mapped peer buffers instead of NCCL calls.
//   push:  every rank stores its payload into slot[rank] of every peer's
//          buffer (NVLink stores), fences at system scope, then bumps the
//          per-writer counter in each peer's buffer (system-scope atomics);
//   pull:  a rank waits until every writer's counter reached this round's
//          target, then reads the slots from its own memory -- summing the
//          gradient slots in rank order, so the all-reduce is deterministic.
// Counters only grow (target = (round + 1) * writer CTAs), so nothing resets.
// ---------------------------------------------------------------------------
constexpr int kMaxPeers = 8;
struct PeerDev {
  int world, rank;
  unsigned long long* cnt_local;              // [2][kMaxPeers]: speeds, gradients
  unsigned long long* cnt_peer[kMaxPeers];
  double* spd_local;                          // [world * n_local]
  double* spd_peer[kMaxPeers];
  float* grd_local;                           // [world][P]
  float* grd_peer[kMaxPeers];
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// spin until every writer's counter reached `want`; returns false on timeout
__device__ bool wait_counters(const PeerDev& X, int which, unsigned long long want,
                              lbbsp_dev_status* st) {
  const unsigned long long t0 = gtimer();
  for (int r = 0; r < X.world; ++r) {
    while (ld_acquire_sys(&X.cnt_local[which * kMaxPeers + r]) < want) {
      if (gtimer() - t0 > 2000000000ull) {  // 2 s: a peer is gone -- fail, do not hang
        set_status(st, LBBSP_NCCL, 0, r, static_cast<long long>(want));
        return false;
      }
    }
  }
  return true;
}

// measured speeds of the local workers -> every rank's v_obs_all
__global__ void peer_speed_kernel(PlanDev D, PeerDev X, int n_phases) {
  tc::pdl_wait();  // the phase stamps of the backward GEMMs
  tc::pdl_launch_dependents();
  const int tid = threadIdx.x;
  for (int i = tid; i < D.n_local; i += blockDim.x) {
    double t;
    const double v = local_speed(D, i, n_phases, &t);
    D.v_obs_local[i] = v;
    const int row = *D.rows;
    if (row < D.max_rows) D.rec_t[static_cast<size_t>(row) * D.n_total + D.rank * D.n_local + i] = t;
    for (int r = 0; r < X.world; ++r) X.spd_peer[r][X.rank * D.n_local + i] = v;
  }
  __threadfence_system();
  __syncthreads();
  __shared__ int ok;
  if (tid == 0) {
    for (int r = 0; r < X.world; ++r) atomicAdd_system(&X.cnt_peer[r][0 * kMaxPeers + X.rank], 1ull);
    ok = wait_counters(X, 0, static_cast<unsigned long long>(*D.round_k) + 1, D.status);
  }
  __syncthreads();
  if (!ok) return;
  for (int i = tid; i < D.n_total; i += blockDim.x) D.v_obs_all[i] = __ldcg(&X.spd_local[i]);
}

// sum of the local worker slabs -> slot[rank] of every rank's gradient buffer
__global__ void __launch_bounds__(256) peer_grad_push_kernel(const float* __restrict__ partial, int n,
                                                             long long P, PeerDev X) {
  const long long nv = P / 4;
  for (long long v = blockIdx.x * 256ll + threadIdx.x; v < nv; v += 256ll * gridDim.x) {
    float4 a = reinterpret_cast<const float4*>(partial)[v];
    for (int g = 1; g < n; ++g) {
      const float4 b = reinterpret_cast<const float4*>(partial + static_cast<long long>(g) * P)[v];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    for (int r = 0; r < X.world; ++r)
      reinterpret_cast<float4*>(X.grd_peer[r] + static_cast<long long>(X.rank) * P)[v] = a;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int r = 0; r < X.world; ++r) atomicAdd_system(&X.cnt_peer[r][1 * kMaxPeers + X.rank], 1ull);
}

// wait for every rank's slot, sum in rank order, SGD apply + bf16 copy
__global__ void __launch_bounds__(256) peer_grad_apply_kernel(long long P, float* grad, float* params,
                                                              bf16* pb, float lr, PeerDev X,
                                                              const long long* round_k,
                                                              int push_ctas,
                                                              lbbsp_dev_status* st) {
  __shared__ int ok;
  if (threadIdx.x == 0)
    ok = wait_counters(X, 1, (static_cast<unsigned long long>(*round_k) + 1) * push_ctas, st);
  __syncthreads();
  if (!ok) return;
  const long long nv = P / 4;
  for (long long v = blockIdx.x * 256ll + threadIdx.x; v < nv; v += 256ll * gridDim.x) {
    float4 a = __ldcg(reinterpret_cast<const float4*>(X.grd_local) + v);
    for (int r = 1; r < X.world; ++r) {
      const float4 b = __ldcg(reinterpret_cast<const float4*>(X.grd_local + static_cast<long long>(r) * P) + v);
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    reinterpret_cast<float4*>(grad)[v] = a;
    float4 w = reinterpret_cast<float4*>(params)[v];
    w.x -= lr * a.x;
    w.y -= lr * a.y;
    w.z -= lr * a.z;
    w.w -= lr * a.w;
    reinterpret_cast<float4*>(params)[v] = w;
    __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(pb) + 2 * v;
    o[0] = __floats2bfloat162_rn(w.x, w.y);
    o[1] = __floats2bfloat162_rn(w.z, w.w);
  }
}

// ---------------------------------------------------------------------------
// One worker per GPU (C3, C5): copy-engine bucket exchange. Each layer's bf16
// gradient bucket is pushed into slot[rank] of every peer's buffer by
// cudaMemcpyAsync (the copy engines move it over NVLink without SMs, so the
// transfer overlaps the persistent backward GEMMs); a one-warp kernel then
// bumps the bucket's arrival counter in each peer. The receiver waits on the
// counters with one CTA and the apply kernel sums the slots in rank order
// (fp32, identical on every rank) and updates the weights.
// Counter layout: cnt[(2 + l) * kMaxPeers + writer], target = round + 1.
// ---------------------------------------------------------------------------
__global__ void peer_bucket_signal_kernel(PeerDev X, int l) {
  __threadfence_system();  // the copies before this kernel are complete in stream order
  const int r = threadIdx.x;
  if (r < X.world && r != X.rank) atomicAdd_system(&X.cnt_peer[r][(2 + l) * kMaxPeers + X.rank], 1ull);
}

__global__ void peer_bucket_wait_kernel(PeerDev X, int l, const long long* round_k,
                                        lbbsp_dev_status* st) {
  const unsigned long long want = static_cast<unsigned long long>(*round_k) + 1;
  const unsigned long long t0 = gtimer();
  const int r = threadIdx.x;
  if (r < X.world && r != X.rank) {
    while (ld_acquire_sys(&X.cnt_local[(2 + l) * kMaxPeers + r]) < want) {
      if (gtimer() - t0 > 2000000000ull) {  // 2 s: a peer is gone -- fail, do not hang
        set_status(st, LBBSP_NCCL, 2 + l, r, static_cast<long long>(want));
        break;
      }
    }
  }
}

// params[seg] -= lr * sum_r slot_r[seg] (own slot = the local bucket), + bf16 copy
__global__ void __launch_bounds__(256) peer_bucket_apply_kernel(PeerDev X, long long seg0, long long n,
                                                                long long P, const bf16* __restrict__ own,
                                                                float* params, bf16* pb, float lr) {
  const long long nv = n / 8;
  const bf16* slots = reinterpret_cast<const bf16*>(X.grd_local);
  for (long long v = blockIdx.x * 256ll + threadIdx.x; v < nv; v += 256ll * gridDim.x) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = 0.f;
    for (int r = 0; r < X.world; ++r) {
      const bf16* src = r == X.rank ? own + seg0 : slots + static_cast<long long>(r) * P + seg0;
      const uint4 q = __ldcg(reinterpret_cast<const uint4*>(src) + v);
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(g2[j]);
        a[2 * j] += f.x;
        a[2 * j + 1] += f.y;
      }
    }
    float4* p4 = reinterpret_cast<float4*>(params + seg0) + 2 * v;
    float4 w0 = p4[0], w1 = p4[1];
    w0.x -= lr * a[0]; w0.y -= lr * a[1]; w0.z -= lr * a[2]; w0.w -= lr * a[3];
    w1.x -= lr * a[4]; w1.y -= lr * a[5]; w1.z -= lr * a[6]; w1.w -= lr * a[7];
    p4[0] = w0;
    p4[1] = w1;
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
    o2[0] = __floats2bfloat162_rn(w0.x, w0.y);
    o2[1] = __floats2bfloat162_rn(w0.z, w0.w);
    o2[2] = __floats2bfloat162_rn(w1.x, w1.y);
    o2[3] = __floats2bfloat162_rn(w1.z, w1.w);
    reinterpret_cast<uint4*>(pb + seg0)[v] = o;
  }
}

// Two-shot variant (N > 2): slice j of a bucket goes only to rank j
// (reduce-scatter by copy engine), rank j sums slice j over the ranks in rank
// order in fp32 and rounds the sum to bf16 (as the NCCL bf16 all-reduce
// does), the bf16 slice sums are copied into every rank's all-gather buffer,
// and every rank applies the whole bucket from it: 2(N-1)/N*P*2 bytes per GPU,
// the ring all-reduce's volume, instead of the one-shot (N-1)*P*2. The owner
// applies the same rounded sum, so every rank holds bitwise equal weights.
// Counters: reduce-scatter arrivals at row 2 + l, all-gather arrivals at row
// 2 + LBBSP_MLP_MAX_LAYERS + l.
__global__ void __launch_bounds__(256) peer_slice_reduce_kernel(PeerDev X, long long s0, long long n,
                                                                long long P, const bf16* __restrict__ own,
                                                                bf16* __restrict__ ag) {
  const long long nv = n / 8;
  const bf16* slots = reinterpret_cast<const bf16*>(X.grd_local);
  for (long long v = blockIdx.x * 256ll + threadIdx.x; v < nv; v += 256ll * gridDim.x) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = 0.f;
    for (int r = 0; r < X.world; ++r) {
      const bf16* src = r == X.rank ? own + s0 : slots + static_cast<long long>(r) * P + s0;
      const uint4 q = __ldcg(reinterpret_cast<const uint4*>(src) + v);
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(g2[j]);
        a[2 * j] += f.x;
        a[2 * j + 1] += f.y;
      }
    }
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) o2[j] = __floats2bfloat162_rn(a[2 * j], a[2 * j + 1]);
    reinterpret_cast<uint4*>(ag + s0)[v] = o;
  }
}

__global__ void peer_signal_row_kernel(PeerDev X, int row) {
  __threadfence_system();
  const int r = threadIdx.x;
  if (r < X.world && r != X.rank) atomicAdd_system(&X.cnt_peer[r][row * kMaxPeers + X.rank], 1ull);
}

__global__ void peer_wait_row_kernel(PeerDev X, int row, const long long* round_k, lbbsp_dev_status* st) {
  const unsigned long long want = static_cast<unsigned long long>(*round_k) + 1;
  const unsigned long long t0 = gtimer();
  const int r = threadIdx.x;
  if (r < X.world && r != X.rank) {
    while (ld_acquire_sys(&X.cnt_local[row * kMaxPeers + r]) < want) {
      if (gtimer() - t0 > 2000000000ull) {
        set_status(st, LBBSP_NCCL, row, r, static_cast<long long>(want));
        break;
      }
    }
  }
}

}  // namespace mlp
}  // namespace lbbsp

// ===========================================================================
// host engine
// ===========================================================================
using namespace lbbsp;
using namespace lbbsp::mlp;

struct lbbsp_mlp {
  lbbsp_mlp_cfg cfg{};
  int L = 0;
  std::vector<int> dims;
  int n_local = 1, n_total = 1, B_total = 0, B_cap = 0, N_data = 0, max_rows = 0;
  bool small_head = false;
  long long P = 0;
  std::vector<long long> off_w, off_b;
  std::vector<void*> allocs;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_speed = nullptr, ev_comm = nullptr;
  cudaEvent_t ev_gather0 = nullptr, ev_gather1 = nullptr;
  cudaEvent_t ev_head0 = nullptr, ev_head1 = nullptr;  // head partial combine beside the backward
  cudaStream_t copy_stream = nullptr;  // e2e input staging (lbbsp_mlp_load_data_async)
  cudaEvent_t ev_staged = nullptr;
  cudaStream_t result_stream = nullptr;  // e2e result reads (D2H beside the next round)
  cudaEvent_t ev_round_done = nullptr;
  long long host_rounds = 0;             // rounds enqueued (the next round's record row)
  // the resident dataset is double-buffered: a round reads buffer `cur`
  // while the next round's inputs are copied into the other one; one graph
  // per buffer (the loss branch's tensor map is bound to the buffer)
  bf16* data_xb[2] = {nullptr, nullptr};
  int* data_yb[2] = {nullptr, nullptr};
  int cur = 0;      // buffer the next round reads
  int cap_buf = 0;  // buffer the graph being captured reads
  cudaEvent_t ev_used[2] = {nullptr, nullptr};  // last round that read buffer b
  cudaEvent_t ev_layer[LBBSP_MLP_MAX_LAYERS] = {};
  cudaEvent_t ev_dx[LBBSP_MLP_MAX_LAYERS] = {};  // dX_l done: the bucketed apply of W_l may run
  cudaStream_t comm_stream = nullptr;
  // copy-engine bucket exchange (one worker per GPU with peers, LBBSP_NCCL_BUCKETS unset)
  cudaStream_t xfer_stream = nullptr;
  cudaEvent_t ev_xfer = nullptr;
  cudaGraphExec_t execb[2] = {nullptr, nullptr};
  cudaGraph_t graphb[2] = {nullptr, nullptr};
  GemmPlan fwd_d0_alt;  // the dataset-loss forward of layer 0 over buffer 1
  ncclComm_t comm = nullptr;
  // NVLink peer exchange (lbbsp_mlp_init_peers): replaces the NCCL calls of
  // the several-workers-per-GPU path when set
  bool peers = false;
  bool ce_ok = false;  // copy-engine bucket exchange usable (bf16 buckets, 8-element aligned)
  bool ce_two_shot = false;  // reduce-scatter + all-gather variant (N > 2)
  PeerDev px{};
  void* peer_buf = nullptr;               // local IPC-exported buffer
  void* peer_map[kMaxPeers] = {};          // opened peer buffers
  size_t peer_off_spd = 0, peer_off_grd = 0;
  int launches = 0;
  // device buffers
  bf16 *data_x = nullptr, *X = nullptr, *pb = nullptr, *logits = nullptr, *dlogits = nullptr;
  int *data_y = nullptr, *y = nullptr, *streams = nullptr;
  float *params = nullptr, *grad = nullptr, *partial = nullptr, *row_scale = nullptr;
  std::vector<bf16*> H, dZ;           // H[l]: output of layer l (l < L-1); dZ[l] grad wrt layer-l output
  std::vector<bf16*> Hd;               // full-dataset forward buffers
  bf16* logits_d = nullptr;
  long long* reg_off = nullptr;
  float* head_part = nullptr;      // [sms][head_vals] small-head CTA partials
  double* head_loss = nullptr;     // [sms]
  unsigned* head_cnt = nullptr;    // [n_local] worker head counters (self-resetting)
  unsigned* head_cnt_d = nullptr;  // [1] dataset-loss head counter
  unsigned* arrive = nullptr;      // observe_train_kernel arrival count (self-resetting)
  float* bias_part = nullptr;      // bias-gradient row-chunk partials (bias_grad_kernel)
  bf16* gradb = nullptr;           // [P] bf16 gradient buckets (bucketed all-reduce path)
  unsigned* bias_cnt = nullptr;    // [n_local][strips] bias_grad_kernel counters (self-resetting)
  unsigned long long* dbg_stamps = nullptr;  // lbbsp_mlp_debug_stamp
  bool use_pdl = true;             // programmatic dependent launch on the worker-phase chain
  long long* reg_len = nullptr;
  int n_reg = 0;
  PlanDev D{};
  lbbsp_predictor pred;
  std::vector<GemmPlan> fwd, dx, dw, fwd_d;
  int n_phases = 0;
  double gemm_flops = 0.0, reduce_bytes = 0.0;
  double* result = nullptr;
  int* dz_end = nullptr;  // [1] local rows rounded up to 64 (one-worker k-split)
  bool use_pair = false;  // one worker per GPU: CTA-pair GEMMs
  bf16** dz_ptrs = nullptr;
  int* dz_widths = nullptr;
  Interference intf{};  // straggler injection state (interference mode)
  // fused worker kernel (784-256-10): forward + head + dW0 in one launch
  bool fused = false;
  bool fused_pair = false;  // the (2,1,1)-cluster variant (c2_fused_pair.cuh)
  bool fused_quad = false;  // the (4,1,1)-cluster variant (c2_fused_quad.cuh)
  CUtensorMap fz_tm[7];
  CUtensorMap fz_gm[2];   // dataset buffer b, box {64, 1}: the pair kernel's in-kernel row gather
  bool fz_gather = false;
  unsigned* fz_comb = nullptr;
  unsigned long long* fz_dbg = nullptr;  // LBBSP_FZ_DEBUG: per-CTA stage stamps
  // e2e plumbing: cached host-buffer lookups (lbbsp_mlp_read_result_async,
  // lbbsp_mlp_step_e2e)
  int* res_host_sizes = nullptr;
  double* res_host_loss = nullptr;
  int* res_dev_sizes = nullptr;
  double* res_dev_loss = nullptr;
  const void* warm_x = nullptr;
  const int* warm_y = nullptr;

  ~lbbsp_mlp() {
    for (void* p : peer_map)
      if (p && p != peer_buf) cudaIpcCloseMemHandle(p);
    if (peer_buf) cudaFree(peer_buf);
    for (int b = 0; b < 2; ++b) {
      if (execb[b]) cudaGraphExecDestroy(execb[b]);
      if (graphb[b]) cudaGraphDestroy(graphb[b]);
      if (ev_used[b]) cudaEventDestroy(ev_used[b]);
    }
    if (comm && nccl_api()) nccl_api()->CommDestroy(comm);
    if (stream) cudaStreamDestroy(stream);
    if (side) cudaStreamDestroy(side);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_gather0) cudaEventDestroy(ev_gather0);
    if (ev_staged) cudaEventDestroy(ev_staged);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (result_stream) cudaStreamDestroy(result_stream);
    if (ev_round_done) cudaEventDestroy(ev_round_done);
    if (ev_gather1) cudaEventDestroy(ev_gather1);
    if (ev_head0) cudaEventDestroy(ev_head0);
    if (ev_head1) cudaEventDestroy(ev_head1);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_speed) cudaEventDestroy(ev_speed);
    if (ev_comm) cudaEventDestroy(ev_comm);
    if (ev_xfer) cudaEventDestroy(ev_xfer);
    if (xfer_stream) cudaStreamDestroy(xfer_stream);
    for (auto& e : ev_layer)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_dx)
      if (e) cudaEventDestroy(e);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    for (void* p : allocs) cudaFree(p);
  }
  template <typename T>
  cudaError_t alloc(T** p, size_t count) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1));
    if (e == cudaSuccess) {
      allocs.push_back(*p);
      e = cudaMemset(*p, 0, sizeof(T) * (count ? count : 1));
    }
    return e;
  }
  template <typename T>
  cudaError_t upload(T** dst, const T* src, size_t count) {
    cudaError_t e = alloc(dst, count);
    if (e == cudaSuccess && count) e = cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyHostToDevice);
    return e;
  }

  Groups groups() const {
    Groups G;
    G.n = n_local;
    G.r0 = D.r0;
    G.r1 = D.r1;
    G.cta0 = D.cta0;
    G.ctan = D.ctan;
    G.intf = intf;
    return G;
  }
  unsigned long long* phase_slot(int p) { return D.timing + 2ll * p * n_local; }

  int enqueue_iteration(cudaStream_t s);
};

namespace {

// grouped GEMM launch helper
int launch_grouped(lbbsp_mlp* m, GemmPlan& p, int mode, unsigned long long* timing, cudaStream_t s) {
  p.args.mode = mode;
  if (p.pair && mode == tc::kKSplit) {
    // k-split over [0, rows) rounded up to the 64-row block (rows past the
    // worker's end are zero in dZ, see zero_dz_tail_kernel)
    p.args.g_r1 = m->dz_end;
  }
  p.args.n_groups = m->n_local;
  p.args.g_r0 = m->D.r0;
  if (!(p.pair && mode == tc::kKSplit)) p.args.g_r1 = m->D.r1;
  p.args.g_cta0 = m->D.cta0;
  p.args.g_ctan = m->D.ctan;
  p.args.timing = timing;
  p.args.intf = m->intf;
  p.ctas = m->D.sm_budget;
  p.pdl = m->use_pdl;
  return gemm_launch(p, s);
}

}  // namespace

int lbbsp_mlp::enqueue_iteration(cudaStream_t s) {
  const bf16* data_x = data_xb[cap_buf];
  const int* data_y = data_yb[cap_buf];
  const Groups G = groups();
  int nl = 0, ph = 0;
  const int sms = D.sm_budget;
  const size_t plan_smem = D.solver == LBBSP_SOLVER_GAMMA ? gamma_plan_smem(n_total) : 0;
  const int gather_ctas = std::max(sms, std::min(sms * 8, (B_cap * (dims[0] / 8) + 1023) / 1024));
  // the pair kernel reads the batch rows from the dataset itself (tile::gather4)
  const bool kgather = fused && fused_pair && fz_gather;
  // single rank: the plan waits for the gather on the device (no graph join);
  // set before either kernel is captured, both read it
  // Kernels serialised by a tool (ncu replay, compute-sanitizer) cannot run the
  // gather beside a spinning plan: join with a graph edge there instead.
  const bool join = getenv("LBBSP_GATHER_JOIN") || getenv("CUDA_INJECTION64_PATH");
  D.gather_ctas = cfg.world == 1 && !join && !kgather ? gather_ctas : 0;
  if (kgather) {
    plan_kernel<<<1, 256, plan_smem, s>>>(D, row_scale);
  } else if (cfg.world == 1 && !join) {  // plan + gather of all B rows in one launch
    GatherArgs ga{streams, B_total, data_x, data_y, dims[0], X, y, partial, P, reg_off, reg_len, n_reg};
    plan_gather_kernel<<<1 + gather_ctas, 256, plan_smem, s>>>(D, row_scale, ga);
  } else if (cfg.world == 1) {  // one rank gathers all B rows: independent of the plan
    LBBSP_CUDA_CHECK(cudaEventRecord(ev_gather0, s));
    LBBSP_CUDA_CHECK(cudaStreamWaitEvent(side, ev_gather0, 0));
    gather_kernel<<<gather_ctas, 256, 0, side>>>(D, streams, B_total, data_x, data_y, dims[0], X, y,
                                                 B_total, partial, P, reg_off, reg_len, n_reg);
    LBBSP_CUDA_CHECK(cudaEventRecord(ev_gather1, side));
    if (join) LBBSP_CUDA_CHECK(cudaStreamWaitEvent(s, ev_gather1, 0));
    plan_kernel<<<1, 256, plan_smem, s>>>(D, row_scale);
  } else {
    plan_kernel<<<1, 256, plan_smem, s>>>(D, row_scale);
    LBBSP_CUDA_CHECK(launch_maybe_pdl(gather_kernel, gather_ctas, 256, 0, s, use_pdl, D,
                                      static_cast<const int*>(streams), B_total,
                                      static_cast<const bf16*>(data_x),
                                      static_cast<const int*>(data_y), dims[0], X, y, 0, partial, P,
                                      static_cast<const long long*>(reg_off),
                                      static_cast<const long long*>(reg_len), n_reg));
  }
  nl += kgather || (cfg.world == 1 && !join) ? 1 : 2;
  if (use_pair) {
    zero_dz_tail_kernel<<<8, 256, 0, s>>>(D, dz_ptrs, dz_widths, L, dz_end, B_cap);
    ++nl;
  }
  const bool bucketed = cfg.world > 1 && n_local == 1 && !small_head;
  const bool ce_buckets = bucketed && peers && gradb && ce_ok;
  // ---- forward (per-worker partitions) ----
  const int Lg = small_head ? L - 1 : L;  // layers on the tensor-core GEMM
  const int hl = L - 1;  // last layer index
  if (fused) {
    // forward + head + dW0 of every worker in one launch (c2_fused.cuh)
    FusedArgs fa{};
    fa.G = G;
    fa.dZ0 = dZ[0];
    fa.W1 = params + off_w[1];
    fa.b0 = params + off_b[0];
    fa.b1 = params + off_b[1];
    fa.y = y;
    fa.row_scale = row_scale;
    fa.slab = partial;
    fa.slab_stride = P;
    fa.off_w0 = off_w[0];
    fa.off_w1 = off_w[1];
    fa.off_b1 = off_b[1];
    fa.off_b0 = off_b[0];
    fa.head_part = head_part;
    fa.done = D.fz_done;
    fa.timing = phase_slot(ph++);
    fa.status = D.status;
    fa.dbg = fz_dbg;
    if (kgather) {
      fa.gather = 1;
      fa.streams = streams;
      fa.kptr = D.k;
      fa.stream_off = D.stream_off;
      fa.data_y = data_y;
      fa.B_total = B_total;
      fa.max_rows = D.max_rows;
    }
    if (fused_quad)
      LBBSP_CUDA_CHECK(launch_maybe_pdl(c2_quad_worker_kernel, sms & ~3, kFqThreads, kFqSmem, s, use_pdl,
                                        fz_tm[0], fz_tm[6], fz_tm[2], fz_tm[3], fz_tm[5], fa));
    else if (fused_pair)
      LBBSP_CUDA_CHECK(launch_maybe_pdl(c2_pair_worker_kernel, sms & ~1, kFpThreads, kFpSmem, s, use_pdl,
                                        kgather ? fz_gm[cap_buf] : fz_tm[0], fz_tm[4], fz_tm[2],
                                        kgather ? fz_gm[cap_buf] : fz_tm[3], fz_tm[5], fa));
    else
      LBBSP_CUDA_CHECK(launch_maybe_pdl(c2_fused_worker_kernel, sms, kFzThreads, kFzSmem, s, use_pdl, fz_tm[0],
                                        fz_tm[1], fz_tm[2], fz_tm[3], fa));
    ++nl;
  } else {
  for (int l = 0; l < Lg; ++l) {
    int rc = launch_grouped(this, fwd[l], tc::kRows, phase_slot(ph++), s);
    if (rc) return rc;
    ++nl;
  }
  // ---- head ----
  if (small_head) {
    const bf16* Hin = L >= 2 ? H[L - 2] : X;
    LBBSP_CUDA_CHECK(launch_maybe_pdl(
        head_mma_kernel<true>, sms, 256, kHeadMmaSmem, s, use_pdl, G, 0, Hin,
        static_cast<const float*>(params + off_w[hl]), static_cast<const float*>(params + off_b[hl]),
        static_cast<const int*>(y), static_cast<const float*>(row_scale), dZ[L - 2], partial, P,
        off_w[hl], off_b[hl], off_b[L - 2], static_cast<double*>(nullptr), head_part, head_loss,
        head_cnt, phase_slot(ph++), static_cast<double*>(nullptr), static_cast<const long long*>(nullptr), 0));
    ++nl;
    // the CTA partials are summed beside the backward GEMMs; joined before the
    // gradient slabs are consumed
    LBBSP_CUDA_CHECK(cudaEventRecord(ev_head0, s));
    LBBSP_CUDA_CHECK(cudaStreamWaitEvent(side, ev_head0, 0));
    head_combine_kernel<<<n_local * kCombineSlices, 256, 0, side>>>(
        G, head_part, partial, P, off_w[hl], off_b[hl], off_b[L - 2]);
    LBBSP_CUDA_CHECK(cudaEventRecord(ev_head1, side));
  } else {
    LBBSP_CUDA_CHECK(launch_softmax_ce(sms, s, use_pdl, G, 0, logits, dims[L], y, row_scale,
                                       dZ[L - 1], nullptr, phase_slot(ph++)));
  }
  ++nl;
  // ---- backward ----
  // One worker per GPU on several GPUs: each layer's gradient segment
  // (W_l | b_l, contiguous in the flat layout) is all-reduced in place on the
  // comm stream as soon as its dW/db are final, overlapping the rest of the
  // backward pass (bucketed allreduce); the speed all-gather follows on the
  // same stream, so the communicator sees one fixed order on every rank.
  for (int l = Lg - 1; l >= 0; --l) {
    if (!(small_head && l == L - 2)) {  // the small head already summed this bias gradient
      unsigned long long* slot = phase_slot(ph++);
      bf16* ob = gradb ? gradb + off_b[l] : nullptr;
      if (getenv("LBBSP_BIAS_SLOT1"))  // A/B: one CTA per partition slot
        bias_grad_kernel<1><<<sms, 256, kBiasSmem, s>>>(G, dZ[l], dims[l + 1], partial, P, off_b[l], bias_part,
                                                        bias_cnt, ob, slot);
      else
        bias_grad_kernel<kBiasCtasPerSlot><<<sms * kBiasCtasPerSlot, 256, kBiasSmem, s>>>(
            G, dZ[l], dims[l + 1], partial, P, off_b[l], bias_part, bias_cnt, ob, slot);
      ++nl;
    }
    int rc = launch_grouped(this, dw[l], tc::kKSplit, phase_slot(ph++), s);
    if (rc) return rc;
    ++nl;
    const long long seg0 = off_w[l], seg1 = l + 1 < L ? off_w[l + 1] : P;
    const long long W = cfg.world;
    auto sl0 = [&](long long r) { return seg0 + ((seg1 - seg0) / 8 * r / W) * 8; };
    bf16* ag_local = peers ? reinterpret_cast<bf16*>(px.grd_local) + W * P : nullptr;
    if (bucketed) {
      // the exchange of this layer's bucket starts as soon as its dW/db are final
      LBBSP_CUDA_CHECK(cudaEventRecord(ev_layer[l], s));
      LBBSP_CUDA_CHECK(cudaStreamWaitEvent(comm_stream, ev_layer[l], 0));
      if (ce_buckets && ce_two_shot) {
        // reduce-scatter: slice r of this bucket -> slot[rank] of rank r
        LBBSP_CUDA_CHECK(cudaStreamWaitEvent(xfer_stream, ev_layer[l], 0));
        // (one stream for all peers: a copy stream per peer measured slower at N=4)
        for (int r = 0; r < cfg.world; ++r) {
          if (r == cfg.rank) continue;
          bf16* dst = reinterpret_cast<bf16*>(px.grd_peer[r]) + static_cast<long long>(cfg.rank) * P + sl0(r);
          LBBSP_CUDA_CHECK(cudaMemcpyAsync(dst, gradb + sl0(r), sizeof(bf16) * (sl0(r + 1) - sl0(r)),
                                           cudaMemcpyDeviceToDevice, xfer_stream));
        }
        peer_signal_row_kernel<<<1, 32, 0, xfer_stream>>>(px, 2 + l);
        // own slice: rank-ordered fp32 sum -> all-gather buffer of every rank
        const long long m0 = sl0(cfg.rank), m1 = sl0(cfg.rank + 1);
        peer_wait_row_kernel<<<1, 32, 0, comm_stream>>>(px, 2 + l, D.round_k, D.status);
        peer_slice_reduce_kernel<<<sms, 256, 0, comm_stream>>>(px, m0, m1 - m0, P, gradb, ag_local);
        for (int r = 0; r < cfg.world; ++r) {
          if (r == cfg.rank) continue;
          bf16* ag_r = reinterpret_cast<bf16*>(px.grd_peer[r]) + W * P;
          LBBSP_CUDA_CHECK(cudaMemcpyAsync(ag_r + m0, ag_local + m0, sizeof(bf16) * (m1 - m0),
                                           cudaMemcpyDeviceToDevice, comm_stream));
        }
        peer_signal_row_kernel<<<1, 32, 0, comm_stream>>>(px, 2 + LBBSP_MLP_MAX_LAYERS + l);
        peer_wait_row_kernel<<<1, 32, 0, comm_stream>>>(px, 2 + LBBSP_MLP_MAX_LAYERS + l, D.round_k,
                                                        D.status);
        nl += 4;
      } else if (ce_buckets) {
        // push this bucket into slot[rank] of every peer (copy engines), then
        // raise the peers' arrival counters; wait for the peers' buckets on
        // the comm stream
        LBBSP_CUDA_CHECK(cudaStreamWaitEvent(xfer_stream, ev_layer[l], 0));
        const size_t bytes = sizeof(bf16) * static_cast<size_t>(seg1 - seg0);
        for (int r = 0; r < cfg.world; ++r) {
          if (r == cfg.rank) continue;
          bf16* dst = reinterpret_cast<bf16*>(px.grd_peer[r]) + static_cast<long long>(cfg.rank) * P + seg0;
          LBBSP_CUDA_CHECK(cudaMemcpyAsync(dst, gradb + seg0, bytes, cudaMemcpyDeviceToDevice, xfer_stream));
        }
        peer_bucket_signal_kernel<<<1, 32, 0, xfer_stream>>>(px, l);
        peer_bucket_wait_kernel<<<1, 32, 0, comm_stream>>>(px, l, D.round_k, D.status);
        nl += 2;
      } else if (gradb) {
        if (nccl_api()->AllReduce(gradb + seg0, gradb + seg0, static_cast<size_t>(seg1 - seg0),
                                  ncclBfloat16, ncclSum, comm, comm_stream) != ncclSuccess)
          return set_error(LBBSP_NCCL, "ncclAllReduce (bucket %d) failed", l);
      } else {
        if (nccl_api()->AllReduce(partial + seg0, partial + seg0, static_cast<size_t>(seg1 - seg0),
                                  ncclFloat, ncclSum, comm, comm_stream) != ncclSuccess)
          return set_error(LBBSP_NCCL, "ncclAllReduce (bucket %d) failed", l);
      }
    }
    if (l > 0) {
      rc = launch_grouped(this, dx[l], tc::kRows, phase_slot(ph++), s);
      if (rc) return rc;
      ++nl;
    }
    if (bucketed) {
      // dX_l reads the bf16 W_l (its B operand): the update of segment l must
      // not overwrite it before that GEMM is done, so the apply waits for it
      // (SGD semantics: every update after the full backward pass)
      if (l > 0) {
        LBBSP_CUDA_CHECK(cudaEventRecord(ev_dx[l], s));
        LBBSP_CUDA_CHECK(cudaStreamWaitEvent(comm_stream, ev_dx[l], 0));
      }
      const float lrf = static_cast<float>(cfg.learning_rate);
      if (ce_buckets && ce_two_shot)
        apply_bf16_kernel<<<sms * 2, 256, 0, comm_stream>>>(ag_local + seg0, seg1 - seg0, params + seg0,
                                                            pb + seg0, lrf);
      else if (ce_buckets)
        peer_bucket_apply_kernel<<<sms * 2, 256, 0, comm_stream>>>(px, seg0, seg1 - seg0, P, gradb, params,
                                                                   pb, lrf);
      else if (gradb)
        apply_bf16_kernel<<<sms * 2, 256, 0, comm_stream>>>(gradb + seg0, seg1 - seg0, params + seg0,
                                                            pb + seg0, lrf);
      else
        reduce_apply_kernel<<<sms * 2, 256, 0, comm_stream>>>(partial + seg0, 1, seg1 - seg0, grad + seg0,
                                                              params + seg0, pb + seg0, lrf, 1, nullptr);
      ++nl;
    }
  }
  }  // !fused
  n_phases = ph;
  // measured speeds; on several GPUs all-gathered (after the gradient buckets)
  const float lr = static_cast<float>(cfg.learning_rate);
  if (cfg.world > 1 && peers && !bucketed) {
    // speeds, all-gathered over NVLink
    LBBSP_CUDA_CHECK(launch_maybe_pdl(peer_speed_kernel, 1, 256, 0, s, use_pdl, D, px, n_phases));
    ++nl;
  } else if (cfg.world > 1 && ce_buckets) {
    // one worker per GPU, copy-engine buckets: the speed all-gather runs over
    // peer memory on the comm stream after the last bucket's apply; its wait
    // for every rank doubles as the round's barrier (no rank refills a peer's
    // bucket slots before that peer has applied them). No NCCL on this path.
    LBBSP_CUDA_CHECK(cudaEventRecord(ev_speed, s));
    LBBSP_CUDA_CHECK(cudaStreamWaitEvent(comm_stream, ev_speed, 0));
    peer_speed_kernel<<<1, 256, 0, comm_stream>>>(D, px, n_phases);
    ++nl;
    LBBSP_CUDA_CHECK(cudaEventRecord(ev_comm, comm_stream));
    LBBSP_CUDA_CHECK(cudaStreamWaitEvent(s, ev_comm, 0));
    // the local buckets must not be overwritten before they left
    LBBSP_CUDA_CHECK(cudaEventRecord(ev_xfer, xfer_stream));
    LBBSP_CUDA_CHECK(cudaStreamWaitEvent(s, ev_xfer, 0));
  } else if (cfg.world > 1) {
    speed_kernel<<<1, 32 * ((n_local + 31) / 32), 0, s>>>(D, n_phases);
    ++nl;
    if (bucketed) {
      LBBSP_CUDA_CHECK(cudaEventRecord(ev_speed, s));
      LBBSP_CUDA_CHECK(cudaStreamWaitEvent(comm_stream, ev_speed, 0));
      if (nccl_api()->AllGather(D.v_obs_local, D.v_obs_all, static_cast<size_t>(n_local), ncclDouble,
                                comm, comm_stream) != ncclSuccess)
        return set_error(LBBSP_NCCL, "ncclAllGather failed");
      LBBSP_CUDA_CHECK(cudaEventRecord(ev_comm, comm_stream));
      LBBSP_CUDA_CHECK(cudaStreamWaitEvent(s, ev_comm, 0));
      if (ce_buckets) {  // the local buckets must not be overwritten before they left
        LBBSP_CUDA_CHECK(cudaEventRecord(ev_xfer, xfer_stream));
        LBBSP_CUDA_CHECK(cudaStreamWaitEvent(s, ev_xfer, 0));
      }
    } else {
      // speeds first: the observe / NARX branch (the usual critical tail)
      // forks right after this small all-gather; the gradient all-reduce
      // follows on the loss branch
      if (nccl_api()->AllGather(D.v_obs_local, D.v_obs_all, static_cast<size_t>(n_local), ncclDouble,
                                comm, s) != ncclSuccess)
        return set_error(LBBSP_NCCL, "ncclAllGather failed");
    }
  }
  // Fork -- the loss branch (apply, full-dataset forward) runs beside the
  // observe branch (history push, NARX training); both join before the next
  // round's plan. step_sync computes the loss (cluster_sim.cpp:445) and trains
  // (:464) independently of each other.
  const bool fork = !getenv("LBBSP_NO_FORK");
  const int nb = (n_total + 1) / 2;
  const bool narx_fused = pred.dev.kind == LBBSP_PRED_NARX && nb + 1 <= num_sms();
  // One rank, fused worker kernel, NARX: the observe / NARX kernel follows the
  // worker kernel on the main stream as a programmatic launch. Its CTAs become
  // resident on the SMs the worker partitions leave free while the workers
  // still run and wait for the workers' results at griddepcontrol.wait (the
  // launch latency leaves the critical path); the loss branch moves to the
  // side stream. (A dry training run there to warm the trainer's code did not
  // shorten the real one: the trainer is fp64-latency bound, ~1.9 us per
  // evaluation at L = 110, scripts/narx_probe.py.)
  const bool early_obs = fork && narx_fused && fused && cfg.world == 1 && use_pdl && !getenv("LBBSP_NO_EARLY_OBSERVE");
  cudaStream_t so = s, sl = s;
  if (fork) {
    LBBSP_CUDA_CHECK(cudaEventRecord(ev_fork, s));
    LBBSP_CUDA_CHECK(cudaStreamWaitEvent(side, ev_fork, 0));
    if (early_obs)
      sl = side;
    else
      so = side;
  }
  // ---- observe branch ----
  if (narx_fused) {
    // at least 116 KB of shared memory: two of these CTAs never share an SM
    // (launched early, beside the worker kernel, they would otherwise pack
    // onto the few SMs the workers leave free and halve each other's fp64
    // and issue rate; the training-set build measured 3 us in place against
    // 1.5 us alone, scripts/fp64/build_lat.cu)
    const size_t tsm = std::max(train_smem_bytes(pred.dev.max_hist), static_cast<size_t>(116 * 1024));
    if (early_obs)
      LBBSP_CUDA_CHECK(launch_maybe_pdl(observe_train_kernel, nb + 1, kTrainThreads, tsm, so, true, D, n_phases,
                                        arrive, tsm, 1));
    else
      observe_train_kernel<<<nb + 1, kTrainThreads, tsm, so>>>(D, cfg.world > 1 ? 0 : n_phases, arrive, tsm, 0);
    ++nl;
  } else {
    observe_kernel<<<1, 256, 0, so>>>(D, cfg.world > 1 ? 0 : n_phases);
    ++nl;
    if (pred.dev.kind == LBBSP_PRED_NARX) {
      LBBSP_CUDA_CHECK(launch_pred_train_from(pred.dev, D.train_first, so));
      ++nl;
    }
  }
  // ---- aggregate + apply (the bucketed path applied per layer above) ----
  // the small head's CTA partials were combined on the side stream
  if (small_head && !fused) LBBSP_CUDA_CHECK(cudaStreamWaitEvent(s, ev_head1, 0));
  if (bucketed) {
  } else if (cfg.world > 1 && peers) {
    // one-shot all-reduce over NVLink peer memory, summed in rank order
    peer_grad_push_kernel<<<sms, 256, 0, s>>>(partial, n_local, P, px);
    peer_grad_apply_kernel<<<sms, 256, 0, s>>>(P, grad, params, pb, lr, px, D.round_k, sms, D.status);
    nl += 2;
  } else if (cfg.world > 1) {
    reduce_apply_kernel<<<sms * 4, 256, 0, s>>>(partial, n_local, P, grad, params, pb, lr, 0, D.stamps);
    ++nl;
    if (nccl_api()->AllReduce(grad, grad, static_cast<size_t>(P), ncclFloat, ncclSum, comm, s) !=
        ncclSuccess)
      return set_error(LBBSP_NCCL, "ncclAllReduce failed");
    reduce_apply_kernel<<<sms * 4, 256, 0, s>>>(grad, 1, P, grad, params, pb, lr, 1, D.stamps);
  } else {
    // not a programmatic launch: early-resident apply CTAs would hold the SMs
    // the (higher-priority) NARX branch needs when the backward ends
    // sized to the parameter count (two float4 per thread, at most 4 CTAs
    // per SM): C2's 0.2 M parameters need ~100 CTAs, and every CTA more
    // shares an SM with the NARX trainings running beside this branch
    const int ra_ctas = static_cast<int>(std::min<long long>(sms * 4ll, std::max(1ll, (P / 4 + 511) / 512)));
    reduce_apply_kernel<<<ra_ctas, 256, 0, sl>>>(partial, n_local, P, grad, params, pb, lr, 1, D.stamps);
  }
  if (!bucketed) ++nl;
  // ---- full-dataset loss (step_sync P9, cluster_sim.cpp:445) ----
  if (D.loss_on) {
    for (int l = 0; l < Lg; ++l) {
      GemmPlan& fp = (l == 0 && cap_buf == 1) ? fwd_d0_alt : fwd_d[l];
      fp.ctas = std::min(fp.ctas, sms) & ~1;
      fp.pdl = use_pdl;
      int rc = gemm_launch(fp, cfg.world == 1 ? sl : s);
      if (rc) return rc;
      ++nl;
    }
    Groups none{};
    none.n = 0;
    if (small_head) {
      const bf16* Hin = L >= 2 ? Hd[L - 2] : data_x;
      LBBSP_CUDA_CHECK(launch_maybe_pdl(
          head_mma_kernel<false>, sms, 256, kHeadMmaSmem, cfg.world == 1 ? sl : s, use_pdl, none, N_data, Hin,
          static_cast<const float*>(params + off_w[hl]), static_cast<const float*>(params + off_b[hl]),
          static_cast<const int*>(data_y), static_cast<const float*>(nullptr),
          static_cast<bf16*>(nullptr), static_cast<float*>(nullptr), 0ll, 0ll, 0ll, 0ll, D.loss_acc,
          head_part, head_loss, head_cnt_d, D.stamps + 6, D.rec_loss, static_cast<const long long*>(D.round_k),
          D.max_rows));
    } else {
      LBBSP_CUDA_CHECK(launch_softmax_ce(sms, cfg.world == 1 ? sl : s, use_pdl, none, N_data, logits_d, dims[L], data_y,
                                         nullptr, nullptr, D.loss_acc, nullptr));
    }
    ++nl;
  }
  if (fork) {
    LBBSP_CUDA_CHECK(cudaEventRecord(ev_join, side));
    LBBSP_CUDA_CHECK(cudaStreamWaitEvent(s, ev_join, 0));
  }
  LBBSP_CUDA_CHECK(cudaGetLastError());
  launches = nl;
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_create(const lbbsp_mlp_cfg* cfg, lbbsp_mlp** out) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return set_error(LBBSP_CUDA, "lbbsp: no CUDA device (the B200 path has no CPU fallback)");
  }
  const lbbsp_mlp_cfg& c = *cfg;
  if (c.n_layers < 1 || c.n_layers > LBBSP_MLP_MAX_LAYERS)
    return set_error(LBBSP_INVALID_ARGUMENT, "mlp: n_layers must be in [1, %d]", LBBSP_MLP_MAX_LAYERS);
  if (c.n_workers_local < 1 || c.world < 1 || c.n_workers_total != c.n_workers_local * c.world)
    return set_error(LBBSP_INVALID_ARGUMENT, "mlp: n_workers_total must equal n_workers_local * world");
  if (c.n_workers_total > LBBSP_MAX_WORKERS)
    return set_error(LBBSP_INVALID_ARGUMENT, "mlp: at most %d workers", LBBSP_MAX_WORKERS);
  if (c.global_batch < c.n_workers_total)
    return set_error(LBBSP_INVALID_ARGUMENT, "simulation: total_budget below worker count");
  if (c.scheme != LBBSP_SCHEME_LBBSP && c.global_batch % c.n_workers_total != 0)
    return set_error(LBBSP_INVALID_ARGUMENT,
                     "simulation: bsp/asp/ssp need total_budget divisible by workers");
  if (c.trace_len < 1 || !c.h_trace_c || !c.h_trace_m || !c.h_trace_mult)
    return set_error(LBBSP_INVALID_ARGUMENT, "mlp: a straggler trace is required");
  const int L = c.n_layers;
  const bool small_head = c.dims[L] <= 16;
  if (small_head && (c.dims[L] != 10 || L < 2 || c.dims[L - 1] != 256))
    return set_error(LBBSP_INVALID_ARGUMENT, "mlp: small heads support the 256->10 classifier");
  for (int l = 0; l <= L; ++l)
    if (c.dims[l] % 8 != 0 && !(small_head && l == L))
      return set_error(LBBSP_INVALID_ARGUMENT, "mlp: layer widths must be multiples of 8");
  if (!small_head && c.dims[L] % 256 != 0)
    return set_error(LBBSP_INVALID_ARGUMENT, "mlp: softmax head width must be a multiple of 256");

  auto M = std::make_unique<lbbsp_mlp>();
  lbbsp_mlp& m = *M;
  m.cfg = c;
  m.L = L;
  m.dims.assign(c.dims, c.dims + L + 1);
  m.n_local = c.n_workers_local;
  m.n_total = c.n_workers_total;
  m.B_total = c.global_batch;
  m.B_cap = c.global_batch;  // a rank can be handed (almost) the whole batch
  m.N_data = c.dataset_size;
  m.small_head = small_head;
  m.use_pdl = !getenv("LBBSP_NO_PDL");
  m.max_rows = c.max_iterations > 0 ? c.max_iterations : 1;
  LBBSP_CUDA_CHECK(cudaStreamCreateWithFlags(&m.stream, cudaStreamNonBlocking));
  {
    int lo = 0, hi = 0;  // the observe / NARX branch is the round's usual critical tail
    LBBSP_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    LBBSP_CUDA_CHECK(cudaStreamCreateWithPriority(&m.side, cudaStreamNonBlocking, hi));
  }
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_fork, cudaEventDisableTiming));
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_gather0, cudaEventDisableTiming));
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_gather1, cudaEventDisableTiming));
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_head0, cudaEventDisableTiming));
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_head1, cudaEventDisableTiming));
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_join, cudaEventDisableTiming));
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_speed, cudaEventDisableTiming));
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_comm, cudaEventDisableTiming));
  for (auto& e : m.ev_layer) LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : m.ev_dx) LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  LBBSP_CUDA_CHECK(cudaStreamCreateWithFlags(&m.comm_stream, cudaStreamNonBlocking));
  LBBSP_CUDA_CHECK(cudaStreamCreateWithFlags(&m.xfer_stream, cudaStreamNonBlocking));
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_xfer, cudaEventDisableTiming));

  // flat parameter layout, 64-element aligned segments
  auto pad = [](long long x) { return (x + 63) / 64 * 64; };
  long long P = 0;
  for (int l = 0; l < L; ++l) {
    m.off_w.push_back(P);
    P += pad(static_cast<long long>(c.dims[l + 1]) * c.dims[l]);
    m.off_b.push_back(P);
    P += pad(c.dims[l + 1]);
  }
  m.P = P;
  const int d0 = c.dims[0];
  LBBSP_CUDA_CHECK(m.alloc(&m.params, P));
  LBBSP_CUDA_CHECK(m.alloc(&m.pb, P));
  LBBSP_CUDA_CHECK(m.alloc(&m.grad, P));
  if (m.n_local > 1 || c.world > 1)
    LBBSP_CUDA_CHECK(m.alloc(&m.partial, static_cast<size_t>(P) * m.n_local));
  else
    m.partial = m.grad;  // one worker: the dW GEMM writes the gradient directly
  // one worker per GPU on several GPUs: the gradient buckets travel in bf16
  // (half the all-reduce bytes; SURVEY 8(d) sizes the C3 all-reduce in bf16)
  if (c.world > 1 && m.n_local == 1 && !small_head && !getenv("LBBSP_FP32_BUCKETS"))
    LBBSP_CUDA_CHECK(m.alloc(&m.gradb, static_cast<size_t>(P)));
  if (small_head) {
    const int nsm = num_sms();
    LBBSP_CUDA_CHECK(m.alloc(&m.head_part, static_cast<size_t>(nsm) * kHeadPartVals));
    LBBSP_CUDA_CHECK(m.alloc(&m.head_loss, static_cast<size_t>(nsm)));
    LBBSP_CUDA_CHECK(m.alloc(&m.head_cnt, static_cast<size_t>(m.n_local)));
    LBBSP_CUDA_CHECK(m.alloc(&m.head_cnt_d, 1));
    LBBSP_CUDA_CHECK(cudaFuncSetAttribute(head_mma_kernel<true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kHeadMmaSmem));
    LBBSP_CUDA_CHECK(cudaFuncSetAttribute(head_mma_kernel<false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kHeadMmaSmem));
  }
  LBBSP_CUDA_CHECK(m.alloc(&m.data_x, static_cast<size_t>(m.N_data) * d0));
  LBBSP_CUDA_CHECK(m.alloc(&m.data_y, m.N_data));
  m.data_xb[0] = m.data_x;
  m.data_yb[0] = m.data_y;
  LBBSP_CUDA_CHECK(m.alloc(&m.data_xb[1], static_cast<size_t>(m.N_data) * d0));
  LBBSP_CUDA_CHECK(m.alloc(&m.data_yb[1], m.N_data));
  LBBSP_CUDA_CHECK(m.alloc(&m.X, static_cast<size_t>(m.B_cap) * d0));
  LBBSP_CUDA_CHECK(m.alloc(&m.y, m.B_cap));
  LBBSP_CUDA_CHECK(m.alloc(&m.row_scale, m.B_cap));
  m.H.assign(L, nullptr);
  m.dZ.assign(L, nullptr);
  m.Hd.assign(L, nullptr);
  for (int l = 0; l < L; ++l) {
    if (l < L - 1) {
      LBBSP_CUDA_CHECK(m.alloc(&m.H[l], static_cast<size_t>(m.B_cap) * c.dims[l + 1]));
      LBBSP_CUDA_CHECK(m.alloc(&m.Hd[l], static_cast<size_t>(m.N_data) * c.dims[l + 1]));
    }
    if (!(small_head && l == L - 1))
      LBBSP_CUDA_CHECK(m.alloc(&m.dZ[l], static_cast<size_t>(m.B_cap) * c.dims[l + 1]));
  }
  if (!small_head) {
    LBBSP_CUDA_CHECK(m.alloc(&m.logits, static_cast<size_t>(m.B_cap) * c.dims[L]));
    LBBSP_CUDA_CHECK(m.alloc(&m.logits_d, static_cast<size_t>(m.N_data) * c.dims[L]));
  }
  // atomic-accumulated partial regions: all biases (+ the small head's W)
  std::vector<long long> ro, rl;
  for (int l = 0; l < L; ++l) {
    ro.push_back(m.off_b[l]);
    rl.push_back(c.dims[l + 1]);
  }
  if (small_head) {
    ro.push_back(m.off_w[L - 1]);
    rl.push_back(static_cast<long long>(c.dims[L]) * c.dims[L - 1]);
  }
  m.n_reg = static_cast<int>(ro.size());
  LBBSP_CUDA_CHECK(m.upload(&m.reg_off, ro.data(), ro.size()));
  LBBSP_CUDA_CHECK(m.upload(&m.reg_len, rl.data(), rl.size()));

  // dataset + parameters (setup-time device generators)
  init_x_kernel<<<512, 256>>>(m.data_x, static_cast<long long>(m.N_data) * d0, c.dataset_seed);
  teacher_labels_kernel<<<m.N_data, 256, c.dims[L] > 32 ? sizeof(float) * d0 : 0>>>(
      m.data_x, m.data_y, d0, c.dims[L], c.dataset_seed);
  for (int l = 0; l < L; ++l)
    init_params_kernel<<<512, 256>>>(m.params, m.pb, m.off_w[l], m.off_b[l], c.dims[l + 1], c.dims[l],
                                     c.seed ^ (0x9a4c0ull + l));
  LBBSP_CUDA_CHECK(cudaGetLastError());

  // sample streams for every round (cluster_sim.cpp:302-307)
  const size_t R = static_cast<size_t>(m.max_rows);
  LBBSP_CUDA_CHECK(m.alloc(&m.streams, R * m.B_total));
  LBBSP_CUDA_CHECK(launch_sample_streams(c.seed, 0, static_cast<int>(R), m.B_total, m.N_data, m.streams,
                                         nullptr));

  // plan state
  PlanDev& D = m.D;
  const int n = m.n_total;
  D.n_total = n;
  D.n_local = m.n_local;
  D.rank = c.rank;
  D.B_total = m.B_total;
  D.scheme = c.scheme;
  D.static_sizes = c.static_sizes;
  int sms = num_sms();
  D.sm_budget = c.sm_budget > 0 && c.sm_budget < sms ? c.sm_budget : sms;
  D.trace_len = c.trace_len;
  const size_t TL = static_cast<size_t>(n) * c.trace_len;
  double *tc_ = nullptr, *tm_ = nullptr, *tx_ = nullptr, *sh = nullptr;
  LBBSP_CUDA_CHECK(m.upload(&tc_, c.h_trace_c, TL));
  LBBSP_CUDA_CHECK(m.upload(&tm_, c.h_trace_m, TL));
  LBBSP_CUDA_CHECK(m.upload(&tx_, c.h_trace_mult, TL));
  D.trace_c = tc_;
  D.trace_m = tm_;
  D.trace_mult = tx_;
  std::vector<double> share(n, 1.0 / m.n_local);
  if (c.h_worker_share) share.assign(c.h_worker_share, c.h_worker_share + n);
  LBBSP_CUDA_CHECK(m.upload(&sh, share.data(), share.size()));
  D.share = sh;
  if (c.static_sizes) {
    int* ss = nullptr;
    LBBSP_CUDA_CHECK(m.upload(&ss, c.h_static_sizes, n));
    D.static_sizes_d = ss;
  }
  LBBSP_CUDA_CHECK(m.alloc(&D.k, 1));
  LBBSP_CUDA_CHECK(m.alloc(&D.rows, 1));
  D.max_rows = m.max_rows;
  LBBSP_CUDA_CHECK(m.alloc(&D.sizes_all, n));
  LBBSP_CUDA_CHECK(m.alloc(&D.r0, m.n_local));
  LBBSP_CUDA_CHECK(m.alloc(&D.r1, m.n_local));
  LBBSP_CUDA_CHECK(m.alloc(&D.cta0, m.n_local));
  LBBSP_CUDA_CHECK(m.alloc(&D.ctan, m.n_local));
  LBBSP_CUDA_CHECK(m.alloc(&D.local_rows, 1));
  LBBSP_CUDA_CHECK(m.alloc(&D.stream_off, 1));
  LBBSP_CUDA_CHECK(m.alloc(&D.c_now, n));
  LBBSP_CUDA_CHECK(m.alloc(&D.m_now, n));
  LBBSP_CUDA_CHECK(m.alloc(&D.v_pred, n));
  LBBSP_CUDA_CHECK(m.alloc(&D.timing, 2ull * kMaxPhases * m.n_local));
  LBBSP_CUDA_CHECK(m.alloc(&D.v_obs_local, m.n_local));
  if (c.world > 1)
    LBBSP_CUDA_CHECK(m.alloc(&D.v_obs_all, n));
  else
    D.v_obs_all = D.v_obs_local;
  LBBSP_CUDA_CHECK(m.alloc(&D.loss_acc, 1));
  LBBSP_CUDA_CHECK(m.alloc(&D.stamps, 16));
  LBBSP_CUDA_CHECK(m.alloc(&D.round_k, 1));
  LBBSP_CUDA_CHECK(m.alloc(&D.v_next, n));
  LBBSP_CUDA_CHECK(m.alloc(&D.nx_c, n));
  LBBSP_CUDA_CHECK(m.alloc(&D.nx_m, n));
  LBBSP_CUDA_CHECK(m.alloc(&D.nx_a, n));
  LBBSP_CUDA_CHECK(m.alloc(&D.nx_intf, m.n_local));
  LBBSP_CUDA_CHECK(m.alloc(&D.vnext_k, 1));
  LBBSP_CUDA_CHECK(cudaMemset(D.vnext_k, 0xff, sizeof(long long)));  // -1
  LBBSP_CUDA_CHECK(m.alloc(&D.obs_seq, 1));
  if (c.straggler_mode != LBBSP_STRAGGLE_INTERFERE && c.straggler_mode != LBBSP_STRAGGLE_SM_CAP)
    return set_error(LBBSP_INVALID_ARGUMENT, "mlp: unknown straggler_mode %d", c.straggler_mode);
  D.straggler_mode = c.straggler_mode;
  if (c.solver != LBBSP_SOLVER_PROPORTIONAL && c.solver != LBBSP_SOLVER_GAMMA)
    return set_error(LBBSP_INVALID_ARGUMENT, "mlp: unknown solver %d", c.solver);
  D.solver = c.solver;
  if (c.observe != LBBSP_OBSERVE_RATE && c.observe != LBBSP_OBSERVE_CAPACITY)
    return set_error(LBBSP_INVALID_ARGUMENT, "mlp: unknown observe %d", c.observe);
  D.observe = c.observe;
  D.plan_fast = n <= 32 && c.solver == LBBSP_SOLVER_PROPORTIONAL && !getenv("LBBSP_PLAN_GENERAL");
  if (c.solver == LBBSP_SOLVER_GAMMA || c.observe == LBBSP_OBSERVE_CAPACITY) {
    if (!c.h_gpu_profiles)
      return set_error(LBBSP_INVALID_ARGUMENT,
                       "mlp: the gamma solver and the capacity observation need h_gpu_profiles (unloaded Gamma per worker)");
    lbbsp_gpu_profile* pr = nullptr;
    LBBSP_CUDA_CHECK(m.upload(&pr, c.h_gpu_profiles, static_cast<size_t>(n)));
    D.prof0 = pr;
  }
  if (c.solver == LBBSP_SOLVER_GAMMA) {
    LBBSP_CUDA_CHECK(cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(gamma_plan_smem(n))));
    LBBSP_CUDA_CHECK(cudaFuncSetAttribute(plan_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(gamma_plan_smem(n))));
  }
  if (c.straggler_mode == LBBSP_STRAGGLE_INTERFERE) {
    float2* w = nullptr;
    LBBSP_CUDA_CHECK(m.alloc(&w, m.n_local));
    D.intf_w = w;
    m.intf.w = w;
    // HBM-bound interference source: larger than the 126 MB L2
    const long long nvec = 192ll * 1024 * 1024 / 16;
    uint4* buf = nullptr;
    LBBSP_CUDA_CHECK(m.alloc(&buf, static_cast<size_t>(nvec)));
    m.intf.buf = buf;
    m.intf.nvec = nvec;
  }
  // end-to-end plumbing (lbbsp_mlp_load_data_async / read_result_async)
  LBBSP_CUDA_CHECK(cudaStreamCreateWithFlags(&m.copy_stream, cudaStreamNonBlocking));
  LBBSP_CUDA_CHECK(cudaStreamCreateWithFlags(&m.result_stream, cudaStreamNonBlocking));
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_round_done, cudaEventDisableTiming));
  LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&m.ev_staged, cudaEventDisableTiming));
  for (auto& e : m.ev_used) LBBSP_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  LBBSP_CUDA_CHECK(m.alloc(&m.result, static_cast<size_t>(m.n_total) + 2));
  LBBSP_CUDA_CHECK(m.alloc(&m.arrive, 1));
  {
    unsigned long long* gd = nullptr;
    LBBSP_CUDA_CHECK(m.alloc(&gd, 1));
    m.D.gather_done = gd;
  }
  {
    int max_w = 8;
    for (int l = 1; l <= L; ++l) max_w = std::max(max_w, c.dims[l]);
    const size_t part = std::max(static_cast<size_t>(num_sms()) * kBiasCols,
                                 static_cast<size_t>(num_sms()) * kBiasCtasPerSlot * kBiasStrip +
                                     static_cast<size_t>(m.n_local) * max_w);
    LBBSP_CUDA_CHECK(m.alloc(&m.bias_part, part));
    LBBSP_CUDA_CHECK(m.alloc(&m.bias_cnt, static_cast<size_t>(m.n_local) * bias_strips(max_w)));
  }
  LBBSP_CUDA_CHECK(cudaFuncSetAttribute(bias_grad_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBiasSmem));
  LBBSP_CUDA_CHECK(cudaFuncSetAttribute(bias_grad_kernel<kBiasCtasPerSlot>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, kBiasSmem));
  LBBSP_CUDA_CHECK(cudaFuncSetAttribute(observe_train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        200 * 1024));
  D.N_data = m.N_data;
  D.loss_on = c.loss_every > 0 ? 1 : 0;
  LBBSP_CUDA_CHECK(m.alloc(&D.train_first, 1));
  LBBSP_CUDA_CHECK(m.alloc(&D.rec_sizes, R * n));
  LBBSP_CUDA_CHECK(m.alloc(&D.rec_vpred, R * n));
  LBBSP_CUDA_CHECK(m.alloc(&D.rec_vobs, R * n));
  LBBSP_CUDA_CHECK(m.alloc(&D.rec_caps, R * n));
  LBBSP_CUDA_CHECK(m.alloc(&D.rec_t, R * n));
  LBBSP_CUDA_CHECK(m.alloc(&D.rec_loss, R));
  LBBSP_CUDA_CHECK(m.alloc(&D.status, 1));

  // predictor bank over all workers (replicated on every rank)
  {
    std::vector<uint64_t> seeds(n);
    for (int i = 0; i < n; ++i) seeds[i] = mix_seed(c.seed, 0x9ced1c70ull, static_cast<uint64_t>(i));
    lbbsp_predictor* tmp = nullptr;
    lbbsp_predictor_cfg pc = c.predictor;
    pc.train.min_history = pc.warmup_iterations;
    int rc = lbbsp_predictor_create(&pc, n, m.max_rows, seeds.data(), nullptr, &tmp);
    if (rc) return rc;
    // adopt the bank's allocations
    m.pred.dev = tmp->dev;
    m.pred.allocs.swap(tmp->allocs);
    delete tmp;
    D.pred = m.pred.dev;
  }

  // GEMM plans (tensor maps on the fixed buffers). One worker per GPU with
  // wide layers runs the CTA-pair kernel (256-row UMMA tiles).
  const int Lg = small_head ? L - 1 : L;
  m.use_pair = m.n_local == 1 && !small_head && !getenv("LBBSP_NO_PAIR");
  for (int l = 0; l <= L && m.use_pair; ++l)
    if (c.dims[l] < 256) m.use_pair = false;
  if (m.use_pair) {
    LBBSP_CUDA_CHECK(m.alloc(&m.dz_end, 1));
    std::vector<bf16*> zp(L, nullptr);
    std::vector<int> zw(L, 0);
    for (int l = 0; l < L; ++l) {
      zp[l] = m.dZ[l];
      zw[l] = c.dims[l + 1];
    }
    LBBSP_CUDA_CHECK(m.upload(&m.dz_ptrs, zp.data(), zp.size()));
    LBBSP_CUDA_CHECK(m.upload(&m.dz_widths, zw.data(), zw.size()));
  }
  m.fwd.resize(Lg);
  m.dx.resize(Lg);
  m.dw.resize(Lg);
  m.fwd_d.resize(Lg);
  double flops = 0.0;
  for (int l = 0; l < Lg; ++l) {
    const int din = c.dims[l], dout = c.dims[l + 1];
    const bf16* Ain = l == 0 ? m.X : m.H[l - 1];
    const bf16* Ain_d = l == 0 ? m.data_x : m.Hd[l - 1];
    const bool last = (l == L - 1);
    // wide tiles (BN=256) unless a worker's share of tiles would leave most of
    // its CTA partition idle (the emulated-worker C2 shapes)
    const double rows_per_worker = static_cast<double>(m.B_total) / c.world / m.n_local;
    const int ctas_per_worker = std::max(1, D.sm_budget / m.n_local);
    // widest N tile that still gives a worker's CTAs enough tiles; the row
    // (forward) GEMMs run on trace-capped partitions, typically about half
    // the nominal share, so they need fewer tiles per nominal CTA (measured
    // on C2, scripts/c2_bn_sweep.py)
    auto pick_bn = [&](double mrows, int ncols, double fill = 0.75) {
      for (int bn : {256, 128}) {
        if (ncols < bn) continue;
        const double tiles = std::ceil(mrows / 128.0) * std::ceil(ncols / static_cast<double>(bn));
        if (tiles >= fill * ctas_per_worker) return bn;
      }
      return 64;
    };
    auto env_bn = [](const char* name, int dflt) {  // tuning override (experiments)
      const char* v = getenv(name);
      const int b = v ? atoi(v) : 0;
      return (b == 64 || b == 128 || b == 256) ? b : dflt;
    };
    const int bn = env_bn("LBBSP_BN_FWD", pick_bn(rows_per_worker, dout, 0.4));
    const int epi = last ? tc::kEpiBiasBf16 : tc::kEpiBiasReluBf16;
    const bool pr = m.use_pair;
    int rc = gemm_plan(&m.fwd[l], Ain, m.pb + m.off_w[l], m.B_cap, dout, din, false, false,
                       pr ? 256 : bn, epi, pr);
    if (rc) return rc;
    m.fwd[l].args.c_bf16 = last ? m.logits : m.H[l];
    m.fwd[l].args.ldc = dout;
    m.fwd[l].args.bias = m.params + m.off_b[l];
    // the dataset forward (loss branch) uses the whole GPU: narrow tiles
    // when its row count alone would leave most SMs idle
    const int bn_d = env_bn("LBBSP_BN_LOSS",
                            std::ceil(m.N_data / 128.0) * std::ceil(dout / 128.0) < sms / 2 ? 64 : bn);
    rc = gemm_plan(&m.fwd_d[l], Ain_d, m.pb + m.off_w[l], m.N_data, dout, din, false, false,
                   pr ? 256 : bn_d, epi, pr);
    if (rc) return rc;
    m.fwd_d[l].args.c_bf16 = last ? m.logits_d : m.Hd[l];
    m.fwd_d[l].args.ldc = dout;
    m.fwd_d[l].args.bias = m.params + m.off_b[l];
    if (l == 0) {  // the same plan over the second dataset buffer
      rc = gemm_plan(&m.fwd_d0_alt, m.data_xb[1], m.pb + m.off_w[l], m.N_data, dout, din, false, false,
                     pr ? 256 : bn_d, epi, pr);
      if (rc) return rc;
      m.fwd_d0_alt.args = m.fwd_d[l].args;
    }
    // dW_l = dZ_l^T A_l : M=dout, N=din, K=rows ; A = dZ_l [rows][dout] MN-major, B = A_l [rows][din] MN-major
    const int bn_w = env_bn("LBBSP_BN_DW", pick_bn(static_cast<double>(dout), din));
    const int bn_x = env_bn("LBBSP_BN_DX", pick_bn(rows_per_worker, din));
    rc = gemm_plan(&m.dw[l], m.dZ[l], Ain, dout, din, m.B_cap, true, true, pr ? 256 : bn_w,
                   m.gradb ? tc::kEpiBf16 : tc::kEpiF32, pr);
    if (rc) return rc;
    m.dw[l].args.c_f32 = m.partial + m.off_w[l];
    if (m.gradb) m.dw[l].args.c_bf16 = m.gradb + m.off_w[l];
    m.dw[l].args.ldc = din;
    m.dw[l].args.group_stride = P;
    if (l > 0) {
      // dZ_{l-1} = (dZ_l W_l) * (H_{l-1} > 0): A = dZ_l [rows][dout] K-major, B = W_l [dout][din] = [K][N] MN-major
      rc = gemm_plan(&m.dx[l], m.dZ[l], m.pb + m.off_w[l], m.B_cap, din, dout, false, true,
                     pr ? 256 : bn_x, tc::kEpiDReluBf16, pr);
      if (rc) return rc;
      m.dx[l].args.c_bf16 = m.dZ[l - 1];
      m.dx[l].args.ldc = din;
      m.dx[l].args.aux = m.H[l - 1];
      m.dx[l].args.ld_aux = din;
    }
    flops += 2.0 * m.B_total / c.world * din * dout * (l > 0 ? 3.0 : 2.0);
  }
  if (small_head) flops += 2.0 * m.B_total / c.world * c.dims[L - 1] * c.dims[L] * 3.0;
  m.gemm_flops = flops;
  // one persistent launch for every worker's forward + head + dW0 on the
  // 784-256-10 MLP (c2_fused.cuh); LBBSP_NO_FUSE=1 keeps the three launches
  m.fused = small_head && L == 2 && c.dims[0] == kFzD0 && c.dims[1] == kHeadDH && !getenv("LBBSP_NO_FUSE");
  if (m.fused) {
    int rc = make_tmap_bf16(&m.fz_tm[0], m.X, kFzD0, m.B_cap, kFzD0, 128);
    if (!rc) rc = make_tmap_bf16(&m.fz_tm[1], m.pb + m.off_w[0], kFzD0, kHeadDH, kFzD0, 256);
    if (!rc) rc = make_tmap_bf16(&m.fz_tm[2], m.dZ[0], kHeadDH, m.B_cap, kHeadDH, 64);
    if (!rc) rc = make_tmap_bf16(&m.fz_tm[3], m.X, kFzD0, m.B_cap, kFzD0, 64);
    if (!rc) rc = make_tmap_bf16(&m.fz_tm[4], m.pb + m.off_w[0], kFzD0, kHeadDH, kFzD0, 128);
    if (!rc)
      rc = make_tmap_f32_3d(&m.fz_tm[5], m.partial + m.off_w[0], kFzD0, kHeadDH, m.n_local, kFzD0, m.P, 128);
    if (rc) return rc;
    // the column-split pair kernel by default (LBBSP_FUSE_SINGLE=1: one CTA per
    // tile). SM-cap mode keeps the single-CTA kernel: its caps follow
    // floor(budget * share * availability) exactly, odd counts included, and
    // the pair kernel needs cluster-aligned (even) partitions
    m.fused_pair = !getenv("LBBSP_FUSE_SINGLE") && c.straggler_mode != LBBSP_STRAGGLE_SM_CAP;
    // in-kernel row gather from the resident dataset, opt-in (LBBSP_KGATHER=1):
    // bitwise the same round, but 32 tile::gather4 requests per 16 KB stage
    // run the worker phase at 50 us against 21 us from the gathered batch
    // (profiles/r02_kgather.txt) -- the TMA unit's request rate, not bytes
    // the quad kernel (four CTAs per tile), opt-in (LBBSP_FUSE_QUAD=1): a
    // CTA's tile takes as long as in the pair kernel (forward 4.5 vs 5.1 us,
    // the head's latency chains unchanged) and a worker's tile wave shrinks
    // from 1152 to 512 rows, so LB-BSP's larger batches need two waves
    // (profiles/r02_quad.txt)
    m.fused_quad = m.fused_pair && getenv("LBBSP_FUSE_QUAD") && !getenv("LBBSP_KGATHER");
    if (m.fused_quad) m.fused_pair = false;
    if (m.fused_quad) rc = make_tmap_bf16(&m.fz_tm[6], m.pb + m.off_w[0], kFzD0, kHeadDH, kFzD0, 64);
    if (rc) return rc;
    m.fz_gather = m.fused_pair && getenv("LBBSP_KGATHER");
    for (int b = 0; b < 2 && m.fz_gather && !rc; ++b)
      rc = make_tmap_bf16(&m.fz_gm[b], m.data_xb[b], kFzD0, m.N_data, kFzD0, 1);
    if (rc) return rc;
    D.cap_align = m.fused_quad ? 4 : m.fused_pair ? 2 : 1;
    unsigned* fd = nullptr;
    LBBSP_CUDA_CHECK(m.alloc(&fd, static_cast<size_t>(m.n_local)));
    D.fz_done = fd;
    LBBSP_CUDA_CHECK(m.alloc(&m.fz_comb, static_cast<size_t>(m.n_local)));
    if (getenv("LBBSP_FZ_DEBUG")) LBBSP_CUDA_CHECK(m.alloc(&m.fz_dbg, static_cast<size_t>(num_sms()) * 16));
    LBBSP_CUDA_CHECK(cudaFuncSetAttribute(c2_fused_worker_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(kFzSmem)));
    LBBSP_CUDA_CHECK(cudaFuncSetAttribute(c2_pair_worker_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(kFpSmem)));
    LBBSP_CUDA_CHECK(cudaFuncSetAttribute(c2_quad_worker_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(kFqSmem)));
  }
  m.reduce_bytes = (m.n_local + 1.0) * P * 4.0 + P * 4.0 + P * 2.0;
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  *out = M.release();
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_destroy(lbbsp_mlp* m) {
  delete m;
  return LBBSP_OK;
}

extern "C" int lbbsp_nccl_unique_id(unsigned char h_id[128]) {
  const NcclApi* api = nccl_api();
  if (!api) return set_error(LBBSP_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != ncclSuccess) return set_error(LBBSP_NCCL, "ncclGetUniqueId failed");
  std::memcpy(h_id, id.internal, 128);
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_init_comm(lbbsp_mlp* m, const unsigned char h_id[128]) {
  if (m->cfg.world <= 1) return LBBSP_OK;
  const NcclApi* api = nccl_api();
  if (!api) return set_error(LBBSP_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  std::memcpy(id.internal, h_id, 128);
  ncclResult_t r = api->CommInitRank(&m->comm, m->cfg.world, id, m->cfg.rank);
  if (r != ncclSuccess) return set_error(LBBSP_NCCL, "ncclCommInitRank: %s", api->GetErrorString(r));
  return LBBSP_OK;
}

// NVLink peer exchange setup: every rank exports one device buffer (CUDA IPC
// handle, 64 bytes); after the handles are all-gathered on the host, every
// rank maps its peers' buffers. Must precede the first lbbsp_mlp_run.
extern "C" int lbbsp_mlp_peer_handle(lbbsp_mlp* m, unsigned char h_handle[64]) {
  if (m->cfg.world > kMaxPeers)
    return set_error(LBBSP_INVALID_ARGUMENT, "mlp: peer exchange supports at most %d GPUs", kMaxPeers);
  if (!m->peer_buf) {
    const int W = m->cfg.world;
    // counters: [2 + LBBSP_MLP_MAX_LAYERS][kMaxPeers] (speeds, gradients, per-bucket arrivals)
    m->peer_off_spd = (sizeof(unsigned long long) * kMaxPeers * (2 + 2 * LBBSP_MLP_MAX_LAYERS) + 255) / 256 * 256;
    m->peer_off_grd = (m->peer_off_spd + sizeof(double) * W * m->n_local + 255) / 256 * 256;
    // gradient region: fp32 slots [W][P] (several workers per GPU), or bf16
    // slots [W][P] + the bf16 all-gather buffer [P] (copy-engine buckets)
    const size_t bytes = m->peer_off_grd + std::max(sizeof(float) * W, sizeof(bf16) * (W + 1)) *
                                               static_cast<size_t>(m->P);
    LBBSP_CUDA_CHECK(cudaMalloc(&m->peer_buf, bytes));
    LBBSP_CUDA_CHECK(cudaMemset(m->peer_buf, 0, bytes));
  }
  cudaIpcMemHandle_t h;
  LBBSP_CUDA_CHECK(cudaIpcGetMemHandle(&h, m->peer_buf));
  std::memcpy(h_handle, &h, 64);
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_init_peers(lbbsp_mlp* m, const unsigned char* h_handles) {
  const int W = m->cfg.world, R = m->cfg.rank;
  if (!m->peer_buf) return set_error(LBBSP_LOGIC, "mlp: lbbsp_mlp_peer_handle first");
  if (m->execb[0] || m->execb[1])
    return set_error(LBBSP_LOGIC, "mlp: peers must be set up before the first round");
  PeerDev& X = m->px;
  X.world = W;
  X.rank = R;
  for (int r = 0; r < W; ++r) {
    if (r == R) {
      m->peer_map[r] = m->peer_buf;
    } else {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, h_handles + 64 * r, 64);
      LBBSP_CUDA_CHECK(cudaIpcOpenMemHandle(&m->peer_map[r], h, cudaIpcMemLazyEnablePeerAccess));
    }
    char* b = static_cast<char*>(m->peer_map[r]);
    X.cnt_peer[r] = reinterpret_cast<unsigned long long*>(b);
    X.spd_peer[r] = reinterpret_cast<double*>(b + m->peer_off_spd);
    X.grd_peer[r] = reinterpret_cast<float*>(b + m->peer_off_grd);
  }
  char* lb = static_cast<char*>(m->peer_buf);
  X.cnt_local = reinterpret_cast<unsigned long long*>(lb);
  X.spd_local = reinterpret_cast<double*>(lb + m->peer_off_spd);
  X.grd_local = reinterpret_cast<float*>(lb + m->peer_off_grd);
  m->peers = true;
  // copy-engine bucket exchange: each bucket (W_l | b_l) moves as whole uint4s.
  // Default at 2 GPUs (one-shot push, C3 no-straggler round 1.31 -> 1.19 ms).
  // At N=4 the one-shot push ((N-1)*P*2 bytes per GPU) measured 1.74 ms and
  // the two-shot variant (ring volume) 1.46 ms against NCCL's 1.42 ms, so
  // N > 2 keeps the NCCL buckets unless LBBSP_CE_BUCKETS=1 (one-shot) or
  // LBBSP_CE_TWO_SHOT=1.
  bool al = m->gradb != nullptr && m->P % 8 == 0 && !getenv("LBBSP_NCCL_BUCKETS") &&
            (W == 2 || getenv("LBBSP_CE_TWO_SHOT") || getenv("LBBSP_CE_BUCKETS"));
  // one-shot push (each GPU sends (N-1)*P*2 bytes, one hop to the apply), or
  // reduce-scatter + all-gather (2(N-1)/N*P*2 bytes per GPU)
  m->ce_two_shot = getenv("LBBSP_CE_TWO_SHOT") != nullptr;
  for (int l = 0; al && l < m->L; ++l) {
    const long long seg0 = m->off_w[l], seg1 = l + 1 < m->L ? m->off_w[l + 1] : m->P;
    al = seg0 % 8 == 0 && (seg1 - seg0) % 8 == 0;
  }
  m->ce_ok = al;
  return LBBSP_OK;
}

extern "C" void* lbbsp_mlp_stream(lbbsp_mlp* m) { return m->stream; }
extern "C" void* lbbsp_mlp_result_stream(lbbsp_mlp* m) { return m->result_stream; }

extern "C" int lbbsp_mlp_run(lbbsp_mlp* m, int iterations) {
  // several GPUs: the peer-memory exchange needs no communicator (several
  // workers per GPU, or one worker per GPU with copy-engine buckets); every
  // other exchange runs on NCCL
  const bool peer_only = m->peers && (m->n_local > 1 || m->ce_ok);
  if (m->cfg.world > 1 && !m->comm && !peer_only)
    return set_error(LBBSP_NCCL, "mlp: world > 1 needs lbbsp_mlp_init_comm (or peers) first");
  for (int i = 0; i < iterations; ++i) {
    const int b = m->cur;
    if (!m->execb[b]) {
      m->cap_buf = b;
      LBBSP_CUDA_CHECK(cudaStreamBeginCapture(m->stream, cudaStreamCaptureModeThreadLocal));
      int rc = m->enqueue_iteration(m->stream);
      cudaError_t e2 = cudaStreamEndCapture(m->stream, &m->graphb[b]);
      if (rc) return rc;
      LBBSP_CUDA_CHECK(e2);
      // honour the side (observe / NARX) stream's higher priority inside the graph
      LBBSP_CUDA_CHECK(cudaGraphInstantiate(&m->execb[b], m->graphb[b], cudaGraphInstantiateFlagUseNodePriority));
    }
    LBBSP_CUDA_CHECK(cudaGraphLaunch(m->execb[b], m->stream));
    LBBSP_CUDA_CHECK(cudaEventRecord(m->ev_used[b], m->stream));
    ++m->host_rounds;
  }
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_records(lbbsp_mlp* m, int max_rows, int* rows, int* sizes, double* v_pred,
                                 double* v_obs, int* caps, double* t_worker, double* loss) {
  LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->stream));
  int r = 0;
  LBBSP_CUDA_CHECK(cudaMemcpy(&r, m->D.rows, sizeof(int), cudaMemcpyDeviceToHost));
  r = std::min(std::min(r, max_rows), m->max_rows);
  *rows = r;
  const size_t n = m->n_total;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    return (dst && bytes) ? cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) : cudaSuccess;
  };
  LBBSP_CUDA_CHECK(cp(sizes, m->D.rec_sizes, sizeof(int) * r * n));
  LBBSP_CUDA_CHECK(cp(v_pred, m->D.rec_vpred, sizeof(double) * r * n));
  LBBSP_CUDA_CHECK(cp(v_obs, m->D.rec_vobs, sizeof(double) * r * n));
  LBBSP_CUDA_CHECK(cp(caps, m->D.rec_caps, sizeof(int) * r * n));
  LBBSP_CUDA_CHECK(cp(t_worker, m->D.rec_t, sizeof(double) * r * n));
  LBBSP_CUDA_CHECK(cp(loss, m->D.rec_loss, sizeof(double) * r));
  if (loss && r > 0) {  // the newest round's loss is still in the accumulator
    double acc = 0.0;
    LBBSP_CUDA_CHECK(cudaMemcpy(&acc, m->D.loss_acc, sizeof(double), cudaMemcpyDeviceToHost));
    loss[r - 1] = m->D.loss_on ? acc / static_cast<double>(m->N_data) : -1.0;
  }
  lbbsp_dev_status st{};
  LBBSP_CUDA_CHECK(cudaMemcpy(&st, m->D.status, sizeof st, cudaMemcpyDeviceToHost));
  if (st.code) return lbbsp_check_status(&st);
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_params(lbbsp_mlp* m, float* h_params, long long* h_offsets,
                                long long* n_params) {
  LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->stream));
  if (n_params) *n_params = m->P;
  if (h_offsets)
    for (int l = 0; l < m->L; ++l) {
      h_offsets[2 * l] = m->off_w[l];
      h_offsets[2 * l + 1] = m->off_b[l];
    }
  if (h_params) LBBSP_CUDA_CHECK(cudaMemcpy(h_params, m->params, sizeof(float) * m->P, cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

namespace {
__global__ void to_bf16_kernel(const float* p, __nv_bfloat16* pb, long long n) {
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) pb[i] = __float2bfloat16_rn(p[i]);
}
}  // namespace

extern "C" int lbbsp_mlp_set_params(lbbsp_mlp* m, const float* h_params) {
  LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->stream));
  LBBSP_CUDA_CHECK(cudaMemcpy(m->params, h_params, sizeof(float) * m->P, cudaMemcpyHostToDevice));
  to_bf16_kernel<<<256, 256, 0, m->stream>>>(m->params, m->pb, m->P);
  LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->stream));
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_dataset(lbbsp_mlp* m, void* h_x_bf16, int* h_labels) {
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  if (h_x_bf16)
    LBBSP_CUDA_CHECK(cudaMemcpy(h_x_bf16, m->data_xb[m->cur], sizeof(bf16) * m->N_data * m->dims[0],
                                cudaMemcpyDeviceToHost));
  if (h_labels)
    LBBSP_CUDA_CHECK(cudaMemcpy(h_labels, m->data_yb[m->cur], sizeof(int) * m->N_data, cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_launches_per_iteration(lbbsp_mlp* m, int* launches) {
  *launches = m->launches;
  return LBBSP_OK;
}

// The next round's inputs go into the dataset buffer the round in flight
// does not read: the host->device copy runs on the copy stream (overlapping
// that round) once the last round that read the buffer is done, and the
// next round -- the graph bound to that buffer -- waits for the copy. No
// device-side copy sits on the round's critical path.
extern "C" int lbbsp_mlp_load_data_async(lbbsp_mlp* m, const void* h_x_bf16, const int* h_labels) {
  const size_t bx = sizeof(bf16) * m->N_data * m->dims[0], by = sizeof(int) * m->N_data;
  const int b = 1 - m->cur;
  LBBSP_CUDA_CHECK(cudaStreamWaitEvent(m->copy_stream, m->ev_used[b], 0));
  LBBSP_CUDA_CHECK(cudaMemcpyAsync(m->data_xb[b], h_x_bf16, bx, cudaMemcpyHostToDevice, m->copy_stream));
  LBBSP_CUDA_CHECK(cudaMemcpyAsync(m->data_yb[b], h_labels, by, cudaMemcpyHostToDevice, m->copy_stream));
  LBBSP_CUDA_CHECK(cudaEventRecord(m->ev_staged, m->copy_stream));
  LBBSP_CUDA_CHECK(cudaStreamWaitEvent(m->stream, m->ev_staged, 0));
  m->cur = b;
  return LBBSP_OK;
}

namespace {
// the round's record row (sizes, loss) straight into mapped page-locked host
// memory: PCIe posted writes from one CTA, no copy-engine DMA
__global__ void result_row_kernel(const int* rec_sizes, const double* rec_loss, long long row, int n,
                                  int* out_sizes, double* out_loss) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) out_sizes[i] = rec_sizes[static_cast<size_t>(row) * n + i];
  if (threadIdx.x == 0) *out_loss = rec_loss[row];
}
__global__ void last_row_kernel(const int* rows, const int* rec_sizes, const double* loss_acc,
                                int n_data, int n, int* out_sizes, double* out_loss) {
  const int r = *rows - 1;
  if (r < 0) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) out_sizes[i] = rec_sizes[static_cast<size_t>(r) * n + i];
  if (threadIdx.x == 0) *out_loss = *loss_acc / static_cast<double>(n_data);
}
}  // namespace

// Page-locked host buffers are written by the kernel itself (zero-copy over
// the unified address space); other host memory goes through a D2H copy.
// The pointer lookup is cached for the last buffer pair (a per-step
// cudaPointerGetAttributes would sit on the host's critical path).
extern "C" int lbbsp_mlp_read_result_async(lbbsp_mlp* m, int* h_sizes, double* h_loss) {
  // One rank, small head, loss every round: the round's record row (sizes,
  // and the loss its loss head wrote) is final when the round ends and no
  // later round writes it -- copy it on the result stream, beside the next
  // round, instead of a kernel on the round's critical path.
  const long long row = m->host_rounds - 1;
  if (h_sizes != m->res_host_sizes || h_loss != m->res_host_loss) {
    cudaPointerAttributes a{}, b{};
    const bool mapped = cudaPointerGetAttributes(&a, h_sizes) == cudaSuccess &&
                        cudaPointerGetAttributes(&b, h_loss) == cudaSuccess &&
                        a.type == cudaMemoryTypeHost && b.type == cudaMemoryTypeHost &&
                        a.devicePointer && b.devicePointer;
    cudaGetLastError();
    m->res_host_sizes = h_sizes;
    m->res_host_loss = h_loss;
    m->res_dev_sizes = mapped ? static_cast<int*>(a.devicePointer) : nullptr;
    m->res_dev_loss = mapped ? static_cast<double*>(b.devicePointer) : nullptr;
  }
  if (m->small_head && m->D.loss_on && m->cfg.world == 1 && m->cfg.loss_every == 1 && row >= 0 &&
      row < m->max_rows) {
    LBBSP_CUDA_CHECK(cudaEventRecord(m->ev_round_done, m->stream));
    LBBSP_CUDA_CHECK(cudaStreamWaitEvent(m->result_stream, m->ev_round_done, 0));
    if (m->res_dev_sizes) {
      // mapped host buffers: one CTA writes them, so the copy engine serves
      // only the next round's upload (a D2H copy queued there delayed it)
      result_row_kernel<<<1, 32, 0, m->result_stream>>>(m->D.rec_sizes, m->D.rec_loss, row, m->n_total,
                                                        m->res_dev_sizes, m->res_dev_loss);
      LBBSP_CUDA_CHECK(cudaGetLastError());
      return LBBSP_OK;
    }
    LBBSP_CUDA_CHECK(cudaMemcpyAsync(h_sizes, m->D.rec_sizes + static_cast<size_t>(row) * m->n_total,
                                     sizeof(int) * m->n_total, cudaMemcpyDeviceToHost, m->result_stream));
    LBBSP_CUDA_CHECK(cudaMemcpyAsync(h_loss, m->D.rec_loss + row, sizeof(double), cudaMemcpyDeviceToHost,
                                     m->result_stream));
    return LBBSP_OK;
  }
  if (m->res_dev_sizes) {
    last_row_kernel<<<1, 256, 0, m->stream>>>(m->D.rows, m->D.rec_sizes, m->D.loss_acc, m->N_data,
                                              m->n_total, m->res_dev_sizes, m->res_dev_loss);
    LBBSP_CUDA_CHECK(cudaGetLastError());
    return LBBSP_OK;
  }
  int* rs = reinterpret_cast<int*>(m->result);
  double* rl = m->result + (m->n_total + 1) / 2 + 1;
  last_row_kernel<<<1, 256, 0, m->stream>>>(m->D.rows, m->D.rec_sizes, m->D.loss_acc, m->N_data,
                                            m->n_total, rs, rl);
  LBBSP_CUDA_CHECK(cudaMemcpyAsync(h_sizes, rs, sizeof(int) * m->n_total, cudaMemcpyDeviceToHost, m->stream));
  LBBSP_CUDA_CHECK(cudaMemcpyAsync(h_loss, rl, sizeof(double), cudaMemcpyDeviceToHost, m->stream));
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_phase_times(lbbsp_mlp* m, double* h_phase_ns, int* n_phases) {
  LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->stream));
  std::vector<unsigned long long> t(2ull * kMaxPhases * m->n_local);
  LBBSP_CUDA_CHECK(cudaMemcpy(t.data(), m->D.timing, sizeof(unsigned long long) * t.size(),
                              cudaMemcpyDeviceToHost));
  *n_phases = m->n_phases;
  for (int p = 0; p < m->n_phases; ++p) {
    unsigned long long s = ~0ull, e = 0;
    for (int i = 0; i < m->n_local; ++i) {
      s = std::min(s, t[2 * (p * m->n_local + i)]);
      e = std::max(e, t[2 * (p * m->n_local + i) + 1]);
    }
    h_phase_ns[p] = (s != ~0ull && e > s) ? static_cast<double>(e - s) : 0.0;
  }
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_worker_phase_times(lbbsp_mlp* m, double* h_ns, int* n_phases) {
  LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->stream));
  std::vector<unsigned long long> t(2ull * kMaxPhases * m->n_local);
  LBBSP_CUDA_CHECK(cudaMemcpy(t.data(), m->D.timing, sizeof(unsigned long long) * t.size(),
                              cudaMemcpyDeviceToHost));
  *n_phases = m->n_phases;
  for (int p = 0; p < m->n_phases; ++p)
    for (int i = 0; i < m->n_local; ++i) {
      const unsigned long long s = t[2 * (p * m->n_local + i)], e = t[2 * (p * m->n_local + i) + 1];
      h_ns[p * m->n_local + i] = (s != ~0ull && e > s) ? static_cast<double>(e - s) : 0.0;
    }
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_work(lbbsp_mlp* m, double* gemm_flops, double* reduce_bytes) {
  if (gemm_flops) *gemm_flops = m->gemm_flops;
  if (reduce_bytes) *reduce_bytes = m->reduce_bytes;
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_rows_per_cta(lbbsp_mlp* m, int* rows) {
  if (!m || !rows) return set_error(LBBSP_INVALID_ARGUMENT, "mlp_rows_per_cta: null argument");
  *rows = m->fused && m->fused_quad ? 32 : m->fused && m->fused_pair ? 64 : 128;
  return LBBSP_OK;
}


// Debug timeline of the last round: stamps[16] then timing[kMaxPhases][n_local][2]
// (globaltimer ns). Not part of the stable C-ABI.
#ifdef LBBSP_NARX_PROF
extern "C" int lbbsp_debug_narx_prof(unsigned long long* out) {
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  LBBSP_CUDA_CHECK(cudaMemcpyFromSymbol(out, g_narx_prof, sizeof(unsigned long long) * 64 * 16));
  return LBBSP_OK;
}
#endif
// Debug (probes only): a one-thread kernel on the engine stream writes
// %globaltimer into slot [0, 8) of a scratch array, so a probe can place the
// graph's first and last kernels against stamps taken just before and after
// the round in stream order (scripts/graph_overhead_probe.py).
__global__ void debug_stamp_kernel(unsigned long long* dst) { *dst = gtimer(); }
extern "C" int lbbsp_mlp_debug_stamp(lbbsp_mlp* m, int slot) {
  if (slot < 0 || slot >= 8) return set_error(LBBSP_INVALID_ARGUMENT, "debug_stamp: slot in [0, 8)");
  if (!m->dbg_stamps) LBBSP_CUDA_CHECK(m->alloc(&m->dbg_stamps, 8));
  debug_stamp_kernel<<<1, 1, 0, m->stream>>>(m->dbg_stamps + slot);
  LBBSP_CUDA_CHECK(cudaGetLastError());
  return LBBSP_OK;
}
extern "C" int lbbsp_mlp_debug_stamps(lbbsp_mlp* m, unsigned long long* out) {
  LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->stream));
  if (!m->dbg_stamps) return set_error(LBBSP_INVALID_ARGUMENT, "debug_stamps: no stamp taken");
  LBBSP_CUDA_CHECK(cudaMemcpy(out, m->dbg_stamps, sizeof(unsigned long long) * 8, cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

extern "C" int lbbsp_mlp_debug_timeline(lbbsp_mlp* m, unsigned long long* out, int* n_phases) {
  LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->stream));
  LBBSP_CUDA_CHECK(cudaMemcpy(out, m->D.stamps, sizeof(unsigned long long) * 16, cudaMemcpyDeviceToHost));
  LBBSP_CUDA_CHECK(cudaMemcpy(out + 16, m->D.timing, sizeof(unsigned long long) * 2 * kMaxPhases * m->n_local,
                              cudaMemcpyDeviceToHost));
  *n_phases = m->n_phases;
  return LBBSP_OK;
}

// One end-to-end step through the C-ABI: stage this step's inputs from host
// memory (H2D on the copy stream, overlapping the round in flight), run the
// round, write its sizes + loss to host memory. The first call with a new
// host buffer pair warms it outside any steady-state step: DMA out of a
// freshly page-locked buffer runs at a third to half of the link rate for its
// first ~100-1000 transfers (113 us vs 38 us for the 1.57 MB dataset,
// profiles/r02_e2e_probe.txt, profiles/r02_h2d_hugepages.txt), so it is
// copied (into both dataset buffers) at least 2048 times and until three
// consecutive copies run within 15% of the fastest (at most 8192 copies).
extern "C" int lbbsp_mlp_step_e2e(lbbsp_mlp* m, const void* h_x_bf16, const int* h_labels, int* h_sizes,
                                  double* h_loss) {
  if (h_x_bf16 != m->warm_x || h_labels != m->warm_y) {
    const size_t bx = sizeof(bf16) * m->N_data * m->dims[0], by = sizeof(int) * m->N_data;
    // first-touch the new host buffers (into the idle dataset buffer; the
    // step below overwrites it again)
    LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->stream));
    LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->copy_stream));
    cudaEvent_t e0, e1;
    LBBSP_CUDA_CHECK(cudaEventCreate(&e0));
    LBBSP_CUDA_CHECK(cudaEventCreate(&e1));
    float best = 1e30f;
    int steady = 0;
    // both dataset buffers (both streams are idle here), at least 2048
    // copies: the slow phase (host->device DMA at a third to half of the
    // link rate) lasted ~100 transfers on some boxes and ~1000 on others,
    // huge-page host buffers included (scripts/e2e_rep_probe.py), at a steady
    // rate -- so "three copies within 15% of the best" alone can stop inside
    // it. One-off, outside any step: ~0.1-0.3 s per new buffer pair.
    for (int i = 0; i < 8192 && (i < 2048 || steady < 3); ++i) {
      const int b = (i & 1) ? m->cur : 1 - m->cur;
      LBBSP_CUDA_CHECK(cudaEventRecord(e0, m->copy_stream));
      LBBSP_CUDA_CHECK(cudaMemcpyAsync(m->data_xb[b], h_x_bf16, bx, cudaMemcpyHostToDevice, m->copy_stream));
      LBBSP_CUDA_CHECK(cudaMemcpyAsync(m->data_yb[b], h_labels, by, cudaMemcpyHostToDevice, m->copy_stream));
      LBBSP_CUDA_CHECK(cudaEventRecord(e1, m->copy_stream));
      LBBSP_CUDA_CHECK(cudaEventSynchronize(e1));
      float ms = 0.f;
      LBBSP_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
      steady = (i >= 8 && ms <= 1.15f * best) ? steady + 1 : 0;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    m->warm_x = h_x_bf16;
    m->warm_y = h_labels;
  }
  int rc = lbbsp_mlp_load_data_async(m, h_x_bf16, h_labels);
  if (rc) return rc;
  rc = lbbsp_mlp_run(m, 1);
  if (rc) return rc;
  return lbbsp_mlp_read_result_async(m, h_sizes, h_loss);
}

// Debug: per-CTA stage stamps of the last fused worker launch ([grid][16]
// globaltimer ns; LBBSP_FZ_DEBUG=1 at create). Not part of the stable C-ABI.
extern "C" int lbbsp_mlp_fused_debug(lbbsp_mlp* m, unsigned long long* out, int* ctas) {
  LBBSP_CUDA_CHECK(cudaStreamSynchronize(m->stream));
  *ctas = m->fz_dbg ? num_sms() : 0;
  if (m->fz_dbg)
    LBBSP_CUDA_CHECK(cudaMemcpy(out, m->fz_dbg, sizeof(unsigned long long) * 16 * num_sms(), cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}
