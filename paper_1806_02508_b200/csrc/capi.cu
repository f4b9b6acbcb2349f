// capi.cu -- the C-ABI of include/lbbsp_c.h and its C++ host runtime.
//
// Host code here only does setup (allocation, seeded generators for the
// dataset / dynamics / NARX initial weights, graph capture) and error
// translation. Every hot-path computation is a kernel in kernels.cu; there is
// no CPU fallback: without a device every compute entry point fails with
// LBBSP_CUDA.
#include <cstdarg>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "exactmath.cuh"
#include "host.cuh"
#include "kernels.cuh"
#include "predictor.cuh"

namespace lbbsp {

static thread_local std::string g_err;

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

// Rng (rng.hpp:24-42) on the host for setup-time draws.
struct HostRng {
  std::mt19937_64 g;
  explicit HostRng(uint64_t s) : g(s) {}
  double uniform() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};

// Reference wording for a device status word (batch_sizer.cpp, sgd.cpp, ...).
static int status_error(const lbbsp_dev_status& st) {
  switch (st.what) {
    case LBBSP_E_CPU_NO_WORKERS: return set_error(st.code, "cpu_allocate: no workers");
    case LBBSP_E_CPU_BUDGET:
      return set_error(st.code, "cpu_allocate: budget %lld below worker count %lld",
                       (long long)st.a, (long long)st.b);
    case LBBSP_E_CPU_SPEED: return set_error(st.code, "cpu_allocate: speeds must be > 0");
    case LBBSP_E_CPU_MIN1: return set_error(st.code, "cpu_allocate: cannot enforce minimum batch");
    case LBBSP_E_GPU_NO_WORKERS: return set_error(st.code, "gpu_allocate: no workers");
    case LBBSP_E_GPU_SLOPE: return set_error(st.code, "gpu_allocate: sec_per_sample must be > 0");
    case LBBSP_E_GPU_BASE: return set_error(st.code, "gpu_allocate: base_time_s must be >= 0");
    case LBBSP_E_GPU_BOUNDS:
      return set_error(st.code, "gpu_allocate: need 1 <= saturation_point <= oom_point");
    case LBBSP_E_GPU_COMM: return set_error(st.code, "gpu_allocate: comm time must be >= 0");
    case LBBSP_E_GPU_BELOW:
      return set_error(st.code, "gpu_allocate: budget %lld below total saturation minimum %lld",
                       (long long)st.a, (long long)st.b);
    case LBBSP_E_GPU_ABOVE:
      return set_error(st.code, "gpu_allocate: budget %lld above total memory capacity %lld",
                       (long long)st.a, (long long)st.b);
    case LBBSP_E_GPU_REPAIR: return set_error(st.code, "gpu_allocate: repair failed");
    case LBBSP_E_GPU_OOM:
      return set_error(st.code, "gpu out of memory: batch %lld exceeds oom point %lld",
                       (long long)st.a, (long long)st.b);
    case LBBSP_E_GRAD_EMPTY: return set_error(st.code, "batch_gradient: empty index set");
    case LBBSP_E_GRAD_INDEX:
      return set_error(st.code, "batch_gradient: sample index out of range");
    case LBBSP_E_AGG_BATCH:
      return set_error(st.code, "aggregate_weighted: batch size must be >= 1");
    case LBBSP_E_MLP_CAPACITY:
      return set_error(st.code, "mlp: round %lld exceeds max_iterations %lld", (long long)st.a,
                       (long long)st.b);
    default: return set_error(st.code, "lbbsp: device status %d/%d", st.code, st.what);
  }
}

// RAII device buffer
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  cudaError_t alloc(size_t count) {
    n = count;
    return cudaMalloc(&p, sizeof(T) * (count ? count : 1));
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

static int require_device() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return set_error(LBBSP_CUDA, "lbbsp: no CUDA device (the B200 path has no CPU fallback)");
  }
  return LBBSP_OK;
}

#define LBBSP_REQUIRE_DEVICE()            \
  do {                                    \
    int _rc = ::lbbsp::require_device();  \
    if (_rc) return _rc;                  \
  } while (0)

// Synchronous helper: run `fn(stream, d_status)`, then check the status word.
template <typename F>
static int run_sync(F&& fn) {
  DBuf<lbbsp_dev_status> st(1);
  LBBSP_CUDA_CHECK(cudaMemset(st.p, 0, sizeof(lbbsp_dev_status)));
  cudaStream_t s = nullptr;
  LBBSP_CUDA_CHECK(fn(s, st.p));
  LBBSP_CUDA_CHECK(cudaStreamSynchronize(s));
  lbbsp_dev_status h{};
  LBBSP_CUDA_CHECK(cudaMemcpy(&h, st.p, sizeof h, cudaMemcpyDeviceToHost));
  if (h.code) return status_error(h);
  return LBBSP_OK;
}

}  // namespace lbbsp

using namespace lbbsp;

// ===========================================================================
// misc
// ===========================================================================
extern "C" const char* lbbsp_last_error(void) { return g_err.c_str(); }
extern "C" int lbbsp_version(void) { return 1; }
extern "C" int lbbsp_check_status(const lbbsp_dev_status* h_status) {
  if (!h_status || h_status->code == 0) return LBBSP_OK;
  return status_error(*h_status);
}

extern "C" int lbbsp_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

// ===========================================================================
// solver
// ===========================================================================
extern "C" int lbbsp_solve_prop(const double* d_speeds, int n, int budget, double speed_floor,
                                int* d_sizes, lbbsp_dev_status* d_status, void* stream) {
  LBBSP_CUDA_CHECK(launch_solve_prop(d_speeds, n, budget, speed_floor, d_sizes, d_status,
                                     static_cast<cudaStream_t>(stream)));
  return LBBSP_OK;
}

extern "C" int lbbsp_solve_gpu(const lbbsp_gpu_profile* d_prof, const double* d_comm, int n,
                               int budget, int* d_sizes, lbbsp_dev_status* d_status,
                               void* stream) {
  LBBSP_CUDA_CHECK(launch_solve_gpu(d_prof, d_comm, n, budget, d_sizes, d_status,
                                    static_cast<cudaStream_t>(stream)));
  return LBBSP_OK;
}

extern "C" int lbbsp_cpu_allocate(const double* h_speeds, int n, int budget, int* h_sizes) {
  LBBSP_REQUIRE_DEVICE();
  if (n < 0) return set_error(LBBSP_INVALID_ARGUMENT, "cpu_allocate: no workers");
  DBuf<double> v(n);
  DBuf<int> out(n);
  if (n) LBBSP_CUDA_CHECK(cudaMemcpy(v.p, h_speeds, sizeof(double) * n, cudaMemcpyHostToDevice));
  int rc = run_sync([&](cudaStream_t s, lbbsp_dev_status* st) {
    return launch_solve_prop(v.p, n, budget, 0.0, out.p, st, s);
  });
  if (rc) return rc;
  if (n) LBBSP_CUDA_CHECK(cudaMemcpy(h_sizes, out.p, sizeof(int) * n, cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

extern "C" int lbbsp_gpu_allocate(const lbbsp_gpu_profile* h_prof, const double* h_comm, int n,
                                  int budget, int* h_sizes) {
  LBBSP_REQUIRE_DEVICE();
  if (n < 0) return set_error(LBBSP_INVALID_ARGUMENT, "gpu_allocate: no workers");
  DBuf<lbbsp_gpu_profile> p(n);
  DBuf<double> c(n);
  DBuf<int> out(n);
  if (n) {
    LBBSP_CUDA_CHECK(cudaMemcpy(p.p, h_prof, sizeof(lbbsp_gpu_profile) * n, cudaMemcpyHostToDevice));
    LBBSP_CUDA_CHECK(cudaMemcpy(c.p, h_comm, sizeof(double) * n, cudaMemcpyHostToDevice));
  }
  int rc = run_sync([&](cudaStream_t s, lbbsp_dev_status* st) {
    return launch_solve_gpu(p.p, c.p, n, budget, out.p, st, s);
  });
  if (rc) return rc;
  if (n) LBBSP_CUDA_CHECK(cudaMemcpy(h_sizes, out.p, sizeof(int) * n, cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

// ===========================================================================
// predictor free functions
// ===========================================================================
extern "C" int lbbsp_narx_init(uint64_t seed, lbbsp_narx_model* out) {
  // narx_init, predictor.cpp:35-44 (setup-time, host)
  HostRng rng(mix_seed(seed, 0x9a4c0ull));
  std::memset(out, 0, sizeof *out);
  for (int j = 0; j < 8; ++j) out->input_weights[j] = rng.uniform(-0.3, 0.3);
  out->hidden_bias = rng.uniform(-0.1, 0.1);
  out->output_weight = rng.uniform(-0.3, 0.3);
  out->output_bias = 0.0;
  out->speed_stddev = out->cpu_stddev = out->mem_stddev = 1.0;
  return LBBSP_OK;
}

extern "C" int lbbsp_ema(const double* h_series, int len, double alpha, double* h_out) {
  if (len <= 0) return set_error(LBBSP_INVALID_ARGUMENT, "ema: empty series");
  if (!(alpha > 0.0 && alpha <= 1.0))
    return set_error(LBBSP_INVALID_ARGUMENT, "ema: alpha must be in (0,1]");
  LBBSP_REQUIRE_DEVICE();
  DBuf<double> s(len), out(1);
  LBBSP_CUDA_CHECK(cudaMemcpy(s.p, h_series, sizeof(double) * len, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(launch_ema(s.p, len, alpha, out.p, nullptr));
  LBBSP_CUDA_CHECK(cudaMemcpy(h_out, out.p, sizeof(double), cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

extern "C" int lbbsp_narx_predict(const lbbsp_narx_model* h_model, const double h_speeds[2],
                                  const double h_cpu[3], const double h_mem[3], double floor,
                                  double* h_out) {
  LBBSP_REQUIRE_DEVICE();
  DBuf<lbbsp_narx_model> m(1);
  DBuf<double> in(8), out(1);
  const double hin[8] = {h_speeds[0], h_speeds[1], h_cpu[0], h_cpu[1], h_cpu[2],
                         h_mem[0],    h_mem[1],    h_mem[2]};
  LBBSP_CUDA_CHECK(cudaMemcpy(m.p, h_model, sizeof *h_model, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(cudaMemcpy(in.p, hin, sizeof hin, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(launch_narx_predict(m.p, in.p, floor, out.p, nullptr));
  LBBSP_CUDA_CHECK(cudaMemcpy(h_out, out.p, sizeof(double), cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

namespace {
__global__ void glibc_tanh_kernel(const double* x, double* y, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    y[i] = glibc_tanh(x[i]);
}
}  // namespace

extern "C" int lbbsp_glibc_tanh(const double* h_x, double* h_y, long long n) {
  LBBSP_REQUIRE_DEVICE();
  if (n < 0) return set_error(LBBSP_INVALID_ARGUMENT, "glibc_tanh: negative length");
  if (n == 0) return LBBSP_OK;
  DBuf<double> x(n), y(n);
  LBBSP_CUDA_CHECK(cudaMemcpy(x.p, h_x, sizeof(double) * n, cudaMemcpyHostToDevice));
  glibc_tanh_kernel<<<148 * 4, 256>>>(x.p, y.p, n);
  LBBSP_CUDA_CHECK(cudaGetLastError());
  LBBSP_CUDA_CHECK(cudaMemcpy(h_y, y.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

extern "C" int lbbsp_narx_train_online(lbbsp_narx_model* h_model, const double* h_speed,
                                       const double* h_cpu, const double* h_mem, int len,
                                       const lbbsp_narx_train_cfg* cfg,
                                       lbbsp_narx_report* h_report, double* h_loss_log) {
  LBBSP_REQUIRE_DEVICE();
  if (len < 0) return set_error(LBBSP_INVALID_ARGUMENT, "narx_train_online: negative length");
  DBuf<lbbsp_narx_model> m(1);
  DBuf<double> v(len), c(len), mm(len);
  DBuf<lbbsp_narx_report> rep(1);
  const int cap = cfg->max_epochs > 0 ? cfg->max_epochs : 1;
  DBuf<double> log(cap);
  DBuf<char> scratch(narx_train_scratch_bytes(len));
  LBBSP_CUDA_CHECK(cudaMemcpy(m.p, h_model, sizeof *h_model, cudaMemcpyHostToDevice));
  if (len) {
    LBBSP_CUDA_CHECK(cudaMemcpy(v.p, h_speed, sizeof(double) * len, cudaMemcpyHostToDevice));
    LBBSP_CUDA_CHECK(cudaMemcpy(c.p, h_cpu, sizeof(double) * len, cudaMemcpyHostToDevice));
    LBBSP_CUDA_CHECK(cudaMemcpy(mm.p, h_mem, sizeof(double) * len, cudaMemcpyHostToDevice));
  }
  LBBSP_CUDA_CHECK(cudaMemset(rep.p, 0, sizeof(lbbsp_narx_report)));
  LBBSP_CUDA_CHECK(launch_narx_train_one(m.p, v.p, c.p, mm.p, len, *cfg, rep.p, log.p, cap,
                                         reinterpret_cast<double*>(scratch.p), nullptr));
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  LBBSP_CUDA_CHECK(cudaMemcpy(h_model, m.p, sizeof *h_model, cudaMemcpyDeviceToHost));
  lbbsp_narx_report r{};
  LBBSP_CUDA_CHECK(cudaMemcpy(&r, rep.p, sizeof r, cudaMemcpyDeviceToHost));
  if (h_report) *h_report = r;
  if (h_loss_log && r.epochs > 0)
    LBBSP_CUDA_CHECK(cudaMemcpy(h_loss_log, log.p, sizeof(double) * std::min(r.epochs, cap),
                                cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

// ===========================================================================
// predictor bank
// ===========================================================================
namespace lbbsp {
// Builds a device predictor bank; used by lbbsp_predictor_create and the sim.
static int make_pred(lbbsp_predictor* P, const lbbsp_predictor_cfg* cfg, int n, int max_hist,
                     const uint64_t* seeds, const lbbsp_narx_model* initial) {
  PredDev& d = P->dev;
  d.n = n;
  d.max_hist = max_hist;
  d.kind = cfg->kind;
  d.alpha = cfg->alpha;
  d.warmup = cfg->warmup_iterations;
  d.floor = cfg->speed_floor;
  d.train = cfg->train;
  const size_t H = static_cast<size_t>(n) * max_hist;
  LBBSP_CUDA_CHECK(P->alloc(&d.hv, H));
  LBBSP_CUDA_CHECK(P->alloc(&d.hc, H));
  LBBSP_CUDA_CHECK(P->alloc(&d.hm, H));
  LBBSP_CUDA_CHECK(P->alloc(&d.ema, n));
  LBBSP_CUDA_CHECK(P->alloc(&d.comm_last, n));
  LBBSP_CUDA_CHECK(P->alloc(&d.comm_ema_lag, n));
  LBBSP_CUDA_CHECK(P->alloc(&d.models, n));
  LBBSP_CUDA_CHECK(P->alloc(&d.reports, n));
  const bool need_scratch = narx_train_min_bytes(max_hist) > train_smem_bytes(max_hist);
  LBBSP_CUDA_CHECK(P->alloc(&d.scratch, need_scratch ? static_cast<size_t>(n) * (narx_train_scratch_bytes(max_hist) / sizeof(double)) : 1));
  LBBSP_CUDA_CHECK(P->alloc(&d.len, 1));
  LBBSP_CUDA_CHECK(P->alloc(&d.cursor, 1));
  std::vector<lbbsp_narx_model> models(n);
  for (int i = 0; i < n; ++i) {
    if (initial)
      models[i] = initial[i];
    else
      lbbsp_narx_init(seeds ? seeds[i] : static_cast<uint64_t>(i), &models[i]);
  }
  LBBSP_CUDA_CHECK(cudaMemcpy(d.models, models.data(), sizeof(lbbsp_narx_model) * n,
                              cudaMemcpyHostToDevice));
  return LBBSP_OK;
}
}  // namespace lbbsp

extern "C" int lbbsp_predictor_create(const lbbsp_predictor_cfg* cfg, int n_workers,
                                      int max_history, const uint64_t* h_seeds,
                                      const lbbsp_narx_model* h_initial, lbbsp_predictor** out) {
  LBBSP_REQUIRE_DEVICE();
  if (n_workers < 1) return set_error(LBBSP_INVALID_ARGUMENT, "predictor: need at least one worker");
  if (max_history < 1) return set_error(LBBSP_INVALID_ARGUMENT, "predictor: max_history must be >= 1");
  if (!(cfg->alpha > 0.0 && cfg->alpha <= 1.0))
    return set_error(LBBSP_INVALID_ARGUMENT, "ema: alpha must be in (0,1]");
  auto P = std::make_unique<lbbsp_predictor>();
  int rc = make_pred(P.get(), cfg, n_workers, max_history, h_seeds, h_initial);
  if (rc) return rc;
  *out = P.release();
  return LBBSP_OK;
}

extern "C" int lbbsp_predictor_destroy(lbbsp_predictor* p) {
  delete p;
  return LBBSP_OK;
}

extern "C" int lbbsp_predictor_observe(lbbsp_predictor* p, const double* d_v, const double* d_c,
                                       const double* d_m, void* stream) {
  LBBSP_CUDA_CHECK(launch_pred_observe(p->dev, d_v, d_c, d_m, nullptr,
                                       static_cast<cudaStream_t>(stream)));
  return LBBSP_OK;
}

extern "C" int lbbsp_predictor_predict(lbbsp_predictor* p, const double* d_c_now,
                                       const double* d_m_now, double* d_v_pred, void* stream) {
  LBBSP_CUDA_CHECK(launch_pred_predict(p->dev, d_c_now, d_m_now, d_v_pred,
                                       static_cast<cudaStream_t>(stream)));
  return LBBSP_OK;
}

extern "C" int lbbsp_predictor_train_rotation(lbbsp_predictor* p, void* stream) {
  LBBSP_CUDA_CHECK(launch_pred_train(p->dev, 1, static_cast<cudaStream_t>(stream)));
  return LBBSP_OK;
}

extern "C" int lbbsp_predictor_train_all(lbbsp_predictor* p, void* stream) {
  LBBSP_CUDA_CHECK(launch_pred_train(p->dev, 0, static_cast<cudaStream_t>(stream)));
  return LBBSP_OK;
}

extern "C" int lbbsp_predictor_get_models(lbbsp_predictor* p, lbbsp_narx_model* h_models) {
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  LBBSP_CUDA_CHECK(cudaMemcpy(h_models, p->dev.models, sizeof(lbbsp_narx_model) * p->dev.n,
                              cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

extern "C" int lbbsp_predictor_history_len(lbbsp_predictor* p, int* h_len) {
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  LBBSP_CUDA_CHECK(cudaMemcpy(h_len, p->dev.len, sizeof(int), cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

// ===========================================================================
// workload: logistic-regression dataset + worker gradients
// ===========================================================================
struct lbbsp_lr_data {
  int n = 0, d = 0;
  DBuf<double> feat, lab;
};

namespace lbbsp {
// generate_dataset (sgd.cpp:32-57) -- setup-time, host generator, uploaded once.
static void host_generate_dataset(uint64_t seed, int n, int d, double noise,
                                  std::vector<double>& feat, std::vector<double>& lab) {
  std::vector<double> truth(d);
  HostRng tr(mix_seed(seed, 0x5e9a7a70ull));
  for (auto& w : truth) w = tr.uniform(-1.0, 1.0);
  HostRng rng(mix_seed(seed, 0xda7a5e7ull));
  feat.assign(static_cast<size_t>(n) * d, 0.0);
  lab.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double* x = feat.data() + static_cast<size_t>(i) * d;
    for (int j = 0; j < d; ++j) x[j] = rng.uniform(-1.0, 1.0);
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += truth[j] * x[j];
    const double margin = s + rng.uniform(-noise, noise);
    lab[i] = margin > 0.0 ? 1.0 : 0.0;
  }
}
}  // namespace lbbsp

extern "C" int lbbsp_lr_data_upload(const double* h_features, const double* h_labels, int n, int d,
                                    lbbsp_lr_data** out) {
  LBBSP_REQUIRE_DEVICE();
  if (n < 1) return set_error(LBBSP_INVALID_ARGUMENT, "generate_dataset: n must be >= 1");
  if (d < 1) return set_error(LBBSP_INVALID_ARGUMENT, "generate_dataset: d must be >= 1");
  auto D = std::make_unique<lbbsp_lr_data>();
  D->n = n;
  D->d = d;
  LBBSP_CUDA_CHECK(D->feat.alloc(static_cast<size_t>(n) * d));
  LBBSP_CUDA_CHECK(D->lab.alloc(n));
  LBBSP_CUDA_CHECK(cudaMemcpy(D->feat.p, h_features, sizeof(double) * n * d, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(cudaMemcpy(D->lab.p, h_labels, sizeof(double) * n, cudaMemcpyHostToDevice));
  *out = D.release();
  return LBBSP_OK;
}

extern "C" int lbbsp_lr_data_create(uint64_t seed, int n, int d, double noise, lbbsp_lr_data** out) {
  if (n < 1) return set_error(LBBSP_INVALID_ARGUMENT, "generate_dataset: n must be >= 1");
  if (d < 1) return set_error(LBBSP_INVALID_ARGUMENT, "generate_dataset: d must be >= 1");
  std::vector<double> feat, lab;
  host_generate_dataset(seed, n, d, noise, feat, lab);
  return lbbsp_lr_data_upload(feat.data(), lab.data(), n, d, out);
}

// generate_dataset / separator_params (sgd.cpp:32-57) into host arrays:
// setup-time generators for the reference-shaped API (include/lbbsp/sgd.hpp)
extern "C" int lbbsp_generate_dataset(uint64_t seed, int n, int d, double noise, double* h_features,
                                      double* h_labels) {
  if (n < 1) return set_error(LBBSP_INVALID_ARGUMENT, "generate_dataset: n must be >= 1");
  if (d < 1) return set_error(LBBSP_INVALID_ARGUMENT, "generate_dataset: d must be >= 1");
  std::vector<double> feat, lab;
  host_generate_dataset(seed, n, d, noise, feat, lab);
  std::memcpy(h_features, feat.data(), sizeof(double) * feat.size());
  std::memcpy(h_labels, lab.data(), sizeof(double) * lab.size());
  return LBBSP_OK;
}

extern "C" int lbbsp_separator_params(uint64_t seed, int d, double* h_out) {
  if (d < 1) return set_error(LBBSP_INVALID_ARGUMENT, "separator_params: d must be >= 1");
  HostRng tr(mix_seed(seed, 0x5e9a7a70ull));
  for (int j = 0; j < d; ++j) h_out[j] = tr.uniform(-1.0, 1.0);
  return LBBSP_OK;
}

// apply_update (sgd.cpp:92-99) on host buffers: the K9 device kernel
// (params -= lr * g, no FMA contraction)
extern "C" int lbbsp_apply_update(double* h_params, int dim, const double* h_grad, double lr) {
  LBBSP_REQUIRE_DEVICE();
  if (dim < 0) return set_error(LBBSP_INVALID_ARGUMENT, "apply_update: gradient dimension mismatch");
  if (dim == 0) return LBBSP_OK;
  DBuf<double> p(dim), g(dim);
  DBuf<int> one(1);
  const int b = 1;
  LBBSP_CUDA_CHECK(cudaMemcpy(p.p, h_params, sizeof(double) * dim, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(cudaMemcpy(g.p, h_grad, sizeof(double) * dim, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(cudaMemcpy(one.p, &b, sizeof(int), cudaMemcpyHostToDevice));
  int rc = run_sync([&](cudaStream_t s, lbbsp_dev_status* st) {
    return launch_aggregate_apply(g.p, one.p, 1, dim, 0, lr, p.p, nullptr, nullptr, st, s);
  });
  if (rc) return rc;
  LBBSP_CUDA_CHECK(cudaMemcpy(h_params, p.p, sizeof(double) * dim, cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

extern "C" int lbbsp_lr_data_destroy(lbbsp_lr_data* data) {
  delete data;
  return LBBSP_OK;
}

extern "C" int lbbsp_lr_data_dim(const lbbsp_lr_data* data, int* n, int* d) {
  *n = data->n;
  *d = data->d;
  return LBBSP_OK;
}

extern "C" int lbbsp_sample_stream(uint64_t seed, int64_t iteration, int budget, int dataset_size,
                                   int* d_indices, void* stream) {
  LBBSP_CUDA_CHECK(launch_sample_streams(seed, iteration, 1, budget, dataset_size, d_indices,
                                         static_cast<cudaStream_t>(stream)));
  return LBBSP_OK;
}

extern "C" int lbbsp_lr_worker_grads(const lbbsp_lr_data* data, const double* d_params,
                                     const int* d_idx, const int* d_sizes, int n_seg,
                                     double* d_grads, lbbsp_dev_status* d_status, void* stream) {
  LBBSP_CUDA_CHECK(launch_lr_worker_grads(data->feat.p, data->lab.p, data->n, data->d, d_params,
                                          d_idx, d_sizes, n_seg, d_grads, d_status,
                                          static_cast<cudaStream_t>(stream)));
  return LBBSP_OK;
}

extern "C" int lbbsp_aggregate_apply(const double* d_grads, const int* d_sizes, int n_seg, int dim,
                                     int weighted, double lr, double* d_params, double* d_agg,
                                     double* d_norm, lbbsp_dev_status* d_status, void* stream) {
  LBBSP_CUDA_CHECK(launch_aggregate_apply(d_grads, d_sizes, n_seg, dim, weighted, lr, d_params,
                                          d_agg, d_norm, d_status,
                                          static_cast<cudaStream_t>(stream)));
  return LBBSP_OK;
}

extern "C" int lbbsp_lr_loss(const lbbsp_lr_data* data, const double* d_params, double* d_loss,
                             void* stream) {
  LBBSP_CUDA_CHECK(launch_lr_loss(data->feat.p, data->lab.p, data->n, data->d, d_params, d_loss,
                                  static_cast<cudaStream_t>(stream)));
  return LBBSP_OK;
}

extern "C" int lbbsp_batch_gradient(const lbbsp_lr_data* data, const double* h_params,
                                    const int* h_indices, int count, double* h_grad) {
  LBBSP_REQUIRE_DEVICE();
  if (count <= 0) return set_error(LBBSP_INVALID_ARGUMENT, "batch_gradient: empty index set");
  DBuf<double> p(data->d), g(data->d);
  DBuf<int> idx(count), sz(1);
  LBBSP_CUDA_CHECK(cudaMemcpy(p.p, h_params, sizeof(double) * data->d, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(cudaMemcpy(idx.p, h_indices, sizeof(int) * count, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(cudaMemcpy(sz.p, &count, sizeof(int), cudaMemcpyHostToDevice));
  int rc = run_sync([&](cudaStream_t s, lbbsp_dev_status* st) {
    return launch_lr_worker_grads(data->feat.p, data->lab.p, data->n, data->d, p.p, idx.p, sz.p, 1,
                                  g.p, st, s);
  });
  if (rc) return rc;
  LBBSP_CUDA_CHECK(cudaMemcpy(h_grad, g.p, sizeof(double) * data->d, cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

extern "C" int lbbsp_loss(const lbbsp_lr_data* data, const double* h_params, double* h_loss) {
  LBBSP_REQUIRE_DEVICE();
  DBuf<double> p(data->d), out(1);
  LBBSP_CUDA_CHECK(cudaMemcpy(p.p, h_params, sizeof(double) * data->d, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(launch_lr_loss(data->feat.p, data->lab.p, data->n, data->d, p.p, out.p, nullptr));
  LBBSP_CUDA_CHECK(cudaMemcpy(h_loss, out.p, sizeof(double), cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

extern "C" int lbbsp_aggregate(const double* h_grads, const int* h_sizes, int n, int dim,
                               int weighted, double* h_out) {
  if (n <= 0) return set_error(LBBSP_INVALID_ARGUMENT, "aggregate: empty gradient list");
  LBBSP_REQUIRE_DEVICE();
  DBuf<double> g(static_cast<size_t>(n) * dim), out(dim);
  DBuf<int> sz(n);
  LBBSP_CUDA_CHECK(cudaMemcpy(g.p, h_grads, sizeof(double) * n * dim, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(cudaMemcpy(sz.p, h_sizes, sizeof(int) * n, cudaMemcpyHostToDevice));
  int rc = run_sync([&](cudaStream_t s, lbbsp_dev_status* st) {
    return launch_aggregate_apply(g.p, sz.p, n, dim, weighted, 0.0, nullptr, out.p, nullptr, st, s);
  });
  if (rc) return rc;
  LBBSP_CUDA_CHECK(cudaMemcpy(h_out, out.p, sizeof(double) * dim, cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

// ===========================================================================
// fused iteration driver (Simulation, cluster_sim.cpp:247-469, 633-643)
// ===========================================================================
struct lbbsp_sim {
  lbbsp_sim_cfg cfg{};
  SimDev dev{};
  AsyncDev adev{};
  bool async = false;
  lbbsp_predictor pred;
  std::vector<void*> allocs;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap_stream = nullptr;
  int launches = 0;
  ~lbbsp_sim() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (cap_stream) cudaStreamDestroy(cap_stream);
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
  template <typename T>
  cudaError_t upload(const T** dst, const std::vector<T>& src) {
    T* p = nullptr;
    cudaError_t e = alloc(&p, src.size());
    if (e != cudaSuccess) return e;
    if (!src.empty()) e = cudaMemcpy(p, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice);
    *dst = p;
    return e;
  }
};

namespace lbbsp {
// make_benchmark_series (cluster_sim.cpp:41-64), host, setup-time.
static void host_benchmark_series(uint64_t seed, const lbbsp_sim_cfg& c, double* cpu, double* mem,
                                  double* mult) {
  HostRng rr(mix_seed(seed, 0xbe9c0ull)), sr(mix_seed(seed, 0x59c1ceull));
  const int L = c.bench_iterations, R = c.bench_regime_length;
  const int regimes = (L + R - 1) / R;
  std::vector<double> levels(std::max(regimes, 1));
  for (int r = 0; r < regimes; ++r)
    levels[r] = (r % 2 == 0) ? rr.uniform(c.bench_high_lo, c.bench_high_hi)
                             : rr.uniform(c.bench_low_lo, c.bench_low_hi);
  for (int k = 0; k < L; ++k) {
    cpu[k] = levels[k / R];
    mem[k] = 1.0;
    mult[k] = sr.uniform() < c.bench_spike_prob ? c.bench_spike_mult : 1.0;
  }
}
}  // namespace lbbsp

extern "C" int lbbsp_benchmark_series(uint64_t seed, int iterations, int regime_length,
                                      double high_lo, double high_hi, double low_lo, double low_hi,
                                      double spike_mult, double spike_prob, double* h_cpu,
                                      double* h_mem, double* h_mult) {
  if (iterations < 1 || regime_length < 1)
    return set_error(LBBSP_INVALID_ARGUMENT, "benchmark series: need iterations, regime >= 1");
  lbbsp_sim_cfg c{};
  c.bench_iterations = iterations;
  c.bench_regime_length = regime_length;
  c.bench_high_lo = high_lo;
  c.bench_high_hi = high_hi;
  c.bench_low_lo = low_lo;
  c.bench_low_hi = low_hi;
  c.bench_spike_mult = spike_mult;
  c.bench_spike_prob = spike_prob;
  host_benchmark_series(seed, c, h_cpu, h_mem, h_mult);
  return LBBSP_OK;
}

extern "C" int lbbsp_sim_create(const lbbsp_sim_cfg* cfg, lbbsp_sim** out) {
  LBBSP_REQUIRE_DEVICE();
  const lbbsp_sim_cfg& c = *cfg;
  const int n = c.n_workers, B = c.total_budget;
  // Simulation ctor validation (cluster_sim.cpp:249-283)
  if (n < 1) return set_error(LBBSP_INVALID_ARGUMENT, "simulation: need at least one worker");
  if (B < n) return set_error(LBBSP_INVALID_ARGUMENT, "simulation: total_budget below worker count");
  if (c.scheme < LBBSP_SCHEME_BSP || c.scheme > LBBSP_SCHEME_LBBSP)
    return set_error(LBBSP_INVALID_ARGUMENT, "simulation: unknown scheme %d", c.scheme);
  if (c.staleness_threshold < 0)
    return set_error(LBBSP_INVALID_ARGUMENT, "simulation: staleness_threshold must be >= 0");
  const bool async = c.scheme == LBBSP_SCHEME_ASP || c.scheme == LBBSP_SCHEME_SSP;
  if (c.scheme != LBBSP_SCHEME_LBBSP && B % n != 0)
    return set_error(LBBSP_INVALID_ARGUMENT,
                     "simulation: bsp/asp/ssp need total_budget divisible by workers");
  if (c.max_updates < 1 || c.max_updates > (1 << 24))
    return set_error(LBBSP_INVALID_ARGUMENT, "simulation: max_updates must be in [1, 2^24]");
  const bool gpu_mode = c.gpu_profiles != nullptr;
  std::vector<int> equal(n);
  for (int i = 0; i < n; ++i) equal[i] = B / n + (i < B % n ? 1 : 0);  // equal_split :209-213
  if (gpu_mode) {
    for (int i = 0; i < n; ++i)
      if (c.scheme != LBBSP_SCHEME_LBBSP && equal[i] > c.gpu_profiles[i].oom_point)
        return set_error(LBBSP_INVALID_ARGUMENT,
                         "simulation: equal split exceeds oom point of worker %d", i);
    if (c.scheme == LBBSP_SCHEME_LBBSP) {  // surfaces infeasible budgets up front (:276-282)
      std::vector<double> zeros(n, 0.0);
      std::vector<int> tmp(n);
      const int rc = lbbsp_gpu_allocate(c.gpu_profiles, zeros.data(), n, B, tmp.data());
      if (rc) return rc;
    }
  }
  auto S = std::make_unique<lbbsp_sim>();
  S->cfg = c;
  SimDev& d = S->dev;
  d.n = n;
  d.B = B;
  d.N = c.dataset_size;
  d.d = c.dataset_dim;
  d.scheme = c.scheme;
  d.gpu_mode = gpu_mode;
  d.base_speed = c.base_speed;
  d.lr = c.learning_rate;
  d.conv_loss = c.convergence_loss;
  d.conv_consec = c.convergence_consecutive;
  d.max_updates = c.max_updates;
  d.seed = c.seed;
  d.base_comm = c.base_comm_s;
  d.bw_worker = c.bw_worker;
  d.bw_at = c.bw_at_iteration;
  d.bw_factor = c.bw_factor;

  // dynamics: presets resolved here (heterogeneity_preset, cluster_sim.cpp:140-197)
  std::vector<double> scpu, smem, phase(n);
  std::vector<lbbsp_straggler> strag;
  int dyn = c.dynamics;
  if (gpu_mode) {
    dyn = LBBSP_DYN_STATIC;
  } else if (c.preset != LBBSP_PRESET_NONE) {
    if (n < 2) return set_error(LBBSP_INVALID_ARGUMENT, "heterogeneity_preset: need n >= 2");
    const double ratio = c.preset == LBBSP_PRESET_HOMO ? 1.0
                         : (c.preset == LBBSP_PRESET_HETERO_L2 || c.preset == LBBSP_PRESET_HETERO_L2_STATIC)
                             ? 0.5
                             : 1.0 / 3.0;
    auto avg = [&](int i) {
      return 1.0 - (1.0 - ratio) * static_cast<double>(i) / static_cast<double>(n - 1);
    };
    if (c.preset == LBBSP_PRESET_HOMO) {
      dyn = LBBSP_DYN_STATIC;
      scpu.assign(n, 1.0);
    } else if (c.preset == LBBSP_PRESET_HETERO_L2_STATIC || c.preset == LBBSP_PRESET_HETERO_L3_STATIC) {
      dyn = LBBSP_DYN_STATIC;
      for (int i = 0; i < n; ++i) scpu.push_back(avg(i));
    } else {
      dyn = LBBSP_DYN_STRAGGLER;
      for (int i = 0; i < n; ++i) {
        lbbsp_straggler s{0.0, 0.0, 0.0, 10};
        if (i > 0) {
          s.on_probability = 0.75;
          s.cpu_consumed = (1.0 - avg(i)) / 0.75;
        }
        strag.push_back(s);
      }
    }
  } else {
    if (c.static_cpu) scpu.assign(c.static_cpu, c.static_cpu + n);
    if (c.static_mem) smem.assign(c.static_mem, c.static_mem + n);
    if (c.stragglers) strag.assign(c.stragglers, c.stragglers + n);
  }
  d.dyn_kind = dyn;
  for (int i = 0; i < n; ++i)  // Dynamics ctor (cluster_sim.cpp:66-75)
    phase[i] = HostRng(mix_seed(c.seed, 0x477a5eull, static_cast<uint64_t>(i))).uniform();
  LBBSP_CUDA_CHECK(S->upload(&d.phase, phase));
  if (!scpu.empty()) LBBSP_CUDA_CHECK(S->upload(&d.static_cpu, scpu));
  if (!smem.empty()) LBBSP_CUDA_CHECK(S->upload(&d.static_mem, smem));
  if (!strag.empty()) LBBSP_CUDA_CHECK(S->upload(&d.strag, strag));
  if (dyn == LBBSP_DYN_BENCHMARK) {
    const int L = c.bench_iterations;
    if (L < 1 || c.bench_regime_length < 1)
      return set_error(LBBSP_INVALID_ARGUMENT, "benchmark series: need iterations, regime >= 1");
    std::vector<double> bc(static_cast<size_t>(n) * L), bm(bc.size()), bx(bc.size());
    for (int i = 0; i < n; ++i)
      host_benchmark_series(mix_seed(c.seed, 0xbe7cull, static_cast<uint64_t>(i)), c,
                            bc.data() + static_cast<size_t>(i) * L, bm.data() + static_cast<size_t>(i) * L,
                            bx.data() + static_cast<size_t>(i) * L);
    d.bench_len = L;
    LBBSP_CUDA_CHECK(S->upload(&d.bcpu, bc));
    LBBSP_CUDA_CHECK(S->upload(&d.bmem, bm));
    LBBSP_CUDA_CHECK(S->upload(&d.bmult, bx));
  }
  if (dyn == LBBSP_DYN_TRACE) {  // Dynamics::at Trace (cluster_sim.cpp:110-115)
    if (!c.trace_offsets || !c.trace_t || !c.trace_cpu || !c.trace_mem)
      return set_error(LBBSP_INVALID_ARGUMENT, "simulation: trace dynamics need trace arrays");
    std::vector<int> off(c.trace_offsets, c.trace_offsets + n + 1);
    for (int i = 0; i < n; ++i)
      if (off[i + 1] <= off[i]) return set_error(LBBSP_INVALID_ARGUMENT, "trace_at: empty trace");
    const size_t P = static_cast<size_t>(off[n]);
    LBBSP_CUDA_CHECK(S->upload(&d.trace_off, off));
    LBBSP_CUDA_CHECK(S->upload(&d.trace_t, std::vector<double>(c.trace_t, c.trace_t + P)));
    LBBSP_CUDA_CHECK(S->upload(&d.trace_c, std::vector<double>(c.trace_cpu, c.trace_cpu + P)));
    LBBSP_CUDA_CHECK(S->upload(&d.trace_m, std::vector<double>(c.trace_mem, c.trace_mem + P)));
  }
  if (gpu_mode) {
    std::vector<lbbsp_gpu_profile> prof(c.gpu_profiles, c.gpu_profiles + n);
    LBBSP_CUDA_CHECK(S->upload(&d.prof, prof));
  }
  LBBSP_CUDA_CHECK(S->upload(&d.equal, equal));

  // dataset + params (cluster_sim.cpp:285-288)
  std::vector<double> feat, lab;
  if (c.dataset_size < 1 || c.dataset_dim < 1)
    return set_error(LBBSP_INVALID_ARGUMENT, "generate_dataset: n and d must be >= 1");
  if (c.dataset_dim > 1024)
    return set_error(LBBSP_INVALID_ARGUMENT, "simulation: dataset_dim above 1024 is not supported");
  host_generate_dataset(c.dataset_seed, c.dataset_size, c.dataset_dim, c.dataset_noise, feat, lab);
  LBBSP_CUDA_CHECK(S->upload(&d.feat, feat));
  LBBSP_CUDA_CHECK(S->upload(&d.lab, lab));
  LBBSP_CUDA_CHECK(S->alloc(&d.params, d.d));
  LBBSP_CUDA_CHECK(S->alloc(&d.grads, static_cast<size_t>(n) * d.d));
  LBBSP_CUDA_CHECK(S->alloc(&d.agg, d.d));

  const size_t R = static_cast<size_t>(c.max_updates);
  // sync: one stream per round; async: one per local iteration j (a worker's
  // j never exceeds the update count, plus the SSP staleness window)
  const size_t J = async ? R + (c.scheme == LBBSP_SCHEME_SSP ? c.staleness_threshold + 2 : 1) : R;
  int* streams = nullptr;
  LBBSP_CUDA_CHECK(S->alloc(&streams, J * B));
  d.streams = streams;
  LBBSP_CUDA_CHECK(S->alloc(&d.k, 1));
  LBBSP_CUDA_CHECK(S->alloc(&d.done, 1));
  LBBSP_CUDA_CHECK(S->alloc(&d.active, 1));
  LBBSP_CUDA_CHECK(S->alloc(&d.converged, 1));
  LBBSP_CUDA_CHECK(S->alloc(&d.below, 1));
  LBBSP_CUDA_CHECK(S->alloc(&d.rows, 1));
  LBBSP_CUDA_CHECK(S->alloc(&d.train_first, 1));
  LBBSP_CUDA_CHECK(S->alloc(&d.c_now, n));
  LBBSP_CUDA_CHECK(S->alloc(&d.m_now, n));
  LBBSP_CUDA_CHECK(S->alloc(&d.vact, n));
  LBBSP_CUDA_CHECK(S->alloc(&d.vpred, n));
  LBBSP_CUDA_CHECK(S->alloc(&d.tp, n));
  LBBSP_CUDA_CHECK(S->alloc(&d.tm, n));
  LBBSP_CUDA_CHECK(S->alloc(&d.sizes, n));
  LBBSP_CUDA_CHECK(S->alloc(&d.offsets, n));
  LBBSP_CUDA_CHECK(S->alloc(&d.wall, 1));
  LBBSP_CUDA_CHECK(S->alloc(&d.now, 1));
  LBBSP_CUDA_CHECK(S->alloc(&d.rec_sc, R));
  LBBSP_CUDA_CHECK(S->alloc(&d.rec_batch, R * n));
  LBBSP_CUDA_CHECK(S->alloc(&d.rec_tp, R * n));
  LBBSP_CUDA_CHECK(S->alloc(&d.rec_tm, R * n));
  LBBSP_CUDA_CHECK(S->alloc(&d.rec_wait, R * n));
  LBBSP_CUDA_CHECK(S->alloc(&d.rec_vpred, R * n));
  LBBSP_CUDA_CHECK(S->alloc(&d.rec_vact, R * n));
  LBBSP_CUDA_CHECK(S->alloc(&d.rec_params, R * d.d));
  LBBSP_CUDA_CHECK(S->alloc(&d.status, 1));

  // per-worker predictors seeded mix_seed(seed, 0x9ced1c70, i) (cluster_sim.cpp:295)
  std::vector<uint64_t> seeds(n);
  for (int i = 0; i < n; ++i) seeds[i] = mix_seed(c.seed, 0x9ced1c70ull, static_cast<uint64_t>(i));
  lbbsp_predictor_cfg pc = c.predictor;
  pc.train.min_history = pc.warmup_iterations;
  std::vector<lbbsp_narx_model> initial;  // PredictorConfig::initial_weights (predictor.cpp:265)
  if (c.narx_weights_path && c.narx_weights_path[0]) {
    lbbsp_narx_model m{};
    if (int rc = lbbsp_narx_load_csv(c.narx_weights_path, &m)) return rc;
    initial.assign(n, m);
  }
  int rc = make_pred(&S->pred, &pc, n, static_cast<int>(J), seeds.data(),
                     initial.empty() ? nullptr : initial.data());
  if (rc) return rc;
  d.pred = S->pred.dev;

  // the whole run's sample streams, generated ahead of the iterations
  LBBSP_CUDA_CHECK(launch_sample_streams(c.seed, 0, static_cast<int>(J), B, c.dataset_size,
                                         streams, nullptr));
  if (async) {
    AsyncDev& A = S->adev;
    S->async = true;
    A.ssp = c.scheme == LBBSP_SCHEME_SSP;
    A.stale = c.staleness_threshold;
    A.ring = c.staleness_threshold + 3;
    A.n_streams = static_cast<int>(J);
    LBBSP_CUDA_CHECK(S->alloc(&A.started, 1));
    LBBSP_CUDA_CHECK(S->alloc(&A.completed, n));
    LBBSP_CUDA_CHECK(S->alloc(&A.running, n));
    LBBSP_CUDA_CHECK(S->alloc(&A.blocked, n));
    LBBSP_CUDA_CHECK(S->alloc(&A.hist_len, n));
    LBBSP_CUDA_CHECK(S->alloc(&A.block_start, n));
    LBBSP_CUDA_CHECK(S->alloc(&A.pending_wait, n));
    LBBSP_CUDA_CHECK(S->alloc(&A.finish, n));
    LBBSP_CUDA_CHECK(S->alloc(&A.inflight_grad, static_cast<size_t>(n) * d.d));
    LBBSP_CUDA_CHECK(S->alloc(&A.inflight, static_cast<size_t>(n) * 8));
    if (A.ssp) {
      LBBSP_CUDA_CHECK(S->alloc(&A.ring_grads, static_cast<size_t>(A.ring) * n * d.d));
      LBBSP_CUDA_CHECK(S->alloc(&A.ring_stats, static_cast<size_t>(A.ring) * n * 6));
      LBBSP_CUDA_CHECK(S->alloc(&A.ring_count, A.ring));
    }
    LBBSP_CUDA_CHECK(S->alloc(&A.last_update, 1));
    LBBSP_CUDA_CHECK(S->alloc(&A.clock, 1));
    LBBSP_CUDA_CHECK(S->alloc(&A.max_skew, 1));
    LBBSP_CUDA_CHECK(S->alloc(&A.rec_worker, R * n));
    LBBSP_CUDA_CHECK(S->alloc(&A.rec_nw, R));
  }
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  *out = S.release();
  return LBBSP_OK;
}

extern "C" int lbbsp_sim_destroy(lbbsp_sim* sim) {
  delete sim;
  return LBBSP_OK;
}

extern "C" int lbbsp_sim_run(lbbsp_sim* sim, int iterations, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (sim->async) {  // ASP/SSP: the whole event loop in one persistent CTA
    if (iterations > 0) LBBSP_CUDA_CHECK(launch_async_sim(sim->dev, sim->adev, iterations, s));
    return LBBSP_OK;
  }
  if (!sim->exec) {
    // warm the function attributes outside capture, then capture one round
    LBBSP_CUDA_CHECK(cudaStreamCreateWithFlags(&sim->cap_stream, cudaStreamNonBlocking));
    LBBSP_CUDA_CHECK(cudaStreamBeginCapture(sim->cap_stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = launch_sim_iteration(sim->dev, sim->cap_stream, &sim->launches);
    cudaError_t e2 = cudaStreamEndCapture(sim->cap_stream, &sim->graph);
    LBBSP_CUDA_CHECK(e);
    LBBSP_CUDA_CHECK(e2);
    LBBSP_CUDA_CHECK(cudaGraphInstantiate(&sim->exec, sim->graph, 0));
  }
  for (int i = 0; i < iterations; ++i) LBBSP_CUDA_CHECK(cudaGraphLaunch(sim->exec, s));
  return LBBSP_OK;
}

extern "C" int lbbsp_sim_status(lbbsp_sim* sim, int* done, int* converged) {
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  int h[2];
  LBBSP_CUDA_CHECK(cudaMemcpy(&h[0], sim->dev.done, sizeof(int), cudaMemcpyDeviceToHost));
  LBBSP_CUDA_CHECK(cudaMemcpy(&h[1], sim->dev.converged, sizeof(int), cudaMemcpyDeviceToHost));
  if (done) *done = h[0];
  if (converged) *converged = h[1];
  lbbsp_dev_status st{};
  LBBSP_CUDA_CHECK(cudaMemcpy(&st, sim->dev.status, sizeof st, cudaMemcpyDeviceToHost));
  if (st.code) return status_error(st);
  return LBBSP_OK;
}

extern "C" int lbbsp_sim_records(lbbsp_sim* sim, int max_rows, int* rows, lbbsp_iter_scalars* sc,
                                 int* batch, double* tp, double* tm, double* wait, double* v_pred,
                                 double* v_actual, double* params) {
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  int r = 0;
  LBBSP_CUDA_CHECK(cudaMemcpy(&r, sim->dev.rows, sizeof(int), cudaMemcpyDeviceToHost));
  r = std::min(r, max_rows);
  *rows = r;
  const int n = sim->dev.n, d = sim->dev.d;
  const SimDev& D = sim->dev;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!dst || bytes == 0) return cudaSuccess;
    return cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
  };
  LBBSP_CUDA_CHECK(cp(sc, D.rec_sc, sizeof(lbbsp_iter_scalars) * r));
  LBBSP_CUDA_CHECK(cp(batch, D.rec_batch, sizeof(int) * r * n));
  LBBSP_CUDA_CHECK(cp(tp, D.rec_tp, sizeof(double) * r * n));
  LBBSP_CUDA_CHECK(cp(tm, D.rec_tm, sizeof(double) * r * n));
  LBBSP_CUDA_CHECK(cp(wait, D.rec_wait, sizeof(double) * r * n));
  LBBSP_CUDA_CHECK(cp(v_pred, D.rec_vpred, sizeof(double) * r * n));
  LBBSP_CUDA_CHECK(cp(v_actual, D.rec_vact, sizeof(double) * r * n));
  LBBSP_CUDA_CHECK(cp(params, D.rec_params, sizeof(double) * r * d));
  return LBBSP_OK;
}

extern "C" int lbbsp_sim_launches_per_iteration(lbbsp_sim* sim, int* launches) {
  if (sim->async)
    *launches = 1;  // one persistent kernel for all updates of a run_rounds call
  else
    *launches = sim->launches ? sim->launches : (sim->dev.pred.kind == LBBSP_PRED_NARX ? 4 : 3);
  return LBBSP_OK;
}

extern "C" int lbbsp_sim_record_workers(lbbsp_sim* sim, int max_rows, int* worker_id,
                                        int* row_workers) {
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  int r = 0;
  LBBSP_CUDA_CHECK(cudaMemcpy(&r, sim->dev.rows, sizeof(int), cudaMemcpyDeviceToHost));
  r = std::min(r, max_rows);
  const int n = sim->dev.n;
  if (sim->async) {
    if (worker_id)
      LBBSP_CUDA_CHECK(cudaMemcpy(worker_id, sim->adev.rec_worker, sizeof(int) * r * n,
                                  cudaMemcpyDeviceToHost));
    if (row_workers)
      LBBSP_CUDA_CHECK(cudaMemcpy(row_workers, sim->adev.rec_nw, sizeof(int) * r,
                                  cudaMemcpyDeviceToHost));
  } else {
    for (int i = 0; i < r; ++i) {
      if (row_workers) row_workers[i] = n;
      for (int w = 0; w < n && worker_id; ++w) worker_id[static_cast<size_t>(i) * n + w] = w;
    }
  }
  return LBBSP_OK;
}

extern "C" int lbbsp_sim_summary(lbbsp_sim* sim, double* total_time_s, int64_t* max_ssp_skew) {
  LBBSP_CUDA_CHECK(cudaDeviceSynchronize());
  double now = 0.0, last = 0.0;
  long long skew = 0;
  LBBSP_CUDA_CHECK(cudaMemcpy(&now, sim->dev.now, sizeof now, cudaMemcpyDeviceToHost));
  if (sim->async) {
    LBBSP_CUDA_CHECK(cudaMemcpy(&last, sim->adev.last_update, sizeof last, cudaMemcpyDeviceToHost));
    LBBSP_CUDA_CHECK(cudaMemcpy(&skew, sim->adev.max_skew, sizeof skew, cudaMemcpyDeviceToHost));
  }
  // result.total_time_s = last_update_time_ > 0 ? last_update_time_ : now_
  if (total_time_s) *total_time_s = last > 0.0 ? last : now;
  if (max_ssp_skew) *max_ssp_skew = skew;
  return LBBSP_OK;
}

extern "C" int lbbsp_sim_metrics(lbbsp_sim* sim, int rmse_from_iteration, lbbsp_metrics* out) {
  double* scratch = nullptr;
  lbbsp_metrics* d_out = nullptr;
  const size_t cap = static_cast<size_t>(sim->dev.max_updates) * sim->dev.n;
  LBBSP_CUDA_CHECK(sim->alloc(&scratch, 2 * cap));
  LBBSP_CUDA_CHECK(sim->alloc(&d_out, 1));
  LBBSP_CUDA_CHECK(launch_sim_metrics(sim->dev, sim->async ? sim->adev.rec_nw : nullptr,
                                      rmse_from_iteration, scratch, d_out, nullptr));
  LBBSP_CUDA_CHECK(cudaMemcpy(out, d_out, sizeof *out, cudaMemcpyDeviceToHost));
  return LBBSP_OK;
}

extern "C" int lbbsp_predictor_series_rmse(int kind, const lbbsp_predictor_cfg* base,
                                           const double* h_cpu, const double* h_mem,
                                           const double* h_mult, int len, double base_speed,
                                           uint64_t seed, int measure_from, double* rmse) {
  LBBSP_REQUIRE_DEVICE();
  if (len < 1) return set_error(LBBSP_INVALID_ARGUMENT, "predictor_series_rmse: nothing to measure");
  lbbsp_predictor_cfg pc = *base;
  pc.kind = kind;
  pc.train.min_history = pc.warmup_iterations;  // SpeedPredictor ctor (predictor.cpp:264)
  lbbsp_predictor P;
  if (int rc = make_pred(&P, &pc, 1, len, &seed, nullptr)) return rc;
  double* series = nullptr;
  double* out2 = nullptr;
  LBBSP_CUDA_CHECK(P.alloc(&series, 3 * static_cast<size_t>(len)));
  LBBSP_CUDA_CHECK(P.alloc(&out2, 2));
  LBBSP_CUDA_CHECK(cudaMemcpy(series, h_cpu, sizeof(double) * len, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(cudaMemcpy(series + len, h_mem, sizeof(double) * len, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(cudaMemcpy(series + 2 * len, h_mult, sizeof(double) * len, cudaMemcpyHostToDevice));
  LBBSP_CUDA_CHECK(launch_series_rmse(P.dev, series, series + len, series + 2 * len, len,
                                      base_speed, measure_from, out2, nullptr));
  double h[2];
  LBBSP_CUDA_CHECK(cudaMemcpy(h, out2, sizeof h, cudaMemcpyDeviceToHost));
  if (h[1] == 0.0)
    return set_error(LBBSP_INVALID_ARGUMENT, "predictor_series_rmse: nothing to measure");
  *rmse = std::sqrt(h[0] / h[1]);
  return LBBSP_OK;
}
