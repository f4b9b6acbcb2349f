/* ORACLE / TEST INFRASTRUCTURE ONLY (see lbbsp_oracle.h).
 *
 * Plain-C restatement of the reference LB-BSP hot path. Each function cites
 * the reference file:line it follows (paths relative to /root/reference/proj).
 * Compiled with -O2 -ffp-contract=off on baseline x86-64 (oracle/Makefile),
 * the same floating-point environment as the reference build, so every
 * result is bit-identical to oracle/_ref/liblbbsp_ref.so. */
#define _GNU_SOURCE
#include "lbbsp_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------------- */
/* rng.hpp:9-42                                                            */
/* ---------------------------------------------------------------------- */

uint64_t orc_mix64(uint64_t z) { /* rng.hpp:9-14 (splitmix64 finaliser) */
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
uint64_t orc_mix_seed2(uint64_t a, uint64_t b) { return orc_mix64(a ^ orc_mix64(b)); } /* :16 */
uint64_t orc_mix_seed3(uint64_t a, uint64_t b, uint64_t c) {                          /* :18 */
  return orc_mix_seed2(orc_mix_seed2(a, b), c);
}

/* std::mt19937_64 (the standard fixes its output bit-for-bit) */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t s) {
  g->mt[0] = s;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull, A = 0xB5026F5AA96619E9ull;
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      g->mt[i] = g->mt[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}

/* Rng::uniform (rng.hpp:31) */
static double rng_uniform(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }
/* Rng::uniform(lo, hi) (rng.hpp:33) */
static double rng_uniform2(mt64* g, double lo, double hi) { return lo + (hi - lo) * rng_uniform(g); }
/* Rng::uniform_int (rng.hpp:36-38) */
static int rng_uniform_int(mt64* g, int lo, int hi) {
  return lo + (int)(rng_uniform(g) * (double)(hi - lo + 1));
}

void orc_rng_u64(uint64_t seed, int count, uint64_t* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int i = 0; i < count; ++i) out[i] = mt64_next(&g);
}
void orc_rng_uniform_int(uint64_t seed, int count, int lo, int hi, int* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int i = 0; i < count; ++i) out[i] = rng_uniform_int(&g, lo, hi);
}

/* ---------------------------------------------------------------------- */
/* batch_sizer.cpp                                                          */
/* ---------------------------------------------------------------------- */

/* cpu_allocate, batch_sizer.cpp:54-99 */
int orc_cpu_allocate(const double* v, int n, int budget, int* out) {
  if (n == 0) return err(LBBSP_INVALID_ARGUMENT, "cpu_allocate: no workers");
  if (budget < n)
    return err(LBBSP_INVALID_ARGUMENT, "cpu_allocate: budget %d below worker count %d", budget, n);
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!(v[i] > 0.0)) return err(LBBSP_INVALID_ARGUMENT, "cpu_allocate: speeds must be > 0");
    sum += v[i];
  }
  double* rem = (double*)malloc(sizeof(double) * (size_t)n);
  int* order = (int*)malloc(sizeof(int) * (size_t)n);
  int assigned = 0;
  for (int i = 0; i < n; ++i) {
    const double share = v[i] / sum * (double)budget;
    const double fl = floor(share);
    out[i] = (int)fl;
    rem[i] = share - fl;
    assigned += (int)fl;
  }
  /* stable_sort by remainder descending == total order (rem desc, index asc);
   * insertion sort is stable */
  for (int i = 0; i < n; ++i) {
    int j = i;
    while (j > 0 && rem[order[j - 1]] < rem[i]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = i;
  }
  for (int k = 0; k < budget - assigned; ++k) out[order[k]] += 1;
  /* min-1 repair from the first max_element (:90-97) */
  int status = 0;
  for (int i = 0; i < n && status == 0; ++i) {
    while (out[i] < 1) {
      int big = 0;
      for (int j = 1; j < n; ++j)
        if (out[j] > out[big]) big = j;
      if (out[big] <= 1) {
        status = err(LBBSP_LOGIC, "cpu_allocate: cannot enforce minimum batch");
        break;
      }
      out[big] -= 1;
      out[i] += 1;
    }
  }
  free(rem);
  free(order);
  return status;
}

/* gpu_time, batch_sizer.cpp:47-50 */
static double gpu_time(const lbbsp_gpu_profile* p, int x, double comm) {
  return p->sec_per_sample * (double)(x > p->saturation_point ? x : p->saturation_point) +
         p->base_time_s + comm;
}

static double clampd(double x, double lo, double hi) { /* std::clamp */
  return x < lo ? lo : (hi < x ? hi : x);
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* validate_gpu_instance, batch_sizer.cpp:18-45 */
static int validate_gpu(const lbbsp_gpu_profile* p, const double* comm, int n, int budget) {
  if (n == 0) return err(LBBSP_INVALID_ARGUMENT, "gpu_allocate: no workers");
  long long lo = 0, hi = 0;
  for (int i = 0; i < n; ++i) {
    if (p[i].sec_per_sample <= 0.0)
      return err(LBBSP_INVALID_ARGUMENT, "gpu_allocate: sec_per_sample must be > 0");
    if (p[i].base_time_s < 0.0)
      return err(LBBSP_INVALID_ARGUMENT, "gpu_allocate: base_time_s must be >= 0");
    if (p[i].saturation_point < 1 || p[i].oom_point < p[i].saturation_point)
      return err(LBBSP_INVALID_ARGUMENT, "gpu_allocate: need 1 <= saturation_point <= oom_point");
    if (comm[i] < 0.0) return err(LBBSP_INVALID_ARGUMENT, "gpu_allocate: comm time must be >= 0");
    lo += p[i].saturation_point;
    hi += p[i].oom_point;
  }
  if (budget < lo)
    return err(LBBSP_INVALID_ARGUMENT, "gpu_allocate: budget %d below total saturation minimum %lld",
               budget, lo);
  if (budget > hi)
    return err(LBBSP_INVALID_ARGUMENT, "gpu_allocate: budget %d above total memory capacity %lld",
               budget, hi);
  return 0;
}

static double demand_at(const lbbsp_gpu_profile* p, const double* comm, int n, double level) {
  double s = 0.0; /* batch_sizer.cpp:110-120 */
  for (int i = 0; i < n; ++i) {
    double x = (level - p[i].base_time_s - comm[i]) / p[i].sec_per_sample;
    x = clampd(x, (double)p[i].saturation_point, (double)p[i].oom_point);
    s += x;
  }
  return s;
}

/* gpu_allocate, batch_sizer.cpp:101-199 */
int orc_gpu_allocate(const lbbsp_gpu_profile* p, const double* comm, int n, int budget, int* out) {
  int st = validate_gpu(p, comm, n, budget);
  if (st) return st;
  double* bp = (double*)malloc(sizeof(double) * (size_t)(2 * n));
  for (int i = 0; i < n; ++i) {
    bp[2 * i] = gpu_time(&p[i], p[i].saturation_point, comm[i]);
    bp[2 * i + 1] = gpu_time(&p[i], p[i].oom_point, comm[i]);
  }
  qsort(bp, (size_t)(2 * n), sizeof(double), cmp_double);
  const double target = (double)budget;
  double level = bp[0];
  if (demand_at(p, comm, n, level) < target) {
    for (int b = 0; b + 1 < 2 * n; ++b) {
      const double t0 = bp[b], t1 = bp[b + 1];
      if (demand_at(p, comm, n, t1) < target) continue;
      double slope = 0.0;
      for (int i = 0; i < n; ++i)
        if (gpu_time(&p[i], p[i].saturation_point, comm[i]) <= t0 &&
            gpu_time(&p[i], p[i].oom_point, comm[i]) > t0)
          slope += 1.0 / p[i].sec_per_sample;
      level = slope > 0.0 ? t0 + (target - demand_at(p, comm, n, t0)) / slope : t1;
      break;
    }
  }
  free(bp);
  int assigned = 0;
  for (int i = 0; i < n; ++i) {
    double x = (level - p[i].base_time_s - comm[i]) / p[i].sec_per_sample;
    x = clampd(x, (double)p[i].saturation_point, (double)p[i].oom_point);
    int xi = (int)floor(x);
    if (xi < p[i].saturation_point) xi = p[i].saturation_point;
    if (xi > p[i].oom_point) xi = p[i].oom_point;
    out[i] = xi;
    assigned += xi;
  }
  while (assigned < budget) { /* :165-180 */
    int best = -1;
    double best_t = INFINITY;
    for (int i = 0; i < n; ++i) {
      if (out[i] >= p[i].oom_point) continue;
      const double t = gpu_time(&p[i], out[i] + 1, comm[i]);
      if (t < best_t) {
        best_t = t;
        best = i;
      }
    }
    out[best] += 1;
    ++assigned;
  }
  while (assigned > budget) { /* :181-197 */
    int worst = -1;
    double worst_t = -1.0;
    for (int i = 0; i < n; ++i) {
      if (out[i] <= p[i].saturation_point) continue;
      const double t = gpu_time(&p[i], out[i], comm[i]);
      if (t > worst_t) {
        worst_t = t;
        worst = i;
      }
    }
    if (worst < 0) return err(LBBSP_LOGIC, "gpu_allocate: repair failed");
    out[worst] -= 1;
    --assigned;
  }
  return 0;
}

/* ---------------------------------------------------------------------- */
/* predictor.cpp                                                            */
/* ---------------------------------------------------------------------- */

/* ema, predictor.cpp:18-25 */
int orc_ema(const double* s, int len, double alpha, double* out) {
  if (len <= 0) return err(LBBSP_INVALID_ARGUMENT, "ema: empty series");
  if (!(alpha > 0.0 && alpha <= 1.0)) return err(LBBSP_INVALID_ARGUMENT, "ema: alpha must be in (0,1]");
  double value = s[0];
  for (int k = 1; k < len; ++k) value = alpha * s[k] + (1.0 - alpha) * value;
  *out = value;
  return 0;
}

/* glibc 2.39 tanh (sysdeps/ieee754/dbl-64/s_tanh.c, fdlibm) calling expm1
 * through its IFUNC; on FMA hosts the __expm1_fma variant (the same fdlibm
 * source built with -mfma, whose contractions are restated here from its
 * disassembly). The reference's NARX calls std::tanh, so bit parity of the
 * device predictor hinges on this exact dataflow. Used only to validate the
 * device port (csrc/exactmath.cuh) on the host. */
static double with_high(double x, uint32_t hi) {
  uint64_t u;
  memcpy(&u, &x, 8);
  u = (u & 0xffffffffull) | ((uint64_t)hi << 32);
  memcpy(&x, &u, 8);
  return x;
}
static uint32_t high_word(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return (uint32_t)(u >> 32);
}
static uint32_t low_word(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return (uint32_t)u;
}

double orc_expm1_glibc_fma(double x) {
  const double o_threshold = 0x1.62e42fefa39efp+9, ln2_hi = 0x1.62e42fee00000p-1,
               ln2_lo = 0x1.a39ef35793c76p-33, invln2 = 0x1.71547652b82fep+0;
  const double Q1 = -0x1.11111111110f4p-5, Q2 = 0x1.a01a019fe5585p-10,
               Q3 = -0x1.4ce199eaadbb7p-14, Q4 = 0x1.0cfca86e65239p-18,
               Q5 = -0x1.afdb76e09c32dp-23;
  uint32_t hx = high_word(x);
  const uint32_t xsb = hx & 0x80000000u;
  hx &= 0x7fffffffu;
  double hi, lo, c = 0.0, t;
  int k;
  if (hx >= 0x4043687Au) {
    if (hx >= 0x40862E42u) {
      if (hx >= 0x7ff00000u) {
        if (((hx & 0xfffff) | low_word(x)) != 0) return x + x;
        return xsb == 0 ? x : -1.0;
      }
      if (x > o_threshold) return 1e300 * 1e300;
    }
    if (xsb != 0) return 1e-300 - 1.0;
  }
  if (hx > 0x3fd62e42u) {
    if (hx < 0x3FF0A2B2u) {
      if (xsb == 0) {
        hi = x - ln2_hi;
        lo = ln2_lo;
        k = 1;
      } else {
        hi = x + ln2_hi;
        lo = -ln2_lo;
        k = -1;
      }
    } else {
      k = (int)(invln2 * x + (xsb == 0 ? 0.5 : -0.5));
      t = (double)k;
      hi = fma(-t, ln2_hi, x); /* fused in __expm1_fma */
      lo = t * ln2_lo;
    }
    x = hi - lo;
    c = (hi - x) - lo;
  } else if (hx < 0x3c900000u) {
    t = 1e300 + x;
    return x - (t - (1e300 + x));
  } else {
    k = 0;
  }
  const double hfx = x * 0.5;
  const double hxs = x * hfx;
  const double R1 = fma(hxs, Q1, 1.0);
  const double R2 = fma(hxs, Q3, Q2);
  const double R3 = fma(hxs, Q5, Q4);
  const double h2 = hxs * hxs;
  const double h4 = h2 * h2;
  const double r1 = fma(h4, R3, fma(h2, R2, R1));
  t = fma(-r1, hfx, 3.0);
  double e = ((r1 - t) / fma(-x, t, 6.0)) * hxs;
  if (k == 0) return x - fma(e, x, -hxs);
  e = fma(e - c, x, -c);
  e -= hxs;
  if (k == -1) return fma(0.5, x - e, -0.5);
  if (k == 1) {
    if (x < -0.25) return (e - (x + 0.5)) * -2.0;
    return fma(x - e, 2.0, 1.0);
  }
  double y;
  if (k <= -2 || k > 56) {
    y = 1.0 - (e - x);
    y = with_high(y, high_word(y) + ((uint32_t)k << 20));
    return y - 1.0;
  }
  if (k < 20) {
    t = with_high(0.0, 0x3ff00000u - (0x200000u >> k));
    y = t - (e - x);
  } else {
    t = with_high(0.0, (uint32_t)(0x3ff - k) << 20);
    y = (x - (e + t)) + 1.0;
  }
  return with_high(y, high_word(y) + ((uint32_t)k << 20));
}

double orc_tanh_glibc_fma(double x) {
  const uint32_t jx = high_word(x), ix = jx & 0x7fffffffu;
  if (ix >= 0x7ff00000u) {
    if (jx & 0x80000000u) return 1.0 / x - 1.0;
    return 1.0 / x + 1.0;
  }
  double z;
  if (ix < 0x40360000u) { /* |x| < 22 */
    if ((ix | low_word(x)) == 0) return x;
    if (ix < 0x3c800000u) return x * (1.0 + x);
    const double ax = fabs(x);
    if (ix >= 0x3ff00000u) {
      const double t = orc_expm1_glibc_fma(ax + ax);
      z = 1.0 - 2.0 / (t + 2.0);
    } else {
      const double t = orc_expm1_glibc_fma(-2.0 * ax);
      z = -t / (t + 2.0);
    }
  } else {
    z = 1.0 - 1e-300;
  }
  return (jx & 0x80000000u) ? -z : z;
}

/* narx_init, predictor.cpp:35-44 */
void orc_narx_init(uint64_t seed, lbbsp_narx_model* m) {
  mt64 g;
  mt64_seed(&g, orc_mix_seed2(seed, 0x9a4c0ull));
  memset(m, 0, sizeof *m);
  for (int j = 0; j < 8; ++j) m->input_weights[j] = rng_uniform2(&g, -0.3, 0.3);
  m->hidden_bias = rng_uniform2(&g, -0.1, 0.1);
  m->output_weight = rng_uniform2(&g, -0.3, 0.3);
  m->output_bias = 0.0;
  m->speed_mean = m->cpu_mean = m->mem_mean = 0.0;
  m->speed_stddev = m->cpu_stddev = m->mem_stddev = 1.0;
}

/* standardize, predictor.cpp:52-60 */
static void standardize(const lbbsp_narx_model* m, const double* v, const double* c,
                        const double* mm, double* z) {
  z[0] = (v[0] - m->speed_mean) / m->speed_stddev;
  z[1] = (v[1] - m->speed_mean) / m->speed_stddev;
  for (int j = 0; j < 3; ++j) z[2 + j] = (c[j] - m->cpu_mean) / m->cpu_stddev;
  for (int j = 0; j < 3; ++j) z[5 + j] = (mm[j] - m->mem_mean) / m->mem_stddev;
}

/* forward, predictor.cpp:62-69 */
static double forward(const lbbsp_narx_model* m, const double* z, double* hidden) {
  double a = m->hidden_bias;
  for (int j = 0; j < 8; ++j) a += m->input_weights[j] * z[j];
  const double h = tanh(a);
  if (hidden) *hidden = h;
  return m->output_weight * h + m->output_bias;
}

/* narx_predict, predictor.cpp:147-153 */
double orc_narx_predict(const lbbsp_narx_model* m, const double* v, const double* c,
                        const double* mm, double floor_) {
  double z[8];
  standardize(m, v, c, mm, z);
  const double out = m->speed_mean + m->speed_stddev * forward(m, z, NULL);
  return out > floor_ ? out : floor_;
}

/* fit_scaler, predictor.cpp:71-82 */
static void fit_scaler(const double* xs, int n, double* mean, double* stddev) {
  *mean = 0.0;
  *stddev = 1.0;
  if (n == 0) return;
  double sum = 0.0;
  for (int i = 0; i < n; ++i) sum += xs[i];
  *mean = sum / (double)n;
  double var = 0.0;
  for (int i = 0; i < n; ++i) var += (xs[i] - *mean) * (xs[i] - *mean);
  var /= (double)n;
  *stddev = var > 1e-18 ? sqrt(var) : 1.0;
}

typedef struct {
  double w[8], hb, ow, ob;
} narx_w;

static void get_w(const lbbsp_narx_model* m, narx_w* w) {
  memcpy(w->w, m->input_weights, sizeof w->w);
  w->hb = m->hidden_bias;
  w->ow = m->output_weight;
  w->ob = m->output_bias;
}
static void put_w(lbbsp_narx_model* m, const narx_w* w) {
  memcpy(m->input_weights, w->w, sizeof w->w);
  m->hidden_bias = w->hb;
  m->output_weight = w->ow;
  m->output_bias = w->ob;
}

static double fwd_w(const narx_w* w, const double* z, double* hidden) {
  double a = w->hb;
  for (int j = 0; j < 8; ++j) a += w->w[j] * z[j];
  const double h = tanh(a);
  if (hidden) *hidden = h;
  return w->ow * h + w->ob;
}

/* mse, predictor.cpp:102-109 */
long long orc_debug_evals = 0; /* test instrumentation: objective evaluations */
static double mse(const narx_w* w, const double* Z, const double* T, int cnt) {
  orc_debug_evals += 1;
  double total = 0.0;
  for (int i = 0; i < cnt; ++i) {
    const double e = fwd_w(w, Z + 8 * i, NULL) - T[i];
    total += e * e;
  }
  return total / (double)cnt;
}

/* narx_train_online, predictor.cpp:155-196 (with build_training_set :89-100,
 * loss_gradient :118-134, apply_step :136-143) */
int orc_narx_train(lbbsp_narx_model* m, const double* v, const double* c, const double* mm,
                   int len, const lbbsp_narx_train_cfg* cfg, lbbsp_narx_report* rep,
                   double* loss_log, int loss_cap) {
  rep->ran = 0;
  rep->epochs = 0;
  rep->final_loss = 0.0;
  const int minh = cfg->min_history > 3 ? cfg->min_history : 3;
  if (len < minh) return 0;
  fit_scaler(v, len, &m->speed_mean, &m->speed_stddev);
  fit_scaler(c, len, &m->cpu_mean, &m->cpu_stddev);
  fit_scaler(mm, len, &m->mem_mean, &m->mem_stddev);
  const int cnt = len - 2;
  double* Z = (double*)malloc(sizeof(double) * 8 * (size_t)cnt);
  double* T = (double*)malloc(sizeof(double) * (size_t)cnt);
  for (int t = 2; t < len; ++t) {
    const double vv[2] = {v[t - 1], v[t - 2]};
    const double cc[3] = {c[t], c[t - 1], c[t - 2]};
    const double m3[3] = {mm[t], mm[t - 1], mm[t - 2]};
    standardize(m, vv, cc, m3, Z + 8 * (t - 2));
    T[t - 2] = (v[t] - m->speed_mean) / m->speed_stddev;
  }
  narx_w w;
  get_w(m, &w);
  double current = mse(&w, Z, T, cnt);
  int stall = 0;
  rep->ran = 1;
  for (int epoch = 0; epoch < cfg->max_epochs; ++epoch) {
    narx_w g;
    memset(&g, 0, sizeof g);
    const double scale = 2.0 / (double)cnt;
    for (int i = 0; i < cnt; ++i) {
      double h = 0.0;
      const double y = fwd_w(&w, Z + 8 * i, &h);
      const double dy = scale * (y - T[i]);
      g.ow += dy * h;
      g.ob += dy;
      const double dz = dy * w.ow * (1.0 - h * h);
      for (int j = 0; j < 8; ++j) g.w[j] += dz * Z[8 * i + j];
      g.hb += dz;
    }
    double step = cfg->step;
    narx_w trial;
#define APPLY_STEP(dst, src, s)                                      \
  do {                                                               \
    dst = src;                                                       \
    for (int j = 0; j < 8; ++j) dst.w[j] -= (s) * g.w[j];            \
    dst.hb -= (s) * g.hb;                                            \
    dst.ow -= (s) * g.ow;                                            \
    dst.ob -= (s) * g.ob;                                            \
  } while (0)
    APPLY_STEP(trial, w, step);
    double next = mse(&trial, Z, T, cnt);
    int halvings = 0;
    while (next > current && halvings < 20) {
      step *= 0.5;
      APPLY_STEP(trial, w, step);
      next = mse(&trial, Z, T, cnt);
      ++halvings;
    }
#undef APPLY_STEP
    if (next > current) break;
    w = trial;
    if (loss_log && rep->epochs < loss_cap) loss_log[rep->epochs] = next;
    ++rep->epochs;
    stall = (current - next < cfg->early_stop_delta) ? stall + 1 : 0;
    current = next;
    if (stall >= cfg->early_stop_patience) break;
  }
  rep->final_loss = current;
  put_w(m, &w);
  free(Z);
  free(T);
  return 0;
}

/* ---------------------------------------------------------------------- */
/* sgd.cpp + coordination.cpp                                               */
/* ---------------------------------------------------------------------- */

static double dotd(const double* a, const double* b, int d) { /* sgd.cpp:14-18 */
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += a[i] * b[i];
  return s;
}
static double log1p_exp(double z) { /* sgd.cpp:20-24 */
  if (z > 0) return z + log1p(exp(-z));
  return log1p(exp(z));
}
static double sigmoid(double z) { /* sgd.cpp:26-30 */
  if (z >= 0) return 1.0 / (1.0 + exp(-z));
  const double e = exp(z);
  return e / (1.0 + e);
}

/* separator_params + generate_dataset, sgd.cpp:32-57 */
int orc_generate_dataset(uint64_t seed, int n, int d, double noise, double* feat, double* labels) {
  if (n < 1) return err(LBBSP_INVALID_ARGUMENT, "generate_dataset: n must be >= 1");
  if (d < 1) return err(LBBSP_INVALID_ARGUMENT, "generate_dataset: d must be >= 1");
  double* truth = (double*)malloc(sizeof(double) * (size_t)d);
  mt64 g;
  mt64_seed(&g, orc_mix_seed2(seed, 0x5e9a7a70ull));
  for (int j = 0; j < d; ++j) truth[j] = rng_uniform2(&g, -1.0, 1.0);
  mt64_seed(&g, orc_mix_seed2(seed, 0xda7a5e7ull));
  for (int i = 0; i < n; ++i) {
    double* x = feat + (size_t)i * d;
    for (int j = 0; j < d; ++j) x[j] = rng_uniform2(&g, -1.0, 1.0);
    const double margin = dotd(truth, x, d) + rng_uniform2(&g, -noise, noise);
    labels[i] = margin > 0.0 ? 1.0 : 0.0;
  }
  free(truth);
  return 0;
}

/* batch_gradient, sgd.cpp:72-90 */
int orc_batch_gradient(const double* feat, const double* labels, int n, int d,
                       const double* params, const int* idx, int count, double* out) {
  if (count <= 0) return err(LBBSP_INVALID_ARGUMENT, "batch_gradient: empty index set");
  for (int j = 0; j < d; ++j) out[j] = 0.0;
  for (int s = 0; s < count; ++s) {
    const int i = idx[s];
    if (i < 0 || i >= n) return err(LBBSP_OUT_OF_RANGE, "batch_gradient: sample index out of range");
    const double* x = feat + (size_t)i * d;
    const double z = dotd(params, x, d);
    const double coeff = sigmoid(z) - labels[i];
    for (int j = 0; j < d; ++j) out[j] += coeff * x[j];
  }
  const double inv = 1.0 / (double)count;
  for (int j = 0; j < d; ++j) out[j] *= inv;
  return 0;
}

/* loss, sgd.cpp:65-70 (sample_loss :59-63) */
int orc_loss(const double* feat, const double* labels, int n, int d, const double* params,
             double* out) {
  if (n <= 0) return err(LBBSP_INVALID_ARGUMENT, "loss: empty dataset");
  double total = 0.0;
  for (int i = 0; i < n; ++i) {
    const double z = dotd(params, feat + (size_t)i * d, d);
    total += log1p_exp(z) - labels[i] * z;
  }
  *out = total / (double)n;
  return 0;
}

/* aggregate_weighted (coordination.cpp:52-68) / aggregate_naive (:39-50) */
int orc_aggregate(const double* grads, const int* sizes, int n, int dim, int weighted, double* out) {
  if (n <= 0) return err(LBBSP_INVALID_ARGUMENT, "aggregate: empty gradient list");
  for (int j = 0; j < dim; ++j) out[j] = 0.0;
  if (weighted) {
    double total = 0.0;
    for (int i = 0; i < n; ++i) {
      if (sizes[i] < 1) return err(LBBSP_INVALID_ARGUMENT, "aggregate_weighted: batch size must be >= 1");
      total += (double)sizes[i];
    }
    for (int i = 0; i < n; ++i) {
      const double w = (double)sizes[i] / total;
      for (int j = 0; j < dim; ++j) out[j] += w * grads[(size_t)i * dim + j];
    }
  } else {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < dim; ++j) out[j] += grads[(size_t)i * dim + j];
    const double inv = 1.0 / (double)n;
    for (int j = 0; j < dim; ++j) out[j] *= inv;
  }
  return 0;
}

/* ---------------------------------------------------------------------- */
/* cluster_sim.cpp                                                          */
/* ---------------------------------------------------------------------- */

typedef struct {
  int iterations, regime_length;
  double hi_lo, hi_hi, lo_lo, lo_hi, spike_mult, spike_prob;
} bench_cfg;

static void bench_default(bench_cfg* b) { /* cluster_sim.hpp:76-83 */
  b->iterations = 1200;
  b->regime_length = 50;
  b->hi_lo = 0.75;
  b->hi_hi = 1.0;
  b->lo_lo = 0.30;
  b->lo_hi = 0.55;
  b->spike_mult = 3.0;
  b->spike_prob = 0.02;
}

/* make_benchmark_series, cluster_sim.cpp:41-64 */
static void benchmark_series(uint64_t seed, const bench_cfg* b, double* cpu, double* mem,
                             double* mult) {
  mt64 rr, sr;
  mt64_seed(&rr, orc_mix_seed2(seed, 0xbe9c0ull));
  mt64_seed(&sr, orc_mix_seed2(seed, 0x59c1ceull));
  const int regimes = (b->iterations + b->regime_length - 1) / b->regime_length;
  const int nl = regimes > 1 ? regimes : 1;
  double* levels = (double*)calloc((size_t)nl, sizeof(double));
  for (int r = 0; r < regimes; ++r)
    levels[r] = (r % 2 == 0) ? rng_uniform2(&rr, b->hi_lo, b->hi_hi) : rng_uniform2(&rr, b->lo_lo, b->lo_hi);
  for (int k = 0; k < b->iterations; ++k) {
    cpu[k] = levels[k / b->regime_length];
    mem[k] = 1.0;
    mult[k] = rng_uniform(&sr) < b->spike_prob ? b->spike_mult : 1.0;
  }
  free(levels);
}

int orc_benchmark_series(uint64_t seed, int iterations, double* cpu, double* mem, double* mult) {
  bench_cfg b;
  bench_default(&b);
  b.iterations = iterations;
  benchmark_series(seed, &b, cpu, mem, mult);
  return 0;
}

/* sample_stream, cluster_sim.cpp:302-307 */
void orc_sample_stream(uint64_t seed, int64_t k, int budget, int dataset_size, int* out) {
  mt64 g;
  mt64_seed(&g, orc_mix_seed3(seed, 0x57e3a9ull, (uint64_t)k));
  for (int i = 0; i < budget; ++i) out[i] = rng_uniform_int(&g, 0, dataset_size - 1);
}

typedef struct {
  int kind; /* LBBSP_DYN_* */
  int n;
  double *static_cpu, *static_mem; /* may be NULL */
  lbbsp_straggler* strag;          /* [n] */
  double* phase;                   /* [n] */
  int bench_len;
  double *bcpu, *bmem, *bmult;     /* [n*bench_len] */
  const int* trace_off;            /* [n+1] (Trace) */
  const double *trace_t, *trace_c, *trace_m;
} dynamics;

/* load_narx_csv, predictor.cpp:215-243: "name,value" rows, any order. */
int orc_narx_load_csv(const char* path, lbbsp_narx_model* out) {
  static const char* names[17] = {"input_weight_0", "input_weight_1", "input_weight_2",
                                  "input_weight_3", "input_weight_4", "input_weight_5",
                                  "input_weight_6", "input_weight_7", "hidden_bias",
                                  "output_weight",  "output_bias",    "speed_mean",
                                  "speed_stddev",   "cpu_mean",       "cpu_stddev",
                                  "mem_mean",       "mem_stddev"};
  double vals[17];
  int have[17] = {0};
  FILE* f = fopen(path, "r");
  if (!f) return err(LBBSP_RUNTIME, "load_narx_csv: cannot open %s", path);
  char line[512];
  while (fgets(line, sizeof line, f)) {
    size_t L = strlen(line);
    if (L && line[L - 1] == '\n') line[--L] = 0;
    if (!L) continue;
    char* comma = strchr(line, ',');
    if (!comma) {
      fclose(f);
      return err(LBBSP_RUNTIME, "load_narx_csv: malformed row '%s'", line);
    }
    *comma = 0;
    for (int j = 0; j < 17; ++j)
      if (!strcmp(line, names[j])) {
        vals[j] = strtod(comma + 1, NULL);
        have[j] = 1;
      }
  }
  fclose(f);
  for (int j = 0; j < 17; ++j)
    if (!have[j]) return err(LBBSP_RUNTIME, "load_narx_csv: missing parameter '%s'", names[j]);
  for (int j = 0; j < 8; ++j) out->input_weights[j] = vals[j];
  out->hidden_bias = vals[8];
  out->output_weight = vals[9];
  out->output_bias = vals[10];
  out->speed_mean = vals[11];
  out->speed_stddev = vals[12];
  out->cpu_mean = vals[13];
  out->cpu_stddev = vals[14];
  out->mem_mean = vals[15];
  out->mem_stddev = vals[16];
  return LBBSP_OK;
}

/* Dynamics::at, cluster_sim.cpp:77-118 -> (cpu, mem, mult) */
static void dyn_at(const dynamics* D, int w, int64_t k, double now, double* c, double* m,
                   double* mult) {
  *c = 1.0;
  *m = 1.0;
  *mult = 1.0;
  switch (D->kind) {
    case LBBSP_DYN_STATIC:
      if (D->static_cpu) *c = D->static_cpu[w];
      if (D->static_mem) *m = D->static_mem[w];
      return;
    case LBBSP_DYN_STRAGGLER: {
      if (!D->strag) return;
      const lbbsp_straggler* s = &D->strag[w];
      if (s->on_probability <= 0.0) return;
      const double q = (double)(k / (s->period > 1 ? s->period : 1));
      const double ph = D->phase[w];
      const int on = floor((q + 1.0 + ph) * s->on_probability) > floor((q + ph) * s->on_probability);
      if (on) {
        *c = 1.0 - s->cpu_consumed;
        *m = 1.0 - s->mem_consumed;
      }
      return;
    }
    case LBBSP_DYN_BENCHMARK: {
      const int64_t idx = k < D->bench_len - 1 ? k : D->bench_len - 1;
      *c = D->bcpu[(size_t)w * D->bench_len + idx];
      *m = D->bmem[(size_t)w * D->bench_len + idx];
      *mult = D->bmult[(size_t)w * D->bench_len + idx];
      return;
    }
    case LBBSP_DYN_TRACE: { /* trace_at, trace.cpp:137-143: latest point at or before now */
      const int lo = D->trace_off[w], hi = D->trace_off[w + 1];
      int p = lo;
      for (int q = lo; q < hi; ++q)
        if (D->trace_t[q] <= now) p = q;
        else break;
      *c = D->trace_c[p];
      *m = D->trace_m[p];
      return;
    }
  }
}

/* equal_split, cluster_sim.cpp:209-213 */
static void equal_split(int total, int n, int* out) {
  for (int i = 0; i < n; ++i) out[i] = total / n + (i < total % n ? 1 : 0);
}

/* MemPenalty + effective_speed, cluster_sim.cpp:22-29 */
static double effective_speed(double base, double c, double m) {
  const double pen = m >= 0.5 ? 1.0 : 0.25 + (1.0 - 0.25) * (m / 0.5);
  return base * c * pen;
}

typedef struct {
  double *v, *c, *m, *comm;
  int len;
  lbbsp_narx_model model;
} worker_rt;

/* SpeedPredictor::predict, predictor.cpp:271-292 */
static double predictor_predict(const lbbsp_predictor_cfg* pc, const worker_rt* rt, double c_now,
                                double m_now) {
  double e = 0.0;
  switch (pc->kind) {
    case LBBSP_PRED_MEMORYLESS:
      return rt->v[rt->len - 1];
    case LBBSP_PRED_PERFECT:
    case LBBSP_PRED_EMA:
      orc_ema(rt->v, rt->len, pc->alpha, &e);
      return e;
    default: {
      const int k = rt->len;
      if (k < pc->warmup_iterations || k < 2) {
        orc_ema(rt->v, rt->len, pc->alpha, &e);
        return e;
      }
      const double vv[2] = {rt->v[k - 1], rt->v[k - 2]};
      const double cc[3] = {c_now, rt->c[k - 1], rt->c[k - 2]};
      const double mm[3] = {m_now, rt->m[k - 1], rt->m[k - 2]};
      return orc_narx_predict(&rt->model, vv, cc, mm, pc->speed_floor);
    }
  }
}

static void predictor_train(const lbbsp_predictor_cfg* pc, worker_rt* rt) {
  if (pc->kind != LBBSP_PRED_NARX) return;
  lbbsp_narx_train_cfg tc = pc->train;
  tc.min_history = pc->warmup_iterations; /* predictor.cpp:264 */
  lbbsp_narx_report rep;
  orc_narx_train(&rt->model, rt->v, rt->c, rt->m, rt->len, &tc, &rep, NULL, 0);
}

/* ---- ASP / SSP: Simulation::step_async (cluster_sim.cpp:486-631) ---------- */
typedef struct {
  const lbbsp_sim_cfg* c;
  int n, B, d, N;
  const double *feat, *lab;
  double* params;
  const int* equal;
  const dynamics* D;
  worker_rt* W;
  int gpu_mode;
} async_ctx;

typedef struct {
  int64_t completed;
  int running, blocked;
  double block_start, pending_wait, finish;
  double* grad;          /* inflight gradient [d] */
  double st[6];          /* x, tp, tm, wait, v_pred, v_act */
  double c, m;           /* inflight resource state */
} async_rt;

/* start_worker, cluster_sim.cpp:504-536 */
static int async_start(const async_ctx* A, async_rt* R, int w, double now, int* stream) {
  const lbbsp_sim_cfg* c = A->c;
  async_rt* rt = &R[w];
  const int64_t j = rt->completed;
  double cc, mm, mult;
  dyn_at(A->D, w, j, now, &cc, &mm, &mult);
  const int x = A->equal[w];
  double tp, va, vp = 0.0;
  if (A->gpu_mode) {
    const lbbsp_gpu_profile* g = &c->gpu_profiles[w];
    if (x > g->oom_point) return err(LBBSP_RUNTIME, "gpu out of memory: batch %d exceeds oom point %d", x, g->oom_point);
    tp = g->sec_per_sample * (double)(x > g->saturation_point ? x : g->saturation_point) + g->base_time_s;
    va = (double)x / tp;
  } else {
    va = effective_speed(c->base_speed, cc, mm) * mult;
    tp = (double)x / va;
    if (A->W[w].len >= 1)
      vp = c->predictor.kind == LBBSP_PRED_PERFECT ? va : predictor_predict(&c->predictor, &A->W[w], cc, mm);
  }
  const double f = (c->bw_worker == w && c->bw_at_iteration <= j) ? c->bw_factor : 1.0;
  const double tm = c->base_comm_s * f;
  orc_sample_stream(c->seed, j, A->B, A->N, stream);
  int off = 0;
  for (int i = 0; i < w; ++i) off += A->equal[i];
  int st = orc_batch_gradient(A->feat, A->lab, A->N, A->d, A->params, stream + off, x, rt->grad);
  if (st) return st;
  rt->st[0] = x;
  rt->st[1] = tp;
  rt->st[2] = tm;
  rt->st[3] = rt->pending_wait;
  rt->st[4] = vp;
  rt->st[5] = va;
  rt->c = cc;
  rt->m = mm;
  rt->pending_wait = 0.0;
  rt->running = 1;
  rt->finish = now + tp + tm;
  return 0;
}

static int64_t min_completed(const async_rt* R, int n) {
  int64_t lo = INT64_MAX;
  for (int i = 0; i < n; ++i) lo = R[i].completed < lo ? R[i].completed : lo;
  return lo;
}

static int async_run(const async_ctx* A, int max_rows, int* count_o, lbbsp_iter_scalars* sc,
                     int* batch_o, double* tp_o, double* tm_o, double* wait_o, double* vpred_o,
                     double* vact_o, double* params_o, int* converged_o, int* worker_o, int* nw_o) {
  const lbbsp_sim_cfg* c = A->c;
  const int n = A->n, d = A->d, ssp = c->scheme == LBBSP_SCHEME_SSP;
  const int64_t stale = c->staleness_threshold;
  const int ring = c->staleness_threshold + 3;
  async_rt* R = (async_rt*)calloc((size_t)n, sizeof(async_rt));
  for (int i = 0; i < n; ++i) R[i].grad = (double*)calloc((size_t)d, sizeof(double));
  double* rg = (double*)calloc((size_t)ring * n * d, sizeof(double));
  double* rs = (double*)calloc((size_t)ring * n * 6, sizeof(double));
  int* rcount = (int*)calloc((size_t)ring, sizeof(int));
  int* stream = (int*)malloc(sizeof(int) * (size_t)A->B);
  double* agg = (double*)malloc(sizeof(double) * (size_t)d);
  int* one = (int*)malloc(sizeof(int));
  double now = 0.0, last_update = 0.0;
  int64_t clock = 0;
  int st = 0, count = 0, below = 0, converged = 0;
  for (int i = 0; i < n && !st; ++i) st = async_start(A, R, i, 0.0, stream); /* ctor (:293-294) */
  while (!st) {
    int next = -1; /* earliest finish, ties to the lowest id */
    for (int i = 0; i < n; ++i) {
      if (!R[i].running) continue;
      if (next < 0 || R[i].finish < R[next].finish) next = i;
    }
    if (next < 0) break;
    async_rt* rt = &R[next];
    worker_rt* W = &A->W[next];
    now = rt->finish;
    rt->running = 0;
    rt->completed += 1;
    W->v[W->len] = rt->st[5]; /* observe (:309-313) */
    W->c[W->len] = rt->c;
    W->m[W->len] = rt->m;
    W->comm[W->len] = rt->st[2];
    W->len += 1;
    predictor_train(&c->predictor, W);
    int rec = 0, slot = 0, nw = 0;
    double lossv = 0.0;
    const double* g_src = NULL;
    if (!ssp) {
      *one = (int)rt->st[0];
      orc_aggregate(rt->grad, one, 1, d, 0, agg);
      g_src = agg;
      nw = 1;
      rec = 1;
    } else {
      slot = (int)((rt->completed - 1) % ring);
      memcpy(rg + ((size_t)slot * n + next) * d, rt->grad, sizeof(double) * d);
      memcpy(rs + ((size_t)slot * n + next) * 6, rt->st, sizeof rt->st);
      if (++rcount[slot] == n) {
        orc_aggregate(rg + (size_t)slot * n * d, A->equal, n, d, 0, agg);
        g_src = agg;
        nw = n;
        rec = 1;
      }
    }
    if (rec) {
      for (int j = 0; j < d; ++j) A->params[j] -= c->learning_rate * g_src[j]; /* apply_update */
      clock += 1;
      double nrm = 0.0;
      for (int j = 0; j < d; ++j) nrm += g_src[j] * g_src[j];
      nrm = sqrt(nrm);
      orc_loss(A->feat, A->lab, A->N, d, A->params, &lossv);
      if (count < max_rows) {
        if (sc) {
          sc[count].k = clock - 1;
          sc[count].grad_norm = nrm;
          sc[count].loss = lossv;
          sc[count].wall_s = now - last_update;
        }
        if (nw_o) nw_o[count] = nw;
        for (int i = 0; i < nw; ++i) {
          const size_t o = (size_t)count * n + i;
          const int wid = ssp ? i : next;
          const double* sv = ssp ? rs + ((size_t)slot * n + i) * 6 : rt->st;
          if (worker_o) worker_o[o] = wid;
          if (batch_o) batch_o[o] = (int)sv[0];
          if (tp_o) tp_o[o] = sv[1];
          if (tm_o) tm_o[o] = sv[2];
          if (wait_o) wait_o[o] = sv[3];
          if (vpred_o) vpred_o[o] = sv[4];
          if (vact_o) vact_o[o] = sv[5];
        }
        if (params_o) memcpy(params_o + (size_t)count * d, A->params, sizeof(double) * d);
      }
      last_update = now;
      if (ssp) rcount[slot] = 0;
    }
    /* restart or park the finisher, then re-check the blocked workers */
    if (!ssp) {
      st = async_start(A, R, next, now, stream);
    } else {
      if (rt->completed - min_completed(R, n) <= stale) {
        st = async_start(A, R, next, now, stream);
      } else {
        rt->blocked = 1;
        rt->block_start = now;
      }
      for (int i = 0; i < n && !st; ++i) {
        if (!R[i].blocked) continue;
        if (R[i].completed - min_completed(R, n) <= stale) {
          R[i].blocked = 0;
          R[i].pending_wait = now - R[i].block_start;
          st = async_start(A, R, i, now, stream);
        }
      }
    }
    if (rec) { /* check_stop (:326-334) */
      ++count;
      below = lossv < c->convergence_loss ? below + 1 : 0;
      if (below >= c->convergence_consecutive) {
        converged = 1;
        break;
      }
      if (count >= c->max_updates) break;
    }
  }
  *count_o = count;
  *converged_o = converged;
  for (int i = 0; i < n; ++i) free(R[i].grad);
  free(R); free(rg); free(rs); free(rcount); free(stream); free(agg); free(one);
  return st;
}

/* Simulation ctor (cluster_sim.cpp:247-296) + run (:633-643) + step_sync
 * (:349-469) for the BSP / LB-BSP schemes. */
int orc_sim_run(const lbbsp_sim_cfg* c, int max_rows, int* rows, lbbsp_iter_scalars* sc,
                int* batch_o, double* tp_o, double* tm_o, double* wait_o, double* vpred_o,
                double* vact_o, double* params_o, int* converged_o, int* worker_o,
                int* nw_o) {
  const int n = c->n_workers;
  const int B = c->total_budget;
  const int gpu_mode = c->gpu_profiles != NULL;
  if (n < 1) return err(LBBSP_INVALID_ARGUMENT, "simulation: need at least one worker");
  if (B < n) return err(LBBSP_INVALID_ARGUMENT, "simulation: total_budget below worker count");
  if (c->scheme < LBBSP_SCHEME_BSP || c->scheme > LBBSP_SCHEME_LBBSP)
    return err(LBBSP_INVALID_ARGUMENT, "simulation: unknown scheme %d", c->scheme);
  if (c->staleness_threshold < 0)
    return err(LBBSP_INVALID_ARGUMENT, "simulation: staleness_threshold must be >= 0");
  const int async = c->scheme == LBBSP_SCHEME_ASP || c->scheme == LBBSP_SCHEME_SSP;
  if (c->scheme != LBBSP_SCHEME_LBBSP && B % n != 0)
    return err(LBBSP_INVALID_ARGUMENT,
               "simulation: bsp/asp/ssp need total_budget divisible by workers");
  int* equal = (int*)malloc(sizeof(int) * (size_t)n);
  equal_split(B, n, equal);
  int st = 0;
  if (gpu_mode) {
    for (int i = 0; i < n; ++i)
      if (c->scheme != LBBSP_SCHEME_LBBSP && equal[i] > c->gpu_profiles[i].oom_point) {
        free(equal);
        return err(LBBSP_INVALID_ARGUMENT, "simulation: equal split exceeds oom point of worker %d", i);
      }
    if (c->scheme == LBBSP_SCHEME_LBBSP) {
      double* zeros = (double*)calloc((size_t)n, sizeof(double));
      int* tmp = (int*)malloc(sizeof(int) * (size_t)n);
      st = orc_gpu_allocate(c->gpu_profiles, zeros, n, B, tmp);
      free(zeros);
      free(tmp);
      if (st) {
        free(equal);
        return st;
      }
    }
  }
  /* dataset + model (cluster_sim.cpp:285-288) */
  const int N = c->dataset_size, d = c->dataset_dim;
  double* feat = (double*)malloc(sizeof(double) * (size_t)N * d);
  double* lab = (double*)malloc(sizeof(double) * (size_t)N);
  st = orc_generate_dataset(c->dataset_seed, N, d, c->dataset_noise, feat, lab);
  if (st) {
    free(equal);
    free(feat);
    free(lab);
    return st;
  }
  double* params = (double*)calloc((size_t)d, sizeof(double));

  /* dynamics (preset or explicit) */
  dynamics D;
  memset(&D, 0, sizeof D);
  D.n = n;
  double* pre_cpu = NULL;
  lbbsp_straggler* pre_strag = NULL;
  if (gpu_mode) {
    D.kind = LBBSP_DYN_STATIC;
  } else if (c->preset != LBBSP_PRESET_NONE) { /* heterogeneity_preset, cluster_sim.cpp:140-197 */
    if (n < 2) {
      free(equal); free(feat); free(lab); free(params);
      return err(LBBSP_INVALID_ARGUMENT, "heterogeneity_preset: need n >= 2");
    }
    const double ratio = c->preset == LBBSP_PRESET_HOMO ? 1.0
                         : (c->preset == LBBSP_PRESET_HETERO_L2 || c->preset == LBBSP_PRESET_HETERO_L2_STATIC)
                             ? 0.5
                             : 1.0 / 3.0;
    if (c->preset == LBBSP_PRESET_HOMO) {
      D.kind = LBBSP_DYN_STATIC;
      pre_cpu = (double*)malloc(sizeof(double) * (size_t)n);
      for (int i = 0; i < n; ++i) pre_cpu[i] = 1.0;
      D.static_cpu = pre_cpu;
    } else if (c->preset == LBBSP_PRESET_HETERO_L2_STATIC || c->preset == LBBSP_PRESET_HETERO_L3_STATIC) {
      D.kind = LBBSP_DYN_STATIC;
      pre_cpu = (double*)malloc(sizeof(double) * (size_t)n);
      for (int i = 0; i < n; ++i) pre_cpu[i] = 1.0 - (1.0 - ratio) * (double)i / (double)(n - 1);
      D.static_cpu = pre_cpu;
    } else {
      D.kind = LBBSP_DYN_STRAGGLER;
      pre_strag = (lbbsp_straggler*)calloc((size_t)n, sizeof(lbbsp_straggler));
      for (int i = 0; i < n; ++i) {
        pre_strag[i].period = 10;
        if (i > 0) {
          const double avg = 1.0 - (1.0 - ratio) * (double)i / (double)(n - 1);
          pre_strag[i].on_probability = 0.75;
          pre_strag[i].cpu_consumed = (1.0 - avg) / 0.75;
          pre_strag[i].period = 10;
        }
      }
      D.strag = pre_strag;
    }
  } else {
    D.kind = c->dynamics;
    D.static_cpu = (double*)c->static_cpu;
    D.static_mem = (double*)c->static_mem;
    D.strag = (lbbsp_straggler*)c->stragglers;
    D.trace_off = c->trace_offsets;
    D.trace_t = c->trace_t;
    D.trace_c = c->trace_cpu;
    D.trace_m = c->trace_mem;
  }
  D.phase = (double*)malloc(sizeof(double) * (size_t)n); /* Dynamics ctor, cluster_sim.cpp:66-75 */
  for (int i = 0; i < n; ++i) {
    mt64 g;
    mt64_seed(&g, orc_mix_seed3(c->seed, 0x477a5eull, (uint64_t)i));
    D.phase[i] = rng_uniform(&g);
  }
  if (D.kind == LBBSP_DYN_BENCHMARK) {
    bench_cfg bc = {c->bench_iterations, c->bench_regime_length, c->bench_high_lo, c->bench_high_hi,
                    c->bench_low_lo,     c->bench_low_hi,        c->bench_spike_mult, c->bench_spike_prob};
    D.bench_len = bc.iterations;
    D.bcpu = (double*)malloc(sizeof(double) * (size_t)n * bc.iterations);
    D.bmem = (double*)malloc(sizeof(double) * (size_t)n * bc.iterations);
    D.bmult = (double*)malloc(sizeof(double) * (size_t)n * bc.iterations);
    for (int i = 0; i < n; ++i)
      benchmark_series(orc_mix_seed3(c->seed, 0xbe7cull, (uint64_t)i), &bc, D.bcpu + (size_t)i * bc.iterations,
                       D.bmem + (size_t)i * bc.iterations, D.bmult + (size_t)i * bc.iterations);
  }

  const int64_t cap = (c->max_updates > 0 ? c->max_updates : 1) + (async ? c->staleness_threshold + 2 : 0);
  lbbsp_narx_model initial; /* PredictorConfig::initial_weights (predictor.cpp:265-266) */
  const int have_initial = c->narx_weights_path && c->narx_weights_path[0];
  if (have_initial) {
    st = orc_narx_load_csv(c->narx_weights_path, &initial);
    if (st) {
      free(equal); free(feat); free(lab); free(params);
      free(D.phase); free(D.bcpu); free(D.bmem); free(D.bmult); free(pre_cpu); free(pre_strag);
      return st;
    }
  }
  worker_rt* W = (worker_rt*)calloc((size_t)n, sizeof(worker_rt));
  for (int i = 0; i < n; ++i) {
    W[i].v = (double*)malloc(sizeof(double) * (size_t)cap);
    W[i].c = (double*)malloc(sizeof(double) * (size_t)cap);
    W[i].m = (double*)malloc(sizeof(double) * (size_t)cap);
    W[i].comm = (double*)malloc(sizeof(double) * (size_t)cap);
    if (have_initial)
      W[i].model = initial;
    else
      orc_narx_init(orc_mix_seed3(c->seed, 0x9ced1c70ull, (uint64_t)i), &W[i].model);
  }
  double *rc = malloc(sizeof(double) * n), *rm = malloc(sizeof(double) * n), *rmult = malloc(sizeof(double) * n);
  double *vact = malloc(sizeof(double) * n), *vpred = malloc(sizeof(double) * n);
  double *tp = malloc(sizeof(double) * n), *tm = malloc(sizeof(double) * n), *tmhat = malloc(sizeof(double) * n);
  int* sizes = malloc(sizeof(int) * n);
  int* stream = malloc(sizeof(int) * (size_t)B);
  double* grads = malloc(sizeof(double) * (size_t)n * d);
  double* agg = malloc(sizeof(double) * (size_t)d);
  int below = 0, converged = 0, count = 0, cursor = 0;
  double now = 0.0; /* Simulation::now_ */

  if (async) {
    async_ctx A = {c, n, B, d, N, feat, lab, params, equal, &D, W, gpu_mode};
    st = async_run(&A, max_rows, &count, sc, batch_o, tp_o, tm_o, wait_o, vpred_o, vact_o,
                   params_o, &converged, worker_o, nw_o);
  }
  for (int64_t k = 0; !async; ++k) {
    /* P1-P3 (:355-367) */
    for (int i = 0; i < n; ++i) {
      dyn_at(&D, i, k, now, &rc[i], &rm[i], &rmult[i]);
      vact[i] = 0.0;
      vpred[i] = 0.0;
      if (!gpu_mode) {
        vact[i] = effective_speed(c->base_speed, rc[i], rm[i]) * rmult[i];
        if (W[i].len >= 1)
          vpred[i] = c->predictor.kind == LBBSP_PRED_PERFECT ? vact[i]
                                                             : predictor_predict(&c->predictor, &W[i], rc[i], rm[i]);
      }
    }
    /* P4 sizes (:371-402) */
    if (c->scheme == LBBSP_SCHEME_LBBSP) {
      if (gpu_mode) {
        int feasible = 1;
        if (k < 2) { /* initial_gpu_sizes, :471-484 */
          for (int i = 0; i < n; ++i) {
            sizes[i] = equal[i];
            if (equal[i] < c->gpu_profiles[i].saturation_point || equal[i] > c->gpu_profiles[i].oom_point)
              feasible = 0;
          }
          if (!feasible) {
            for (int i = 0; i < n; ++i) tmhat[i] = 0.0;
            st = orc_gpu_allocate(c->gpu_profiles, tmhat, n, B, sizes);
          }
        } else {
          for (int i = 0; i < n; ++i) orc_ema(W[i].comm, W[i].len - 1, c->predictor.alpha, &tmhat[i]);
          st = orc_gpu_allocate(c->gpu_profiles, tmhat, n, B, sizes);
        }
      } else if (k == 0) {
        memcpy(sizes, equal, sizeof(int) * n);
      } else {
        double* sp = malloc(sizeof(double) * n);
        for (int i = 0; i < n; ++i) sp[i] = vpred[i] > c->predictor.speed_floor ? vpred[i] : c->predictor.speed_floor;
        st = orc_cpu_allocate(sp, n, B, sizes);
        free(sp);
      }
      if (st) break;
    } else {
      memcpy(sizes, equal, sizeof(int) * n);
    }
    /* P5 timing (:404-420) */
    double wall = 0.0;
    for (int i = 0; i < n; ++i) {
      const int x = sizes[i];
      if (gpu_mode) {
        const lbbsp_gpu_profile* g = &c->gpu_profiles[i];
        if (x < 1) { st = err(LBBSP_INVALID_ARGUMENT, "gpu_compute_time: batch must be >= 1"); break; }
        if (x > g->oom_point) {
          st = err(LBBSP_RUNTIME, "gpu out of memory: batch %d exceeds oom point %d", x, g->oom_point);
          break;
        }
        tp[i] = g->sec_per_sample * (double)(x > g->saturation_point ? x : g->saturation_point) + g->base_time_s;
        vact[i] = (double)x / tp[i];
      } else {
        tp[i] = (double)x / vact[i];
      }
      double f = 1.0; /* CommModel::tm_at, :13-20 */
      if (c->bw_worker == i && c->bw_at_iteration <= k) f = c->bw_factor;
      tm[i] = c->base_comm_s * f;
      if (tp[i] + tm[i] > wall) wall = tp[i] + tm[i];
    }
    if (st) break;
    /* P6-P8 (:422-439) */
    orc_sample_stream(c->seed, k, B, N, stream);
    int off = 0;
    for (int i = 0; i < n; ++i) {
      st = orc_batch_gradient(feat, lab, N, d, params, stream + off, sizes[i], grads + (size_t)i * d);
      if (st) break;
      off += sizes[i];
    }
    if (st) break;
    orc_aggregate(grads, sizes, n, d, c->scheme == LBBSP_SCHEME_LBBSP, agg);
    for (int j = 0; j < d; ++j) params[j] -= c->learning_rate * agg[j]; /* apply_update sgd.cpp:92-99 */
    /* P9 record (:441-456) */
    double nrm = 0.0;
    for (int j = 0; j < d; ++j) nrm += agg[j] * agg[j];
    nrm = sqrt(nrm);
    double lossv = 0.0;
    orc_loss(feat, lab, N, d, params, &lossv);
    if (count < max_rows) {
      if (sc) {
        sc[count].k = k;
        sc[count].grad_norm = nrm;
        sc[count].loss = lossv;
        sc[count].wall_s = wall;
      }
      for (int i = 0; i < n; ++i) {
        const size_t o = (size_t)count * n + i;
        if (batch_o) batch_o[o] = sizes[i];
        if (tp_o) tp_o[o] = tp[i];
        if (tm_o) tm_o[o] = tm[i];
        if (wait_o) wait_o[o] = wall - tp[i] - tm[i];
        if (vpred_o) vpred_o[o] = vpred[i];
        if (vact_o) vact_o[o] = vact[i];
      }
      if (params_o) memcpy(params_o + (size_t)count * d, params, sizeof(double) * d);
      if (nw_o) nw_o[count] = n;
      if (worker_o)
        for (int i = 0; i < n; ++i) worker_o[(size_t)count * n + i] = i;
    }
    ++count;
    /* P10 observe + train_rotation (:458-464, :309-324) */
    for (int i = 0; i < n; ++i) {
      W[i].v[W[i].len] = vact[i];
      W[i].c[W[i].len] = rc[i];
      W[i].m[W[i].len] = rm[i];
      W[i].comm[W[i].len] = tm[i];
      W[i].len += 1;
    }
    if (c->predictor.kind == LBBSP_PRED_NARX) {
      const int bud = (n + 1) / 2;
      for (int j = 0; j < bud; ++j) predictor_train(&c->predictor, &W[(cursor + j) % n]);
      cursor = (cursor + bud) % n;
    }
    now += wall; /* :466 */
    /* check_stop (:326-334) */
    below = lossv < c->convergence_loss ? below + 1 : 0;
    if (below >= c->convergence_consecutive) {
      converged = 1;
      break;
    }
    if (count >= c->max_updates) break;
  }
  *rows = count < max_rows ? count : max_rows;
  if (converged_o) *converged_o = converged;

  for (int i = 0; i < n; ++i) {
    free(W[i].v); free(W[i].c); free(W[i].m); free(W[i].comm);
  }
  free(W); free(rc); free(rm); free(rmult); free(vact); free(vpred); free(tp); free(tm); free(tmhat);
  free(sizes); free(stream); free(grads); free(agg); free(equal); free(feat); free(lab); free(params);
  free(D.phase); free(D.bcpu); free(D.bmem); free(D.bmult); free(pre_cpu); free(pre_strag);
  return st;
}

/* Replay driver: see oracle/ref_capi.cpp ref_replay_cpu (same contract). */
int orc_replay_cpu(const lbbsp_predictor_cfg* pc, const uint64_t* seeds, int n, int budget,
                   int iters, const double* v_obs, const double* c_obs, const double* m_obs,
                   int* sizes_out, double* v_pred_out) {
  worker_rt* W = (worker_rt*)calloc((size_t)n, sizeof(worker_rt));
  for (int i = 0; i < n; ++i) {
    W[i].v = malloc(sizeof(double) * (size_t)(iters + 1));
    W[i].c = malloc(sizeof(double) * (size_t)(iters + 1));
    W[i].m = malloc(sizeof(double) * (size_t)(iters + 1));
    orc_narx_init(seeds[i], &W[i].model);
  }
  int* equal = malloc(sizeof(int) * n);
  equal_split(budget, n, equal);
  double* vp = malloc(sizeof(double) * n);
  int st = 0, cursor = 0;
  for (int k = 0; k < iters && !st; ++k) {
    for (int i = 0; i < n; ++i) {
      const size_t o = (size_t)k * n + i;
      vp[i] = 0.0;
      if (W[i].len >= 1)
        vp[i] = pc->kind == LBBSP_PRED_PERFECT ? v_obs[o] : predictor_predict(pc, &W[i], c_obs[o], m_obs[o]);
    }
    int* sz = sizes_out + (size_t)k * n;
    if (k == 0) {
      memcpy(sz, equal, sizeof(int) * n);
    } else {
      double* sp = malloc(sizeof(double) * n);
      for (int i = 0; i < n; ++i) sp[i] = vp[i] > pc->speed_floor ? vp[i] : pc->speed_floor;
      st = orc_cpu_allocate(sp, n, budget, sz);
      free(sp);
    }
    for (int i = 0; i < n; ++i) {
      const size_t o = (size_t)k * n + i;
      if (v_pred_out) v_pred_out[o] = vp[i];
      W[i].v[W[i].len] = v_obs[o];
      W[i].c[W[i].len] = c_obs[o];
      W[i].m[W[i].len] = m_obs[o];
      W[i].len += 1;
    }
    if (pc->kind == LBBSP_PRED_NARX) {
      const int bud = (n + 1) / 2;
      for (int j = 0; j < bud; ++j) predictor_train(pc, &W[(cursor + j) % n]);
      cursor = (cursor + bud) % n;
    }
  }
  for (int i = 0; i < n; ++i) {
    free(W[i].v); free(W[i].c); free(W[i].m);
  }
  free(W); free(equal); free(vp);
  return st;
}

/* ---------------------------------------------------------------------- */
/* Generalised NARX (delay d, hidden h) -- the C4 sweep shape. Restates     */
/* predictor.cpp:35-196 with the lag structure and width as parameters:     */
/* inputs {v_{t-1..t-d}, c_{t..t-d}, m_{t..t-d}} (I = 3d+2), h tanh units,   */
/* one linear output. Parameter layout (double[P], P = h*I + 2h + 1 + 6):    */
/*   W1[h][I] | b1[h] | w2[h] | b2 | speed_mean, speed_std, cpu_mean,        */
/*   cpu_std, mem_mean, mem_std.                                             */
/* At (d, h) = (2, 1) every operation and its order equals the reference,    */
/* so results are bit-identical (tests/test_oracle.py pins that).            */
/* ---------------------------------------------------------------------- */
int orc_narxg_param_count(int d, int h) { return h * (3 * d + 2) + 2 * h + 1 + 6; }

/* narx_init generalised (predictor.cpp:35-44): same draw order */
void orc_narxg_init(uint64_t seed, int d, int h, double* p) {
  const int I = 3 * d + 2;
  mt64 g;
  mt64_seed(&g, orc_mix_seed2(seed, 0x9a4c0ull));
  for (int j = 0; j < h * I; ++j) p[j] = rng_uniform2(&g, -0.3, 0.3);
  for (int j = 0; j < h; ++j) p[h * I + j] = rng_uniform2(&g, -0.1, 0.1);
  for (int j = 0; j < h; ++j) p[h * I + h + j] = rng_uniform2(&g, -0.3, 0.3);
  p[h * I + 2 * h] = 0.0;
  double* sc = p + h * I + 2 * h + 1;
  sc[0] = 0.0; sc[1] = 1.0; sc[2] = 0.0; sc[3] = 1.0; sc[4] = 0.0; sc[5] = 1.0;
}

static double narxg_fwd(const double* p, int I, int h, const double* x, double* hid) {
  double y = 0.0;
  for (int j = 0; j < h; ++j) {
    double a = p[h * I + j];                       /* hidden bias */
    for (int i = 0; i < I; ++i) a += p[j * I + i] * x[i];
    const double t = tanh(a);
    if (hid) hid[j] = t;
    y += p[h * I + h + j] * t;                     /* output weight */
  }
  return y + p[h * I + 2 * h];                     /* output bias */
}

static void narxg_inputs(const double* sc, int d, const double* v, const double* c,
                         const double* m, int t, double* x) {
  for (int l = 0; l < d; ++l) x[l] = (v[t - 1 - l] - sc[0]) / sc[1];
  for (int l = 0; l <= d; ++l) x[d + l] = (c[t - l] - sc[2]) / sc[3];
  for (int l = 0; l <= d; ++l) x[2 * d + 1 + l] = (m[t - l] - sc[4]) / sc[5];
}

/* narx_predict generalised (predictor.cpp:147-153); windows most recent first */
double orc_narxg_predict(const double* p, int d, int h, const double* vlags, const double* cwin,
                         const double* mwin, double floor_) {
  const int I = 3 * d + 2;
  const double* sc = p + h * I + 2 * h + 1;
  double x[256];
  for (int l = 0; l < d; ++l) x[l] = (vlags[l] - sc[0]) / sc[1];
  for (int l = 0; l <= d; ++l) x[d + l] = (cwin[l] - sc[2]) / sc[3];
  for (int l = 0; l <= d; ++l) x[2 * d + 1 + l] = (mwin[l] - sc[4]) / sc[5];
  const double out = sc[0] + sc[1] * narxg_fwd(p, I, h, x, NULL);
  return out > floor_ ? out : floor_;
}

/* narx_train_online generalised (predictor.cpp:155-196). fixed_epochs > 0
 * disables the early stop (throughput mode of the C4 sweep). */
int orc_narxg_train(double* p, int d, int h, const double* v, const double* c, const double* m,
                    int len, const lbbsp_narx_train_cfg* cfg, int fixed_epochs,
                    lbbsp_narx_report* rep, double* loss_log, int loss_cap) {
  const int I = 3 * d + 2, P = h * I + 2 * h + 1;
  rep->ran = 0; rep->epochs = 0; rep->final_loss = 0.0;
  const int minh = cfg->min_history > d + 1 ? cfg->min_history : d + 1;
  if (len < minh) return 0;
  double* sc = p + P;
  fit_scaler(v, len, &sc[0], &sc[1]);
  fit_scaler(c, len, &sc[2], &sc[3]);
  fit_scaler(m, len, &sc[4], &sc[5]);
  const int cnt = len - d;
  double* Z = (double*)malloc(sizeof(double) * (size_t)I * cnt);
  double* T = (double*)malloc(sizeof(double) * (size_t)cnt);
  for (int t = d; t < len; ++t) {
    narxg_inputs(sc, d, v, c, m, t, Z + (size_t)I * (t - d));
    T[t - d] = (v[t] - sc[0]) / sc[1];
  }
  double* w = (double*)malloc(sizeof(double) * P);
  double* g = (double*)malloc(sizeof(double) * P);
  double* tr = (double*)malloc(sizeof(double) * P);
  double* hid = (double*)malloc(sizeof(double) * h);
  memcpy(w, p, sizeof(double) * P);
#define NARXG_MSE(wt, out)                                               \
  do {                                                                   \
    double tot_ = 0.0;                                                   \
    for (int i_ = 0; i_ < cnt; ++i_) {                                   \
      const double e_ = narxg_fwd(wt, I, h, Z + (size_t)I * i_, NULL) - T[i_]; \
      tot_ += e_ * e_;                                                   \
    }                                                                    \
    out = tot_ / (double)cnt;                                            \
  } while (0)
  double current;
  NARXG_MSE(w, current);
  int stall = 0;
  rep->ran = 1;
  const int max_ep = fixed_epochs > 0 ? fixed_epochs : cfg->max_epochs;
  for (int epoch = 0; epoch < max_ep; ++epoch) {
    for (int k = 0; k < P; ++k) g[k] = 0.0;
    const double scale = 2.0 / (double)cnt;
    for (int i = 0; i < cnt; ++i) {
      const double* x = Z + (size_t)I * i;
      const double y = narxg_fwd(w, I, h, x, hid);
      const double dy = scale * (y - T[i]);
      for (int j = 0; j < h; ++j) {
        g[h * I + h + j] += dy * hid[j];                  /* output weight */
        if (j == 0) g[h * I + 2 * h] += dy;                /* output bias   */
        const double dz = dy * w[h * I + h + j] * (1.0 - hid[j] * hid[j]);
        for (int q = 0; q < I; ++q) g[j * I + q] += dz * x[q];
        g[h * I + j] += dz;                                /* hidden bias   */
      }
    }
    double step = cfg->step, next;
    for (int k = 0; k < P; ++k) tr[k] = w[k] - step * g[k];
    NARXG_MSE(tr, next);
    int halvings = 0;
    while (next > current && halvings < 20) {
      step *= 0.5;
      for (int k = 0; k < P; ++k) tr[k] = w[k] - step * g[k];
      NARXG_MSE(tr, next);
      ++halvings;
    }
    if (next > current) break;
    memcpy(w, tr, sizeof(double) * P);
    if (loss_log && rep->epochs < loss_cap) loss_log[rep->epochs] = next;
    ++rep->epochs;
    stall = (current - next < cfg->early_stop_delta) ? stall + 1 : 0;
    current = next;
    if (fixed_epochs <= 0 && stall >= cfg->early_stop_patience) break;
  }
#undef NARXG_MSE
  rep->final_loss = current;
  memcpy(p, w, sizeof(double) * P);
  free(Z); free(T); free(w); free(g); free(tr); free(hid);
  return 0;
}
