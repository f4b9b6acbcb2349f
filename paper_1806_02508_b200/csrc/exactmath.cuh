// exactmath.cuh -- device arithmetic that reproduces the reference's fp64
// results bit-for-bit.
//
// The reference core is built for baseline x86-64 (SSE2, no FMA),
// so every product and sum is individually rounded. nvcc would otherwise
// contract a*b+c into DFMA; the _rn intrinsics below are never contracted.
// The one place the reference DOES see fused ops is glibc's tanh -> expm1
// IFUNC, which selects __expm1_fma on FMA hosts; glibc_tanh() restates that
// exact dataflow (validated against host libm by the oracle restatement
// orc_tanh_glibc_fma and on device by tests/test_gpu_core.py::
// test_device_tanh_bit_exact_vs_glibc / test_device_tanh_batch_bit_exact_vs_host_libm).
#pragma once
#include <cstdint>

namespace lbbsp {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// a / b for a standardisation (x - mean) / stddev. __ddiv_rn leaves its
// inline fast path for a called slow path when the numerator is zero (or
// tiny), and constant series make (x - mean) = 0 for a third of the NARX
// training set. A zero numerator over a positive divisor is the numerator
// itself (+0 / b = +0, -0 / b = -0, b = +inf included), so it is divided as
// 1.0 (fast path) and the quotient replaced; every other input divides
// unchanged -- bit-identical to ddiv for all inputs. (A plain select would be
// if-converted into a division of the zero, slow path included.)
__device__ __forceinline__ double ddiv_std(double a, double b) {
  const bool z = a == 0.0 && b > 0.0;
  const double q = __ddiv_rn(z ? 1.0 : a, b);
  return z ? a : q;
}
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

__device__ __forceinline__ uint32_t hi_word(double x) {
  return static_cast<uint32_t>(__double2hiint(x));
}
__device__ __forceinline__ uint32_t lo_word(double x) {
  return static_cast<uint32_t>(__double2loint(x));
}
__device__ __forceinline__ double with_hi(double x, uint32_t hi) {
  return __hiloint2double(static_cast<int>(hi), __double2loint(x));
}

// glibc 2.39 __expm1_fma (fdlibm s_expm1.c compiled with -mfma); constants
// read from libm's .rodata (see oracle/lbbsp_oracle.c orc_expm1_glibc_fma).
//
// Written without data-dependent branches so that a warp whose lanes fall in
// different argument ranges does not serialise them: the argument reduction is
// one formula for every k (for k = 0 it gives hi = x, lo = 0, c = 0 and for
// k = +-1 it gives glibc's x -+ ln2_hi / +-ln2_lo, each bit-identical to the
// branchy source), and every final combination is formed and the one glibc
// returns is selected. Only the non-finite / overflow inputs branch.
__device__ __forceinline__ double glibc_expm1(double x) {
  const double o_threshold = 0x1.62e42fefa39efp+9, ln2_hi = 0x1.62e42fee00000p-1,
               ln2_lo = 0x1.a39ef35793c76p-33, invln2 = 0x1.71547652b82fep+0;
  const double Q1 = -0x1.11111111110f4p-5, Q2 = 0x1.a01a019fe5585p-10,
               Q3 = -0x1.4ce199eaadbb7p-14, Q4 = 0x1.0cfca86e65239p-18,
               Q5 = -0x1.afdb76e09c32dp-23;
  uint32_t hx = hi_word(x);
  const uint32_t xsb = hx & 0x80000000u;
  hx &= 0x7fffffffu;
  if (hx >= 0x40862E42u) {  // |x| >= 709.78: inf, nan, overflow, -1
    if (hx >= 0x7ff00000u) {
      if (((hx & 0xfffffu) | lo_word(x)) != 0) return dadd(x, x);
      return xsb == 0 ? x : -1.0;
    }
    if (x > o_threshold) return __int_as_float(0x7f800000);  // +inf
  }
  const bool neg_one = hx >= 0x4043687Au && xsb != 0;  // tiny - one rounds to -1
  const bool tiny = hx < 0x3c900000u;                  // |x| < 2^-54 (inexact only)
  int k = 0;
  if (hx > 0x3fd62e42u)
    k = hx < 0x3FF0A2B2u ? (xsb == 0 ? 1 : -1)
                         : static_cast<int>(dadd(dmul(invln2, x), xsb == 0 ? 0.5 : -0.5));
  const double tk = static_cast<double>(k);
  const double hi = dfma(-tk, ln2_hi, x);
  const double lo = dmul(tk, ln2_lo);
  const double xr = dsub(hi, lo);
  const double c = dsub(dsub(hi, xr), lo);
  const double hfx = dmul(xr, 0.5);
  const double hxs = dmul(xr, hfx);
  const double R1 = dfma(hxs, Q1, 1.0);
  const double R2 = dfma(hxs, Q3, Q2);
  const double R3 = dfma(hxs, Q5, Q4);
  const double h2 = dmul(hxs, hxs);
  const double h4 = dmul(h2, h2);
  const double r1 = dfma(h4, R3, dfma(h2, R2, R1));
  const double t = dfma(-r1, hfx, 3.0);
  const double e = dmul(ddiv(dsub(r1, t), dfma(-xr, t, 6.0)), hxs);
  // k == 0
  const double res0 = dsub(xr, dfma(e, xr, -hxs));
  // k != 0
  const double e2 = dsub(dfma(dsub(e, c), xr, -c), hxs);
  const double res_m1 = dfma(0.5, dsub(xr, e2), -0.5);
  const double res_p1 = xr < -0.25 ? dmul(dsub(e2, dadd(xr, 0.5)), -2.0)
                                   : dfma(dsub(xr, e2), 2.0, 1.0);
  const uint32_t kshift = static_cast<uint32_t>(k) << 20;
  const double ya = dsub(1.0, dsub(e2, xr));                      // k <= -2 || k > 56
  const double res_a = dsub(with_hi(ya, hi_word(ya) + kshift), 1.0);
  const int kb = k > 0 && k < 20 ? k : 1;                         // k < 20
  const double tb = __hiloint2double(static_cast<int>(0x3ff00000u - (0x200000u >> kb)), 0);
  const double yb = dsub(tb, dsub(e2, xr));
  const double res_b = with_hi(yb, hi_word(yb) + kshift);
  const int kc = k >= 20 && k <= 56 ? k : 20;                     // 20 <= k <= 56
  const double tc = __hiloint2double(static_cast<int>(static_cast<uint32_t>(0x3ff - kc) << 20), 0);
  const double yc = dadd(dsub(xr, dadd(e2, tc)), 1.0);
  const double res_c = with_hi(yc, hi_word(yc) + kshift);
  double r = (k <= -2 || k > 56) ? res_a : (k < 20 ? res_b : res_c);
  r = k == 1 ? res_p1 : r;
  r = k == -1 ? res_m1 : r;
  r = k == 0 ? res0 : r;
  r = tiny ? x : r;
  return neg_one ? -1.0 : r;
}

// glibc 2.39 tanh (sysdeps/ieee754/dbl-64/s_tanh.c; no FMA in tanh itself):
// the two |x| ranges share one expm1 and one division (numerator selected),
// and the zero / tiny / saturated results are selected, so lanes stay converged.
__device__ __forceinline__ double glibc_tanh(double x) {
  const uint32_t jx = hi_word(x), ix = jx & 0x7fffffffu;
  if (ix >= 0x7ff00000u) {
    if (jx & 0x80000000u) return dsub(ddiv(1.0, x), 1.0);
    return dadd(ddiv(1.0, x), 1.0);
  }
  const double ax = fabs(x);
  const bool big = ix >= 0x3ff00000u;
  const double t = glibc_expm1(big ? dadd(ax, ax) : dmul(-2.0, ax));
  const double den = dadd(t, 2.0);
  const double q = ddiv(big ? 2.0 : -t, den);
  double z = big ? dsub(1.0, q) : q;
  z = ix >= 0x40360000u ? 1.0 : z;  // |x| >= 22: one - tiny
  z = (jx & 0x80000000u) ? -z : z;
  z = ix < 0x3c800000u ? dmul(x, dadd(1.0, x)) : z;  // |x| < 2^-55
  return (ix | lo_word(x)) == 0 ? x : z;
}

// ---- rng.hpp:9-42 ----------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t a, uint64_t b) {
  return mix64(a ^ mix64(b));
}
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t a, uint64_t b, uint64_t c) {
  return mix_seed(mix_seed(a, b), c);
}

__device__ __forceinline__ uint64_t mt64_temper(uint64_t x) {
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}

__device__ __forceinline__ uint64_t mt64_twist_one(uint64_t cur, uint64_t next, uint64_t far) {
  const uint64_t x = (cur & 0xFFFFFFFF80000000ull) | (next & 0x7FFFFFFFull);
  return far ^ (x >> 1) ^ ((x & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
}

// Rng::uniform() then uniform_int(lo, lo+range-1) (rng.hpp:31,36-38)
__device__ __forceinline__ int uniform_int_from(uint64_t u, int lo, int range) {
  const double f = dmul(static_cast<double>(u >> 11), 0x1.0p-53);
  return lo + static_cast<int>(dmul(f, static_cast<double>(range)));
}

__device__ __forceinline__ double uniform_from(uint64_t u) {
  return dmul(static_cast<double>(u >> 11), 0x1.0p-53);
}

}  // namespace lbbsp
