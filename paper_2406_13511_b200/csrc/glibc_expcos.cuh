// glibc_expcos.cuh — bit-exact ports of the `exp` and `cos` the reference's
// log-normal length sampler calls, and that sampler.
//
// workload.cpp:112-118,136-141 (next_standard_normal, sample_length kLogNormal):
//   u1 = 1 - u,  u2 = u'                        (two engine outputs, always)
//   z   = sqrt(-2.0 * log(u1)) * cos(2 pi * u2)
//   raw = exp(mu + sigma * z)
//   len = clamp(min(raw > 1e18 ? 1e18 : llround(raw), cap), 1, limit)
// The reference is compiled without FMA contraction (no -march; oracle/Makefile
// adds -ffp-contract=off), so the products and sums around the library calls
// are plain _rn operations here.  `log` is csrc/glibc_log.cuh.  On x86-64 with
// AVX2+FMA, glibc 2.39's IFUNCs select the FMA builds of
//   - exp: sysdeps/ieee754/dbl-64/e_exp.c (2^(k/128) table, degree-5 poly);
//   - cos: sysdeps/ieee754/dbl-64/s_sin.c __cos (do_cos / do_sin /
//     TAYLOR_SIN / reduce_sincos over __sincostab).
// The operation order and every fused multiply-add below were read off the
// machine code of those variants in this image's libm.so.6 (__exp_fma at
// 0x79b60, __cos_fma at 0x7bad0); the constants are in glibc_expcos_data.h
// (tools/extract_glibc_expcos.py).  tests/test_workload_gen.py checks the host
// build of this file against the host libm on millions of arguments, and the
// device build against the host build.
//
// Domain notes.  cos is called on [0, 2 pi) only (u2 in [0, 1)), which takes
// the first three branches of __cos (|x| < 105414350); exp's argument paths
// with |x| >= 512 (glibc's specialcase) only decide whether raw is above 1e18
// or below 0.5, so they return +inf / +0 here, which give the same length.
#pragma once

#include <stdint.h>

#include "glibc_expcos_data.h"
#include "glibc_log.cuh"

namespace scls_glibc {

#if defined(__CUDACC__)
static __device__ const uint64_t kExpTabDev[256] = SCLS_GLIBC_EXP_TAB;
static __device__ const uint64_t kSinCosTabDev[440] = SCLS_GLIBC_SINCOS_TAB;
#endif
static const uint64_t kExpTabHost[256] = SCLS_GLIBC_EXP_TAB;
static const uint64_t kSinCosTabHost[440] = SCLS_GLIBC_SINCOS_TAB;

SCLS_HD double tab_d(const uint64_t* t, int i) {
#if defined(__CUDA_ARCH__)
  return f_dbl(__ldg((const unsigned long long*)t + i));
#else
  return f_dbl(t[i]);
#endif
}
SCLS_HD uint64_t tab_u(const uint64_t* t, int i) {
#if defined(__CUDA_ARCH__)
  return __ldg((const unsigned long long*)t + i);
#else
  return t[i];
#endif
}
SCLS_HD const uint64_t* exp_tab() {
#if defined(__CUDA_ARCH__)
  return kExpTabDev;
#else
  return kExpTabHost;
#endif
}
SCLS_HD const uint64_t* sincos_tab() {
#if defined(__CUDA_ARCH__)
  return kSinCosTabDev;
#else
  return kSinCosTabHost;
#endif
}
SCLS_HD double f_abs(double x) { return f_dbl(f_bits(x) & 0x7fffffffffffffffull); }
SCLS_HD double f_neg(double x) { return f_dbl(f_bits(x) ^ 0x8000000000000000ull); }

// exp(x), __exp_fma (e_exp.c): kd = fma(x, N/ln2, shift); r = x - kd ln2/N in two
// fused steps; tmp = fma(r2^2, fma(r, C5, C4), fma(r2, fma(r, C3, C2), tail + r));
// result = fma(scale, tmp, scale).
SCLS_HD double exp_fma(double x) {
  const uint64_t ix = f_bits(x);
  const uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x3fu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return f_add(1.0, x);  // |x| < 2^-54
    // |x| >= 512 (glibc's specialcase / overflow / underflow): see the header
    if (x != x) return x;
    return (ix >> 63) ? 0.0 : f_dbl(0x7ff0000000000000ull);
  }
  const double shift = f_dbl(kExpShift);
  const double kd0 = f_fma(x, f_dbl(kExpInvLn2N), shift);
  const uint64_t ki = f_bits(kd0);
  const double kd = f_sub(kd0, shift);
  double r = f_fma(kd, f_dbl(kExpNegLn2hiN), x);
  r = f_fma(kd, f_dbl(kExpNegLn2loN), r);
  const int idx = 2 * (int)(ki & 127u);
  const uint64_t top = ki << 45;
  const uint64_t* T = exp_tab();
  const double tail = tab_d(T, idx);
  const uint64_t sbits = tab_u(T, idx + 1) + top;
  const double p23 = f_fma(r, f_dbl(kExpC3), f_dbl(kExpC2));
  const double tr = f_add(r, tail);
  const double r2 = f_mul(r, r);
  const double p45 = f_fma(r, f_dbl(kExpC5), f_dbl(kExpC4));
  const double a = f_fma(p23, r2, tr);
  const double r4 = f_mul(r2, r2);
  const double tmp = f_fma(r4, p45, a);
  const double scale = f_dbl(sbits);
  return f_fma(scale, tmp, scale);
}

// s_sin.c do_cos(x, dx) as __cos_fma computes it (x of either sign).
SCLS_HD double cos_do_cos(double x, double dx) {
  if (x < 0) dx = f_neg(dx);
  const double big = f_dbl(kCos_big);
  const double ax = f_abs(x);
  const double u = f_add(ax, big);
  const double xr = f_add(f_sub(ax, f_sub(u, big)), dx);
  const int k = (int)(uint32_t)f_bits(u) << 2;
  const uint64_t* S = sincos_tab();
  const double xx = f_mul(xr, xr);
  const double p = f_fma(xx, f_dbl(kCos_sn5), f_dbl(kCos_sn3));
  const double s = f_fma(f_mul(xr, xx), p, xr);
  double c = f_fma(xx, f_dbl(kCos_cs6), f_dbl(kCos_cs4));
  c = f_fma(xx, c, f_dbl(kCos_cs2));
  c = f_mul(xx, c);
  const double sn = tab_d(S, k), ssn = tab_d(S, k + 1), cs = tab_d(S, k + 2), ccs = tab_d(S, k + 3);
  double cor = f_fma(f_neg(s), ssn, ccs);
  cor = f_fma(f_neg(c), cs, cor);
  cor = f_fma(f_neg(s), sn, cor);
  return f_add(cs, cor);
}

// TAYLOR_SIN(a*a, a, da): a + (fma(xx, fma(POLY(xx), a, -0.5 da), da)).
SCLS_HD double cos_taylor_sin(double a, double da) {
  const double xx = f_mul(a, a);
  double p = f_fma(xx, f_dbl(kCos_s5), f_dbl(kCos_s4));
  p = f_fma(xx, p, f_dbl(kCos_s3));
  p = f_fma(xx, p, f_dbl(kCos_s2));
  p = f_fma(xx, p, f_dbl(kCos_s1));
  const double h = f_mul(da, f_dbl(kCos_cs2));
  const double q = f_fma(p, a, f_neg(h));
  const double t = f_fma(xx, q, da);
  return f_add(a, t);
}

// s_sin.c do_sin(x, dx) as __cos_fma computes it.
SCLS_HD double cos_do_sin(double x, double dx) {
  if (f_abs(x) < f_dbl(kCos_taylor_lim)) return cos_taylor_sin(x, dx);
  if (x <= 0) dx = f_neg(dx);
  const double big = f_dbl(kCos_big);
  const double ax = f_abs(x);
  const double u = f_add(ax, big);
  const double xr = f_sub(ax, f_sub(u, big));
  const int k = (int)(uint32_t)f_bits(u) << 2;
  const uint64_t* S = sincos_tab();
  const double xx = f_mul(xr, xr);
  const double p = f_fma(xx, f_dbl(kCos_sn5), f_dbl(kCos_sn3));
  const double s = f_add(xr, f_fma(f_mul(xr, xx), p, dx));
  double c = f_fma(xx, f_dbl(kCos_cs6), f_dbl(kCos_cs4));
  c = f_fma(xx, c, f_dbl(kCos_cs2));
  c = f_fma(dx, xr, f_mul(xx, c));
  const double sn = tab_d(S, k), ssn = tab_d(S, k + 1), cs = tab_d(S, k + 2), ccs = tab_d(S, k + 3);
  double cor = f_fma(s, ccs, ssn);
  cor = f_fma(f_neg(c), sn, cor);
  cor = f_fma(s, cs, cor);
  const double r = f_add(sn, cor);
  return f_dbl((f_bits(r) & 0x7fffffffffffffffull) | (f_bits(x) & 0x8000000000000000ull));  // copysign
}

// cos(x) for |x| < 105414350 (the sampler's [0, 2 pi)), __cos_fma's branches.
SCLS_HD double cos_fma(double x) {
  const uint32_t k = (uint32_t)(f_bits(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;            // |x| < 2^-27
  if (k < 0x3feb6000u) return cos_do_cos(x, 0.0);  // |x| < 0.855469
  if (k < 0x400368fdu) {                      // |x| < 2.426265: sin(pi/2 - |x|)
    const double y = f_sub(f_dbl(kCos_hp0), f_abs(x));
    const double a = f_add(y, f_dbl(kCos_hp1));
    const double da = f_add(f_sub(y, a), f_dbl(kCos_hp1));
    return cos_do_sin(a, da);
  }
  // reduce_sincos: x = n pi/2 + (a + da), the pi/2 split in four parts
  const double toint = f_dbl(kCos_toint);
  const double t = f_fma(x, f_dbl(kCos_hpinv), toint);
  const double xn = f_sub(t, toint);
  const int n = (int)(f_bits(t) & 3u);
  double y = f_fma(f_neg(xn), f_dbl(kCos_mp1), x);
  y = f_fma(f_neg(xn), f_dbl(kCos_mp2), y);
  const double pp3 = f_dbl(kCos_pp3), pp4 = f_dbl(kCos_pp4);
  const double t2 = f_fma(f_neg(xn), pp3, y);
  double db = f_fma(f_neg(xn), pp3, f_sub(y, t2));
  const double b = f_fma(f_neg(xn), pp4, t2);
  db = f_add(db, f_fma(f_neg(xn), pp4, f_sub(t2, b)));
  // do_sincos(a, da, n + 1)
  const double r = ((n + 1) & 1) ? cos_do_cos(b, db) : cos_do_sin(b, db);
  return ((n + 1) & 2) ? f_neg(r) : r;
}

// sample_length, kLogNormal (workload.cpp:136-141), from the request's two
// engine outputs; cap = dist.cap, limit = max_{input,gen}_limit.
SCLS_HD int lognormal_length(double mu, double sigma, long long cap, int limit, uint64_t w0, uint64_t w1) {
  const double u1 = f_sub(1.0, f_mul((double)(w0 >> 11), 0x1.0p-53));
  const double u2 = f_mul((double)(w1 >> 11), 0x1.0p-53);
  const double two_pi = 6.283185307179586;  // 2.0 * std::numbers::pi, folded by the compiler
#if defined(__CUDA_ARCH__)
  const double rad = __dsqrt_rn(f_mul(-2.0, log_fma(u1)));
#else
  const double rad = std::sqrt(f_mul(-2.0, log_fma(u1)));
#endif
  const double z = f_mul(rad, cos_fma(f_mul(two_pi, u2)));
  const double raw = exp_fma(f_add(mu, f_mul(sigma, z)));
  long long rounded;
  if (raw > 1e18) {
    rounded = 1000000000000000000ll;
  } else {
#if defined(__CUDA_ARCH__)
    rounded = llround(raw);
#else
    rounded = std::llround(raw);
#endif
  }
  if (rounded > cap) rounded = cap;
  if (rounded < 1) return 1;
  if (rounded > limit) return limit;
  return (int)rounded;
}

}  // namespace scls_glibc
