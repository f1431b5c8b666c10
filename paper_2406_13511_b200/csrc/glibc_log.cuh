// glibc_log.cuh — bit-exact port of the `log` the reference calls.
//
// The reference draws exponential inter-arrival gaps as -std::log(1 - u) / rate
// (workload.cpp:106-110).  On an x86-64 host with FMA (the survey box and the
// GPU boxes), glibc 2.39's IFUNC dispatches `log` to the FMA build of
// sysdeps/ieee754/dbl-64/e_log.c (ARM optimized-routines, 128-entry table).
// That build contracts several a*b+c into vfmadd; the exact operation order
// below was read off the machine code of that variant in this image's
// libm.so.6 (the resolver's AVX2+FMA target) and is spelled with explicit
// fma / mul / add so neither compiler may re-contract it:
//   - main path:  x = 2^k z, r = fma(z, invc, -1), w = fma(k, ln2hi, logc),
//                 hi = w + r, lo = fma(k, ln2lo, (w - hi) + r),
//                 y = fma(r*r2, fma(fma(r, A4, A3), r2, fma(r, A2, A1)), fma(r2, A0, lo)) + hi
//   - |x - 1| < 0x1p-4: the poly1 evaluation with the 2^27 split of r.
// Constants: glibc_log_data.h (tools/extract_glibc_log.py).  Checked bit for bit
// against the host libm (tests/test_workload_gen.py).
#pragma once

#include <stdint.h>

#include "glibc_log_data.h"

#if defined(__CUDACC__)
#define SCLS_HD __host__ __device__ __forceinline__
#else
#define SCLS_HD inline
#endif

namespace scls_glibc {

#if defined(__CUDA_ARCH__)
SCLS_HD double f_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
SCLS_HD double f_mul(double a, double b) { return __dmul_rn(a, b); }
SCLS_HD double f_add(double a, double b) { return __dadd_rn(a, b); }
SCLS_HD double f_sub(double a, double b) { return __dsub_rn(a, b); }
SCLS_HD uint64_t f_bits(double x) { return (uint64_t)__double_as_longlong(x); }
SCLS_HD double f_dbl(uint64_t u) { return __longlong_as_double((long long)u); }
#else
}  // namespace scls_glibc
#include <cmath>
#include <cstring>
namespace scls_glibc {
// Host build: compiled with -ffp-contract=off, so only the explicit fma fuses.
SCLS_HD double f_fma(double a, double b, double c) { return std::fma(a, b, c); }
SCLS_HD double f_mul(double a, double b) { return a * b; }
SCLS_HD double f_add(double a, double b) { return a + b; }
SCLS_HD double f_sub(double a, double b) { return a - b; }
SCLS_HD uint64_t f_bits(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}
SCLS_HD double f_dbl(uint64_t u) {
  double x;
  std::memcpy(&x, &u, 8);
  return x;
}
#endif

// The (invc, logc) table: a global-memory copy for the device (lanes index it
// independently, so constant memory would serialise) and a host copy.
#if defined(__CUDACC__)
static __device__ const double kTabDev[256] = SCLS_GLIBC_LOG_TAB;
#endif
static const double kTabHost[256] = SCLS_GLIBC_LOG_TAB;

// log(x) as glibc 2.39's FMA variant computes it, for every double x.
SCLS_HD double log_fma(double x) {
#if defined(__CUDA_ARCH__)
  const double* kTab = kTabDev;
#else
  const double* kTab = kTabHost;
#endif
  uint64_t ix = f_bits(x);
  if (ix - 0x3fee000000000000ull < 0x3090000000000ull) {
    // 1 - 0x1p-4 <= x < 1 + 0x1.09p-4
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double r = f_sub(x, 1.0);
    double p = f_fma(r, kB2, kB1);
    double q = f_fma(r, kB5, kB4);
    const double s = f_fma(r, kB8, kB7);
    const double r2 = f_mul(r, r);
    p = f_fma(r2, kB3, p);
    q = f_fma(r2, kB6, q);
    const double r3 = f_mul(r, r2);
    double t = f_fma(r2, kB9, s);
    t = f_fma(r3, kB10, t);
    t = f_fma(t, r3, q);
    t = f_fma(t, r3, p);
    const double w2 = f_fma(r, 0x1p27, r);
    const double rhi = f_fma(-0x1p27, r, w2);
    const double rhi2 = f_mul(rhi, rhi);
    const double rlo = f_sub(r, rhi);
    const double hi = f_fma(rhi2, kB0, r);
    const double lo0 = f_sub(r, hi);
    const double rs = f_add(r, rhi);
    double lo = f_fma(rhi2, kB0, lo0);
    lo = f_fma(f_mul(kB0, rlo), rs, lo);
    const double y = f_fma(t, r3, lo);
    return f_add(hi, y);
  }
  const uint32_t top = (uint32_t)(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    // zero, subnormal, negative, inf, nan
    if ((ix << 1) == 0) return -f_dbl(0x7ff0000000000000ull);  // -inf (divide by zero)
    if (ix == 0x7ff0000000000000ull) return x;                  // +inf
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return f_dbl(0x7ff8000000000000ull);  // nan
    ix = f_bits(f_mul(x, 0x1p52)) - (52ull << 52);               // subnormal: normalise
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = (int)((tmp >> 45) & 127);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
#if defined(__CUDA_ARCH__)
  const double invc = __ldg(kTab + 2 * i), logc = __ldg(kTab + 2 * i + 1);
#else
  const double invc = kTab[2 * i], logc = kTab[2 * i + 1];
#endif
  const double z = f_dbl(iz);
  const double kd = (double)k;
  const double w = f_fma(kd, kLn2hi, logc);
  const double r = f_fma(z, invc, -1.0);
  const double a = f_fma(r, kA2, kA1);
  const double hi = f_add(r, w);
  const double r2 = f_mul(r, r);
  double lo = f_add(f_sub(w, hi), r);
  lo = f_fma(kd, kLn2lo, lo);
  const double rr2 = f_mul(r, r2);
  double b = f_fma(r, kA4, kA3);
  const double lo2 = f_fma(r2, kA0, lo);
  b = f_fma(b, r2, a);
  const double y = f_fma(rr2, b, lo2);
  return f_add(y, hi);
}

}  // namespace scls_glibc
