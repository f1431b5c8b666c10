// scls_common.cuh — device-side restatement of the serving-time and KV-memory
// estimators (reference cost_model.cpp:30-51, memory_model.cpp:28-90) with
// the reference's exact fp64 association order.  Every product and sum is an
// explicit round-to-nearest intrinsic so no FMA contraction can occur,
// whatever the compile flags (the reference Release build has no FMA).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "scls_capi.h"

#define SCLS_DEV __device__ __forceinline__

namespace scls {

constexpr int kWarp = 32;
constexpr int kMaxRules = SCLS_MAX_RULES;

// Latency model coefficients (cost_model.h:29-39), device copy.
struct Lat {
  double p1, p2, p3, p4, d1, d2, d3, d4;
};

// Memory model (memory_model.h:20-53), device copy.  `budget` caches the
// reference's right-hand side zeta * available_mem() (memory_model.cpp:63),
// which it recomputes identically on every call.
struct Mem {
  int32_t kind;
  int32_t n_rules;
  double delta;
  double budget;
  double zeta;
  double avail;
  int32_t thr[kMaxRules];
  int32_t max_n[kMaxRules];
};

inline Lat make_lat(const scls_latency& m) {
  return Lat{m.p1, m.p2, m.p3, m.p4, m.d1, m.d2, m.d3, m.d4};
}

inline Mem make_mem(const scls_memory& m) {
  Mem r{};
  r.kind = m.kind;
  r.n_rules = m.n_rules;
  r.delta = m.delta;
  // memory_model.cpp:54-59 then :63, same operation order on the host.
  volatile double avail = m.m_cap - m.m_model;
  avail = avail - m.m_engine;
  r.avail = avail;
  r.zeta = m.zeta;
  volatile double budget = m.zeta * r.avail;
  r.budget = budget;
  for (int i = 0; i < kMaxRules; ++i) {
    r.thr[i] = m.rule_threshold[i];
    r.max_n[i] = m.rule_max_n[i];
  }
  return r;
}

// cost_model.cpp:30-33 (Eq. 3): p1*n*l + p2*n + p3*l + p4, left to right.
SCLS_DEV double prefill_time(const Lat& m, int n, int l_in) {
  const double dn = (double)n, dl = (double)l_in;
  double v = __dmul_rn(__dmul_rn(m.p1, dn), dl);
  v = __dadd_rn(v, __dmul_rn(m.p2, dn));
  v = __dadd_rn(v, __dmul_rn(m.p3, dl));
  return __dadd_rn(v, m.p4);
}

// cost_model.cpp:35-38 (Eq. 4).
SCLS_DEV double decode_step_time(const Lat& m, int ctx, int n) {
  const double dn = (double)n, dl = (double)ctx;
  double v = __dmul_rn(__dmul_rn(m.d1, dn), dl);
  v = __dadd_rn(v, __dmul_rn(m.d2, dn));
  v = __dadd_rn(v, __dmul_rn(m.d3, dl));
  return __dadd_rn(v, m.d4);
}

// cost_model.cpp:40-47 (Eq. 2 closed form).  sum_l depends only on
// (l_in, l_out), so callers that sweep n may hoist it (decode_sum_l).
SCLS_DEV double decode_sum_l(int l_in, int l_out) {
  const double k = (double)l_out;
  // k * l_in + k * (k + 1.0) / 2.0
  return __dadd_rn(__dmul_rn(k, (double)l_in),
                   __ddiv_rn(__dmul_rn(k, __dadd_rn(k, 1.0)), 2.0));
}

SCLS_DEV double decode_time_from_sum(const Lat& m, int n, double sum_l, int l_out) {
  if (l_out <= 0) return 0.0;
  const double dn = (double)n, k = (double)l_out;
  // (d1*n + d3) * sum_l + (d2*n + d4) * k
  return __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(m.d1, dn), m.d3), sum_l),
                   __dmul_rn(__dadd_rn(__dmul_rn(m.d2, dn), m.d4), k));
}

SCLS_DEV double decode_time(const Lat& m, int n, int l_in, int l_out) {
  if (l_out <= 0) return 0.0;
  return decode_time_from_sum(m, n, decode_sum_l(l_in, l_out), l_out);
}

// cost_model.cpp:49-51 (Eq. 1).
SCLS_DEV double batch_serve_time(const Lat& m, int n, int l_in, int l_out) {
  return __dadd_rn(prefill_time(m, n, l_in), decode_time(m, n, l_in, l_out));
}

// memory_model.cpp:28-31 (Eq. 5): (l_in + l_out) * n * delta.
SCLS_DEV double kv_cache_mem(double delta, int n, int l_in, int l_out) {
  return __dmul_rn(__dmul_rn(__dadd_rn((double)l_in, (double)l_out), (double)n), delta);
}

// memory_model.cpp:61-70 (Eq. 7/9, Alg. 2).
SCLS_DEV bool would_oom(const Mem& m, int n, int l_in, int slice) {
  if (m.kind == SCLS_MEM_ANALYTIC) return kv_cache_mem(m.delta, n, l_in, slice) > m.budget;
  const int total = l_in + slice;
  for (int i = 0; i < m.n_rules; ++i)
    if (total > m.thr[i]) return n > m.max_n[i];
  return n > m.max_n[m.n_rules - 1];
}

// memory_model.cpp:72-90 (Eq. 8): floor estimate nudged onto the exact
// would_oom boundary; capped at 1e9.
SCLS_DEV int max_batch_size(const Mem& m, int l_in, int slice) {
  if (m.kind == SCLS_MEM_RULE_TABLE) {
    const int total = l_in + slice;
    for (int i = 0; i < m.n_rules; ++i)
      if (total > m.thr[i]) return m.max_n[i];
    return m.max_n[m.n_rules - 1];
  }
  const double per_request = __dmul_rn(m.delta, __dadd_rn((double)l_in, (double)slice));
  const double quotient = floor(__ddiv_rn(__dmul_rn(m.zeta, m.avail), per_request));
  if (quotient >= 1e9) return 1000000000;
  int n = (int)quotient;
  if (n < 0) n = 0;
  while (n > 0 && would_oom(m, n, l_in, slice)) --n;
  while (n < 1000000000 && !would_oom(m, n + 1, l_in, slice)) ++n;
  return n;
}

// Order-preserving map of a double onto uint64 (radix keys).  -0.0 is
// canonicalised to +0.0 because the reference compares with `<`, under which
// the two are equal (batcher.cpp:35-38, offloader.cpp:34-37).
SCLS_DEV uint64_t ordered_bits(double x) {
  // -0.0 and +0.0 share a key; negatives flip every bit, others only the sign.
  const uint64_t u = x == 0.0 ? 0ull : (uint64_t)__double_as_longlong(x);
  const uint64_t m = (uint64_t)((int64_t)u >> 63);
  return u ^ (m | 0x8000000000000000ull);
}

}  // namespace scls
