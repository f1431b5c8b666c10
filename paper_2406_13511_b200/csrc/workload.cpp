// workload.cpp — scls_generate: host-side Poisson trace generation with the
// reference's exact sampler (workload.cpp:100-181): std::mt19937_64, the top
// 53 bits per uniform, exponential gaps through glibc `log`, histogram /
// uniform / log-normal length draws truncated to [1, limit].  Traces are an
// input of the simulator, produced once and uploaded; generation is not part
// of the device hot path (SURVEY §8(f) row 1 moves it on-device).
#include <cmath>
#include <cstdint>
#include <random>
#include <string>

#include "scls_capi.h"

namespace scls {
scls_status set_error(struct scls_ctx* ctx, scls_status st, const std::string& msg);
}

namespace {

double uniform01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

int draw_int(int lo, int hi, std::mt19937_64& g) {
  const double u = uniform01(g);
  return lo + static_cast<int>(u * (static_cast<double>(hi) - lo + 1.0));
}

int truncate_len(long long v, int limit) { return v < 1 ? 1 : (v > limit ? limit : static_cast<int>(v)); }

int draw_length(const scls_length_dist& d, int limit, std::mt19937_64& g) {
  if (d.kind == SCLS_DIST_UNIFORM) return truncate_len(draw_int(d.lo, d.hi, g), limit);
  if (d.kind == SCLS_DIST_LOGNORMAL) {
    const double u1 = 1.0 - uniform01(g);
    const double u2 = uniform01(g);
    const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
    const double raw = std::exp(d.mu + d.sigma * z);
    const long long r = raw > 1e18 ? static_cast<long long>(1e18) : std::llround(raw);
    return truncate_len(r < d.cap ? r : d.cap, limit);
  }
  const double u = uniform01(g);
  double cdf = 0.0;
  int bucket = d.n_buckets - 1;
  for (int i = 0; i < d.n_buckets; ++i) {
    cdf += d.weights[i];
    if (u < cdf) {
      bucket = i;
      break;
    }
  }
  return truncate_len(draw_int(d.edges[bucket], d.edges[bucket + 1], g), limit);
}

scls_status check_dist(scls_ctx* ctx, const scls_length_dist& d) {
  using scls::set_error;
  if (d.kind == SCLS_DIST_UNIFORM) {
    if (d.lo < 1 || d.hi < d.lo) return set_error(ctx, SCLS_ERR_ERROR, "uniform length distribution requires 1 <= lo <= hi");
  } else if (d.kind == SCLS_DIST_LOGNORMAL) {
    if (!(d.sigma > 0.0) || d.cap < 1) return set_error(ctx, SCLS_ERR_ERROR, "log-normal length distribution requires sigma > 0 and cap >= 1");
  } else if (d.kind == SCLS_DIST_HISTOGRAM) {
    if (d.n_buckets < 1 || d.n_buckets > SCLS_MAX_BUCKETS) return set_error(ctx, SCLS_ERR_ERROR, "histogram needs k weights and k+1 edges, k >= 1");
    for (int i = 0; i < d.n_buckets; ++i)
      if (d.edges[i] < 1 || d.edges[i] > d.edges[i + 1]) return set_error(ctx, SCLS_ERR_ERROR, "histogram edges must be >= 1 and non-decreasing");
    double total = 0.0;
    for (int i = 0; i < d.n_buckets; ++i) {
      if (d.weights[i] < 0.0) return set_error(ctx, SCLS_ERR_ERROR, "histogram weights must be non-negative");
      total += d.weights[i];
    }
    if (std::abs(total - 1.0) > 1e-9) return set_error(ctx, SCLS_ERR_ERROR, "histogram weights must sum to 1 within 1e-9");
  } else {
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "unknown length distribution kind");
  }
  return SCLS_OK;
}

}  // namespace

namespace scls {
// validate(const WorkloadSpec&) (workload.cpp:84-98), shared with the device
// generator (workload_gen.cu).
scls_status validate_workload_spec(scls_ctx* ctx, const scls_workload_spec& spec) {
  if (!(spec.rate > 0.0)) return set_error(ctx, SCLS_ERR_ERROR, "workload rate must be > 0");
  if (spec.duration_s < 0.0) return set_error(ctx, SCLS_ERR_ERROR, "workload duration must be >= 0");
  if (spec.max_input_limit < 1 || spec.max_gen_limit < 1) return set_error(ctx, SCLS_ERR_ERROR, "length limits must be >= 1");
  scls_status st = check_dist(ctx, spec.input_len_dist);
  if (st) return st;
  return check_dist(ctx, spec.gen_len_dist);
}
}  // namespace scls

extern "C" scls_status scls_generate(const scls_workload_spec* spec, int64_t cap, int64_t* n, double* arrival,
                                     int32_t* input_len, int32_t* gen_len) {
  using scls::set_error;
  if (!spec || !n || (cap > 0 && (!arrival || !input_len || !gen_len)))
    return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  *n = 0;
  scls_status st = scls::validate_workload_spec(nullptr, *spec);
  if (st) return st;
  std::mt19937_64 g(spec->seed);
  double clock = 0.0;
  int64_t k = 0;
  for (;;) {
    clock += -std::log(1.0 - uniform01(g)) / spec->rate;
    if (clock > spec->duration_s) break;
    const int in = draw_length(spec->input_len_dist, spec->max_input_limit, g);
    const int gl = draw_length(spec->gen_len_dist, spec->max_gen_limit, g);
    if (k < cap) {
      arrival[k] = clock;
      input_len[k] = in;
      gen_len[k] = gl;
    }
    ++k;
  }
  *n = k;
  return k > cap ? SCLS_ERR_CAPACITY : SCLS_OK;
}

extern "C" scls_status scls_make_pool(int64_t n, uint64_t seed, int32_t* input_len, double* arrival,
                                      int64_t* id, int32_t* gen_len) {
  if (n < 0 || (n > 0 && (!input_len || !arrival || !id)))
    return scls::set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  std::mt19937_64 g(seed);
  for (int64_t i = 0; i < n; ++i) {
    id[i] = i;
    arrival[i] = uniform01(g) * 100.0;
    input_len[i] = 1 + static_cast<int>(uniform01(g) * 1024.0);
    const int gl = 1 + static_cast<int>(uniform01(g) * 1024.0);
    if (gen_len) gen_len[i] = gl;
  }
  return SCLS_OK;
}
