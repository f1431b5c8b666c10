// fit.cpp — scls_fit_latency: the latency-model fit of cost_model.cpp:96-160
// (SURVEY §8(f) row 4).  A 4-parameter least-squares problem per phase on a
// few hundred profile samples, so it stays on the host (no device work would
// pay for itself here).
//
// Per phase (prefill, decode) the reference builds the design matrix
// [n*l, n, l, 1] and the latency target, solves it with Eigen's
// ColPivHouseholderQR, refuses rank < 4, and reports the coefficients and
// rmse = sqrt(|design * coef - target|^2 / m); then `validate` (cost_model.cpp
// :70-87).  Here: Householder QR with column pivoting written out (pivot = the
// column of largest remaining norm; rank = diagonal entries of R above
// eps * min(m, 4) * max|R_kk|, Eigen's default threshold), back substitution,
// and the same checks and error messages.  Floating-point results agree with
// the reference within the north star's 1e-9 relative tolerance
// (tests/test_fit.py), not bit for bit: the solver's operation order is not
// the reference's.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <set>
#include <string>
#include <vector>

#include "scls_capi.h"

namespace scls {
scls_status set_error(struct scls_ctx* ctx, scls_status st, const std::string& msg);
}

namespace {

struct PhaseFit {
  double c[4];
  double rmse;
};

scls_status fit_phase(const scls_profile_sample* s, int64_t n, int32_t phase, const char* name, PhaseFit* out) {
  std::vector<const scls_profile_sample*> rows;
  std::set<int> sizes, lengths;
  for (int64_t i = 0; i < n; ++i) {
    if (s[i].phase != phase) continue;
    rows.push_back(&s[i]);
    sizes.insert(s[i].batch_size);
    lengths.insert(s[i].length);
  }
  if (rows.size() < 4 || sizes.size() < 2 || lengths.size() < 2)
    return scls::set_error(nullptr, SCLS_ERR_INSUFFICIENT_SAMPLES,
                           std::string(name) +
                               " fit needs >= 4 samples spanning >= 2 batch sizes and >= 2 lengths, got " +
                               std::to_string(rows.size()) + " samples / " + std::to_string(sizes.size()) +
                               " sizes / " + std::to_string(lengths.size()) + " lengths");
  const int m = (int)rows.size();
  std::vector<double> A((size_t)m * 4), b(m), A0, b0;
  for (int i = 0; i < m; ++i) {
    const double nn = rows[i]->batch_size, l = rows[i]->length;
    A[i * 4 + 0] = nn * l;
    A[i * 4 + 1] = nn;
    A[i * 4 + 2] = l;
    A[i * 4 + 3] = 1.0;
    b[i] = rows[i]->latency_s;
  }
  A0 = A;
  b0 = b;
  int perm[4] = {0, 1, 2, 3};
  double diag[4] = {0, 0, 0, 0}, maxpivot = 0.0;
  const int kmax = std::min(m, 4);
  for (int k = 0; k < kmax; ++k) {
    // pivot: the remaining column of largest norm below row k
    int pc = k;
    double best = -1.0;
    for (int c = k; c < 4; ++c) {
      double s2 = 0.0;
      for (int i = k; i < m; ++i) s2 += A[i * 4 + c] * A[i * 4 + c];
      if (s2 > best) {
        best = s2;
        pc = c;
      }
    }
    if (pc != k) {
      for (int i = 0; i < m; ++i) std::swap(A[i * 4 + k], A[i * 4 + pc]);
      std::swap(perm[k], perm[pc]);
    }
    // Householder reflector for A[k:, k]
    double norm = 0.0;
    for (int i = k; i < m; ++i) norm += A[i * 4 + k] * A[i * 4 + k];
    norm = std::sqrt(norm);
    if (norm == 0.0) {
      diag[k] = 0.0;
      continue;
    }
    const double alpha = A[k * 4 + k] > 0 ? -norm : norm;
    std::vector<double> v(m - k);
    for (int i = k; i < m; ++i) v[i - k] = A[i * 4 + k];
    v[0] -= alpha;
    double vv = 0.0;
    for (double x : v) vv += x * x;
    if (vv > 0.0) {
      for (int c = k; c < 4; ++c) {
        double d = 0.0;
        for (int i = k; i < m; ++i) d += v[i - k] * A[i * 4 + c];
        const double f = 2.0 * d / vv;
        for (int i = k; i < m; ++i) A[i * 4 + c] -= f * v[i - k];
      }
      double d = 0.0;
      for (int i = k; i < m; ++i) d += v[i - k] * b[i];
      const double f = 2.0 * d / vv;
      for (int i = k; i < m; ++i) b[i] -= f * v[i - k];
    }
    diag[k] = std::fabs(A[k * 4 + k]);
    maxpivot = std::max(maxpivot, diag[k]);
  }
  const double thr = maxpivot * (std::numeric_limits<double>::epsilon() * 4.0);
  int rank = 0;
  for (int k = 0; k < kmax; ++k) rank += diag[k] > thr;
  if (rank < 4)
    return scls::set_error(nullptr, SCLS_ERR_INSUFFICIENT_SAMPLES,
                           std::string(name) + " samples give a rank-deficient design matrix");
  double x[4];
  for (int k = 3; k >= 0; --k) {
    double s2 = b[k];
    for (int c = k + 1; c < 4; ++c) s2 -= A[k * 4 + c] * x[c];
    x[k] = s2 / A[k * 4 + k];
  }
  for (int k = 0; k < 4; ++k) out->c[perm[k]] = x[k];
  double rss = 0.0;
  for (int i = 0; i < m; ++i) {
    const double r =
        A0[i * 4 + 0] * out->c[0] + A0[i * 4 + 1] * out->c[1] + A0[i * 4 + 2] * out->c[2] + A0[i * 4 + 3] * out->c[3] -
        b0[i];
    rss += r * r;
  }
  out->rmse = std::sqrt(rss / (double)m);
  return SCLS_OK;
}

}  // namespace

extern "C" scls_status scls_fit_latency(const scls_profile_sample* samples, int64_t n, int32_t n_cap, int32_t l_cap,
                                        scls_latency* out) {
  if (!out || n < 0 || (n > 0 && !samples)) return scls::set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  PhaseFit pf, df;
  scls_status st = fit_phase(samples, n, 0, "prefill", &pf);
  if (st) return st;
  st = fit_phase(samples, n, 1, "decode", &df);
  if (st) return st;
  scls_latency m{};
  m.p1 = pf.c[0];
  m.p2 = pf.c[1];
  m.p3 = pf.c[2];
  m.p4 = pf.c[3];
  m.d1 = df.c[0];
  m.d2 = df.c[1];
  m.d3 = df.c[2];
  m.d4 = df.c[3];
  m.rmse_prefill = pf.rmse;
  m.rmse_decode = df.rmse;
  m.n_cap = n_cap;
  m.l_cap = l_cap;
  st = scls_validate_latency(&m);  // cost_model.cpp:156 validate(m)
  if (st) return st;
  *out = m;
  return SCLS_OK;
}
