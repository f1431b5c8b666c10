/* scls_oracle.c — CPU restatement of the reference SCLS path, plain C11.
 *
 * TEST INFRASTRUCTURE ONLY (see scls_oracle.h).  Every function cites the
 * reference file:line it restates (paths relative to
 * /root/reference/proj/core).  Floating-point expressions keep the
 * reference's exact association order; the build uses -ffp-contract=off,
 * matching the reference Release build (no -march, hence no FMA).
 */
#define _GNU_SOURCE
#include "scls_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "scls_loghash.h"

static _Thread_local char g_err[512];
static _Thread_local int64_t g_err_request = -1;

static scls_status fail(scls_status st, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return st;
}

size_t orc_last_error(char* buf, size_t cap) {
  size_t n = strlen(g_err);
  if (buf && cap) {
    size_t k = n < cap - 1 ? n : cap - 1;
    memcpy(buf, g_err, k);
    buf[k] = 0;
  }
  return n;
}
int64_t orc_last_request_id(void) { return g_err_request; }

/* ---- estimators ---------------------------------------------------------- */

/* cost_model.cpp:30-33 (Eq. 3) */
double orc_prefill_time(const scls_latency* m, int32_t n, int32_t l_in) {
  const double dn = n, dl = l_in;
  return m->p1 * dn * dl + m->p2 * dn + m->p3 * dl + m->p4;
}

/* cost_model.cpp:35-38 (Eq. 4) */
double orc_decode_step_time(const scls_latency* m, int32_t ctx, int32_t n) {
  const double dn = n, dl = ctx;
  return m->d1 * dn * dl + m->d2 * dn + m->d3 * dl + m->d4;
}

/* cost_model.cpp:40-47 (Eq. 2, arithmetic-series closed form) */
double orc_decode_time(const scls_latency* m, int32_t n, int32_t l_in, int32_t l_out) {
  if (l_out <= 0) return 0.0;
  const double k = l_out;
  const double sum_l = k * (double)l_in + k * (k + 1.0) / 2.0;
  return (m->d1 * n + m->d3) * sum_l + (m->d2 * n + m->d4) * k;
}

/* cost_model.cpp:49-51 (Eq. 1) */
double orc_batch_serve_time(const scls_latency* m, int32_t n, int32_t l_in, int32_t l_out) {
  return orc_prefill_time(m, n, l_in) + orc_decode_time(m, n, l_in, l_out);
}

/* memory_model.cpp:28-31 (Eq. 5) */
static double kv_cache_mem(double delta, int32_t n, int32_t l_in, int32_t l_out) {
  return ((double)l_in + (double)l_out) * (double)n * delta;
}

/* memory_model.cpp:54-59 (Eq. 6) */
static double available_mem(const scls_memory* m) { return m->m_cap - m->m_model - m->m_engine; }

/* memory_model.cpp:61-70 (Eq. 7/9, Alg. 2) */
int32_t orc_would_oom(const scls_memory* m, int32_t n, int32_t l_in, int32_t slice) {
  if (m->kind == SCLS_MEM_ANALYTIC)
    return kv_cache_mem(m->delta, n, l_in, slice) > m->zeta * available_mem(m);
  const int32_t total = l_in + slice;
  for (int i = 0; i < m->n_rules; ++i)
    if (total > m->rule_threshold[i]) return n > m->rule_max_n[i];
  return n > m->rule_max_n[m->n_rules - 1];
}

/* memory_model.cpp:72-90 (Eq. 8 with the boundary nudge) */
int32_t orc_max_batch_size(const scls_memory* m, int32_t l_in, int32_t slice) {
  if (m->kind == SCLS_MEM_RULE_TABLE) {
    const int32_t total = l_in + slice;
    for (int i = 0; i < m->n_rules; ++i)
      if (total > m->rule_threshold[i]) return m->rule_max_n[i];
    return m->rule_max_n[m->n_rules - 1];
  }
  const double per_request = m->delta * ((double)l_in + slice);
  const double quotient = floor(m->zeta * available_mem(m) / per_request);
  if (quotient >= 1e9) return 1000000000;
  int32_t n = (int32_t)quotient;
  if (n < 0) n = 0;
  while (n > 0 && orc_would_oom(m, n, l_in, slice)) --n;
  while (n < 1000000000 && !orc_would_oom(m, n + 1, l_in, slice)) ++n;
  return n;
}

/* sched_policies.cpp:59-61 (Eq. 12) */
double orc_next_interval(double lambda, double gamma, double min_load) {
  const double a = lambda * min_load;
  return a < gamma ? gamma : a; /* std::max(a, gamma) returns a unless a < gamma */
}

/* cost_model.cpp:55-87 */
static int negative_on_corner(double c1, double c2, double c3, double c4, int n_cap, int l_cap) {
  const int ns[2] = {1, n_cap}, ls[2] = {1, l_cap};
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      const double v = c1 * (double)ns[a] * (double)ls[b] + c2 * ns[a] + c3 * ls[b] + c4;
      if (!(v >= 0.0)) return 1;
    }
  return 0;
}

scls_status orc_validate_latency(const scls_latency* m) {
  const double c[8] = {m->p1, m->p2, m->p3, m->p4, m->d1, m->d2, m->d3, m->d4};
  for (int i = 0; i < 8; ++i)
    if (!isfinite(c[i]))
      return fail(SCLS_ERR_DEGENERATE_MODEL, "latency model has a non-finite coefficient");
  if (m->n_cap < 1 || m->l_cap < 1)
    return fail(SCLS_ERR_DEGENERATE_MODEL, "latency model operating range caps must be >= 1");
  if (negative_on_corner(m->p1, m->p2, m->p3, m->p4, m->n_cap, m->l_cap))
    return fail(SCLS_ERR_DEGENERATE_MODEL,
                "latency model predicts negative prefill time within operating range");
  if (negative_on_corner(m->d1, m->d2, m->d3, m->d4, m->n_cap, m->l_cap))
    return fail(SCLS_ERR_DEGENERATE_MODEL,
                "latency model predicts negative decode-step time within operating range");
  return SCLS_OK;
}

/* memory_model.cpp:92-120 */
scls_status orc_validate_memory(const scls_memory* m) {
  if (m->kind == SCLS_MEM_ANALYTIC) {
    const double v[5] = {m->m_cap, m->m_model, m->m_engine, m->delta, m->zeta};
    for (int i = 0; i < 5; ++i)
      if (!isfinite(v[i])) return fail(SCLS_ERR_ERROR, "memory model has a non-finite field");
    if (!(m->m_cap > m->m_model + m->m_engine))
      return fail(SCLS_ERR_ERROR, "memory model needs m_cap > m_model + m_engine");
    if (!(m->delta > 0.0)) return fail(SCLS_ERR_ERROR, "memory model needs delta > 0");
    if (!(m->zeta > 0.0 && m->zeta <= 1.0))
      return fail(SCLS_ERR_ERROR, "memory model needs zeta in (0, 1]");
    return SCLS_OK;
  }
  if (m->n_rules < 1) return fail(SCLS_ERR_ERROR, "rule-table memory model needs >= 1 row");
  for (int i = 0; i < m->n_rules; ++i) {
    if (m->rule_max_n[i] < 1) return fail(SCLS_ERR_ERROR, "rule-table max batch sizes must be >= 1");
    if (i > 0) {
      if (m->rule_threshold[i] >= m->rule_threshold[i - 1])
        return fail(SCLS_ERR_ERROR, "rule-table thresholds must be strictly decreasing");
      if (m->rule_max_n[i] < m->rule_max_n[i - 1])
        return fail(SCLS_ERR_ERROR,
                    "rule-table max batch sizes must not decrease as thresholds do");
    }
  }
  return SCLS_OK;
}

/* sched_policies.cpp:45-57 */
scls_status orc_validate_sched(const scls_sched_cfg* c) {
  if (!(c->lambda > 0.0 && c->lambda < 1.0)) return fail(SCLS_ERR_ERROR, "lambda must lie in (0, 1)");
  if (!(c->gamma > 0.0)) return fail(SCLS_ERR_ERROR, "gamma must be > 0");
  if (c->slice_len < 1) return fail(SCLS_ERR_ERROR, "slice_len must be >= 1");
  if (c->max_gen_limit < c->slice_len)
    return fail(SCLS_ERR_ERROR, "slice_len must not exceed max_gen_limit");
  if (c->fixed_batch_size < 1) return fail(SCLS_ERR_ERROR, "fixed_batch_size must be >= 1");
  if (c->max_concurrent < 1) return fail(SCLS_ERR_ERROR, "max_concurrent must be >= 1");
  if (c->worker_count < 1) return fail(SCLS_ERR_ERROR, "worker_count must be >= 1");
  return SCLS_OK;
}

/* ---- batcher ------------------------------------------------------------- */

typedef struct {
  int32_t eff;
  double arrival;
  int64_t id;
  int32_t idx;
} sort_item;

/* batcher.cpp:35-38: tuple (effective_input_len, arrival_time, id) < */
static int cmp_item(const void* pa, const void* pb) {
  const sort_item* a = (const sort_item*)pa;
  const sort_item* b = (const sort_item*)pb;
  if (a->eff != b->eff) return a->eff < b->eff ? -1 : 1;
  if (a->arrival < b->arrival) return -1;
  if (b->arrival < a->arrival) return 1;
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  return 0;
}

/* Core of batch_requests (batcher.cpp:26-87) over an already-built item
 * array; shared by the public entry point and the SCLS tick.  Outputs the
 * sorted items in place, the segment starts (seg[0..nb]) and nb. */
static scls_status batch_core(int32_t n, sort_item* items, int32_t slice_len,
                              const scls_latency* lat, const scls_memory* mem,
                              int32_t* seg, int64_t* nb_out) {
  *nb_out = 0;
  if (n == 0) return SCLS_OK;
  qsort(items, (size_t)n, sizeof *items, cmp_item); /* strict total order: == std::sort */
  /* batcher.cpp:40-46 singleton feasibility, first offender in sorted order */
  for (int32_t i = 0; i < n; ++i) {
    if (orc_would_oom(mem, 1, items[i].eff, slice_len)) {
      g_err_request = items[i].id;
      snprintf(g_err, sizeof g_err,
               "request %lld does not fit memory even as a singleton batch",
               (long long)items[i].id);
      return SCLS_ERR_INFEASIBLE_REQUEST;
    }
  }
  /* batcher.cpp:48-67 the DP (Eq. 10) */
  double* total = (double*)calloc((size_t)(uint32_t)n + 1, sizeof(double));
  int32_t* split = (int32_t*)calloc((size_t)(uint32_t)n + 1, sizeof(int32_t));
  for (int32_t i = 1; i <= n; ++i) {
    const int32_t len_i = items[i - 1].eff;
    split[i] = i - 1;
    total[i] = total[i - 1] + orc_batch_serve_time(lat, 1, len_i, slice_len);
    for (int32_t j = i - 1; j > 0 && !orc_would_oom(mem, i - j + 1, len_i, slice_len); --j) {
      const double t = total[j - 1] + orc_batch_serve_time(lat, i - j + 1, len_i, slice_len);
      if (t < total[i]) {
        total[i] = t;
        split[i] = j - 1;
      }
    }
  }
  /* batcher.cpp:69-73 backtrack, then ascending segment order */
  int64_t nb = 0;
  for (int32_t i = n; i > 0; i = split[i]) ++nb;
  int64_t b = nb;
  seg[nb] = n;
  for (int32_t i = n; i > 0; i = split[i]) seg[--b] = split[i];
  free(total);
  free(split);
  *nb_out = nb;
  return SCLS_OK;
}

/* batcher.h:40-43 / batcher.cpp:26-87 */
scls_status orc_batch_requests(int64_t n, const int32_t* eff_len, const double* arrival,
                               const int64_t* id, int32_t slice_len,
                               const scls_latency* lat, const scls_memory* mem,
                               int64_t first_batch_id, int64_t* n_batches,
                               int32_t* seg_begin, int32_t* l_in, double* est,
                               int64_t* batch_id, int64_t* member_id) {
  *n_batches = 0;
  if (n == 0) {
    seg_begin[0] = 0;
    return SCLS_OK;
  }
  sort_item* items = (sort_item*)malloc((size_t)n * sizeof *items);
  for (int64_t i = 0; i < n; ++i)
    items[i] = (sort_item){eff_len[i], arrival[i], id[i], (int32_t)i};
  int64_t nb = 0;
  scls_status st = batch_core((int32_t)n, items, slice_len, lat, mem, seg_begin, &nb);
  if (st == SCLS_OK) {
    /* batcher.cpp:75-86 emit: id, l_in = last member's eff, est = c(l_in, size) */
    for (int64_t b = 0; b < nb; ++b) {
      const int32_t beg = seg_begin[b], end = seg_begin[b + 1];
      batch_id[b] = first_batch_id + b;
      l_in[b] = items[end - 1].eff;
      est[b] = orc_batch_serve_time(lat, end - beg, l_in[b], slice_len);
    }
    for (int64_t p = 0; p < n; ++p) member_id[p] = items[p].id;
    *n_batches = nb;
  }
  free(items);
  return st;
}

/* ---- offloader ----------------------------------------------------------- */

typedef struct {
  double est;
  int64_t idx;
} off_item;

/* offloader.cpp:34-37: stable_sort by est descending == sort by (est desc, index asc) */
static int cmp_off(const void* pa, const void* pb) {
  const off_item* a = (const off_item*)pa;
  const off_item* b = (const off_item*)pb;
  if (a->est > b->est) return -1;
  if (b->est > a->est) return 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

/* offloader.cpp:25-54 (Eq. 11, max-min placement); loads/ids mutated in place */
static scls_status offload_core(int64_t nb, const int64_t* batch_id, const double* est,
                                int32_t nw, const int32_t* wid, double* load,
                                int64_t* out_b, int32_t* out_w) {
  if (nb == 0) return SCLS_OK;
  if (nw == 0) return fail(SCLS_ERR_NO_WORKERS, "cannot offload batches: no workers configured");
  off_item* order = (off_item*)malloc((size_t)nb * sizeof *order);
  for (int64_t i = 0; i < nb; ++i) order[i] = (off_item){est[i], i};
  qsort(order, (size_t)nb, sizeof *order, cmp_off);
  for (int64_t k = 0; k < nb; ++k) {
    int32_t t = 0;
    for (int32_t w = 0; w < nw; ++w)
      if (load[w] < load[t] || (load[w] == load[t] && wid[w] < wid[t])) t = w;
    load[t] += est[order[k].idx];
    out_b[k] = batch_id[order[k].idx];
    out_w[k] = wid[t];
  }
  free(order);
  return SCLS_OK;
}

scls_status orc_offload(int64_t nb, const int64_t* batch_id, const double* est,
                        int32_t n_workers, const int32_t* worker_id, double* load_inout,
                        int64_t* out_batch_id, int32_t* out_worker) {
  return offload_core(nb, batch_id, est, n_workers, worker_id, load_inout, out_batch_id,
                      out_worker);
}

/* ---- workload (workload.cpp:100-181) ------------------------------------- */

typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

/* std::mt19937_64 (the standard's parameters; seeding per [rand.eng.mers]) */
static void mt_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* workload.cpp:100-102 */
static double next_uniform(mt64* g) { return (double)(mt_next(g) >> 11) * 0x1.0p-53; }

/* workload.cpp:120-123 */
static int uniform_int(int lo, int hi, mt64* g) {
  const double u = next_uniform(g);
  return lo + (int)(u * ((double)hi - lo + 1.0));
}

/* workload.cpp:125-129 */
static int clamp_length(long long v, int limit) {
  if (v < 1) return 1;
  if (v > limit) return limit;
  return (int)v;
}

/* workload.cpp:133-161 */
static int sample_length(const scls_length_dist* d, int limit, mt64* g) {
  switch (d->kind) {
    case SCLS_DIST_UNIFORM:
      return clamp_length(uniform_int(d->lo, d->hi, g), limit);
    case SCLS_DIST_LOGNORMAL: {
      /* workload.cpp:112-118 Box-Muller */
      const double u1 = 1.0 - next_uniform(g);
      const double u2 = next_uniform(g);
      const double z = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
      const double raw = exp(d->mu + d->sigma * z);
      const long long rounded = raw > 1e18 ? (long long)1e18 : llround(raw);
      return clamp_length(rounded < d->cap ? rounded : d->cap, limit);
    }
    default: {
      const double u = next_uniform(g);
      double cdf = 0.0;
      int bucket = d->n_buckets - 1;
      for (int i = 0; i < d->n_buckets; ++i) {
        cdf += d->weights[i];
        if (u < cdf) {
          bucket = i;
          break;
        }
      }
      return clamp_length(uniform_int(d->edges[bucket], d->edges[bucket + 1], g), limit);
    }
  }
}

/* workload.cpp:56-98 */
static scls_status validate_dist(const scls_length_dist* d) {
  switch (d->kind) {
    case SCLS_DIST_UNIFORM:
      if (d->lo < 1 || d->hi < d->lo)
        return fail(SCLS_ERR_ERROR, "uniform length distribution requires 1 <= lo <= hi");
      return SCLS_OK;
    case SCLS_DIST_LOGNORMAL:
      if (!(d->sigma > 0.0) || d->cap < 1)
        return fail(SCLS_ERR_ERROR, "log-normal length distribution requires sigma > 0 and cap >= 1");
      return SCLS_OK;
    default: {
      if (d->n_buckets < 1 || d->n_buckets > SCLS_MAX_BUCKETS)
        return fail(SCLS_ERR_ERROR, "histogram needs k weights and k+1 edges, k >= 1");
      for (int i = 0; i < d->n_buckets; ++i)
        if (d->edges[i] < 1 || d->edges[i] > d->edges[i + 1])
          return fail(SCLS_ERR_ERROR, "histogram edges must be >= 1 and non-decreasing");
      double total = 0.0;
      for (int i = 0; i < d->n_buckets; ++i) {
        if (d->weights[i] < 0.0) return fail(SCLS_ERR_ERROR, "histogram weights must be non-negative");
        total += d->weights[i];
      }
      if (fabs(total - 1.0) > 1e-9) return fail(SCLS_ERR_ERROR, "histogram weights must sum to 1 within 1e-9");
      return SCLS_OK;
    }
  }
}

/* workload.cpp:106-110 + 163-181 */
scls_status orc_generate(const scls_workload_spec* s, int64_t cap, int64_t* n, double* arrival,
                         int32_t* input_len, int32_t* gen_len) {
  *n = 0;
  if (!(s->rate > 0.0)) return fail(SCLS_ERR_ERROR, "workload rate must be > 0");
  if (s->duration_s < 0.0) return fail(SCLS_ERR_ERROR, "workload duration must be >= 0");
  if (s->max_input_limit < 1 || s->max_gen_limit < 1) return fail(SCLS_ERR_ERROR, "length limits must be >= 1");
  scls_status st = validate_dist(&s->input_len_dist);
  if (st) return st;
  if ((st = validate_dist(&s->gen_len_dist))) return st;
  mt64 g;
  mt_seed(&g, s->seed);
  double clock = 0.0;
  int64_t k = 0;
  for (;;) {
    clock += -log(1.0 - next_uniform(&g)) / s->rate;
    if (clock > s->duration_s) break;
    const int32_t in = sample_length(&s->input_len_dist, s->max_input_limit, &g);
    const int32_t gl = sample_length(&s->gen_len_dist, s->max_gen_limit, &g);
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

/* bench_batcher.cpp:27-42 make_pool (the reference microbenchmark's pool) */
scls_status orc_make_pool(int64_t n, uint64_t seed, int32_t* input_len, double* arrival,
                          int64_t* id, int32_t* gen_len) {
  mt64 g;
  mt_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) {
    id[i] = i;
    arrival[i] = next_uniform(&g) * 100.0;
    input_len[i] = 1 + (int)(next_uniform(&g) * 1024.0);
    const int gl = 1 + (int)(next_uniform(&g) * 1024.0);
    if (gen_len) gen_len[i] = gl;
  }
  return SCLS_OK;
}

/* ---- simulator (sim_engine.cpp, sched_policies.cpp) ---------------------- */

#define GROW(ptr, len, cap)                                                   \
  do {                                                                        \
    if ((len) >= (cap)) {                                                     \
      (cap) = (cap) ? 2 * (cap) : 64;                                         \
      (ptr) = realloc((ptr), (size_t)(cap) * sizeof *(ptr));                  \
    }                                                                         \
  } while (0)

enum { EV_ARRIVAL, EV_TICK, EV_BATCH_DONE, EV_POLICY, EV_END }; /* sim_engine.h:33 */
enum { K_ARRIVAL, K_TICK, K_DISPATCH, K_BATCH_START, K_BATCH_END, K_COMPLETE }; /* event_log.h:27-34 */

typedef struct { double time; uint64_t seq; int kind; int64_t request; int32_t worker; } sim_event;

typedef struct {
  int64_t id;
  int64_t* req;
  int32_t n, l_in, planned_l_out;
  double est;
} batch_t;

typedef struct { batch_t b; int32_t served; } queued_batch;

typedef struct {
  queued_batch* q;
  int64_t qhead, qlen, qcap;
  int has_in_flight;
  batch_t in_flight;
  int32_t in_flight_l_out;
  double busy_until;
  double load;
} worker_t;

typedef struct { int64_t* v; int64_t head, len, cap; } deque_t;

static void dq_push(deque_t* d, int64_t x) {
  if (d->head + d->len >= d->cap) {
    if (d->head > 0 && d->len < d->cap / 2) {
      memmove(d->v, d->v + d->head, (size_t)d->len * sizeof *d->v);
      d->head = 0;
    } else {
      d->cap = d->cap ? 2 * d->cap : 64;
      d->v = realloc(d->v, (size_t)d->cap * sizeof *d->v);
    }
  }
  d->v[d->head + d->len++] = x;
}
static int64_t dq_pop(deque_t* d) {
  int64_t x = d->v[d->head++];
  --d->len;
  return x;
}

typedef struct {
  int64_t* running; int32_t n_running, cap_running;
  deque_t waiting;
  int boundary_scheduled;
  int64_t segment_id;
  int32_t segment_n, segment_l_in, segment_iterations;
} ils_inst;

typedef struct {
  /* config */
  const scls_sched_cfg* cfg;
  const scls_latency* lat;
  const scls_memory* mem;
  /* requests (request.h:32-49) */
  int64_t n;
  const double* arrival;
  const int32_t* orig;
  const int32_t* true_gen;
  int32_t* generated;
  int32_t* slices;
  unsigned char* has_first_dispatch;
  /* engine */
  double clock;
  uint64_t next_seq;
  sim_event* heap; int64_t heap_len, heap_cap;
  worker_t* workers;
  int64_t completed;
  /* policy state */
  int64_t next_batch_id;
  int64_t* pool; int64_t pool_len, pool_cap; /* SCLS */
  deque_t* pending; int64_t rr;              /* SLS */
  ils_inst* inst;                            /* ILS */
  /* event log */
  scls_event_record* rec; int64_t rec_len, rec_cap;
  scls_member* mem_rec; int64_t mem_len, mem_cap;
} sim_t;

/* sim_engine.h:100-105: (time, seq) min-order */
static int ev_before(const sim_event* a, const sim_event* b) {
  if (a->time != b->time) return a->time < b->time;
  return a->seq < b->seq;
}

/* sim_engine.cpp:43-46 */
static void push_event(sim_t* s, double time, int kind, int64_t req, int32_t worker) {
  GROW(s->heap, s->heap_len, s->heap_cap);
  sim_event e = {time, s->next_seq++, kind, req, worker};
  int64_t i = s->heap_len++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!ev_before(&e, &s->heap[p])) break;
    s->heap[i] = s->heap[p];
    i = p;
  }
  s->heap[i] = e;
}

static sim_event pop_event(sim_t* s) {
  sim_event top = s->heap[0];
  sim_event last = s->heap[--s->heap_len];
  int64_t i = 0;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= s->heap_len) break;
    if (c + 1 < s->heap_len && ev_before(&s->heap[c + 1], &s->heap[c])) ++c;
    if (!ev_before(&s->heap[c], &last)) break;
    s->heap[i] = s->heap[c];
    i = c;
  }
  if (s->heap_len > 0) s->heap[i] = last;
  return top;
}

static scls_event_record* add_rec(sim_t* s, int kind) {
  GROW(s->rec, s->rec_len, s->rec_cap);
  scls_event_record* r = &s->rec[s->rec_len++];
  memset(r, 0, sizeof *r);
  r->t = s->clock;
  r->kind = kind;
  r->request = -1;
  r->worker = -1;
  r->batch = -1;
  r->member_offset = s->mem_len;
  return r;
}

static void add_member(sim_t* s, scls_event_record* r, int64_t req, int32_t eff, int32_t pad,
                       int32_t gen, int32_t invalid) {
  GROW(s->mem_rec, s->mem_len, s->mem_cap);
  s->mem_rec[s->mem_len++] = (scls_member){req, eff, pad, gen, invalid};
  r->member_count++;
}

static int32_t eff_len(const sim_t* s, int64_t id) { return s->orig[id] + s->generated[id]; }
static int32_t remaining(const sim_t* s, int64_t id) { return s->true_gen[id] - s->generated[id]; }
static int is_done(const sim_t* s, int64_t id) { return s->generated[id] >= s->true_gen[id]; }

/* sim_engine.cpp:63-84 */
static void start_next_batch(sim_t* s, int32_t wi) {
  worker_t* w = &s->workers[wi];
  if (w->has_in_flight || w->qlen == 0) return;
  queued_batch qb = w->q[w->qhead++];
  --w->qlen;
  scls_event_record* r = add_rec(s, K_BATCH_START);
  r->worker = wi;
  r->batch = qb.b.id;
  r->n = qb.b.n;
  r->l_in = qb.b.l_in;
  const double serve_s = orc_batch_serve_time(s->lat, qb.b.n, qb.b.l_in, qb.served);
  w->busy_until = s->clock + serve_s;
  w->in_flight = qb.b;
  w->has_in_flight = 1;
  w->in_flight_l_out = qb.served;
  push_event(s, w->busy_until, EV_BATCH_DONE, -1, wi);
}

/* sim_engine.cpp:56-61 */
static void enqueue_batch(sim_t* s, int32_t wi, batch_t b, int32_t served) {
  worker_t* w = &s->workers[wi];
  if (w->qhead + w->qlen >= w->qcap) {
    if (w->qhead > 0) {
      memmove(w->q, w->q + w->qhead, (size_t)w->qlen * sizeof *w->q);
      w->qhead = 0;
    }
    if (w->qlen >= w->qcap) {
      w->qcap = w->qcap ? 2 * w->qcap : 16;
      w->q = realloc(w->q, (size_t)w->qcap * sizeof *w->q);
    }
  }
  w->q[w->qhead + w->qlen++] = (queued_batch){b, served};
  if (!w->has_in_flight) start_next_batch(s, wi);
}

/* sim_engine.cpp:86-99 */
static void complete_request(sim_t* s, int64_t id, int32_t wi, double* completion) {
  completion[id] = s->clock;
  ++s->completed;
  scls_event_record* r = add_rec(s, K_COMPLETE);
  r->request = id;
  r->worker = wi;
  r->response_s = s->clock - s->arrival[id];
  r->slices = s->slices[id];
}

/* sched_policies.cpp:72-80 */
static int32_t slice_served_l_out(const sim_t* s, const batch_t* b, int32_t slice_len) {
  int32_t served = 0;
  for (int32_t i = 0; i < b->n; ++i) {
    int32_t rem = remaining(s, b->req[i]);
    int32_t v = rem < slice_len ? rem : slice_len;
    if (v > served) served = v;
  }
  return served;
}

/* sched_policies.cpp:90-147 SCLS tick */
static scls_status scls_on_tick(sim_t* s) {
  const scls_sched_cfg* cfg = s->cfg;
  const int32_t W = cfg->worker_count;
  int64_t nb = 0;
  batch_t* batches = NULL;
  if (s->pool_len > 0) {
    const int32_t n = (int32_t)s->pool_len;
    sort_item* items = (sort_item*)malloc((size_t)n * sizeof *items);
    for (int32_t i = 0; i < n; ++i) {
      const int64_t id = s->pool[i];
      items[i] = (sort_item){eff_len(s, id), s->arrival[id], id, i};
    }
    s->pool_len = 0;
    int32_t* seg = (int32_t*)malloc(((size_t)n + 1) * sizeof *seg);
    scls_status st = batch_core(n, items, cfg->slice_len, s->lat, s->mem, seg, &nb);
    if (st) {
      free(items);
      free(seg);
      return st;
    }
    batches = (batch_t*)malloc((size_t)nb * sizeof *batches);
    for (int64_t b = 0; b < nb; ++b) {
      const int32_t beg = seg[b], end = seg[b + 1];
      batch_t* bt = &batches[b];
      bt->id = s->next_batch_id + b;
      bt->n = end - beg;
      bt->req = (int64_t*)malloc((size_t)bt->n * sizeof(int64_t));
      for (int32_t k = beg; k < end; ++k) bt->req[k - beg] = items[k].id;
      bt->l_in = items[end - 1].eff;
      bt->planned_l_out = cfg->slice_len;
      bt->est = orc_batch_serve_time(s->lat, bt->n, bt->l_in, cfg->slice_len);
    }
    s->next_batch_id += nb;
    free(items);
    free(seg);
  }
  /* sched_policies.cpp:104-112 offload against the current load estimates */
  double* load = (double*)malloc((size_t)W * sizeof(double));
  int32_t* wid = (int32_t*)malloc((size_t)W * sizeof(int32_t));
  for (int32_t w = 0; w < W; ++w) {
    load[w] = s->workers[w].load;
    wid[w] = w;
  }
  int64_t* ob = (int64_t*)malloc(((size_t)nb + 1) * sizeof(int64_t));
  int32_t* ow = (int32_t*)malloc(((size_t)nb + 1) * sizeof(int32_t));
  if (nb > 0) {
    int64_t* bid = (int64_t*)malloc((size_t)nb * sizeof(int64_t));
    double* est = (double*)malloc((size_t)nb * sizeof(double));
    for (int64_t b = 0; b < nb; ++b) {
      bid[b] = batches[b].id;
      est[b] = batches[b].est;
    }
    offload_core(nb, bid, est, W, wid, load, ob, ow);
    free(bid);
    free(est);
  }
  for (int32_t w = 0; w < W; ++w) s->workers[w].load = load[w];
  /* sched_policies.cpp:114-132 dispatch in assignment order */
  for (int64_t k = 0; k < nb; ++k) {
    batch_t* b = &batches[ob[k] - batches[0].id];
    scls_event_record* r = add_rec(s, K_DISPATCH);
    r->worker = ow[k];
    r->batch = b->id;
    r->n = b->n;
    r->l_in = b->l_in;
    r->planned_l_out = b->planned_l_out;
    r->est_serve_s = b->est;
    for (int32_t i = 0; i < b->n; ++i) s->has_first_dispatch[b->req[i]] = 1;
    const int32_t served = slice_served_l_out(s, b, cfg->slice_len);
    enqueue_batch(s, ow[k], *b, served);
  }
  /* sched_policies.cpp:134-146 */
  double min_load = INFINITY;
  for (int32_t w = 0; w < W; ++w)
    if (s->workers[w].load < min_load) min_load = s->workers[w].load;
  const double interval = orc_next_interval(cfg->lambda, cfg->gamma, min_load);
  scls_event_record* r = add_rec(s, K_TICK);
  r->n = (int32_t)nb;
  r->next_interval_s = interval;
  push_event(s, s->clock + interval, EV_TICK, -1, -1);
  free(load);
  free(wid);
  free(ob);
  free(ow);
  free(batches);
  return SCLS_OK;
}

/* sched_policies.cpp:149-188 */
static void scls_on_batch_done(sim_t* s, int32_t wi, batch_t* b, int32_t served,
                               double* completion) {
  scls_event_record* end = add_rec(s, K_BATCH_END);
  end->worker = wi;
  end->batch = b->id;
  end->n = b->n;
  end->l_in = b->l_in;
  end->planned_l_out = b->planned_l_out;
  end->served_l_out = served;
  int64_t* finished = (int64_t*)malloc((size_t)b->n * sizeof(int64_t));
  int32_t nf = 0;
  for (int32_t i = 0; i < b->n; ++i) {
    const int64_t id = b->req[i];
    const int32_t eff = eff_len(s, id);
    const int32_t rem = remaining(s, id);
    const int32_t gen = rem < served ? rem : served;
    add_member(s, &s->rec[s->rec_len - 1], id, eff, b->l_in - eff, gen, served - gen);
    s->generated[id] += gen;
    s->slices[id] += 1;
    if (is_done(s, id) || s->generated[id] >= s->cfg->max_gen_limit) {
      finished[nf++] = id;
    } else {
      GROW(s->pool, s->pool_len, s->pool_cap);
      s->pool[s->pool_len++] = id;
    }
  }
  (void)end;
  for (int32_t i = 0; i < nf; ++i) complete_request(s, finished[i], wi, completion);
  free(finished);
  /* offloader.cpp:56-59 complete_batch */
  worker_t* w = &s->workers[wi];
  w->load -= b->est;
  if (w->load < 0.0) w->load = 0.0;
}

/* sched_policies.cpp:207-243 */
static void sls_try_dispatch(sim_t* s, int32_t wi) {
  worker_t* w = &s->workers[wi];
  deque_t* q = &s->pending[wi];
  if (w->has_in_flight || w->qlen != 0 || q->len == 0) return;
  const scls_sched_cfg* cfg = s->cfg;
  batch_t b;
  b.id = s->next_batch_id++;
  const int32_t take = cfg->fixed_batch_size < q->len ? cfg->fixed_batch_size : (int32_t)q->len;
  b.req = (int64_t*)malloc((size_t)take * sizeof(int64_t));
  b.n = take;
  b.l_in = 0;
  int32_t l_out = 0;
  for (int32_t i = 0; i < take; ++i) {
    const int64_t id = dq_pop(q);
    b.req[i] = id;
    if (s->orig[id] > b.l_in) b.l_in = s->orig[id];
    const int32_t g = s->true_gen[id] < cfg->max_gen_limit ? s->true_gen[id] : cfg->max_gen_limit;
    if (g > l_out) l_out = g;
    s->has_first_dispatch[id] = 1;
  }
  b.planned_l_out = l_out;
  b.est = orc_batch_serve_time(s->lat, b.n, b.l_in, l_out);
  scls_event_record* r = add_rec(s, K_DISPATCH);
  r->worker = wi;
  r->batch = b.id;
  r->n = b.n;
  r->l_in = b.l_in;
  r->planned_l_out = b.planned_l_out;
  r->est_serve_s = b.est;
  enqueue_batch(s, wi, b, l_out);
}

/* sched_policies.cpp:245-273 */
static void sls_on_batch_done(sim_t* s, int32_t wi, batch_t* b, int32_t served,
                              double* completion) {
  scls_event_record* end = add_rec(s, K_BATCH_END);
  end->worker = wi;
  end->batch = b->id;
  end->n = b->n;
  end->l_in = b->l_in;
  end->planned_l_out = b->planned_l_out;
  end->served_l_out = served;
  const int64_t ridx = s->rec_len - 1;
  for (int32_t i = 0; i < b->n; ++i) {
    const int64_t id = b->req[i];
    const int32_t g = s->true_gen[id] < s->cfg->max_gen_limit ? s->true_gen[id] : s->cfg->max_gen_limit;
    add_member(s, &s->rec[ridx], id, s->orig[id], b->l_in - s->orig[id], g, served - g);
    s->generated[id] = g;
    s->slices[id] = 1;
  }
  for (int32_t i = 0; i < b->n; ++i) complete_request(s, b->req[i], wi, completion);
  sls_try_dispatch(s, wi);
}

/* sched_policies.cpp:292-391 ILS iteration boundary */
static void ils_on_policy_event(sim_t* s, int32_t wi, double* completion) {
  const scls_sched_cfg* cfg = s->cfg;
  ils_inst* in = &s->inst[wi];
  const double now = s->clock;
  int64_t* exits = (int64_t*)malloc(((size_t)in->n_running + 1) * sizeof(int64_t));
  int32_t ne = 0;
  if (in->n_running > 0) {
    in->segment_iterations += 1;
    for (int32_t i = 0; i < in->n_running; ++i) {
      const int64_t id = in->running[i];
      s->generated[id] += 1;
      if (is_done(s, id) || s->generated[id] >= cfg->max_gen_limit) exits[ne++] = id;
    }
    /* order-preserving erase of every exit */
    int32_t k = 0;
    for (int32_t i = 0; i < in->n_running; ++i) {
      const int64_t id = in->running[i];
      int gone = 0;
      for (int32_t e = 0; e < ne; ++e) gone |= exits[e] == id;
      if (!gone) in->running[k++] = id;
    }
    in->n_running = k;
  }
  int64_t* joins = (int64_t*)malloc(((size_t)cfg->max_concurrent + 1) * sizeof(int64_t));
  int32_t nj = 0;
  while (in->n_running < cfg->max_concurrent && in->waiting.len > 0) {
    const int64_t id = dq_pop(&in->waiting);
    GROW(in->running, in->n_running, in->cap_running);
    in->running[in->n_running++] = id;
    joins[nj++] = id;
  }
  const int changed = ne > 0 || nj > 0;
  if (changed && in->segment_id >= 0 && in->segment_iterations > 0) {
    scls_event_record* r = add_rec(s, K_BATCH_END);
    r->worker = wi;
    r->batch = in->segment_id;
    r->n = in->segment_n;
    r->l_in = in->segment_l_in;
    r->planned_l_out = in->segment_iterations;
    r->served_l_out = in->segment_iterations;
    in->segment_id = -1;
  }
  for (int32_t e = 0; e < ne; ++e) complete_request(s, exits[e], wi, completion);
  if (in->n_running == 0) {
    in->boundary_scheduled = 0;
    free(exits);
    free(joins);
    return;
  }
  int32_t max_ctx = 0;
  for (int32_t i = 0; i < in->n_running; ++i) {
    const int32_t e = eff_len(s, in->running[i]);
    if (e > max_ctx) max_ctx = e;
  }
  if (changed) {
    in->segment_id = s->next_batch_id++;
    in->segment_n = in->n_running;
    in->segment_l_in = max_ctx;
    in->segment_iterations = 0;
    scls_event_record* r = add_rec(s, K_BATCH_START);
    r->worker = wi;
    r->batch = in->segment_id;
    r->n = in->segment_n;
    r->l_in = in->segment_l_in;
  }
  double it = orc_decode_step_time(s->lat, max_ctx, in->n_running);
  for (int32_t j = 0; j < nj; ++j) {
    const int64_t id = joins[j];
    s->slices[id] = 1;
    s->has_first_dispatch[id] = 1;
    it += orc_prefill_time(s->lat, 1, s->orig[id]);
    scls_event_record* r = add_rec(s, K_DISPATCH);
    r->worker = wi;
    r->batch = in->segment_id;
    r->request = id;
    r->n = 1;
    r->l_in = s->orig[id];
    r->planned_l_out = remaining(s, id);
    r->est_serve_s = 0.0;
  }
  push_event(s, now + it, EV_POLICY, -1, wi);
  in->boundary_scheduled = 1;
  free(exits);
  free(joins);
}

static int cmp_dbl(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y);
}

/* metrics.cpp:30-117 over the log s->rec; fills r (and the histogram) */
static scls_status compute_metrics(const sim_t* s, int32_t W, scls_trace_result* r,
                                   int32_t hist_bins, int64_t* hist) {
  uint64_t hc = SCLS_FNV_OFFSET, hd = SCLS_FNV_OFFSET, ht = SCLS_FNV_OFFSET, hl = SCLS_FNV_OFFSET;
  double first_arrival = INFINITY, last_completion = -INFINITY;
  double* responses = (double*)malloc(((size_t)s->n + 1) * sizeof(double));
  double* last_end = (double*)calloc((size_t)W + 1, sizeof(double));
  int64_t nresp = 0, pad = 0, inval = 0, bc = 0, bm = 0, er = 0, nd = 0, nt = 0;
  for (int64_t k = 0; k < s->rec_len; ++k) {
    const scls_event_record* e = &s->rec[k];
    hl = scls_hash_record(hl, e->kind, e->t, e->request, e->worker, e->batch, e->n, e->l_in,
                          e->planned_l_out, e->served_l_out, e->est_serve_s, e->input_len,
                          e->gen_len, e->response_s, e->slices, e->next_interval_s,
                          e->member_count);
    for (int32_t m = 0; m < e->member_count; ++m) {
      const scls_member* mm = &s->mem_rec[e->member_offset + m];
      hl = scls_hash_member(hl, mm->request, mm->effective_input, mm->pad, mm->gen, mm->invalid);
    }
    switch (e->kind) {
      case K_ARRIVAL:
        if (e->t < first_arrival) first_arrival = e->t;
        break;
      case K_COMPLETE:
        if (e->t > last_completion) last_completion = e->t;
        responses[nresp++] = e->response_s;
        if (hist && e->slices >= 0 && e->slices < hist_bins) hist[e->slices] += 1;
        hc = scls_fnv_bytes(hc, (uint64_t)e->request);
        ht = scls_fnv_bytes(ht, scls_dbits(e->t));
        break;
      case K_DISPATCH:
        hd = scls_fnv_bytes(hd, (uint64_t)e->batch);
        hd = scls_fnv_bytes(hd, (uint64_t)(int64_t)e->worker);
        hd = scls_fnv_bytes(hd, (uint64_t)(int64_t)e->n);
        hd = scls_fnv_bytes(hd, (uint64_t)(int64_t)e->l_in);
        ++nd;
        break;
      case K_TICK: ++nt; break;
      case K_BATCH_END:
        ++bc;
        bm += e->n;
        if (e->served_l_out < e->planned_l_out) ++er;
        for (int32_t m = 0; m < e->member_count; ++m) {
          pad += s->mem_rec[e->member_offset + m].pad;
          inval += s->mem_rec[e->member_offset + m].invalid;
        }
        if (e->worker >= 0 && e->worker < W && e->t > last_end[e->worker]) last_end[e->worker] = e->t;
        break;
      default: break;
    }
  }
  r->h_complete_ids = hc; r->h_dispatch = hd; r->h_complete_t = ht; r->h_log = hl;
  r->n_events = s->rec_len; r->n_dispatches = nd; r->n_ticks = nt;
  r->total_pad = pad; r->total_invalid = inval; r->batch_count = bc; r->batch_members = bm;
  r->early_returns = er; r->completed = nresp;
  r->sim_clock = s->rec_len ? s->rec[s->rec_len - 1].t : 0.0;
  scls_status st = SCLS_OK;
  if (s->rec_len == 0) {
    st = fail(SCLS_ERR_EMPTY_LOG, "cannot compute metrics from an empty log");
  } else if (nresp == 0) {
    st = fail(SCLS_ERR_EMPTY_LOG, "log contains no completed requests");
  } else {
    const double span = last_completion - first_arrival;
    const double completed = (double)nresp;
    r->throughput = span > 0.0 ? completed / span : 0.0;
    double sum = 0.0;
    for (int64_t i = 0; i < nresp; ++i) sum += responses[i];
    r->avg_response_s = sum / completed;
    qsort(responses, (size_t)nresp, sizeof(double), cmp_dbl);
    size_t rank = (size_t)ceil(0.95 * (double)nresp);
    r->p95_response_s = responses[(rank > 1 ? rank : 1) - 1];
    if (W > 0) {
      double mean = 0.0;
      for (int32_t w = 0; w < W; ++w) mean += last_end[w];
      mean /= (double)W;
      double var = 0.0;
      for (int32_t w = 0; w < W; ++w) var += (last_end[w] - mean) * (last_end[w] - mean);
      var /= (double)W;
      r->ct_std_s = sqrt(var);
    }
    r->avg_pad_tokens = (double)pad / completed;
    r->avg_invalid_tokens = (double)inval / completed;
    r->avg_batch_size = bc > 0 ? (double)bm / (double)bc : 0.0;
    r->early_return_ratio = bc > 0 ? (double)er / (double)bc : 0.0;
  }
  free(responses);
  free(last_end);
  return st;
}

/* Simulator::Simulator + run (sim_engine.cpp:26-41, 101-168) for one trace */
static void simulate_one(int64_t n, const double* arrival, const int32_t* in_len,
                         const int32_t* gen_len, const scls_sched_cfg* cfg,
                         const scls_latency* lat, const scls_memory* mem,
                         scls_trace_result* r, int32_t hist_bins, int64_t* hist,
                         scls_event_log* log, int64_t trace) {
  memset(r, 0, sizeof *r);
  r->worker_count = cfg->worker_count;
  r->error_request_id = -1;
  r->n_requests = n;
  if (hist) memset(hist, 0, (size_t)hist_bins * sizeof(int64_t));
  g_err_request = -1;
  scls_status st;
  if ((st = orc_validate_sched(cfg)) || (st = orc_validate_latency(lat)) ||
      (st = orc_validate_memory(mem))) {
    r->status = st;
    return;
  }
  if (!(cfg->horizon_s > 0.0)) {
    r->status = fail(SCLS_ERR_ERROR, "simulation horizon must be > 0");
    return;
  }
  /* sim_engine.cpp:102-114: stable sort by (arrival, id) must leave ids 0..n-1 */
  for (int64_t i = 1; i < n; ++i)
    if (arrival[i] < arrival[i - 1]) {
      r->status = fail(SCLS_ERR_ERROR, "workload request ids must be 0..n-1 in arrival order");
      return;
    }
  const int32_t W = cfg->worker_count;
  sim_t s;
  memset(&s, 0, sizeof s);
  s.cfg = cfg; s.lat = lat; s.mem = mem; s.n = n;
  s.arrival = arrival; s.orig = in_len; s.true_gen = gen_len;
  s.generated = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  s.slices = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  s.has_first_dispatch = (unsigned char*)calloc((size_t)n + 1, 1);
  double* completion = (double*)calloc((size_t)n + 1, sizeof(double));
  s.workers = (worker_t*)calloc((size_t)W, sizeof(worker_t));
  /* sim_engine.cpp:116-120 */
  for (int64_t i = 0; i < n; ++i) push_event(&s, arrival[i], EV_ARRIVAL, i, -1);
  push_event(&s, cfg->horizon_s, EV_END, -1, -1);
  if (cfg->policy == SCLS_POLICY_SCLS) {
    push_event(&s, 0.0, EV_TICK, -1, -1); /* sched_policies.cpp:84 */
  } else if (cfg->policy == SCLS_POLICY_SLS) {
    s.pending = (deque_t*)calloc((size_t)W, sizeof(deque_t));
  } else {
    s.inst = (ils_inst*)calloc((size_t)W, sizeof(ils_inst));
    for (int32_t w = 0; w < W; ++w) s.inst[w].segment_id = -1;
  }
  st = SCLS_OK;
  /* sim_engine.cpp:123-166 */
  while (s.completed < n) {
    if (s.heap_len == 0) {
      st = fail(SCLS_ERR_ERROR, "event queue drained with requests incomplete");
      break;
    }
    const sim_event ev = pop_event(&s);
    s.clock = ev.time;
    if (ev.kind == EV_ARRIVAL) {
      scls_event_record* a = add_rec(&s, K_ARRIVAL);
      a->request = ev.request;
      a->input_len = in_len[ev.request];
      a->gen_len = gen_len[ev.request];
      if (cfg->policy == SCLS_POLICY_SCLS) {
        GROW(s.pool, s.pool_len, s.pool_cap);
        s.pool[s.pool_len++] = ev.request;
      } else if (cfg->policy == SCLS_POLICY_SLS) {
        /* sched_policies.cpp:194-201 */
        const int32_t w = (int32_t)(s.rr++ % W);
        dq_push(&s.pending[w], ev.request);
        push_event(&s, s.clock, EV_POLICY, -1, w);
      } else {
        /* sched_policies.cpp:279-290 */
        const int32_t w = (int32_t)(s.rr++ % W);
        ils_inst* in = &s.inst[w];
        dq_push(&in->waiting, ev.request);
        if (in->n_running == 0 && !in->boundary_scheduled) {
          push_event(&s, s.clock, EV_POLICY, -1, w);
          in->boundary_scheduled = 1;
        }
      }
    } else if (ev.kind == EV_TICK) {
      if (cfg->policy == SCLS_POLICY_SCLS) {
        st = scls_on_tick(&s);
        if (st) {
          r->error_request_id = g_err_request;
          break;
        }
      }
    } else if (ev.kind == EV_POLICY) {
      if (cfg->policy == SCLS_POLICY_SLS) sls_try_dispatch(&s, ev.worker);
      else if (cfg->policy == SCLS_POLICY_ILS) ils_on_policy_event(&s, ev.worker, completion);
    } else if (ev.kind == EV_BATCH_DONE) {
      worker_t* w = &s.workers[ev.worker];
      batch_t b = w->in_flight;
      const int32_t served = w->in_flight_l_out;
      w->has_in_flight = 0;
      if (cfg->policy == SCLS_POLICY_SCLS) scls_on_batch_done(&s, ev.worker, &b, served, completion);
      else if (cfg->policy == SCLS_POLICY_SLS) sls_on_batch_done(&s, ev.worker, &b, served, completion);
      free(b.req);
      start_next_batch(&s, ev.worker);
    } else {
      st = fail(SCLS_ERR_NON_TERMINATION, "simulated clock reached horizon");
      break;
    }
  }
  if (st == SCLS_OK) st = compute_metrics(&s, W, r, hist_bins, hist);
  r->status = st;
  if (log && trace < log->n_logged) {
    scls_event_record* dst = log->records + trace * log->rec_cap;
    scls_member* dm = log->members + trace * log->mem_cap;
    for (int64_t k = 0; k < s.rec_len && k < log->rec_cap; ++k) dst[k] = s.rec[k];
    for (int64_t k = 0; k < s.mem_len && k < log->mem_cap; ++k) dm[k] = s.mem_rec[k];
    log->rec_count[trace] = s.rec_len;
    log->mem_count[trace] = s.mem_len;
  }
  /* release */
  for (int32_t w = 0; w < W; ++w) {
    worker_t* wk = &s.workers[w];
    for (int64_t q = 0; q < wk->qlen; ++q) free(wk->q[wk->qhead + q].b.req);
    if (wk->has_in_flight) free(wk->in_flight.req);
    free(wk->q);
    if (s.pending) free(s.pending[w].v);
    if (s.inst) {
      free(s.inst[w].running);
      free(s.inst[w].waiting.v);
    }
  }
  free(s.workers); free(s.pending); free(s.inst); free(s.pool); free(s.heap);
  free(s.generated); free(s.slices); free(s.has_first_dispatch); free(completion);
  free(s.rec); free(s.mem_rec);
}

typedef struct {
  int32_t n_traces;
  const int64_t* off;
  const double* arrival;
  const int32_t* in_len;
  const int32_t* gen_len;
  const scls_sched_cfg* cfgs;
  const int32_t* cfg_index;
  const scls_latency* lat;
  const scls_memory* mem;
  scls_trace_result* results;
  int32_t hist_bins;
  int64_t* hist;
  scls_event_log* log;
  int32_t next;
  pthread_mutex_t mu;
} sim_job;

static void* sim_worker(void* p) {
  sim_job* j = (sim_job*)p;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int32_t t = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (t >= j->n_traces) return NULL;
    const int64_t b = j->off[t], e = j->off[t + 1];
    const scls_sched_cfg* c = &j->cfgs[j->cfg_index ? j->cfg_index[t] : 0];
    simulate_one(e - b, j->arrival + b, j->in_len + b, j->gen_len + b, c, j->lat, j->mem,
                 &j->results[t], j->hist_bins, j->hist ? j->hist + (int64_t)t * j->hist_bins : NULL,
                 j->log, t);
  }
}

scls_status orc_simulate(int32_t n_traces, const int64_t* req_offset, const double* arrival,
                         const int32_t* input_len, const int32_t* gen_len,
                         const scls_sched_cfg* cfgs, const int32_t* cfg_index,
                         const scls_latency* lat, const scls_memory* mem,
                         scls_trace_result* results, int32_t hist_bins, int64_t* slice_hist,
                         scls_event_log* log, int32_t n_threads) {
  sim_job j = {n_traces, req_offset, arrival, input_len, gen_len, cfgs, cfg_index, lat, mem,
               results, hist_bins, slice_hist, log, 0, PTHREAD_MUTEX_INITIALIZER};
  if (n_threads <= 1) {
    sim_worker(&j);
    return SCLS_OK;
  }
  pthread_t* th = (pthread_t*)malloc((size_t)n_threads * sizeof(pthread_t));
  for (int32_t i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, sim_worker, &j);
  for (int32_t i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  free(th);
  return SCLS_OK;
}
