// ref_capi.cpp — C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with
// /root/reference/proj/core/src/*.cpp (namespace renamed slicesim -> scls_ref)
// into oracle/_ref/libscls_ref.so.  It is the checker for the C restatement
// (oracle/scls_oracle.c) and for the CUDA path, and the `--impl reference`
// CPU arm of bench.py.  Nothing in the product links or loads it.
//
// Each function is a thin adapter: it builds the reference's own value types
// from the C-ABI structs of include/scls_capi.h, calls the reference API
// (batcher.h:40-43, offloader.h:39-44, sim_engine.h:61-67, metrics.h:41,
// workload.h:78, cost_model.h:54-66, memory_model.h:62-66) and flattens the
// results back.  Exceptions become scls_status codes (errors.h:26-87).

#include <algorithm>
#include <atomic>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "slicesim/batcher.h"
#include "slicesim/cost_model.h"
#include "slicesim/errors.h"
#include "slicesim/event_log.h"
#include "slicesim/memory_model.h"
#include "slicesim/metrics.h"
#include "slicesim/offloader.h"
#include "slicesim/run_config.h"
#include "slicesim/sched_policies.h"
#include "slicesim/sim_engine.h"
#include "slicesim/workload.h"

#include "scls_capi.h"
#include "scls_loghash.h"

namespace S = slicesim;  // renamed to scls_ref by -Dslicesim=scls_ref

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_request = -1;

scls_status map_exception() {
  g_err_request = -1;  // only an InfeasibleRequestError names a request
  try {
    throw;
  } catch (const S::InfeasibleRequestError& e) {
    g_err = e.what();
    g_err_request = e.request_id;
    return SCLS_ERR_INFEASIBLE_REQUEST;
  } catch (const S::InsufficientSamplesError& e) {
    g_err = e.what();
    return SCLS_ERR_INSUFFICIENT_SAMPLES;
  } catch (const S::DegenerateModelError& e) {
    g_err = e.what();
    return SCLS_ERR_DEGENERATE_MODEL;
  } catch (const S::WrongKindError& e) {
    g_err = e.what();
    return SCLS_ERR_WRONG_KIND;
  } catch (const S::NoWorkersError& e) {
    g_err = e.what();
    return SCLS_ERR_NO_WORKERS;
  } catch (const S::ParseError& e) {
    g_err = e.what();
    return SCLS_ERR_PARSE;
  } catch (const S::LimitViolationError& e) {
    g_err = e.what();
    return SCLS_ERR_LIMIT_VIOLATION;
  } catch (const S::EmptyLogError& e) {
    g_err = e.what();
    return SCLS_ERR_EMPTY_LOG;
  } catch (const S::NonTerminationError& e) {
    g_err = e.what();
    return SCLS_ERR_NON_TERMINATION;
  } catch (const S::Error& e) {
    g_err = e.what();
    return SCLS_ERR_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SCLS_ERR_INVALID_ARGUMENT;
  }
}

S::LatencyModel to_ref(const scls_latency& m) {
  S::LatencyModel r;
  r.p1 = m.p1; r.p2 = m.p2; r.p3 = m.p3; r.p4 = m.p4;
  r.d1 = m.d1; r.d2 = m.d2; r.d3 = m.d3; r.d4 = m.d4;
  r.rmse_prefill = m.rmse_prefill;
  r.rmse_decode = m.rmse_decode;
  r.n_cap = m.n_cap;
  r.l_cap = m.l_cap;
  return r;
}

// Field-by-field (no validation), like a default-constructed MemoryModel the
// tests then fill in; the factories validate where the caller asks for it.
S::MemoryModel to_ref(const scls_memory& m) {
  S::MemoryModel r;
  if (m.kind == SCLS_MEM_ANALYTIC) {
    r.kind = S::MemoryModel::Kind::kAnalytic;
    r.m_cap = m.m_cap; r.m_model = m.m_model; r.m_engine = m.m_engine;
    r.delta = m.delta; r.zeta = m.zeta;
  } else {
    r.kind = S::MemoryModel::Kind::kRuleTable;
    for (int i = 0; i < m.n_rules; ++i)
      r.rules.push_back({m.rule_threshold[i], m.rule_max_n[i]});
  }
  return r;
}

S::SchedulerConfig to_ref(const scls_sched_cfg& c) {
  S::SchedulerConfig r;
  r.policy = c.policy == SCLS_POLICY_SCLS ? S::PolicyKind::kScls
             : c.policy == SCLS_POLICY_SLS ? S::PolicyKind::kSls
                                           : S::PolicyKind::kIls;
  r.slice_len = c.slice_len;
  r.max_gen_limit = c.max_gen_limit;
  r.lambda = c.lambda;
  r.gamma = c.gamma;
  r.fixed_batch_size = c.fixed_batch_size;
  r.max_concurrent = c.max_concurrent;
  r.worker_count = c.worker_count;
  return r;
}

S::LengthDist to_ref(const scls_length_dist& d) {
  switch (d.kind) {
    case SCLS_DIST_UNIFORM: return S::LengthDist::uniform(d.lo, d.hi);
    case SCLS_DIST_LOGNORMAL: return S::LengthDist::log_normal(d.mu, d.sigma, d.cap);
    default: {
      std::vector<int> edges(d.edges, d.edges + d.n_buckets + 1);
      std::vector<double> weights(d.weights, d.weights + d.n_buckets);
      return S::LengthDist::histogram(std::move(edges), std::move(weights));
    }
  }
}

// hash = false skips the FNV digests (h_* stay 0): what remains is one
// counting pass over the log (completions, slice histogram, batch counters).
void fill_result(const S::EventLog& log, scls_trace_result* r, int32_t hist_bins,
                 int64_t* hist, scls_event_log* out_log, int64_t trace, bool hash = true) {
  uint64_t hc = SCLS_FNV_OFFSET, hd = SCLS_FNV_OFFSET, ht = SCLS_FNV_OFFSET,
           hl = SCLS_FNV_OFFSET;
  int64_t nd = 0, nt = 0, pad = 0, inval = 0, bc = 0, bm = 0, er = 0, done = 0;
  scls_event_record* recs = nullptr;
  scls_member* mems = nullptr;
  int64_t rec_n = 0, mem_n = 0;
  bool logging = out_log && trace < out_log->n_logged;
  if (logging) {
    recs = out_log->records + trace * out_log->rec_cap;
    mems = out_log->members + trace * out_log->mem_cap;
  }
  for (const S::EventRecord& e : log.events) {
    const int32_t kind = static_cast<int32_t>(e.kind);
    if (hash) {
    hl = scls_hash_record(hl, kind, e.t, e.request, e.worker, e.batch, e.n, e.l_in,
                          e.planned_l_out, e.served_l_out, e.est_serve_s,
                          e.input_len, e.gen_len, e.response_s, e.slices,
                          e.next_interval_s, static_cast<int32_t>(e.members.size()));
    for (const S::MemberAccounting& m : e.members)
      hl = scls_hash_member(hl, m.request, m.effective_input, m.pad, m.gen, m.invalid);
    }
    switch (e.kind) {
      case S::EventKind::kComplete:
        if (hash) {
          hc = scls_fnv_bytes(hc, static_cast<uint64_t>(e.request));
          ht = scls_fnv_bytes(ht, scls_dbits(e.t));
        }
        ++done;
        if (hist && e.slices >= 0 && e.slices < hist_bins)
          hist[trace * hist_bins + e.slices] += 1;
        break;
      case S::EventKind::kDispatch:
        if (hash) {
          hd = scls_fnv_bytes(hd, static_cast<uint64_t>(e.batch));
          hd = scls_fnv_bytes(hd, static_cast<uint64_t>(static_cast<int64_t>(e.worker)));
          hd = scls_fnv_bytes(hd, static_cast<uint64_t>(static_cast<int64_t>(e.n)));
          hd = scls_fnv_bytes(hd, static_cast<uint64_t>(static_cast<int64_t>(e.l_in)));
        }
        ++nd;
        break;
      case S::EventKind::kTick: ++nt; break;
      case S::EventKind::kBatchEnd:
        ++bc;
        bm += e.n;
        if (e.served_l_out < e.planned_l_out) ++er;
        for (const S::MemberAccounting& m : e.members) {
          pad += m.pad;
          inval += m.invalid;
        }
        break;
      default: break;
    }
    if (logging) {
      if (rec_n < out_log->rec_cap) {
        scls_event_record& o = recs[rec_n];
        o.t = e.t; o.est_serve_s = e.est_serve_s; o.response_s = e.response_s;
        o.next_interval_s = e.next_interval_s; o.request = e.request; o.batch = e.batch;
        o.kind = kind; o.worker = e.worker; o.n = e.n; o.l_in = e.l_in;
        o.planned_l_out = e.planned_l_out; o.served_l_out = e.served_l_out;
        o.input_len = e.input_len; o.gen_len = e.gen_len; o.slices = e.slices;
        o.member_count = static_cast<int32_t>(e.members.size());
        o.member_offset = mem_n;
      }
      for (const S::MemberAccounting& m : e.members) {
        if (mem_n < out_log->mem_cap)
          mems[mem_n] = scls_member{m.request, m.effective_input, m.pad, m.gen, m.invalid};
        ++mem_n;
      }
      ++rec_n;
    }
  }
  if (logging) {
    out_log->rec_count[trace] = rec_n;
    out_log->mem_count[trace] = mem_n;
  }
  r->h_complete_ids = hash ? hc : 0;
  r->h_dispatch = hash ? hd : 0;
  r->h_complete_t = hash ? ht : 0;
  r->h_log = hash ? hl : 0;
  r->n_events = static_cast<int64_t>(log.events.size());
  r->n_dispatches = nd;
  r->n_ticks = nt;
  r->total_pad = pad;
  r->total_invalid = inval;
  r->batch_count = bc;
  r->batch_members = bm;
  r->early_returns = er;
  r->completed = done;
  r->sim_clock = log.events.empty() ? 0.0 : log.events.back().t;
}

}  // namespace

extern "C" {

size_t ref_last_error(char* buf, size_t cap) {
  if (buf && cap) {
    const size_t n = std::min(cap - 1, g_err.size());
    std::memcpy(buf, g_err.data(), n);
    buf[n] = '\0';
  }
  return g_err.size();
}

int64_t ref_last_request_id(void) { return g_err_request; }

double ref_batch_serve_time(const scls_latency* m, int32_t n, int32_t l_in, int32_t l_out) {
  return S::batch_serve_time(to_ref(*m), n, l_in, l_out);
}
double ref_prefill_time(const scls_latency* m, int32_t n, int32_t l_in) {
  return S::prefill_time(to_ref(*m), n, l_in);
}
double ref_decode_step_time(const scls_latency* m, int32_t ctx, int32_t n) {
  return S::decode_step_time(to_ref(*m), ctx, n);
}
double ref_decode_time(const scls_latency* m, int32_t n, int32_t l_in, int32_t l_out) {
  return S::decode_time(to_ref(*m), n, l_in, l_out);
}
int32_t ref_would_oom(const scls_memory* m, int32_t n, int32_t l_in, int32_t slice) {
  return to_ref(*m).would_oom(n, l_in, slice) ? 1 : 0;
}
int32_t ref_max_batch_size(const scls_memory* m, int32_t l_in, int32_t slice) {
  return to_ref(*m).max_batch_size(l_in, slice);
}
double ref_next_interval(double lambda, double gamma, double min_load) {
  return S::next_interval(lambda, gamma, min_load);
}

// cost_model.cpp:140-160 fit, the reference's own (built here against the
// Eigen stand-in of oracle/ref_shims): the checker of scls_fit_latency.
scls_status ref_fit_latency(const scls_profile_sample* s, int64_t n, int32_t n_cap, int32_t l_cap,
                            scls_latency* out) {
  try {
    std::vector<S::ProfileSample> v(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      v[i].phase = s[i].phase == 0 ? S::Phase::kPrefill : S::Phase::kDecode;
      v[i].batch_size = s[i].batch_size;
      v[i].length = s[i].length;
      v[i].latency_s = s[i].latency_s;
    }
    const S::LatencyModel m = S::fit(v, n_cap, l_cap);
    *out = scls_latency{m.p1, m.p2, m.p3, m.p4, m.d1, m.d2, m.d3, m.d4, m.rmse_prefill, m.rmse_decode,
                        m.n_cap, m.l_cap};
    return SCLS_OK;
  } catch (...) {
    return map_exception();
  }
}

scls_status ref_validate_latency(const scls_latency* m) {
  try { S::validate(to_ref(*m)); return SCLS_OK; } catch (...) { return map_exception(); }
}
scls_status ref_validate_memory(const scls_memory* m) {
  try { S::validate(to_ref(*m)); return SCLS_OK; } catch (...) { return map_exception(); }
}
scls_status ref_validate_sched(const scls_sched_cfg* c) {
  try { S::validate(to_ref(*c)); return SCLS_OK; } catch (...) { return map_exception(); }
}

// batcher.h:40-43.  Outputs: n_batches, seg_begin[nb+1] (positions in batch
// order), l_in[nb], est[nb], batch_id[nb], member_id[n].
scls_status ref_batch_requests(int64_t n, const int32_t* eff_len, const double* arrival,
                               const int64_t* id, int32_t slice_len,
                               const scls_latency* lat, const scls_memory* mem,
                               int64_t first_batch_id, int64_t* n_batches,
                               int32_t* seg_begin, int32_t* l_in, double* est,
                               int64_t* batch_id, int64_t* member_id) {
  try {
    std::vector<S::Request> reqs(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      reqs[i].id = id[i];
      reqs[i].arrival_time = arrival[i];
      reqs[i].orig_input_len = eff_len[i];
    }
    const auto batches = S::batch_requests(reqs, slice_len, to_ref(*lat), to_ref(*mem),
                                           first_batch_id);
    *n_batches = static_cast<int64_t>(batches.size());
    int32_t pos = 0;
    for (size_t b = 0; b < batches.size(); ++b) {
      seg_begin[b] = pos;
      l_in[b] = batches[b].l_in;
      est[b] = batches[b].est_serve_time;
      batch_id[b] = batches[b].id;
      for (S::RequestId r : batches[b].requests) member_id[pos++] = r;
    }
    seg_begin[batches.size()] = pos;
    return SCLS_OK;
  } catch (...) {
    return map_exception();
  }
}

// offloader.h:39-40.
scls_status ref_offload(int64_t nb, const int64_t* batch_id, const double* est,
                        int32_t n_workers, const int32_t* worker_id, double* load_inout,
                        int64_t* out_batch_id, int32_t* out_worker) {
  try {
    std::vector<S::Batch> batches(static_cast<size_t>(nb));
    for (int64_t b = 0; b < nb; ++b) {
      batches[b].id = batch_id[b];
      batches[b].est_serve_time = est[b];
    }
    std::vector<S::WorkerLoad> loads(static_cast<size_t>(n_workers));
    for (int32_t w = 0; w < n_workers; ++w) loads[w] = {worker_id[w], load_inout[w]};
    const auto asg = S::offload(batches, loads);
    for (size_t i = 0; i < asg.size(); ++i) {
      out_batch_id[i] = asg[i].first;
      out_worker[i] = asg[i].second;
    }
    for (int32_t w = 0; w < n_workers; ++w) load_inout[w] = loads[w].load_estimate;
    return SCLS_OK;
  } catch (...) {
    return map_exception();
  }
}

// workload.h:78.
scls_status ref_generate(const scls_workload_spec* spec, int64_t cap, int64_t* n,
                         double* arrival, int32_t* input_len, int32_t* gen_len) {
  try {
    S::WorkloadSpec w;
    w.rate = spec->rate;
    w.duration_s = spec->duration_s;
    w.input_len_dist = to_ref(spec->input_len_dist);
    w.gen_len_dist = to_ref(spec->gen_len_dist);
    w.max_input_limit = spec->max_input_limit;
    w.max_gen_limit = spec->max_gen_limit;
    w.seed = spec->seed;
    const auto reqs = S::generate(w);
    *n = static_cast<int64_t>(reqs.size());
    for (int64_t i = 0; i < *n && i < cap; ++i) {
      arrival[i] = reqs[i].arrival_time;
      input_len[i] = reqs[i].orig_input_len;
      gen_len[i] = reqs[i].true_gen_len;
    }
    return *n > cap ? SCLS_ERR_CAPACITY : SCLS_OK;
  } catch (...) {
    return map_exception();
  }
}

// One Simulator::run + compute per trace (sim_engine.h:61-67, metrics.h:41),
// traces spread over `n_threads` host threads (independent runs may execute
// concurrently, sim_engine.h:55-58).  Returns the first failing status only
// for argument errors; per-trace failures land in results[t].status.
scls_status ref_simulate(int32_t n_traces, const int64_t* req_offset, const double* arrival,
                         const int32_t* input_len, const int32_t* gen_len,
                         const scls_sched_cfg* cfgs, const int32_t* cfg_index,
                         const scls_latency* lat, const scls_memory* mem,
                         scls_trace_result* results, int32_t hist_bins, int64_t* slice_hist,
                         scls_event_log* log, int32_t n_threads) {
  const S::LatencyModel latency = to_ref(*lat);
  const S::MemoryModel memory = to_ref(*mem);
  std::atomic<int32_t> next{0};
  auto worker = [&]() {
    for (;;) {
      const int32_t t = next.fetch_add(1);
      if (t >= n_traces) return;
      const scls_sched_cfg& c = cfgs[cfg_index ? cfg_index[t] : 0];
      scls_trace_result* r = &results[t];
      std::memset(r, 0, sizeof *r);
      r->worker_count = c.worker_count;
      r->error_request_id = -1;
      const int64_t b = req_offset[t], e = req_offset[t + 1];
      r->n_requests = e - b;
      if (slice_hist) std::fill(slice_hist + t * hist_bins, slice_hist + (t + 1) * hist_bins, 0);
      try {
        std::vector<S::Request> reqs(static_cast<size_t>(e - b));
        for (int64_t i = b; i < e; ++i) {
          S::Request& q = reqs[i - b];
          q.id = i - b;
          q.arrival_time = arrival[i];
          q.orig_input_len = input_len[i];
          q.true_gen_len = gen_len[i];
        }
        S::Simulator sim(to_ref(c), latency, memory, c.horizon_s);
        auto policy = S::make_scheduler(to_ref(c).policy);
        const S::EventLog elog = sim.run(std::move(reqs), *policy);
        fill_result(elog, r, hist_bins, slice_hist, log, t);
        const S::MetricsReport rep = S::compute(elog);
        r->throughput = rep.throughput;
        r->avg_response_s = rep.avg_response_s;
        r->p95_response_s = rep.p95_response_s;
        r->ct_std_s = rep.ct_std_s;
        r->avg_pad_tokens = rep.avg_pad_tokens;
        r->avg_invalid_tokens = rep.avg_invalid_tokens;
        r->avg_batch_size = rep.avg_batch_size;
        r->early_return_ratio = rep.early_return_ratio;
        r->status = SCLS_OK;
      } catch (...) {
        r->status = map_exception();
        r->error_request_id = g_err_request;
      }
    }
  };
  if (n_threads <= 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int32_t i = 0; i < n_threads; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
  }
  return SCLS_OK;
}

// The reference's sweep body (experiment.cpp:62-85 / run_experiment :39-60)
// for n_traces x n_cfgs jobs: per trace, generate(spec) once (workload.h:78),
// then for every config Simulator::run + compute (sim_engine.h:61-67,
// metrics.h:41) -- exactly the work of one reference sweep value -- plus one
// digest-free counting pass over each log for the parity record.  Traces
// are spread over n_threads host threads (independent runs may execute
// concurrently, sim_engine.h:55-58).  Job j = c * n_traces + t.
scls_status ref_run_sweep(int32_t n_traces, const scls_workload_spec* specs, int32_t n_cfgs,
                          const scls_sched_cfg* cfgs, const scls_latency* lat, const scls_memory* mem,
                          scls_trace_result* results, int32_t hist_bins, int64_t* slice_hist,
                          int32_t n_threads) {
  const S::LatencyModel latency = to_ref(*lat);
  const S::MemoryModel memory = to_ref(*mem);
  std::atomic<int32_t> next{0};
  auto worker = [&]() {
    for (;;) {
      const int32_t t = next.fetch_add(1);
      if (t >= n_traces) return;
      std::vector<S::Request> reqs;
      scls_status gen_status = SCLS_OK;
      try {
        S::WorkloadSpec w;
        w.rate = specs[t].rate;
        w.duration_s = specs[t].duration_s;
        w.input_len_dist = to_ref(specs[t].input_len_dist);
        w.gen_len_dist = to_ref(specs[t].gen_len_dist);
        w.max_input_limit = specs[t].max_input_limit;
        w.max_gen_limit = specs[t].max_gen_limit;
        w.seed = specs[t].seed;
        reqs = S::generate(w);
      } catch (...) {
        gen_status = map_exception();
      }
      for (int32_t c = 0; c < n_cfgs; ++c) {
        const int64_t j = (int64_t)c * n_traces + t;
        scls_trace_result* r = &results[j];
        std::memset(r, 0, sizeof *r);
        r->worker_count = cfgs[c].worker_count;
        r->error_request_id = -1;
        r->n_requests = static_cast<int64_t>(reqs.size());
        if (slice_hist) std::fill(slice_hist + j * hist_bins, slice_hist + (j + 1) * hist_bins, 0);
        if (gen_status != SCLS_OK) {
          r->status = gen_status;
          continue;
        }
        try {
          S::Simulator sim(to_ref(cfgs[c]), latency, memory, cfgs[c].horizon_s);
          auto policy = S::make_scheduler(to_ref(cfgs[c]).policy);
          const S::EventLog elog = sim.run(reqs, *policy);
          fill_result(elog, r, hist_bins, slice_hist, nullptr, j, false);
          const S::MetricsReport rep = S::compute(elog);
          r->throughput = rep.throughput;
          r->avg_response_s = rep.avg_response_s;
          r->p95_response_s = rep.p95_response_s;
          r->ct_std_s = rep.ct_std_s;
          r->avg_pad_tokens = rep.avg_pad_tokens;
          r->avg_invalid_tokens = rep.avg_invalid_tokens;
          r->avg_batch_size = rep.avg_batch_size;
          r->early_return_ratio = rep.early_return_ratio;
          r->status = SCLS_OK;
        } catch (...) {
          r->status = map_exception();
          r->error_request_id = g_err_request;
        }
      }
    }
  };
  if (n_threads <= 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int32_t i = 0; i < n_threads; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
  }
  return SCLS_OK;
}

// Event log JSONL of one run (event_log.cpp:39-96) and the report JSON
// (metrics.cpp:119-135), for byte-identity checks.
scls_status ref_run_jsonl(int64_t n, const double* arrival, const int32_t* input_len,
                          const int32_t* gen_len, const scls_sched_cfg* c,
                          const scls_latency* lat, const scls_memory* mem,
                          const char* log_path, const char* report_path) {
  try {
    std::vector<S::Request> reqs(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      reqs[i].id = i;
      reqs[i].arrival_time = arrival[i];
      reqs[i].orig_input_len = input_len[i];
      reqs[i].true_gen_len = gen_len[i];
    }
    S::Simulator sim(to_ref(*c), to_ref(*lat), to_ref(*mem), c->horizon_s);
    auto policy = S::make_scheduler(to_ref(*c).policy);
    const S::EventLog elog = sim.run(std::move(reqs), *policy);
    if (log_path) elog.save_jsonl(log_path);
    if (report_path) S::save_report(S::compute(elog), report_path);
    return SCLS_OK;
  } catch (...) {
    return map_exception();
  }
}

}  // extern "C"
