// device_run.cpp — one simulation with its full event log on the B200, and
// the conversions the drop-in needs around it: the device records ->
// EventLog (event_log.h:41-84), the device report -> MetricsReport
// (metrics.h:26-36), and the device status -> the reference's exception
// (sim_engine.cpp:159-163, metrics.cpp:31,75, batcher.cpp:40-46).
#include <algorithm>
#include <cmath>
#include <string>

#include "dropin.h"

namespace slicesim {
namespace b200 {

LoggedRun run_logged(const scls_sched_cfg& c, const scls_latency& lat, const scls_memory& mem, int32_t hist_bins,
                     const scls_workload_spec* spec, const std::vector<Request>* workload) {
  scls_ctx* ctx = context();
  LoggedRun out;
  int64_t n = 0;
  std::vector<double> arr;
  std::vector<int32_t> inp, gen;
  if (spec) {
    // Poisson count: mean + 12 sigma + 64 (the device generator's own cap)
    const double mean = std::max(0.0, spec->rate * spec->duration_s);
    n = static_cast<int64_t>(mean + 12.0 * std::sqrt(mean) + 64.0);
  } else {
    n = static_cast<int64_t>(workload->size());
    arr.resize(n);
    inp.resize(n);
    gen.resize(n);
    for (int64_t i = 0; i < n; ++i) {
      arr[i] = (*workload)[i].arrival_time;
      inp[i] = (*workload)[i].orig_input_len;
      gen[i] = (*workload)[i].true_gen_len;
    }
  }
  int64_t rec_cap = 6 * n + 64, mem_cap = 4 * n + 64;
  out.hist.assign(std::max(hist_bins, 1), 0);
  for (int attempt = 0; attempt < 2; ++attempt) {
    out.recs.assign(static_cast<std::size_t>(rec_cap), scls_event_record{});
    out.mems.assign(static_cast<std::size_t>(mem_cap), scls_member{});
    out.rc = out.mc = 0;
    scls_event_log lg{1, rec_cap, mem_cap, out.recs.data(), out.mems.data(), &out.rc, &out.mc};
    out.res = scls_trace_result{};
    if (spec) {
      check(ctx, scls_run_experiments(ctx, 1, spec, &c, &lat, &mem, &out.res, hist_bins, out.hist.data(), &lg,
                                      SCLS_MEM_HOST));
    } else {
      const int64_t offs[2] = {0, n};
      check(ctx, scls_simulate(ctx, 1, offs, arr.data(), inp.data(), gen.data(), 1, &c, nullptr, &lat, &mem,
                               &out.res, hist_bins, out.hist.data(), &lg, SCLS_MEM_HOST));
    }
    if (out.rc <= rec_cap && out.mc <= mem_cap) return out;
    rec_cap = out.rc;  // the device counts past capacity: resize once
    mem_cap = out.mc;
  }
  throw Error("device event log capacity could not be established");
}

void raise_status(const LoggedRun& r, double horizon_s) {
  const scls_trace_result& res = r.res;
  switch (res.status) {
    case SCLS_OK:
      return;
    case SCLS_ERR_INFEASIBLE_REQUEST:
      throw InfeasibleRequestError(res.error_request_id, "request " + std::to_string(res.error_request_id) +
                                                             " does not fit memory even as a singleton batch");
    case SCLS_ERR_NON_TERMINATION: {
      int64_t done = 0;
      for (int64_t k = 0; k < std::min<int64_t>(r.rc, static_cast<int64_t>(r.recs.size())); ++k)
        done += r.recs[static_cast<std::size_t>(k)].kind == 5;
      throw NonTerminationError("simulated clock reached horizon " + std::to_string(horizon_s) + " s with " +
                                std::to_string(done) + " of " + std::to_string(res.n_requests) +
                                " requests completed");
    }
    case SCLS_ERR_EMPTY_LOG:
      if (r.rc == 0) throw EmptyLogError("cannot compute metrics from an empty log");
      throw EmptyLogError("log contains no completed requests");
    default:
      throw Error("device simulation failed with status " + std::to_string(res.status));
  }
}

EventLog to_event_log(const LoggedRun& r, int worker_count) {
  EventLog log;
  log.worker_count = worker_count;
  log.events.reserve(static_cast<std::size_t>(r.rc));
  for (int64_t k = 0; k < r.rc; ++k) {
    const scls_event_record& d = r.recs[static_cast<std::size_t>(k)];
    EventRecord e;
    e.t = d.t;
    e.kind = static_cast<EventKind>(d.kind);
    e.request = d.request;
    e.worker = d.worker;
    e.batch = d.batch;
    e.n = d.n;
    e.l_in = d.l_in;
    e.planned_l_out = d.planned_l_out;
    e.served_l_out = d.served_l_out;
    e.est_serve_s = d.est_serve_s;
    e.input_len = d.input_len;
    e.gen_len = d.gen_len;
    e.response_s = d.response_s;
    e.slices = d.slices;
    e.next_interval_s = d.next_interval_s;
    e.members.reserve(static_cast<std::size_t>(d.member_count));
    for (int32_t j = 0; j < d.member_count; ++j) {
      const scls_member& m = r.mems[static_cast<std::size_t>(d.member_offset + j)];
      e.members.push_back(MemberAccounting{m.request, m.effective_input, m.pad, m.gen, m.invalid});
    }
    log.add(std::move(e));
  }
  return log;
}

MetricsReport to_report(const scls_trace_result& r, const int64_t* hist, int32_t hist_bins) {
  // metrics.cpp:30-117, computed online by the device in the reference's
  // summation orders; the histogram fraction is count / completed (:109-111)
  MetricsReport m;
  m.throughput = r.throughput;
  m.avg_response_s = r.avg_response_s;
  m.p95_response_s = r.p95_response_s;
  m.ct_std_s = r.ct_std_s;
  m.avg_pad_tokens = r.avg_pad_tokens;
  m.avg_invalid_tokens = r.avg_invalid_tokens;
  m.avg_batch_size = r.avg_batch_size;
  m.early_return_ratio = r.early_return_ratio;
  const double completed = static_cast<double>(r.completed);
  for (int32_t s = 0; s < hist_bins; ++s)
    if (hist[s] > 0) m.slice_count_hist[s] = static_cast<double>(hist[s]) / completed;
  return m;
}

int32_t report_hist_bins(const scls_sched_cfg& c) {
  // a request is served at most ceil(max_gen_limit / slice_len) slices
  return c.slice_len > 0 ? std::max(2, (c.max_gen_limit + c.slice_len - 1) / c.slice_len + 2) : 2;
}

}  // namespace b200
}  // namespace slicesim
