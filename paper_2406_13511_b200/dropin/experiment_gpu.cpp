// experiment_gpu.cpp — drop-in replacement of the reference's
// core/src/experiment.cpp.  run_experiment keeps its structure (models →
// workload → Simulator::run, now on the B200 → compute).  sweep
// (experiment.h:52-53) is the data-parallel entry point: instead of one run
// after another it builds every run of the sweep and simulates all of them
// in ONE call (one warp per trace), reading the reports the device computes
// online (metrics.cpp:30-117, bit for bit).  Generated workloads (uniform,
// log-normal and histogram lengths) are generated on the device too
// (scls_run_experiments, bit-exact with generate()); only trace files are
// loaded on the host and simulated with scls_simulate.  Errors surface in
// value order, as the sequential reference would raise them.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <ostream>
#include <sstream>

#include "dropin.h"
#include "slicesim/experiment.h"
#include "slicesim/sim_engine.h"
#include "slicesim/workload.h"

namespace slicesim {

LatencyModel resolve_latency_model(const std::string& path) {
  if (path.empty()) return builtin_latency_model();
  return load_latency_model(path);
}

MemoryModel resolve_memory_model(const std::string& path) {
  if (path.empty()) return builtin_memory_model();
  if (path == "builtin-analytic") return builtin_analytic_memory_model();
  return load_memory_model(path);
}

namespace {

std::vector<Request> load_workload(const RunConfig& cfg) {
  if (cfg.workload_from_trace) {
    if (cfg.trace_path.empty()) throw Error("workload.kind = trace requires workload.trace = <path>");
    return load_trace(cfg.trace_path, cfg.workload.max_input_limit, cfg.workload.max_gen_limit);
  }
  return generate(cfg.workload);
}

RunConfig with_value(const RunConfig& base, const std::string& param, double value) {
  RunConfig cfg = base;
  if (param == "rate") cfg.workload.rate = value;
  else if (param == "slice_len") cfg.sched.slice_len = static_cast<int>(std::llround(value));
  else if (param == "workers") cfg.sched.worker_count = static_cast<int>(std::llround(value));
  else throw Error("unknown sweep parameter '" + param + "' (expected rate, slice_len, or workers)");
  return cfg;
}

// Whether generate(cfg.workload) can run on the device (scls_run_experiments).
bool device_generated(const RunConfig& cfg) {
  const WorkloadSpec& w = cfg.workload;
  auto ok = [](const LengthDist& d) {
    return d.kind != LengthDist::Kind::kHistogram || d.weights.size() <= SCLS_MAX_BUCKETS;
  };
  return !cfg.workload_from_trace && ok(w.input_len_dist) && ok(w.gen_len_dist);
}

scls_length_dist to_c(const LengthDist& d) {
  scls_length_dist c{};
  c.kind = d.kind == LengthDist::Kind::kUniform ? SCLS_DIST_UNIFORM
           : d.kind == LengthDist::Kind::kLogNormal ? SCLS_DIST_LOGNORMAL : SCLS_DIST_HISTOGRAM;
  c.lo = d.lo;
  c.hi = d.hi;
  c.mu = d.mu;
  c.sigma = d.sigma;
  c.cap = d.cap;
  c.n_buckets = static_cast<int32_t>(d.weights.size());
  for (std::size_t i = 0; i < d.edges.size() && i <= SCLS_MAX_BUCKETS; ++i) c.edges[i] = d.edges[i];
  for (std::size_t i = 0; i < d.weights.size() && i < SCLS_MAX_BUCKETS; ++i) c.weights[i] = d.weights[i];
  return c;
}

scls_workload_spec to_c(const WorkloadSpec& w) {
  scls_workload_spec c{};
  c.rate = w.rate;
  c.duration_s = w.duration_s;
  c.input_len_dist = to_c(w.input_len_dist);
  c.gen_len_dist = to_c(w.gen_len_dist);
  c.max_input_limit = w.max_input_limit;
  c.max_gen_limit = w.max_gen_limit;
  c.seed = w.seed;
  return c;
}

}  // namespace

RunResult run_experiment(const RunConfig& cfg) {
  // experiment.cpp:39-60: models -> workload -> Simulator::run -> compute.
  // Uniform / histogram workloads are generated on the device
  // (scls_run_experiments, bit-exact with generate()); the run's event log and
  // its MetricsReport both come from the device (metrics.cpp:30-117 computed
  // online, bit for bit), so neither generate() nor compute() runs on the
  // host.  Trace files and log-normal lengths are loaded / generated on the host.
  const LatencyModel latency = resolve_latency_model(cfg.latency_model_path);
  const MemoryModel memory = resolve_memory_model(cfg.memory_model_path);
  std::vector<Request> requests;
  scls_workload_spec spec{};
  const bool on_dev = device_generated(cfg);
  if (on_dev) {
    validate(cfg.workload);  // generate()'s own check (workload.cpp:86-98), same exception
    spec = to_c(cfg.workload);
  } else {
    requests = load_workload(cfg);
  }
  Simulator check_cfg(cfg.sched, latency, memory, cfg.horizon_s);  // constructor validation (sim_engine.cpp:32-35)
  const scls_sched_cfg c = b200::to_c(cfg.sched, cfg.horizon_s);
  const int32_t bins = b200::report_hist_bins(c);
  RunResult result;
  if (!on_dev) {
    // Simulator::run's own preconditions (sim_engine.cpp:102-114) on the host-built workload
    std::stable_sort(requests.begin(), requests.end(), [](const Request& a, const Request& b) {
      if (a.arrival_time != b.arrival_time) return a.arrival_time < b.arrival_time;
      return a.id < b.id;
    });
    for (std::size_t i = 0; i < requests.size(); ++i)
      if (requests[i].id != static_cast<RequestId>(i))
        throw Error("workload request ids must be 0..n-1 in arrival order");
    if (requests.empty()) throw EmptyLogError("cannot compute metrics from an empty log");
  }
  const b200::LoggedRun r = b200::run_logged(c, b200::to_c(latency), b200::to_c(memory), bins,
                                             on_dev ? &spec : nullptr, on_dev ? nullptr : &requests);
  b200::raise_status(r, cfg.horizon_s);
  result.log = b200::to_event_log(r, cfg.sched.worker_count);
  result.report = b200::to_report(r.res, r.hist.data(), bins);
  return result;
}

std::vector<SweepRow> sweep(const RunConfig& base, const std::string& param,
                            const std::vector<double>& values) {
  if (values.empty()) throw Error("sweep requires at least one value");
  const std::size_t nv = values.size();
  // Host preparation per value; failures are deferred so they surface in value order.
  std::vector<std::exception_ptr> early(nv);
  std::vector<std::vector<Request>> work(nv);
  std::vector<char> on_dev(nv, 0);
  std::vector<scls_workload_spec> specs(nv);
  std::vector<scls_sched_cfg> cfgs(nv);
  std::vector<scls_latency> lats(nv);
  std::vector<scls_memory> mems(nv);
  for (std::size_t v = 0; v < nv; ++v) {
    try {
      const RunConfig cfg = with_value(base, param, values[v]);
      const LatencyModel lat = resolve_latency_model(cfg.latency_model_path);
      const MemoryModel mem = resolve_memory_model(cfg.memory_model_path);
      if (device_generated(cfg)) {
        validate(cfg.workload);  // generate()'s own check, same exception
        specs[v] = to_c(cfg.workload);
        on_dev[v] = 1;
      } else {
        work[v] = load_workload(cfg);
      }
      Simulator check(cfg.sched, lat, mem, cfg.horizon_s);  // constructor validation
      cfgs[v] = b200::to_c(cfg.sched, cfg.horizon_s);
      lats[v] = b200::to_c(lat);
      mems[v] = b200::to_c(mem);
    } catch (...) {
      early[v] = std::current_exception();
    }
  }
  // Runs sharing models go to the device together (models are per call).
  std::vector<SweepRow> rows(nv);
  std::vector<scls_trace_result> res(nv);
  std::vector<int32_t> done(nv, 0);
  scls_ctx* ctx = b200::context();
  int32_t hist_bins = 2;
  for (std::size_t v = 0; v < nv; ++v)
    if (!early[v] && cfgs[v].slice_len > 0)
      hist_bins = std::max<int32_t>(hist_bins, (cfgs[v].max_gen_limit + cfgs[v].slice_len - 1) / cfgs[v].slice_len + 2);
  std::vector<int64_t> hist(nv * static_cast<std::size_t>(hist_bins));
  for (std::size_t v0 = 0; v0 < nv; ++v0) {
    if (early[v0] || done[v0]) continue;
    std::vector<std::size_t> group;
    for (std::size_t v = v0; v < nv; ++v)
      if (!early[v] && !done[v] && on_dev[v] == on_dev[v0] &&
          std::memcmp(&lats[v], &lats[v0], sizeof(scls_latency)) == 0 &&
          std::memcmp(&mems[v], &mems[v0], sizeof(scls_memory)) == 0)
        group.push_back(v);
    std::vector<int64_t> offs(1, 0);
    std::vector<double> arr;
    std::vector<int32_t> inp, gen, idx;
    std::vector<scls_sched_cfg> gc;
    for (std::size_t g = 0; g < group.size(); ++g) {
      for (const Request& r : work[group[g]]) {
        arr.push_back(r.arrival_time);
        inp.push_back(r.orig_input_len);
        gen.push_back(r.true_gen_len);
      }
      offs.push_back(static_cast<int64_t>(arr.size()));
      gc.push_back(cfgs[group[g]]);
      idx.push_back(static_cast<int32_t>(g));
    }
    std::vector<scls_trace_result> gr(group.size());
    std::vector<int64_t> gh(group.size() * hist_bins);
    if (on_dev[v0]) {
      std::vector<scls_workload_spec> gs;
      for (std::size_t v : group) gs.push_back(specs[v]);
      scls_multi* m = group.size() > 1 ? b200::multi() : nullptr;
      if (m) {  // the runs sharded over every visible GPU, results gathered over NCCL
        const scls_status st = scls_multi_run_experiments(m, static_cast<int32_t>(group.size()), gs.data(), gc.data(),
                                                          &lats[v0], &mems[v0], gr.data(), hist_bins, gh.data(),
                                                          nullptr);
        if (st != SCLS_OK) {
          char buf[1024];
          scls_multi_last_error(m, buf, sizeof buf);
          throw Error(std::string("B200 multi-GPU sweep failed: ") + buf);
        }
      } else {
        // metrics only (no log digests): the sweep keeps reports, not logs
        scls_set_option(ctx, SCLS_OPT_SIM_DIGESTS, 0);
        const scls_status st = scls_run_experiments(ctx, static_cast<int32_t>(group.size()), gs.data(), gc.data(),
                                                    &lats[v0], &mems[v0], gr.data(), hist_bins, gh.data(), nullptr,
                                                    SCLS_MEM_HOST);
        scls_set_option(ctx, SCLS_OPT_SIM_DIGESTS, 1);
        b200::check(ctx, st);
      }
    } else {
      scls_set_option(ctx, SCLS_OPT_SIM_DIGESTS, 0);
      const scls_status st = scls_simulate(ctx, static_cast<int32_t>(group.size()), offs.data(), arr.data(),
                                           inp.data(), gen.data(), static_cast<int32_t>(gc.size()), gc.data(),
                                           idx.data(), &lats[v0], &mems[v0], gr.data(), hist_bins, gh.data(), nullptr,
                                           SCLS_MEM_HOST);
      scls_set_option(ctx, SCLS_OPT_SIM_DIGESTS, 1);
      b200::check(ctx, st);
    }
    for (std::size_t g = 0; g < group.size(); ++g) {
      res[group[g]] = gr[g];
      std::copy(gh.begin() + g * hist_bins, gh.begin() + (g + 1) * hist_bins, hist.begin() + group[g] * hist_bins);
      done[group[g]] = 1;
    }
  }
  for (std::size_t v = 0; v < nv; ++v) {
    if (early[v]) std::rethrow_exception(early[v]);
    const scls_trace_result& r = res[v];
    if (r.status != SCLS_OK) {
      // the failing value re-runs alone with its event log, which raises the
      // reference's exact exception and message (sim_engine.cpp:159-163, ...)
      (void)run_experiment(with_value(base, param, values[v]));
      throw Error("device simulation failed with status " + std::to_string(r.status));
    }
    SweepRow& row = rows[v];
    row.value = values[v];
    row.report = b200::to_report(r, hist.data() + v * hist_bins, hist_bins);
  }
  return rows;
}

namespace {
std::string format_double(double v) {
  std::ostringstream out;
  out.precision(17);
  out << v;
  return out.str();
}
}  // namespace

void write_sweep_csv(std::ostream& out, const std::string& param, const std::vector<SweepRow>& rows) {
  out << param
      << ",throughput,avg_response_s,p95_response_s,ct_std_s,avg_pad_tokens,avg_invalid_tokens,"
         "avg_batch_size,slice_count_hist,early_return_ratio\n";
  for (const SweepRow& row : rows) {
    const MetricsReport& r = row.report;
    std::string hist;
    for (const auto& [slices, fraction] : r.slice_count_hist) {
      if (!hist.empty()) hist += ';';
      hist += std::to_string(slices) + ':' + format_double(fraction);
    }
    out << format_double(row.value) << ',' << format_double(r.throughput) << ','
        << format_double(r.avg_response_s) << ',' << format_double(r.p95_response_s) << ','
        << format_double(r.ct_std_s) << ',' << format_double(r.avg_pad_tokens) << ','
        << format_double(r.avg_invalid_tokens) << ',' << format_double(r.avg_batch_size) << ',' << hist << ','
        << format_double(r.early_return_ratio) << '\n';
  }
}

}  // namespace slicesim
