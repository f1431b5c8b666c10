// sim_engine_gpu.cpp — drop-in replacement of the reference's
// core/src/sim_engine.cpp: Simulator::run (sim_engine.h:61-67) executes on the
// B200 via scls_simulate (one trace, full event log) and returns the same
// EventLog record for record.
//
// The device runs the three built-in policies (make_scheduler,
// sched_policies.h:136).  A user-defined Scheduler subclass cannot run on the
// device and is rejected with Error — there is no CPU fallback.  The hook
// entry points the policies use from inside a host event loop
// (enqueue_batch, schedule_tick, ...) are therefore unreachable and throw.
#include <algorithm>
#include <string>
#include <vector>

#include "dropin.h"
#include "slicesim/sim_engine.h"

namespace slicesim {

Simulator::Simulator(SchedulerConfig cfg, LatencyModel latency, MemoryModel memory, double horizon_s)
    : cfg_(std::move(cfg)), latency_(latency), memory_(std::move(memory)), horizon_s_(horizon_s) {
  // sim_engine.cpp:32-35 semantics: the same validators, the same errors.
  validate(cfg_);
  validate(latency_);
  validate(memory_);
  if (!(horizon_s_ > 0.0)) throw Error("simulation horizon must be > 0");
  workers_.resize(static_cast<std::size_t>(cfg_.worker_count));
  for (std::size_t i = 0; i < workers_.size(); ++i) workers_[i].id = static_cast<WorkerId>(i);
  log_.worker_count = cfg_.worker_count;
}

namespace {
[[noreturn]] void host_hook() {
  throw Error("the B200 simulator runs the built-in policies on the device; "
              "Simulator hooks are not callable from host code");
}
}  // namespace

void Simulator::enqueue_batch(WorkerId, Batch, int) { host_hook(); }
void Simulator::schedule_tick(double) { host_hook(); }
void Simulator::schedule_policy_event(double, WorkerId) { host_hook(); }
void Simulator::complete_request(RequestId, WorkerId) { host_hook(); }

namespace {
// The post-run Simulator state the reference leaves behind (clock(),
// request(id), workers()), rebuilt from the device event log in log order:
//   - request progress: first dispatch (sched_policies.cpp:128,225,373),
//     generated / slices (:174-175 SCLS, :266-267 SLS, :304,372 ILS) and
//     completion time (sim_engine.cpp:86-99);
//   - worker load_estimate (SCLS): offload's += est in dispatch order
//     (offloader.cpp:50, written back at sched_policies.cpp:111) and
//     complete_batch's clamped -= est at each batch end (offloader.cpp:56-59);
//   - busy_until: the end of the worker's last served batch (sim_engine.cpp:80;
//     ILS never enqueues batches, so it stays 0).
void replay(const EventLog& log, int policy, int max_gen, std::vector<Request>& reqs,
            std::vector<WorkerSim>& workers) {
  std::vector<double> disp_t, est;  // per batch id (SCLS / SLS)
  auto slot = [](std::vector<double>& v, int64_t b) -> double& {
    if (b >= (int64_t)v.size()) v.resize((size_t)b + 1, 0.0);
    return v[(size_t)b];
  };
  for (const EventRecord& e : log.events) {
    if (e.kind == EventKind::kDispatch) {
      if (policy == SCLS_POLICY_ILS) {
        Request& r = reqs[(size_t)e.request];
        r.slices_served = 1;
        if (!r.first_dispatch_time) r.first_dispatch_time = e.t;
        continue;
      }
      slot(disp_t, e.batch) = e.t;
      slot(est, e.batch) = e.est_serve_s;
      if (policy == SCLS_POLICY_SCLS) workers[(size_t)e.worker].load_estimate += e.est_serve_s;
    } else if (e.kind == EventKind::kBatchEnd) {
      if (policy == SCLS_POLICY_ILS) continue;
      WorkerSim& w = workers[(size_t)e.worker];
      w.busy_until = e.t;
      for (const MemberAccounting& m : e.members) {
        Request& r = reqs[(size_t)m.request];
        if (!r.first_dispatch_time) r.first_dispatch_time = slot(disp_t, e.batch);
        r.generated_so_far += m.gen;
        r.slices_served += 1;
      }
      if (policy == SCLS_POLICY_SCLS) {
        w.load_estimate -= slot(est, e.batch);
        if (w.load_estimate < 0.0) w.load_estimate = 0.0;
      }
    } else if (e.kind == EventKind::kComplete) {
      Request& r = reqs[(size_t)e.request];
      r.completion_time = e.t;
      if (policy == SCLS_POLICY_ILS) r.generated_so_far = std::min(r.true_gen_len, max_gen);
    }
  }
}
}  // namespace

EventLog Simulator::run(std::vector<Request> workload, Scheduler& policy) {
  std::stable_sort(workload.begin(), workload.end(), [](const Request& a, const Request& b) {
    if (a.arrival_time != b.arrival_time) return a.arrival_time < b.arrival_time;
    return a.id < b.id;
  });
  for (std::size_t i = 0; i < workload.size(); ++i)
    if (workload[i].id != static_cast<RequestId>(i))
      throw Error("workload request ids must be 0..n-1 in arrival order");
  scls_sched_cfg c = b200::to_c(cfg_, horizon_s_);
  if (dynamic_cast<SclsScheduler*>(&policy)) c.policy = SCLS_POLICY_SCLS;
  else if (dynamic_cast<SlsScheduler*>(&policy)) c.policy = SCLS_POLICY_SLS;
  else if (dynamic_cast<IlsScheduler*>(&policy)) c.policy = SCLS_POLICY_ILS;
  else throw Error("custom Scheduler subclasses cannot run on the B200 device simulator");
  const int64_t n = static_cast<int64_t>(workload.size());
  requests_ = workload;
  if (n == 0) return std::move(log_);
  const scls_latency lat = b200::to_c(latency_);
  const scls_memory mem = b200::to_c(memory_);
  const b200::LoggedRun r = b200::run_logged(c, lat, mem, 0, nullptr, &workload);
  if (r.res.status != SCLS_ERR_EMPTY_LOG) b200::raise_status(r, horizon_s_);  // compute() raises that one
  log_ = b200::to_event_log(r, cfg_.worker_count);
  replay(log_, c.policy, cfg_.max_gen_limit, requests_, workers_);
  clock_ = r.res.sim_clock;
  return std::move(log_);
}

}  // namespace slicesim
