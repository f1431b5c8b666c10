// post_run_state.cpp — prints the Simulator state a run leaves behind
// (sim_engine.h:64-79: clock(), request(id), workers()) and the NonTermination
// message, for the three policies on a few generated workloads.  Built
// against the reference core (post_run_state_ref) and against the B200
// drop-in (post_run_state_b200); tests/test_reference_suite.py compares the
// two outputs byte for byte.
#include <cstdio>
#include <string>

#include "slicesim/cost_model.h"
#include "slicesim/errors.h"
#include "slicesim/memory_model.h"
#include "slicesim/run_config.h"
#include "slicesim/sched_policies.h"
#include "slicesim/sim_engine.h"
#include "slicesim/workload.h"

using namespace slicesim;

static void dump(const char* tag, Simulator& sim, std::size_t n) {
  std::printf("%s clock=%.17g\n", tag, sim.clock());
  for (std::size_t i = 0; i < n; ++i) {
    const Request& r = sim.request(static_cast<RequestId>(i));
    std::printf("r %zu gen=%d slices=%d first=%.17g done=%.17g\n", i, r.generated_so_far, r.slices_served,
                r.first_dispatch_time ? *r.first_dispatch_time : -1.0,
                r.completion_time ? *r.completion_time : -1.0);
  }
  for (const WorkerSim& w : sim.workers())
    std::printf("w %d load=%.17g busy_until=%.17g idle=%d queued=%zu\n", w.id, w.load_estimate, w.busy_until,
                (int)w.idle(), w.local_queue.size());
}

int main() {
  const PolicyKind kinds[3] = {PolicyKind::kScls, PolicyKind::kSls, PolicyKind::kIls};
  const char* names[3] = {"scls", "sls", "ils"};
  for (int workers : {1, 3, 8}) {
    for (int k = 0; k < 3; ++k) {
      RunConfig rc = default_run_config();
      rc.workload.rate = 4.0 * workers;
      rc.workload.duration_s = 40.0;
      rc.workload.seed = 11 + workers;
      SchedulerConfig cfg = rc.sched;
      cfg.policy = kinds[k];
      cfg.worker_count = workers;
      const std::vector<Request> reqs = generate(rc.workload);
      const LatencyModel lat = builtin_latency_model();
      const MemoryModel mem = builtin_memory_model();
      Simulator sim(cfg, lat, mem);
      auto policy = make_scheduler(kinds[k]);
      sim.run(reqs, *policy);
      const std::string tag = std::string(names[k]) + " W=" + std::to_string(workers);
      dump(tag.c_str(), sim, reqs.size());
      // the same workload against a horizon it cannot reach
      Simulator short_sim(cfg, lat, mem, 25.0);
      auto p2 = make_scheduler(kinds[k]);
      try {
        short_sim.run(reqs, *p2);
        std::printf("%s horizon: no error\n", tag.c_str());
      } catch (const NonTerminationError& e) {
        std::printf("%s horizon: %s\n", tag.c_str(), e.what());
      }
    }
  }
  return 0;
}
