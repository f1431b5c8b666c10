// poison_host_path.cpp — linked only into build/refsuite/slicesim_b200_strict:
// the reference's host generate() (workload.cpp:163-181) and compute()
// (metrics.cpp:30-117) abort.  That binary's `run` / `sweep` on generated
// uniform / histogram workloads must still produce byte-identical outputs
// (tests/test_cli_dropin.py), proving the B200 drop-in generates the workload
// and computes the report on the device, not on the host.
#include <cstdio>
#include <cstdlib>

#include "slicesim/metrics.h"
#include "slicesim/workload.h"

namespace slicesim {

std::vector<Request> generate(const WorkloadSpec&) {
  std::fprintf(stderr, "poisoned host generate() called\n");
  std::abort();
}

MetricsReport compute(const EventLog&) {
  std::fprintf(stderr, "poisoned host compute() called\n");
  std::abort();
}

}  // namespace slicesim
