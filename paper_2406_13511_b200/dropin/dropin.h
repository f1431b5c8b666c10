// dropin.h — shared glue of the B200 drop-in for the reference library.
//
// The files in this directory are meant to REPLACE four translation units of
// the reference's libslicesim_core (core/src/batcher.cpp, offloader.cpp,
// sim_engine.cpp, experiment.cpp): they define the same functions with the
// same signatures and exception behaviour, against the reference's own
// headers, and run the work on the B200 through the C-ABI
// (include/scls_capi.h, libscls_b200.so).  See INTEGRATION.md.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "scls_capi.h"
#include "slicesim/cost_model.h"
#include "slicesim/errors.h"
#include "slicesim/event_log.h"
#include "slicesim/memory_model.h"
#include "slicesim/metrics.h"
#include "slicesim/request.h"
#include "slicesim/sched_policies.h"

namespace slicesim {
namespace b200 {

// One scls_ctx per host thread (the C-ABI contract), created on first use on
// device 0 (SCLS_DEVICE overrides).  Throws Error when no device is usable:
// the drop-in has no CPU fallback.
scls_ctx* context();

// All visible GPUs for device-generated sweeps (scls_multi: contiguous run
// shards, NCCL gather); nullptr with a single GPU.  SCLS_DEVICES=k caps it
// at devices 0..k-1; a list ("0,1", or "0,0" to shard on one GPU) names them.
scls_multi* multi();

// Rethrows the last failure of `ctx` as the matching reference exception
// (errors.h:26-87).
[[noreturn]] void raise(scls_ctx* ctx, scls_status st);
inline void check(scls_ctx* ctx, scls_status st) {
  if (st != SCLS_OK) raise(ctx, st);
}

// One run with its full device event log (device_run.cpp): the workload is
// generated on the device from `spec` (uniform / histogram lengths), or
// taken from `workload`.  Throws only for C-ABI failures; the run's own
// status is in res (raise_status maps it onto the reference's exceptions).
struct LoggedRun {
  std::vector<scls_event_record> recs;
  std::vector<scls_member> mems;
  int64_t rc = 0, mc = 0;
  scls_trace_result res{};
  std::vector<int64_t> hist;
};
LoggedRun run_logged(const scls_sched_cfg& c, const scls_latency& lat, const scls_memory& mem, int32_t hist_bins,
                     const scls_workload_spec* spec, const std::vector<Request>* workload);
void raise_status(const LoggedRun& r, double horizon_s);
EventLog to_event_log(const LoggedRun& r, int worker_count);
MetricsReport to_report(const scls_trace_result& r, const int64_t* hist, int32_t hist_bins);
int32_t report_hist_bins(const scls_sched_cfg& c);

scls_latency to_c(const LatencyModel& m);
scls_memory to_c(const MemoryModel& m);
scls_sched_cfg to_c(const SchedulerConfig& c, double horizon_s);

}  // namespace b200
}  // namespace slicesim
