// sim.cu — placeholder until the device simulator lands.
#include "sim.cuh"

namespace scls {
scls_status set_error(scls_ctx* ctx, scls_status st, const std::string& msg);
}

extern "C" scls_status scls_simulate(scls_ctx* ctx, int32_t, const int64_t*, const double*, const int32_t*,
                                     const int32_t*, int32_t, const scls_sched_cfg*, const int32_t*,
                                     const scls_latency*, const scls_memory*, scls_trace_result*, int32_t,
                                     int64_t*, scls_event_log*, int32_t) {
  return scls::set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "scls_simulate: not built yet");
}
