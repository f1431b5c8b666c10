// batcher.cuh — device entry points of the scheduling core (batch_requests,
// offload), callable from the C-ABI layer and from the fused SCLS tick.
#pragma once

#include "ctx.h"

namespace scls {

struct BatchInputs {
  int64_t n;
  const int32_t* eff;      // device
  const double* arrival;   // device
  const int64_t* id;       // device
  int32_t slice_len;
  const scls_latency* lat; // host
  const scls_memory* mem;  // host
};

struct BatchOutputs {  // device buffers; order/member_id may be null
  int32_t* order;
  int32_t* seg_begin;  // capacity n+1
  int32_t* l_in;       // capacity n
  double* est;         // capacity n
  int64_t* member_id;
};

// Internal buffers of the last call, for tests and profiling.
struct BatchTrace {
  const double* T;
  const int32_t* split;
  const int32_t* Lrow;
  const int32_t* perm;
  int32_t k_max;
  int32_t n_runs;
  int32_t cost_entries;
};

scls_status batch_requests_device(scls_ctx* ctx, const BatchInputs& in, const BatchOutputs& out,
                                  int64_t* nb_out, BatchTrace* trace);

// Pools of up to 4096 requests: the same results in four launches and one
// host read-back (small.cu).
bool small_pool_eligible(int64_t n);
scls_status batch_requests_small(scls_ctx* ctx, const BatchInputs& in, const BatchOutputs& out, int64_t* nb_out);

// offloader.cpp:25-54 on device arrays; loads/worker ids on device, mutated
// in place; outputs the assignment sequence.
scls_status offload_device(scls_ctx* ctx, int64_t nb, const int64_t* batch_id, const double* est,
                           int32_t n_workers, const int32_t* worker_id, double* load,
                           int64_t* out_batch_id, int32_t* out_worker);

}  // namespace scls
