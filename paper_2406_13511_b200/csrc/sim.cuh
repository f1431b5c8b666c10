// sim.cuh — device discrete-event simulator (reference sim_engine.cpp and
// the three policies of sched_policies.cpp), one trace per warp.
#pragma once

#include "ctx.h"

namespace scls {

// Per-trace scratch layout (byte offsets from the trace's arena base).
struct SimLayout {
  int64_t gen, sl, resp;                                  // per request
  int64_t pool, sk, sk2, sv, T, split, segs, tlog;        // SCLS tick
  int64_t p_eff, p_g, p_t, p_s, p_a;                      // SCLS pool records
  int64_t b_start, b_n, b_lin, b_served, b_next, b_est;   // SCLS batches
  int64_t tl_g, tl_t, tl_e, tl_s, tl_a;                   // SCLS slot state
  int64_t fifo, pf_t, pf_seq, pf_w, run, ex;              // SLS / ILS
  int64_t ct, cp, cr, ra, cn;                             // ILS / SLS completion records, slot arrivals
  int64_t isum;                                           // ILS: per-instance phase-1 summaries (split kernels)
  int64_t ws;                                             // worker slots (W > 32)
  int64_t total;
};

// Bytes reserved per worker slot of the wide variant (sizeof(WorkerState) in
// sim.cu, checked there): W > 32 workers keep their state in the arena,
// ceil(W / 32) slots per lane.
constexpr int64_t kWorkerSlotBytes = 128;

__host__ __device__ inline int64_t sim_align(int64_t x) { return (x + 15) & ~(int64_t)15; }

// n requests, W workers, per-worker FIFO capacity cap_w = ceil(n/W),
// cap = total slices (SCLS tick-log / batch capacity), mc = ILS running cap.
__host__ __device__ inline SimLayout sim_layout(int64_t n, int32_t W, int32_t policy, int64_t cap,
                                                int32_t mc) {
  SimLayout L{};
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o = sim_align(o + bytes);
    return at;
  };
  const int64_t n1 = n + 1;
  const int64_t cap_w = W > 0 ? (n + W - 1) / W : 0;
  // per-request progress; SCLS carries it in its pool records instead
  L.gen = take(policy == SCLS_POLICY_SCLS ? 0 : 4 * n1);
  L.sl = take(policy == SCLS_POLICY_SCLS ? 0 : 4 * n1);
  L.resp = take(8 * n1);
  if (policy == SCLS_POLICY_SCLS) {
    // Repooled requests carry their whole record (id, effective input,
    // generated, true gen, slices, arrival), written contiguously at batch
    // completion, so a tick never chases per-request arrays by id; fresh
    // arrivals are the id range since the last tick (their input rows).
    L.pool = take(4 * n1);
    L.p_eff = take(4 * n1);
    // {generated, true gen, slices, -, arrival, -}: 32 B per repooled record,
    // gathered by pool slot in the tick's rows pass (one sector per member)
    o = (o + 31) & ~(int64_t)31;
    L.p_g = take(32 * n1);
    L.p_t = L.p_s = L.p_a = 0;
    L.sk = take(8 * n1);
    L.sk2 = take(8 * n1);
    L.sv = take(4 * n1);
    L.T = take(8 * (n1 + 1));
    L.split = take(4 * (n1 + 1));
    L.segs = take(4 * (n1 + 1));
    // the tick log: per batched slot the request's state when it was batched
    // {id, generated, true gen, effective input, slices, -, arrival}, 32 B,
    // so offload and batch completion read slot-contiguous records instead
    // of chasing request ids
    o = (o + 31) & ~(int64_t)31;
    L.tlog = take(32 * (cap + 1));
    L.tl_g = L.tl_t = L.tl_e = L.tl_s = L.tl_a = 0;
    o = (o + 31) & ~(int64_t)31;
    L.b_start = take(32 * (cap + 1));  // {start, n, l_in, served; est; next} per batch
    L.b_n = L.b_lin = L.b_served = L.b_next = L.b_est = 0;
  } else if (policy == SCLS_POLICY_SLS) {
    L.fifo = take(4 * (W * cap_w + 1));
    L.pf_t = take(8 * n1);
    L.pf_seq = take(8 * n1);
    L.pf_w = take(4 * n1);
    L.ct = take(8 * (W * cap_w + 1));
    L.cp = take(8 * (W * cap_w + 1));
    L.cr = take(8 * (W * cap_w + 1));
    L.cn = take(4 * (W * cap_w + 1));
    L.isum = take(64 * ((int64_t)W + 1));
  } else {
    L.fifo = take(4 * (W * cap_w + 1));
    L.run = take(16 * ((int64_t)W * mc + 1));
    L.ex = take(4 * ((int64_t)mc + 1));
    L.ct = take(8 * (W * cap_w + 1));
    L.cp = take(8 * (W * cap_w + 1));
    L.cr = take(8 * (W * cap_w + 1));
    L.ra = take(8 * ((int64_t)W * mc + 1));
    L.isum = take(48 * ((int64_t)W + 1));
  }
  L.ws = take(W > 32 ? kWorkerSlotBytes * 32 * (((int64_t)W + 31) / 32) : 0);
  L.total = (o + 127) & ~(int64_t)127;  // trace arenas 128 B aligned (the 32 B records stay in one sector)
  return L;
}

}  // namespace scls
