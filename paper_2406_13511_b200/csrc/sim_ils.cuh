// sim_ils.cuh — lean metrics-only ILS simulator (included by sim.cu).
//
// The same semantics as run_trace<ILS> (reference sched_policies.cpp:275-391,
// sim_engine.cpp:101-168, metrics.cpp:30-117) for the sweep path, where only
// the report is needed (no digests, no event log).  ILS is the event-heaviest
// policy (~309k boundaries per 600 s trace), so this kernel keeps only what
// the report depends on: per-instance registers in lane w, running requests
// as {id, join_iter, lim, inp} slots, the response array, and counters.  For
// ILS every completion has exactly one slice and segment records carry no
// members, so pad / invalid / early-return totals are identically zero.
#pragma once

namespace scls {
namespace {

constexpr int kIlsRunSmem = 128;  // running slots per warp kept in shared memory (W * MC)
constexpr int kOwnBuckets = 1024;  // owner table of the rounds' distinct-key certificate

__device__ __forceinline__ unsigned opaque_u32(unsigned x) {
  unsigned y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ double opaque_f64(double x) {
  double y;
  asm volatile("mov.b64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// Keys of event times: with every time provably positive (see `pos` in the
// kernel) the raw IEEE bits already order them, otherwise ordered_bits().
template <bool kPos>
__device__ __forceinline__ uint64_t time_key(double t) {
  return kPos ? (uint64_t)__double_as_longlong(t) : ordered_bits(t);
}

// Push order of pending events.  The reference orders simultaneous events by
// a global sequence number taken at push time (sim_engine.cpp:101-168).  The
// lean kernel processes several independent boundaries per step ("rounds",
// below), so it records the push order as (round, key of the pushing event):
// rounds are processed in order, one push per lane per round, and within a
// round the pushing events have distinct times processed in time order --
// the same total order as the reference's counter.
struct PushOrder {
  unsigned round;
  uint64_t pkey;
};

// Fast rounds: membership of every instance is fixed until the next arrival
// (or the horizon), so each instance's boundaries follow from its own state.
// With bound = min(limit, every fast instance's SECOND boundary, every other
// instance's pending event), all fast pending events before `bound` are the
// next events in the reference's global order (each push lands at or after
// `bound`), and they are processed together.  A round stops the run when it
// is empty (the next event is an arrival, the horizon, a membership change
// or needs the tie-break) or when two of its events share a time.
template <bool kPos>
__device__ __forceinline__ void ils_fast_rounds(int lane, int W, int MC, double next_arr, double horizon,
                                                const Lat& lat, int n_run, int f_head, int f_tail, int next_exit,
                                                int& it_cnt, int& seg_it, int& mctx, double& ev_t, PushOrder& po,
                                                unsigned& round_ctr, uint8_t* own) {
  const bool has = lane < W && ev_t != dinf();
  bool fast = has && n_run > 0 && it_cnt + 1 < next_exit && !(f_tail > f_head && n_run < MC);
  const uint64_t limit = time_key<kPos>(fmin(next_arr, horizon));
  // Opaque copies: at the 64-register cap the compiler would otherwise
  // rematerialise these (I2F + 2 DMUL) on every round.
  const double dn = (double)n_run;
  const double a1 = opaque_f64(__dmul_rn(lat.d1, dn)), a2 = opaque_f64(__dmul_rn(lat.d2, dn));
  auto step = [&](int ctx) {
    const double dl = (double)ctx;
    return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a1, dl), a2), __dmul_rn(lat.d3, dl)), lat.d4);
  };
  uint64_t key = has ? time_key<kPos>(ev_t) : ~0ull;
  double tnext = __dadd_rn(ev_t, step(mctx + 1));
  for (;;) {
    const uint64_t cand = fast ? time_key<kPos>(tnext) : key;
    const unsigned ch = (unsigned)(cand >> 32), cl = (unsigned)cand;
    const unsigned mh = __reduce_min_sync(FULL, ch);
    const unsigned ml = __reduce_min_sync(FULL, ch == mh ? cl : 0xffffffffu);
    const uint64_t m = ((uint64_t)mh << 32) | ml;
    const uint64_t bound = m < limit ? m : limit;
    const bool in = fast && key < bound;
    const unsigned S = __ballot_sync(FULL, in);
    if (!S) break;
    if (S & (S - 1u)) {
      // Distinct keys are certified by a bucket mask over low key bits with
      // one bucket per member (cheap REDUX.OR); only an inconclusive mask
      // pays for the exact MATCH (distinct sentinels: keys in the round are
      // < limit < ~lane).
      // Distinct keys are certified by an owner table in shared memory: each
      // member writes its lane id into bucket h(key) and reads it back; a
      // member that finds another lane's id (a tie, or a bucket collision --
      // ~2% of rounds with 1024 buckets) sends the round to the exact but slow
      // MATCH (~450 cycles on B200 vs ~80 for the table).
      bool clash = false;
      if (in) {
        const unsigned lo = (unsigned)key;
        const unsigned h = (lo ^ (lo >> 10) ^ (unsigned)(key >> 32)) & (kOwnBuckets - 1);
        own[h] = (uint8_t)lane;
        __syncwarp(S);
        clash = own[h] != (uint8_t)lane;
      }
      if (__any_sync(FULL, clash)) {
        const unsigned same = __match_any_sync(FULL, in ? key : ~(uint64_t)lane);
        if (__any_sync(FULL, same & (same - 1u))) break;
      }
    }
    if (in) {
      it_cnt += 1;
      seg_it += 1;
      mctx += 1;
      po.round = round_ctr;
      po.pkey = key;
      ev_t = tnext;
      key = time_key<kPos>(ev_t);
      fast = it_cnt + 1 < next_exit;
      tnext = __dadd_rn(ev_t, step(mctx + 1));
    }
    ++round_ctr;
  }
}

// Earliest pending instance event by (time, push order); the reference's
// queue order (sim_engine.cpp:101-168).  Returns the lane, -1 if none.
__device__ __forceinline__ int argmin_pending(double ev_t, const PushOrder& po, bool has, int lane, double* bt) {
  const uint64_t key = has ? ordered_bits(ev_t) : ~0ull;
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mh = __reduce_min_sync(FULL, hi);
  const unsigned ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xffffffffu);
  unsigned tie = __ballot_sync(FULL, hi == mh && lo == ml);
  if (tie & (tie - 1u)) {
    bool in = (tie >> lane) & 1u;
    const unsigned r = __reduce_min_sync(FULL, in ? po.round : 0xffffffffu);
    in = in && po.round == r;
    const unsigned ph = (unsigned)(po.pkey >> 32), pl = (unsigned)po.pkey;
    const unsigned mph = __reduce_min_sync(FULL, in ? ph : 0xffffffffu);
    in = in && ph == mph;
    const unsigned mpl = __reduce_min_sync(FULL, in ? pl : 0xffffffffu);
    tie = __ballot_sync(FULL, in && pl == mpl);
  }
  const int w = __ffs(tie) - 1;
  *bt = shfl_d(has ? ev_t : dinf(), w);
  return w;
}

__device__ void finish_report(int lane, scls_trace_result* R, int status, int n, int W, int completed,
                              double first_arrival, double last_completion, double* resp, int32_t* bins,
                              double last_end, long long total_pad, long long total_inv, long long batch_count,
                              long long batch_members, long long early, long long n_events, long long n_disp,
                              long long n_ticks, double clock) {
  if (status == SCLS_OK && (n_events == 0 || completed == 0)) status = SCLS_ERR_EMPTY_LOG;
  double thr = 0.0, avg = 0.0, p95 = 0.0, ctstd = 0.0;
  if (status == SCLS_OK) {
    const double span = last_completion - first_arrival;
    const double comp = (double)completed;
    thr = span > 0.0 ? __ddiv_rn(comp, span) : 0.0;
    // sum in completion order (metrics.cpp:83-85) and nearest-rank p95 (metrics.cpp:87-91)
    double sum = 0.0;
    resp_stats(lane, completed, resp, bins, &sum, &p95);
    avg = __ddiv_rn(sum, comp);
    double mean = 0.0, var = 0.0;
    for (int w = 0; w < W; ++w) mean = __dadd_rn(mean, shfl_d(last_end, w));
    mean = __ddiv_rn(mean, (double)W);
    for (int w = 0; w < W; ++w) {
      const double d = __dadd_rn(shfl_d(last_end, w), -mean);
      var = __dadd_rn(var, __dmul_rn(d, d));
    }
    var = __ddiv_rn(var, (double)W);
    ctstd = __dsqrt_rn(var);
  }
  if (lane == 0) {
    memset(R, 0, sizeof *R);
    R->status = status;
    R->worker_count = W;
    R->error_request_id = -1;
    R->n_requests = n;
    if (status != SCLS_OK) return;
    const double comp = (double)completed;
    R->completed = completed;
    R->throughput = thr;
    R->avg_response_s = avg;
    R->p95_response_s = p95;
    R->ct_std_s = ctstd;
    R->avg_pad_tokens = __ddiv_rn((double)total_pad, comp);
    R->avg_invalid_tokens = __ddiv_rn((double)total_inv, comp);
    R->avg_batch_size = batch_count > 0 ? __ddiv_rn((double)batch_members, (double)batch_count) : 0.0;
    R->early_return_ratio = batch_count > 0 ? __ddiv_rn((double)early, (double)batch_count) : 0.0;
    R->total_pad = total_pad;
    R->total_invalid = total_inv;
    R->batch_count = batch_count;
    R->batch_members = batch_members;
    R->early_returns = early;
    R->n_events = n_events;
    R->n_dispatches = n_disp;
    R->n_ticks = n_ticks;
    R->sim_clock = clock;
  }
}

#ifndef SCLS_ILS_MINB
#define SCLS_ILS_MINB 7  // 28 warps/SM: one wave for 4096 traces, 72 registers
#endif
__global__ void __launch_bounds__(kSimWarps * 32, SCLS_ILS_MINB)
    sim_ils_lean_kernel(SimParams P, const int32_t* __restrict__ list, int32_t count,
                        const int32_t* __restrict__ dcount) {
  if (dcount) count = *dcount;  // fallback launches: the job count lives on the device
  __shared__ int32_t sbins[kSimWarps][256];
  __shared__ int4 srun[kSimWarps][kIlsRunSmem];
  __shared__ uint8_t sown[kSimWarps][kOwnBuckets];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;  // launches use 1 or kSimWarps warps per CTA
  if (g >= count) return;
  const int t = list[g];
  if (t < 0) return;  // an empty slot (small launches: one job per CTA)
  int32_t* bins = sbins[warp];
  const int ts = P.src ? P.src[t] : t;  // source trace of job t
  const int64_t r0 = P.req_off[ts];
  const int n = (int)(P.req_off[ts + 1] - r0);
  const double* __restrict__ arr = P.arr + r0;
  const int32_t* __restrict__ inp = P.inp + r0;
  const int32_t* __restrict__ tg = P.tg + r0;
  const int ci = P.cfg_index ? P.cfg_index[t] : 0;
  const int W = P.cfgs[ci].W, MC = P.cfgs[ci].MC, G = P.cfgs[ci].G;
  const double horizon = P.cfgs[ci].horizon;
  const Lat& lat = P.lat;
  scls_trace_result* R = &P.res[t];
  int64_t* hist = P.hist ? P.hist + (int64_t)t * P.hist_bins : nullptr;

  int status = P.cfg_ok[ci] ? SCLS_OK : SCLS_ERR_ERROR;
  if (status == SCLS_OK) status = trace_input_status(arr, inp, tg, n, lane);
  if (hist)
    for (int i = lane; i < P.hist_bins; i += 32) hist[i] = 0;
  if (status != SCLS_OK) {
    finish_report(lane, R, status, n, W, 0, 0.0, 0.0, nullptr, bins, 0.0, 0, 0, 0, 0, 0, 0, 0, 0, 0.0);
    return;
  }
  char* base = P.arena + P.trace_base[t];
  const SimLayout Lay = sim_layout(n, W, SCLS_POLICY_ILS, P.trace_cap[t], MC);
  double* resp = (double*)(base + Lay.resp);
  // Running slots in this warp's shared memory when W * MC fits (global
  // arena otherwise).  Waiting FIFOs need no storage: arrivals go round-robin
  // in id order (sched_policies.cpp:280), so instance w's k-th arrival is
  // request w + k * W and a FIFO is just its (head, tail) counters.
  int4* run_base = W * MC <= kIlsRunSmem ? srun[warp] : (int4*)(base + Lay.run);

  // instance registers (lane w < W)
  double ev_t = dinf(), last_end = 0.0;
  PushOrder po = {~0u, ~0ull};
  int n_run = 0, boundary = 0, seg_n = 0, seg_lin = 0, seg_it = 0, it_cnt = 0, next_exit = 0, mctx = 0;
  int seg_id = -1, f_head = 0, f_tail = 0;
  // trace registers (uniform)
  // Round counter of PushOrder: one round per processed step, so it wraps only
  // after 2^32 steps of one trace (far beyond any horizon the sweeps use).
  unsigned round_ctr = 0;
  // The first arrival event is arr[0] and the last event of a finished run is
  // its last completion, so neither first_arrival nor the clock is carried.
  double next_arr = n > 0 ? arr[0] : dinf();
  double last_completion = -dinf();
  int cur = 0, completed = 0, rr = 0, next_batch = 0;
  unsigned batch_count = 0, n_disp = 0;  // <= 2n and <= n
  long long batch_members = 0, n_events = 0;
  const unsigned lt = (1u << lane) - 1u;
  // Every event time is positive when arrivals are, the horizon is, and each
  // step time is (nonnegative coefficients with d2 or d4 positive: a boundary
  // always has n >= 1 running).  Then raw IEEE bits order the times.
  const bool pos = n > 0 && arr[0] > 0.0 && horizon > 0.0 && lat.p1 >= 0.0 && lat.p2 >= 0.0 && lat.p3 >= 0.0 &&
                   lat.p4 >= 0.0 && lat.d1 >= 0.0 && lat.d2 >= 0.0 && lat.d3 >= 0.0 && lat.d4 >= 0.0 &&
                   (lat.d2 > 0.0 || lat.d4 > 0.0);

#ifdef SCLS_ILS_PROF  // debug build: per-phase clock64 totals into hist[4..15]
  long long prof[10] = {0}, tp = clock64();
#define ILS_PROF(i)                \
  do {                             \
    const long long tq = clock64(); \
    prof[i] += tq - tp;            \
    tp = tq;                       \
  } while (0)
#else
#define ILS_PROF(i) \
  do {              \
  } while (0)
#endif
  while (completed < n) {
    ILS_PROF(9);
    // ---- fast lane: unchanged iterations (see run_trace<ILS>) -------------------
    // While no instance changes membership, the next arrival and the horizon are
    // fixed, so one precomputed key bounds the run: the loop stops at the first
    // event at or past min(next arrival, horizon) (arrivals win ties), at a time
    // tie between instances, or when the winner's next boundary changes
    // membership.  The tie mask doubles as the winner's lane bit.  The winner's
    // next step time is computed one iteration ahead, off the critical path.
    if (pos)
      ils_fast_rounds<true>(lane, W, MC, next_arr, horizon, lat, n_run, f_head, f_tail, next_exit, it_cnt, seg_it,
                            mctx, ev_t, po, round_ctr, sown[warp]);
    else
      ils_fast_rounds<false>(lane, W, MC, next_arr, horizon, lat, n_run, f_head, f_tail, next_exit, it_cnt, seg_it,
                             mctx, ev_t, po, round_ctr, sown[warp]);
    ILS_PROF(0);
    // ---- general step ----------------------------------------------------------------
    double na_t;
    const int na_w = argmin_pending(ev_t, po, lane < W && ev_t != dinf(), lane, &na_t);
    ILS_PROF(1);
    if (next_arr <= fmin(na_t, horizon)) {  // arrival (seq < n): sched_policies.cpp:279-290
      const int id = cur++;
      const double clock = next_arr;
      next_arr = cur < n ? arr[cur] : dinf();
      ++n_events;
      const int w = rr;  // == id % W
      rr = rr + 1 == W ? 0 : rr + 1;
      const bool wake = shfl_i(n_run == 0 && !boundary, w);  // idle instance: boundary at `clock`
      (void)id;
      if (lane == w) {
        ++f_tail;
        if (wake) {
          ev_t = clock;
          po.round = round_ctr;
          po.pkey = 0;
          boundary = 1;
        }
      }
      if (wake) ++round_ctr;
      ILS_PROF(2);
      continue;
    }
    if (horizon <= na_t) {  // EndOfRun precedes every later event
      status = SCLS_ERR_NON_TERMINATION;
      break;
    }
    // ---- an instance boundary with a membership change (sched_policies.cpp:292-391)
    const int w = na_w;
    const double now = na_t;
    int4* run = run_base + (int64_t)w * MC;
    const int nr = shfl_i(n_run, w);
    const int it1 = shfl_i(it_cnt, w) + (nr > 0 ? 1 : 0);
    const int head = shfl_i(f_head, w), tail = shfl_i(f_tail, w);
    if (lane == w) {
      ev_t = dinf();
      po.round = ~0u;
      if (nr > 0) {
        it_cnt = it1;
        seg_it += 1;
      }
    }
    // retire (survivors compacted in order; exits complete in member order,
    // their responses written straight to resp) and admit FCFS
    int nexit = 0, keep = 0;
    for (int b0 = 0; b0 < nr; b0 += 32) {
      const int i = b0 + lane;
      const bool ok = i < nr;
      int4 v = make_int4(0, 0, 0, 0);
      bool ex = false;
      if (ok) {
        v = run[i];
        ex = it1 - v.y >= v.z;
      }
      const unsigned em = __ballot_sync(FULL, ok && ex);
      const unsigned km = __ballot_sync(FULL, ok && !ex);
      __syncwarp();
      if (ok && ex) resp[completed + nexit + __popc(em & lt)] = now - arr[v.x];
      if (ok && !ex) run[keep + __popc(km & lt)] = v;
      nexit += __popc(em);
      keep += __popc(km);
      __syncwarp();
    }
    ILS_PROF(3);
    const int njoin = min(MC - keep, tail - head);
    for (int j = lane; j < njoin; j += 32) {
      const int id = w + (head + j) * W;
      run[keep + j] = make_int4(id, it1, min(tg[id], G), inp[id]);
    }
    __syncwarp();
    const int nr_new = keep + njoin;
    if (lane == w) {
      f_head = head + njoin;
      n_run = nr_new;
    }
    ILS_PROF(4);
    const bool changed = nexit > 0 || njoin > 0;
    if (changed && shfl_i(seg_id, w) >= 0 && shfl_i(seg_it, w) > 0) {  // batch_end record
      ++batch_count;
      batch_members += shfl_i(seg_n, w);
      ++n_events;
      if (lane == w) {
        seg_id = -1;
        last_end = fmax(last_end, now);
      }
    }
    if (nexit > 0) {  // completions (responses written above)
      completed += nexit;
      n_events += nexit;
      last_completion = now;
    }
    __syncwarp();
    if (nr_new == 0) {
      if (lane == w) boundary = 0;
      continue;
    }
    ILS_PROF(5);
    int mc = 0, nx = 0x7fffffff;
    for (int i = lane; i < nr_new; i += 32) {
      const int4 v = run[i];
      mc = max(mc, v.w + (it1 - v.y));
      nx = min(nx, v.y + v.z);
    }
    mc = __reduce_max_sync(FULL, mc);
    nx = __reduce_min_sync(FULL, nx);
    if (changed) {  // batch_start record
      ++n_events;
      if (lane == w) {
        seg_id = next_batch;
        seg_n = nr_new;
        seg_lin = mc;
        seg_it = 0;
      }
      ++next_batch;
    }
    double it = decode_step_time(lat, mc, nr_new);
    for (int j = 0; j < njoin; ++j) it = __dadd_rn(it, prefill_time(lat, 1, run[keep + j].w));
    n_disp += njoin;
    n_events += njoin;
    if (lane == w) {
      mctx = mc;
      next_exit = nx;
      ev_t = __dadd_rn(now, it);
      po.round = round_ctr;
      po.pkey = 0;
      boundary = 1;
    }
    ++round_ctr;
    ILS_PROF(6);
  }
  (void)seg_lin;
#ifdef SCLS_ILS_PROF
  if (hist && P.hist_bins >= 14 && lane == 0)
    for (int i = 0; i < 10; ++i) hist[4 + i] = prof[i];
#endif
  if (hist && status == SCLS_OK && P.hist_bins > 1 && lane == 0) hist[1] = completed;
  finish_report(lane, R, status, n, W, completed, n > 0 ? arr[0] : dinf(), last_completion, resp, bins, last_end, 0,
                0, batch_count, batch_members, 0, n_events, n_disp, 0, last_completion);
}

}  // namespace
}  // namespace scls
