// sim_indep.cuh — metrics-only ILS and SLS simulators with independent instance
// (worker) lanes (included by sim.cu after sim_ils.cuh).  ILS first; SLS at the end.
//
// ILS instances never interact.  Arrivals are assigned round-robin in id
// order (sched_policies.cpp:279-281), so instance w sees exactly the requests
// w, w + W, w + 2W, ...; its boundaries (sched_policies.cpp:292-391) read and
// write only its own queue, running set and segment, and its wake-up fires
// after the arrivals that share its instant (seq < n, sim_engine.cpp:116-119).
// The reference's global (time, seq) order therefore matters for exactly one
// report field: avg_response_s sums the responses in global completion order
// (metrics.cpp:83-85).  Everything else is a count, a max, a per-worker value
// or an order-free selection (p95).
//
// So lane w simulates instance w on its own, at its own pace — no warp
// reduction per event, and an unchanged iteration costs one dependent DADD
// (the step time depends only on the context length, so it is computed ahead)
// — and records each completion as (t, push time of its boundary, response).
// A W-way warp merge then replays the completions in the reference's order:
// by time, then by the push order of the completing boundaries.  Two
// boundaries of different instances at the same time were pushed by their
// instances' previous boundaries, so the earlier push time wins; an exact tie
// of both times would need the push order one level further back, and such a
// job is handed to the exact lock-step kernel (sim_ils_lean_kernel) through a
// device-side fallback list instead.
//
// NonTermination (sim_engine.cpp:160-164): EndOfRun (horizon, seq n) precedes
// every boundary at or after the horizon and every arrival after it, so the
// run fails iff some instance still has work when its next event reaches it.
#pragma once

namespace scls {
namespace {

struct IlsRec {
  double* t;   // completion time
  double* tp;  // push time of the completing boundary (its instance's previous boundary)
  double* r;   // response (t - arrival)
};

#ifndef SCLS_MERGE_SORT
#define SCLS_MERGE_SORT 1
#endif
// per policy: ILS keeps the W-way merge (alone 16.7 vs 18.1 ms sorted, the
// step the same), SLS sorts (8.07 -> 7.88 ms alone)
#ifndef SCLS_MERGE_SORT_ILS
#define SCLS_MERGE_SORT_ILS 0
#endif
#ifndef SCLS_MERGE_WIN
#define SCLS_MERGE_WIN 256
#endif
#ifndef SCLS_INDEP_RUN
#define SCLS_INDEP_RUN 128
#endif
constexpr int kMergeWin = SCLS_MERGE_WIN;  // merge window entries per warp (time key + response), reused as p95 bins
constexpr int kIndepRun = SCLS_INDEP_RUN;  // ILS running slots per warp (W * MC), shared memory
// Replays the W per-instance completion lists (sorted; list w of lane w,
// comp records) in the reference's global order -- time, then push time of
// the completing event -- into resp[0, completed).  Each instance streams its
// records through a shared-memory window (kMergeWin / W entries, refilled by
// the whole warp).  A step selects by a 32-bit fixed-point image of the time
// (monotone, so its minimum holds the minimum time; one REDUX); only lanes
// sharing that image compare the exact 64-bit keys.  With run lengths (cn:
// the batch size at a batch's first record), the winner emits the whole run
// -- members of one batch share (time, push time) and complete in member
// order within the one event.
// Returns true on an exact (time, push time) tie between instances, which
// needs the push order one level further back: the caller hands the job to
// the lock-step kernel.
__device__ bool merge_completions(int lane, int W, int comp, int completed, double last_completion, int64_t cap_w,
                                  const double* __restrict__ ct, const double* __restrict__ cp,
                                  const double* __restrict__ cr, const int32_t* __restrict__ cn,
                                  double* __restrict__ resp, uint64_t* wt, double* wr, uint32_t* wq, uint8_t* wn) {
  __syncwarp();  // every lane's completion records (written in the simulation phase) are visible
  const bool runs = cn != nullptr;
  const int ws = kMergeWin / W;
  const int mine = lane < W ? comp : 0;
  double t_lo = mine > 0 ? ct[lane * cap_w] : dinf();
  for (int o = 16; o; o >>= 1) t_lo = fmin(t_lo, __shfl_xor_sync(FULL, t_lo, o));
  const double span = __dsub_rn(last_completion, t_lo);
  const double scale = completed > 0 && span > 0.0 ? __ddiv_rn(4294967040.0, span) : 0.0;
  int k = 0, h = 0;  // records consumed; head position in the window
  int carry_run = 0;  // rest of a run that a window refill cut
  unsigned need = __ballot_sync(FULL, mine > 0);
  uint64_t kt = ~0ull;
  uint32_t kq = 0xffffffffu;
  for (int i = 0;;) {
    while (need) {  // refill the windows of the instances in `need`
      const int q = __ffs(need) - 1;
      need &= need - 1u;
      const int kk = shfl_i(k, q), mq = shfl_i(mine, q);
      for (int e = lane; e < ws; e += 32) {
        const int64_t idx = kk + e;
        if (idx < mq) {
          const double tv = ct[q * cap_w + idx];
          wt[q * ws + e] = ordered_bits(tv);
          wq[q * ws + e] = (uint32_t)__dmul_rn(__dsub_rn(tv, t_lo), scale);
          wr[q * ws + e] = cr[q * cap_w + idx];
          if (runs) wn[q * ws + e] = (uint8_t)min(cn[q * cap_w + idx], 255);
        }
      }
      __syncwarp();
      if (lane == q) {
        h = 0;
        kt = wt[q * ws];
        kq = wq[q * ws];
        if (carry_run > 0) wn[q * ws] = (uint8_t)carry_run;
        carry_run = 0;
      }
    }
    if (i >= completed) break;
    const unsigned mq = __reduce_min_sync(FULL, kq);
    unsigned win = __ballot_sync(FULL, kq == mq);
    if (win & (win - 1u)) {  // same fixed-point image: exact time, then push order
      bool in = (win >> lane) & 1u;
      const unsigned hi = (unsigned)(kt >> 32), lo = (unsigned)kt;
      const unsigned mh = __reduce_min_sync(FULL, in ? hi : 0xffffffffu);
      in = in && hi == mh;
      const unsigned ml = __reduce_min_sync(FULL, in ? lo : 0xffffffffu);
      in = in && lo == ml;
      win = __ballot_sync(FULL, in);
      if (win & (win - 1u)) {
        const uint64_t kp = in ? ordered_bits(cp[lane * cap_w + k]) : ~0ull;
        const unsigned ph = (unsigned)(kp >> 32), pl = (unsigned)kp;
        const unsigned mph = __reduce_min_sync(FULL, ph);
        const unsigned mpl = __reduce_min_sync(FULL, ph == mph ? pl : 0xffffffffu);
        win = __ballot_sync(FULL, in && ph == mph && pl == mpl);
        if (win & (win - 1u)) return true;
      }
    }
    const int wl = __ffs(win) - 1;
    bool refill = false;
    if (!runs) {  // ILS: one record per step, i advances by one on every lane
      if (lane == wl) {
        resp[i] = wr[lane * ws + h];
        ++k;
        ++h;
        if (k == mine) {
          kt = ~0ull;
          kq = 0xffffffffu;
        } else if (h == ws) {
          refill = true;
        } else {
          kt = wt[lane * ws + h];
          kq = wq[lane * ws + h];
        }
      }
      ++i;
      need = __ballot_sync(FULL, refill);
      continue;
    }
    int emitted = 0;
    if (lane == wl) {
      // a run: the rest of this batch (at most 255 per step), same event
      int left = runs ? max((int)wn[lane * ws + h], 1) : 1;
      do {
        resp[i + emitted] = wr[lane * ws + h];
        ++emitted;
        ++k;
        ++h;
        --left;
        if (k == mine) {
          kt = ~0ull;
          kq = 0xffffffffu;
          break;
        }
        if (h == ws) {
          refill = true;
          break;
        }
        kt = wt[lane * ws + h];
        kq = wq[lane * ws + h];
      } while (left > 0);
      if (refill && left > 0) carry_run = left;
    }
    i += shfl_i(emitted, wl);
    need = __ballot_sync(FULL, refill);
  }
  return false;
}

// The same replay by sorting instead of a W-way merge (SCLS_MERGE_SORT, the
// split kernels' default): every completion becomes a 64-bit key -- the
// 32-bit fixed-point image of its time over its source (record index << 5 |
// instance) -- and a warp LSD radix sort on the image (4 passes, stable, so
// equal images stay in instance-major order) orders the job in ~2.5 warp
// instructions per completion, where a merge step costs ~50.  Equal images
// from different instances are then put in exact (time, push time) order by
// an insertion sort of their run (lane 0; rare), which also detects the exact
// cross-instance tie that needs the lock-step kernel (returns true).  kA and
// kB are per-job scratch of >= completed keys each (kB may alias resp); the
// responses land in resp in the reference's order.
__device__ bool sort_completions(int lane, int W, int comp, int completed, double last_completion, int64_t cap_w,
                                 const double* __restrict__ ct, const double* __restrict__ cp,
                                 const double* __restrict__ cr, double* resp, uint64_t* kA, uint64_t* kB,
                                 int32_t* bins) {
  if (completed == 0) return false;
  const int mine = lane < W ? comp : 0;
  double t_lo = mine > 0 ? ct[lane * cap_w] : dinf();
  for (int o = 16; o; o >>= 1) t_lo = fmin(t_lo, __shfl_xor_sync(FULL, t_lo, o));
  const double span = __dsub_rn(last_completion, t_lo);
  const double scale = span > 0.0 ? __ddiv_rn(4294967040.0, span) : 0.0;
  int off = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, off, o);
    if (lane >= o) off += y;
  }
  off -= mine;
  for (int w = 0; w < W; ++w) {
    const int cw = __shfl_sync(FULL, mine, w), ow = __shfl_sync(FULL, off, w);
    for (int i = lane; i < cw; i += 32) {
      const double tv = ct[w * cap_w + i];
      const uint32_t q = (uint32_t)__dmul_rn(__dsub_rn(tv, t_lo), scale);
      kA[ow + i] = ((uint64_t)q << 32) | ((uint32_t)i << 5) | (uint32_t)w;
    }
  }
  __syncwarp();
  uint64_t* keys = warp_radix_sort(completed, kA, nullptr, kB, nullptr, 64, lane, bins, 32) ? kB : kA;
  auto rec = [&](uint64_t k) { return (int64_t)(k & 31u) * cap_w + (int64_t)((uint32_t)k >> 5); };
  int fixed_end = 0;  // runs [.., fixed_end) already put in exact order
  for (int c = 0; c + 1 < completed; c += 32) {
    const int i = c + lane;
    bool f = false;
    if (i + 1 < completed) {
      const uint64_t a = keys[i], b = keys[i + 1];
      f = (a >> 32) == (b >> 32) && (a & 31u) != (b & 31u);
    }
    for (unsigned m = __ballot_sync(FULL, f); m; m &= m - 1u) {
      const int p = c + __ffs(m) - 1;
      int tie = 0;
      if (lane == 0 && p >= fixed_end) {
        const uint32_t img = (uint32_t)(keys[p] >> 32);
        int a = p, b = p + 2;
        while (a > 0 && (uint32_t)(keys[a - 1] >> 32) == img) --a;
        while (b < completed && (uint32_t)(keys[b] >> 32) == img) ++b;
        for (int x = a + 1; x < b && !tie; ++x) {  // stable insertion sort by exact (time, push time)
          const uint64_t kx = keys[x];
          const double tx = ct[rec(kx)], px = cp[rec(kx)];
          int y = x - 1;
          for (; y >= a; --y) {
            const uint64_t ky = keys[y];
            const double ty = ct[rec(ky)], py = cp[rec(ky)];
            if (ty < tx || (ty == tx && py < px)) break;
            if (ty == tx && py == px) {
              tie = (ky & 31u) != (kx & 31u);  // the same event of one instance keeps its order
              break;
            }
            keys[y + 1] = ky;
          }
          keys[y + 1] = kx;
        }
        fixed_end = b;
      }
      __syncwarp();
      fixed_end = __shfl_sync(FULL, fixed_end, 0);
      if (__shfl_sync(FULL, tie, 0)) return true;
    }
  }
  __syncwarp();
  for (int i = lane; i < completed; i += 32) resp[i] = cr[rec(keys[i])];
  return false;
}

#ifndef SCLS_ILS_INDEP_MINB
#define SCLS_ILS_INDEP_MINB 4
#endif
#ifndef SCLS_PACK_SLOTS
#define SCLS_PACK_SLOTS 192  // W = 8, MC = 12: two jobs per warp, one wave of 4096 jobs
#endif
constexpr int kPackSlots = SCLS_PACK_SLOTS;  // ILS running slots per warp: the pack's traces x W x MC
#ifndef SCLS_ILS_PACK_MAX
#define SCLS_ILS_PACK_MAX 2
#endif
constexpr int kIlsPackMax = SCLS_ILS_PACK_MAX;  // jobs per pack (their merges run in series)
// dynamic shared memory of sim_ils_indep_kernel: per warp, the running slots
// (int4), their arrival times (double) and a boundary's join inputs (int)
constexpr size_t kIlsPackSmem = (size_t)kSimWarps * kPackSlots * (sizeof(int4) + sizeof(double) + sizeof(int32_t));
// Split mode (SCLS_OPT ILS split, default on): the simulation kernel packs up
// to 32 / W jobs per warp (all lanes busy) and writes each instance's phase-1
// summary next to its completion records; a second kernel merges and reports
// every job with a warp of its own, so the merges no longer run in series
// behind a pack.
#ifndef SCLS_ILS_PACK_SPLIT
#define SCLS_ILS_PACK_SPLIT 4
#endif
constexpr int kIlsPackMaxSplit = SCLS_ILS_PACK_SPLIT;
constexpr int kPackSlotsSplit = 2 * kPackSlots;
constexpr size_t kIlsPackSmemSplit =
    (size_t)kSimWarps * kPackSlotsSplit * (sizeof(int4) + sizeof(double) + sizeof(int32_t));
struct IlsSum {  // one instance's phase-1 totals (48 B, sim_layout isum)
  int32_t comp, stuck, n_disp, batch_count;
  long long n_ev, batch_members;
  double last_comp, last_end;
};
static_assert(sizeof(IlsSum) == 48, "sim.cuh isum region");

// Packs.  A warp takes a pack of up to min(kIlsPackMax = 2, 32 / W,
// kPackSlots / (W * MC)) jobs of one config (host: pack_off / jobs); in phase 1 lane gi * W + w simulates instance w of job
// gi, so with W = 8 all 32 lanes do work instead of 8.  The merges and
// reports then run job by job over the whole warp.
struct PackJob {
  int t, n;
  const double* arr;
  char* base;
  SimLayout Lay;
  int64_t cap_w;
};

__device__ __forceinline__ PackJob pack_job(const SimParams& P, int t, int W, int policy, int MC) {
  PackJob j;
  j.t = t;
  const int ts = P.src ? P.src[t] : t;
  const int64_t r0 = P.req_off[ts];
  j.n = (int)(P.req_off[ts + 1] - r0);
  j.arr = P.arr + r0;
  j.base = P.arena + P.trace_base[t];
  j.Lay = sim_layout(j.n, W, policy, P.trace_cap[t], MC);
  j.cap_w = (j.n + W - 1) / W;
  return j;
}

// Validates each job of the pack (Simulator::Simulator, sim_engine.cpp:32-35,
// 102-114) and reports the failed ones; returns the mask of jobs to simulate.
__device__ unsigned pack_validate(const SimParams& P, const int32_t* jobs, int np, int ci, int W, int lane,
                                  int32_t* bins) {
  unsigned ok = 0;
  for (int q = 0; q < np; ++q) {
    const int t = jobs[q];
    const int ts = P.src ? P.src[t] : t;
    const int64_t r0 = P.req_off[ts];
    const int n = (int)(P.req_off[ts + 1] - r0);
    const double* arr = P.arr + r0;
    int status = P.cfg_ok[ci] ? SCLS_OK : SCLS_ERR_ERROR;
    if (status == SCLS_OK) status = trace_input_status(arr, P.inp + r0, P.tg + r0, n, lane);
    int64_t* hist = P.hist ? P.hist + (int64_t)t * P.hist_bins : nullptr;
    if (hist)
      for (int i = lane; i < P.hist_bins; i += 32) hist[i] = 0;
    if (status != SCLS_OK)
      finish_report(lane, &P.res[t], status, n, W, 0, 0.0, 0.0, nullptr, bins, 0.0, 0, 0, 0, 0, 0, 0, 0, 0, 0.0);
    else
      ok |= 1u << q;
  }
  return ok;
}

// Phase 2 of one ILS job (lanes < W hold its instances' phase-1 totals):
// the completions in the reference's global order, then the report.
__device__ void ils_finish_job(const SimParams& P, int t, int W, int MC, int lane, const IlsSum& s, uint64_t* wt,
                               double* wr, uint32_t* wq, int32_t* bins, int32_t* fb_count, int32_t* fb_list) {
  const bool in = lane < W;
  int c = in ? s.comp : 0, st = in ? s.stuck : 0, nd = in ? s.n_disp : 0, bc = in ? s.batch_count : 0;
  long long ne = in ? s.n_ev : 0, bm = in ? s.batch_members : 0;
  double lc = in ? s.last_comp : -dinf(), le = in ? s.last_end : 0.0;
  const PackJob J = pack_job(P, t, W, SCLS_POLICY_ILS, MC);
  scls_trace_result* R = &P.res[J.t];
  int64_t* hist = P.hist ? P.hist + (int64_t)J.t * P.hist_bins : nullptr;
  if (__any_sync(FULL, st)) {
    finish_report(lane, R, SCLS_ERR_NON_TERMINATION, J.n, W, 0, 0.0, 0.0, nullptr, bins, 0.0, 0, 0, 0, 0, 0, 0, 0,
                  0, 0.0);
    return;
  }
  const int completed = __reduce_add_sync(FULL, c);
  const long long n_events = J.n + __reduce_add_sync(FULL, (unsigned)ne);  // per-instance counts fit 32 bits
  const int n_disp_all = __reduce_add_sync(FULL, nd);
  const int batch_all = __reduce_add_sync(FULL, bc);
  for (int o = 16; o; o >>= 1) bm += __shfl_xor_sync(FULL, bm, o);
  double last_completion = lc;
  for (int o = 16; o; o >>= 1) last_completion = fmax(last_completion, __shfl_xor_sync(FULL, last_completion, o));
  double* resp = (double*)(J.base + J.Lay.resp);
  const bool tie =
      SCLS_MERGE_SORT && SCLS_MERGE_SORT_ILS && J.cap_w < (1 << 27)
          ? sort_completions(lane, W, c, completed, last_completion, J.cap_w, (const double*)(J.base + J.Lay.ct),
                             (const double*)(J.base + J.Lay.cp), (const double*)(J.base + J.Lay.cr), resp,
                             (uint64_t*)(J.base + J.Lay.gen), (uint64_t*)resp, bins)
          : merge_completions(lane, W, c, completed, last_completion, J.cap_w, (const double*)(J.base + J.Lay.ct),
                              (const double*)(J.base + J.Lay.cp), (const double*)(J.base + J.Lay.cr), nullptr, resp,
                              wt, wr, wq, nullptr);
  if (tie) {  // the exact lock-step kernel re-runs this job
    if (lane == 0) fb_list[atomicAdd(fb_count, 1)] = J.t;
    return;
  }
  __syncwarp();
  if (hist && P.hist_bins > 1 && lane == 0) hist[1] = completed;
  finish_report(lane, R, SCLS_OK, J.n, W, completed, J.n > 0 ? J.arr[0] : dinf(), last_completion, resp, bins, le,
                0, 0, batch_all, bm, 0, n_events, n_disp_all, 0, last_completion);
}

template <bool kSplit>
__global__ void __launch_bounds__(kSimWarps * 32, SCLS_ILS_INDEP_MINB)
    sim_ils_indep_kernel(SimParams P, const int32_t* __restrict__ pack_off, const int32_t* __restrict__ jobs,
                         int32_t count, int32_t* __restrict__ fb_count, int32_t* __restrict__ fb_list) {
  constexpr int kSlots = kSplit ? kPackSlotsSplit : kPackSlots;
  __shared__ uint64_t swin_t[kSplit ? 1 : kSimWarps][kSplit ? 1 : kMergeWin];
  __shared__ double swin_r[kSplit ? 1 : kSimWarps][kSplit ? 1 : kMergeWin];
  __shared__ uint32_t swin_q[kSplit ? 1 : kSimWarps][kSplit ? 1 : kMergeWin];
  __shared__ int32_t sbins_split[kSplit ? kSimWarps : 1][kSplit ? 256 : 1];
  extern __shared__ __align__(16) unsigned char ils_dyn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int4* srun = (int4*)ils_dyn + warp * kSlots;  // running slots
  double* sra = (double*)(ils_dyn + (size_t)kSimWarps * kSlots * sizeof(int4)) + warp * kSlots;
  int32_t* sjin = (int32_t*)(ils_dyn + (size_t)kSimWarps * kSlots * (sizeof(int4) + sizeof(double))) +
                  warp * kSlots;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;  // launches use 1 or kSimWarps warps per CTA
  if (g >= count) return;
  const int p0 = pack_off[g], np = pack_off[g + 1] - p0;
  if (np <= 0) return;  // an empty slot (small launches: one pack per CTA)
  const int32_t* pj = jobs + p0;
  int32_t* bins = kSplit ? sbins_split[warp] : (int32_t*)swin_t[warp];  // p95 bins (after the merge)
  const int ci = P.cfg_index ? P.cfg_index[pj[0]] : 0;  // one config per pack
  const int W = P.cfgs[ci].W, MC = P.cfgs[ci].MC, G = P.cfgs[ci].G;
  const double horizon = P.cfgs[ci].horizon;
  const Lat& lat = P.lat;
  unsigned okm = pack_validate(P, pj, np, ci, W, lane, bins);
  if (kSplit) {  // jobs reported here (invalid) or handed to the fallback: the merge kernel skips them
    const bool fits = np * W * MC <= kSlots;
    if (lane == 0)
      for (int q = 0; q < np; ++q)
        if (!((okm >> q) & 1u) || !fits) {
          const PackJob Jq = pack_job(P, pj[q], W, SCLS_POLICY_ILS, MC);
          ((IlsSum*)(Jq.base + Jq.Lay.isum))->stuck = -1;
        }
    __syncwarp();
  }
  if (okm && np * W * MC > kSlots) {  // running slots do not fit this warp's shared memory (np == 1)
    if (lane == 0)
      for (int q = 0; q < np; ++q)
        if ((okm >> q) & 1u) fb_list[atomicAdd(fb_count, 1)] = pj[q];
    return;
  }

  // ---- phase 1: lane gi * W + w simulates instance w of job gi -----------------------
  int comp = 0, batch_count = 0, n_disp = 0, stuck = 0;
  long long batch_members = 0, n_ev = 0;
  double last_end = 0.0, last_comp = -dinf();
  {
    const int gi = lane / W, w = lane - gi * W;
    const bool active = gi < np && ((okm >> gi) & 1u);
    const PackJob J = pack_job(P, active ? pj[gi] : pj[0], W, SCLS_POLICY_ILS, MC);
    const int n = J.n;
    const double* __restrict__ arr = J.arr;
    const int64_t r0 = P.req_off[P.src ? P.src[active ? pj[gi] : pj[0]] : (active ? pj[gi] : pj[0])];
    const int32_t* __restrict__ inp = P.inp + r0;
    const int32_t* __restrict__ tg = P.tg + r0;
    const int64_t cap_w = J.cap_w;
    // running slots {exit iteration, join iteration, input, -} + their
    // arrival times, sorted by exit iteration (see the boundary below)
    int4* run = srun + lane * MC;
    double* ra = sra + lane * MC;
    int* jin = sjin + lane * MC;
    IlsRec rec{(double*)(J.base + J.Lay.ct) + w * cap_w, (double*)(J.base + J.Lay.cp) + w * cap_w,
               (double*)(J.base + J.Lay.cr) + w * cap_w};
    const int n_mine = active && w < n ? (n - 1 - w) / W + 1 : 0;  // requests w, w + W, ...
    int f_head = 0, f_tail = 0;  // joined / arrived (FIFO as counters)
    int n_run = 0, it_cnt = 0, seg_it = 0, seg_n = 0, room = 0;
    int mxd = (-2147483647 - 1);  // max over the running set of (input - join iteration)
    bool seg = false, boundary = false;
    double ev_t = dinf(), t_push = 0.0;
    double a1 = 0.0, a2 = 0.0, dl = 0.0;  // step-time terms of the current membership, next context
    // request stream prefetch: the next two arrivals, and the next join's data
    double next_arr = n_mine > 0 ? arr[w] : dinf();
    double next_arr2 = n_mine > 1 ? arr[w + W] : dinf();
    double j_a = n_mine > 0 ? arr[w] : 0.0;
    int j_i = n_mine > 0 ? inp[w] : 0, j_g = n_mine > 0 ? tg[w] : 0;
    bool live = n_mine > 0;
    auto step = [&](double x) {
      return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a1, x), a2), __dmul_rn(lat.d3, x)), lat.d4);
    };
    // Each outer trip: this lane's run of unchanged iterations (four per inner
    // trip, branch-free), then its next arrival or membership-changing boundary.
    for (;;) {
      const double stop = fmin(next_arr, horizon);
      if (live && boundary && n_run > 0 && !(f_tail > f_head && n_run < MC)) {
        while (room > 0 && ev_t < stop) {
          const double x1 = __dadd_rn(dl, 1.0), x2 = __dadd_rn(dl, 2.0), x3 = __dadd_rn(dl, 3.0),
                       x4 = __dadd_rn(dl, 4.0);
          const double s0 = step(dl), s1 = step(x1), s2 = step(x2), s3 = step(x3);
          const double b1 = __dadd_rn(ev_t, s0), b2 = __dadd_rn(b1, s1), b3 = __dadd_rn(b2, s2),
                       b4 = __dadd_rn(b3, s3);
          const bool c1 = (room > 1) & (b1 < stop);
          const bool c2 = c1 & (room > 2) & (b2 < stop);
          const bool c3 = c2 & (room > 3) & (b3 < stop);
          const int k = 1 + (int)c1 + (int)c2 + (int)c3;
          t_push = c3 ? b3 : (c2 ? b2 : (c1 ? b1 : ev_t));
          ev_t = c3 ? b4 : (c2 ? b3 : (c1 ? b2 : b1));
          dl = c3 ? x4 : (c2 ? x3 : (c1 ? x2 : x1));
          room -= k;
          it_cnt += k;
          seg_it += k;
        }
      }
      const bool arrive = live && next_arr <= ev_t && next_arr <= horizon;
      const bool slow = live && !arrive && boundary && ev_t < next_arr && ev_t < horizon;
      if (!__any_sync(FULL, arrive || slow)) break;
      if (arrive) {
        // on_arrival (sched_policies.cpp:279-290)
        ++f_tail;
        if (n_run == 0 && !boundary) {  // wake: boundary at this instant, after the arrivals
          boundary = true;
          ev_t = next_arr;
          t_push = next_arr;
        }
        next_arr = next_arr2;
        next_arr2 = f_tail + 1 < n_mine ? arr[w + (f_tail + 1) * W] : dinf();
      } else if (slow) {
      // a boundary (sched_policies.cpp:292-391): retire, compact, admit FCFS,
      // and the next step's context / first exit, in one pass over the slots
      const double now = ev_t;
      const int nr = n_run;
      const int it1 = it_cnt + (nr > 0 ? 1 : 0);
      if (nr > 0) {
        it_cnt = it1;
        ++seg_it;
      }
      // The running set is kept sorted by exit iteration, descending, ties
      // with the earliest joined last: a boundary's exits are a suffix
      // (completed back to front = join order, sched_policies.cpp:300-313),
      // a join is an insertion, and the first exit is the last slot.  The
      // largest (input - join) over the set is kept in a register and
      // rescanned only when its slot exits.
      int nexit = 0;
      bool lost_max = false;
      while (nexit < nr) {
        const int q = nr - 1 - nexit;
        const int4 v = run[q];  // {exit iteration, join iteration, input, -}
        if (v.x > it1) break;
        rec.t[comp + nexit] = now;
        rec.tp[comp + nexit] = t_push;
        rec.r[comp + nexit] = now - ra[q];
        lost_max |= v.z - v.y == mxd;
        ++nexit;
      }
      int keep = nr - nexit;
      if (lost_max) {
        mxd = (-2147483647 - 1);
        for (int q = 0; q < keep; ++q) {
          const int4 v = run[q];
          mxd = max(mxd, v.z - v.y);
        }
      }
      const int njoin = min(MC - keep, f_tail - f_head);
      for (int j = 0; j < njoin; ++j) {
        const int lim = min(j_g, G);
        const int ex = it1 + lim;
        int pos = keep + j;
        while (pos > 0 && run[pos - 1].x <= ex) {  // slots exiting no later move behind it
          run[pos] = run[pos - 1];
          ra[pos] = ra[pos - 1];
          --pos;
        }
        run[pos] = make_int4(ex, it1, j_i, 0);
        ra[pos] = j_a;
        jin[j] = j_i;
        mxd = max(mxd, j_i - it1);
        ++f_head;
        if (f_head < n_mine) {
          const int id = w + f_head * W;
          j_a = arr[id];
          j_i = inp[id];
          j_g = tg[id];
        }
      }
      const int nr_new = keep + njoin;
      n_run = nr_new;
      const int mc = mxd + it1;
      const int nx = nr_new > 0 ? run[nr_new - 1].x : 0x7fffffff;
      const bool changed = nexit > 0 || njoin > 0;
      if (changed && seg && seg_it > 0) {  // batch_end record
        ++batch_count;
        batch_members += seg_n;
        ++n_ev;
        seg = false;
        last_end = fmax(last_end, now);
      }
      if (nexit > 0) {
        comp += nexit;
        n_ev += nexit;
        last_comp = now;
      }
      if (nr_new == 0) {
        boundary = false;
        ev_t = dinf();
      } else {
        if (changed) {  // batch_start record
          ++n_ev;
          seg = true;
          seg_n = nr_new;
          seg_it = 0;
        }
        double it = decode_step_time(lat, mc, nr_new);
        for (int j = 0; j < njoin; ++j) it = __dadd_rn(it, prefill_time(lat, 1, jin[j]));
        n_disp += njoin;
        n_ev += njoin;
        const double dn = (double)nr_new;
        a1 = __dmul_rn(lat.d1, dn);
        a2 = __dmul_rn(lat.d2, dn);
        dl = (double)(mc + 1);
        room = nx - it_cnt - 1;
        t_push = now;
        ev_t = __dadd_rn(now, it);
      }
      }
      live = live && (comp < n_mine);
    }
    stuck = comp < n_mine;
  }

  if (kSplit) {  // the merge kernel takes it from here
    const int gi = lane / W, w = lane - gi * W;
    if (gi < np && ((okm >> gi) & 1u)) {
      const PackJob J = pack_job(P, pj[gi], W, SCLS_POLICY_ILS, MC);
      IlsSum* sp = (IlsSum*)(J.base + J.Lay.isum) + w;
      *sp = IlsSum{comp, stuck, n_disp, batch_count, n_ev, batch_members, last_comp, last_end};
    }
    return;
  }
  // ---- phase 2, job by job: the completions in the reference's global order ----------
  for (int q = 0; q < np; ++q) {
    if (!((okm >> q) & 1u)) continue;
    __syncwarp();
    const bool in = lane < W;
    const int src = in ? q * W + lane : lane;  // lane w < W takes instance w of job q
    int c = shfl_i(comp, src), st = shfl_i(stuck, src), nd = shfl_i(n_disp, src), bc = shfl_i(batch_count, src);
    long long ne = shfl_l(n_ev, src), bm = shfl_l(batch_members, src);
    double lc = shfl_d(last_comp, src), le = shfl_d(last_end, src);
    if (!in) {
      c = st = nd = bc = 0;
      ne = bm = 0;
      lc = -dinf();
      le = 0.0;
    }
    const PackJob J = pack_job(P, pj[q], W, SCLS_POLICY_ILS, MC);
    scls_trace_result* R = &P.res[J.t];
    int64_t* hist = P.hist ? P.hist + (int64_t)J.t * P.hist_bins : nullptr;
    if (__any_sync(FULL, st)) {
      finish_report(lane, R, SCLS_ERR_NON_TERMINATION, J.n, W, 0, 0.0, 0.0, nullptr, bins, 0.0, 0, 0, 0, 0, 0, 0, 0,
                    0, 0.0);
      continue;
    }
    const int completed = __reduce_add_sync(FULL, c);
    const long long n_events = J.n + __reduce_add_sync(FULL, (unsigned)ne);  // per-instance counts fit 32 bits
    const int n_disp_all = __reduce_add_sync(FULL, nd);
    const int batch_all = __reduce_add_sync(FULL, bc);
    for (int o = 16; o; o >>= 1) bm += __shfl_xor_sync(FULL, bm, o);
    double last_completion = lc;
    for (int o = 16; o; o >>= 1) last_completion = fmax(last_completion, __shfl_xor_sync(FULL, last_completion, o));
    double* resp = (double*)(J.base + J.Lay.resp);
    const bool tie = merge_completions(lane, W, c, completed, last_completion, J.cap_w,
                                       (const double*)(J.base + J.Lay.ct), (const double*)(J.base + J.Lay.cp),
                                       (const double*)(J.base + J.Lay.cr), nullptr, resp, swin_t[warp], swin_r[warp],
                                       swin_q[warp], nullptr);
    if (tie) {  // the exact lock-step kernel re-runs this job
      if (lane == 0) fb_list[atomicAdd(fb_count, 1)] = J.t;
      continue;
    }
    __syncwarp();
    if (hist && P.hist_bins > 1 && lane == 0) hist[1] = completed;
    finish_report(lane, R, SCLS_OK, J.n, W, completed, J.n > 0 ? J.arr[0] : dinf(), last_completion, resp, bins, le,
                  0, 0, batch_all, bm, 0, n_events, n_disp_all, 0, last_completion);
  }
}


// The split ILS's phase 2: one warp per job (list order, longest first).
__global__ void __launch_bounds__(kSimWarps * 32) sim_ils_merge_kernel(SimParams P, const int32_t* __restrict__ list,
                                                                      int32_t count, int32_t* __restrict__ fb_count,
                                                                      int32_t* __restrict__ fb_list) {
  // sort mode: the radix bins / p95 bins only (256 ints); merge mode: the windows too
  constexpr bool kSort = SCLS_MERGE_SORT && SCLS_MERGE_SORT_ILS;
  constexpr int kWin = kSort ? 128 : kMergeWin, kWin2 = kSort ? 1 : kMergeWin;
  __shared__ uint64_t swin_t[kSimWarps][kWin];
  __shared__ double swin_r[kSimWarps][kWin2];
  __shared__ uint32_t swin_q[kSimWarps][kWin2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;
  if (g >= count) return;
#ifdef SCLS_SKIP_MERGE  // timing experiment only: no reports
  return;
#endif
  const int t = list[g];
  if (t < 0) return;
  const int ci = P.cfg_index ? P.cfg_index[t] : 0;
  const int W = P.cfgs[ci].W, MC = P.cfgs[ci].MC;
  const PackJob J = pack_job(P, t, W, SCLS_POLICY_ILS, MC);
  const IlsSum* sp = (const IlsSum*)(J.base + J.Lay.isum);
  if (__shfl_sync(FULL, lane == 0 ? sp[0].stuck : 0, 0) == -1) return;  // reported / re-run elsewhere
  IlsSum s{};
  if (lane < W) s = sp[lane];
  ils_finish_job(P, t, W, MC, lane, s, swin_t[warp], swin_r[warp], swin_q[warp], (int32_t*)swin_t[warp], fb_count,
                 fb_list);
}

// ---- SLS with independent worker lanes ------------------------------------------------
// SLS workers never interact either: arrivals go round-robin in id order
// (sched_policies.cpp:194-201), a worker dispatches only from its own FIFO
// when idle (:207-243), and its batch ends complete only its members
// (:245-273).  Within a worker, same-instant events run arrivals first (seq <
// n), then in the worker's own push order; a policy event that finds the
// worker busy or its FIFO empty changes nothing, so the worker's timeline is:
// dispatch when idle after the arrivals of an instant, and at every batch end.
// Completions are recorded as (t, push time = the batch's start, response)
// with the batch size at its first member, and merged like ILS.
#ifndef SCLS_SLS_INDEP_MINB
#define SCLS_SLS_INDEP_MINB 7  // one wave of 4096 traces (7.3 ms vs 8.8 ms at 4)
#endif
// Split mode (like ILS): the simulation kernel packs 32 / W jobs of one
// config per warp and writes each worker's totals (64 B, sim_layout isum);
// sim_sls_merge_kernel merges and reports a job per warp.
struct SlsSum {
  int32_t comp, stuck, n_disp, batch_count;
  long long n_ev, batch_members, total_pad, total_inv;
  double last_comp, last_end;
};
static_assert(sizeof(SlsSum) == 64, "sim.cuh isum region (SLS)");

// Phase 2 of one SLS job (lanes < W hold its workers' totals).
__device__ void sls_finish_job(const SimParams& P, int t, int W, int lane, const SlsSum& s, uint64_t* wt,
                               double* wr, uint32_t* wq, uint8_t* wn, int32_t* bins, int32_t* fb_count,
                               int32_t* fb_list) {
  const int ts = P.src ? P.src[t] : t;
  const int64_t r0 = P.req_off[ts];
  const int n = (int)(P.req_off[ts + 1] - r0);
  const double* __restrict__ arr = P.arr + r0;
  scls_trace_result* R = &P.res[t];
  int64_t* hist = P.hist ? P.hist + (int64_t)t * P.hist_bins : nullptr;
  char* base = P.arena + P.trace_base[t];
  const SimLayout Lay = sim_layout(n, W, SCLS_POLICY_SLS, P.trace_cap[t], 1);
  double* resp = (double*)(base + Lay.resp);
  const int64_t cap_w = (n + W - 1) / W;
  const bool in = lane < W;
  const int comp = in ? s.comp : 0, stuck = in ? s.stuck : 0;
  long long n_ev = in ? s.n_ev : 0, batch_members = in ? s.batch_members : 0;
  long long total_pad = in ? s.total_pad : 0, total_inv = in ? s.total_inv : 0;
  const int n_disp = in ? s.n_disp : 0, batch_count = in ? s.batch_count : 0;
  const double last_comp = in ? s.last_comp : -dinf(), last_end0 = in ? s.last_end : 0.0;
  if (__any_sync(FULL, stuck)) {
    finish_report(lane, R, SCLS_ERR_NON_TERMINATION, n, W, 0, 0.0, 0.0, nullptr, bins, 0.0, 0, 0, 0, 0, 0, 0, 0, 0,
                  0.0);
    return;
  }
  const int completed = __reduce_add_sync(FULL, comp);
  const long long n_events = n + __reduce_add_sync(FULL, (unsigned)n_ev);
  const int n_disp_all = __reduce_add_sync(FULL, n_disp);
  const int batch_all = __reduce_add_sync(FULL, batch_count);
  double last_end = last_end0;
  for (int o = 16; o; o >>= 1) {
    batch_members += __shfl_xor_sync(FULL, batch_members, o);
    total_pad += __shfl_xor_sync(FULL, total_pad, o);
    total_inv += __shfl_xor_sync(FULL, total_inv, o);
  }
  double last_completion = last_comp;
  for (int o = 16; o; o >>= 1) last_completion = fmax(last_completion, __shfl_xor_sync(FULL, last_completion, o));
  bool tie = false;
  if (W == 1) {  // one list: already in completion order
    const double* cr = (const double*)(base + Lay.cr);
    __syncwarp();
    for (int i = lane; i < completed; i += 32) resp[i] = cr[i];
  } else {
    tie = SCLS_MERGE_SORT && cap_w < (1 << 27)
              ? sort_completions(lane, W, comp, completed, last_completion, cap_w, (const double*)(base + Lay.ct),
                                 (const double*)(base + Lay.cp), (const double*)(base + Lay.cr), resp,
                                 (uint64_t*)(base + Lay.gen), (uint64_t*)resp, bins)
              : merge_completions(lane, W, comp, completed, last_completion, cap_w, (const double*)(base + Lay.ct),
                                  (const double*)(base + Lay.cp), (const double*)(base + Lay.cr),
                                  (const int32_t*)(base + Lay.cn), resp, wt, wr, wq, wn);
  }
  if (tie) {  // the exact lock-step kernel re-runs this job
    if (lane == 0) fb_list[atomicAdd(fb_count, 1)] = t;
    return;
  }
  __syncwarp();
  if (hist && P.hist_bins > 1 && lane == 0) hist[1] = completed;
  finish_report(lane, R, SCLS_OK, n, W, completed, n > 0 ? arr[0] : dinf(), last_completion, resp, bins, last_end,
                total_pad, total_inv, batch_all, batch_members, 0, n_events, n_disp_all, 0, last_completion);
}

// Phase 1 of SLS for worker w of job t (this lane), into *out.
__device__ __forceinline__ void sls_simulate_worker(const SimParams& P, int t, int W, int w, bool active, SlsSum* out) {
  const int ts = P.src ? P.src[t] : t;
  const int64_t r0 = P.req_off[ts];
  const int n = (int)(P.req_off[ts + 1] - r0);
  const double* __restrict__ arr = P.arr + r0;
  const int32_t* __restrict__ inp = P.inp + r0;
  const int32_t* __restrict__ tg = P.tg + r0;
  const int ci = P.cfg_index ? P.cfg_index[t] : 0;
  const int B = P.cfgs[ci].B, G = P.cfgs[ci].G;
  const double horizon = P.cfgs[ci].horizon;
  const Lat& lat = P.lat;
  char* base = P.arena + P.trace_base[t];
  const SimLayout Lay = sim_layout(n, W, SCLS_POLICY_SLS, P.trace_cap[t], 1);
  const int64_t cap_w = (n + W - 1) / W;
  int comp = 0, batch_count = 0, n_disp = 0;
  long long batch_members = 0, n_ev = 0, total_pad = 0, total_inv = 0;
  double last_end = 0.0, last_comp = -dinf();
  double* rt = (double*)(base + Lay.ct) + w * cap_w;
  double* rp = (double*)(base + Lay.cp) + w * cap_w;
  double* rr = (double*)(base + Lay.cr) + w * cap_w;
  int32_t* rn = (int32_t*)(base + Lay.cn) + w * cap_w;
  const int n_mine = active && w < n ? (n - 1 - w) / W + 1 : 0;  // requests w, w + W, ...
  int f_head = 0, f_tail = 0;  // dispatched / arrived (FIFO as counters)
  bool busy = false;
  int b_head = 0, b_n = 0, b_lin = 0, b_lout = 0;  // in-flight batch: FIFO positions [b_head, b_head + b_n)
  double done_t = dinf(), b_start = 0.0;
  double next_arr = n_mine > 0 ? arr[w] : dinf();
  double next_arr2 = n_mine > 1 ? arr[w + W] : dinf();
  bool live = n_mine > 0;
  // try_dispatch at `now` (sched_policies.cpp:207-243): FCFS batch of <= B
  // from the FIFO, started at once (enqueue_batch + start_next_batch)
  auto dispatch = [&](double now) {
    const int take = min(B, f_tail - f_head);
    int lin = 0, lout = 0;
    long long so = 0, sg = 0;
    for (int j0 = 0; j0 < take; j0 += 4) {  // four members per trip, loads first
      int o[4], gm[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int id = w + (f_head + j0 + u) * W;
        o[u] = j0 + u < take ? inp[id] : 0;
        gm[u] = j0 + u < take ? min(tg[id], G) : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        lin = max(lin, o[u]);
        lout = max(lout, gm[u]);
        so += o[u];
        sg += gm[u];
      }
    }
    // batch_end accounting (sched_policies.cpp:255-266): pad = l_in - orig,
    // invalid = served - min(gen, G), summed over members
    total_pad += (long long)take * lin - so;
    total_inv += (long long)take * lout - sg;
    b_head = f_head;
    b_n = take;
    b_lin = lin;
    b_lout = lout;
    f_head += take;
    busy = true;
    b_start = now;
    done_t = __dadd_rn(now, batch_serve_time(lat, take, lin, lout));
    n_disp += 1;
    n_ev += 2;  // dispatch + batch_start
  };
  for (;;) {
    const bool arrive = live && next_arr <= done_t && next_arr <= horizon;  // arrivals first at an instant
    const bool done = live && !arrive && busy && done_t < next_arr && done_t < horizon;
    if (!__any_sync(FULL, arrive || done)) break;
    if (arrive) {
      // on_arrival (sched_policies.cpp:194-201) + its policy event, which runs
      // after every arrival of this instant
      const double now = next_arr;
      ++f_tail;
      next_arr = next_arr2;
      next_arr2 = f_tail + 1 < n_mine ? arr[w + (f_tail + 1) * W] : dinf();
      if (!busy && next_arr != now) dispatch(now);
    } else if (done) {
      // BatchDone (sim_engine.cpp:151-158, sched_policies.cpp:245-273)
      const double now = done_t;
      ++batch_count;
      batch_members += b_n;
      last_end = fmax(last_end, now);
      for (int j0 = 0; j0 < b_n; j0 += 4) {  // four members per trip, loads first
        double av[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) av[u] = j0 + u < b_n ? arr[w + (b_head + j0 + u) * W] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u;
          if (j < b_n) {
            rt[comp + j] = now;
            rp[comp + j] = b_start;
            rr[comp + j] = now - av[u];
            rn[comp + j] = j == 0 ? b_n : 0;
          }
        }
      }
      comp += b_n;
      n_ev += 1 + b_n;  // batch_end + completions
      last_comp = now;
      busy = false;
      done_t = dinf();
      if (f_tail > f_head) dispatch(now);
    }
    live = live && comp < n_mine;
  }
  *out = SlsSum{comp, comp < n_mine ? 1 : 0, n_disp, batch_count, n_ev, batch_members, total_pad, total_inv,
                last_comp, last_end};
}

__global__ void __launch_bounds__(kSimWarps * 32, SCLS_SLS_INDEP_MINB)
    sim_sls_indep_kernel(SimParams P, const int32_t* __restrict__ list, int32_t count, int32_t* __restrict__ fb_count,
                         int32_t* __restrict__ fb_list) {
  __shared__ uint64_t swin_t[kSimWarps][kMergeWin];
  __shared__ double swin_r[kSimWarps][kMergeWin];
  __shared__ uint32_t swin_q[kSimWarps][kMergeWin];
  __shared__ uint8_t swin_n[kSimWarps][kMergeWin];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;  // launches use 1 or kSimWarps warps per CTA
  if (g >= count) return;
  const int t = list[g];
  if (t < 0) return;  // an empty slot (small launches: one job per CTA)
  int32_t* bins = (int32_t*)swin_t[warp];  // p95 bins (after the merge)
  const int ci = P.cfg_index ? P.cfg_index[t] : 0;
  const int W = P.cfgs[ci].W;
  if (!pack_validate(P, &t, 1, ci, W, lane, bins)) return;
  SlsSum s;
  sls_simulate_worker(P, t, W, lane, lane < W, &s);
  sls_finish_job(P, t, W, lane, s, swin_t[warp], swin_r[warp], swin_q[warp], swin_n[warp], bins, fb_count, fb_list);
}

// Split SLS, phase 1: packs of up to 32 / W jobs (pack_off / jobs), lane
// gi * W + w simulates worker w of job gi; totals into the job's isum region.
__global__ void __launch_bounds__(kSimWarps * 32, SCLS_SLS_INDEP_MINB)
    sim_sls_pack_kernel(SimParams P, const int32_t* __restrict__ pack_off, const int32_t* __restrict__ jobs,
                        int32_t count) {
  __shared__ int32_t sbins[kSimWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;
  if (g >= count) return;
  const int p0 = pack_off[g], np = pack_off[g + 1] - p0;
  if (np <= 0) return;
  const int32_t* pj = jobs + p0;
  const int ci = P.cfg_index ? P.cfg_index[pj[0]] : 0;  // one config per pack
  const int W = P.cfgs[ci].W;
  const unsigned okm = pack_validate(P, pj, np, ci, W, lane, sbins[warp]);
  if (lane == 0)
    for (int q = 0; q < np; ++q)
      if (!((okm >> q) & 1u)) {  // reported by pack_validate: the merge kernel skips it
        const int t = pj[q];
        const int ts = P.src ? P.src[t] : t;
        const int n = (int)(P.req_off[ts + 1] - P.req_off[ts]);
        const SimLayout Lay = sim_layout(n, W, SCLS_POLICY_SLS, P.trace_cap[t], 1);
        ((SlsSum*)(P.arena + P.trace_base[t] + Lay.isum))->stuck = -1;
      }
  __syncwarp();
  const int gi = lane / W, w = lane - gi * W;
  const bool active = gi < np && ((okm >> gi) & 1u);
  const int t = pj[active ? gi : 0];
  SlsSum s;
  sls_simulate_worker(P, t, W, w, active, &s);
  if (active) {
    const int ts = P.src ? P.src[t] : t;
    const int n = (int)(P.req_off[ts + 1] - P.req_off[ts]);
    const SimLayout Lay = sim_layout(n, W, SCLS_POLICY_SLS, P.trace_cap[t], 1);
    ((SlsSum*)(P.arena + P.trace_base[t] + Lay.isum))[w] = s;
  }
}

// Split SLS, phase 2: a warp per job (list order).
__global__ void __launch_bounds__(kSimWarps * 32) sim_sls_merge_kernel(SimParams P, const int32_t* __restrict__ list,
                                                                      int32_t count, int32_t* __restrict__ fb_count,
                                                                      int32_t* __restrict__ fb_list) {
  constexpr int kWin = SCLS_MERGE_SORT ? 128 : kMergeWin, kWin2 = SCLS_MERGE_SORT ? 1 : kMergeWin;
  __shared__ uint64_t swin_t[kSimWarps][kWin];
  __shared__ double swin_r[kSimWarps][kWin2];
  __shared__ uint32_t swin_q[kSimWarps][kWin2];
  __shared__ uint8_t swin_n[kSimWarps][kWin2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;
  if (g >= count) return;
#ifdef SCLS_SKIP_MERGE  // timing experiment only: no reports
  return;
#endif
  const int t = list[g];
  if (t < 0) return;
  const int ci = P.cfg_index ? P.cfg_index[t] : 0;
  const int W = P.cfgs[ci].W;
  const int ts = P.src ? P.src[t] : t;
  const int n = (int)(P.req_off[ts + 1] - P.req_off[ts]);
  const SimLayout Lay = sim_layout(n, W, SCLS_POLICY_SLS, P.trace_cap[t], 1);
  const SlsSum* sp = (const SlsSum*)(P.arena + P.trace_base[t] + Lay.isum);
  if (__shfl_sync(FULL, lane == 0 ? sp[0].stuck : 0, 0) == -1) return;
  SlsSum s{};
  if (lane < W) s = sp[lane];
  sls_finish_job(P, t, W, lane, s, swin_t[warp], swin_r[warp], swin_q[warp], swin_n[warp], (int32_t*)swin_t[warp],
                 fb_count, fb_list);
}
}  // namespace
}  // namespace scls
