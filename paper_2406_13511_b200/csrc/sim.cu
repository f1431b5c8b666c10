// sim.cu — the slice-by-slice discrete-event serving simulator on device:
// reference sim_engine.cpp:26-168 with the SCLS / SLS / ILS policies of
// sched_policies.cpp:84-391 and the report of metrics.cpp:30-117, batched as
// ONE TRACE PER WARP across thousands of independent traces.
//
// Exactness.  Events are processed in the reference's (time, seq) order:
// arrivals carry seq 0..n-1, EndOfRun seq n, every later push the next seq
// (sim_engine.cpp:43-46, 116-120).  Non-arrival events live in per-lane
// slots (lane w = worker / instance w; at most one pending BatchDone or ILS
// boundary per worker, sim_engine.h:100-119), the SCLS tick in one uniform
// slot, SLS's deferred dispatch checks in a FIFO (pushed at the current
// clock, hence already in (time, seq) order).  Every fp64 expression keeps
// the reference's association order; sums that the reference accumulates
// in a fixed order (response sum, ILS iteration time, ct-std) are
// accumulated in that order.
//
// Per-trace state lives in a per-trace arena (sim_layout) in global memory;
// worker state lives in the lanes' registers (W <= 32; wider configs run a
// variant with ceil(W / 32) worker slots per lane in the trace's arena, any W).  The SCLS tick runs
// the scheduling core warp-wide: LSD radix sort of the pool by
// (eff, arrival-rank == id), the Eq. 10 DP with a per-config cost table, the
// backtrack, the stable descending estimate order and the max-min offload.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "radix.cuh"
#include "scls_common.cuh"
#include "scls_loghash.h"
#include "sim.cuh"

namespace scls {
namespace {

constexpr unsigned FULL = 0xffffffffu;
#ifndef SCLS_SIM_WARPS
#define SCLS_SIM_WARPS 4
#endif
constexpr int kSimWarps = SCLS_SIM_WARPS;  // traces per CTA
#ifndef SCLS_SPLIT_SMEM
#define SCLS_SPLIT_SMEM 256
#endif
#ifndef SCLS_SIM_MINB
#define SCLS_SIM_MINB 7
#endif
constexpr int kSplitSmem = SCLS_SPLIT_SMEM;
#ifndef SCLS_FAR_U
#define SCLS_FAR_U 4
#endif
#ifndef SCLS_KEYS_U
#define SCLS_KEYS_U 2
#endif
constexpr int kFarU = SCLS_FAR_U;    // tick DP: far sources per trip (loads first)
constexpr int kKeysU = SCLS_KEYS_U;  // tick keys: pool rows per lane per trip
#ifndef SCLS_HIST_U
#define SCLS_HIST_U 2
#endif
constexpr int kHistU = SCLS_HIST_U;  // radix histogram: keys per lane per trip
#ifndef SCLS_ROWS_U
#define SCLS_ROWS_U 2
#endif
constexpr int kRowsU = SCLS_ROWS_U;  // tick rows: sorted rows per lane per trip
#ifndef SCLS_EMIT_U
#define SCLS_EMIT_U 1
#endif
constexpr int kEmitU = SCLS_EMIT_U;  // tick emit: served l_out scan unroll
#ifndef SCLS_PUSH_U
#define SCLS_PUSH_U 4
#endif
constexpr int kPushU = SCLS_PUSH_U;
#ifndef SCLS_SIM_DISCARD
#define SCLS_SIM_DISCARD 0  // 1: dead SCLS tick scratch and consumed tick-log lines dropped from L2 (measured slower)
#endif
#ifndef SCLS_CHAIN_ALWAYS
#define SCLS_CHAIN_ALWAYS 1  // the tick DP's chain mode also for launches with few jobs (windows <= 32)
#endif
#ifndef SCLS_DP_PUSH
#define SCLS_DP_PUSH 1  // tick DP chain mode, windows <= 32: the next tile's far candidates ride this tile's chain
#endif
#ifndef SCLS_DP_PAIR
#define SCLS_DP_PAIR 1  // tick DP chain: two steps per broadcast (T[tb+s] formed on every lane)
#endif
#ifndef SCLS_DP_BRANCHFREE
#define SCLS_DP_BRANCHFREE 0  // tick DP: clamped loads + selects instead of divergent branches
#endif
#ifndef SCLS_DP_SELECT_ACCEPT
#define SCLS_DP_SELECT_ACCEPT 1  // tick DP chain: the accept as a select (loads stay conditional)
#endif
#ifndef SCLS_DP_SELECT_FAR
#define SCLS_DP_SELECT_FAR 1  // tick DP far candidates: the accept as a select
#endif  // tick DP decision rounds: final sources pushed per trip

struct SimCfg {
  int32_t policy, S, G, B, MC, W;
  double lambda, gamma, horizon;
  int32_t table;  // cost-table index (SCLS), -1 otherwise
  int32_t mono;   // monotone cost model (dp_mono.cuh): the tick DP may use decision rounds
};

struct SimParams {
  int32_t n_traces;  // jobs
  const int64_t* req_off;  // per source trace
  const int32_t* src;      // job -> source trace (null: identity)
  const double* arr;
  const int32_t* inp;
  const int32_t* tg;
  const SimCfg* cfgs;
  const int32_t* cfg_index;
  const uint8_t* cfg_ok;
  Lat lat;
  int32_t Lmax;
  const int32_t* Kt;    // [table][L]
  const int32_t* coff;  // [table][L] -> offset of c(L, 1) in cost
  const double* cost;
  char* arena;
  const int64_t* trace_base;
  const int64_t* trace_cap;
  scls_trace_result* res;
  int32_t hist_bins;
  int64_t* hist;
  scls_event_record* recs;
  scls_member* mems;
  int64_t rec_cap, mem_cap;
  int64_t* rec_count;
  int64_t* mem_count;
  int32_t n_logged;
};

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000ll); }

// Per-trace input checks, run before any arena write: arrivals in order
// (sim_engine.cpp:102-114 -> Error) and lengths >= 1.  generate() clamps both
// lengths to [1, limit] (workload.cpp:120-128); a hand-built Request with a
// length < 1 would drive the reference's counters negative, which no device
// policy models (the SCLS sort key packs eff >= 1, the arena is sized by
// ceil(gen / S) slices), so such a trace is refused as INVALID_ARGUMENT.
__device__ __forceinline__ int trace_input_status(const double* arr, const int32_t* inp, const int32_t* tg, int n,
                                                  int lane) {
  int order = 0, len = 0;
  for (int i = lane; i < n; i += 32) {
    if (i > 0) order |= arr[i] < arr[i - 1];
    len |= inp[i] < 1 || tg[i] < 1;
  }
  if (__any_sync(0xffffffffu, order)) return SCLS_ERR_ERROR;
  if (__any_sync(0xffffffffu, len)) return SCLS_ERR_INVALID_ARGUMENT;
  return SCLS_OK;
}

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(FULL, v, src); }
__device__ __forceinline__ int shfl_i(int v, int src) { return __shfl_sync(FULL, v, src); }
__device__ __forceinline__ long long shfl_l(long long v, int src) { return __shfl_sync(FULL, v, src); }

// Drop the L2 lines that lie wholly inside [lo, hi) without writing them
// back (discard.global.L2): for arena scratch that is dead -- every later
// read of it is preceded by a write of the same bytes -- so its dirty lines
// neither cost a DRAM write-back nor hold L2 capacity the live tick log and
// pool records need.  Lines shared with a neighbouring range are kept.
__device__ __forceinline__ void l2_discard(const void* lo, const void* hi, int lane) {
#if SCLS_SIM_DISCARD
  uintptr_t a = ((uintptr_t)lo + 127) & ~(uintptr_t)127;
  const uintptr_t e = (uintptr_t)hi & ~(uintptr_t)127;
  for (a += (uintptr_t)128 * lane; a < e; a += (uintptr_t)128 * 32)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
#endif
}

// ---- event-log sink: counters always, digests / records on demand ------------------

template <bool kHash, bool kLog>
struct Sink {
  uint64_t hc, hd, ht, hl;
  int64_t n_events, n_disp, n_ticks;
  scls_event_record* rec;
  scls_member* mem;
  int64_t rec_cap, mem_cap, rec_n, mem_n;

  __device__ void init(scls_event_record* r, scls_member* m, int64_t rc, int64_t mc) {
    hc = hd = ht = hl = SCLS_FNV_OFFSET;
    n_events = n_disp = n_ticks = 0;
    rec = r;
    mem = m;
    rec_cap = rc;
    mem_cap = mc;
    rec_n = mem_n = 0;
  }
  // Uniform call (all lanes, same arguments); lane 0 writes the record.
  __device__ void record(int lane, int32_t kind, double t, int64_t request, int32_t worker,
                         int64_t batch, int32_t n, int32_t l_in, int32_t planned, int32_t served,
                         double est, int32_t input_len, int32_t gen_len, double response,
                         int32_t slices, double next_interval, int32_t members) {
    ++n_events;
    if (kind == 2) ++n_disp;
    if (kind == 1) ++n_ticks;
    if (kHash) {
      hl = scls_hash_record(hl, kind, t, request, worker, batch, n, l_in, planned, served, est,
                            input_len, gen_len, response, slices, next_interval, members);
      if (kind == 5) {
        hc = scls_fnv_bytes(hc, (uint64_t)request);
        ht = scls_fnv_bytes(ht, scls_dbits(t));
      } else if (kind == 2) {
        hd = scls_fnv_bytes(hd, (uint64_t)batch);
        hd = scls_fnv_bytes(hd, (uint64_t)(int64_t)worker);
        hd = scls_fnv_bytes(hd, (uint64_t)(int64_t)n);
        hd = scls_fnv_bytes(hd, (uint64_t)(int64_t)l_in);
      }
    }
    if (kLog) {
      if (lane == 0 && rec_n < rec_cap) {
        scls_event_record& o = rec[rec_n];
        o.t = t;
        o.est_serve_s = est;
        o.response_s = response;
        o.next_interval_s = next_interval;
        o.request = request;
        o.batch = batch;
        o.kind = kind;
        o.worker = worker;
        o.n = n;
        o.l_in = l_in;
        o.planned_l_out = planned;
        o.served_l_out = served;
        o.input_len = input_len;
        o.gen_len = gen_len;
        o.slices = slices;
        o.member_count = members;
        o.member_offset = mem_n;
      }
      ++rec_n;
    }
  }
  // Members of the last batch_end record: one chunk of up to 32 lanes.
  __device__ void members(int lane, int cnt, int64_t request, int32_t eff, int32_t pad,
                          int32_t gen, int32_t inv) {
    if (kHash) {
      for (int i = 0; i < cnt; ++i) {
        hl = scls_hash_member(hl, shfl_l(request, i), shfl_i(eff, i), shfl_i(pad, i),
                              shfl_i(gen, i), shfl_i(inv, i));
      }
    }
    if (kLog) {
      if (lane < cnt && mem_n + lane < mem_cap)
        mem[mem_n + lane] = scls_member{request, eff, pad, gen, inv};
      mem_n += cnt;
    }
  }
};

// ---- warp helpers -------------------------------------------------------------

// (t, seq) lexicographic min over lanes [0, 2^rounds); returns the winning lane.
__device__ __forceinline__ int argmin_event(double t, unsigned long long s, int lane, int rounds,
                                            double* bt, unsigned long long* bs) {
  int bl = lane;
  for (int r = 0; r < rounds; ++r) {
    const int o = 1 << r;
    const double ot = __shfl_xor_sync(FULL, t, o);
    const unsigned long long os = __shfl_xor_sync(FULL, s, o);
    const int ol = __shfl_xor_sync(FULL, bl, o);
    if (ot < t || (ot == t && os < s)) {
      t = ot;
      s = os;
      bl = ol;
    }
  }
  *bt = shfl_d(t, 0);
  *bs = __shfl_sync(FULL, s, 0);
  return shfl_i(bl, 0);
}

// (t, seq) lexicographic min over the lanes with has == true, by warp
// reductions on the order-preserving bits of t (seq only on exact time ties).
__device__ __forceinline__ int argmin_event_redux(double t, unsigned long long s, bool has, int lane,
                                                  double* bt, unsigned long long* bs) {
  const uint64_t key = has ? ordered_bits(t) : ~0ull;
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mh = __reduce_min_sync(FULL, hi);
  const unsigned ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xffffffffu);
  unsigned tie = __ballot_sync(FULL, hi == mh && lo == ml);
  if (__popc(tie) > 1) {
    const bool in = (tie >> lane) & 1u;
    const unsigned sh = (unsigned)(s >> 32), sl = (unsigned)s;
    const unsigned msh = __reduce_min_sync(FULL, in ? sh : 0xffffffffu);
    const unsigned msl = __reduce_min_sync(FULL, in && sh == msh ? sl : 0xffffffffu);
    tie = __ballot_sync(FULL, in && sh == msh && sl == msl);
  }
  const int w = __ffs(tie) - 1;
  *bt = has ? t : dinf();
  *bt = shfl_d(*bt, w);
  *bs = __shfl_sync(FULL, s, w);
  return w;
}

// Stable LSD radix sort of n (key, val) pairs on key bits [lo, bits), warp-wide,
// ping-ponging between (k, v) and (k2, v2).  Returns true when the result is
// in (k2, v2).  bins: 256 ints of this warp's shared memory.  Bits below `lo`
// ride along (a payload packed under the sort key).
__device__ bool warp_radix_sort(int n, uint64_t* k, int32_t* v, uint64_t* k2, int32_t* v2, int bits,
                                int lane, int32_t* bins, int lo = 0) {
  bool swapped = false;
  const unsigned lt = (1u << lane) - 1u;
  for (int shift = lo; shift < bits; shift += 8) {
    const uint32_t mask = bits - shift >= 8 ? 0xffu : ((1u << (bits - shift)) - 1u);
    for (int i = lane; i < 256; i += 32) bins[i] = 0;
    __syncwarp();
    for (int base = 0; base < n; base += 32 * kHistU) {  // kHistU keys per lane per trip, loads first
      uint64_t kk[kHistU];
#pragma unroll
      for (int u = 0; u < kHistU; ++u) kk[u] = base + 32 * u + lane < n ? k[base + 32 * u + lane] : 0ull;
#pragma unroll
      for (int u = 0; u < kHistU; ++u)
        if (base + 32 * u + lane < n) atomicAdd(&bins[(kk[u] >> shift) & mask], 1);
    }
    __syncwarp();
    {  // exclusive scan of 256 bins: 8 per lane
      int loc[8], s = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        loc[q] = bins[lane * 8 + q];
        s += loc[q];
      }
      int incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      int run = incl - s;
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        bins[lane * 8 + q] = run;
        run += loc[q];
      }
    }
    __syncwarp();
    // the next chunk's key is loaded before this chunk's scatter (the keys
    // are only read here; the scatter writes the other buffer)
    uint64_t next_key = lane < n ? k[lane] : 0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const bool ok = i < n;
      const uint64_t key = next_key;
      next_key = base + 32 + lane < n ? k[base + 32 + lane] : 0;
      const int32_t val = (ok && v) ? v[i] : 0;
      const int d = ok ? (int)((key >> shift) & mask) : 256 + lane;
      const unsigned peers = __match_any_sync(FULL, d);
      const int prior = ok ? bins[d] : 0;
      const int dst = prior + __popc(peers & lt);
      __syncwarp();
      if (ok && lane == __ffs(peers) - 1) bins[d] = prior + __popc(peers);
      if (ok) {
        k2[dst] = key;
        if (v) v2[dst] = val;
      }
      __syncwarp();
    }
    uint64_t* tk = k;
    k = k2;
    k2 = tk;
    int32_t* tv = v;
    v = v2;
    v2 = tv;
    swapped = !swapped;
    __syncwarp();
  }
  return swapped;
}

__device__ __forceinline__ int bits_of(uint32_t x) { return x ? 32 - __clz(x) : 0; }

// The digit of a warp radix select: the smallest d with sum(bins[0..d]) > want
// (want < the bins' total); want becomes the rank inside that digit.  Each
// lane owns 8 consecutive digits, one warp scan finds the owner.
__device__ __forceinline__ int select_digit(const int32_t* bins, int& want, int lane) {
  int c[8], s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    c[u] = bins[lane * 8 + u];
    s += c[u];
  }
  int incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  const int owner = __ffs(__ballot_sync(FULL, incl > want)) - 1;
  int digit = 0, acc = incl - s;
  if (lane == owner) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (acc + c[u] > want) {
        digit = lane * 8 + u;
        break;
      }
      acc += c[u];
    }
  }
  digit = __shfl_sync(FULL, digit, owner);
  want -= __shfl_sync(FULL, acc, owner);
  return digit;
}

// Report statistics over resp[0, completed) (completed > 0): the sum in
// completion order (metrics.cpp:83-85: coalesced loads one chunk ahead, then
// 32 dependent DADDs per chunk on broadcast values, every lane holding the
// sum) and the nearest-rank p95 (metrics.cpp:87-91) by a radix select on the
// order-preserving bits, whose first pass shares the sum's loads (the ILS /
// SLS reports; out of line it cost the merge kernels 8%).
#ifndef SCLS_RESP_STATS_INLINE
#define SCLS_RESP_STATS_INLINE 1
#endif
#if SCLS_RESP_STATS_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
void resp_stats(int lane, int completed, const double* resp, int32_t* bins, double* sum_out,
                                        double* p95_out) {
  const size_t rk = (size_t)ceil(__dmul_rn(0.95, (double)completed));
  int want = (int)(rk > 1 ? rk : 1) - 1;
  double sum = 0.0;
  for (int i = lane; i < 256; i += 32) bins[i] = 0;
  __syncwarp();
  double v = lane < completed ? resp[lane] : 0.0;
  for (int c = 0; c < completed; c += 32) {
    const double vn = c + 32 + lane < completed ? resp[c + 32 + lane] : 0.0;
    if (c + lane < completed) atomicAdd(&bins[ordered_bits(v) >> 56], 1);
    const int m = min(32, completed - c);
    for (int j = 0; j < m; ++j) sum = __dadd_rn(sum, __shfl_sync(FULL, v, j));
    v = vn;
  }
  __syncwarp();
  uint64_t prefix = (uint64_t)select_digit(bins, want, lane) << 56;
  __syncwarp();
  for (int shift = 48; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) bins[i] = 0;
    __syncwarp();
    const uint64_t hi_mask = ~0ull << (shift + 8);
    for (int i = lane; i < completed; i += 32) {
      const uint64_t k = ordered_bits(resp[i]);
      if ((k & hi_mask) == prefix) atomicAdd(&bins[(k >> shift) & 0xff], 1);
    }
    __syncwarp();
    prefix |= (uint64_t)select_digit(bins, want, lane) << shift;
    __syncwarp();
  }
  const uint64_t u = (prefix & 0x8000000000000000ull) ? (prefix & ~0x8000000000000000ull) : ~prefix;
  *sum_out = sum;
  *p95_out = __longlong_as_double((long long)u);
}

// Per-worker (SCLS/SLS) / per-instance (ILS) state.  Worker w lives in lane
// w & 31, slot w >> 5 of that lane's slots: V = 1 (W <= 32, one slot in
// registers) or V = kWideV (any W > 32, the reference's worker_count >= 1 of
// sched_policies.cpp:56: ceil(W / 32) slots per lane in the trace's arena,
// slot q of lane l at index 32 q + l, so a warp's 32 lanes touch 32
// consecutive slots).
constexpr int kWideV = 2;  // template tag of the arena-slot variant
struct WorkerState {
  double ev_t = dinf();  // pending BatchDone / ILS boundary
  unsigned long long ev_s = ~0ull;
  double load = 0.0, last_end = 0.0;
  int busy = 0, infl = -1, q_head = -1, q_tail = -1;
  int f_head = 0, f_tail = 0;  // SLS pending / ILS waiting FIFO
  int inf_start = 0, inf_n = 0, inf_lin = 0, inf_lout = 0;  // SLS in-flight batch
  long long inf_id = 0;
  int n_run = 0, boundary = 0, seg_n = 0, seg_lin = 0, seg_it = 0;  // ILS
  int it_cnt = 0, next_exit = 0, mctx = 0;
  long long seg_id = -1;
};
static_assert(sizeof(WorkerState) <= kWorkerSlotBytes, "sim.cuh kWorkerSlotBytes");

// A lane's worker slots: V = 1 one register-resident slot; otherwise nv
// slots in the arena.
template <int V>
struct Slots {
  WorkerState r;
  WorkerState* g = nullptr;
  int nv = 1;
  __device__ __forceinline__ WorkerState& operator[](int q) { return V == 1 ? r : g[q * 32]; }
};

// The (t, seq)-earliest pending worker event (seqs are distinct), or -1.
template <int V>
__device__ __forceinline__ int argmin_worker_event(Slots<V>& ws, int W, int lane, double* bt,
                                                   unsigned long long* bs) {
  if (V == 1) return argmin_event_redux(ws[0].ev_t, ws[0].ev_s, lane < W && ws[0].ev_t != dinf(), lane, bt, bs);
  double t = dinf();
  unsigned long long s = ~0ull;
  int v = 0;
  for (int q = 0; q < ws.nv; ++q) {
    const bool ok = q * 32 + lane < W && ws[q].ev_t != dinf();
    if (ok && (ws[q].ev_t < t || (ws[q].ev_t == t && ws[q].ev_s < s))) {
      t = ws[q].ev_t;
      s = ws[q].ev_s;
      v = q;
    }
  }
  const int l = argmin_event_redux(t, s, t != dinf(), lane, bt, bs);
  return shfl_i(v, l) * 32 + l;
}

// The worker with the minimal (load, worker id) (offloader.cpp:41-48).
template <int V>
__device__ __forceinline__ int argmin_worker_load(Slots<V>& ws, int W, int lane) {
  double bt;
  unsigned long long bs;
  if (V == 1)  // loads are >= 0, so (load, lane) keys order exactly
    return argmin_event_redux(ws[0].load, (unsigned long long)lane, lane < W, lane, &bt, &bs);
  double ld = dinf();
  int v = 0;
  bool has = false;
  for (int q = 0; q < ws.nv; ++q)
    if (q * 32 + lane < W && (!has || ws[q].load < ld)) {  // ascending slots: ties keep the lower id
      ld = ws[q].load;
      v = q;
      has = true;
    }
  const int w = v * 32 + lane;
  const int l = argmin_event_redux(ld, (unsigned long long)w, has, lane, &bt, &bs);
  return shfl_i(w, l);
}

// min over workers of load (sched_policies.cpp:134-146).
template <int V>
__device__ __forceinline__ double min_worker_load(Slots<V>& ws, int W, int lane) {
  double ml = dinf();
  for (int q = 0; q < ws.nv; ++q)
    if (q * 32 + lane < W) ml = fmin(ml, ws[q].load);
  for (int o = 16; o; o >>= 1) ml = fmin(ml, __shfl_xor_sync(FULL, ml, o));
  return ml;
}

// ---- the per-trace simulation -------------------------------------------------------

// SCLS records (sim.cuh layout): a repooled request's state by pool slot, and
// a tick-log entry per batched slot; 32 B each, read as one 16 B vector and
// one double from the same sector.
struct __align__(32) PoolRec {
  int4 gts;  // generated, true gen, slices, -
  double a;  // arrival
  double pad;
};
struct __align__(32) TickRec {
  int4 igte;  // id, generated, true gen, effective input
  int32_t s, pad;
  double a;   // arrival
};
struct __align__(32) BatchRec {
  int4 d;      // tick-log start, members, l_in, served l_out
  double est;  // estimated serve time
  int32_t next, pad;  // next batch in its worker's queue
};
static_assert(sizeof(PoolRec) == 32 && sizeof(TickRec) == 32 && sizeof(BatchRec) == 32, "sim.cuh SCLS record sizes");

template <int POL, bool kHash, bool kLog, int V>
__device__ void run_trace(const SimParams& P, int t, int lane, int32_t* bins, int32_t* ssplit, double* sT) {
  const int ts = P.src ? P.src[t] : t;  // source trace of job t
  const int64_t r0 = P.req_off[ts];
  const int n = (int)(P.req_off[ts + 1] - r0);
  const double* __restrict__ arr = P.arr + r0;
  const int32_t* __restrict__ inp = P.inp + r0;
  const int32_t* __restrict__ tg = P.tg + r0;
  const int ci = P.cfg_index ? P.cfg_index[t] : 0;
  const SimCfg C = P.cfgs[ci];
  scls_trace_result* R = &P.res[t];
  int64_t* hist = P.hist ? P.hist + (int64_t)t * P.hist_bins : nullptr;
  const int W = C.W;
  const bool logging = kLog && t < P.n_logged;

  // Constructor validation (host-checked per config) and the arrival-order
  // rule (sim_engine.cpp:102-114).
  int status = P.cfg_ok[ci] ? SCLS_OK : SCLS_ERR_ERROR;
  if (status == SCLS_OK) status = trace_input_status(arr, inp, tg, n, lane);
  if (hist)
    for (int i = lane; i < P.hist_bins; i += 32) hist[i] = 0;
  if (status != SCLS_OK) {
    if (lane == 0) {
      memset(R, 0, sizeof *R);
      R->status = status;
      R->worker_count = W;
      R->error_request_id = -1;
      R->n_requests = n;
    }
    return;
  }

  char* base = P.arena + P.trace_base[t];
  const SimLayout Lay = sim_layout(n, W, POL, P.trace_cap[t], C.MC);
  int32_t* gen = (int32_t*)(base + Lay.gen);
  int32_t* sl = (int32_t*)(base + Lay.sl);
  double* resp = (double*)(base + Lay.resp);
  if (POL != SCLS_POLICY_SCLS)
    for (int i = lane; i < n; i += 32) {
      gen[i] = 0;
      sl[i] = 0;
    }

  Sink<kHash, kLog> sink;
  sink.init(logging ? P.recs + (int64_t)t * P.rec_cap : nullptr,
            logging ? P.mems + (int64_t)t * P.mem_cap : nullptr, logging ? P.rec_cap : 0,
            logging ? P.mem_cap : 0);

  // Worker / instance state: worker w in lane WL(w), slot WK(w) (see WorkerState).
  Slots<V> ws;
  if (V != 1) {
    ws.g = (WorkerState*)(base + Lay.ws) + lane;
    ws.nv = (W + 31) >> 5;
    for (int q = 0; q < ws.nv; ++q) ws.g[q * 32] = WorkerState();
  }
#define WK(w) ws[V == 1 ? 0 : ((w) >> 5)]
#define WL(w) (V == 1 ? (w) : ((w) & 31))
#define MINE(w) (lane == WL(w))

  // Trace-wide uniform state.
  unsigned long long next_seq = (unsigned long long)n + 1;  // arrivals 0..n-1, EndOfRun n
  double clock = 0.0;
  int cur = 0, completed = 0;
  long long next_batch = 0;
  int rr = 0;  // round-robin cursor (sched_policies.cpp:195,280: rr_++ % W), kept wrapped
  double first_arrival = dinf(), last_completion = -dinf();
  long long total_pad = 0, total_inv = 0, batch_count = 0, batch_members = 0, early = 0;
  double tick_t = dinf();
  unsigned long long tick_s = ~0ull;
  int pool_len = 0, tl_pos = 0, arr_lo = 0;
  int pf_head = 0, pf_tail = 0;  // SLS policy FIFO
  int err_req = -1;
  status = SCLS_OK;

  // Policy-specific arena views.
  int32_t* pool = (int32_t*)(base + Lay.pool);  // SCLS pool records: id, eff, generated, true gen, slices, arrival
  int32_t* p_eff = (int32_t*)(base + Lay.p_eff);
  PoolRec* prec = (PoolRec*)(base + Lay.p_g);  // repooled records by pool slot
  uint64_t* sk = (uint64_t*)(base + Lay.sk);
  uint64_t* sk2 = (uint64_t*)(base + Lay.sk2);
  int32_t* sv = (int32_t*)(base + Lay.sv);
  double* Tg = (double*)(base + Lay.T);
  int32_t* split_g = (int32_t*)(base + Lay.split);
  int32_t* segs = (int32_t*)(base + Lay.segs);
  TickRec* tlog = (TickRec*)(base + Lay.tlog);  // the tick log
  // batches: {tick-log start, members, l_in, served l_out}, estimate, next in
  // the worker queue -- one 32 B record
  BatchRec* brec = (BatchRec*)(base + Lay.b_start);
  const int cap_w = W > 0 ? (n + W - 1) / W : 0;
  int32_t* fifo_base = (int32_t*)(base + Lay.fifo);
  double* pf_t = (double*)(base + Lay.pf_t);
  unsigned long long* pf_seq = (unsigned long long*)(base + Lay.pf_seq);
  int32_t* pf_w = (int32_t*)(base + Lay.pf_w);
  int32_t* run_base = (int32_t*)(base + Lay.run);
  int32_t* ex_base = (int32_t*)(base + Lay.ex);
  const int32_t* Kt = C.table >= 0 ? P.Kt + (int64_t)C.table * (P.Lmax + 1) : nullptr;
  const int32_t* coff = C.table >= 0 ? P.coff + (int64_t)C.table * (P.Lmax + 1) : nullptr;
  const double* cost = P.cost;
  const Lat& lat = P.lat;  // stays in the kernel parameter (constant) bank: frees 16 registers

#ifdef SCLS_SIM_PROF  // debug build: SCLS per-phase clock64 totals into hist[4..15]
  long long prof[12] = {0}, tp = clock64();
#define SIM_PROF(i)                                 \
  do {                                              \
    if (POL == SCLS_POLICY_SCLS) {                  \
      const long long tq = clock64();               \
      prof[i] += tq - tp;                           \
      tp = tq;                                      \
    }                                               \
  } while (0)
#else
#define SIM_PROF(i) \
  do {              \
  } while (0)
#endif
  if (POL == SCLS_POLICY_SCLS) {  // sched_policies.cpp:84: first tick at 0
    tick_t = 0.0;
    tick_s = next_seq++;
  }

  // ---- shared event handlers -------------------------------------------------------

  // sim_engine.cpp:86-99 complete_request for a chunk of `cnt` ids in lane order.
  auto complete_chunk = [&](int cnt, int id, int worker) {
    if (lane < cnt) {
      resp[completed + lane] = clock - arr[id];
      const int s = sl[id];
      if (hist && s >= 0 && s < P.hist_bins) atomicAdd((unsigned long long*)&hist[s], 1ull);
    }
    for (int i = 0; i < cnt; ++i) {
      const int rid = shfl_i(id, i);
      const int s = shfl_i(lane < cnt ? sl[id] : 0, i);
      sink.record(lane, 5, clock, rid, worker, -1, 0, 0, 0, 0, 0.0, 0, 0, clock - arr[rid], s, 0.0, 0);
    }
    completed += cnt;
    if (cnt > 0) last_completion = clock;
  };

  // sim_engine.cpp:63-84 start_next_batch (SCLS: batches queued per worker).
  auto start_next_scls = [&](int w) {
    const int b = shfl_i(WK(w).busy, WL(w)) ? -1 : shfl_i(WK(w).q_head, WL(w));
    if (b < 0) return;
    const int nb_next = brec[b].next;
    if (MINE(w)) {
      WorkerState& k = WK(w);
      k.q_head = nb_next;
      if (k.q_head < 0) k.q_tail = -1;
    }
    const int4 d = brec[b].d;
    const int bn = d.y, blin = d.z, bsv = d.w;
    sink.record(lane, 3, clock, -1, w, b, bn, blin, 0, 0, 0.0, 0, 0, 0.0, 0, 0.0, 0);
    const double serve = batch_serve_time(lat, bn, blin, bsv);
    if (MINE(w)) {
      WorkerState& k = WK(w);
      k.busy = 1;
      k.infl = b;
      k.ev_t = __dadd_rn(clock, serve);
      k.ev_s = next_seq;
    }
    ++next_seq;
  };

  // SLS try_dispatch (sched_policies.cpp:207-243): FCFS batch of <= B from
  // the worker's FIFO; starts at once (the worker is idle, queue empty).
  auto sls_try_dispatch = [&](int w) {
    const int bz = shfl_i(WK(w).busy, WL(w));
    const int head = shfl_i(WK(w).f_head, WL(w)), tail = shfl_i(WK(w).f_tail, WL(w));
    if (bz || tail == head) return;
    const int take = min(C.B, tail - head);
    const int32_t* q = fifo_base + (int64_t)w * cap_w;
    int lin = 0, lout = 0;
    for (int b0 = 0; b0 < take; b0 += 32) {
      const int i = b0 + lane;
      if (i < take) {
        const int id = q[head + i];
        lin = max(lin, inp[id]);
        lout = max(lout, min(tg[id], C.G));
      }
    }
    lin = __reduce_max_sync(FULL, lin);
    lout = __reduce_max_sync(FULL, lout);
    const long long bid = next_batch++;
    const double est = batch_serve_time(lat, take, lin, lout);
    sink.record(lane, 2, clock, -1, w, bid, take, lin, lout, 0, est, 0, 0, 0.0, 0, 0.0, 0);
    sink.record(lane, 3, clock, -1, w, bid, take, lin, 0, 0, 0.0, 0, 0, 0.0, 0, 0.0, 0);
    if (MINE(w)) {
      WorkerState& k = WK(w);
      k.f_head = head + take;
      k.busy = 1;
      k.inf_start = head;
      k.inf_n = take;
      k.inf_lin = lin;
      k.inf_lout = lout;
      k.inf_id = bid;
      k.ev_t = __dadd_rn(clock, est);  // serve time == est (served l_out == planned)
      k.ev_s = next_seq;
    }
    ++next_seq;
  };

  // ---- the SCLS tick (sched_policies.cpp:90-147) ------------------------------------
  auto scls_tick = [&]() -> int {
    int nb = 0;
    // the pool: repooled records [0, pool_len), then the arrivals since the
    // last tick, ids [arr_lo, cur), whose state is their input row
    const int n_rec = pool_len, a_lo = arr_lo;
    const int P_ = pool_len + (cur - arr_lo);
    arr_lo = cur;
    if (P_ > 0) {
      // 1. order the pool by (eff, id); ids are arrival ranks (sim_engine.cpp:110-114).
      //    key = eff << (idb + pb) | id << pb | pool slot: the slot rides under
      //    the sort key, so the rows pass reads each request's record from the
      //    pool (written contiguously at arrival / repooling) instead of
      //    chasing per-request arrays by id.
      const int idb = bits_of((uint32_t)max(n - 1, 1));
      const int pb = bits_of((uint32_t)max(P_ - 1, 1));
      // eff <= Lmax; the slot fits under the key for any n < 2^20 (huge traces
      // sort a slot array alongside)
      const bool packed = idb + pb + bits_of((uint32_t)P.Lmax) <= 64;
      const int sh = packed ? pb : 0;
      int32_t* slot_v = segs;      // free until the backtrack
      int32_t* slot_v2 = split_g;  // free until the DP
      uint32_t emax = 0;
      for (int i0 = lane; i0 < P_; i0 += 32 * kKeysU) {
        int id[kKeysU], e[kKeysU];
#pragma unroll
        for (int u = 0; u < kKeysU; ++u) {
          const int i = i0 + 32 * u;
          id[u] = i < n_rec ? pool[i] : a_lo + (i - n_rec);
          e[u] = i < n_rec ? p_eff[i] : (i < P_ ? inp[id[u]] : 0);
        }
#pragma unroll
        for (int u = 0; u < kKeysU; ++u) {
          const int i = i0 + 32 * u;
          if (i < P_) {
            emax = max(emax, (uint32_t)e[u]);
            sk[i] = ((uint64_t)e[u] << (idb + sh)) | ((uint64_t)id[u] << sh) | (packed ? (uint64_t)i : 0ull);
            if (!packed) slot_v[i] = i;
          }
        }
      }
      emax = __reduce_max_sync(FULL, emax);
      const int top = idb + sh + bits_of(emax);
      __syncwarp();
      SIM_PROF(2);
      const bool sw = packed ? warp_radix_sort(P_, sk, nullptr, sk2, nullptr, top, lane, bins, sh)
                             : warp_radix_sort(P_, sk, slot_v, sk2, slot_v2, top, lane, bins);
      const uint64_t* keys = sw ? sk2 : sk;
      const int32_t* slots = sw ? slot_v2 : slot_v;
      SIM_PROF(3);
      const int kb_id = sh;  // id field position in the sorted key
      const uint64_t idmask = (1ull << idb) - 1ull;
      const uint64_t pmask = (1ull << pb) - 1ull;
      // 2. rows: the batched state of every member, L, K(L) and its cost row,
      //    singleton feasibility (batcher.cpp:40-46)
      int bad = 0x7fffffff;
#if SCLS_DP_PUSH
      int kmx = 0;  // the largest K(L) of the pool
#endif
      for (int i0 = lane; i0 < P_; i0 += 32 * kRowsU) {  // kRowsU rows per lane per trip, loads first
        uint64_t key[kRowsU];
        int q[kRowsU];
#pragma unroll
        for (int u = 0; u < kRowsU; ++u) {
          const bool ok = i0 + 32 * u < P_;
          key[u] = ok ? keys[i0 + 32 * u] : 0ull;
          q[u] = packed ? (int)(key[u] & pmask) : (ok ? slots[i0 + 32 * u] : 0);
        }
        int id[kRowsU], L[kRowsU], g_[kRowsU], t_[kRowsU], s_[kRowsU], k_[kRowsU];
        double a_[kRowsU];
#pragma unroll
        for (int u = 0; u < kRowsU; ++u) {
          const bool ok = i0 + 32 * u < P_;
          id[u] = (int)((key[u] >> kb_id) & idmask);
          L[u] = (int)(key[u] >> (kb_id + idb));
          // a repooled record, or a fresh arrival (slot >= n_rec: its input row)
          const bool rec = ok && q[u] < n_rec;
          int4 pr = make_int4(0, 0, 0, 0);
          double pa = 0.0;
          if (rec) {
            pr = prec[q[u]].gts;
            pa = prec[q[u]].a;
          }
          g_[u] = pr.x;
          t_[u] = rec ? pr.y : (ok ? tg[id[u]] : 0);
          s_[u] = pr.z;
          a_[u] = rec ? pa : (ok ? arr[id[u]] : 0.0);
          k_[u] = ok && L[u] <= P.Lmax ? __ldg(Kt + L[u]) : 0;
        }
#pragma unroll
        for (int u = 0; u < kRowsU; ++u) {
          const int i = i0 + 32 * u;
          if (i < P_) {
            const int64_t qq = tl_pos + i;
            tlog[qq].igte = make_int4(id[u], g_[u], t_[u], L[u]);
            tlog[qq].s = s_[u];
            tlog[qq].a = a_[u];
            sv[i] = L[u];
            if (L[u] > P.Lmax || k_[u] == 0) bad = min(bad, i);
#if SCLS_DP_PUSH
            kmx = max(kmx, k_[u]);
#endif
          }
        }
      }
      bad = __reduce_min_sync(FULL, bad);
#if SCLS_DP_PUSH
      kmx = __reduce_max_sync(FULL, kmx);
#endif
      __syncwarp();
      if (bad != 0x7fffffff) {
        err_req = tlog[tl_pos + bad].igte.x;
        return SCLS_ERR_INFEASIBLE_REQUEST;
      }
      SIM_PROF(4);
      // 3. the DP (batcher.cpp:48-67): tiles of 32 rows, far+mid then the chain.
      //    T and split live in this warp's shared memory when the pool fits.
      //    Cost loads are issued ahead of the dependent adds (4-wide batches
      //    in the far part, a 2-deep pipeline along the chain).
      const bool small = P_ <= kSplitSmem;
      int32_t* split = small ? ssplit : split_g;
      double* T = small ? sT : Tg;
      if (lane == 0) {
        T[0] = 0.0;
        split[0] = 0;
      }
      __syncwarp();
      const double kInf = dinf();
#if SCLS_DP_PUSH
      // chain mode with every window <= 32: a row's sources other than its
      // own tile's are all in the previous tile, whose chain offers them to
      // it in ascending order (accN), so the far loop is skipped
      const bool push = !C.mono && kmx <= 32;
      double accN = kInf;
      int kbN = 0;
#endif
      for (int tb = 0; tb < P_; tb += 32) {
        SIM_PROF(5);
        const int r = tb + 1 + lane;
        const bool valid = r <= P_;
        const int L = valid ? sv[r - 1] : 0;
        const int Wr = valid ? min(__ldg(Kt + L), r) : 0;
        const double* crow = cost + (valid ? __ldg(coff + L) - 1 : 0);
        double acc = kInf;
        int kb = 0;
        const int wmax = __reduce_max_sync(FULL, Wr);
        // candidates with j <= tb, ascending j (k descending)
#if SCLS_DP_PUSH
        if (push && tb > 0) {
          acc = accN;
          kb = kbN;
        } else {
#else
        {
#endif
        int j = max(0, tb + 1 - wmax);
#if SCLS_DP_BRANCHFREE
        {
          // k = r - j >= 1 here (j <= tb < r); loads from min(k, Wr), selects
          const int kcap = max(Wr, 1);
          for (; j + kFarU - 1 <= tb; j += kFarU) {
            double tv[kFarU], cv[kFarU];
#pragma unroll
            for (int u = 0; u < kFarU; ++u) {
              tv[u] = T[j + u];
              cv[u] = __ldg(crow + min(r - (j + u), kcap));
            }
#pragma unroll
            for (int u = 0; u < kFarU; ++u) {
              const int k = r - (j + u);
              const double cand = __dadd_rn(tv[u], cv[u]);
              const bool tk = k <= Wr && cand <= acc;
              acc = tk ? cand : acc;
              kb = tk ? k : kb;
            }
          }
          for (; j <= tb; ++j) {
            const int k = r - j;
            const double cand = __dadd_rn(T[j], __ldg(crow + min(k, kcap)));
            const bool tk = k <= Wr && cand <= acc;
            acc = tk ? cand : acc;
            kb = tk ? k : kb;
          }
        }
#else
        for (; j + kFarU - 1 <= tb; j += kFarU) {
          double tv[kFarU], cv[kFarU];
#pragma unroll
          for (int u = 0; u < kFarU; ++u) {
            const int k = r - (j + u);
            tv[u] = T[j + u];
            cv[u] = k <= Wr ? __ldg(crow + k) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kFarU; ++u) {
            const int k = r - (j + u);
#if SCLS_DP_SELECT_FAR
            const double cand = __dadd_rn(tv[u], cv[u]);
            const bool tk = k <= Wr && cand <= acc;
            acc = tk ? cand : acc;
            kb = tk ? k : kb;
#else
            if (k <= Wr) {
              const double cand = __dadd_rn(tv[u], cv[u]);
              if (cand <= acc) {
                acc = cand;
                kb = k;
              }
            }
#endif
          }
        }
        for (; j <= tb; ++j) {
          const double Tj = T[j];
          const int k = r - j;
          if (k <= Wr) {
            const double cand = __dadd_rn(Tj, __ldg(crow + k));
            if (cand <= acc) {
              acc = cand;
              kb = k;
            }
          }
        }
#endif
        }
        SIM_PROF(11);  // tile setup + far candidates (the rest of the tile goes to slot 5)
        if (C.mono) {
          // decision rounds (dp_mono.cuh): with T[0..a] final, a pending row
          // whose best candidate from sources <= a is strictly below
          // LB = T[a] + c(L_r, 1) is final -- no later source reaches LB.
          // The leading run of decided rows becomes final and is pushed into
          // the rows still pending; row a+1 is always decided.
          bool pend = valid;
          int a = tb;
          double ta = T[tb];
          const double c1r = valid ? __ldg(crow + 1) : 0.0;
          for (;;) {
            const double lb = __dadd_rn(ta, c1r);
            const bool und = pend && r != a + 1 && !(acc < lb);
            const unsigned um = __ballot_sync(FULL, und);
            const int first = um ? __ffs(um) - 1 : 32;  // lanes below it are final
            if (pend && lane < first) {
              T[r] = acc;
              split[r] = r - kb;
              pend = false;
            }
            if (!um) break;
            const int a2 = tb + first;  // new frontier: rows a+1 .. a2 are final
            // push sources j in (a, a2], ascending j (descending k, ties to the smaller k)
            for (int j = a + 1; j <= a2; j += kPushU) {
              double tv[kPushU], cv[kPushU];
#pragma unroll
              for (int u = 0; u < kPushU; ++u) {
                const int jj = min(j + u, a2);
                tv[u] = shfl_d(acc, jj - tb - 1);
                const int k = r - (j + u);
                cv[u] = pend && j + u <= a2 && k >= 1 && k <= Wr ? __ldg(crow + k) : 0.0;
              }
#pragma unroll
              for (int u = 0; u < kPushU; ++u) {
                const int k = r - (j + u);
                if (pend && j + u <= a2 && k >= 1 && k <= Wr) {
                  const double cand = __dadd_rn(tv[u], cv[u]);
                  if (cand <= acc) {
                    acc = cand;
                    kb = k;
                  }
                }
              }
            }
            ta = shfl_d(acc, a2 - tb - 1);
            a = a2;
          }
          __syncwarp();
          continue;
        }
        // the in-tile chain: row tb+s finalises at step s-1 (lane s-1) after
        // T[tb+s-1] arrives; step s offers k = lane + 2 - s to this lane
        double Tj = T[tb];
        const int rows = min(32, P_ - tb);
        // step s is valid for this lane iff 2 <= s <= rows and 1 <= k <= Wr,
        // i.e. s in [s_lo, s_lo + cnt): one unsigned compare per step
        const int s_lo = max(2, lane + 2 - Wr);
        const int cnt = max(0, min(rows, lane + 1) - s_lo + 1);
        auto kval = [&](int s) { return (unsigned)(s - s_lo) < (unsigned)cnt; };
#if SCLS_DP_BRANCHFREE
        // branch-free steps: every step loads a cost from a clamped, always
        // valid k and selects; the accept is a select, not a divergent branch
        const int kcap = max(Wr, 1);
        auto ck = [&](int k) { return __ldg(crow + min(max(k, 1), kcap)); };
        double c1 = 0.0;                                   // step s (never valid at s = 1)
        double c2 = kval(2) ? ck(lane) : 0.0;              // step s + 1
        for (int s = 1; s <= rows; ++s) {
          const double c0 = c1;
          c1 = c2;
          const double cl = ck(lane - s);  // k = lane + 2 - (s + 2)
          c2 = kval(s + 2) ? cl : 0.0;
          const double cand = __dadd_rn(Tj, c0);
          const bool tk = kval(s) && cand <= acc;
          acc = tk ? cand : acc;
          kb = tk ? lane + 2 - s : kb;
          Tj = shfl_d(acc, s - 1);
        }
#elif SCLS_DP_PAIR
        // Two steps per broadcast.  T[tb+s] is lane s-1's acc after its k = 1
        // candidate at step s: min-select of fl(T[tb+s-1] + c(L, 1)) against
        // its acc before step s -- the same operands and the same accept as
        // on that lane, so every lane forms it itself from (acc, c(L, 1)) of
        // lane s-1, shuffled one pair ahead, and step s+1 needs no broadcast:
        // one shuffle latency per two rows on the chain instead of one per row.
        const double* __restrict__ cp = crow + lane;       // c(L_r, lane + 2 - s) = cp[2 - s]
        const double c1own = valid ? __ldg(crow + 1) : 0.0;
#if SCLS_DP_PUSH
        // the next tile's row r + 32 takes source tb+s-1 at step s with
        // k' = 34 + lane - s (<= its window <= 32, so s >= 2)
        const int rN = r + 32;
        const bool vN = push && rN <= P_;
        const int LN = vN ? sv[rN - 1] : 0;
        const int WrN = vN ? min(__ldg(Kt + LN), rN) : 0;
        const double* __restrict__ cpN = cost + (vN ? __ldg(coff + LN) - 1 : 0) + 34 + lane;  // cpN[-s]
        auto kvN = [&](int st) { return 34 + lane - st <= WrN; };
        accN = kInf;
        kbN = 0;
        double caN = kvN(2) ? __ldg(cpN - 2) : 0.0, cbN = kvN(3) ? __ldg(cpN - 3) : 0.0;
#endif
        Tj = shfl_d(acc, 0);  // step 1 offers nothing (sources <= tb were the far part): T[tb+1]
        double Ab = shfl_d(acc, 1), c1b = shfl_d(c1own, 1);  // lane 1 before step 2
        double ca = kval(2) ? __ldg(cp) : 0.0;               // step 2
        double cb = kval(3) ? __ldg(cp - 1) : 0.0;           // step 3
        int s = 2;
        for (; s + 1 <= rows; s += 2) {
          const double na = kval(s + 2) ? __ldg(cp - s) : 0.0;      // step s + 2
          const double nb = kval(s + 3) ? __ldg(cp - s - 1) : 0.0;  // step s + 3
          const double t1 = __dadd_rn(Tj, c1b);
          const double Ts = t1 <= Ab ? t1 : Ab;  // T[tb+s]
          const double cand = __dadd_rn(Tj, ca);  // step s: source tb+s-1
          const bool tk = kval(s) && cand <= acc;
          acc = tk ? cand : acc;
          kb = tk ? lane + 2 - s : kb;
          const double cand2 = __dadd_rn(Ts, cb);  // step s+1: source tb+s
          const bool tk2 = kval(s + 1) && cand2 <= acc;
          acc = tk2 ? cand2 : acc;
          kb = tk2 ? lane + 1 - s : kb;
#if SCLS_DP_PUSH
          {
            const double naN = kvN(s + 2) ? __ldg(cpN - s - 2) : 0.0;
            const double nbN = kvN(s + 3) ? __ldg(cpN - s - 3) : 0.0;
            const double d1 = __dadd_rn(Tj, caN);
            const bool u1 = kvN(s) && d1 <= accN;
            accN = u1 ? d1 : accN;
            kbN = u1 ? 34 + lane - s : kbN;
            const double d2 = __dadd_rn(Ts, cbN);
            const bool u2 = kvN(s + 1) && d2 <= accN;
            accN = u2 ? d2 : accN;
            kbN = u2 ? 33 + lane - s : kbN;
            caN = naN;
            cbN = nbN;
          }
#endif
          Tj = shfl_d(acc, s);  // T[tb+s+1]: lane s is final after step s+1
          Ab = shfl_d(acc, s + 1);
          c1b = shfl_d(c1own, s + 1);
          ca = na;
          cb = nb;
        }
        if (s == rows) {  // a last single step
          const double cand = __dadd_rn(Tj, ca);
          const bool tk = kval(s) && cand <= acc;
          acc = tk ? cand : acc;
          kb = tk ? lane + 2 - s : kb;
        }
#if SCLS_DP_PUSH
        if (rows == 32) {  // then s == 32: sources tb+31 (Tj) and tb+32 (lane 31's final acc)
          const double d1 = __dadd_rn(Tj, caN);
          const bool u1 = kvN(32) && d1 <= accN;
          accN = u1 ? d1 : accN;
          kbN = u1 ? 2 + lane : kbN;
          const double Tl = shfl_d(acc, 31);
          const double d2 = __dadd_rn(Tl, cbN);
          const bool u2 = kvN(33) && d2 <= accN;
          accN = u2 ? d2 : accN;
          kbN = u2 ? 1 + lane : kbN;
        }
#endif
#else
        const double* __restrict__ cp = crow + lane;       // c(L_r, lane + 2 - s) = cp[2 - s]
        double c1 = 0.0;                                   // step s (never valid at s = 1)
        double c2 = kval(2) ? __ldg(cp) : 0.0;             // step s + 1
        for (int s = 1; s <= rows; ++s) {
          const double c0 = c1;
          c1 = c2;
          c2 = kval(s + 2) ? __ldg(cp - s) : 0.0;  // k = lane + 2 - (s + 2)
#if SCLS_DP_SELECT_ACCEPT
          const double cand = __dadd_rn(Tj, c0);
          const bool tk = kval(s) && cand <= acc;
          acc = tk ? cand : acc;
          kb = tk ? lane + 2 - s : kb;
#else
          if (kval(s)) {
            const double cand = __dadd_rn(Tj, c0);
            if (cand <= acc) {
              acc = cand;
              kb = lane + 2 - s;
            }
          }
#endif
          Tj = shfl_d(acc, s - 1);
        }
#endif
        if (valid) {
          T[r] = acc;
          split[r] = r - kb;
        }
        __syncwarp();
      }
      SIM_PROF(5);
      // 4. backtrack (batcher.cpp:69-73): segment ends, reversed
      int cnt = 0;
      for (int i = P_; i > 0; i = split[i]) {
        if (lane == 0) segs[cnt] = i;
        ++cnt;
      }
      __syncwarp();
      nb = cnt;
      // 5. emit batches in ascending segment order (batcher.cpp:75-86)
      for (int b0 = 0; b0 < nb; b0 += 32) {
        const int b = b0 + lane;
        if (b < nb) {
          const int end = segs[nb - 1 - b];
          const int beg = b == 0 ? 0 : segs[nb - b];
          const int bi = (int)next_batch + b;
          const int L = sv[end - 1];
          brec[bi].est = cost[coff[L] - 1 + (end - beg)];
          // slice_served_l_out (sched_policies.cpp:72-80): max over members
          int served = 0;
#pragma unroll kEmitU
          for (int q = tl_pos + beg; q < tl_pos + end; ++q) {
            const int4 v = tlog[q].igte;
            served = max(served, min(v.z - v.y, C.S));
          }
          brec[bi].d = make_int4(tl_pos + beg, end - beg, L, served);
        }
      }
      tl_pos += P_;
      pool_len = 0;
      __syncwarp();
    }
    SIM_PROF(6);
    const int first = (int)next_batch;
    next_batch += nb;
    // 6. offload (offloader.cpp:25-54): stable est-descending order, then the
    //    greedy min-(load, worker) placement against the lane loads.
    int32_t* order = segs;  // reuse
    if (nb > 0) {
      if (nb <= 32) {
        const double e = lane < nb ? brec[first + lane].est : -dinf();
        int rank = 0;
        for (int q = 0; q < nb; ++q) {
          const double eq = shfl_d(e, q);
          rank += (eq > e) || (eq == e && q < lane);
        }
        if (lane < nb) order[rank] = lane;
      } else {
        for (int i = lane; i < nb; i += 32) {
          sk[i] = ~ordered_bits(brec[first + i].est);
          sv[i] = i;
        }
        __syncwarp();
        const bool sw = warp_radix_sort(nb, sk, sv, sk2, (int32_t*)Tg, 64, lane, bins);
        const int32_t* ord = sw ? (const int32_t*)Tg : sv;
        for (int i = lane; i < nb; i += 32) order[i] = ord[i];
      }
      __syncwarp();
    }
    for (int k = 0; k < nb; ++k) {
      const int b = first + order[k];
      const double e = brec[b].est;
      const int w = argmin_worker_load<V>(ws, W, lane);  // min (load, worker id)
      if (MINE(w)) WK(w).load = __dadd_rn(WK(w).load, e);
      // dispatch record (served l_out computed at emit), enqueue
      const int4 d = brec[b].d;
      const int bn = d.y;
      sink.record(lane, 2, clock, -1, w, b, bn, d.z, C.S, 0, e, 0, 0, 0.0, 0, 0.0, 0);
      if (lane == 0) brec[b].next = -1;
      const int tail = shfl_i(WK(w).q_tail, WL(w));
      if (lane == 0 && tail >= 0) brec[tail].next = b;
      if (MINE(w)) {
        WorkerState& k = WK(w);
        if (k.q_tail < 0) k.q_head = b;
        k.q_tail = b;
      }
      __syncwarp();
      start_next_scls(w);
    }
    SIM_PROF(7);
    // the tick's scratch is dead until the next tick rewrites it: the pool
    // records it consumed, the sort keys, rows, T / split and segments
    if (P_ > 0) {
      const int m = max(P_, nb);
      l2_discard(prec, prec + n_rec, lane);
      l2_discard(pool, pool + n_rec, lane);
      l2_discard(p_eff, p_eff + n_rec, lane);
      l2_discard(sk, sk + m, lane);
      l2_discard(sk2, sk2 + m, lane);
      l2_discard(sv, sv + m + 1, lane);
      l2_discard(Tg, Tg + m + 1, lane);
      l2_discard(split_g, split_g + m + 1, lane);
      l2_discard(segs, segs + nb + 1, lane);
    }
    // sched_policies.cpp:134-146: adaptive interval from the post-offload loads
    const double ml = min_worker_load<V>(ws, W, lane);
    const double a = __dmul_rn(C.lambda, ml);
    const double interval = a < C.gamma ? C.gamma : a;
    sink.record(lane, 1, clock, -1, -1, -1, nb, 0, 0, 0, 0.0, 0, 0, 0.0, 0, interval, 0);
    tick_t = __dadd_rn(clock, interval);
    tick_s = next_seq++;
    return SCLS_OK;
  };

  // SCLS on_batch_done (sched_policies.cpp:149-188) for worker w, batch b.
  auto scls_done = [&](int w, int b) {
    const int4 d = brec[b].d;
    const int bn = d.y, bst = d.x, lin = d.z, served = d.w;
    const double best = brec[b].est;
    sink.record(lane, 4, clock, -1, w, b, bn, lin, C.S, served, 0.0, 0, 0, 0.0, 0, 0.0, bn);
    ++batch_count;
    batch_members += bn;
    early += served < C.S;
    const unsigned lt = (1u << lane) - 1u;
    int nfin = 0;
    int32_t* fin = sv;  // finished members' slots, member order (reused scratch)
    // One chunk (bn <= 32, the common case): the completions come straight
    // from the member registers, still after this chunk's member records.
    const bool one = bn <= 32;
    for (int b0 = 0; b0 < bn; b0 += 32) {
      const int i = b0 + lane;
      const bool ok = i < bn;
      int id = 0, eff = 0, g = 0, pad = 0, inv = 0, s1 = 0;
      double ta = 0.0;
      bool done = false;
      int ng = 0, tgv = 0;
      if (ok) {
        const int q = bst + i;
        const int4 v = tlog[q].igte;
        id = v.x;
        const int gsf = v.y;
        tgv = v.z;
        eff = v.w;
        s1 = tlog[q].s + 1;
        ta = tlog[q].a;
        g = min(tgv - gsf, served);
        pad = lin - eff;
        inv = served - g;
        ng = gsf + g;
        done = ng >= tgv || ng >= C.G;
      }
      const int cnt = min(32, bn - b0);
      sink.members(lane, cnt, id, eff, pad, g, inv);
      total_pad += __reduce_add_sync(FULL, ok ? pad : 0);
      total_inv += __reduce_add_sync(FULL, ok ? inv : 0);
      const unsigned fm = __ballot_sync(FULL, ok && done);
      const unsigned pm = __ballot_sync(FULL, ok && !done);
      if (ok && !done) {  // repooled in member order with its record (sched_policies.cpp:176-181)
        const int d = pool_len + __popc(pm & lt);
        pool[d] = id;
        p_eff[d] = eff + g;
        prec[d].gts = make_int4(ng, tgv, s1, 0);
        prec[d].a = ta;
      }
      pool_len += __popc(pm);
      if (one) {
        const int cnt = __popc(fm);
        const int pos = __popc(fm & lt);
        const double r = clock - ta;
        if (ok && done) {
          resp[completed + pos] = r;
          if (hist && s1 < P.hist_bins) atomicAdd((unsigned long long*)&hist[s1], 1ull);
        }
        if (kHash || kLog)
          for (unsigned m = fm; m; m &= m - 1) {
            const int src = __ffs(m) - 1;
            sink.record(lane, 5, clock, shfl_i(id, src), w, -1, 0, 0, 0, 0, 0.0, 0, 0, shfl_d(r, src),
                        shfl_i(s1, src), 0.0, 0);
          }
        else
          sink.n_events += cnt;
        completed += cnt;
        if (cnt > 0) last_completion = clock;
        break;
      }
      if (ok && done) fin[nfin + __popc(fm & lt)] = bst + i;
      nfin += __popc(fm);
    }
    __syncwarp();
    for (int c0 = 0; c0 < nfin; c0 += 32) {  // completions from the slot state
      const int cnt = min(32, nfin - c0);
      const int q = lane < cnt ? fin[c0 + lane] : 0;
      const int id = lane < cnt ? tlog[q].igte.x : 0;
      const double r = lane < cnt ? clock - tlog[q].a : 0.0;
      const int s = lane < cnt ? tlog[q].s + 1 : 0;
      if (lane < cnt) {
        resp[completed + lane] = r;
        if (hist && s < P.hist_bins) atomicAdd((unsigned long long*)&hist[s], 1ull);
      }
      for (int i = 0; i < cnt; ++i)
        sink.record(lane, 5, clock, shfl_i(id, i), w, -1, 0, 0, 0, 0, 0.0, 0, 0, shfl_d(r, i), shfl_i(s, i), 0.0, 0);
      completed += cnt;
      if (cnt > 0) last_completion = clock;
    }
    if (MINE(w)) {
      WorkerState& k = WK(w);
      k.last_end = fmax(k.last_end, clock);
      k.load = k.load - best;  // offloader.cpp:56-59 complete_batch
      if (k.load < 0.0) k.load = 0.0;
    }
    // this batch's tick-log entries are consumed (the log is append-only)
    __syncwarp();
    l2_discard(tlog + bst, tlog + bst + bn, lane);
  };

  // SLS on_batch_done (sched_policies.cpp:245-273).
  auto sls_done = [&](int w) {
    const int start = shfl_i(WK(w).inf_start, WL(w)), bn = shfl_i(WK(w).inf_n, WL(w)),
              lin = shfl_i(WK(w).inf_lin, WL(w)), lout = shfl_i(WK(w).inf_lout, WL(w));
    const long long bid = shfl_l(WK(w).inf_id, WL(w));
    sink.record(lane, 4, clock, -1, w, bid, bn, lin, lout, lout, 0.0, 0, 0, 0.0, 0, 0.0, bn);
    ++batch_count;
    batch_members += bn;
    const int32_t* q = fifo_base + (int64_t)w * cap_w;
    for (int b0 = 0; b0 < bn; b0 += 32) {
      const int i = b0 + lane;
      const bool ok = i < bn;
      int id = 0, g = 0, pad = 0, inv = 0, orig = 0;
      if (ok) {
        id = q[start + i];
        orig = inp[id];
        g = min(tg[id], C.G);
        pad = lin - orig;
        inv = lout - g;
        gen[id] = g;
        sl[id] = 1;
      }
      const int cnt = min(32, bn - b0);
      sink.members(lane, cnt, id, orig, pad, g, inv);
      total_pad += __reduce_add_sync(FULL, ok ? pad : 0);
      total_inv += __reduce_add_sync(FULL, ok ? inv : 0);
    }
    __syncwarp();
    for (int c0 = 0; c0 < bn; c0 += 32) {
      const int cnt = min(32, bn - c0);
      const int id = lane < cnt ? q[start + c0 + lane] : 0;
      complete_chunk(cnt, id, w);
    }
    if (MINE(w)) {
      WorkerState& k = WK(w);
      k.last_end = fmax(k.last_end, clock);
      k.busy = 0;
    }
    sls_try_dispatch(w);
  };

  // ILS iteration boundary (sched_policies.cpp:292-391) for instance w.
  // Running requests live in per-instance slots {id, join_iter, lim, inp}
  // with lim = min(true_gen, max_gen_limit): a request's generated count is
  // it_cnt - join_iter, and it exits at the first boundary where that
  // reaches lim.  next_exit = min(join_iter + lim) and mctx (max effective
  // input over running) are kept per instance, so an iteration that neither
  // retires nor admits anyone (the common case) is O(1) and touches no memory.
  auto ils_event = [&](int w) {
    const unsigned lt = (1u << lane) - 1u;
    const double now = clock;
    int4* run = (int4*)run_base + (int64_t)w * C.MC;
    const int32_t* wq = fifo_base + (int64_t)w * cap_w;
    const int wl = WL(w);
    const int nr = shfl_i(WK(w).n_run, wl);
    const int it1 = shfl_i(WK(w).it_cnt, wl) + (nr > 0 ? 1 : 0);
    const int head = shfl_i(WK(w).f_head, wl), tail = shfl_i(WK(w).f_tail, wl);
    const bool exit_possible = nr > 0 && it1 >= shfl_i(WK(w).next_exit, wl);
    const bool join_possible = tail > head && (nr < C.MC || exit_possible);
    if (nr > 0 && !exit_possible && !join_possible) {  // unchanged iteration
      if (lane == wl) {
        WorkerState& k = WK(w);
        k.it_cnt = it1;
        k.seg_it += 1;
        k.mctx += 1;
        k.ev_t = __dadd_rn(now, decode_step_time(lat, k.mctx, nr));
        k.ev_s = next_seq;
      }
      ++next_seq;
      return;
    }
    if (nr > 0 && lane == wl) {
      WK(w).it_cnt = it1;
      WK(w).seg_it += 1;
    }
    // retire: survivors compacted in order, exits in member order
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
      if (ok && ex) ex_base[nexit + __popc(em & lt)] = v.x;
      if (ok && !ex) run[keep + __popc(km & lt)] = v;
      nexit += __popc(em);
      keep += __popc(km);
      __syncwarp();
    }
    // admit FCFS up to max_concurrent
    const int njoin = min(C.MC - keep, tail - head);
    for (int j = lane; j < njoin; j += 32) {
      const int id = wq[head + j];
      run[keep + j] = make_int4(id, it1, min(tg[id], C.G), inp[id]);
    }
    __syncwarp();
    const int nr_new = keep + njoin;
    if (lane == wl) {
      WK(w).f_head = head + njoin;
      WK(w).n_run = nr_new;
    }
    const bool changed = nexit > 0 || njoin > 0;
    const long long sid = shfl_l(WK(w).seg_id, wl);
    const int sit = shfl_i(WK(w).seg_it, wl);
    if (changed && sid >= 0 && sit > 0) {
      const int sn = shfl_i(WK(w).seg_n, wl), slin = shfl_i(WK(w).seg_lin, wl);
      sink.record(lane, 4, now, -1, w, sid, sn, slin, sit, sit, 0.0, 0, 0, 0.0, 0, 0.0, 0);
      ++batch_count;
      batch_members += sn;
      if (lane == wl) {
        WK(w).seg_id = -1;
        WK(w).last_end = fmax(WK(w).last_end, now);
      }
    }
    for (int c0 = 0; c0 < nexit; c0 += 32) {
      const int cnt = min(32, nexit - c0);
      const int id = lane < cnt ? ex_base[c0 + lane] : 0;
      __syncwarp();
      complete_chunk(cnt, id, w);
    }
    if (nr_new == 0) {
      if (lane == wl) WK(w).boundary = 0;
      return;
    }
    int mc = 0, nx = 0x7fffffff;
    for (int i = lane; i < nr_new; i += 32) {
      const int4 v = run[i];
      mc = max(mc, v.w + (it1 - v.y));
      nx = min(nx, v.y + v.z);
    }
    mc = __reduce_max_sync(FULL, mc);
    nx = __reduce_min_sync(FULL, nx);
    long long cur_seg = sid;
    if (changed) {
      cur_seg = next_batch++;
      if (lane == wl) {
        WorkerState& k = WK(w);
        k.seg_id = cur_seg;
        k.seg_n = nr_new;
        k.seg_lin = mc;
        k.seg_it = 0;
      }
      sink.record(lane, 3, now, -1, w, cur_seg, nr_new, mc, 0, 0, 0.0, 0, 0, 0.0, 0, 0.0, 0);
    }
    double it = decode_step_time(lat, mc, nr_new);
    for (int j = 0; j < njoin; ++j) {
      const int4 v = run[keep + j];
      if (lane == 0) sl[v.x] = 1;
      it = __dadd_rn(it, prefill_time(lat, 1, v.w));
      // planned_l_out = remaining_gen() = true_gen (nothing generated yet), sched_policies.cpp:384
      sink.record(lane, 2, now, v.x, w, cur_seg, 1, v.w, tg[v.x], 0, 0.0, 0, 0, 0.0, 0, 0.0, 0);
    }
    if (lane == wl) {
      WorkerState& k = WK(w);
      k.mctx = mc;
      k.next_exit = nx;
      k.ev_t = __dadd_rn(now, it);
      k.ev_s = next_seq;
      k.boundary = 1;
    }
    ++next_seq;
  };

  // ---- the event loop (sim_engine.cpp:123-166) ------------------------------------
  bool dirty = true;
  double next_arr = n > 0 ? arr[0] : dinf();
  double na_t = dinf();
  unsigned long long na_s = ~0ull;
  int na_w = -1;  // -1: tick / FIFO head, >= 0: lane slot
  while (completed < n) {
    if (POL == SCLS_POLICY_ILS && V == 1) {
      WorkerState& k = ws[0];
      // Fast lane: consecutive boundary events of instances whose iteration
      // neither retires nor admits anyone (see ils_event) — the bulk of an
      // ILS run.  Same (time, seq) order, same arithmetic as ils_event's
      // unchanged branch; anything else falls through to the general path.
      // Each lane keeps the order-preserving key of its pending event and a
      // "next boundary is unchanged" flag; only the winner's lane changes
      // per step, the winner's time is rebuilt from the reduced key, and any
      // exact time tie is left to the general path (which orders by seq).
      const bool has = lane < W && k.ev_t != dinf();
      uint64_t key = has ? ordered_bits(k.ev_t) : ~0ull;
      bool mine_fast = has && k.n_run > 0 && k.it_cnt + 1 < k.next_exit && !(k.f_tail > k.f_head && k.n_run < C.MC);
      // decode_step_time(mctx, n) = ((d1*n)*l + d2*n) + d3*l + d4: the n terms are fixed in a run
      const double dn = (double)k.n_run;
      const double a1 = __dmul_rn(lat.d1, dn), a2 = __dmul_rn(lat.d2, dn);
      for (;;) {
        const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
        const unsigned mh = __reduce_min_sync(FULL, hi);
        const unsigned ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xffffffffu);
        const unsigned tie = __ballot_sync(FULL, hi == mh && lo == ml);
        if (tie & (tie - 1u)) break;  // equal times: the general path orders by seq
        const int w = __ffs(tie) - 1;
        const uint64_t kmin = ((uint64_t)mh << 32) | ml;
        if (kmin == ~0ull) break;
        const double bt = __longlong_as_double(
            (long long)((kmin & 0x8000000000000000ull) ? (kmin & ~0x8000000000000000ull) : ~kmin));
        if (next_arr <= fmin(bt, C.horizon) || C.horizon <= bt) break;
        if (!((__ballot_sync(FULL, mine_fast) >> w) & 1u)) break;
        clock = bt;
        if (lane == w) {
          k.it_cnt += 1;
          k.seg_it += 1;
          k.mctx += 1;
          const double dl = (double)k.mctx;
          const double it = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a1, dl), a2), __dmul_rn(lat.d3, dl)), lat.d4);
          k.ev_t = __dadd_rn(bt, it);
          k.ev_s = next_seq;
          key = ordered_bits(k.ev_t);
          mine_fast = k.it_cnt + 1 < k.next_exit;
        }
        ++next_seq;
      }
      dirty = true;
    }
    if (dirty) {
      double bt;
      unsigned long long bs;
      const int bw = argmin_worker_event<V>(ws, W, lane, &bt, &bs);
      na_t = bt;
      na_s = bs;
      na_w = bw;
      if (POL == SCLS_POLICY_SCLS) {
        if (tick_t < na_t || (tick_t == na_t && tick_s < na_s)) {
          na_t = tick_t;
          na_s = tick_s;
          na_w = -1;
        }
      } else if (POL == SCLS_POLICY_SLS && pf_head < pf_tail) {
        const double ft = pf_t[pf_head];
        const unsigned long long fs = pf_seq[pf_head];
        if (ft < na_t || (ft == na_t && fs < na_s)) {
          na_t = ft;
          na_s = fs;
          na_w = -1;
        }
      }
      dirty = false;
    }
    SIM_PROF(0);
    const double bound = fmin(na_t, C.horizon);
    if (next_arr <= bound) {  // next_arr = arr[cur], +INF once all arrived
      // Arrival(s): seq < n, so they precede any non-arrival event at the same time.
      if (POL == SCLS_POLICY_SCLS) {
        // SCLS arrivals only append to the pool: take every arrival <= bound.
        int cnt = 0;
        for (;;) {
          const int i = cur + cnt + lane;
          const bool ok = i < n && arr[i] <= bound;
          const unsigned m = __ballot_sync(FULL, ok);
          const int run = (~m) ? __ffs(~m) - 1 : 32;
          cnt += run;
          if (run < 32) break;
        }
        if (first_arrival == dinf()) first_arrival = arr[cur];

        if (kHash || kLog) {
          for (int i = 0; i < cnt; ++i) {
            const int id = cur + i;
            sink.record(lane, 0, arr[id], id, -1, -1, 0, 0, 0, 0, 0.0, inp[id], tg[id], 0.0, 0, 0.0, 0);
          }
        } else {
          sink.n_events += cnt;
        }
        clock = arr[cur + cnt - 1];
        cur += cnt;  // pooled as the id range [arr_lo, cur) until the next tick
        next_arr = cur < n ? arr[cur] : dinf();
        __syncwarp();
        SIM_PROF(1);
        continue;
      }
      const int id = cur++;
      next_arr = cur < n ? arr[cur] : dinf();
      clock = arr[id];
      if (first_arrival == dinf()) first_arrival = clock;
      sink.record(lane, 0, clock, id, -1, -1, 0, 0, 0, 0, 0.0, inp[id], tg[id], 0.0, 0, 0.0, 0);
      const int w = rr;
      rr = rr + 1 == W ? 0 : rr + 1;
      if (POL == SCLS_POLICY_SLS) {  // sched_policies.cpp:194-201
        if (MINE(w)) fifo_base[(int64_t)w * cap_w + WK(w).f_tail++] = id;
        if (lane == 0) {
          pf_t[pf_tail] = clock;
          pf_seq[pf_tail] = next_seq;
          pf_w[pf_tail] = w;
        }
        ++pf_tail;
        ++next_seq;
        dirty = dirty || pf_tail - pf_head == 1;
      } else {  // ILS, sched_policies.cpp:279-290
        if (MINE(w)) fifo_base[(int64_t)w * cap_w + WK(w).f_tail++] = id;
        const int wake = shfl_i(WK(w).n_run == 0 && !WK(w).boundary, WL(w));
        if (wake) {
          if (MINE(w)) {
            WorkerState& k = WK(w);
            k.ev_t = clock;
            k.ev_s = next_seq;
            k.boundary = 1;
          }
          ++next_seq;
          dirty = true;
        }
      }
      __syncwarp();
      continue;
    }
    if (C.horizon <= na_t) {  // EndOfRun (horizon, n) precedes (na_t, na_s > n)
      status = SCLS_ERR_NON_TERMINATION;
      break;
    }
    clock = na_t;
    dirty = true;
    if (na_w < 0) {
      if (POL == SCLS_POLICY_SCLS) {
        tick_t = dinf();
        tick_s = ~0ull;
        SIM_PROF(8);
        status = scls_tick();
        SIM_PROF(9);
        if (status != SCLS_OK) break;
      } else {  // SLS deferred dispatch check
        const int w = pf_w[pf_head];
        ++pf_head;
        sls_try_dispatch(w);
      }
    } else {
      const int w = na_w;
      if (MINE(w)) {
        WK(w).ev_t = dinf();
        WK(w).ev_s = ~0ull;
      }
      if (POL == SCLS_POLICY_SCLS) {
        const int b = shfl_i(WK(w).infl, WL(w));
        if (MINE(w)) {
          WK(w).busy = 0;
          WK(w).infl = -1;
        }
        SIM_PROF(8);
        scls_done(w, b);
        start_next_scls(w);
        SIM_PROF(10);
      } else if (POL == SCLS_POLICY_SLS) {
        sls_done(w);
      } else {
        ils_event(w);
      }
    }
    __syncwarp();
  }

  SIM_PROF(8);
#ifdef SCLS_SIM_PROF
  if (POL == SCLS_POLICY_SCLS && hist && P.hist_bins >= 16 && lane == 0)
    for (int i = 0; i < 12; ++i) hist[4 + i] = prof[i];
#endif
  // ---- report (metrics.cpp:30-117) ------------------------------------------------------
  if (status == SCLS_OK && (sink.n_events == 0 || completed == 0)) status = SCLS_ERR_EMPTY_LOG;
  double thr = 0.0, avg = 0.0, p95 = 0.0, ctstd = 0.0;
  if (status == SCLS_OK) {
    const double span = last_completion - first_arrival;
    const double comp = (double)completed;
    thr = span > 0.0 ? __ddiv_rn(comp, span) : 0.0;
    // mean in completion order (metrics.cpp:83-85).  SCLS keeps this lane-0
    // loop and the serial digit scan below: resp_stats() here measured 33.5
    // -> 35.8 ms (inlined) / 36.4 ms (out of line) for the SCLS launch -- code
    // layout and register allocation of the event loop, not this once-per-trace work.
    double sum = 0.0;
    if (lane == 0)
      for (int i = 0; i < completed; ++i) sum = __dadd_rn(sum, resp[i]);
    sum = shfl_d(sum, 0);
    avg = __ddiv_rn(sum, comp);
    // nearest-rank p95 (metrics.cpp:87-91): radix select of the rank-th smallest
    const size_t rk = (size_t)ceil(__dmul_rn(0.95, comp));
    int want = (int)(rk > 1 ? rk : 1) - 1;
    uint64_t prefix = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = lane; i < 256; i += 32) bins[i] = 0;
      __syncwarp();
      const uint64_t hi_mask = shift == 56 ? 0ull : (~0ull << (shift + 8));
      for (int i = lane; i < completed; i += 32) {
        const uint64_t k = ordered_bits(resp[i]);
        if ((k & hi_mask) == prefix) atomicAdd(&bins[(k >> shift) & 0xff], 1);
      }
      __syncwarp();
      int digit = 0;
      if (lane == 0) {
        int acc = 0;
        for (int d = 0; d < 256; ++d) {
          if (acc + bins[d] > want) {
            digit = d;
            break;
          }
          acc += bins[d];
        }
        want -= acc;
      }
      digit = shfl_i(digit, 0);
      want = shfl_i(want, 0);
      prefix |= (uint64_t)digit << shift;
      __syncwarp();
    }
    {
      const uint64_t u = (prefix & 0x8000000000000000ull) ? (prefix & ~0x8000000000000000ull) : ~prefix;
      p95 = __longlong_as_double((long long)u);
    }
    // population std of per-worker last batch end (metrics.cpp:93-101)
    double mean = 0.0, var = 0.0;
    for (int w = 0; w < W; ++w) mean = __dadd_rn(mean, shfl_d(WK(w).last_end, WL(w)));
    mean = __ddiv_rn(mean, (double)W);
    for (int w = 0; w < W; ++w) {
      const double d = __dadd_rn(shfl_d(WK(w).last_end, WL(w)), -mean);
      var = __dadd_rn(var, __dmul_rn(d, d));
    }
    var = __ddiv_rn(var, (double)W);
    ctstd = __dsqrt_rn(var);
  }
  if (status != SCLS_OK && hist)  // no report => no slice histogram either
    for (int i = lane; i < P.hist_bins; i += 32) hist[i] = 0;
  if (lane == 0 && status != SCLS_OK) {
    // A failed run has no report (the reference throws, metrics.cpp is never
    // reached): only the status and the offending request are defined.
    memset(R, 0, sizeof *R);
    R->status = status;
    R->worker_count = W;
    R->error_request_id = status == SCLS_ERR_INFEASIBLE_REQUEST ? err_req : -1;
    R->n_requests = n;
    if (logging) {
      P.rec_count[t] = sink.rec_n;
      P.mem_count[t] = sink.mem_n;
    }
  } else if (lane == 0) {
    R->status = status;
    R->worker_count = W;
    R->error_request_id = -1;
    R->n_requests = n;
    R->completed = completed;
    const double comp = (double)completed;
    R->throughput = thr;
    R->avg_response_s = avg;
    R->p95_response_s = p95;
    R->ct_std_s = ctstd;
    R->avg_pad_tokens = status == SCLS_OK ? __ddiv_rn((double)total_pad, comp) : 0.0;
    R->avg_invalid_tokens = status == SCLS_OK ? __ddiv_rn((double)total_inv, comp) : 0.0;
    R->avg_batch_size = status == SCLS_OK && batch_count > 0
                            ? __ddiv_rn((double)batch_members, (double)batch_count) : 0.0;
    R->early_return_ratio = status == SCLS_OK && batch_count > 0
                                ? __ddiv_rn((double)early, (double)batch_count) : 0.0;
    R->total_pad = total_pad;
    R->total_invalid = total_inv;
    R->batch_count = batch_count;
    R->batch_members = batch_members;
    R->early_returns = early;
    R->n_events = sink.n_events;
    R->n_dispatches = sink.n_disp;
    R->n_ticks = sink.n_ticks;
    R->h_complete_ids = kHash ? sink.hc : 0;
    R->h_dispatch = kHash ? sink.hd : 0;
    R->h_complete_t = kHash ? sink.ht : 0;
    R->h_log = kHash ? sink.hl : 0;
    R->sim_clock = clock;
    if (logging) {
      P.rec_count[t] = sink.rec_n;
      P.mem_count[t] = sink.mem_n;
    }
  }
#undef WK
#undef WL
#undef MINE
}

template <int POL, bool kHash, bool kLog, int V = 1>
__global__ void __launch_bounds__(kSimWarps * 32, POL == SCLS_POLICY_SCLS ? SCLS_SIM_MINB : 8) sim_kernel(SimParams p, const int32_t* __restrict__ list,
                                                              int32_t count, const int32_t* __restrict__ dcount = nullptr) {
  if (dcount) count = *dcount;  // fallback launches: the job count lives on the device
  __shared__ int32_t bins[kSimWarps][256];
  __shared__ int32_t ssplit[POL == SCLS_POLICY_SCLS ? kSimWarps : 1][POL == SCLS_POLICY_SCLS ? kSplitSmem + 1 : 1];
  __shared__ double sT[POL == SCLS_POLICY_SCLS ? kSimWarps : 1][POL == SCLS_POLICY_SCLS ? kSplitSmem + 1 : 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;  // launches use 1 or kSimWarps warps per CTA
  if (g >= count) return;
  if (list[g] < 0) return;  // an empty slot (small launches: one job per CTA)
  run_trace<POL, kHash, kLog, V>(p, list[g], lane, bins[warp], ssplit[POL == SCLS_POLICY_SCLS ? warp : 0],
                              sT[POL == SCLS_POLICY_SCLS ? warp : 0]);
}

}  // namespace
}  // namespace scls

#include "sim_ils.cuh"
#include "sim_indep.cuh"

namespace scls {
namespace {

// Σ_i ceil(min(gen_i, G) / S): the exact number of (request, slice) pairs a
// SCLS run serves, i.e. the tick-log and batch capacity of the trace.
__global__ void slice_caps_kernel(int32_t n_traces, const int64_t* __restrict__ req_off,
                                  const int32_t* __restrict__ src, const int32_t* __restrict__ tg, const SimCfg* __restrict__ cfgs,
                                  const int32_t* __restrict__ cfg_index, int64_t* __restrict__ caps) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n_traces) return;
  const SimCfg c = cfgs[cfg_index ? cfg_index[warp] : 0];
  long long s = 0;
  if (c.policy == SCLS_POLICY_SCLS && c.S > 0)
    for (int64_t i = req_off[src ? src[warp] : warp] + lane; i < req_off[(src ? src[warp] : warp) + 1]; i += 32) {
      const int g = min(tg[i], c.G);
      s += g >= 1 ? (g + c.S - 1) / c.S : 1;  // lengths < 1 are refused by the kernel; keep the arena sane
    }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  if (lane == 0) caps[warp] = s;
}

__global__ void max_reduce_kernel(int64_t n, const int32_t* __restrict__ x, int32_t* __restrict__ out) {
  int m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, x[i]);
  m = __reduce_max_sync(FULL, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Per-config cost tables: K(L) = max_batch_size(L, S) and c(L, k) for
// k <= min(K(L), kcap) (cost_model.cpp:49-51, memory_model.cpp:72-90).
__global__ void k_table_kernel(int32_t Lmax, int32_t S, int32_t kcap, Mem mem, int32_t* __restrict__ Kt,
                               int32_t* __restrict__ need) {
  const int L = blockIdx.x * blockDim.x + threadIdx.x;
  if (L > Lmax) return;
  if (L == 0) {
    Kt[0] = 0;
    need[0] = 0;
    return;
  }
  const int K = would_oom(mem, 1, L, S) ? 0 : max_batch_size(mem, L, S);
  Kt[L] = K;
  need[L] = min(K, kcap);
}

__global__ void cost_fill_kernel(int32_t Lmax, int32_t S, Lat lat, const int32_t* __restrict__ need,
                                 const int32_t* __restrict__ off, int32_t base, double* __restrict__ cost) {
  for (int L = blockIdx.x; L <= Lmax; L += gridDim.x) {
    const int nk = need[L];
    const double sum_l = decode_sum_l(L, S);
    for (int k = threadIdx.x + 1; k <= nk; k += blockDim.x)
      cost[base + off[L] + k - 1] = __dadd_rn(prefill_time(lat, k, L), decode_time_from_sum(lat, k, sum_l, S));
  }
}

__global__ void coff_kernel(int32_t Lmax, const int32_t* __restrict__ off, int32_t base, int32_t* __restrict__ coff) {
  const int L = blockIdx.x * blockDim.x + threadIdx.x;
  if (L <= Lmax) coff[L] = base + off[L];
}

}  // namespace

static scls_status validate_cfg_host(const scls_sched_cfg& c) {
  if (!(c.lambda > 0.0 && c.lambda < 1.0)) return SCLS_ERR_ERROR;
  if (!(c.gamma > 0.0)) return SCLS_ERR_ERROR;
  if (c.slice_len < 1 || c.max_gen_limit < c.slice_len) return SCLS_ERR_ERROR;
  if (c.fixed_batch_size < 1 || c.max_concurrent < 1 || c.worker_count < 1) return SCLS_ERR_ERROR;
  if (c.policy < 0 || c.policy > 2) return SCLS_ERR_ERROR;
  if (!(c.horizon_s > 0.0)) return SCLS_ERR_ERROR;
  return SCLS_OK;
}

}  // namespace scls

using namespace scls;

extern "C" scls_status scls_validate_latency(const scls_latency* m);
extern "C" scls_status scls_validate_memory(const scls_memory* m);

// The simulator entry (shared by scls_simulate and scls_simulate_grid): job j
// runs source trace src[j] (identity when null) under config job_cfg[j].
// in_mem: where arrival/input_len/gen_len and req_offset live (SCLS_MEM_HOST,
// SCLS_MEM_DEVICE, or kMemDeviceArrays: arrays on the device, req_offset on
// the host); mem: where results / slice_hist / log live.
constexpr int32_t kMemDeviceArrays = 2;
static scls_status simulate_core(scls_ctx* ctx, int32_t n_src, const int64_t* req_offset, const double* arrival,
                                 const int32_t* input_len, const int32_t* gen_len, int32_t n_cfgs,
                                 const scls_sched_cfg* cfgs, int32_t n_traces, const std::vector<int32_t>& h_src,
                                 const std::vector<int32_t>& h_idx, const scls_latency* lat,
                                 const scls_memory* memm, scls_trace_result* results, int32_t hist_bins,
                                 int64_t* slice_hist, scls_event_log* log, int32_t mem, int32_t in_mem) {
  // n_traces counts jobs below; h_off / inputs are per source trace.
  const bool has_src = !h_src.empty();
  const bool cfg_index = !h_idx.empty();
  cudaStream_t s = ctx->stream;
  // Host-side copies of the small arguments.
  std::vector<int64_t> h_off(n_src + 1);
  if (in_mem == SCLS_MEM_DEVICE) {
    SCLS_CUDA(cudaMemcpy(h_off.data(), req_offset, sizeof(int64_t) * (n_src + 1), cudaMemcpyDeviceToHost));
  } else {
    std::memcpy(h_off.data(), req_offset, sizeof(int64_t) * (n_src + 1));
  }
  const int64_t total = h_off[n_src] - h_off[0];
  if (h_off[0] != 0 || total < 0) return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "req_offset must start at 0");
  int64_t nmax = 0;
  for (int t = 0; t < n_src; ++t) {
    const int64_t nt = h_off[t + 1] - h_off[t];
    if (nt < 0 || nt >= (1ll << 30)) return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad trace size");
    nmax = std::max(nmax, nt);
  }
  auto src_of = [&](int j) { return has_src ? h_src[j] : j; };
  // Configs: validate (Simulator::Simulator, sim_engine.cpp:32-35), limits.
  const bool model_ok = scls_validate_latency(lat) == SCLS_OK && scls_validate_memory(memm) == SCLS_OK;
  // dp_mono.cuh: non-negative coefficients + a valid memory model make every
  // tick's T non-decreasing, so the tick DP can decide rows in rounds
  const bool mono = model_ok && !std::signbit(lat->p1) && !std::signbit(lat->p2) && !std::signbit(lat->p3) &&
                    !std::signbit(lat->p4) && !std::signbit(lat->d1) && !std::signbit(lat->d2) &&
                    !std::signbit(lat->d3) && !std::signbit(lat->d4);
  std::vector<SimCfg> hc(n_cfgs);
  std::vector<uint8_t> hok(n_cfgs);
  int n_tables = 0;
  int32_t Gmax = 1;
  for (int c = 0; c < n_cfgs; ++c) {
    const scls_sched_cfg& x = cfgs[c];
    hok[c] = model_ok && validate_cfg_host(x) == SCLS_OK;
    hc[c] = SimCfg{x.policy, x.slice_len, x.max_gen_limit, x.fixed_batch_size, x.max_concurrent,
                   x.worker_count, x.lambda, x.gamma, x.horizon_s, -1, mono && ctx->dp_mode != 1};
    if (hok[c] && x.policy == SCLS_POLICY_SCLS) hc[c].table = n_tables++;
    if (hok[c]) Gmax = std::max(Gmax, x.max_gen_limit);
    if (hok[c] && x.policy == SCLS_POLICY_ILS) hc[c].MC = std::max(1, std::min<int32_t>(x.max_concurrent, (int32_t)nmax));
  }
  // Stage requests.
  const double* d_arr = arrival;
  const int32_t* d_inp = input_len;
  const int32_t* d_tg = gen_len;
  int64_t* d_off = (int64_t*)ctx->buf(kSlotSim + 0, sizeof(int64_t) * (n_src + 1));
  int32_t* d_src = has_src ? (int32_t*)ctx->buf(kSlotSim + 23, sizeof(int32_t) * n_traces) : nullptr;
  if (has_src && !d_src) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  SimCfg* d_cfg = (SimCfg*)ctx->buf(kSlotSim + 1, sizeof(SimCfg) * n_cfgs);
  uint8_t* d_ok = (uint8_t*)ctx->buf(kSlotSim + 2, n_cfgs);
  int32_t* d_idx = cfg_index ? (int32_t*)ctx->buf(kSlotSim + 3, sizeof(int32_t) * n_traces) : nullptr;
  if (!d_off || !d_cfg || !d_ok || (cfg_index && !d_idx)) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  SCLS_CUDA(cudaEventRecord(ctx->ev[0], s));
  if (in_mem == SCLS_MEM_HOST && total > 0) {
    double* a = (double*)ctx->buf(kSlotSim + 4, sizeof(double) * total);
    int32_t* b = (int32_t*)ctx->buf(kSlotSim + 5, sizeof(int32_t) * total);
    int32_t* g = (int32_t*)ctx->buf(kSlotSim + 6, sizeof(int32_t) * total);
    if (!a || !b || !g) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
    SCLS_CUDA(cudaMemcpyAsync(a, arrival, sizeof(double) * total, cudaMemcpyHostToDevice, s));
    SCLS_CUDA(cudaMemcpyAsync(b, input_len, sizeof(int32_t) * total, cudaMemcpyHostToDevice, s));
    SCLS_CUDA(cudaMemcpyAsync(g, gen_len, sizeof(int32_t) * total, cudaMemcpyHostToDevice, s));
    d_arr = a;
    d_inp = b;
    d_tg = g;
  }
  SCLS_CUDA(cudaMemcpyAsync(d_off, h_off.data(), sizeof(int64_t) * (n_src + 1), cudaMemcpyHostToDevice, s));
  if (d_src) SCLS_CUDA(cudaMemcpyAsync(d_src, h_src.data(), sizeof(int32_t) * n_traces, cudaMemcpyHostToDevice, s));
  SCLS_CUDA(cudaMemcpyAsync(d_cfg, hc.data(), sizeof(SimCfg) * n_cfgs, cudaMemcpyHostToDevice, s));
  SCLS_CUDA(cudaMemcpyAsync(d_ok, hok.data(), n_cfgs, cudaMemcpyHostToDevice, s));
  if (d_idx) SCLS_CUDA(cudaMemcpyAsync(d_idx, h_idx.data(), sizeof(int32_t) * n_traces, cudaMemcpyHostToDevice, s));
  // Max input length (for the L range of the cost tables), on device.
  int32_t in_max = 1;
  {
    int32_t* d_max = (int32_t*)ctx->buf(kSlotSim + 21, sizeof(int32_t));
    if (!d_max) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
    SCLS_CUDA(cudaMemsetAsync(d_max, 0, sizeof(int32_t), s));
    if (total > 0) {
      max_reduce_kernel<<<std::min(div_up(total, 256), ctx->sm_count * 8), 256, 0, s>>>(total, d_inp, d_max);
      SCLS_LAUNCHED();
    }
    SCLS_CUDA(cudaMemcpyAsync(&in_max, d_max, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  }
  int64_t* d_caps = (int64_t*)ctx->buf(kSlotSim + 7, sizeof(int64_t) * n_traces);
  if (!d_caps) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  slice_caps_kernel<<<div_up((int64_t)n_traces * 32, 256), 256, 0, s>>>(n_traces, d_off, d_src, d_tg, d_cfg, d_idx, d_caps);
  SCLS_LAUNCHED();
  std::vector<int64_t> caps(n_traces);
  SCLS_CUDA(cudaMemcpyAsync(caps.data(), d_caps, sizeof(int64_t) * n_traces, cudaMemcpyDeviceToHost, s));
  SCLS_CUDA(cudaStreamSynchronize(s));
  in_max = std::max(in_max, 1);
  // Cost tables (one per SCLS config): L in [0, Lmax], k <= min(K(L), nmax).
  const int32_t Lmax = (int32_t)std::min<int64_t>((int64_t)in_max + Gmax, 1 << 24);
  int32_t* d_Kt = nullptr;
  int32_t* d_coff = nullptr;
  double* d_cost = nullptr;
  if (n_tables > 0) {
    d_Kt = (int32_t*)ctx->buf(kSlotSim + 8, sizeof(int32_t) * (size_t)n_tables * (Lmax + 1));
    d_coff = (int32_t*)ctx->buf(kSlotSim + 9, sizeof(int32_t) * (size_t)n_tables * (Lmax + 1));
    int32_t* need = (int32_t*)ctx->buf(kSlotSim + 10, sizeof(int32_t) * (Lmax + 2));
    int32_t* off = (int32_t*)ctx->buf(kSlotSim + 11, sizeof(int32_t) * (Lmax + 2));
    if (!d_Kt || !d_coff || !need || !off) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
    const Mem dm = make_mem(*memm);
    std::vector<int32_t> totals(n_tables);
    int64_t grand = 0;
    for (int c = 0; c < n_cfgs; ++c) {
      if (hc[c].table < 0) continue;
      int32_t* Kt = d_Kt + (size_t)hc[c].table * (Lmax + 1);
      k_table_kernel<<<div_up(Lmax + 1, 256), 256, 0, s>>>(Lmax, hc[c].S, (int32_t)std::max<int64_t>(nmax, 1), dm, Kt, need);
      SCLS_LAUNCHED();
      scls_status st = scan_exclusive(ctx, Lmax + 1, need, off, off + Lmax + 1);
      if (st) return st;
      int32_t* d_kmax = (int32_t*)ctx->buf(kSlotSim + 29, sizeof(int32_t) * 2);
      if (!d_kmax) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
      SCLS_CUDA(cudaMemsetAsync(d_kmax, 0, sizeof(int32_t), s));
      max_reduce_kernel<<<std::min(div_up(Lmax + 1, 256), ctx->sm_count * 8), 256, 0, s>>>(Lmax + 1, need, d_kmax);
      SCLS_LAUNCHED();
      int32_t tot = 0, kmax = 0;
      SCLS_CUDA(cudaMemcpyAsync(&tot, off + Lmax + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      SCLS_CUDA(cudaMemcpyAsync(&kmax, d_kmax, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      SCLS_CUDA(cudaStreamSynchronize(s));
      // Tick DP variant: when every window fits one 32-row tile the in-tile
      // chain (two steps per broadcast, the next tile's far candidates on
      // it) beats the decision rounds -- in a contended sweep (C5: it issues
      // less) and, since round 2's paired / pushed chain, also for single
      // traces (C1 1.68 -> 1.61, C2 12.3 -> 11.4, C4 377 -> 354 ms);
      // SCLS_CHAIN_ALWAYS 0 keeps the rounds for launches with <= one job per SM.
      if (kmax <= 32 && ctx->dp_mode == 0) {
        int64_t jobs = 0;
        for (int t = 0; t < n_traces; ++t) jobs += (cfg_index ? h_idx[t] : 0) == c;
        if (jobs > ctx->sm_count || SCLS_CHAIN_ALWAYS) hc[c].mono = 0;
      }
      if (grand + tot > (1ll << 30)) return set_error(ctx, SCLS_ERR_CAPACITY, "simulator cost tables exceed 2^30 entries");
      totals[hc[c].table] = tot;
      // c(L, k) entries are written after the buffer is sized; remember the
      // per-table base via the coff table (base + off[L]).
      coff_kernel<<<div_up(Lmax + 1, 256), 256, 0, s>>>(Lmax, off, (int32_t)grand, d_coff + (size_t)hc[c].table * (Lmax + 1));
      SCLS_LAUNCHED();
      grand += tot;
    }
    // the tick-DP variant may have changed per config (above)
    SCLS_CUDA(cudaMemcpyAsync(d_cfg, hc.data(), sizeof(SimCfg) * n_cfgs, cudaMemcpyHostToDevice, s));
    d_cost = (double*)ctx->buf(kSlotSim + 12, sizeof(double) * (size_t)std::max<int64_t>(grand, 1));
    if (!d_cost) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
    const Lat dl = make_lat(*lat);
    int64_t base = 0;
    for (int c = 0; c < n_cfgs; ++c) {
      if (hc[c].table < 0) continue;
      // recompute need/off for this table (cheap) and fill its entries
      int32_t* Kt = d_Kt + (size_t)hc[c].table * (Lmax + 1);
      k_table_kernel<<<div_up(Lmax + 1, 256), 256, 0, s>>>(Lmax, hc[c].S, (int32_t)std::max<int64_t>(nmax, 1), dm, Kt, need);
      SCLS_LAUNCHED();
      scls_status st = scan_exclusive(ctx, Lmax + 1, need, off, nullptr);
      if (st) return st;
      cost_fill_kernel<<<std::min(Lmax + 1, ctx->sm_count * 8), 128, 0, s>>>(Lmax, hc[c].S, dl, need, off, (int32_t)base, d_cost);
      SCLS_LAUNCHED();
      base += totals[hc[c].table];
    }
  }
  // Per-trace arenas.
  std::vector<int64_t> tbase(n_traces + 1, 0);
  for (int t = 0; t < n_traces; ++t) {
    const SimCfg& c = hc[cfg_index ? h_idx[t] : 0];
    const int64_t nt = h_off[src_of(t) + 1] - h_off[src_of(t)];
    tbase[t + 1] = tbase[t] + sim_layout(nt, std::max(c.W, 1), c.policy, caps[t], std::max(c.MC, 1)).total;
  }
  int64_t* d_tbase = (int64_t*)ctx->buf(kSlotSim + 13, sizeof(int64_t) * (n_traces + 1));
  int64_t* d_tcap = (int64_t*)ctx->buf(kSlotSim + 14, sizeof(int64_t) * n_traces);
  char* arena = (char*)ctx->buf(kSlotSim + 15, (size_t)std::max<int64_t>(tbase[n_traces], 16));
  if (!d_tbase || !d_tcap || !arena) return set_error(ctx, SCLS_ERR_CUDA, "simulator arena allocation failed");
  SCLS_CUDA(cudaMemcpyAsync(d_tbase, tbase.data(), sizeof(int64_t) * (n_traces + 1), cudaMemcpyHostToDevice, s));
  SCLS_CUDA(cudaMemcpyAsync(d_tcap, caps.data(), sizeof(int64_t) * n_traces, cudaMemcpyHostToDevice, s));
  // Results / histogram / log buffers.
  scls_trace_result* d_res = results;
  int64_t* d_hist = slice_hist;
  if (mem == SCLS_MEM_HOST) {
    d_res = (scls_trace_result*)ctx->buf(kSlotSim + 16, sizeof(scls_trace_result) * n_traces);
    d_hist = hist_bins > 0 ? (int64_t*)ctx->buf(kSlotSim + 17, sizeof(int64_t) * (size_t)n_traces * hist_bins) : nullptr;
    if (!d_res || (hist_bins > 0 && !d_hist)) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  }
  SimParams p{};
  p.n_traces = n_traces;
  p.req_off = d_off;
  p.src = d_src;
  p.arr = d_arr;
  p.inp = d_inp;
  p.tg = d_tg;
  p.cfgs = d_cfg;
  p.cfg_index = d_idx;
  p.cfg_ok = d_ok;
  p.lat = make_lat(*lat);
  p.Lmax = Lmax;
  p.Kt = d_Kt;
  p.coff = d_coff;
  p.cost = d_cost;
  p.arena = arena;
  p.trace_base = d_tbase;
  p.trace_cap = d_tcap;
  p.res = d_res;
  p.hist_bins = hist_bins;
  p.hist = d_hist;
  const bool want_log = log && log->n_logged > 0;
  if (want_log) {
    const int64_t nl = std::min<int64_t>(log->n_logged, n_traces);
    p.n_logged = (int32_t)nl;
    p.rec_cap = log->rec_cap;
    p.mem_cap = log->mem_cap;
    if (mem == SCLS_MEM_HOST) {
      p.recs = (scls_event_record*)ctx->buf(kSlotSim + 18, sizeof(scls_event_record) * (size_t)nl * log->rec_cap);
      p.mems = (scls_member*)ctx->buf(kSlotSim + 19, sizeof(scls_member) * (size_t)std::max<int64_t>(nl * log->mem_cap, 1));
      int64_t* cnts = (int64_t*)ctx->buf(kSlotSim + 20, sizeof(int64_t) * 2 * nl);
      if (!p.recs || !p.mems || !cnts) return set_error(ctx, SCLS_ERR_CUDA, "log allocation failed");
      p.rec_count = cnts;
      p.mem_count = cnts + nl;
    } else {
      p.recs = log->records;
      p.mems = log->members;
      p.rec_count = log->rec_count;
      p.mem_count = log->mem_count;
    }
  }
  SCLS_CUDA(cudaEventRecord(ctx->ev[1], s));
  // One launch per policy over that policy's traces (compile-time policy
  // keeps each kernel lean); invalid configs ride along (status Error).
  // lists[3 + pol]: configs with more than 32 workers (the wide variant).
  std::vector<int32_t> lists[6];
  for (int t = 0; t < n_traces; ++t) {
    const SimCfg& c = hc[cfg_index ? h_idx[t] : 0];
    const int pol = c.policy;
    lists[((pol >= 0 && pol <= 2) ? pol : 0) + (c.W > 32 ? 3 : 0)].push_back(t);
  }
  // Longest jobs first (work ~ requests; SCLS: served slices): a launch that
  // needs more than one wave of warps starts its slowest jobs first and fills
  // the tail with short ones.  A launch with at most one job per SM (a single
  // trace, a small grid) gives every job a CTA of its own (the other warps of
  // the CTA get no job, -1), so no two jobs share an SM's L1.
  size_t n_slots = 0;
  for (auto& l : lists) {
    auto work = [&](int32_t t) {
      const SimCfg& c = hc[cfg_index ? h_idx[t] : 0];
      return c.policy == SCLS_POLICY_SCLS ? caps[t] : h_off[src_of(t) + 1] - h_off[src_of(t)];
    };
    std::stable_sort(l.begin(), l.end(), [&](int32_t a, int32_t b) { return work(a) > work(b); });
    if (l.size() > 1 && l.size() <= (size_t)ctx->sm_count) {
      std::vector<int32_t> spread;
      spread.reserve(l.size() * kSimWarps);
      for (int32_t t : l) {
        spread.push_back(t);
        for (int w = 1; w < kSimWarps; ++w) spread.push_back(-1);
      }
      l.swap(spread);
    }
    n_slots += l.size();
  }
  int32_t* d_lists = (int32_t*)ctx->buf(kSlotSim + 22, sizeof(int32_t) * (n_slots + 3));
  if (!d_lists) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  {
    std::vector<int32_t> flat;
    flat.reserve(n_slots);
    for (auto& l : lists) flat.insert(flat.end(), l.begin(), l.end());
    SCLS_CUDA(cudaMemcpyAsync(d_lists, flat.data(), sizeof(int32_t) * n_slots, cudaMemcpyHostToDevice, s));
  }
  const bool hash = ctx->sim_digests;
  // Packs for the independent-lane ILS kernel (sim_indep.cuh): up to
  // min(kIlsPackMax = 2, 32 / W, kPackSlots / (W * MC)) jobs of one config
  // per warp, packs in
  // LPT order of their longest job; one pack per CTA for small launches.
  auto make_packs = [&](const std::vector<int32_t>& l, bool ils, std::vector<int32_t>& off,
                        std::vector<int32_t>& flat) {
    std::vector<std::vector<int32_t>> packs, open(n_cfgs);
    auto work = [&](int32_t t) { return h_off[src_of(t) + 1] - h_off[src_of(t)]; };
    for (int32_t t : l) {
      if (t < 0) continue;
      const int ci = cfg_index ? h_idx[t] : 0;
      const SimCfg& c = hc[ci];
      int G = std::max(1, 32 / std::max(c.W, 1));
      if (ils) G = std::max(1, std::min(G, (ctx->ils_split ? kPackSlotsSplit : kPackSlots) /
                                              std::max(1, c.W * std::max(c.MC, 1))));
      if (ils) G = std::min(G, ctx->ils_split ? kIlsPackMaxSplit : kIlsPackMax);
      open[ci].push_back(t);
      if ((int)open[ci].size() == G) {
        packs.push_back(std::move(open[ci]));
        open[ci].clear();
      }
    }
    for (auto& o : open)
      if (!o.empty()) packs.push_back(std::move(o));
    std::stable_sort(packs.begin(), packs.end(),
                     [&](const std::vector<int32_t>& a, const std::vector<int32_t>& b) { return work(a[0]) > work(b[0]); });
    const bool spread = packs.size() > 1 && packs.size() <= (size_t)ctx->sm_count;
    off.assign(1, 0);
    flat.clear();
    for (auto& pk : packs) {
      flat.insert(flat.end(), pk.begin(), pk.end());
      off.push_back((int32_t)flat.size());
      if (spread)
        for (int w = 1; w < kSimWarps; ++w) off.push_back((int32_t)flat.size());
    }
  };
  const bool indep = !want_log && !hash;
  std::vector<int32_t> pk_off[3], pk_jobs[3];
  int32_t* d_pk[3] = {nullptr, nullptr, nullptr};
  for (int pol : {SCLS_POLICY_ILS, SCLS_POLICY_SLS}) {
    if (!indep || ctx->ils_lockstep || lists[pol].empty()) continue;
    if (pol == SCLS_POLICY_SLS && !ctx->ils_split) continue;  // SLS packs only in split mode
    make_packs(lists[pol], pol == SCLS_POLICY_ILS, pk_off[pol], pk_jobs[pol]);
    const size_t m = pk_off[pol].size() + pk_jobs[pol].size();
    d_pk[pol] = (int32_t*)ctx->buf(kSlotSim + 26 + pol, sizeof(int32_t) * m);
    if (!d_pk[pol]) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
    std::vector<int32_t> h(pk_off[pol]);
    h.insert(h.end(), pk_jobs[pol].begin(), pk_jobs[pol].end());
    SCLS_CUDA(cudaMemcpyAsync(d_pk[pol], h.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, s));
  }
  // lock-step fallback lists of the independent-lane kernels, one per policy
  // (the per-policy launches may run concurrently)
  int32_t* d_fb_ils = (int32_t*)ctx->buf(kSlotSim + 24, sizeof(int32_t) * (n_traces + 1));
  int32_t* d_fb_sls = (int32_t*)ctx->buf(kSlotSim + 25, sizeof(int32_t) * (n_traces + 1));
  if (!d_fb_ils || !d_fb_sls) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  // Per-policy launches; with more than one policy they run concurrently on
  // forked streams so one kernel's tail overlaps the others' work.
  int n_pol = 0;
  for (int q = 0; q < 3; ++q) n_pol += !lists[q].empty() || !lists[3 + q].empty();
  const bool fork = ctx->sim_concurrent && n_pol > 1;
  if (fork) {
#ifndef SCLS_SIM_PRIO
#define SCLS_SIM_PRIO 0
#endif
    // SCLS_SIM_PRIO 1: the SCLS launch's stream (side[SCLS]) at the greatest
    // priority, so its pending CTAs are placed before the other policies'
    for (int q = 0; q < 3; ++q)
      if (!ctx->side[q]) {
        int lo = 0, hi = 0;
        SCLS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        SCLS_CUDA(cudaStreamCreateWithPriority(&ctx->side[q], cudaStreamNonBlocking,
                                               SCLS_SIM_PRIO && q == SCLS_POLICY_SCLS ? hi : lo));
      }
    SCLS_CUDA(cudaEventRecord(ctx->ev[8], s));
  }
  int64_t at = 0;
  int k = 0;
#ifndef SCLS_SIM_ORDER
#define SCLS_SIM_ORDER 0
#endif
  constexpr int kOrder[3][3] = {{SCLS_POLICY_ILS, SCLS_POLICY_SCLS, SCLS_POLICY_SLS},
                                {SCLS_POLICY_SCLS, SCLS_POLICY_ILS, SCLS_POLICY_SLS},
                                {SCLS_POLICY_SCLS, SCLS_POLICY_SLS, SCLS_POLICY_ILS}};
  for (int pol : kOrder[SCLS_SIM_ORDER]) {  // longest first
    const int32_t cnt = (int32_t)lists[pol].size(), wcnt = (int32_t)lists[3 + pol].size();
    int64_t off = 0, woff = 0;
    for (int q = 0; q < pol; ++q) off += (int64_t)lists[q].size();
    for (int q = 0; q < 3 + pol; ++q) woff += (int64_t)lists[q].size();
    if (cnt == 0 && wcnt == 0) continue;
    cudaStream_t ls = s;
    if (fork) {
      ls = ctx->side[pol];
      SCLS_CUDA(cudaStreamWaitEvent(ls, ctx->ev[8], 0));
    }
    const int wpb = kSimWarps;
    const int grid = div_up(cnt, wpb);
    const int32_t* l = d_lists + off;
    at += cnt;
#define SCLS_SIM_LAUNCH(POLV)                                                                      \
  if (want_log) sim_kernel<POLV, true, true><<<grid, wpb * 32, 0, ls>>>(p, l, cnt);          \
  else if (hash) sim_kernel<POLV, true, false><<<grid, wpb * 32, 0, ls>>>(p, l, cnt);        \
  else sim_kernel<POLV, false, false><<<grid, wpb * 32, 0, ls>>>(p, l, cnt);
#define SCLS_SIM_LAUNCH_WIDE(POLV)                                                                     \
  if (want_log) sim_kernel<POLV, true, true, kWideV><<<wgrid, wpb * 32, 0, ls>>>(p, wl, wcnt);   \
  else if (hash) sim_kernel<POLV, true, false, kWideV><<<wgrid, wpb * 32, 0, ls>>>(p, wl, wcnt); \
  else sim_kernel<POLV, false, false, kWideV><<<wgrid, wpb * 32, 0, ls>>>(p, wl, wcnt);
    if (wcnt > 0) {  // more than 32 workers: the lock-step kernel with 32 worker slots per lane
      const int wgrid = div_up(wcnt, wpb);
      const int32_t* wl = d_lists + woff;
      if (pol == SCLS_POLICY_SCLS) { SCLS_SIM_LAUNCH_WIDE(SCLS_POLICY_SCLS) }
      else if (pol == SCLS_POLICY_SLS) { SCLS_SIM_LAUNCH_WIDE(SCLS_POLICY_SLS) }
      else { SCLS_SIM_LAUNCH_WIDE(SCLS_POLICY_ILS) }
      SCLS_LAUNCHED();
    }
#undef SCLS_SIM_LAUNCH_WIDE
    if (cnt == 0) {
    } else if (pol == SCLS_POLICY_SCLS) { SCLS_SIM_LAUNCH(SCLS_POLICY_SCLS) }
    else if (pol == SCLS_POLICY_SLS && !want_log && !hash && !ctx->ils_lockstep) {
      // independent worker lanes; exact cross-worker ties re-run in lock step
      SCLS_CUDA(cudaMemsetAsync(d_fb_sls, 0, sizeof(int32_t), ls));
      if (ctx->ils_split) {  // packs of 32 / W jobs simulate, then a warp per job merges
        const int32_t npk = (int32_t)pk_off[pol].size() - 1;
        sim_sls_pack_kernel<<<div_up(npk, wpb), wpb * 32, 0, ls>>>(p, d_pk[pol], d_pk[pol] + npk + 1, npk);
        SCLS_LAUNCHED();
        sim_sls_merge_kernel<<<grid, wpb * 32, 0, ls>>>(p, l, cnt, d_fb_sls, d_fb_sls + 1);
      } else {
        sim_sls_indep_kernel<<<grid, wpb * 32, 0, ls>>>(p, l, cnt, d_fb_sls, d_fb_sls + 1);
      }
      SCLS_LAUNCHED();
      sim_kernel<SCLS_POLICY_SLS, false, false><<<grid, wpb * 32, 0, ls>>>(p, d_fb_sls + 1, cnt, d_fb_sls);
    }
    else if (pol == SCLS_POLICY_SLS) { SCLS_SIM_LAUNCH(SCLS_POLICY_SLS) }
    else if (!want_log && !hash && ctx->ils_lockstep) sim_ils_lean_kernel<<<grid, wpb * 32, 0, ls>>>(p, l, cnt, nullptr);
    else if (!want_log && !hash) {
      // independent instance lanes; jobs with an exact cross-instance time tie
      // are re-run by the lock-step kernel from a device-side list
      SCLS_CUDA(cudaMemsetAsync(d_fb_ils, 0, sizeof(int32_t), ls));
      const int32_t npk = (int32_t)pk_off[pol].size() - 1;
      if (ctx->ils_split) {
        SCLS_CUDA(cudaFuncSetAttribute(sim_ils_indep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kIlsPackSmemSplit));
        sim_ils_indep_kernel<true><<<div_up(npk, wpb), wpb * 32, kIlsPackSmemSplit, ls>>>(
            p, d_pk[pol], d_pk[pol] + npk + 1, npk, d_fb_ils, d_fb_ils + 1);
        SCLS_LAUNCHED();
        sim_ils_merge_kernel<<<grid, wpb * 32, 0, ls>>>(p, l, cnt, d_fb_ils, d_fb_ils + 1);
      } else {
        SCLS_CUDA(cudaFuncSetAttribute(sim_ils_indep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kIlsPackSmem));
        sim_ils_indep_kernel<false><<<div_up(npk, wpb), wpb * 32, kIlsPackSmem, ls>>>(
            p, d_pk[pol], d_pk[pol] + npk + 1, npk, d_fb_ils, d_fb_ils + 1);
      }
      SCLS_LAUNCHED();
      sim_ils_lean_kernel<<<grid, wpb * 32, 0, ls>>>(p, d_fb_ils + 1, cnt, d_fb_ils);
    }
    else { SCLS_SIM_LAUNCH(SCLS_POLICY_ILS) }
#undef SCLS_SIM_LAUNCH
    if (cnt > 0) SCLS_LAUNCHED();
    if (fork) {
      SCLS_CUDA(cudaEventRecord(ctx->ev[9 + k], ls));
      SCLS_CUDA(cudaStreamWaitEvent(s, ctx->ev[9 + k], 0));
    }
    ++k;
  }
  (void)at;
  SCLS_CUDA(cudaEventRecord(ctx->ev[2], s));
  if (mem == SCLS_MEM_HOST) {
    SCLS_CUDA(cudaMemcpyAsync(results, d_res, sizeof(scls_trace_result) * n_traces, cudaMemcpyDeviceToHost, s));
    if (hist_bins > 0)
      SCLS_CUDA(cudaMemcpyAsync(slice_hist, d_hist, sizeof(int64_t) * (size_t)n_traces * hist_bins, cudaMemcpyDeviceToHost, s));
    if (want_log) {
      const int64_t nl = p.n_logged;
      SCLS_CUDA(cudaMemcpyAsync(log->rec_count, p.rec_count, sizeof(int64_t) * nl, cudaMemcpyDeviceToHost, s));
      SCLS_CUDA(cudaMemcpyAsync(log->mem_count, p.mem_count, sizeof(int64_t) * nl, cudaMemcpyDeviceToHost, s));
      SCLS_CUDA(cudaMemcpyAsync(log->records, p.recs, sizeof(scls_event_record) * (size_t)nl * log->rec_cap, cudaMemcpyDeviceToHost, s));
      if (log->mem_cap > 0)
        SCLS_CUDA(cudaMemcpyAsync(log->members, p.mems, sizeof(scls_member) * (size_t)nl * log->mem_cap, cudaMemcpyDeviceToHost, s));
    }
  }
  SCLS_CUDA(cudaEventRecord(ctx->ev[3], s));
  SCLS_CUDA(cudaStreamSynchronize(s));
  cudaEventElapsedTime(&ctx->timings[0], ctx->ev[0], ctx->ev[3]);
  cudaEventElapsedTime(&ctx->timings[6], ctx->ev[1], ctx->ev[2]);
  cudaEventElapsedTime(&ctx->timings[2], ctx->ev[0], ctx->ev[1]);
  return SCLS_OK;
}

extern "C" scls_status scls_simulate(scls_ctx* ctx, int32_t n_traces, const int64_t* req_offset,
                                     const double* arrival, const int32_t* input_len,
                                     const int32_t* gen_len, int32_t n_cfgs, const scls_sched_cfg* cfgs,
                                     const int32_t* cfg_index, const scls_latency* lat,
                                     const scls_memory* memm, scls_trace_result* results,
                                     int32_t hist_bins, int64_t* slice_hist, scls_event_log* log,
                                     int32_t mem) {
  if (!ctx) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null context");
  ctx->err.clear();
  ctx->err_request = -1;
  ctx->launches = 0;
  std::fill(ctx->timings, ctx->timings + 8, 0.f);
  SCLS_CUDA(cudaSetDevice(ctx->device));
  if (n_traces < 0 || n_cfgs < 1 || !cfgs || !lat || !memm || !results || !req_offset || hist_bins < 0 ||
      (hist_bins > 0 && !slice_hist))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n_traces == 0) return SCLS_OK;
  std::vector<int32_t> h_idx;
  if (cfg_index) {
    h_idx.resize(n_traces);
    if (mem == SCLS_MEM_DEVICE)
      SCLS_CUDA(cudaMemcpy(h_idx.data(), cfg_index, sizeof(int32_t) * n_traces, cudaMemcpyDeviceToHost));
    else
      std::memcpy(h_idx.data(), cfg_index, sizeof(int32_t) * n_traces);
    for (int32_t v : h_idx)
      if (v < 0 || v >= n_cfgs) return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "cfg_index out of range");
  }
  return simulate_core(ctx, n_traces, req_offset, arrival, input_len, gen_len, n_cfgs, cfgs, n_traces, {}, h_idx,
                       lat, memm, results, hist_bins, slice_hist, log, mem, mem);
}

extern "C" scls_status scls_simulate_grid(scls_ctx* ctx, int32_t n_traces, const int64_t* req_offset,
                                          const double* arrival, const int32_t* input_len,
                                          const int32_t* gen_len, int32_t n_cfgs, const scls_sched_cfg* cfgs,
                                          const scls_latency* lat, const scls_memory* memm,
                                          scls_trace_result* results, int32_t hist_bins, int64_t* slice_hist,
                                          scls_event_log* log, int32_t mem) {
  if (!ctx) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null context");
  ctx->err.clear();
  ctx->err_request = -1;
  ctx->launches = 0;
  std::fill(ctx->timings, ctx->timings + 8, 0.f);
  SCLS_CUDA(cudaSetDevice(ctx->device));
  if (n_traces < 0 || n_cfgs < 1 || !cfgs || !lat || !memm || !results || !req_offset || hist_bins < 0 ||
      (hist_bins > 0 && !slice_hist) || (int64_t)n_traces * n_cfgs > INT32_MAX)
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n_traces == 0) return SCLS_OK;
  const int32_t n_jobs = n_traces * n_cfgs;
  std::vector<int32_t> h_src(n_jobs), h_idx(n_jobs);
  for (int32_t j = 0; j < n_jobs; ++j) {
    h_src[j] = j % n_traces;
    h_idx[j] = j / n_traces;
  }
  return simulate_core(ctx, n_traces, req_offset, arrival, input_len, gen_len, n_cfgs, cfgs, n_jobs, h_src, h_idx,
                       lat, memm, results, hist_bins, slice_hist, log, mem, mem);
}

namespace scls {
scls_status generate_device(scls_ctx* ctx, int32_t n_specs, const scls_workload_spec* specs,
                            std::vector<int64_t>& h_off, double** arr, int32_t** inp, int32_t** gen);
}

// Generate n_specs traces on the device, then run the jobs (h_src, h_idx) on
// them; grid = true builds the every-config-on-every-trace job list.
static scls_status run_generated(scls_ctx* ctx, int32_t n_specs, const scls_workload_spec* specs, int32_t n_cfgs,
                                 const scls_sched_cfg* cfgs, bool grid, const scls_latency* lat,
                                 const scls_memory* memm, scls_trace_result* results, int32_t hist_bins,
                                 int64_t* slice_hist, scls_event_log* log, int32_t mem) {
  if (!ctx) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null context");
  ctx->err.clear();
  ctx->err_request = -1;
  ctx->launches = 0;
  std::fill(ctx->timings, ctx->timings + 8, 0.f);
  SCLS_CUDA(cudaSetDevice(ctx->device));
  if (n_specs < 0 || n_cfgs < 1 || !cfgs || !lat || !memm || !results || (n_specs > 0 && !specs) ||
      hist_bins < 0 || (hist_bins > 0 && !slice_hist) || (int64_t)n_specs * n_cfgs > INT32_MAX ||
      (!grid && n_cfgs != n_specs))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n_specs == 0) return SCLS_OK;
  cudaStream_t s = ctx->stream;
  SCLS_CUDA(cudaEventRecord(ctx->ev[14], s));
  std::vector<int64_t> h_off;
  double* d_arr = nullptr;
  int32_t* d_inp = nullptr;
  int32_t* d_gen = nullptr;
  scls_status st = generate_device(ctx, n_specs, specs, h_off, &d_arr, &d_inp, &d_gen);
  if (st) return st;
  SCLS_CUDA(cudaEventRecord(ctx->ev[15], s));
  const int32_t n_jobs = grid ? n_specs * n_cfgs : n_specs;
  std::vector<int32_t> h_src, h_idx(n_jobs);
  if (grid) {
    h_src.resize(n_jobs);
    for (int32_t j = 0; j < n_jobs; ++j) {
      h_src[j] = j % n_specs;
      h_idx[j] = j / n_specs;
    }
  } else {
    for (int32_t j = 0; j < n_jobs; ++j) h_idx[j] = j;
  }
  // offsets on the host, request arrays on the device
  st = simulate_core(ctx, n_specs, h_off.data(), d_arr, d_inp, d_gen, n_cfgs, cfgs, n_jobs, h_src, h_idx, lat,
                     memm, results, hist_bins, slice_hist, log, mem, kMemDeviceArrays);
  if (st) return st;
  float gen_ms = 0.f, all_ms = 0.f;
  cudaEventElapsedTime(&gen_ms, ctx->ev[14], ctx->ev[15]);
  cudaEventElapsedTime(&all_ms, ctx->ev[14], ctx->ev[3]);
  ctx->timings[7] = gen_ms;
  ctx->timings[0] = all_ms;
  return SCLS_OK;
}

extern "C" scls_status scls_run_sweep(scls_ctx* ctx, int32_t n_traces, const scls_workload_spec* specs,
                                      int32_t n_cfgs, const scls_sched_cfg* cfgs, const scls_latency* lat,
                                      const scls_memory* memm, scls_trace_result* results, int32_t hist_bins,
                                      int64_t* slice_hist, scls_event_log* log, int32_t mem) {
  return run_generated(ctx, n_traces, specs, n_cfgs, cfgs, true, lat, memm, results, hist_bins, slice_hist, log,
                       mem);
}

extern "C" scls_status scls_run_experiments(scls_ctx* ctx, int32_t n_runs, const scls_workload_spec* specs,
                                            const scls_sched_cfg* cfgs, const scls_latency* lat,
                                            const scls_memory* memm, scls_trace_result* results, int32_t hist_bins,
                                            int64_t* slice_hist, scls_event_log* log, int32_t mem) {
  return run_generated(ctx, n_runs, specs, n_runs, cfgs, false, lat, memm, results, hist_bins, slice_hist, log,
                       mem);
}
