// dp_mono.cuh — the Eq. 10 DP (reference batcher.cpp:48-67) for one large
// pool when the cost model is MONOTONE, replacing the serial chain by an
// exact decision test.
//
// Monotone case: every latency coefficient has a clear sign bit (>= +0) and
// the memory model is valid (analytic, or a rule table with decreasing
// thresholds and non-decreasing caps).  Then, computed exactly as the
// reference computes it,
//   * c(L, k) = batch_serve_time(k, L, S) is non-decreasing in L and in k
//     (sums and products of non-negative monotone terms; fl() is monotone);
//   * the window K(L) is non-increasing in L;
// and therefore T is non-decreasing: every candidate of row j,
// fl(T[j-k] + c(L_j, k)), is >= fl(T[j-k] + c(L_{j-1}, k-1)) >= T[j-1]
// (k >= 2), and fl(T[j-1] + c(L_j, 1)) >= T[j-1].
//
// Decision test.  Let T[0..a] be final and row r > a+1.  Every candidate of
// r whose source j lies in (a, r-1] satisfies
//   fl(T[j] + c(L_r, r-j)) >= fl(T[a] + c(L_r, 1)) =: LB_r.
// If the exact minimum F_r over the sources j <= a is strictly below LB_r,
// no later source can reach or tie it: T[r] = F_r with F_r's k, exactly what
// the reference's full scan returns.  Row a+1 itself is always final (all its
// sources are <= a).
//
// Warp roles (16 warps, warp w on SMSP w % 4): warp 0 = main (rows of the
// current tile), warps 4 / 8 / 12 = stagers (row metadata 3 tiles ahead and
// c(L, 1..64) once per run of equal L in the tile, 2 tiles ahead: ~1 load per
// stager thread per tile instead of 2,048 per-row cost loads on the
// helpers), the other 12 = helpers (far candidates one tile ahead).
// Per tile of 32 rows (lane m of warp 0 <-> row 32t+1+m):
//   far   sources j <= 32(t-1): helper warps one tile ahead; each of the 12
//         helper warps scans one k-segment of every row (lane m <-> row m),
//         lane-serial (no per-row reductions), then one helper merges the
//         12 partial minima in ascending-k order;
//   mid   sources in the previous tile: main warp at tile start, 4
//         interleaved partial minima (short dependency chains);
//   then ROUNDS: decide every pending row against LB; the leading run of
//   decided rows becomes final, the frontier moves past it, its T values are
//   pushed into the rows still pending, repeat.  On C3 a tile takes 1-2 rounds
//   instead of 32 chain steps.
// Ties: every partial minimum keeps the smallest k among equal values and the
// merges compare (value, k) lexicographically — the reference's ascending-k
// scan with strict `<`.
#pragma once

#include "dp_chain.cuh"

namespace scls {

constexpr int kMonoSegs = kDpHelpers;  // 12 k-segments per row per CTA
constexpr int kDpMaxCluster = 4;       // CTAs per DP cluster (dp_mono_kernel<., kC>)
#ifndef SCLS_DP_FAR_TOP
#define SCLS_DP_FAR_TOP 48
#endif
constexpr int kFarTop = SCLS_DP_FAR_TOP;  // far k's near the window, split finer

// Shared memory of dp_mono_kernel<., kC>.  kC > 1 stages 96 costs per row
// (the near-far band k <= 95 of CTA 0's helpers) and holds the peers'
// far-far partials in a 3-deep ring (Q).
template <int kC>
struct DpMonoSmemT {
  static constexpr int kStage = kC > 1 ? 96 : kDpStageK;
  double ring[kDpRing];              // 32 KB of recent T
  double cs[kC > 1 ? 3 : 1][kStage][32];   // kC > 1: staged c(L_r, 1..kStage), +INF past W_r
  double cr[kC > 1 ? 1 : 3][32][64];      // kC == 1: c(L, 1..64) per run of equal L in the tile,
                                          // +INF past the run's K(L) (W_r = min(K, r) adds only
                                          // k <= r, which j >= 0 already enforces)
  int32_t rs[3][32];                      // kC == 1: the run slot of each row
  double Pv[2][kMonoSegs][32];       // CTA 0 helpers' partial minima per segment
  int32_t Pk[2][kMonoSegs][32];
  double Qv[3][32];                  // a peer's merged far-far minimum per row (kC > 1)
  int32_t Qk[3][32];
  unsigned long long tiles_done;     // CTA 0: tiles whose T is final (read by the peers)
  unsigned long long far_done;       // a peer: far-far tiles whose Q entry is final (read by CTA 0)
  double Fv[2][32];                  // merged far minimum per row
  int32_t Fk[2][32];
  int32_t W[4][32];
  int32_t CB[4][32];
  int32_t sp[4][32];                 // split of the last tiles (ring mode: flushed a tile later)
  long long arrive_t[16];            // SCLS_DP_PROF_ARRIVE diagnostics: each warp's barrier arrival
};
using DpMonoSmem = DpMonoSmemT<1>;

// ---- thread-block-cluster primitives (DSMEM stores, counters at cluster scope)
__device__ __forceinline__ uint32_t dp_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t dp_mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t dp_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void dp_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Monotone counters at cluster scope.  A writer orders its CTA's earlier
// shared-memory writes (made visible to it by a CTA barrier) before the
// counter with a cumulative release fence; readers poll with acquire loads,
// so no phase aliasing however far one side runs ahead.
__device__ __forceinline__ void dp_fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
__device__ __forceinline__ void dp_st_count(unsigned long long* c, unsigned long long v) {
  asm volatile("st.relaxed.cluster.shared::cta.u64 [%0], %1;" ::"r"(dp_smem_u32(c)), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long dp_ld_acquire(uint32_t cluster_addr) {
  unsigned long long v;
  asm volatile("ld.acquire.cluster.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(cluster_addr) : "memory");
  return v;
}
__device__ __forceinline__ double dp_ld_remote(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int32_t dp_ld_remote_s32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
// Polls a (local or remote) counter until it reaches target; a bounded spin
// turns a protocol error into a trap (a launch error) instead of a hung GPU.
__device__ __forceinline__ void dp_wait_count(uint32_t cluster_addr, unsigned long long target) {
  for (uint32_t it = 0;; ++it) {
    if (dp_ld_acquire(cluster_addr) >= target) return;
    if (it > (1u << 27)) __trap();
    __nanosleep(20);
  }
}

// (v, k) lexicographic "a before b": smaller value, ties to the smaller k.
__device__ __forceinline__ bool lex_lt(double va, int ka, double vb, int kb) {
  return va < vb || (va == vb && ka < kb);
}

// kC > 1 (a thread-block cluster of kC CTAs, !kGlobalT): CTA 0 runs the
// kernel below; CTAs 1..kC-1 are far-candidate helpers only.  Their 12
// helper warps take far segments 12 rank .. 12 rank + 11 of every row (the
// 12 kC segments split the k range as the 12 did), read T from their own ring
// -- after each tile's barrier an idle warp of CTA 0 publishes tiles_done
// (release fence + store); a peer's helper warp 0 polls it (acquire) and
// copies the tile's 32 T values out of CTA 0's ring over DSMEM.  Every
// exchange is a pull of data the owner finished in its own shared memory:
// the owner publishes a monotone counter after a release fence, the reader
// polls it with acquire loads and then loads over DSMEM.
// Pv/Pk are double-buffered by tile parity: a peer writes far(u) only after
// tile u-2 is final, and CTA 0 merged far(u-2) before finishing tile u-3.
template <bool kGlobalT, int kC = 1>
__global__ void __launch_bounds__(kDpThreads, 1)
    dp_mono_kernel(int32_t n, const int32_t* __restrict__ Krow, const int32_t* __restrict__ cbase,
                   const double* __restrict__ cost, double* __restrict__ T, int32_t* __restrict__ split,
                   unsigned long long* __restrict__ prof, const int32_t* __restrict__ gate = nullptr,
                   int32_t gate_id = 0) {
  if (gate && *gate != gate_id) return;  // small-pool launches: the DP kernel the device did not choose
  extern __shared__ __align__(16) unsigned char dp_smem_raw[];
  using Smem = DpMonoSmemT<kC>;
  Smem& sm = *reinterpret_cast<Smem*>(dp_smem_raw);
  constexpr int kStage = Smem::kStage;
  constexpr int M = kDpRing - 1;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
#ifndef SCLS_DP_MAIN_HI
#define SCLS_DP_MAIN_HI 1
#endif
  // Role index of this warp.  Hardware warp w issues on SMSP w % 4, and an
  // SMSP's arbiter prefers the highest warp id among eligible warps: with
  // SCLS_DP_MAIN_HI the main warp (role 0) is hardware warp 12, so the
  // stagers sharing its SMSP (roles 4 / 8 / 12 = warps 8 / 4 / 0) never take
  // an issue slot it could use.
  const int tid = threadIdx.x, lane = tid & 31, hw_warp = tid >> 5;
  const int warp = SCLS_DP_MAIN_HI && (hw_warp & 3) == 0 ? 12 - hw_warp : hw_warp;
  const bool helper = (warp & 3) != 0;
  const int h = warp - 1 - (warp >> 2);  // helper index 0..11
  const int ht = h * 32 + lane;
  const int ntiles = (n + 31) >> 5;
  static_assert(kC >= 1 && kC <= kDpMaxCluster && (kC == 1 || !kGlobalT), "cluster variant: T in the ring");
  // kC == 1: the 12 helper warps split every row's far k range.  kC > 1: the
  // peers' 12 (kC - 1) warps split the far-far range (sources <= 32(u-2)).
  constexpr int kSegs = kC > 1 ? kMonoSegs * (kC - 1) : kMonoSegs;
  const int rank = kC > 1 ? (int)dp_cluster_rank() : 0;
  const int g = kC > 1 ? h + kMonoSegs * (rank - 1) : h;  // this helper warp's far segment

#ifndef SCLS_DP_STAGERS
#define SCLS_DP_STAGERS 1
#endif
  // kC == 1: warps 4, 8, 12 (idle otherwise: SMSP 0 is left to the main
  // warp) load the row metadata and stage the cost block, so the 12 helper
  // warps only scan far candidates.
#ifndef SCLS_DP_STAGER_WARPS
#define SCLS_DP_STAGER_WARPS 3
#endif
  constexpr bool kStagers = SCLS_DP_STAGERS && kC == 1;
  constexpr int kStThreads = 32 * SCLS_DP_STAGER_WARPS;  // warps 4 (, 8, 12)
  const bool stager = kStagers && warp != 0 && (warp & 3) == 0 && (warp >> 2) <= SCLS_DP_STAGER_WARPS;
  const int sidx = ((warp >> 2) - 1) * 32 + lane;  // 0..95 in the stager warps
  const bool meta_thread = kStagers ? (stager && sidx < 32) : (helper && h == 0);
  auto load_meta = [&](int u) {
    if (meta_thread && u < ntiles) {
      const int r = (u << 5) + 1 + lane;
      sm.W[u & 3][lane] = r <= n ? Krow[r - 1] : 0;
      sm.CB[u & 3][lane] = r <= n ? cbase[r - 1] : 0;
    }
  };
  // Staging c(L_r, 1..64) of tile u: stage_load issues the global loads
  // into registers, stage_store writes them (+INF past W_r) to shared
  // memory — far() runs in between so the loads' latency is hidden.
  constexpr int kPer = (32 * kStage + kDpHelperThreads - 1) / kDpHelperThreads;
  auto stage_load = [&](int u, double* v) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) v[i] = kInf;
    if (u >= ntiles) return;
    const int W = sm.W[u & 3][lane], CB = sm.CB[u & 3][lane];  // row m == lane for every i
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = ht + i * kDpHelperThreads;
      const int k = 1 + (e >> 5);
      if (e < 32 * kStage && k <= W) v[i] = cost[CB + k];
    }
  };
  auto stage_store = [&](int u, const double* v) {
    if (u >= ntiles) return;
    const int b = u % 3;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = ht + i * kDpHelperThreads;
      if (e < 32 * kStage) sm.cs[b][e >> 5][e & 31] = v[i];
    }
  };
  auto stage_costs = [&](int u) {
    double v[kPer];
    stage_load(u, v);
    stage_store(u, v);
  };
  constexpr int kPerS = (32 * kStage + kStThreads - 1) / kStThreads;
  auto stage_costs_st = [&](int u) {  // the stager warps' staging of tile u, one row per run
    if (u >= ntiles) return;
    const int r = (u << 5) + 1 + lane;
    const bool okr = r <= n;
    const int CBm = sm.CB[u & 3][lane];
    const unsigned heads = __ballot_sync(0xffffffffu, okr && (lane == 0 || sm.CB[u & 3][lane - 1] != CBm));
    const int last = 31 - __clz(__ballot_sync(0xffffffffu, okr));
    const int nrun = __popc(heads);
    const int b = u % 3;
    if (sidx < 32) sm.rs[b][lane] = okr ? __popc(heads & ((2u << lane) - 1u)) - 1 : 0;
#ifndef SCLS_DP_ST_PRE
#define SCLS_DP_ST_PRE 0
#endif
    // the first SCLS_DP_ST_PRE entries per thread: every load issued before any store
    auto cost_of = [&](int e) {
      const int q = e >> 6, k = (e & 63) + 1;
      const int h0 = __fns(heads, 0, q + 1);                       // the run's first row
      const unsigned after = heads & ~((2u << h0) - 1u);
      const int h1 = after ? __ffs(after) - 2 : last;              // its last row: the largest window
      const int kq = sm.W[u & 3][h1];
      return k <= kq ? cost[sm.CB[u & 3][h0] + k] : kInf;
    };
    int e = sidx;
    if (SCLS_DP_ST_PRE > 0) {
      double cv[SCLS_DP_ST_PRE > 0 ? SCLS_DP_ST_PRE : 1];
#pragma unroll
      for (int i = 0; i < SCLS_DP_ST_PRE; ++i) {
        const int ei = e + i * kStThreads;
        cv[i] = ei < nrun * 64 ? cost_of(ei) : kInf;
      }
#pragma unroll
      for (int i = 0; i < SCLS_DP_ST_PRE; ++i) {
        const int ei = e + i * kStThreads;
        if (ei < nrun * 64) sm.cr[b][ei >> 6][ei & 63] = cv[i];
      }
      e += SCLS_DP_ST_PRE * kStThreads;
    }
    for (; e < nrun * 64; e += kStThreads) sm.cr[b][e >> 6][e & 63] = cost_of(e);
  };
  // c(L_r, k) of this lane's row in tile buffer b (k <= 64); rsl = sm.rs[b][lane]
  auto csv = [&](int b, int rsl, int k) -> double {
    if (kStagers) return sm.cr[b][rsl][k - 1];
    return sm.cs[b][k - 1][lane];
  };
  // This warp's segment g of the far candidates of row r (lane) over the
  // sources j <= jtop (k >= r - jtop): (value, k) lexicographic minimum.
  auto seg_scan = [&](int u, int jtop, int W, int cb, double& best, int& bk) {
    const int r = (u << 5) + 1 + lane;
    const int jmax = jtop;
    const int kmin = r - jmax;
    const int span = W - kmin + 1;
    if (span > 0) {
      // Two tiers: the top kFarTop k's (the batch sizes near the window, where
      // the minimum of these monotone costs lives and pruning rarely holds)
      // in kMonoSegs/2 short segments, the rest in the other half (mostly
      // pruned by the bound below) -- the helpers' work evens out.
      constexpr int kHalf = kSegs / 2;
      const int top = min(span, kFarTop);
      const int rest = span - top;
#ifndef SCLS_DP_FAR_RR
#define SCLS_DP_FAR_RR 2
#endif
      if (SCLS_DP_FAR_RR == 2 || (SCLS_DP_FAR_RR && g < kHalf)) {
        // The rest in chunks of 8 k's dealt round-robin over the kHalf
        // helpers, each chunk pruned on its own: the unpruned band near the
        // optimum spreads over all of them instead of landing on one
        // helper's contiguous segment (the tile waits for the slowest).
        const double ub = __dadd_rn(kGlobalT ? T[r - W] : sm.ring[(r - W) & M], cost[cb + W]);
        double b2 = kInf;
        int k2 = 0;
        // SCLS_DP_FAR_RR 2: all kSegs helpers deal the whole span [kmin, W]
#ifndef SCLS_DP_FAR_CHUNK
#define SCLS_DP_FAR_CHUNK 16
#endif
        constexpr int kCh = SCLS_DP_FAR_CHUNK;
        constexpr int kDeal = SCLS_DP_FAR_RR == 2 ? kSegs : kHalf;
        const int lim = SCLS_DP_FAR_RR == 2 ? span : rest;
#ifndef SCLS_DP_PRUNE_PRE
#define SCLS_DP_PRUNE_PRE 0
#endif
        // the first SCLS_DP_PRUNE_PRE chunks' bounds loaded together, ahead of the scans
        double lbv[SCLS_DP_PRUNE_PRE > 0 ? SCLS_DP_PRUNE_PRE : 1];
#pragma unroll
        for (int i = 0; i < SCLS_DP_PRUNE_PRE; ++i) {
          const int c0 = g * kCh + i * kDeal * kCh;
          const int k0 = kmin + min(c0, lim - 1), k1 = min(kmin + lim - 1, k0 + kCh - 1);
          lbv[i] = __dadd_rn(kGlobalT ? T[r - k1] : sm.ring[(r - k1) & M], cost[cb + k0]);
        }
        int ci = 0;
        for (int c0 = g * kCh; c0 < lim; c0 += kDeal * kCh, ++ci) {
          const int k0 = kmin + c0, k1 = min(kmin + lim - 1, k0 + kCh - 1);
          double lb;
          if (SCLS_DP_PRUNE_PRE > 0 && ci < SCLS_DP_PRUNE_PRE) {
            lb = lbv[0];
#pragma unroll
            for (int i = 1; i < SCLS_DP_PRUNE_PRE; ++i) lb = ci == i ? lbv[i] : lb;
          } else {
            lb = __dadd_rn(kGlobalT ? T[r - k1] : sm.ring[(r - k1) & M], cost[cb + k0]);
          }
          if (lb > ub) continue;
          double tv[kCh], cv[kCh];
#pragma unroll
          for (int i = 0; i < kCh; ++i) {
            const int k = min(k0 + i, k1);
            const int j = r - k;
            tv[i] = kGlobalT ? T[j] : sm.ring[j & M];
            cv[i] = cost[cb + k];
          }
#pragma unroll
          for (int i = 0; i < kCh; ++i) {
            const double cand = k0 + i <= k1 ? __dadd_rn(tv[i], cv[i]) : kInf;
            if (i & 1) {
              if (cand < b2) {
                b2 = cand;
                k2 = k0 + i;
              }
            } else if (cand < best) {
              best = cand;
              bk = k0 + i;
            }
          }
        }
        if (lex_lt(b2, k2, best, bk)) {
          best = b2;
          bk = k2;
        }
        return;
      }
      int k0, k1;
      if (g < kHalf) {
        const int len = (rest + kHalf - 1) / kHalf;
        k0 = kmin + g * len;
        k1 = min(kmin + rest - 1, k0 + len - 1);
      } else {
        const int len = (top + kHalf - 1) / kHalf;
        k0 = kmin + rest + (g - kHalf) * len;
        k1 = min(W, k0 + len - 1);
      }
      // Exact segment pruning (monotone T and c): every candidate of the
      // segment is >= fl(T[r-k1] + c(L_r, k0)).  If that bound exceeds an
      // actual candidate of the row (k = W, the full window), no candidate
      // of the segment can be the row's minimum or tie it.
      bool skip = k0 > k1;
      if (!skip) {
        const double ub = __dadd_rn(kGlobalT ? T[r - W] : sm.ring[(r - W) & M], cost[cb + W]);
        const double lb = __dadd_rn(kGlobalT ? T[r - k1] : sm.ring[(r - k1) & M], cost[cb + k0]);
        skip = lb > ub;
      }
      // chunks of 8: loads first, then two interleaved ascending-k minima
      double b2 = kInf;
      int k2 = 0;
      for (int kc = k0; !skip && kc <= k1; kc += 8) {
        double tv[8], cv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int k = min(kc + i, k1);
          const int j = r - k;
          tv[i] = kGlobalT ? T[j] : sm.ring[j & M];
          cv[i] = cost[cb + k];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double cand = kc + i <= k1 ? __dadd_rn(tv[i], cv[i]) : kInf;
          if (i & 1) {
            if (cand < b2) {
              b2 = cand;
              k2 = kc + i;
            }
          } else if (cand < best) {
            best = cand;
            bk = kc + i;
          }
        }
      }
      if (lex_lt(b2, k2, best, bk)) {
        best = b2;
        bk = k2;
      }
    }
  };
  // merge of 12 partials (per-warp loads, then a tree); folds into (fv, fk2)
  auto merge12 = [&](const double (*Pv_)[32], const int32_t (*Pk_)[32], double& fv, int& fk2) {
    double v[kMonoSegs];
    int k[kMonoSegs];
#pragma unroll
    for (int s2 = 0; s2 < kMonoSegs; ++s2) {
      v[s2] = Pv_[s2][lane];
      k[s2] = Pk_[s2][lane];
    }
#pragma unroll
    for (int span2 = 1; span2 < kMonoSegs; span2 <<= 1) {
#pragma unroll
      for (int s2 = 0; s2 + span2 < kMonoSegs; s2 += 2 * span2) {
        if (lex_lt(v[s2 + span2], k[s2 + span2], v[s2], k[s2])) {
          v[s2] = v[s2 + span2];
          k[s2] = k[s2 + span2];
        }
      }
    }
    if (lex_lt(v[0], k[0], fv, fk2)) {
      fv = v[0];
      fk2 = k[0];
    }
  };
  // Far candidates of tile u (sources j <= 32(u-1)), merged into Fv/Fk by
  // helper 0 of CTA 0.  kC == 1: the 12 helpers' k-segments of every row.
  // kC > 1: CTA 0's helpers take the near-far band (the 32 sources of tile
  // u-2, costs from the staged cs block) and merge it with the peers'
  // far-far segments of tile u (Q ring, delivered over DSMEM).
  auto far = [&](int u) {
    if (u >= ntiles) return;
    double best = kInf;
    int bk = 0;
    if (kC == 1) {
      seg_scan(u, (u - 1) << 5, sm.W[u & 3][lane], sm.CB[u & 3][lane], best, bk);
    } else {
      const int r = (u << 5) + 1 + lane;
      const int lo = r - sm.W[u & 3][lane];
      const int jn0 = max(0, ((u - 2) << 5) + 1), jn1 = (u - 1) << 5;
      const int cb3 = u % 3;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int j = jn0 + h + q * kMonoSegs;
        if (j <= jn1 && j >= lo && r <= n) {
          const int k = r - j;  // 1 + lane .. 64 + lane, staged (+INF past W_r)
          const double cand = __dadd_rn(sm.ring[j & M], sm.cs[cb3][k - 1][lane]);
          if (lex_lt(cand, k, best, bk)) {
            best = cand;
            bk = k;
          }
        }
      }
    }
    sm.Pv[u & 1][h][lane] = best;
    sm.Pk[u & 1][h][lane] = bk;
#ifndef SCLS_DP_MAIN_MERGE
#define SCLS_DP_MAIN_MERGE 1
#endif
    // kC == 1: the main warp merges the 12 partials itself at the start of
    // tile u (after the tile barrier), so the helpers' barrier and helper 0's
    // merge leave the helpers' path
    if (kC == 1 && SCLS_DP_MAIN_MERGE) return;
    asm volatile("bar.sync 1, %0;" ::"n"(kDpHelperThreads));
    if (h == 0) {
      double fv = kInf;
      int fk2 = 0;
      merge12(sm.Pv[u & 1], sm.Pk[u & 1], fv, fk2);
      if (kC > 1) {
        // each peer's merged far-far minima of tile u, pulled over DSMEM once
        // the peer has published them (acquire)
#pragma unroll 1
        for (int p = 1; p < kC; ++p) {
          dp_wait_count(dp_mapa(dp_smem_u32(&sm.far_done), p), (unsigned long long)u);
          const double qv = dp_ld_remote(dp_mapa(dp_smem_u32(&sm.Qv[u % 3][lane]), p));
          const int qk = dp_ld_remote_s32(dp_mapa(dp_smem_u32(&sm.Qk[u % 3][lane]), p));
          if (lex_lt(qv, qk, fv, fk2)) {
            fv = qv;
            fk2 = qk;
          }
        }
      }
      sm.Fv[u & 1][lane] = fv;
      sm.Fk[u & 1][lane] = fk2;
    }
  };
  // A peer's far-far segments of tile u (sources j <= 32(u-2)): its 12
  // helper warps' partials (Pv, local), merged by its helper 0 into Q[u % 3],
  // then published (warp-wide release fence, far_done = u) for CTA 0 to pull.
  // Q[u % 3] is rewritten for tile u + 3 only after tiles_done >= u + 1,
  // i.e. after CTA 0 consumed it while finishing tile u - 1.
  auto far_far = [&](int u, int W, int cb) {
    double best = kInf;
    int bk = 0;
    if (u >= 2) seg_scan(u, (u - 2) << 5, W, cb, best, bk);
    sm.Pv[u & 1][h][lane] = best;
    sm.Pk[u & 1][h][lane] = bk;
    asm volatile("bar.sync 1, %0;" ::"n"(kDpHelperThreads));
    if (h == 0) {
      double fv = kInf;
      int fk2 = 0;
      merge12(sm.Pv[u & 1], sm.Pk[u & 1], fv, fk2);
      sm.Qv[u % 3][lane] = fv;
      sm.Qk[u % 3][lane] = fk2;
      __syncwarp();
      dp_fence_cluster();
      if (lane == 0) dp_st_count(&sm.far_done, (unsigned long long)u);
    }
  };
  if (kC > 1) {
    if (tid == 0) {
      sm.ring[0] = 0.0;
      sm.tiles_done = 0;
      sm.far_done = 0;
    }
    dp_cluster_sync();
    if (rank != 0) {
      // peer: far_far(u) (sources <= 32(u-2)) once tiles 0..u-3 are final --
      // helper warp 0 polls CTA 0's tiles_done and copies tile u-3's T into
      // this CTA's ring; CTA 0 needs the result only at the end of tile u-1,
      // two tiles later
      if (helper) {
        int Wn = 0, CBn = 0;
        auto meta = [&](int u, int& W_, int& CB_) {
          const int r = (u << 5) + 1 + lane;
          W_ = u < ntiles && r <= n ? Krow[r - 1] : 0;
          CB_ = u < ntiles && r <= n ? cbase[r - 1] : 0;
        };
        meta(1, Wn, CBn);
        const uint32_t done0 = dp_mapa(dp_smem_u32(&sm.tiles_done), 0);
        for (int u = 1; u < ntiles; ++u) {
          const int Wc = Wn, CBc = CBn;
          meta(u + 1, Wn, CBn);
          if (u >= 3) {
            if (h == 0) {
              dp_wait_count(done0, (unsigned long long)(u - 2));
              const int r = ((u - 3) << 5) + 1 + lane;
              if (r <= n) sm.ring[r & M] = dp_ld_remote(dp_mapa(dp_smem_u32(&sm.ring[r & M]), 0));
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kDpHelperThreads));
          }
          far_far(u, Wc, CBc);
        }
      }
      dp_cluster_sync();  // keep this CTA's shared memory alive until CTA 0 is done
      return;
    }
  }
  if (tid == 0) {
    sm.ring[0] = 0.0;
    T[0] = 0.0;
    split[0] = 0;
  }
  if (kStagers ? stager : helper) {
    load_meta(0);
    load_meta(1);
    load_meta(2);
  }
  // Stagers: the row metadata of tile t + 3 is loaded into registers during
  // tile t - 1 and stored during tile t, so each tile's stager work waits on
  // one global load latency (the costs of tile t + 2), not two in series.
  int pm_w = 0, pm_cb = 0;
  auto meta_prefetch = [&](int u) {
    if (meta_thread && u < ntiles) {
      const int r = (u << 5) + 1 + lane;
      pm_w = r <= n ? Krow[r - 1] : 0;
      pm_cb = r <= n ? cbase[r - 1] : 0;
    }
  };
  if (kStagers && stager) meta_prefetch(3);
#ifndef SCLS_DP_DEFER_TS
#define SCLS_DP_DEFER_TS 1
#endif
  // Ring mode: the main warp leaves T (ring) and split (sp) in shared memory;
  // the first stager warp writes tile u's rows to global during tile u + 1
  // (the backtrack reads them after the kernel), so no global store sits on
  // the main warp's path to the tile barrier.
  constexpr bool kDeferTS = SCLS_DP_DEFER_TS && kStagers && !kGlobalT;
  auto flush_ts = [&](int u) {
    const int r = (u << 5) + 1 + lane;
    if (sidx < 32 && r <= n) {
      T[r] = sm.ring[r & M];
      split[r] = sm.sp[u & 3][lane];
    }
  };
  __syncthreads();
  if (kStagers && stager) {
    stage_costs_st(0);
    stage_costs_st(1);
  }
  if (helper) {
    if (!kStagers) {
      stage_costs(0);
      stage_costs(1);
    }
    for (int m = ht; m < 32; m += kDpHelperThreads) {
      sm.Fv[0][m] = kInf;
      sm.Fk[0][m] = 0;
    }
    for (int e = ht; e < kMonoSegs * 32; e += kDpHelperThreads) {  // tile 0 has no far sources
      sm.Pv[0][e >> 5][e & 31] = kInf;
      sm.Pk[0][e >> 5][e & 31] = 0;
    }
  }
  __syncthreads();

  long long c_a = 0, c_b = 0, c_c = 0, c_d = 0, c_e = 0, c_mid = 0, n_rounds = 0, c_sl = 0, c_hl = 0, c_top = 0;
#ifndef SCLS_DP_PIPE
#define SCLS_DP_PIPE 0
#endif
  // Ring mode, one CTA: the tile barrier split into two named barriers.  The
  // main warp's tile t needs the producers' (helpers + stagers) work of their
  // iteration t - 1 (far(t), costs staged earlier): barrier kBarFar, arrived
  // by the producers, synced by the main warp.  The producers' iteration t
  // needs the main warp's tile t - 1 (T in the ring, the buffers it read):
  // barrier kBarTile, arrived by the main warp, synced by the producers.  A
  // producer never runs more than one iteration ahead, so each barrier has at
  // most one phase outstanding; the main warp no longer waits for the
  // producers at the end of its tile, only (rarely) at the start of the next.
#ifdef SCLS_DP_PROF_ARRIVE
  constexpr bool kProfArrive = true;
#else
  constexpr bool kProfArrive = false;
#endif
  constexpr bool kPipe = SCLS_DP_PIPE && kC == 1 && kStagers && !kGlobalT;
  constexpr int kBarFar = 2, kBarTile = 3;
#ifndef SCLS_DP_MID_HELPERS
#define SCLS_DP_MID_HELPERS 0
#endif
  // The mid candidates (sources in the previous tile) on the helpers: at the
  // start of tile t each helper folds ~3 of the 32 sources into its own far
  // partial of tile t, then arrives on kBarMid; the main warp waits there and
  // merges the 12 partials as before -- its 32-candidate mid scan leaves the
  // critical path.
  constexpr bool kMidH = SCLS_DP_MID_HELPERS && kC == 1 && kStagers && SCLS_DP_MAIN_MERGE && !kPipe;
  constexpr int kBarMid = 4, kMidThreads = 32 * (kMonoSegs + 1);
  auto mid_fold = [&](int u) {
    const int uB = u << 5;
    const int b = u % 3, rs_ = sm.rs[b][lane];
    double best = sm.Pv[u & 1][h][lane];
    int bk = sm.Pk[u & 1][h][lane];
    for (int jj = h; jj < 32; jj += kMonoSegs) {  // ascending j
      const int j = uB - 31 + jj;
      if (j >= 0) {
        const int k = lane + 32 - jj;
        const double cand = __dadd_rn(sm.ring[j & M], csv(b, rs_, k));
        if (lex_lt(cand, k, best, bk)) {
          best = cand;
          bk = k;
        }
      }
    }
    sm.Pv[u & 1][h][lane] = best;
    sm.Pk[u & 1][h][lane] = bk;
  };
  for (int t = 0; t < ntiles; ++t) {
    const int tB = t << 5;
    if (kPipe && t > 0) {
      if (warp == 0)
        asm volatile("bar.sync %0, %1;" ::"n"(kBarFar), "n"(kDpThreads) : "memory");
      else
        asm volatile("bar.sync %0, %1;" ::"n"(kBarTile), "n"(kDpThreads) : "memory");
    }
    const long long t0 = prof ? clock64() : 0;
    long long t1 = t0, t2 = t0;
    if (warp == 0) {
      const int cbuf = t % 3;
      const int rsl = kStagers ? sm.rs[cbuf][lane] : 0;
      const int r = tB + 1 + lane;
      // far: the helpers' 12 partial minima (kC == 1) or their merge, first
      // -- independent of the ring loads below
      double acc = kInf;
      int kb = 0;
      if (kC == 1 && SCLS_DP_MAIN_MERGE) {
        if (kMidH) asm volatile("bar.sync %0, %1;" ::"n"(kBarMid), "n"(kMidThreads) : "memory");
        merge12(sm.Pv[t & 1], sm.Pk[t & 1], acc, kb);
      } else {
        acc = sm.Fv[t & 1][lane];
        kb = sm.Fk[t & 1][lane];
      }
      // mid: sources j = tB-31 .. tB (k = lane+32-jj), 4 interleaved chains.
      // Skipped when it cannot win (exact, monotone case): every mid
      // candidate of row r is >= fl(T[tB-31] + c(L_r, lane+1)) -- T is
      // non-decreasing in j and c in k -- so a row whose far minimum is
      // strictly below that bound keeps it; on C3 the optimum batch (~89
      // rows) lies in the far range and the whole warp usually skips.
#ifndef SCLS_DP_MID_SKIP
#define SCLS_DP_MID_SKIP 0
#endif
      bool mid_needed = true;
      if (SCLS_DP_MID_SKIP) {
        const double lbm = __dadd_rn(sm.ring[max(tB - 31, 0) & M], csv(cbuf, rsl, lane + 1));
        mid_needed = __any_sync(0xffffffffu, !(lbm > acc));
      }
      if (!kMidH && mid_needed) {
      double va[8] = {kInf, kInf, kInf, kInf, kInf, kInf, kInf, kInf};
      int ka[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double tv[8], cv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int jj = c * 8 + i;
          tv[i] = sm.ring[(tB - 31 + jj) & M];
          cv[i] = csv(cbuf, rsl, lane + 32 - jj);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int jj = c * 8 + i;
          const int q = jj & 7;
          const int k = lane + 32 - jj;
          // j ascending = k descending: <= keeps the smallest k
          const double cand = tB - 31 + jj >= 0 ? __dadd_rn(tv[i], cv[i]) : kInf;
          if (cand <= va[q] && tB - 31 + jj >= 0) {
            va[q] = cand;
            ka[q] = k;
          }
        }
      }
#ifndef SCLS_DP_MID_TREE
#define SCLS_DP_MID_TREE 0
#endif
      if (SCLS_DP_MID_TREE) {  // the 8 chains' minima by a (value, k) tree: 3 dependent steps, not 8
#pragma unroll
        for (int span = 1; span < 8; span <<= 1) {
#pragma unroll
          for (int q = 0; q + span < 8; q += 2 * span)
            if (lex_lt(va[q + span], ka[q + span], va[q], ka[q])) {
              va[q] = va[q + span];
              ka[q] = ka[q + span];
            }
        }
        if (lex_lt(va[0], ka[0], acc, kb)) {
          acc = va[0];
          kb = ka[0];
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (lex_lt(va[q], ka[q], acc, kb)) {
            acc = va[q];
            kb = ka[q];
          }
      }
      }  // !kMidH
      // rounds
      if (prof) c_mid += clock64() - t0;
      const double c1 = csv(cbuf, rsl, 1);
      int p0 = 0;  // first pending lane; frontier a = tB + p0
      const int rows = min(32, n - tB);
      double Ta = sm.ring[tB & M];
      while (p0 < rows) {
        ++n_rounds;
        const double lb = __dadd_rn(Ta, c1);
        const bool fin = lane == p0 || (lane > p0 && acc < lb);
        const unsigned m = __ballot_sync(0xffffffffu, fin) >> p0;
        const int d = min((~m) ? __ffs(~m) - 1 : 32 - p0, rows - p0);
        const int p1 = p0 + d;  // lanes [p0, p1) are final
        if (p1 >= rows) break;
        // the final rows [p0, p1) join the ring; push them into lanes >= p1
        if (lane >= p0 && lane < p1) sm.ring[r & M] = acc;
        __syncwarp();
        Ta = sm.ring[(tB + p1) & M];
        double vA = kInf, vB = kInf;
        int kA = 0, kB = 0;
        for (int i0 = p0; i0 < p1; i0 += 8) {
          double tv[8], cv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int i = min(i0 + q, p1 - 1);
            tv[q] = sm.ring[(tB + 1 + i) & M];
            const int k = lane - i;
            cv[q] = csv(cbuf, rsl, k >= 1 ? k : 1);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int i = i0 + q;
            const int k = lane - i;
            const bool ok = i < p1 && k >= 1;
            const double cand = ok ? __dadd_rn(tv[q], cv[q]) : kInf;
            if (q & 1) {
              if (ok && cand <= vB) {
                vB = cand;
                kB = k;
              }
            } else if (ok && cand <= vA) {
              vA = cand;
              kA = k;
            }
          }
        }
        if (lane >= p1) {
          if (lex_lt(vA, kA, acc, kb)) {
            acc = vA;
            kb = kA;
          }
          if (lex_lt(vB, kB, acc, kb)) {
            acc = vB;
            kb = kB;
          }
        }
        p0 = p1;
      }
      if (r <= n) {
        if (kDeferTS) {  // a stager stores tile t's T and split to global during tile t + 1
          sm.sp[t & 3][lane] = r - kb;
        } else {
          T[r] = acc;
          split[r] = r - kb;
        }
        sm.ring[r & M] = acc;
      }
      t1 = t2 = prof ? clock64() : 0;
    } else if (kStagers && stager) {
      if (meta_thread && t + 3 < ntiles) {
        sm.W[(t + 3) & 3][lane] = pm_w;
        sm.CB[(t + 3) & 3][lane] = pm_cb;
      }
      meta_prefetch(t + 4);
      if (kDeferTS && t > 0) flush_ts(t - 1);
      stage_costs_st(t + 2);
      t1 = prof ? clock64() : 0;
    } else if (helper) {
      if (kStagers) {
        if (kMidH) {
          mid_fold(t);
          asm volatile("bar.arrive %0, %1;" ::"n"(kBarMid), "n"(kMidThreads) : "memory");
        }
        t1 = prof ? clock64() : 0;
        far(t + 1);
      } else {
        load_meta(t + 3);
        double sv[kPer];
        stage_load(t + 2, sv);
        t1 = prof ? clock64() : 0;
        far(t + 1);
        stage_store(t + 2, sv);
      }
      t2 = prof ? clock64() : 0;
    }
#ifdef SCLS_DP_PROF_ARRIVE
    if (prof && lane == 0) sm.arrive_t[warp] = clock64();
#endif
    if (!kPipe) {
      __syncthreads();
    } else if (t + 1 < ntiles) {
      if (warp == 0)
        asm volatile("bar.arrive %0, %1;" ::"n"(kBarTile), "n"(kDpThreads) : "memory");
      else
        asm volatile("bar.arrive %0, %1;" ::"n"(kBarFar), "n"(kDpThreads) : "memory");
    }
    if (kC > 1 && warp == 4 && lane == 0) {  // off the main warp's path: publish tile t
      dp_fence_cluster();
      dp_st_count(&sm.tiles_done, (unsigned long long)(t + 1));
    }
    if (prof) {
      const long long t3 = clock64();
#ifdef SCLS_DP_PROF_ARRIVE
      // main warp: how long after its own arrival the last warp arrived, who
      // that was, and the release latency after the last arrival
      if (warp == 0 && lane == 0) {
        long long last = sm.arrive_t[0];
        int who = 0;
        for (int q = 1; q < 16; ++q)
          if (sm.arrive_t[q] > last) {
            last = sm.arrive_t[q];
            who = q;
          }
        c_d += last - sm.arrive_t[0];
        c_e += t3 - last;
        if (who != 0 && (who & 3) == 0) ++c_sl;  // a stager arrived last
        else if (who != 0) {                    // a helper arrived last
          ++c_hl;
          const int hw = who;  // role index; its helper index (far segment)
          if (hw - 1 - (hw >> 2) >= kMonoSegs / 2) ++c_top;
        }
      }
#endif
      if (warp == 0) {
        c_a += t1 - t0;
        c_b += t3 - t1;
      } else if (helper) {
        c_c += t1 - t0;
        c_d += t2 - t1;
        c_e += t3 - t2;
      } else if (stager) {
        c_c += t1 - t0;  // SCLS_DP_PROF_STAGER: the stagers' work per tile
      }
    }
  }
  if (kPipe) __syncthreads();
  if (kDeferTS && stager && ntiles > 0) flush_ts(ntiles - 1);  // after a barrier that follows the last tile
  if (prof && lane == 0) {
    if (warp == 0) {
#ifdef SCLS_DP_PROF_ARRIVE  // [2] last arrival after main's, [3] release latency, [4] / [5] stager / helper last
      atomicAdd(&prof[2], (unsigned long long)c_d);
      atomicAdd(&prof[3], (unsigned long long)c_e);
      atomicAdd(&prof[4], (unsigned long long)c_sl);
      atomicAdd(&prof[5], (unsigned long long)c_hl);
      atomicAdd(&prof[6], (unsigned long long)c_top);
#endif
      atomicAdd(&prof[0], (unsigned long long)c_a);
      atomicAdd(&prof[1], (unsigned long long)c_b);
      if (!kProfArrive) {
        atomicAdd(&prof[6], (unsigned long long)c_mid);
        atomicAdd(&prof[7], (unsigned long long)n_rounds);
      }
    } else if (stager) {
#ifdef SCLS_DP_PROF_STAGER  // diagnostics: the slowest stager's work instead of the helpers' waits
      atomicMax(&prof[4], (unsigned long long)c_c);
#endif
    } else if (helper && !kProfArrive) {
      atomicAdd(&prof[2], (unsigned long long)c_c);
      atomicAdd(&prof[3], (unsigned long long)c_d);
#if defined(SCLS_DP_PROF_MAXFAR)  // diagnostics: the slowest helper's far cycles instead of the waits
      atomicMax(&prof[4], (unsigned long long)c_d);
#elif defined(SCLS_DP_PROF_STAGER)
#else
      atomicAdd(&prof[4], (unsigned long long)c_e);
#endif
      atomicAdd(&prof[5], 1ull);
    }
  }
  if (kC > 1) dp_cluster_sync();  // the peers' shared memory stays valid until CTA 0 is done
}

}  // namespace scls
