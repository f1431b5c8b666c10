// dp_chain.cuh — the Eq. 10 DP chain (reference batcher.cpp:48-67) for one
// large pool, one CTA.
//
//   T[0] = 0,  T[r] = min_{1<=k<=W_r} T[r-k] + c(L_r, k),  ties -> smallest k
//
// Rows are processed in tiles of 32; lane m of the main warp (warp 0) owns
// row r = 32t + 1 + m of tile t (the "current" row) and row r + 32 of tile
// t + 1 (the "next" row).  A row's candidates split by the age of T[j]:
//   far   j <= 32(t-1)         helper warps, one tile ahead (warp argmin)
//   mid   32(t-1) < j < 32t    main warp, pushed into the "next" row while
//                              the previous tile's chain runs
//   near  32t <= j < r         main warp, the serial in-tile chain
// Every push visits k strictly decreasing, and `cand <= acc` makes the
// smallest k win ties; far is merged under the same rule (mid wins ties).
// The result is exactly the reference's ascending-k scan with strict `<`.
//
// Helper warps (warp % 4 != 0, so the main warp owns SMSP 0) run a software
// pipeline: row metadata 3 tiles ahead, the 32 x 64 cost block c(L_r, 1..64)
// 2 tiles ahead, far candidates 1 tile ahead.  The main warp touches only
// shared memory and registers.
//
// kIntCmp: when every cost is a non-negative double (no sign bit), so is
// every T and every candidate, and the order of the values equals the order
// of their bit patterns read as int64 — an exact, cheaper comparison on the
// chain than DSETP.
#pragma once

#include "scls_common.cuh"

namespace scls {

#ifndef SCLS_DPC_PAIR
#define SCLS_DPC_PAIR 1  // the in-tile chain takes two steps per broadcast
#endif

constexpr int kDpThreads = 512;
constexpr int kDpRing = 4096;   // ring of recent T values
constexpr int kDpStageK = 64;   // staged costs per row (mid+near need k <= 63)
constexpr int kDpHelpers = kDpThreads / 32 - kDpThreads / 128;  // 12
constexpr int kDpHelperThreads = kDpHelpers * 32;

struct DpSmem {
  double ring[kDpRing];              // 32 KB
  double cs[3][kDpStageK][32];       // 48 KB, [buf][k-1][lane]
  double Fv[2][32];
  int32_t Fk[2][32];
  int32_t W[4][32];
  int32_t CB[4][32];
};

template <bool kIntCmp>
__device__ __forceinline__ bool le(double a, double b) {
  if (kIntCmp) return __double_as_longlong(a) <= __double_as_longlong(b);
  return a <= b;
}

template <bool kGlobalT, bool kIntCmp>
__global__ void __launch_bounds__(kDpThreads, 1)
    dp_chain_kernel(int32_t n, const int32_t* __restrict__ Krow, const int32_t* __restrict__ cbase,
                    const double* __restrict__ cost, double* __restrict__ T,
                    int32_t* __restrict__ split, unsigned long long* __restrict__ prof,
                    const int32_t* __restrict__ gate = nullptr, int32_t gate_id = 0) {
  // small-pool launches (small.cu) start both DP kernels; the one the device
  // chose runs, the other returns
  if (gate && *gate != gate_id) return;
  extern __shared__ __align__(16) unsigned char dp_smem_raw[];
  DpSmem& sm = *reinterpret_cast<DpSmem*>(dp_smem_raw);
  constexpr int M = kDpRing - 1;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool helper = (warp & 3) != 0;
  const int h = warp - 1 - (warp >> 2);  // helper index 0..11
  const int ht = h * 32 + lane;          // helper thread index 0..383
  const int ntiles = (n + 31) >> 5;

  // Helper pipeline stages, each for one tile u.
  auto load_meta = [&](int u) {
    if (h == 0 && u < ntiles) {
      const int r = (u << 5) + 1 + lane;
      sm.W[u & 3][lane] = r <= n ? Krow[r - 1] : 0;
      sm.CB[u & 3][lane] = r <= n ? cbase[r - 1] : 0;
    }
  };
  auto stage_costs = [&](int u) {
    // c(L_r, k) for k = 1..64; +INF where k > W_r, so the main warp can take
    // every candidate unconditionally (a row's k = 1 candidate is always
    // finite and comes last, so an INF never survives).
    if (u >= ntiles) return;
    const int b = u % 3;
    constexpr int kPer = (32 * kDpStageK + kDpHelperThreads - 1) / kDpHelperThreads;
    double v[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = ht + i * kDpHelperThreads;
      v[i] = kInf;
      if (e < 32 * kDpStageK) {
        const int m = e & 31, k = 1 + (e >> 5);
        if (k <= sm.W[u & 3][m]) v[i] = cost[sm.CB[u & 3][m] + k];
      }
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = ht + i * kDpHelperThreads;
      if (e < 32 * kDpStageK) sm.cs[b][e >> 5][e & 31] = v[i];
    }
  };
  auto far = [&](int u) {  // far candidates of tile u: j <= 32(u-1)
    if (u >= ntiles) return;
    const int jmax = (u - 1) << 5;
    for (int m = h; m < 32; m += kDpHelpers) {
      const int r = (u << 5) + 1 + m;
      const int W = sm.W[u & 3][m];
      const int cb = sm.CB[u & 3][m];
      double best = kInf;
      int bk = 0;
      if (r - jmax > W) {  // no far candidates for this row (uniform)
        if (lane == 0) {
          sm.Fv[u & 1][m] = kInf;
          sm.Fk[u & 1][m] = 0;
        }
        continue;
      }
      int k = r - jmax + lane;
#pragma unroll 4
      for (; k <= W; k += 32) {
        const int j = r - k;
        const double tv = kGlobalT ? T[j] : sm.ring[j & M];
        const double cand = __dadd_rn(tv, cost[cb + k]);
        if (cand < best) {  // lane-local k ascending: strict < keeps the smallest k
          best = cand;
          bk = k;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
        if (ov < best || (ov == best && ok < bk)) {
          best = ov;
          bk = ok;
        }
      }
      if (lane == 0) {
        sm.Fv[u & 1][m] = best;
        sm.Fk[u & 1][m] = bk;
      }
    }
  };

  if (tid == 0) {
    sm.ring[0] = 0.0;
    T[0] = 0.0;
    split[0] = 0;
  }
  // Prologue: metadata for tiles 0..2, costs for tiles 0..1, far for tile 0
  // (empty: every k would reach below row 0).
  if (helper) {
    load_meta(0);
    load_meta(1);
    load_meta(2);
  }
  __syncthreads();
  if (helper) {
    stage_costs(0);
    stage_costs(1);
    for (int m = ht; m < 32; m += kDpHelperThreads) {
      sm.Fv[0][m] = kInf;
      sm.Fk[0][m] = 0;
    }
  }
  __syncthreads();

  // Main-warp registers: the next tile's accumulator (mid candidates).
  double accN = kInf;
  int kbN = 0;
  double Tlast = 0.0;  // T[32t], the last value of the previous tile
  // Phase counters (prof != nullptr): cycles in [0] main chain, [1] main
  // barrier wait, [2] helper meta+staging, [3] helper far, [4] helper wait.
  long long c_a = 0, c_b = 0, c_c = 0, c_d = 0, c_e = 0;
  for (int t = 0; t < ntiles; ++t) {
    const int tB = t << 5;
    const long long t0 = prof ? clock64() : 0;
    long long t1 = t0, t2 = t0;
    if (warp == 0) {
      const int cb = t % 3, nb = (t + 1) % 3;
      const int Wr = sm.W[t & 3][lane];
      const int WrN = sm.W[(t + 1) & 3][lane];
      // merge: far (larger k) then mid (accN) — mid wins ties.
      double acc = sm.Fv[t & 1][lane];
      int kb = sm.Fk[t & 1][lane];
      if (le<kIntCmp>(accN, acc)) {
        acc = accN;
        kb = kbN;
      }
      accN = kInf;
      kbN = 0;
      // near-chain costs for the current rows: step s uses k = lane + 1 - s
      // (+INF when k < 1; staged +INF when k > W).
      double cn[32];
#pragma unroll
      for (int s = 0; s < 32; ++s) cn[s] = (s <= lane) ? sm.cs[cb][lane - s][lane] : kInf;
      // next-tile costs, step s >= 1 uses k2 = 33 + lane - s; prefetched
      // kAhead steps early so no shared-memory latency sits in a step.
      constexpr int kAhead = 8;
      double c2[33];
#pragma unroll
      for (int s = 1; s <= kAhead; ++s) c2[s] = sm.cs[nb][32 + lane - s][lane];
      double Tj = Tlast;
#if SCLS_DPC_PAIR
      // Two steps per broadcast: T[tB+s+1] is lane s's acc after its k = 1
      // candidate at step s -- every lane forms it from lane s's (acc before
      // step s, c(L, 1)), shuffled a pair ahead, with the same operands and
      // the same accept as lane s, so step s+1 needs no broadcast.
      const double c1own = sm.cs[cb][0][lane];
      double Ab = __shfl_sync(0xffffffffu, acc, 0), c1b = __shfl_sync(0xffffffffu, c1own, 0);
#pragma unroll
      for (int s = 0; s < 32; s += 2) {
        if (s + kAhead <= 31 && s + kAhead >= 1) c2[s + kAhead] = sm.cs[nb][32 + lane - s - kAhead][lane];
        if (s + 1 + kAhead <= 31) c2[s + 1 + kAhead] = sm.cs[nb][32 + lane - s - 1 - kAhead][lane];
        const double t1 = __dadd_rn(Tj, c1b);
        const double Tn = le<kIntCmp>(t1, Ab) ? t1 : Ab;  // T[tB+s+1]
        // step s: T[tB+s], k = lane+1-s; the next-tile row with k2 = 33+lane-s
        const double cand = __dadd_rn(Tj, cn[s]);
        const bool take = le<kIntCmp>(cand, acc);
        acc = take ? cand : acc;
        kb = take ? lane + 1 - s : kb;
        if (s >= 1) {
          const double cand2 = __dadd_rn(Tj, c2[s]);
          const bool take2 = le<kIntCmp>(cand2, accN);
          accN = take2 ? cand2 : accN;
          kbN = take2 ? 33 + lane - s : kbN;
        }
        // step s+1: T[tB+s+1]
        const double candb = __dadd_rn(Tn, cn[s + 1]);
        const bool takeb = le<kIntCmp>(candb, acc);
        acc = takeb ? candb : acc;
        kb = takeb ? lane - s : kb;
        const double cand2b = __dadd_rn(Tn, c2[s + 1]);
        const bool take2b = le<kIntCmp>(cand2b, accN);
        accN = take2b ? cand2b : accN;
        kbN = take2b ? 32 + lane - s : kbN;
        Tj = __shfl_sync(0xffffffffu, acc, s + 1);
        if (s + 2 < 32) {
          Ab = __shfl_sync(0xffffffffu, acc, s + 2);
          c1b = __shfl_sync(0xffffffffu, c1own, s + 2);
        }
      }
#else
#pragma unroll
      for (int s = 0; s < 32; ++s) {
        if (s + kAhead <= 31 && s + kAhead >= 1) c2[s + kAhead] = sm.cs[nb][32 + lane - s - kAhead][lane];
        // current row r = tB+1+lane receives T[tB+s] with k = lane+1-s
        const double cand = __dadd_rn(Tj, cn[s]);
        const bool take = le<kIntCmp>(cand, acc);
        acc = take ? cand : acc;
        kb = take ? lane + 1 - s : kb;
        // next-tile row r+32 receives T[tB+s] (s >= 1) with k2 = 33+lane-s
        if (s >= 1) {
          const double cand2 = __dadd_rn(Tj, c2[s]);
          const bool take2 = le<kIntCmp>(cand2, accN);
          accN = take2 ? cand2 : accN;
          kbN = take2 ? 33 + lane - s : kbN;
        }
        Tj = __shfl_sync(0xffffffffu, acc, s);
      }
#endif
      // T[tB+32] reaches the next rows as step s = 0 of the next chain.
      Tlast = Tj;
      const int r = tB + 1 + lane;
      if (r <= n) {
        T[r] = acc;
        split[r] = r - kb;
        sm.ring[r & M] = acc;
      }
      t1 = t2 = prof ? clock64() : 0;
    } else if (helper) {
      load_meta(t + 3);
      stage_costs(t + 2);
      t1 = prof ? clock64() : 0;
      far(t + 1);
      t2 = prof ? clock64() : 0;
    }
    __syncthreads();
    if (prof) {
      const long long t3 = clock64();
      if (warp == 0) {
        c_a += t1 - t0;
        c_b += t3 - t1;
      } else if (helper) {
        c_c += t1 - t0;
        c_d += t2 - t1;
        c_e += t3 - t2;
      }
    }
  }
  if (prof && lane == 0) {
    if (warp == 0) {
      atomicAdd(&prof[0], (unsigned long long)c_a);
      atomicAdd(&prof[1], (unsigned long long)c_b);
    } else if (helper) {
      atomicAdd(&prof[2], (unsigned long long)c_c);
      atomicAdd(&prof[3], (unsigned long long)c_d);
      atomicAdd(&prof[4], (unsigned long long)c_e);
      atomicAdd(&prof[5], 1ull);
    }
  }
}

}  // namespace scls
