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

constexpr int kMonoSegs = kDpHelpers;  // 12 k-segments per row
#ifndef SCLS_DP_FAR_TOP
#define SCLS_DP_FAR_TOP 48
#endif
constexpr int kFarTop = SCLS_DP_FAR_TOP;  // far k's near the window, split finer

struct DpMonoSmem {
  double ring[kDpRing];          // 32 KB of recent T
  double cs[3][kDpStageK][32];   // 48 KB staged c(L_r, 1..64), +INF past W_r
  double Pv[2][kMonoSegs][32];   // far partial minima per segment
  int32_t Pk[2][kMonoSegs][32];
  double Fv[2][32];              // merged far minimum per row
  int32_t Fk[2][32];
  int32_t W[4][32];
  int32_t CB[4][32];
};

// (v, k) lexicographic "a before b": smaller value, ties to the smaller k.
__device__ __forceinline__ bool lex_lt(double va, int ka, double vb, int kb) {
  return va < vb || (va == vb && ka < kb);
}

template <bool kGlobalT>
__global__ void __launch_bounds__(kDpThreads, 1)
    dp_mono_kernel(int32_t n, const int32_t* __restrict__ Krow, const int32_t* __restrict__ cbase,
                   const double* __restrict__ cost, double* __restrict__ T, int32_t* __restrict__ split,
                   unsigned long long* __restrict__ prof, const int32_t* __restrict__ gate = nullptr,
                   int32_t gate_id = 0) {
  if (gate && *gate != gate_id) return;  // small-pool launches: the DP kernel the device did not choose
  extern __shared__ __align__(16) unsigned char dp_smem_raw[];
  DpMonoSmem& sm = *reinterpret_cast<DpMonoSmem*>(dp_smem_raw);
  constexpr int M = kDpRing - 1;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool helper = (warp & 3) != 0;
  const int h = warp - 1 - (warp >> 2);  // helper index 0..11
  const int ht = h * 32 + lane;
  const int ntiles = (n + 31) >> 5;

  auto load_meta = [&](int u) {
    if (h == 0 && u < ntiles) {
      const int r = (u << 5) + 1 + lane;
      sm.W[u & 3][lane] = r <= n ? Krow[r - 1] : 0;
      sm.CB[u & 3][lane] = r <= n ? cbase[r - 1] : 0;
    }
  };
  // Staging c(L_r, 1..64) of tile u: stage_load issues the global loads
  // into registers, stage_store writes them (+INF past W_r) to shared
  // memory — far() runs in between so the loads' latency is hidden.
  constexpr int kPer = (32 * kDpStageK + kDpHelperThreads - 1) / kDpHelperThreads;
  auto stage_load = [&](int u, double* v) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) v[i] = kInf;
    if (u >= ntiles) return;
    const int W = sm.W[u & 3][lane], CB = sm.CB[u & 3][lane];  // row m == lane for every i
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = ht + i * kDpHelperThreads;
      const int k = 1 + (e >> 5);
      if (e < 32 * kDpStageK && k <= W) v[i] = cost[CB + k];
    }
  };
  auto stage_store = [&](int u, const double* v) {
    if (u >= ntiles) return;
    const int b = u % 3;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = ht + i * kDpHelperThreads;
      if (e < 32 * kDpStageK) sm.cs[b][e >> 5][e & 31] = v[i];
    }
  };
  auto stage_costs = [&](int u) {
    double v[kPer];
    stage_load(u, v);
    stage_store(u, v);
  };
  // Far candidates of tile u (sources j <= 32(u-1)): helper h scans the h-th
  // k-segment of row m = lane, then (after a helper-only barrier) helper 0
  // merges the segments in ascending k.
  auto far = [&](int u) {
    if (u >= ntiles) return;
    const int jmax = (u - 1) << 5;
    const int r = (u << 5) + 1 + lane;
    const int W = sm.W[u & 3][lane];
    const int cb = sm.CB[u & 3][lane];
    const int kmin = r - jmax;
    const int span = W - kmin + 1;
    double best = kInf;
    int bk = 0;
    if (span > 0) {
      // Two tiers: the top kFarTop k's (the batch sizes near the window, where
      // the minimum of these monotone costs lives and pruning rarely holds)
      // in kMonoSegs/2 short segments, the rest in the other half (mostly
      // pruned by the bound below) -- the helpers' work evens out.
      constexpr int kHalf = kMonoSegs / 2;
      const int top = min(span, kFarTop);
      const int rest = span - top;
      int k0, k1;
      if (h < kHalf) {
        const int len = (rest + kHalf - 1) / kHalf;
        k0 = kmin + h * len;
        k1 = min(kmin + rest - 1, k0 + len - 1);
      } else {
        const int len = (top + kHalf - 1) / kHalf;
        k0 = kmin + rest + (h - kHalf) * len;
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
    sm.Pv[u & 1][h][lane] = best;
    sm.Pk[u & 1][h][lane] = bk;
    asm volatile("bar.sync 1, %0;" ::"n"(kDpHelperThreads));
    if (h == 0) {
      // merge the 12 segments (ascending k): all loads first, then a tree of
      // (value, k) lexicographic minima — ties go to the smaller k.
      double v[kMonoSegs];
      int k[kMonoSegs];
#pragma unroll
      for (int s2 = 0; s2 < kMonoSegs; ++s2) {
        v[s2] = sm.Pv[u & 1][s2][lane];
        k[s2] = sm.Pk[u & 1][s2][lane];
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
      sm.Fv[u & 1][lane] = v[0];
      sm.Fk[u & 1][lane] = k[0];
    }
  };

  if (tid == 0) {
    sm.ring[0] = 0.0;
    T[0] = 0.0;
    split[0] = 0;
  }
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

  long long c_a = 0, c_b = 0, c_c = 0, c_d = 0, c_e = 0, c_mid = 0, n_rounds = 0;
  for (int t = 0; t < ntiles; ++t) {
    const int tB = t << 5;
    const long long t0 = prof ? clock64() : 0;
    long long t1 = t0, t2 = t0;
    if (warp == 0) {
      const int cbuf = t % 3;
      const int r = tB + 1 + lane;
      // mid: sources j = tB-31 .. tB (k = lane+32-jj), 4 interleaved chains
      double va[8] = {kInf, kInf, kInf, kInf, kInf, kInf, kInf, kInf};
      int ka[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double tv[8], cv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int jj = c * 8 + i;
          tv[i] = sm.ring[(tB - 31 + jj) & M];
          cv[i] = sm.cs[cbuf][lane + 31 - jj][lane];
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
      double acc = sm.Fv[t & 1][lane];
      int kb = sm.Fk[t & 1][lane];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (lex_lt(va[q], ka[q], acc, kb)) {
          acc = va[q];
          kb = ka[q];
        }
      // rounds
      if (prof) c_mid += clock64() - t0;
      const double c1 = sm.cs[cbuf][0][lane];
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
            cv[q] = sm.cs[cbuf][k >= 1 ? k - 1 : 0][lane];
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
        T[r] = acc;
        split[r] = r - kb;
        sm.ring[r & M] = acc;
      }
      t1 = t2 = prof ? clock64() : 0;
    } else if (helper) {
      load_meta(t + 3);
      double sv[kPer];
      stage_load(t + 2, sv);
      t1 = prof ? clock64() : 0;
      far(t + 1);
      stage_store(t + 2, sv);
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
      atomicAdd(&prof[6], (unsigned long long)c_mid);
      atomicAdd(&prof[7], (unsigned long long)n_rounds);
    } else if (helper) {
      atomicAdd(&prof[2], (unsigned long long)c_c);
      atomicAdd(&prof[3], (unsigned long long)c_d);
      atomicAdd(&prof[4], (unsigned long long)c_e);
      atomicAdd(&prof[5], 1ull);
    }
  }
}

}  // namespace scls
