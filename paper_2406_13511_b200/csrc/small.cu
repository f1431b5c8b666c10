// small.cu — batch_requests (reference batcher.cpp:26-87) for pools of up to
// kSmallPool requests: the per-tick sizes of a live scheduler (SURVEY §8(a):
// pools of ~460 on average, 1.5k-30k at the extremes; bench_batcher.cpp
// sweeps 16..4096).  The multi-kernel path (batcher.cu) is built for 1M
// pools: ~150 launches and 4 host round trips, which at these sizes ARE the
// latency.  Here the whole call is four launches and one host read-back:
//
//   prep   one CTA: the order by (eff, arrival, id, position) in shared
//          memory (a bitonic network on three 64-bit words per member for
//          pools up to 1024, stable LSD radix passes above), then per sorted
//          row L, K(L) and singleton feasibility (batcher.cpp:40-46), the
//          runs of equal L, and the cost table c(L, k) per run
//          (cost_model.cpp:49-51); the DP kernel to use is decided on device
//   DP     dp_mono_kernel / dp_chain_kernel (both launched; the one the
//          device did not choose returns at once)
//   post   one CTA: the backtrack over split[] in shared memory
//          (batcher.cpp:69-73), batch emission (:75-86), member ids.
//
// Same results as the large path bit for bit: the same total order, the same
// tie rules, the same cost expressions (scls_common.cuh).
#include <algorithm>
#include <cmath>

#include "batcher.cuh"
#include "dp_chain.cuh"
#include "dp_mono.cuh"
#include "radix.cuh"
#include "scls_common.cuh"

extern "C" scls_status scls_validate_memory(const scls_memory* m);

namespace scls {

constexpr int kSmallPool = 4096;
constexpr int kSmallThreads = 1024;
constexpr int kSmallWarps = kSmallThreads / 32;

namespace {

// Device-side results the host reads once (one pinned copy).
struct SmallState {
  int32_t status;        // SCLS_OK / INFEASIBLE_REQUEST / CAPACITY
  int32_t gate;          // 1: monotone decision kernel, 0: chain kernel
  int32_t nb;
  int32_t k_max;
  int64_t err_request;
  int64_t cost_entries;
};

struct SmallSmem {
  uint64_t key[2][kSmallPool];
  int32_t perm[2][kSmallPool];
  int32_t cnt[kSmallWarps][256];  // per-warp digit counts, then scatter offsets
  int32_t tot[256];
  int32_t wsum[kSmallWarps];
  unsigned long long red[6];
  int32_t first_bad;
  int32_t kmax;
};

__device__ __forceinline__ uint64_t bias64(int64_t x) { return (uint64_t)x ^ 0x8000000000000000ull; }
__device__ __forceinline__ uint64_t bias32(int32_t x) { return (uint64_t)((uint32_t)x ^ 0x80000000u); }

// Block-wide exclusive scan of one int per thread (kSmallThreads threads).
__device__ int block_exclusive_scan(int v, int32_t* wsum, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(~0u, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = wsum[lane];
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(~0u, wi, o);
      if (lane >= o) wi += y;
    }
    wsum[lane] = wi - w;
    if (lane == 31) *total = wi;  // written through shared memory by the caller's pointer
  }
  __syncthreads();
  const int r = wsum[warp] + incl - v;
  __syncthreads();
  return r;
}

// One stable LSD pass on bits [shift, shift + 8) of key[src] (perm rides
// along) into key[src ^ 1].  Warp w owns positions [w*C, (w+1)*C); the
// element order (warp, iteration, lane) is the input order, so equal digits
// keep their order.
__device__ void block_radix_pass(SmallSmem& sm, int src, int n, int shift) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int C = (n + kSmallWarps - 1) / kSmallWarps;
  const int b0 = warp * C, b1 = min(n, b0 + C);
  for (int i = threadIdx.x; i < kSmallWarps * 256; i += kSmallThreads) (&sm.cnt[0][0])[i] = 0;
  __syncthreads();
  for (int p = b0 + lane; p < b1; p += 32) atomicAdd(&sm.cnt[warp][(sm.key[src][p] >> shift) & 0xff], 1);
  __syncthreads();
  // offsets: digit-major, warp-minor
  if (threadIdx.x < 256) {
    int s = 0;
    for (int w = 0; w < kSmallWarps; ++w) s += sm.cnt[w][threadIdx.x];
    sm.tot[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the 256 digit totals, 8 per lane
    int loc[8], s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      loc[q] = sm.tot[lane * 8 + q];
      s += loc[q];
    }
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(~0u, incl, o);
      if (lane >= o) incl += y;
    }
    int run = incl - s;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      sm.tot[lane * 8 + q] = run;
      run += loc[q];
    }
  }
  __syncthreads();
  if (threadIdx.x < 256) {
    int run = sm.tot[threadIdx.x];
    for (int w = 0; w < kSmallWarps; ++w) {
      const int c = sm.cnt[w][threadIdx.x];
      sm.cnt[w][threadIdx.x] = run;
      run += c;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int base = b0; base < b1; base += 32) {
    const int p = base + lane;
    const bool ok = p < b1;
    const uint64_t k = ok ? sm.key[src][p] : 0;
    const int32_t v = ok ? sm.perm[src][p] : 0;
    const int d = ok ? (int)((k >> shift) & 0xff) : 256 + lane;
    const unsigned peers = __match_any_sync(~0u, d);
    const int prior = ok ? sm.cnt[warp][d] : 0;
    __syncwarp();
    if (ok) {
      const int dst = prior + __popc(peers & lt);
      sm.key[src ^ 1][dst] = k;
      sm.perm[src ^ 1][dst] = v;
      if (lane == __ffs(peers) - 1) sm.cnt[warp][d] = prior + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSmallThreads, 1)
    small_prep_kernel(int32_t n, const int32_t* __restrict__ eff, const double* __restrict__ arr,
                      const int64_t* __restrict__ id, int32_t S, Lat lat, Mem mem, int32_t mono_ok,
                      int32_t force_mono, int64_t cost_cap, int32_t* __restrict__ perm_out,
                      int32_t* __restrict__ Krow, int32_t* __restrict__ cbase, double* __restrict__ cost,
                      int32_t* __restrict__ run_scratch, SmallState* __restrict__ st) {
  extern __shared__ __align__(16) unsigned char small_smem_raw[];
  SmallSmem& sm = *reinterpret_cast<SmallSmem*>(small_smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 6) sm.red[tid] = (tid & 1) ? 0ull : ~0ull;  // (min, max) x (id, arrival, eff)
  if (tid == 0) {
    sm.first_bad = 0x7fffffff;
    sm.kmax = 0;
    st->gate = -1;  // no DP kernel runs unless this call reaches the end
  }
  __syncthreads();
  // The order (eff, arrival, id), input position last: pools of up to
  // kSmallThreads by a bitonic network (few stages, no histogram rounds),
  // larger ones by the stable LSD passes.
  int src = 0;
  if (n <= kSmallThreads) {
    // a bitonic network in shared memory on three 64-bit words per member --
    //    A = eff | arrival[63:32], B = arrival[31:0] | id[63:32],
    //    C = id[31:0] | position -- compared lexicographically: 10 stages for
    //    16 members, where the LSD passes (up to 11, each a full 256-bin
    //    histogram round over 32 warps) cost 28 us; at 4096 members the
    //    network's 78 stages lose to them (measured 122 vs 94 us)
    uint64_t* const wa = sm.key[0];
    uint64_t* const wb = sm.key[1];
    uint64_t* const wc = reinterpret_cast<uint64_t*>(&sm.perm[0][0]);  // perm[2][kSmallPool] = kSmallPool words
    int P = 2;
    while (P < n) P <<= 1;
    for (int i = tid; i < P; i += kSmallThreads) {
      if (i < n) {
        const uint64_t a = ordered_bits(arr[i]), d = bias64(id[i]);
        wa[i] = bias32(eff[i]) << 32 | a >> 32;
        wb[i] = a << 32 | d >> 32;
        wc[i] = d << 32 | (uint64_t)(uint32_t)i;
      } else {
        wa[i] = wb[i] = wc[i] = ~0ull;
      }
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = tid; t < (P >> 1); t += kSmallThreads) {
          const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), h = i + j;  // j is a power of two
          const uint64_t a0 = wa[i], a1 = wa[h], b0 = wb[i], b1 = wb[h], c0 = wc[i], c1 = wc[h];
          const bool gt = a0 != a1 ? a0 > a1 : (b0 != b1 ? b0 > b1 : c0 > c1);
          if (gt == ((i & k) == 0)) {  // ascending blocks swap a greater first element
            wa[i] = a1;
            wa[h] = a0;
            wb[i] = b1;
            wb[h] = b0;
            wc[i] = c1;
            wc[h] = c0;
          }
        }
        __syncthreads();
      }
    }
    const int32_t pos = tid < n ? (int32_t)(uint32_t)wc[tid] : 0;  // n <= kSmallThreads here
    __syncthreads();
    if (tid < n) sm.perm[0][tid] = pos;
    __syncthreads();
  } else {
    // 1. key ranges (so that fields / bits that never vary cost no pass)
    {
      unsigned long long mn[3] = {~0ull, ~0ull, ~0ull}, mx[3] = {0, 0, 0};
      for (int i = tid; i < n; i += kSmallThreads) {
        const uint64_t f[3] = {bias64(id[i]), ordered_bits(arr[i]), bias32(eff[i])};
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          mn[q] = min(mn[q], (unsigned long long)f[q]);
          mx[q] = max(mx[q], (unsigned long long)f[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          mn[q] = min(mn[q], __shfl_xor_sync(~0u, mn[q], o));
          mx[q] = max(mx[q], __shfl_xor_sync(~0u, mx[q], o));
        }
        if (lane == 0) {
          atomicMin(&sm.red[2 * q], mn[q]);
          atomicMax(&sm.red[2 * q + 1], mx[q]);
        }
      }
    }
    __syncthreads();
    // 2. stable LSD sort, field by field from the least significant: id,
    //    arrival, eff (batcher.cpp:35-38 tuple order)
    for (int i = tid; i < n; i += kSmallThreads) sm.perm[0][i] = i;
    __syncthreads();
    for (int q = 0; q < 3; ++q) {
      const uint64_t lo = sm.red[2 * q], range = sm.red[2 * q + 1] - lo;
      const int bits = range ? 64 - __clzll((long long)range) : 0;
      if (bits == 0) continue;
      for (int p = tid; p < n; p += kSmallThreads) {
        const int i = sm.perm[src][p];
        const uint64_t f = q == 0 ? bias64(id[i]) : (q == 1 ? ordered_bits(arr[i]) : bias32(eff[i]));
        sm.key[src][p] = f - lo;
      }
      __syncthreads();
      for (int shift = 0; shift < bits; shift += 8) {
        block_radix_pass(sm, src, n, shift);
        src ^= 1;
      }
    }
  }
  // 3. rows: L, K(L) (memory_model.cpp:72-90), singleton feasibility, runs
  int32_t* flag_excl = run_scratch;                 // n
  int32_t* run_first = run_scratch + kSmallPool;    // n_runs
  int32_t* run_need = run_scratch + 2 * kSmallPool; // n_runs
  constexpr int kPer = kSmallPool / kSmallThreads;  // rows per thread, contiguous
  int L[kPer], K[kPer], fl[kPer];
  int kmax = 0, nfl = 0;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int p = tid * kPer + u;
    L[u] = K[u] = fl[u] = 0;
    if (p < n) {
      const int i = sm.perm[src][p];
      perm_out[p] = i;
      L[u] = eff[i];
      fl[u] = (p == 0 || eff[sm.perm[src][p - 1]] != L[u]) ? 1 : 0;
      if (would_oom(mem, 1, L[u], S)) {
        atomicMin(&sm.first_bad, p);
      } else {
        const int kk = max_batch_size(mem, L[u], S);
        K[u] = kk < p + 1 ? kk : p + 1;
        kmax = max(kmax, K[u]);
      }
      Krow[p] = K[u];
      nfl += fl[u];
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) kmax = max(kmax, __shfl_xor_sync(~0u, kmax, o));
  if (lane == 0) atomicMax(&sm.kmax, kmax);
  __shared__ int total;
  const int base = block_exclusive_scan(nfl, sm.wsum, &total);
  if (sm.first_bad != 0x7fffffff) {  // batcher.cpp:40-46: the first offender in sorted order
    if (tid == 0) {
      st->status = SCLS_ERR_INFEASIBLE_REQUEST;
      st->err_request = id[sm.perm[src][sm.first_bad]];
      st->nb = 0;
    }
    return;
  }
  const int n_runs = total;
  {  // run index per row; each run's first row and largest usable window
    int r = base - 1;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int p = tid * kPer + u;
      if (p < n) {
        r += fl[u];
        flag_excl[p] = r;
        if (fl[u]) run_first[r] = p;
        if (p == n - 1) run_need[r] = K[u];
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int p = tid * kPer + u;
    if (p < n - 1 && flag_excl[p + 1] != flag_excl[p]) run_need[flag_excl[p]] = K[u];
  }
  __syncthreads();
  // run offsets into the cost table (exclusive scan of run_need)
  int need[kPer], nsum = 0;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int r = tid * kPer + u;
    need[u] = r < n_runs ? run_need[r] : 0;
    nsum += need[u];
  }
  const int obase = block_exclusive_scan(nsum, sm.wsum, &total);
  int32_t* run_off = run_scratch + 3 * kSmallPool;
  {
    int o = obase;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int r = tid * kPer + u;
      if (r < n_runs) run_off[r] = o;
      o += need[u];
    }
  }
  if ((int64_t)total > cost_cap) {
    if (tid == 0) {
      st->status = SCLS_ERR_CAPACITY;
      st->nb = 0;
    }
    return;
  }
  __syncthreads();
  // 4. cost rows c(L, 1..need) per run (cost_model.cpp:49-51, hoisted sum_l)
  for (int r = warp; r < n_runs; r += kSmallWarps) {
    const int Lr = eff[sm.perm[src][run_first[r]]];
    const int nd = run_need[r], off = run_off[r];
    const double sum_l = decode_sum_l(Lr, S);
    for (int k = lane + 1; k <= nd; k += 32)
      cost[off + k - 1] = __dadd_rn(prefill_time(lat, k, Lr), decode_time_from_sum(lat, k, sum_l, S));
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int p = tid * kPer + u;
    if (p < n) cbase[p] = run_off[flag_excl[p]] - 1;
  }
  if (tid == 0) {
    st->status = SCLS_OK;
    st->k_max = sm.kmax;
    st->gate = mono_ok && (sm.kmax > 32 || force_mono) ? 1 : 0;
    st->cost_entries = total;
  }
}

// The backtrack (batcher.cpp:69-73) in shared memory, then the batches in
// ascending segment order (:75-86) and the member ids.
__global__ void __launch_bounds__(kSmallThreads, 1)
    small_post_kernel(int32_t n, const int32_t* __restrict__ split, const int32_t* __restrict__ perm,
                      const int32_t* __restrict__ eff, const int64_t* __restrict__ id, int32_t S, Lat lat,
                      int32_t* __restrict__ seg_begin, int32_t* __restrict__ l_in, double* __restrict__ est,
                      int32_t* __restrict__ order, int64_t* __restrict__ member, SmallState* __restrict__ st) {
  __shared__ int32_t ssplit[kSmallPool + 1];
  __shared__ int32_t ends[kSmallPool + 1];
  __shared__ int nb_s;
  if (st->status != SCLS_OK) return;
  const int tid = threadIdx.x;
  for (int r = tid; r <= n; r += kSmallThreads) ssplit[r] = split[r];
  __syncthreads();
  if (tid == 0) {  // segment ends from n back to 0 (reversed)
    int cnt = 0;
    for (int i = n; i > 0; i = ssplit[i]) ends[cnt++] = i;
    nb_s = cnt;
  }
  __syncthreads();
  const int nb = nb_s;
  for (int b = tid; b < nb; b += kSmallThreads) {
    const int end = ends[nb - 1 - b];
    const int beg = b == 0 ? 0 : ends[nb - b];
    const int L = eff[perm[end - 1]];
    seg_begin[b] = beg;
    l_in[b] = L;
    est[b] = batch_serve_time(lat, end - beg, L, S);
  }
  if (tid == 0) {
    seg_begin[nb] = n;
    st->nb = nb;
  }
  for (int p = tid; p < n; p += kSmallThreads) {
    const int i = perm[p];
    if (order) order[p] = i;
    if (member) member[p] = id[i];
  }
}

}  // namespace

bool small_pool_eligible(int64_t n) { return n > 0 && n <= kSmallPool; }

scls_status batch_requests_small(scls_ctx* ctx, const BatchInputs& in, const BatchOutputs& out, int64_t* nb_out) {
  cudaStream_t s = ctx->stream;
  const int32_t n = (int32_t)in.n;
  *nb_out = 0;
  const Lat lat = make_lat(*in.lat);
  const Mem mem = make_mem(*in.mem);
  const bool int_cmp = !std::signbit(in.lat->p1) && !std::signbit(in.lat->p2) && !std::signbit(in.lat->p3) &&
                       !std::signbit(in.lat->p4) && !std::signbit(in.lat->d1) && !std::signbit(in.lat->d2) &&
                       !std::signbit(in.lat->d3) && !std::signbit(in.lat->d4);
  const bool mono_ok = int_cmp && scls_validate_memory(in.mem) == SCLS_OK && ctx->dp_mode != 1;
  // cost table bound: every run needs at most min(K(L), n) entries, K(L) <= K(1)
  // for a valid memory model (windows shrink as L grows); else <= n
  int64_t kcap = n;
  if (scls_validate_memory(in.mem) == SCLS_OK) {
    if (in.mem->kind == SCLS_MEM_RULE_TABLE) {  // K(L) is some row's max_n
      int64_t m = 1;
      for (int i = 0; i < in.mem->n_rules; ++i) m = std::max<int64_t>(m, in.mem->rule_max_n[i]);
      kcap = std::min(kcap, m);
    } else {  // K(L) <= K(1) ~ zeta * avail / (delta * (1 + S)), plus the nudge
      const double q = std::floor(mem.zeta * mem.avail / (mem.delta * (1.0 + in.slice_len)));
      if (q >= 0.0 && q < 1e9) kcap = std::min<int64_t>(kcap, (int64_t)q + 64);
    }
  }
  const int64_t cost_cap = (int64_t)n * kcap;
  // scratch (slots of batcher.cu's range are free: this path replaces it)
  int32_t* perm = (int32_t*)ctx->buf(0, sizeof(int32_t) * n);
  int32_t* Krow = (int32_t*)ctx->buf(1, sizeof(int32_t) * n);
  int32_t* cbase = (int32_t*)ctx->buf(2, sizeof(int32_t) * n);
  double* cost = (double*)ctx->buf(3, sizeof(double) * (size_t)std::max<int64_t>(cost_cap, 1));
  int32_t* runs = (int32_t*)ctx->buf(4, sizeof(int32_t) * 4 * kSmallPool);
  double* T = (double*)ctx->buf(5, sizeof(double) * (n + 1));
  int32_t* split = (int32_t*)ctx->buf(6, sizeof(int32_t) * (n + 1));
  SmallState* dst = (SmallState*)ctx->buf(7, sizeof(SmallState));
  SmallState* hst = (SmallState*)ctx->host_pinned(sizeof(SmallState));
  if (!perm || !Krow || !cbase || !cost || !runs || !T || !split || !dst || !hst)
    return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  SCLS_CUDA(cudaEventRecord(ctx->ev[0], s));
  static bool attr_set = false;
  if (!attr_set) {
    SCLS_CUDA(cudaFuncSetAttribute(small_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sizeof(SmallSmem)));
    attr_set = true;
  }
  small_prep_kernel<<<1, kSmallThreads, sizeof(SmallSmem), s>>>(n, in.eff, in.arrival, in.id, in.slice_len, lat, mem,
                                                                 mono_ok ? 1 : 0, ctx->dp_mode == 2 ? 1 : 0, cost_cap,
                                                                 perm, Krow, cbase, cost, runs, dst);
  SCLS_LAUNCHED();
  SCLS_CUDA(cudaEventRecord(ctx->ev[1], s));
  SCLS_CUDA(cudaEventRecord(ctx->ev[2], s));
  // both DP kernels; the gate (device) lets one of them run
  const bool global_t = n + 64 > kDpRing;
  auto launch = [&](auto kern, size_t bytes, int32_t gate_id) -> scls_status {
    SCLS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    kern<<<1, kDpThreads, bytes, s>>>(n, Krow, cbase, cost, T, split, ctx->dp_prof, &dst->gate, gate_id);
    SCLS_LAUNCHED();
    return SCLS_OK;
  };
  scls_status stt = SCLS_OK;
  if (mono_ok)
    stt = global_t ? launch(dp_mono_kernel<true>, sizeof(DpMonoSmem), 1)
                   : launch(dp_mono_kernel<false>, sizeof(DpMonoSmem), 1);
  if (stt) return stt;
  if (global_t)
    stt = int_cmp ? launch(dp_chain_kernel<true, true>, sizeof(DpSmem), 0)
                  : launch(dp_chain_kernel<true, false>, sizeof(DpSmem), 0);
  else
    stt = int_cmp ? launch(dp_chain_kernel<false, true>, sizeof(DpSmem), 0)
                  : launch(dp_chain_kernel<false, false>, sizeof(DpSmem), 0);
  if (stt) return stt;
  SCLS_CUDA(cudaEventRecord(ctx->ev[3], s));
  small_post_kernel<<<1, kSmallThreads, 0, s>>>(n, split, perm, in.eff, in.id, in.slice_len, lat, out.seg_begin,
                                                 out.l_in, out.est, out.order, out.member_id, dst);
  SCLS_LAUNCHED();
  SCLS_CUDA(cudaEventRecord(ctx->ev[4], s));
  SCLS_CUDA(cudaMemcpyAsync(hst, dst, sizeof(SmallState), cudaMemcpyDeviceToHost, s));
  SCLS_CUDA(cudaStreamSynchronize(s));
  if (hst->status == SCLS_ERR_INFEASIBLE_REQUEST) {
    ctx->err_request = hst->err_request;
    return set_error(ctx, SCLS_ERR_INFEASIBLE_REQUEST,
                     "request " + std::to_string(hst->err_request) + " does not fit memory even as a singleton batch");
  }
  if (hst->status != SCLS_OK) return set_error(ctx, SCLS_ERR_CAPACITY, "small-pool cost table bound exceeded");
  ctx->dp_last_mono = hst->gate == 1;
  *nb_out = hst->nb;
  return SCLS_OK;
}

}  // namespace scls
