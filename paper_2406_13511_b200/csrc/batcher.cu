// batcher.cu — device batch_requests (reference batcher.cpp:26-87, Alg. 1 /
// Eq. 10), bit-exact.
//
// Phases (all on the context stream):
//   1. key analysis     min/max of eff, id and arrival bits (one pass)
//   2. pool ordering    stable LSD radix sort, field by field from least to
//                       most significant: id, arrival, eff — the reference's
//                       tuple order (batcher.cpp:35-38); fields whose range is
//                       a single value cost no pass
//   3. windows + costs  per sorted row: L = eff, K = would_oom boundary
//                       (memory_model.cpp:61-90); per distinct L ("run") the
//                       cost row c(L,k) = batch_serve_time(k, L, S) for every k
//                       a row of that run can use (cost_model.cpp:49-51)
//   4. DP chain         dp_chain_kernel: T[r] = min_k T[r-k] + c(L_r, k) with
//                       the reference's smallest-k tie rule
//   5. backtrack        pointer doubling over split[] marks the segment ends
//                       on the path from n (batcher.cpp:69-73), then compaction
//   6. emit             l_in = last member's eff, est = c(l_in, size)
#include <algorithm>
#include <cmath>
#include <cstring>

#include "batcher.cuh"
#include "radix.cuh"
#include "dp_chain.cuh"
#include "dp_mono.cuh"
#include "scls_common.cuh"

extern "C" scls_status scls_validate_memory(const scls_memory* m);

namespace scls {
namespace {

enum : int {
  kSlotKeys = 0, kSlotVals, kSlotKeysAlt, kSlotValsAlt, kSlotStats, kSlotLrow, kSlotKrow,
  kSlotFlag, kSlotRunIdx, kSlotRunFirst, kSlotRunNeed, kSlotRunOff, kSlotCost, kSlotT,
  kSlotSplit, kSlotJump, kSlotMark, kSlotMarkScan,
};

// ---- 1. key analysis --------------------------------------------------------

struct KeyStats {
  unsigned long long eff_min, eff_max;  // biased int32
  unsigned long long id_min, id_max;    // biased int64
  unsigned long long arr_min, arr_max;  // ordered_bits
  // second round (after sort)
  int first_infeasible;                 // sorted position, INT_MAX if none
  int k_max;                            // max window over rows
  int n_runs;
  int bucket_overflow;                  // the eff-bucket sort met a bucket above kBucketCap
  long long cost_entries;
};

__device__ __forceinline__ uint64_t bias64(int64_t x) { return (uint64_t)x ^ 0x8000000000000000ull; }
__device__ __forceinline__ uint64_t bias32(int32_t x) { return (uint64_t)((uint32_t)x ^ 0x80000000u); }

__global__ void key_stats_kernel(int64_t n, const int32_t* __restrict__ eff,
                                 const int64_t* __restrict__ id, const double* __restrict__ arr,
                                 KeyStats* st) {
  uint64_t emn = ~0ull, emx = 0, imn = ~0ull, imx = 0, amn = ~0ull, amx = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t e = bias32(eff[i]), d = bias64(id[i]), a = ordered_bits(arr[i]);
    emn = min(emn, e); emx = max(emx, e);
    imn = min(imn, d); imx = max(imx, d);
    amn = min(amn, a); amx = max(amx, a);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    emn = min(emn, __shfl_xor_sync(~0u, emn, o)); emx = max(emx, __shfl_xor_sync(~0u, emx, o));
    imn = min(imn, __shfl_xor_sync(~0u, imn, o)); imx = max(imx, __shfl_xor_sync(~0u, imx, o));
    amn = min(amn, __shfl_xor_sync(~0u, amn, o)); amx = max(amx, __shfl_xor_sync(~0u, amx, o));
  }
  // one set of atomics per block (per-warp atomics on six addresses contend)
  __shared__ uint64_t red[6][32];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = emn; red[1][w] = emx; red[2][w] = imn; red[3][w] = imx; red[4][w] = amn; red[5][w] = amx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < nw; ++q) {
      emn = min(emn, red[0][q]); emx = max(emx, red[1][q]);
      imn = min(imn, red[2][q]); imx = max(imx, red[3][q]);
      amn = min(amn, red[4][q]); amx = max(amx, red[5][q]);
    }
    atomicMin(&st->eff_min, emn); atomicMax(&st->eff_max, emx);
    atomicMin(&st->id_min, imn); atomicMax(&st->id_max, imx);
    atomicMin(&st->arr_min, amn); atomicMax(&st->arr_max, amx);
  }
}

__global__ void init_stats_kernel(KeyStats* st) {
  st->eff_min = st->id_min = st->arr_min = ~0ull;
  st->eff_max = st->id_max = st->arr_max = 0;
  st->first_infeasible = 0x7fffffff;
  st->k_max = 0;
  st->n_runs = 0;
  st->bucket_overflow = 0;
  st->cost_entries = 0;
}

// ---- 2. field keys -------------------------------------------------------------

enum Field { kFieldId, kFieldArrival, kFieldEff };

template <Field F>
__global__ void gather_key_kernel(int64_t n, const int32_t* __restrict__ vals,
                                  const int32_t* __restrict__ eff, const int64_t* __restrict__ id,
                                  const double* __restrict__ arr, uint64_t base,
                                  uint64_t* __restrict__ keys, bool identity,
                                  int32_t* __restrict__ vals_out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int32_t i = identity ? (int32_t)p : vals[p];
  if (identity) vals_out[p] = (int32_t)p;
  uint64_t k;
  if (F == kFieldId) k = bias64(id[i]);
  else if (F == kFieldArrival) k = ordered_bits(arr[i]);
  else k = bias32(eff[i]);
  keys[p] = k - base;
}

// ---- 3. rows, windows, runs, costs -------------------------------------------------

__global__ void rows_kernel(int64_t n, const int32_t* __restrict__ perm,
                            const int32_t* __restrict__ eff, int32_t slice, Mem mem,
                            int32_t* __restrict__ Lrow, int32_t* __restrict__ Krow,
                            int32_t* __restrict__ flag, KeyStats* st) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int kmax = 0;
  const int32_t L = p < n ? eff[perm[p]] : 0;
  if (p < n) {
    Lrow[p] = L;
    // batcher.cpp:40-46: singleton feasibility; first offender in sorted order.
    if (would_oom(mem, 1, L, slice)) {
      atomicMin(&st->first_infeasible, (int)p);
      Krow[p] = 0;
    } else {
      // batcher.cpp:58-59 extends k while !would_oom(k, L, S); would_oom is
      // monotone in n, so the scan stops exactly at max_batch_size (Eq. 8).
      const int K = max_batch_size(mem, L, slice);
      const int64_t row = p + 1;
      Krow[p] = (int32_t)(K < row ? K : row);
      kmax = Krow[p];
    }
  }
  // the previous row's L from the neighbouring lane (lane 0 gathers it)
  int32_t Lp = __shfl_up_sync(~0u, L, 1);
  if ((threadIdx.x & 31) == 0 && p > 0 && p < n) Lp = eff[perm[p - 1]];
  if (p < n) flag[p] = (p == 0 || Lp != L) ? 1 : 0;
  // k_max: one atomic per block (per-warp atomics on one address serialise)
  __shared__ int32_t wmax[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) kmax = max(kmax, __shfl_xor_sync(~0u, kmax, o));
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = kmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) kmax = max(kmax, wmax[w]);
    if (kmax) atomicMax(&st->k_max, kmax);
  }
}

// For each run (maximal block of equal L): first sorted position and the
// largest k any of its rows can use: max over rows of min(K, row) = the
// last row's window (K is constant over a run, rows grow).
__global__ void runs_kernel(int64_t n, const int32_t* __restrict__ flag,
                            const int32_t* run_excl, const int32_t* __restrict__ Krow,
                            int32_t* run_of_row, int32_t* __restrict__ run_first,
                            int32_t* __restrict__ run_need) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int32_t run = run_excl[p] + flag[p] - 1;
  run_of_row[p] = run;
  if (flag[p]) run_first[run] = (int32_t)p;
  if (p == n - 1 || flag[p + 1]) run_need[run] = Krow[p];
}

__global__ void row_cbase_kernel(int64_t n, const int32_t* __restrict__ run_of_row,
                                 const int32_t* __restrict__ run_off, int32_t* __restrict__ cbase) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) cbase[p] = run_off[run_of_row[p]] - 1;
}

__global__ void cost_table_kernel(int32_t n_runs, const int32_t* __restrict__ run_first,
                                  const int32_t* __restrict__ run_need,
                                  const int32_t* __restrict__ run_off,
                                  const int32_t* __restrict__ Lrow, int32_t slice, Lat lat,
                                  double* __restrict__ cost) {
  for (int run = blockIdx.x; run < n_runs; run += gridDim.x) {
    const int L = Lrow[run_first[run]];
    const int need = run_need[run];
    const int off = run_off[run];
    const double sum_l = decode_sum_l(L, slice);
    for (int k = threadIdx.x + 1; k <= need; k += blockDim.x) {
      // batch_serve_time(k, L, S) == prefill + decode with the hoisted sum_l.
      cost[off + k - 1] = __dadd_rn(prefill_time(lat, k, L),
                                    decode_time_from_sum(lat, k, sum_l, slice));
    }
  }
}

// ---- 5. backtrack by pointer doubling --------------------------------------------

__global__ void jump_kernel(int32_t n, const int32_t* __restrict__ prev, int32_t* __restrict__ next) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r <= n) next[r] = prev[prev[r]];
}

__global__ void mark_init_kernel(int32_t n, int32_t* __restrict__ mark) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r <= n) mark[r] = (r == n) ? 1 : 0;
}

__global__ void mark_kernel(int32_t n, const int32_t* __restrict__ jump, int32_t* __restrict__ mark) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r <= n && mark[r]) mark[jump[r]] = 1;
}

__global__ void compact_kernel(int32_t n, const int32_t* __restrict__ mark,
                               const int32_t* __restrict__ pos, int32_t* __restrict__ seg) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n && mark[r]) seg[pos[r]] = r;
  if (r == n) seg[pos[n - 1] + mark[n - 1]] = n;
}

// ---- 6. emit --------------------------------------------------------------------------

__global__ void emit_batches_kernel(int32_t nb, const int32_t* __restrict__ seg,
                                    const int32_t* __restrict__ Lrow, int32_t slice, Lat lat,
                                    int32_t* __restrict__ l_in, double* __restrict__ est) {
  const int32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int32_t beg = seg[b], end = seg[b + 1];
  const int32_t L = Lrow[end - 1];
  l_in[b] = L;
  est[b] = batch_serve_time(lat, end - beg, L, slice);
}

__global__ void emit_members_kernel(int64_t n, const int32_t* __restrict__ perm,
                                    const int64_t* __restrict__ id, int32_t* __restrict__ order,
                                    int64_t* __restrict__ member) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int32_t i = perm[p];
  if (order) order[p] = i;
  if (member) member[p] = id[i];
}

}  // namespace

scls_status batch_requests_device(scls_ctx* ctx, const BatchInputs& in, const BatchOutputs& out,
                                  int64_t* nb_out, BatchTrace* trace) {
  cudaStream_t s = ctx->stream;
  const int64_t n = in.n;
  *nb_out = 0;
  if (n == 0) return SCLS_OK;
  if (n >= 0x7fffffffLL) return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "pool larger than 2^31-1");
  if (small_pool_eligible(n) && !trace && !ctx->force_large_path) return batch_requests_small(ctx, in, out, nb_out);
  const Lat lat = make_lat(*in.lat);
  const Mem mem = make_mem(*in.mem);
  const int threads = 256;
  const int grid_n = div_up(n, threads);

  // ---- 1. key analysis
  KeyStats* st = (KeyStats*)ctx->buf(kSlotStats, sizeof(KeyStats));
  KeyStats* hst = (KeyStats*)ctx->host_pinned(sizeof(KeyStats));
  if (!st || !hst) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  SCLS_CUDA(cudaEventRecord(ctx->ev[0], s));
  init_stats_kernel<<<1, 1, 0, s>>>(st);
  SCLS_LAUNCHED();
  key_stats_kernel<<<std::min(grid_n, ctx->sm_count * 8), threads, 0, s>>>(n, in.eff, in.id,
                                                                           in.arrival, st);
  SCLS_LAUNCHED();
  // The key ranges reach the host only when the LSD sort needs them (forced,
  // or after an eff-bucket overflow): the bucket sort plans on the device.
  KeyStats ks{};

  // ---- 2. sort by (eff, arrival, id): eff buckets sorted in shared memory,
  //         or the stable LSD radix sort field by field
  uint64_t* keys = (uint64_t*)ctx->buf(kSlotKeys, sizeof(uint64_t) * n);
  uint64_t* keys2 = (uint64_t*)ctx->buf(kSlotKeysAlt, sizeof(uint64_t) * n);
  int32_t* vals = (int32_t*)ctx->buf(kSlotVals, sizeof(int32_t) * n);
  int32_t* vals2 = (int32_t*)ctx->buf(kSlotValsAlt, sizeof(int32_t) * n);
  if (!keys || !keys2 || !vals || !vals2) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  auto lsd_sort = [&]() -> scls_status {
    bool identity = true;
    struct FieldPlan {
      Field f;
      uint64_t lo, hi;
    } plan[3] = {{kFieldId, ks.id_min, ks.id_max},
                 {kFieldArrival, ks.arr_min, ks.arr_max},
                 {kFieldEff, ks.eff_min, ks.eff_max}};
    for (const FieldPlan& fp : plan) {
      const int bits = bit_width(fp.hi - fp.lo);
      if (bits == 0) continue;
      switch (fp.f) {
        case kFieldId:
          gather_key_kernel<kFieldId><<<grid_n, threads, 0, s>>>(n, vals, in.eff, in.id, in.arrival,
                                                                 fp.lo, keys, identity, vals);
          break;
        case kFieldArrival:
          gather_key_kernel<kFieldArrival><<<grid_n, threads, 0, s>>>(n, vals, in.eff, in.id,
                                                                      in.arrival, fp.lo, keys,
                                                                      identity, vals);
          break;
        default:
          gather_key_kernel<kFieldEff><<<grid_n, threads, 0, s>>>(n, vals, in.eff, in.id, in.arrival,
                                                                  fp.lo, keys, identity, vals);
          break;
      }
      SCLS_LAUNCHED();
      identity = false;
      bool swapped = false;
      scls_status stt = radix_sort_pairs(ctx, n, keys, vals, keys2, vals2, 0, bits, &swapped);
      if (stt) return stt;
      if (swapped) {
        std::swap(keys, keys2);
        std::swap(vals, vals2);
      }
    }
    if (identity) {
      // Every key field constant: the order is the input order.
      gather_key_kernel<kFieldEff><<<grid_n, threads, 0, s>>>(n, vals, in.eff, in.id, in.arrival, 0,
                                                              keys, true, vals);
      SCLS_LAUNCHED();
    }
    return SCLS_OK;
  };
  // eff buckets unless forced off; a pool they do not fit (eff range, average
  // or largest bucket) sets bucket_overflow on the device and is re-sorted by
  // the LSD path after the rows pass's read-back, below
  const bool bucketed = !ctx->force_lsd_sort;
  if (bucketed) {
    scls_status stt0 = bucket_sort_perm(ctx, n, in.eff, in.arrival, in.id, &st->eff_min, vals,
                                        &st->bucket_overflow);
    if (stt0) return stt0;
  } else {
    SCLS_CUDA(cudaMemcpyAsync(hst, st, sizeof(KeyStats), cudaMemcpyDeviceToHost, s));
    SCLS_CUDA(cudaStreamSynchronize(s));
    ks = *hst;
    scls_status stt0 = lsd_sort();
    if (stt0) return stt0;
  }
  const int32_t* perm = vals;
  SCLS_CUDA(cudaEventRecord(ctx->ev[1], s));

  // ---- 3. rows, windows, runs, cost table
  int32_t* Lrow = (int32_t*)ctx->buf(kSlotLrow, sizeof(int32_t) * n);
  int32_t* Krow = (int32_t*)ctx->buf(kSlotKrow, sizeof(int32_t) * n);
  int32_t* flag = (int32_t*)ctx->buf(kSlotFlag, sizeof(int32_t) * n);
  int32_t* run_excl = (int32_t*)ctx->buf(kSlotRunIdx, sizeof(int32_t) * n);
  if (!Lrow || !Krow || !flag || !run_excl) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  auto rows_pass = [&]() -> scls_status {
    rows_kernel<<<grid_n, threads, 0, s>>>(n, perm, in.eff, in.slice_len, mem, Lrow, Krow, flag, st);
    SCLS_LAUNCHED();
    scls_status st2 = scan_exclusive(ctx, n, flag, run_excl, &st->n_runs);
    if (st2) return st2;
    SCLS_CUDA(cudaMemcpyAsync(hst, st, sizeof(KeyStats), cudaMemcpyDeviceToHost, s));
    SCLS_CUDA(cudaStreamSynchronize(s));
    return SCLS_OK;
  };
  scls_status stt = rows_pass();
  if (stt) return stt;
  if (bucketed && hst->bucket_overflow) {
    // no eff buckets for this pool: redo the order with the LSD sort, on the
    // key ranges of the rows pass's read-back
    ks = *hst;
    init_stats_kernel<<<1, 1, 0, s>>>(st);
    SCLS_LAUNCHED();
    stt = lsd_sort();
    if (stt) return stt;
    perm = vals;
    stt = rows_pass();
    if (stt) return stt;
  }
  if (hst->first_infeasible != 0x7fffffff) {
    // batcher.cpp:40-46: InfeasibleRequestError for the first offender.
    int32_t idx = 0;
    int64_t rid = 0;
    SCLS_CUDA(cudaMemcpy(&idx, perm + hst->first_infeasible, sizeof idx, cudaMemcpyDeviceToHost));
    SCLS_CUDA(cudaMemcpy(&rid, in.id + idx, sizeof rid, cudaMemcpyDeviceToHost));
    ctx->err_request = rid;
    return set_error(ctx, SCLS_ERR_INFEASIBLE_REQUEST,
                     "request " + std::to_string(rid) +
                         " does not fit memory even as a singleton batch");
  }
  const int32_t n_runs = hst->n_runs;
  const int32_t k_max = hst->k_max;
  int32_t* run_first = (int32_t*)ctx->buf(kSlotRunFirst, sizeof(int32_t) * n_runs);
  int32_t* run_need = (int32_t*)ctx->buf(kSlotRunNeed, sizeof(int32_t) * n_runs);
  int32_t* run_off = (int32_t*)ctx->buf(kSlotRunOff, sizeof(int32_t) * (n_runs + 1));
  if (!run_first || !run_need || !run_off) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  // run index per row overwrites the exclusive scan in place (flag stays).
  runs_kernel<<<grid_n, threads, 0, s>>>(n, flag, run_excl, Krow, run_excl, run_first, run_need);
  SCLS_LAUNCHED();
  stt = scan_exclusive(ctx, n_runs, run_need, run_off, run_off + n_runs);
  if (stt) return stt;
  // Every run needs at most k_max entries: when n_runs * k_max is small the
  // table is sized by that bound and the exact total stays on the device
  // (no second host round trip); otherwise it is read back and checked.
  int64_t total_cost = (int64_t)n_runs * std::max(k_max, 1);
  if (total_cost > ((int64_t)1 << 24)) {
    SCLS_CUDA(cudaMemcpyAsync(&hst->first_infeasible, run_off + n_runs, sizeof(int32_t),
                              cudaMemcpyDeviceToHost, s));
    SCLS_CUDA(cudaStreamSynchronize(s));
    total_cost = hst->first_infeasible;
    if (total_cost < 0 || total_cost > (int64_t)1 << 28)
      return set_error(ctx, SCLS_ERR_CAPACITY, "candidate cost table exceeds 2^28 entries");
  }
  double* cost = (double*)ctx->buf(kSlotCost, sizeof(double) * (size_t)std::max<int64_t>(total_cost, 1));
  if (!cost) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  cost_table_kernel<<<std::min(n_runs, ctx->sm_count * 16), 128, 0, s>>>(
      n_runs, run_first, run_need, run_off, Lrow, in.slice_len, lat, cost);
  SCLS_LAUNCHED();
  SCLS_CUDA(cudaEventRecord(ctx->ev[2], s));

  // ---- 4. DP chain
  double* T = (double*)ctx->buf(kSlotT, sizeof(double) * (n + 1));
  int32_t* split = (int32_t*)ctx->buf(kSlotSplit, sizeof(int32_t) * (n + 1));
  if (!T || !split) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  // cost base per row (cost[cbase[p] + k] = c(L_p, k)), reusing the flag slot
  int32_t* cbase = flag;
  row_cbase_kernel<<<grid_n, threads, 0, s>>>(n, run_excl, run_off, cbase);
  SCLS_LAUNCHED();
  const size_t smem = sizeof(DpSmem);
  const bool global_t = k_max + 64 > kDpRing;
  const bool int_cmp = !std::signbit(in.lat->p1) && !std::signbit(in.lat->p2) && !std::signbit(in.lat->p3) &&
                       !std::signbit(in.lat->p4) && !std::signbit(in.lat->d1) && !std::signbit(in.lat->d2) &&
                       !std::signbit(in.lat->d3) && !std::signbit(in.lat->d4);
  auto launch = [&](auto kern, size_t bytes) -> scls_status {
    SCLS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    kern<<<1, kDpThreads, bytes, s>>>((int32_t)n, Krow, cbase, cost, T, split, ctx->dp_prof, nullptr, 0);
    SCLS_LAUNCHED();
    return SCLS_OK;
  };
  // Monotone cost model (dp_mono.cuh): non-negative coefficients and a valid
  // memory model make T provably non-decreasing -> exact decision rounds.
  // When every window fits in one tile (k_max <= 32, e.g. the rule-table
  // engines) the chain kernel's in-tile pushes beat the decision rounds.
  const bool monotone = int_cmp && scls_validate_memory(in.mem) == SCLS_OK && ctx->dp_mode != 1 &&
                        (k_max > 32 || ctx->dp_mode == 2);
  ctx->dp_last_mono = monotone;
  // A thread-block cluster spreads the far candidates over kC SMs
  // (dp_mono.cuh); SCLS_OPT_DP_CLUSTER picks kC (1 = one CTA).
  auto launch_cluster = [&](auto kern, int csize, size_t bytes) -> bool {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(kDpThreads);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, (int32_t)n, (const int32_t*)Krow, (const int32_t*)cbase, (const double*)cost, T,
                           split, ctx->dp_prof, (const int32_t*)nullptr, (int32_t)0) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    SCLS_LAUNCHED();
    return true;
  };
  if (monotone) {
    bool done = false;
    if (!global_t && ctx->dp_cluster == 4) done = launch_cluster(dp_mono_kernel<false, 4>, 4, sizeof(DpMonoSmemT<4>));
    if (!global_t && ctx->dp_cluster == 2) done = launch_cluster(dp_mono_kernel<false, 2>, 2, sizeof(DpMonoSmemT<2>));
    if (!done)
      stt = global_t ? launch(dp_mono_kernel<true>, sizeof(DpMonoSmem)) : launch(dp_mono_kernel<false>, sizeof(DpMonoSmem));
    ctx->dp_last_cluster = done ? ctx->dp_cluster : 1;
  } else if (global_t) {
    stt = int_cmp ? launch(dp_chain_kernel<true, true>, smem) : launch(dp_chain_kernel<true, false>, smem);
  } else {
    stt = int_cmp ? launch(dp_chain_kernel<false, true>, smem) : launch(dp_chain_kernel<false, false>, smem);
  }
  if (stt) return stt;
  SCLS_CUDA(cudaEventRecord(ctx->ev[3], s));

  // ---- 5. backtrack: mark the ancestors of n in the split forest
  int levels = 1;
  while (((int64_t)1 << levels) <= n) ++levels;
  int32_t* jump = (int32_t*)ctx->buf(kSlotJump, sizeof(int32_t) * (size_t)(n + 1) * levels);
  int32_t* mark = (int32_t*)ctx->buf(kSlotMark, sizeof(int32_t) * (n + 1));
  int32_t* mpos = (int32_t*)ctx->buf(kSlotMarkScan, sizeof(int32_t) * (n + 1));
  if (!jump || !mark || !mpos) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  const int grid_n1 = div_up(n + 1, threads);
  SCLS_CUDA(cudaMemcpyAsync(jump, split, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
  for (int l = 1; l < levels; ++l) {
    jump_kernel<<<grid_n1, threads, 0, s>>>((int32_t)n, jump + (size_t)(l - 1) * (n + 1),
                                            jump + (size_t)l * (n + 1));
    SCLS_LAUNCHED();
  }
  mark_init_kernel<<<grid_n1, threads, 0, s>>>((int32_t)n, mark);
  SCLS_LAUNCHED();
  for (int l = levels - 1; l >= 0; --l) {
    mark_kernel<<<grid_n1, threads, 0, s>>>((int32_t)n, jump + (size_t)l * (n + 1), mark);
    SCLS_LAUNCHED();
  }
  stt = scan_exclusive(ctx, n, mark, mpos, &st->n_runs);
  if (stt) return stt;
  compact_kernel<<<grid_n1, threads, 0, s>>>((int32_t)n, mark, mpos, out.seg_begin);
  SCLS_LAUNCHED();
  SCLS_CUDA(cudaMemcpyAsync(&hst->n_runs, &st->n_runs, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SCLS_CUDA(cudaStreamSynchronize(s));
  const int32_t nb = hst->n_runs;

  // ---- 6. emit
  emit_batches_kernel<<<div_up(nb, threads), threads, 0, s>>>(nb, out.seg_begin, Lrow,
                                                               in.slice_len, lat, out.l_in, out.est);
  SCLS_LAUNCHED();
  if (out.order || out.member_id) {
    emit_members_kernel<<<grid_n, threads, 0, s>>>(n, perm, in.id, out.order, out.member_id);
    SCLS_LAUNCHED();
  }
  SCLS_CUDA(cudaEventRecord(ctx->ev[4], s));
  *nb_out = nb;
  if (trace) {
    trace->T = T;
    trace->split = split;
    trace->Lrow = Lrow;
    trace->perm = perm;
    trace->k_max = k_max;
    trace->n_runs = n_runs;
    trace->cost_entries = total_cost;
  }
  return SCLS_OK;
}

}  // namespace scls
