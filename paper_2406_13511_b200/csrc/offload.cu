// offload.cu — max-min batch placement (reference offloader.cpp:25-59,
// Eq. 11) on device.
//
//   1. stable sort of batch indices by est_serve_time descending
//      (offloader.cpp:34-37): LSD radix on ~ordered_bits(est), ties keep
//      creation order because the sort is stable;
//   2. the greedy pass: each batch goes to the worker minimising
//      (load, worker_id) — the reference's scan (offloader.cpp:39-47) keeps
//      the first minimum, so the index breaks remaining ties — then that
//      load grows by the estimate.  The pass is a serial chain over batches;
//      it runs in one thread with the loads in registers and a log2(W)-deep
//      compare tree (W <= 8), or in one warp with a shuffle argmin (W <= 32),
//      or in one CTA (any W).
#include <algorithm>

#include "batcher.cuh"
#include "radix.cuh"
#include "scls_common.cuh"

namespace scls {
namespace {

enum : int { kSlotOKeys = 16, kSlotOVals, kSlotOKeysAlt, kSlotOValsAlt, kSlotORange };

__global__ void est_keys_kernel(int64_t nb, const double* __restrict__ est,
                                uint64_t* __restrict__ keys, int32_t* __restrict__ vals,
                                unsigned long long* range) {
  uint64_t mn = ~0ull, mx = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = ~ordered_bits(est[i]);  // descending
    keys[i] = k;
    vals[i] = (int32_t)i;
    mn = min(mn, k);
    mx = max(mx, k);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(~0u, mn, o));
    mx = max(mx, __shfl_xor_sync(~0u, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&range[0], mn);
    atomicMax(&range[1], mx);
  }
}

__global__ void sub_keys_kernel(int64_t nb, uint64_t* __restrict__ keys, const unsigned long long* range) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nb) keys[i] -= range[0];
}

__global__ void init_range_kernel(unsigned long long* range) {
  range[0] = ~0ull;
  range[1] = 0;
}

// (load, id, index) lexicographic "a before b" — the reference's selection.
__device__ __forceinline__ bool wins(double la, int ia, int xa, double lb, int ib, int xb) {
  return la < lb || (la == lb && (ia < ib || (ia == ib && xa < xb)));
}

template <int W>
__global__ void greedy_small_kernel(int64_t nb, const int32_t* __restrict__ order,
                                    const int64_t* __restrict__ batch_id,
                                    const double* __restrict__ est, int32_t nw,
                                    const int32_t* __restrict__ worker_id,
                                    double* __restrict__ load, int64_t* __restrict__ out_b,
                                    int32_t* __restrict__ out_w) {
  if (threadIdx.x != 0) return;
  double l[W];
  int id[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    l[w] = w < nw ? load[w] : __longlong_as_double(0x7ff0000000000000ll);
    id[w] = w < nw ? worker_id[w] : 0x7fffffff;
  }
  int32_t nxt = nb > 0 ? order[0] : 0;
  double e_nxt = nb > 0 ? est[nxt] : 0.0;
  for (int64_t k = 0; k < nb; ++k) {
    const int32_t cur = nxt;
    const double e = e_nxt;
    if (k + 1 < nb) {  // prefetch the next batch off the chain
      nxt = order[k + 1];
      e_nxt = est[nxt];
    }
    // Tournament over the W slots.
    double bl[W];
    int bi[W], bx[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      bl[w] = l[w];
      bi[w] = id[w];
      bx[w] = w;
    }
#pragma unroll
    for (int span = 1; span < W; span <<= 1) {
#pragma unroll
      for (int w = 0; w + span < W; w += 2 * span) {
        if (wins(bl[w + span], bi[w + span], bx[w + span], bl[w], bi[w], bx[w])) {
          bl[w] = bl[w + span];
          bi[w] = bi[w + span];
          bx[w] = bx[w + span];
        }
      }
    }
    const int t = bx[0];
#pragma unroll
    for (int w = 0; w < W; ++w)
      if (w == t) l[w] = __dadd_rn(l[w], e);
    out_b[k] = batch_id[cur];
    out_w[k] = bi[0];
  }
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (w < nw) load[w] = l[w];
}

__global__ void greedy_warp_kernel(int64_t nb, const int32_t* __restrict__ order,
                                   const int64_t* __restrict__ batch_id,
                                   const double* __restrict__ est, int32_t nw,
                                   const int32_t* __restrict__ worker_id,
                                   double* __restrict__ load, int64_t* __restrict__ out_b,
                                   int32_t* __restrict__ out_w) {
  const int lane = threadIdx.x;
  double l = lane < nw ? load[lane] : __longlong_as_double(0x7ff0000000000000ll);
  const int id = lane < nw ? worker_id[lane] : 0x7fffffff;
  for (int64_t k = 0; k < nb; ++k) {
    const int32_t cur = order[k];
    const double e = est[cur];
    double bl = l;
    int bi = id, bx = lane;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ol = __shfl_xor_sync(~0u, bl, o);
      const int oi = __shfl_xor_sync(~0u, bi, o);
      const int ox = __shfl_xor_sync(~0u, bx, o);
      if (wins(ol, oi, ox, bl, bi, bx)) {
        bl = ol;
        bi = oi;
        bx = ox;
      }
    }
    if (lane == bx) l = __dadd_rn(l, e);
    if (lane == 0) {
      out_b[k] = batch_id[cur];
      out_w[k] = bi;
    }
  }
  if (lane < nw) load[lane] = l;
}

// Any W: one CTA, loads in shared memory, block argmin per batch.
__global__ void greedy_block_kernel(int64_t nb, const int32_t* __restrict__ order,
                                    const int64_t* __restrict__ batch_id,
                                    const double* __restrict__ est, int32_t nw,
                                    const int32_t* __restrict__ worker_id,
                                    double* __restrict__ load, int64_t* __restrict__ out_b,
                                    int32_t* __restrict__ out_w) {
  __shared__ double sl[32];
  __shared__ int si[32], sx[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int64_t k = 0; k < nb; ++k) {
    double bl = __longlong_as_double(0x7ff0000000000000ll);
    int bi = 0x7fffffff, bx = 0x7fffffff;
    for (int w = tid; w < nw; w += blockDim.x) {
      const double lw = load[w];
      if (wins(lw, worker_id[w], w, bl, bi, bx)) {
        bl = lw;
        bi = worker_id[w];
        bx = w;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ol = __shfl_xor_sync(~0u, bl, o);
      const int oi = __shfl_xor_sync(~0u, bi, o);
      const int ox = __shfl_xor_sync(~0u, bx, o);
      if (wins(ol, oi, ox, bl, bi, bx)) {
        bl = ol;
        bi = oi;
        bx = ox;
      }
    }
    if (lane == 0) {
      sl[warp] = bl;
      si[warp] = bi;
      sx[warp] = bx;
    }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < nwarps; ++q)
        if (wins(sl[q], si[q], sx[q], sl[0], si[0], sx[0])) {
          sl[0] = sl[q];
          si[0] = si[q];
          sx[0] = sx[q];
        }
      const int32_t cur = order[k];
      load[sx[0]] = __dadd_rn(load[sx[0]], est[cur]);
      out_b[k] = batch_id[cur];
      out_w[k] = si[0];
    }
    __syncthreads();
  }
}

}  // namespace

scls_status offload_device(scls_ctx* ctx, int64_t nb, const int64_t* batch_id, const double* est,
                           int32_t nw, const int32_t* worker_id, double* load,
                           int64_t* out_batch_id, int32_t* out_worker) {
  if (nb == 0) return SCLS_OK;
  if (nw <= 0) return set_error(ctx, SCLS_ERR_NO_WORKERS, "cannot offload batches: no workers configured");
  cudaStream_t s = ctx->stream;
  uint64_t* keys = (uint64_t*)ctx->buf(kSlotOKeys, sizeof(uint64_t) * nb);
  int32_t* vals = (int32_t*)ctx->buf(kSlotOVals, sizeof(int32_t) * nb);
  uint64_t* keys2 = (uint64_t*)ctx->buf(kSlotOKeysAlt, sizeof(uint64_t) * nb);
  int32_t* vals2 = (int32_t*)ctx->buf(kSlotOValsAlt, sizeof(int32_t) * nb);
  unsigned long long* range = (unsigned long long*)ctx->buf(kSlotORange, 2 * sizeof(uint64_t));
  unsigned long long* hrange = (unsigned long long*)ctx->host_pinned(2 * sizeof(uint64_t));
  if (!keys || !vals || !keys2 || !vals2 || !range || !hrange)
    return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  init_range_kernel<<<1, 1, 0, s>>>(range);
  SCLS_LAUNCHED();
  const int grid = std::min(div_up(nb, 256), ctx->sm_count * 8);
  est_keys_kernel<<<grid, 256, 0, s>>>(nb, est, keys, vals, range);
  SCLS_LAUNCHED();
  SCLS_CUDA(cudaMemcpyAsync(hrange, range, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  SCLS_CUDA(cudaStreamSynchronize(s));
  const int bits = bit_width(hrange[1] - hrange[0]);
  const int32_t* order = vals;
  if (bits > 0) {
    sub_keys_kernel<<<div_up(nb, 256), 256, 0, s>>>(nb, keys, range);
    SCLS_LAUNCHED();
    bool swapped = false;
    scls_status st = radix_sort_pairs(ctx, nb, keys, vals, keys2, vals2, 0, bits, &swapped);
    if (st) return st;
    order = swapped ? vals2 : vals;
  }
  if (nw <= 1) greedy_small_kernel<1><<<1, 32, 0, s>>>(nb, order, batch_id, est, nw, worker_id, load, out_batch_id, out_worker);
  else if (nw <= 2) greedy_small_kernel<2><<<1, 32, 0, s>>>(nb, order, batch_id, est, nw, worker_id, load, out_batch_id, out_worker);
  else if (nw <= 4) greedy_small_kernel<4><<<1, 32, 0, s>>>(nb, order, batch_id, est, nw, worker_id, load, out_batch_id, out_worker);
  else if (nw <= 8) greedy_small_kernel<8><<<1, 32, 0, s>>>(nb, order, batch_id, est, nw, worker_id, load, out_batch_id, out_worker);
  else if (nw <= 32) greedy_warp_kernel<<<1, 32, 0, s>>>(nb, order, batch_id, est, nw, worker_id, load, out_batch_id, out_worker);
  else greedy_block_kernel<<<1, 256, 0, s>>>(nb, order, batch_id, est, nw, worker_id, load, out_batch_id, out_worker);
  SCLS_LAUNCHED();
  return SCLS_OK;
}

}  // namespace scls
