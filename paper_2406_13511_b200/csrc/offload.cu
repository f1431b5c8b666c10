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

enum : int { kSlotOKeys = 18, kSlotOVals, kSlotOKeysAlt, kSlotOValsAlt, kSlotORange, kSlotOEst, kSlotOSlots };

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

// Worker slots are renumbered in (worker_id, index) order once per call, so
// the reference's tie rule (lowest worker_id, then first position,
// offloader.cpp:39-47) becomes "lowest slot wins ties" and a comparison tree
// only needs `right < left` on the load.
__global__ void slot_order_kernel(int32_t nw, const int32_t* __restrict__ worker_id,
                                  int32_t* __restrict__ slot_src, int32_t* __restrict__ slot_id) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int32_t i = 0; i < nw; ++i) {  // insertion sort by (id, index); W is small
    const int32_t id = worker_id[i];
    int32_t j = i;
    while (j > 0 && slot_id[j - 1] > id) {
      slot_id[j] = slot_id[j - 1];
      slot_src[j] = slot_src[j - 1];
      --j;
    }
    slot_id[j] = id;
    slot_src[j] = i;
  }
}

__global__ void gather_sorted_kernel(int64_t nb, const int32_t* __restrict__ order,
                                     const int64_t* __restrict__ batch_id,
                                     const double* __restrict__ est, double* __restrict__ est_sorted,
                                     int64_t* __restrict__ out_b) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  const int32_t i = order[k];
  est_sorted[k] = est[i];
  out_b[k] = batch_id[i];
}

__global__ void slot_to_worker_kernel(int64_t nb, const int32_t* __restrict__ slot_id,
                                      int32_t* __restrict__ out_w) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nb) out_w[k] = slot_id[out_w[k]];
}

constexpr int kChunk = 2048;

// p ? a : b as an opaque selp, so the front end cannot turn a select over an
// unrolled register array into an indexed (local-memory) access.
__device__ __forceinline__ double select_if(bool p, double a, double b) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tselp.f64 %0, %2, %3, q;\n\t}"
      : "=d"(r)
      : "r"((unsigned)p), "d"(a), "d"(b));
  return r;
}

// Thread 0 runs the serial greedy chain over the sorted estimates with the W
// loads in registers and a log2(W)-deep comparison tree; warp 1 streams the
// next chunk of estimates into shared memory meanwhile.
template <int W>
__global__ void __launch_bounds__(64) greedy_small_kernel(int64_t nb, const double* __restrict__ est_sorted,
                                                          int32_t nw, const int32_t* __restrict__ slot_src,
                                                          double* __restrict__ load,
                                                          int32_t* __restrict__ out_slot) {
  __shared__ double se[2][kChunk];
  const int tid = threadIdx.x;
  const int nchunks = (int)((nb + kChunk - 1) / kChunk);
  if (tid >= 32) {
    for (int i = tid - 32; i < kChunk && i < nb; i += 32) se[0][i] = est_sorted[i];
  }
  double l[W];
#pragma unroll
  for (int w = 0; w < W; ++w) l[w] = (tid == 0 && w < nw) ? load[slot_src[w]] : __longlong_as_double(0x7ff0000000000000ll);
  __syncthreads();
  for (int c = 0; c < nchunks; ++c) {
    const int64_t base = (int64_t)c * kChunk;
    if (tid >= 32 && c + 1 < nchunks) {
      const int64_t nb2 = base + kChunk;
      for (int i = tid - 32; i < kChunk && nb2 + i < nb; i += 32) se[(c + 1) & 1][i] = est_sorted[nb2 + i];
    }
    if (tid == 0) {
      const int cnt = (int)min((int64_t)kChunk, nb - base);
      const double* e = se[c & 1];
      for (int i = 0; i < cnt; ++i) {
        double bl[W];
        int bx[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
          bl[w] = l[w];
          bx[w] = w;
        }
#pragma unroll
        for (int span = 1; span < W; span <<= 1) {
#pragma unroll
          for (int w = 0; w + span < W; w += 2 * span) {
            if (bl[w + span] < bl[w]) {
              bl[w] = bl[w + span];
              bx[w] = bx[w + span];
            }
          }
        }
        // every candidate sum is formed while the tree runs; the winner's is
        // then selected -- no indexed update, so l[] stays in registers
        const double ei = e[i];
        double nl[W];
#pragma unroll
        for (int w = 0; w < W; ++w) nl[w] = __dadd_rn(l[w], ei);
#pragma unroll
        for (int w = 0; w < W; ++w) l[w] = select_if(bx[0] == w, nl[w], l[w]);
        out_slot[base + i] = bx[0];
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
#pragma unroll
    for (int w = 0; w < W; ++w)
      if (w < nw) load[slot_src[w]] = l[w];
  }
}

// 9..32 workers: lane = slot, shuffle argmin with lower lane winning ties.
__global__ void greedy_warp_kernel(int64_t nb, const double* __restrict__ est_sorted, int32_t nw,
                                   const int32_t* __restrict__ slot_src, double* __restrict__ load,
                                   int32_t* __restrict__ out_slot) {
  const int lane = threadIdx.x;
  double l = lane < nw ? load[slot_src[lane]] : __longlong_as_double(0x7ff0000000000000ll);
  double e_next = nb > 0 ? est_sorted[0] : 0.0;
  for (int64_t k = 0; k < nb; ++k) {
    const double e = e_next;
    if (k + 1 < nb) e_next = est_sorted[k + 1];
    double bl = l;
    int bx = lane;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ol = __shfl_xor_sync(~0u, bl, o);
      const int ox = __shfl_xor_sync(~0u, bx, o);
      if (ol < bl || (ol == bl && ox < bx)) {
        bl = ol;
        bx = ox;
      }
    }
    if (lane == bx) l = __dadd_rn(l, e);
    if (lane == 0) out_slot[k] = bx;
  }
  if (lane < nw) load[slot_src[lane]] = l;
}

// Any W: one CTA, loads in global memory, block argmin per batch.
__global__ void greedy_block_kernel(int64_t nb, const double* __restrict__ est_sorted, int32_t nw,
                                    const int32_t* __restrict__ slot_src, double* __restrict__ load,
                                    int32_t* __restrict__ out_slot) {
  __shared__ double sl[32];
  __shared__ int sx[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int64_t k = 0; k < nb; ++k) {
    double bl = __longlong_as_double(0x7ff0000000000000ll);
    int bx = 0x7fffffff;
    for (int w = tid; w < nw; w += blockDim.x) {
      const double lw = load[slot_src[w]];
      if (lw < bl || (lw == bl && w < bx)) {
        bl = lw;
        bx = w;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ol = __shfl_xor_sync(~0u, bl, o);
      const int ox = __shfl_xor_sync(~0u, bx, o);
      if (ol < bl || (ol == bl && ox < bx)) {
        bl = ol;
        bx = ox;
      }
    }
    if (lane == 0) {
      sl[warp] = bl;
      sx[warp] = bx;
    }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < nwarps; ++q)
        if (sl[q] < sl[0] || (sl[q] == sl[0] && sx[q] < sx[0])) {
          sl[0] = sl[q];
          sx[0] = sx[q];
        }
      double* lp = &load[slot_src[sx[0]]];
      *lp = __dadd_rn(*lp, est_sorted[k]);
      out_slot[k] = sx[0];
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
  double* est_sorted = (double*)ctx->buf(kSlotOEst, sizeof(double) * nb);
  int32_t* slot_src = (int32_t*)ctx->buf(kSlotOSlots, sizeof(int32_t) * 2 * (size_t)nw);
  if (!est_sorted || !slot_src) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  int32_t* slot_id = slot_src + nw;
  slot_order_kernel<<<1, 1, 0, s>>>(nw, worker_id, slot_src, slot_id);
  SCLS_LAUNCHED();
  gather_sorted_kernel<<<div_up(nb, 256), 256, 0, s>>>(nb, order, batch_id, est, est_sorted, out_batch_id);
  SCLS_LAUNCHED();
  if (nw <= 1) greedy_small_kernel<1><<<1, 64, 0, s>>>(nb, est_sorted, nw, slot_src, load, out_worker);
  else if (nw <= 2) greedy_small_kernel<2><<<1, 64, 0, s>>>(nb, est_sorted, nw, slot_src, load, out_worker);
  else if (nw <= 4) greedy_small_kernel<4><<<1, 64, 0, s>>>(nb, est_sorted, nw, slot_src, load, out_worker);
  else if (nw <= 8) greedy_small_kernel<8><<<1, 64, 0, s>>>(nb, est_sorted, nw, slot_src, load, out_worker);
  else if (nw <= 32) greedy_warp_kernel<<<1, 32, 0, s>>>(nb, est_sorted, nw, slot_src, load, out_worker);
  else greedy_block_kernel<<<1, 256, 0, s>>>(nb, est_sorted, nw, slot_src, load, out_worker);
  SCLS_LAUNCHED();
  slot_to_worker_kernel<<<div_up(nb, 256), 256, 0, s>>>(nb, slot_id, out_worker);
  SCLS_LAUNCHED();
  return SCLS_OK;
}

}  // namespace scls
