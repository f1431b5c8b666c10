// radix.cu — stable LSD radix sort (8-bit digits) and exclusive scan.
//
// Sort pass = histogram kernel + scan of the digit-major count table +
// scatter kernel.  Ranks inside a tile are made stable with warp-level
// __match_any_sync: a warp walks its 256-element segment in 8 rounds of 32,
// each element's rank = earlier same-digit elements in the warp segment
// (per-warp smem counters) + earlier peers in the round; warps are then
// prefixed per digit.  Tile = 8 warps x 256 = 2048 elements.
#include "radix.cuh"

namespace scls {
namespace {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kItems = 8;
constexpr int kTile = kBlock * kItems;
constexpr int kBins = 256;

__global__ void __launch_bounds__(kBlock) radix_hist_kernel(const uint64_t* __restrict__ keys,
                                                            int64_t n, int shift, uint32_t mask,
                                                            int32_t* __restrict__ counts,
                                                            int nblocks) {
  __shared__ int32_t h[kBins];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  h[tid] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile + w * (32 * kItems);
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int64_t e = base + i * 32 + lane;
    if (e < n) atomicAdd(&h[(keys[e] >> shift) & mask], 1);
  }
  __syncthreads();
  counts[(int64_t)tid * nblocks + blockIdx.x] = h[tid];
}

__global__ void __launch_bounds__(kBlock) radix_scatter_kernel(
    const uint64_t* __restrict__ keys, const int32_t* __restrict__ vals,
    uint64_t* __restrict__ okeys, int32_t* __restrict__ ovals, int64_t n, int shift,
    uint32_t mask, const int32_t* __restrict__ offsets, int nblocks) {
  __shared__ int32_t wcnt[kWarps][kBins];
  __shared__ int32_t goff[kBins];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int q = 0; q < kWarps; ++q) wcnt[q][tid] = 0;
  goff[tid] = offsets[(int64_t)tid * nblocks + blockIdx.x];
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile + w * (32 * kItems);
  const unsigned lt = (1u << lane) - 1u;
  uint64_t k[kItems];
  int32_t v[kItems];
  int32_t d[kItems];
  int32_t rank[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int64_t e = base + i * 32 + lane;
    const bool valid = e < n;
    k[i] = valid ? keys[e] : 0;
    v[i] = valid ? vals[e] : 0;
    d[i] = valid ? (int32_t)((k[i] >> shift) & mask) : kBins + lane;
    const unsigned peers = __match_any_sync(0xffffffffu, d[i]);
    const int leader = __ffs(peers) - 1;
    const int prior = valid ? wcnt[w][d[i]] : 0;
    rank[i] = prior + __popc(peers & lt);
    __syncwarp();
    if (valid && lane == leader) wcnt[w][d[i]] = prior + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    int run = 0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) {
      const int c = wcnt[q][tid];
      wcnt[q][tid] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    if (d[i] < kBins) {
      const int pos = goff[d[i]] + wcnt[w][d[i]] + rank[i];
      okeys[pos] = k[i];
      ovals[pos] = v[i];
    }
  }
}

// ---- exclusive scan ------------------------------------------------------

constexpr int kScanBlock = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanBlock * kScanItems;

__global__ void __launch_bounds__(kScanBlock) scan_tiles_kernel(const int32_t* __restrict__ in,
                                                                int32_t* __restrict__ out,
                                                                int64_t n,
                                                                int32_t* __restrict__ tile_sums) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int32_t x[kScanItems];
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    x[i] = (base + i < n) ? in[base + i] : 0;
    s += x[i];
  }
  // Block-wide exclusive scan of the per-thread sums (warp 31 handled
  // separately because its base slot doubles as the total).
  __shared__ int32_t ws[32];
  __shared__ int32_t tot;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int32_t v = ws[lane];
    int32_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= o) vi += y;
    }
    ws[lane] = vi - v;
    if (lane == 31) tot = vi;
  }
  __syncthreads();
  int32_t run = ws[w] + incl - s;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += x[i];
  }
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void scan_add_kernel(int32_t* __restrict__ out, int64_t n,
                                const int32_t* __restrict__ tile_off) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += tile_off[i / kScanTile];
}

__global__ void total_kernel(const int32_t* __restrict__ in, const int32_t* __restrict__ ex,
                             int64_t n, int32_t* __restrict__ total) {
  *total = n ? ex[n - 1] + in[n - 1] : 0;
}

}  // namespace

static scls_status scan_level(scls_ctx* ctx, int64_t n, const int32_t* in, int32_t* out,
                              int32_t* d_total, int level) {
  if (n <= 0) {
    if (d_total) SCLS_CUDA(cudaMemsetAsync(d_total, 0, sizeof(int32_t), ctx->stream));
    return SCLS_OK;
  }
  const int tiles = div_up(n, kScanTile);
  int32_t* sums = (int32_t*)ctx->buf(kSlotScan + 2 * level, sizeof(int32_t) * (size_t)(tiles + 1));
  int32_t* offs = (int32_t*)ctx->buf(kSlotScan + 2 * level + 1, sizeof(int32_t) * (size_t)(tiles + 1));
  if (!sums || !offs) return set_error(ctx, SCLS_ERR_CUDA, "scratch allocation failed");
  scan_tiles_kernel<<<tiles, kScanBlock, 0, ctx->stream>>>(in, out, n, sums);
  SCLS_LAUNCHED();
  if (tiles > 1) {
    scls_status st = scan_level(ctx, tiles, sums, offs, nullptr, level + 1);
    if (st) return st;
    scan_add_kernel<<<div_up(n, 256), 256, 0, ctx->stream>>>(out, n, offs);
    SCLS_LAUNCHED();
  }
  if (d_total) {
    total_kernel<<<1, 1, 0, ctx->stream>>>(in, out, n, d_total);
    SCLS_LAUNCHED();
  }
  return SCLS_OK;
}

scls_status scan_exclusive(scls_ctx* ctx, int64_t n, const int32_t* in, int32_t* out,
                           int32_t* d_total) {
  return scan_level(ctx, n, in, out, d_total, 0);
}

scls_status radix_sort_pairs(scls_ctx* ctx, int64_t n, uint64_t* keys, int32_t* vals,
                             uint64_t* keys_alt, int32_t* vals_alt, int begin_bit,
                             int end_bit, bool* swapped) {
  *swapped = false;
  if (n <= 1 || end_bit <= begin_bit) return SCLS_OK;
  const int nblocks = div_up(n, kTile);
  const int64_t table = (int64_t)kBins * nblocks;
  int32_t* counts = (int32_t*)ctx->buf(kSlotRadixCounts, sizeof(int32_t) * (size_t)table);
  int32_t* offs = (int32_t*)ctx->buf(kSlotRadixOffs, sizeof(int32_t) * (size_t)table);
  if (!counts || !offs) return set_error(ctx, SCLS_ERR_CUDA, "scratch allocation failed");
  uint64_t *ki = keys, *ko = keys_alt;
  int32_t *vi = vals, *vo = vals_alt;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    const int bits = end_bit - shift < 8 ? end_bit - shift : 8;
    const uint32_t mask = (1u << bits) - 1u;
    radix_hist_kernel<<<nblocks, kBlock, 0, ctx->stream>>>(ki, n, shift, mask, counts, nblocks);
    SCLS_LAUNCHED();
    scls_status st = scan_exclusive(ctx, table, counts, offs, nullptr);
    if (st) return st;
    radix_scatter_kernel<<<nblocks, kBlock, 0, ctx->stream>>>(ki, vi, ko, vo, n, shift, mask,
                                                              offs, nblocks);
    SCLS_LAUNCHED();
    uint64_t* tk = ki; ki = ko; ko = tk;
    int32_t* tv = vi; vi = vo; vo = tv;
    *swapped = !*swapped;
  }
  return SCLS_OK;
}

}  // namespace scls
