// radix.cu — stable LSD radix sort (8-bit digits) and exclusive scan.
//
// Sort pass = histogram kernel + scan of the digit-major count table +
// scatter kernel.  Ranks inside a tile are made stable with warp-level
// __match_any_sync: a warp walks its 256-element segment in 8 rounds of 32,
// each element's rank = earlier same-digit elements in the warp segment
// (per-warp smem counters) + earlier peers in the round; warps are then
// prefixed per digit.  Tile = 8 warps x 256 = 2048 elements.
#include "radix.cuh"
#include "scls_common.cuh"

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


// ---- eff-bucket sort ------------------------------------------------------

__device__ __forceinline__ uint64_t eb_bias64(int64_t x) { return (uint64_t)x ^ 0x8000000000000000ull; }

// The bucket plan from the device key stats (biased-int32 eff min / max):
// usable when the eff range has at most kBucketMaxBins values and the
// average bucket fits the shared-memory sort with room to spare.
struct EbPlan {
  bool ok;
  int32_t emin, nbins;
};
__device__ __forceinline__ EbPlan eb_plan(int64_t n, const unsigned long long* erng) {
  const uint64_t lo = erng[0], hi = erng[1];
  const uint64_t r = hi - lo;
  EbPlan pl;
  pl.ok = hi >= lo && r < (uint64_t)kBucketMaxBins && n <= (int64_t)(r + 1) * (kBucketCap * 3 / 4);
  pl.emin = (int32_t)((uint32_t)lo ^ 0x80000000u);
  pl.nbins = pl.ok ? (int32_t)r + 1 : 0;
  return pl;
}

// Histogram of eff - emin.  Small bin counts (<= kEbSmemBins): a shared
// histogram per block of kEbChunk elements, then one global add per bin per
// block; larger ranges: warp-aggregated global adds.
constexpr int kEbSmemBins = 8192;
constexpr int kEbChunk = 4096;  // 256 blocks for a 1M pool
__global__ void __launch_bounds__(512) ebucket_hist_kernel(int64_t n, const int32_t* __restrict__ eff,
                                                           const unsigned long long* __restrict__ erng,
                                                           int32_t* __restrict__ counts) {
  __shared__ int32_t h[kEbSmemBins];
  const EbPlan pl = eb_plan(n, erng);
  if (!pl.ok) return;
  const int32_t emin = pl.emin, nbins = pl.nbins;
  const int64_t lo = (int64_t)blockIdx.x * kEbChunk, hi = min(n, lo + kEbChunk);
  if (nbins <= kEbSmemBins) {
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&h[eff[i] - emin], 1);
    __syncthreads();
    for (int b = threadIdx.x; b < nbins; b += blockDim.x)
      if (h[b]) atomicAdd(&counts[b], h[b]);
    return;
  }
  for (int64_t base = lo; base < hi; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool ok = i < hi;
    const int b = ok ? eff[i] - emin : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    if (ok && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&counts[b], __popc(peers));
  }
}

// One CTA: exclusive offsets of <= kBucketMaxBins counts, a cursor copy, and
// the overflow flag for buckets beyond kBucketCap.
__global__ void __launch_bounds__(1024) ebucket_scan_kernel(int64_t n, const unsigned long long* __restrict__ erng,
                                                            const int32_t* __restrict__ counts,
                                                            int32_t* __restrict__ offs,
                                                            int32_t* __restrict__ cursor,
                                                            int32_t* __restrict__ overflow) {
  __shared__ int32_t ws[32];
  const EbPlan pl = eb_plan(n, erng);
  if (!pl.ok) {
    if (threadIdx.x == 0) *overflow = 1;
    return;
  }
  const int32_t nbins = pl.nbins;
  const int per = (nbins + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int sum = 0, mx = 0;
  for (int q = 0; q < per; ++q) {
    const int b = b0 + q;
    if (b < nbins) {
      const int c = counts[b];
      sum += c;
      mx = max(mx, c);
    }
  }
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int v = ws[lane];
    int vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= o) vi += y;
    }
    ws[lane] = vi - v;
  }
  __syncthreads();
  int run = ws[w] + incl - sum;
  for (int q = 0; q < per; ++q) {
    const int b = b0 + q;
    if (b < nbins) {
      offs[b] = run;
      cursor[b] = run;
      run += counts[b];
    }
  }
  if (mx > kBucketCap) *overflow = 1;
}

// Scatter positions into their eff buckets.  Small bin counts: a block
// reserves each bin's range for its kEbChunk elements with one global add,
// then ranks locally in shared memory (the order inside a bucket does not
// matter: the bucket sort's last key is the position).
__global__ void __launch_bounds__(512) ebucket_scatter_kernel(int64_t n, const int32_t* __restrict__ eff,
                                                              const unsigned long long* __restrict__ erng,
                                                              int32_t* __restrict__ cursor,
                                                              int32_t* __restrict__ idx) {
  __shared__ int32_t h[kEbSmemBins];
  const EbPlan pl = eb_plan(n, erng);
  if (!pl.ok) return;
  const int32_t emin = pl.emin, nbins = pl.nbins;
  const int64_t lo = (int64_t)blockIdx.x * kEbChunk, hi = min(n, lo + kEbChunk);
  const int lane = threadIdx.x & 31;
  if (nbins <= kEbSmemBins) {
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&h[eff[i] - emin], 1);
    __syncthreads();
    for (int b = threadIdx.x; b < nbins; b += blockDim.x)
      if (h[b]) h[b] = atomicAdd(&cursor[b], h[b]);
    __syncthreads();
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) idx[atomicAdd(&h[eff[i] - emin], 1)] = (int32_t)i;
    return;
  }
  for (int64_t base = lo; base < hi; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool ok = i < hi;
    const int b = ok ? eff[i] - emin : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    const int leader = __ffs(peers) - 1;
    int at = 0;
    if (ok && lane == leader) at = atomicAdd(&cursor[b], __popc(peers));
    at = __shfl_sync(0xffffffffu, at, leader);
    if (ok) idx[at + __popc(peers & ((1u << lane) - 1u))] = (int32_t)i;
  }
}

// One CTA per bucket (grid-stride).  Fast path: every member gets a 21-bit
// image of its arrival, (ordered_bits(arrival) - bucket min) >> shift with
// the shift that fits the bucket's range in 21 bits -- monotone in the
// arrival -- and the 32-bit key image << 11 | slot is sorted by a bitonic
// network held in registers (four members per thread: partners 1-2 apart in
// the thread, 4-64 apart by warp shuffles, 128+ apart through shared
// memory).  That orders the bucket up to runs of equal images, which are then
// put in (arrival, id, position) order by an insertion sort of the full keys.
// A run longer than kEbTieRun (e.g. a bucket of equal arrivals) sends the
// bucket to the full-key bitonic sort in shared memory.
constexpr int kEbThreads = 512;  // four members per thread: kBucketCap = 2048
constexpr int kEbPer = 4;
constexpr int kEbImgBits = 21, kEbSlotBits = 11;
constexpr int kEbTieRun = 32;
static_assert(kEbPer * kEbThreads == kBucketCap && (1 << kEbSlotBits) == kBucketCap, "bucket geometry");

__device__ __forceinline__ bool eb_less_full(int xa, int xb, const double* arr, const int64_t* id) {
  const uint64_t a0 = ordered_bits(arr[xa]), a1 = ordered_bits(arr[xb]);
  if (a0 != a1) return a0 < a1;
  const int64_t i0 = id[xa], i1 = id[xb];
  if (i0 != i1) return i0 < i1;
  return xa < xb;
}

// Compare-exchange seen from one member: keep the min when m == 0, the max
// when m == ~0 (min of the complements).
__device__ __forceinline__ uint32_t eb_keep(uint32_t mine, uint32_t other, uint32_t m) {
  return min(mine ^ m, other ^ m) ^ m;
}

__global__ void __launch_bounds__(kEbThreads) ebucket_sort_kernel(int64_t n, const unsigned long long* __restrict__ erng,
                                                                  const int32_t* __restrict__ counts,
                                                                  const int32_t* __restrict__ offs,
                                                                  const int32_t* __restrict__ idx,
                                                                  const double* __restrict__ arr,
                                                                  const int64_t* __restrict__ id,
                                                                  int32_t* __restrict__ perm) {
  __shared__ uint64_t ka[kBucketCap], ki[kBucketCap];  // fast path: two 32-bit stage buffers in ka
  __shared__ uint32_t kx[kBucketCap];                  // fast path: slot -> position
  __shared__ uint64_t red[2][kEbThreads / 32];
  uint32_t* const sbuf0 = (uint32_t*)ka;
  uint32_t* const sbuf1 = sbuf0 + kBucketCap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int e0 = kEbPer * tid;
  const EbPlan pl = eb_plan(n, erng);
  if (!pl.ok) {  // no buckets: a valid (identity) permutation for the caller's rows pass, then the LSD sort
    for (int64_t i = (int64_t)blockIdx.x * kEbThreads + tid; i < n; i += (int64_t)gridDim.x * kEbThreads)
      perm[i] = (int32_t)i;
    return;
  }
  const int32_t nbins = pl.nbins;
  for (int b = blockIdx.x; b < nbins; b += gridDim.x) {
    const int c = counts[b];
    if (c == 0) continue;
    const int o = offs[b];
    if (c > kBucketCap) {  // overflow (the caller re-sorts): positions only, so the rows pass reads valid rows
      for (int q = tid; q < c; q += kEbThreads) perm[o + q] = idx[o + q];
      continue;
    }
    if (c == 1) {
      if (tid == 0) perm[o] = idx[o];
      continue;
    }
    int P = 128;
    while (P < c) P <<= 1;
    // ---- images
    uint64_t ob[kEbPer];
    uint64_t mn = ~0ull, mx = 0ull;
#pragma unroll
    for (int h = 0; h < kEbPer; ++h) {
      ob[h] = 0;
      if (e0 + h < c) {
        const int x = idx[o + e0 + h];
        kx[e0 + h] = (uint32_t)x;
        ob[h] = ordered_bits(arr[x]);
        mn = min(mn, ob[h]);
        mx = max(mx, ob[h]);
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      mn = min(mn, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)mn, d));
      mx = max(mx, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)mx, d));
    }
    if (lane == 0) {
      red[0][warp] = mn;
      red[1][warp] = mx;
    }
    __syncthreads();
    mn = red[0][0];
    mx = red[1][0];
#pragma unroll
    for (int w = 1; w < kEbThreads / 32; ++w) {
      mn = min(mn, red[0][w]);
      mx = max(mx, red[1][w]);
    }
    const uint64_t span = mx - mn;
    const int sh = span ? max(0, 64 - kEbImgBits - __clzll((long long)span)) : 0;
    uint32_t k[kEbPer];
#pragma unroll
    for (int h = 0; h < kEbPer; ++h)
      k[h] = e0 + h < c ? (uint32_t)((ob[h] - mn) >> sh) << kEbSlotBits | (uint32_t)(e0 + h) : ~0u;
    // ---- bitonic network on the 32-bit keys (all distinct)
    const bool act = e0 < P;  // warp-uniform (P >= 128)
    int buf = 0;
    for (int kk = 2; kk <= P; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        if (j >= 4) {
          // the four members share (i & j) and (i & kk): one direction per thread
          const uint32_t m = ((e0 & j) == 0) == ((e0 & kk) == 0) ? 0u : ~0u;
          if (j >= 128) {
            uint32_t* sb = buf ? sbuf1 : sbuf0;
            buf ^= 1;
            if (act) *(uint4*)(sb + e0) = make_uint4(k[0], k[1], k[2], k[3]);
            __syncthreads();
            if (act) {
              const uint4 p = *(const uint4*)(sb + (e0 ^ j));
              k[0] = eb_keep(k[0], p.x, m);
              k[1] = eb_keep(k[1], p.y, m);
              k[2] = eb_keep(k[2], p.z, m);
              k[3] = eb_keep(k[3], p.w, m);
            }
          } else if (act) {
#pragma unroll
            for (int h = 0; h < kEbPer; ++h) k[h] = eb_keep(k[h], __shfl_xor_sync(0xffffffffu, k[h], j >> 2), m);
          }
        } else if (act) {
          // partners inside the thread: (0, 2), (1, 3) for j = 2; (0, 1), (2, 3) for j = 1
          auto cx = [&](uint32_t& a, uint32_t& z, int i) {
            const bool asc = (i & kk) == 0;
            const uint32_t lo = min(a, z), hi = max(a, z);
            a = asc ? lo : hi;
            z = asc ? hi : lo;
          };
          if (j == 2) {
            cx(k[0], k[2], e0);
            cx(k[1], k[3], e0 + 1);
          } else {
            cx(k[0], k[1], e0);
            cx(k[2], k[3], e0 + 2);
          }
        }
      }
    }
    // ---- runs of equal images
    uint32_t* sk = buf ? sbuf1 : sbuf0;  // not the buffer the last shared stage read
    if (act) *(uint4*)(sk + e0) = make_uint4(k[0], k[1], k[2], k[3]);
    __syncthreads();
    bool tie = false;
#pragma unroll
    for (int h = 0; h < kEbPer; ++h) {
      const int i = e0 + h;
      tie |= i + 1 < c && (sk[i] >> kEbSlotBits) == (sk[i + 1] >> kEbSlotBits);
    }
    bool slow = false;
    if (__syncthreads_or(tie)) {
      // a run starts at s when image(s) == image(s + 1) != image(s - 1)
      int run_len = 0;
#pragma unroll
      for (int h = 0; h < kEbPer; ++h) {
        const int s = e0 + h;
        const uint32_t is = sk[s] >> kEbSlotBits;
        if (s + 1 < c && is == (sk[s + 1] >> kEbSlotBits) && (s == 0 || (sk[s - 1] >> kEbSlotBits) != is)) {
          int e = s + 2;
          while (e < c && (sk[e] >> kEbSlotBits) == is && e - s <= kEbTieRun) ++e;
          run_len = max(run_len, e - s);
        }
      }
      slow = __syncthreads_or(run_len > kEbTieRun);
      if (!slow) {
#pragma unroll
        for (int h = 0; h < kEbPer; ++h) {
          const int s = e0 + h;
          const uint32_t is = sk[s] >> kEbSlotBits;
          if (s + 1 < c && is == (sk[s + 1] >> kEbSlotBits) && (s == 0 || (sk[s - 1] >> kEbSlotBits) != is)) {
            int e = s + 1;
            while (e < c && (sk[e] >> kEbSlotBits) == is) ++e;
            for (int i = s + 1; i < e; ++i) {  // insertion sort of [s, e) by the full key
              const uint32_t v = sk[i];
              const int xv = (int)kx[v & (kBucketCap - 1)];
              int q = i;
              while (q > s && eb_less_full(xv, (int)kx[sk[q - 1] & (kBucketCap - 1)], arr, id)) {
                sk[q] = sk[q - 1];
                --q;
              }
              sk[q] = v;
            }
          }
        }
        __syncthreads();
      }
    }
    if (!slow) {
      for (int q = tid; q < c; q += kEbThreads) perm[o + q] = (int32_t)kx[sk[q] & (kBucketCap - 1)];
      __syncthreads();
      continue;
    }
    // ---- long runs of equal images: bitonic sort on the full keys
    for (int q = tid; q < P; q += kEbThreads) {
      if (q < c) {
        const int x = idx[o + q];
        ka[q] = ordered_bits(arr[x]);
        ki[q] = eb_bias64(id[x]);
        kx[q] = (uint32_t)x;
      } else {
        ka[q] = ki[q] = ~0ull;
        kx[q] = ~0u;
      }
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = tid; t < (P >> 1); t += kEbThreads) {
          const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), h = i + j;  // j is a power of two
          const uint64_t a0 = ka[i], a1 = ka[h], i0 = ki[i], i1 = ki[h];
          const uint32_t x0 = kx[i], x1 = kx[h];
          const bool gt = a0 > a1 || (a0 == a1 && (i0 > i1 || (i0 == i1 && x0 > x1)));
          if (gt == ((i & k) == 0)) {  // ascending blocks swap a greater first element
            ka[i] = a1;
            ka[h] = a0;
            ki[i] = i1;
            ki[h] = i0;
            kx[i] = x1;
            kx[h] = x0;
          }
        }
        __syncthreads();
      }
    }
    for (int q = tid; q < c; q += kEbThreads) perm[o + q] = (int32_t)kx[q];
    __syncthreads();
  }
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

scls_status bucket_sort_perm(scls_ctx* ctx, int64_t n, const int32_t* eff, const double* arr,
                             const int64_t* id, const unsigned long long* d_eff_range, int32_t* perm,
                             int32_t* d_overflow) {
  cudaStream_t s = ctx->stream;
  int32_t* counts = (int32_t*)ctx->buf(kSlotBucket + 0, sizeof(int32_t) * kBucketMaxBins);
  int32_t* offs = (int32_t*)ctx->buf(kSlotBucket + 1, sizeof(int32_t) * kBucketMaxBins);
  int32_t* cursor = (int32_t*)ctx->buf(kSlotBucket + 2, sizeof(int32_t) * kBucketMaxBins);
  int32_t* idx = (int32_t*)ctx->buf(kSlotBucket + 3, sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1));
  if (!counts || !offs || !cursor || !idx) return set_error(ctx, SCLS_ERR_CUDA, "scratch allocation failed");
  SCLS_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * kBucketMaxBins, s));
  const int grid = (int)div_up(n, kEbChunk);
  ebucket_hist_kernel<<<grid, 512, 0, s>>>(n, eff, d_eff_range, counts);
  SCLS_LAUNCHED();
  ebucket_scan_kernel<<<1, 1024, 0, s>>>(n, d_eff_range, counts, offs, cursor, d_overflow);
  SCLS_LAUNCHED();
  ebucket_scatter_kernel<<<grid, 512, 0, s>>>(n, eff, d_eff_range, cursor, idx);
  SCLS_LAUNCHED();
  // four 512-thread CTAs per SM; buckets grid-strided
  ebucket_sort_kernel<<<ctx->sm_count * 4, kEbThreads, 0, s>>>(n, d_eff_range, counts, offs, idx, arr, id, perm);
  SCLS_LAUNCHED();
  return SCLS_OK;
}

}  // namespace scls
