// workload_gen.cu — device trace generation: generate() (workload.cpp:163-181)
// for thousands of WorkloadSpecs at once, bit-exact with the reference.
//
// The reference's sampler per trace (workload.cpp:100-181):
//   engine = std::mt19937_64(seed)
//   loop: clock += -log(1 - u) / rate      u = (engine() >> 11) * 2^-53
//         if clock > duration: stop
//         input = sample_length(input dist), gen = sample_length(gen dist)
// Every request consumes a FIXED number of engine outputs D = 1 + d(input) +
// d(gen) (uniform: 1, histogram: 2), so request r owns outputs [rD, rD + D)
// and the stopping gap is output nD.  The only serial dependence is the
// arrival clock (an fp64 running sum that must be added in order).
//
// Layout: one warp per trace.  The warp keeps the 312-word MT state in shared
// memory and regenerates it 312 outputs at a time in two lane-parallel phases
// (libstdc++ _M_gen_rand: k < 156 reads x[k+156] old; k >= 156 reads x[k-156]
// new, and k = 311 reads the new x[0]); the tempered outputs land in a
// per-warp window with the < D leftover outputs of the previous block in
// front.  Requests are sampled one per lane (log via csrc/glibc_log.cuh, the
// FMA variant of glibc 2.39's log the reference links), then the warp adds the
// gaps to the clock in request order (32 dependent DADDs per 32 requests,
// the same sums as the reference) and writes coalesced SoA rows.
//
// Output rows go to a capped per-trace region (cap from a Poisson tail bound;
// an overflow is detected and the launch repeated with the exact counts),
// then are compacted into the contiguous req_offset layout the simulator
// reads (scls_simulate, sim_engine.cpp:102-114: ids = arrival ranks).
//
// Log-normal lengths (Box-Muller, two outputs per draw) use bit-exact ports of
// glibc's FMA `exp` and `cos` (csrc/glibc_expcos.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "ctx.h"
#include "glibc_expcos.cuh"
#include "glibc_log.cuh"
#include "scls_capi.h"

namespace scls {

scls_status validate_workload_spec(scls_ctx* ctx, const scls_workload_spec& spec);

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kGenWarps = 4;
constexpr int kMtN = 312;
constexpr int kWin = kMtN + 8;
constexpr uint64_t kMatA = 0xb5026f5aa96619e9ull;
constexpr uint64_t kUpper = 0xffffffff80000000ull;  // top 33 bits (r = 31)
constexpr uint64_t kLower = 0x000000007fffffffull;

__device__ __forceinline__ uint64_t temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71d67fffeda60000ull;
  z ^= (z << 37) & 0xfff7eee000000000ull;
  z ^= z >> 43;
  return z;
}

// u = (engine() >> 11) * 0x1.0p-53 (workload.cpp:100-102)
__device__ __forceinline__ double unit(uint64_t x) { return __dmul_rn((double)(x >> 11), 0x1.0p-53); }

// uniform_int (workload.cpp:120-123): lo + (int)(u * ((double)hi - lo + 1.0))
__device__ __forceinline__ int uniform_int(int lo, int hi, uint64_t x) {
  const double span = __dadd_rn(__dsub_rn((double)hi, (double)lo), 1.0);
  return lo + __double2int_rz(__dmul_rn(unit(x), span));
}

__device__ __forceinline__ int clamp_len(int v, int limit) { return v < 1 ? 1 : (v > limit ? limit : v); }

// sample_length (workload.cpp:133-161); w points at this request's outputs
// for the distribution.
__device__ __forceinline__ int sample_len(const scls_length_dist& d, int limit, const uint64_t* w) {
  if (d.kind == SCLS_DIST_UNIFORM) return clamp_len(uniform_int(d.lo, d.hi, w[0]), limit);
  if (d.kind == SCLS_DIST_LOGNORMAL) return scls_glibc::lognormal_length(d.mu, d.sigma, d.cap, limit, w[0], w[1]);
  const double u = unit(w[0]);
  double cdf = 0.0;
  int bucket = d.n_buckets - 1;
  for (int i = 0; i < d.n_buckets; ++i) {
    cdf = __dadd_rn(cdf, d.weights[i]);
    if (u < cdf) {
      bucket = i;
      break;
    }
  }
  return clamp_len(uniform_int(d.edges[bucket], d.edges[bucket + 1], w[1]), limit);
}

// engine outputs per draw: uniform 1; histogram (bucket, value) and
// log-normal (Box-Muller u1, u2: workload.cpp:112-118) 2
__device__ __forceinline__ int draws(const scls_length_dist& d) { return d.kind == SCLS_DIST_UNIFORM ? 1 : 2; }

__global__ void __launch_bounds__(kGenWarps * 32)
    gen_kernel(int32_t n_specs, const scls_workload_spec* __restrict__ specs, const int64_t* __restrict__ cap_off,
               double* __restrict__ arr, int32_t* __restrict__ inp, int32_t* __restrict__ gen,
               int64_t* __restrict__ count) {
  __shared__ uint64_t s_mt[kGenWarps][kMtN];
  __shared__ uint64_t s_win[kGenWarps][kWin];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * kGenWarps + w;
  if (t >= n_specs) return;
  const scls_workload_spec& sp = specs[t];
  const double rate = sp.rate, dur = sp.duration_s;
  const int max_in = sp.max_input_limit, max_gen = sp.max_gen_limit;
  const int d_in = draws(sp.input_len_dist);
  const int D = 1 + d_in + draws(sp.gen_len_dist);
  const int64_t base = cap_off[t], cap = cap_off[t + 1] - base;
  uint64_t* mt = s_mt[w];
  uint64_t* win = s_win[w];
  // std::mt19937_64(seed): x0 = seed, x_i = f * (x_{i-1} ^ (x_{i-1} >> 62)) + i
  if (lane == 0) {
    uint64_t x = sp.seed;
    mt[0] = x;
    for (int i = 1; i < kMtN; ++i) {
      x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
      mt[i] = x;
    }
  }
  __syncwarp();
  int carry = 0;
  int64_t cnt = 0;
  double clock = 0.0;
  bool done = false;
  while (!done) {
    // _M_gen_rand: phase A (k < 156) then phase B (k >= 156), 32 words at a
    // time; every lane reads before any lane of its chunk writes.
#pragma unroll 1
    for (int ph = 0; ph < 2; ++ph) {
#pragma unroll
      for (int c = 0; c < kMtN / 2; c += 32) {
        const int k = ph * (kMtN / 2) + c + lane;
        const bool act = c + lane < kMtN / 2;
        uint64_t nv = 0;
        if (act) {
          const uint64_t y = (mt[k] & kUpper) | (mt[k + 1 == kMtN ? 0 : k + 1] & kLower);
          const int m = k < kMtN / 2 ? k + kMtN / 2 : k - kMtN / 2;
          nv = mt[m] ^ (y >> 1) ^ ((y & 1ull) ? kMatA : 0ull);
        }
        __syncwarp();
        if (act) mt[k] = nv;
        __syncwarp();
      }
    }
    for (int j = lane; j < kMtN; j += 32) win[carry + j] = temper(mt[j]);
    __syncwarp();
    const int avail = carry + kMtN;
    const int nblk = avail / D;  // requests whose D outputs are all in the window
    for (int c = 0; c < nblk && !done; c += 32) {
      const int q = c + lane;
      const bool valid = q < nblk;
      double gap = 0.0;
      if (valid) {
        // next_exponential (workload.cpp:106-110): -log(1 - u) / rate
        const double u = unit(win[q * D]);
        gap = __ddiv_rn(-scls_glibc::log_fma(__dsub_rn(1.0, u)), rate);
      }
      // clock += gap, in request order (the same running sum as the reference)
      const int m = min(32, nblk - c);
      double mine = 0.0;
      for (int j = 0; j < m; ++j) {
        clock = __dadd_rn(clock, __shfl_sync(FULL, gap, j));
        if (j == lane) mine = clock;
      }
      const unsigned over = __ballot_sync(FULL, valid && mine > dur);
      const int nv = over ? __ffs(over) - 1 : m;  // requests before the stopping gap
      if (over) done = true;
      if (lane < nv) {
        const int in = sample_len(sp.input_len_dist, max_in, win + q * D + 1);
        const int gl = sample_len(sp.gen_len_dist, max_gen, win + q * D + 1 + d_in);
        const int64_t idx = cnt + lane;
        if (idx < cap) {
          arr[base + idx] = mine;
          inp[base + idx] = in;
          gen[base + idx] = gl;
        }
      }
      cnt += nv;
    }
    if (done) break;
    // carry the < D outputs of a request that straddles the block boundary
    const int left = avail - nblk * D;
    uint64_t v = lane < left ? win[nblk * D + lane] : 0ull;
    __syncwarp();
    if (lane < left) win[lane] = v;
    __syncwarp();
    carry = left;
  }
  if (lane == 0) count[t] = cnt;
}

// Capped layout -> contiguous req_offset layout (one warp per trace).
__global__ void compact_kernel(int32_t n, const int64_t* __restrict__ cap_off, const int64_t* __restrict__ off,
                               const double* __restrict__ a0, const int32_t* __restrict__ i0,
                               const int32_t* __restrict__ g0, double* __restrict__ a1, int32_t* __restrict__ i1,
                               int32_t* __restrict__ g1) {
  const int t = blockIdx.x;
  if (t >= n) return;
  const int64_t src = cap_off[t], dst = off[t], len = off[t + 1] - dst;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
    a1[dst + i] = a0[src + i];
    i1[dst + i] = i0[src + i];
    g1[dst + i] = g0[src + i];
  }
}

// Device copy of the ported log, for the bit-exactness test against libm.
// fn: 0 log, 1 exp, 2 cos (the device ports, for the bit-exactness checks)
__global__ void libm_kernel(int32_t fn, int64_t n, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fn == 0 ? scls_glibc::log_fma(x[i]) : fn == 1 ? scls_glibc::exp_fma(x[i]) : scls_glibc::cos_fma(x[i]);
}

}  // namespace

// Generates every spec's trace on the device.  On success h_off holds the
// n_specs + 1 request offsets and *arr/*inp/*gen point at ctx scratch (slots
// kSlotGen..) holding the concatenated traces.
scls_status generate_device(scls_ctx* ctx, int32_t n_specs, const scls_workload_spec* specs,
                            std::vector<int64_t>& h_off, double** arr, int32_t** inp, int32_t** gen) {
  cudaStream_t s = ctx->stream;
  for (int t = 0; t < n_specs; ++t) {
    scls_status st = validate_workload_spec(ctx, specs[t]);
    if (st) return st;
    if (!(specs[t].rate * specs[t].duration_s < 1e9))
      return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "device generator: rate * duration must be < 1e9");
  }
  // Capacity per trace: mean + 12 sigma + 64 of the Poisson count.
  std::vector<int64_t> cap_off(n_specs + 1, 0);
  for (int t = 0; t < n_specs; ++t) {
    const double mean = specs[t].rate * specs[t].duration_s;
    cap_off[t + 1] = cap_off[t] + (int64_t)std::ceil(mean + 12.0 * std::sqrt(mean) + 64.0);
  }
  scls_workload_spec* d_specs = (scls_workload_spec*)ctx->buf(kSlotGen + 0, sizeof(scls_workload_spec) * n_specs);
  int64_t* d_capoff = (int64_t*)ctx->buf(kSlotGen + 1, sizeof(int64_t) * (n_specs + 1));
  int64_t* d_cnt = (int64_t*)ctx->buf(kSlotGen + 2, sizeof(int64_t) * (n_specs + 1));
  if (!d_specs || !d_capoff || !d_cnt) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  SCLS_CUDA(cudaMemcpyAsync(d_specs, specs, sizeof(scls_workload_spec) * n_specs, cudaMemcpyHostToDevice, s));
  std::vector<int64_t> cnt(n_specs);
  double* a0 = nullptr;
  int32_t* i0 = nullptr;
  int32_t* g0 = nullptr;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const int64_t total_cap = std::max<int64_t>(cap_off[n_specs], 1);
    a0 = (double*)ctx->buf(kSlotGen + 3, sizeof(double) * total_cap);
    i0 = (int32_t*)ctx->buf(kSlotGen + 4, sizeof(int32_t) * total_cap);
    g0 = (int32_t*)ctx->buf(kSlotGen + 5, sizeof(int32_t) * total_cap);
    if (!a0 || !i0 || !g0) return set_error(ctx, SCLS_ERR_CUDA, "generator allocation failed");
    SCLS_CUDA(cudaMemcpyAsync(d_capoff, cap_off.data(), sizeof(int64_t) * (n_specs + 1), cudaMemcpyHostToDevice, s));
    gen_kernel<<<div_up(n_specs, kGenWarps), kGenWarps * 32, 0, s>>>(n_specs, d_specs, d_capoff, a0, i0, g0, d_cnt);
    SCLS_LAUNCHED();
    SCLS_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int64_t) * n_specs, cudaMemcpyDeviceToHost, s));
    SCLS_CUDA(cudaStreamSynchronize(s));
    bool over = false;
    for (int t = 0; t < n_specs; ++t) over |= cnt[t] > cap_off[t + 1] - cap_off[t];
    if (!over) break;
    if (attempt == 1) return set_error(ctx, SCLS_ERR_CUDA, "device generator: capacity retry failed");
    for (int t = 0; t < n_specs; ++t) cap_off[t + 1] = cap_off[t] + std::max<int64_t>(cnt[t], 1);
  }
  h_off.assign(n_specs + 1, 0);
  for (int t = 0; t < n_specs; ++t) h_off[t + 1] = h_off[t] + cnt[t];
  const int64_t total = std::max<int64_t>(h_off[n_specs], 1);
  double* a1 = (double*)ctx->buf(kSlotGen + 6, sizeof(double) * total);
  int32_t* i1 = (int32_t*)ctx->buf(kSlotGen + 7, sizeof(int32_t) * total);
  int32_t* g1 = (int32_t*)ctx->buf(kSlotGen + 8, sizeof(int32_t) * total);
  int64_t* d_off = (int64_t*)ctx->buf(kSlotGen + 9, sizeof(int64_t) * (n_specs + 1));
  if (!a1 || !i1 || !g1 || !d_off) return set_error(ctx, SCLS_ERR_CUDA, "generator allocation failed");
  SCLS_CUDA(cudaMemcpyAsync(d_off, h_off.data(), sizeof(int64_t) * (n_specs + 1), cudaMemcpyHostToDevice, s));
  if (h_off[n_specs] > 0) {
    compact_kernel<<<n_specs, 256, 0, s>>>(n_specs, d_capoff, d_off, a0, i0, g0, a1, i1, g1);
    SCLS_LAUNCHED();
  }
  *arr = a1;
  *inp = i1;
  *gen = g1;
  return SCLS_OK;
}

}  // namespace scls

using namespace scls;

extern "C" scls_status scls_generate_batch(scls_ctx* ctx, int32_t n_specs, const scls_workload_spec* specs,
                                           int64_t cap, int64_t* req_offset, double* arrival, int32_t* input_len,
                                           int32_t* gen_len, int32_t mem) {
  if (!ctx) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null context");
  ctx->err.clear();
  ctx->err_request = -1;
  ctx->launches = 0;
  std::fill(ctx->timings, ctx->timings + 8, 0.f);
  SCLS_CUDA(cudaSetDevice(ctx->device));
  if (n_specs < 0 || (n_specs > 0 && (!specs || !req_offset)) || cap < 0 ||
      (cap > 0 && (!arrival || !input_len || !gen_len)))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n_specs == 0) {
    if (mem == SCLS_MEM_DEVICE) SCLS_CUDA(cudaMemset(req_offset, 0, sizeof(int64_t)));
    else req_offset[0] = 0;
    return SCLS_OK;
  }
  cudaStream_t s = ctx->stream;
  SCLS_CUDA(cudaEventRecord(ctx->ev[0], s));
  std::vector<int64_t> h_off;
  double* a = nullptr;
  int32_t* in = nullptr;
  int32_t* g = nullptr;
  scls_status st = generate_device(ctx, n_specs, specs, h_off, &a, &in, &g);
  if (st) return st;
  const int64_t total = h_off[n_specs];
  const cudaMemcpyKind k = mem == SCLS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  SCLS_CUDA(cudaMemcpyAsync(req_offset, h_off.data(), sizeof(int64_t) * (n_specs + 1),
                            mem == SCLS_MEM_DEVICE ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost, s));
  if (total > cap) {
    SCLS_CUDA(cudaStreamSynchronize(s));
    return set_error(ctx, SCLS_ERR_CAPACITY, "generated requests exceed cap");
  }
  if (total > 0) {
    SCLS_CUDA(cudaMemcpyAsync(arrival, a, sizeof(double) * total, k, s));
    SCLS_CUDA(cudaMemcpyAsync(input_len, in, sizeof(int32_t) * total, k, s));
    SCLS_CUDA(cudaMemcpyAsync(gen_len, g, sizeof(int32_t) * total, k, s));
  }
  SCLS_CUDA(cudaEventRecord(ctx->ev[1], s));
  SCLS_CUDA(cudaStreamSynchronize(s));
  cudaEventElapsedTime(&ctx->timings[7], ctx->ev[0], ctx->ev[1]);
  ctx->timings[0] = ctx->timings[7];
  return SCLS_OK;
}

extern "C" scls_status scls_debug_log(scls_ctx* ctx, int64_t n, const double* x, double* y, int32_t mem) {
  return scls_debug_libm(ctx, 0, n, x, y, mem);
}

extern "C" scls_status scls_debug_libm(scls_ctx* ctx, int32_t fn, int64_t n, const double* x, double* y,
                                       int32_t mem) {
  if (!ctx) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null context");
  SCLS_CUDA(cudaSetDevice(ctx->device));
  if (fn < 0 || fn > 2 || n < 0 || (n > 0 && (!x || !y)))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n == 0) return SCLS_OK;
  cudaStream_t s = ctx->stream;
  const double* dx = x;
  double* dy = y;
  if (mem == SCLS_MEM_HOST) {
    double* b = (double*)ctx->buf(kSlotStage + 0, sizeof(double) * 2 * n);
    if (!b) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
    SCLS_CUDA(cudaMemcpyAsync(b, x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    dx = b;
    dy = b + n;
  }
  libm_kernel<<<std::min(div_up(n, 256), ctx->sm_count * 8), 256, 0, s>>>(fn, n, dx, dy);
  SCLS_LAUNCHED();
  if (mem == SCLS_MEM_HOST) SCLS_CUDA(cudaMemcpyAsync(y, dy, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  SCLS_CUDA(cudaStreamSynchronize(s));
  return SCLS_OK;
}
