// ubench_chain.cu — latency floors of the DP chain's building blocks on the
// local GPU (single warp, dependent chains), in SM cycles and ns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool lei(double a, double b) { return __double_as_longlong(a) <= __double_as_longlong(b); }

template <int MODE>
__global__ void chain(const double* __restrict__ c, double* out, long long* cyc, unsigned long long* ns, int iters) {
  const int lane = threadIdx.x;
  double acc = c[lane], t = c[lane + 32], acc2 = c[lane + 64];
  int kb = 0;
  const double cc = c[lane + 64], c1 = c[lane + 65];
  __syncwarp();
  const long long c0 = clock64();
  const uint64_t g0 = gtime();
#pragma unroll 8
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {  // dependent DADD
      t = __dadd_rn(t, cc);
    } else if (MODE == 1) {  // dadd + dsetp/sel
      const double cand = __dadd_rn(t, cc);
      const bool tk = cand <= acc;
      acc = tk ? cand : acc;
      kb = tk ? i : kb;
      t = acc;
    } else if (MODE == 2) {  // dadd + int64 compare/sel
      const double cand = __dadd_rn(t, cc);
      const bool tk = lei(cand, acc);
      acc = tk ? cand : acc;
      kb = tk ? i : kb;
      t = acc;
    } else if (MODE == 3) {  // shfl.f64 (register index)
      t = __shfl_sync(0xffffffffu, t, i & 31);
    } else if (MODE == 4) {  // DP step, dsetp
      const double cand = __dadd_rn(t, cc);
      const bool tk = cand <= acc;
      acc = tk ? cand : acc;
      kb = tk ? i : kb;
      t = __shfl_sync(0xffffffffu, acc, i & 31);
    } else if (MODE == 5) {  // DP step, int compare
      const double cand = __dadd_rn(t, cc);
      const bool tk = lei(cand, acc);
      acc = tk ? cand : acc;
      kb = tk ? i : kb;
      t = __shfl_sync(0xffffffffu, acc, i & 31);
    } else if (MODE == 6) {  // 2-row lookahead: dadd, dadd, int-min (counts 2 rows)
      const double a = __dadd_rn(__dadd_rn(t, cc), c1);
      t = lei(a, acc2) ? a : acc2;
      acc2 = __dadd_rn(acc2, cc);
    } else {  // value-only DP step: dadd, int-min, shfl
      const double cand = __dadd_rn(t, cc);
      acc = lei(cand, acc) ? cand : acc;
      t = __shfl_sync(0xffffffffu, acc, i & 31);
    }
  }
  const uint64_t g1 = gtime();
  const long long c1_ = clock64();
  out[lane] = t + acc + kb + acc2;
  if (lane == 0) {
    cyc[MODE] = c1_ - c0;
    ns[MODE] = g1 - g0;
  }
}

int main() {
  double *c, *out;
  long long* cyc;
  unsigned long long* ns;
  cudaMalloc(&c, 128 * 8);
  cudaMalloc(&out, 32 * 8);
  cudaMallocManaged(&cyc, 128);
  cudaMallocManaged(&ns, 128);
  double h[128];
  for (int i = 0; i < 128; ++i) h[i] = 1e-3 * (i + 1);
  cudaMemcpy(c, h, sizeof h, cudaMemcpyHostToDevice);
  const int iters = 1 << 20;
  for (int rep = 0; rep < 2; ++rep) {
    chain<0><<<1, 32>>>(c, out, cyc, ns, iters);
    chain<1><<<1, 32>>>(c, out, cyc, ns, iters);
    chain<2><<<1, 32>>>(c, out, cyc, ns, iters);
    chain<3><<<1, 32>>>(c, out, cyc, ns, iters);
    chain<4><<<1, 32>>>(c, out, cyc, ns, iters);
    chain<5><<<1, 32>>>(c, out, cyc, ns, iters);
    chain<6><<<1, 32>>>(c, out, cyc, ns, iters);
    chain<7><<<1, 32>>>(c, out, cyc, ns, iters);
    cudaDeviceSynchronize();
  }
  const char* names[8] = {"dadd", "dadd+dsetp/sel", "dadd+i64cmp/sel", "shfl.f64",
                          "step dsetp (dadd,cmp,sel,shfl)", "step i64cmp", "2-row lookahead (per 2 rows)",
                          "value-only step i64"};
  for (int m = 0; m < 8; ++m)
    printf("%-34s %7.2f cyc/iter  %7.3f ns/iter  (%.0f MHz)\n", names[m], (double)cyc[m] / iters,
           (double)ns[m] / iters, (double)cyc[m] / (double)ns[m] * 1e3);
  return 0;
}
