// Dependent-chain latency of warp-wide primitives on sm_100a (cycles/op).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_warpops tools/ubench_warpops.cu
#include <cstdio>
#include <cstdint>
#define N 2048
template <int OP>
__global__ void k(unsigned seed, unsigned long long* out, unsigned* sink) {
  unsigned x = seed ^ threadIdx.x;
  const uint64_t y = ((uint64_t)seed << 32) | (seed * 7u);
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    if (OP == 0) x = __reduce_min_sync(0xffffffffu, x) + threadIdx.x;
    else if (OP == 1) x = __reduce_or_sync(0xffffffffu, x) ^ threadIdx.x;
    else if (OP == 2) x = __match_any_sync(0xffffffffu, y + x) ^ threadIdx.x;
    else if (OP == 3) x = __match_any_sync(0xffffffffu, x) ^ threadIdx.x;
    else if (OP == 4) x = __ballot_sync(0xffffffffu, x & 1) ^ threadIdx.x;
    else if (OP == 5) x = __shfl_sync(0xffffffffu, x, (x + 1) & 31) + 1;
    else if (OP == 6) x = __any_sync(0xffffffffu, x & 1) + x * 3;
    else if (OP == 7) x = x * 3 + threadIdx.x;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[OP] = (unsigned long long)(t1 - t0);
  sink[threadIdx.x] = x;
}
template <int OP>
void run(unsigned long long* d, unsigned* s, const char* name) {
  k<OP><<<1, 32>>>(12345, d, s);
  k<OP><<<1, 32>>>(12345, d, s);
  unsigned long long h[8];
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("%-14s %.1f cycles/op (incl. the dependent int op)\n", name, (double)h[OP] / N);
}
int main() {
  unsigned long long* d; unsigned* s; cudaMalloc(&d, 64); cudaMalloc(&s, 128);
  run<0>(d, s, "redux.min");
  run<1>(d, s, "redux.or");
  run<2>(d, s, "match.any.b64");
  run<3>(d, s, "match.any.b32");
  run<4>(d, s, "ballot");
  run<5>(d, s, "shfl.idx");
  run<6>(d, s, "vote.any");
  run<7>(d, s, "imad");
  return 0;
}
