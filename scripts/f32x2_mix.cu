// Packed/scalar fp32 mix on sm_100a: fp32 operations per second when each
// iteration issues NP packed adds (add.rn.f32x2, 2 ops each) and NS scalar
// FFMA over 8 independent chains, a full chip of warps. Tells whether
// FADD2 mixed with scalar FFMA keeps the FP32 pipe's 128 ops/clk/SM while
// using fewer issue slots. Development microbenchmark.
#include <cstdio>
#include <cuda_runtime.h>

template <int NP, int NS, int NM>
__global__ void k(float* out, int iters, float s) {
  float a[8];
  unsigned long long p[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = ((unsigned long long)__float_as_uint(a[i]) << 32) | __float_as_uint(a[i + 4]);
  const unsigned long long ps = ((unsigned long long)__float_as_uint(s) << 32) | __float_as_uint(s);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int j = 0; j < NP; ++j) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[j & 3]) : "l"(ps));
#pragma unroll
      for (int j = 0; j < NS; ++j) a[j & 7] = __fmaf_rn(a[j & 7], s, s);
#pragma unroll
      for (int j = 0; j < NM; ++j) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a[(j + 3) & 7]));
    }
  }
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += a[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc += __uint_as_float((unsigned)p[i]) + __uint_as_float((unsigned)(p[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int NP, int NS, int NM>
void run(float* d, int blocks, int threads, int iters, double clk_ghz) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<NP, NS, NM><<<blocks, threads>>>(d, 10, 0.999f);
  cudaEventRecord(e0);
  k<NP, NS, NM><<<blocks, threads>>>(d, iters, 0.999f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double n = (double)blocks * threads * iters * 8;
  const double ops = n * (2 * NP + NS), inst = n * (NP + NS + NM);
  printf("packed %2d scalar %2d mufu %d : %.2f T fp32-op/s, %.2f T thread-inst/s, %.1f%% of 37.2 T op\n", NP, NS, NM,
         ops / ms / 1e9, inst / ms / 1e9, 100 * ops / ms / 1e9 / 37.2);
}

int main() {
  float* d;
  const int blocks = 148 * 4, threads = 512;
  cudaMalloc(&d, blocks * threads * 4);
  const int it = 4000;
  run<0, 24, 0>(d, blocks, threads, it, 1.9);
  run<12, 0, 0>(d, blocks, threads, it, 1.9);
  run<4, 16, 0>(d, blocks, threads, it, 1.9);
  run<7, 10, 0>(d, blocks, threads, it, 1.9);
  run<8, 8, 0>(d, blocks, threads, it, 1.9);
  run<0, 23, 1>(d, blocks, threads, it, 1.9);
  run<7, 9, 1>(d, blocks, threads, it, 1.9);
  run<4, 15, 1>(d, blocks, threads, it, 1.9);
  return 0;
}
