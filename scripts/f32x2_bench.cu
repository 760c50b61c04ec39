// Throughput of packed fp32 (FADD2/FMUL2/FFMA2, PTX *.rn.f32x2) vs scalar
// FADD/FMUL/FFMA on sm_100a: the same number of fp32 operations per thread,
// 8 independent chains, a full chip of warps. Development microbenchmark.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  return ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(a);
}

template <int MODE>  // 0 scalar fma, 1 packed fma, 2 scalar add, 3 packed add, 4 scalar mul, 5 packed mul
__global__ void k(float* out, int iters, float s) {
  float a[8];
  unsigned long long p[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = pk(a[2 * i], a[2 * i + 1]);
  const unsigned long long ps = pk(s, s);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __fmaf_rn(a[i], s, s);
      } else if (MODE == 1) {
#pragma unroll
        for (int i = 0; i < 4; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[i]) : "l"(ps));
      } else if (MODE == 2) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __fadd_rn(a[i], s);
      } else if (MODE == 3) {
#pragma unroll
        for (int i = 0; i < 4; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(ps));
      } else if (MODE == 4) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __fmul_rn(a[i], s);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(ps));
      }
    }
  }
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += a[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc += __uint_as_float((unsigned)p[i]) + __uint_as_float((unsigned)(p[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(const char* name, float* d, int blocks, int threads, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<blocks, threads>>>(d, 10, 0.999f);
  cudaEventRecord(e0);
  k<MODE><<<blocks, threads>>>(d, iters, 0.999f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)blocks * threads * iters * 16 * 8;  // fp32 operations
  printf("%-14s %8.3f ms  %7.2f T fp32-op/s\n", name, ms, ops / (ms * 1e-3) / 1e12);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 8, iters = 4000;
  float* d;
  cudaMalloc(&d, sizeof(float) * blocks * threads);
  run<0>("ffma scalar", d, blocks, threads, iters);
  run<1>("ffma2 packed", d, blocks, threads, iters);
  run<2>("fadd scalar", d, blocks, threads, iters);
  run<3>("fadd2 packed", d, blocks, threads, iters);
  run<4>("fmul scalar", d, blocks, threads, iters);
  run<5>("fmul2 packed", d, blocks, threads, iters);
  return 0;
}
