// Load-path microbenchmark for gz_kernel's LL exchange: 144 CTAs x 512
// threads each read an L2-resident 64 KB region (8-byte words, consecutive
// lanes consecutive words) with different load flavours, back to back; the
// cycles per pass tell whether strong (.relaxed.gpu) loads coalesce.
// Development microbenchmark (scripts/, not part of librd).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(const unsigned long long* src, unsigned long long* out, int words, int passes, long long* cyc) {
  const unsigned long long* p = src + (size_t)blockIdx.x * words;
  unsigned long long acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < passes; ++it) {
    for (int i = threadIdx.x * (MODE == 2 ? 2 : 1); i < words; i += blockDim.x * (MODE == 2 ? 2 : 1)) {
      unsigned long long x, y = 0;
      if (MODE == 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p + i));
      if (MODE == 1) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(x) : "l"(p + i));
      if (MODE == 2) asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(p + i));
      if (MODE == 3) asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(x) : "l"(p + i));
      acc += x + y;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / passes;
  if (acc == 42) out[0] = acc;
}

template <int MODE>
void run(const char* name, const unsigned long long* d, unsigned long long* o, long long* cyc, int words) {
  k<MODE><<<144, 512>>>(d, o, words, 2, cyc);
  k<MODE><<<144, 512>>>(d, o, words, 20, cyc);
  cudaDeviceSynchronize();
  long long h[144];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 144; ++i) m += h[i];
  printf("%-22s %6d words/CTA: %8.0f cycles per pass (%.1f B/cycle/SM)\n", name, words, m / 144, words * 8.0 / (m / 144));
}

int main() {
  const int words = 8192;  // 64 KB per CTA
  unsigned long long *d, *o;
  long long* cyc;
  cudaMalloc(&d, (size_t)144 * words * 8);
  cudaMemset(d, 1, (size_t)144 * words * 8);
  cudaMalloc(&o, 64);
  cudaMalloc(&cyc, 144 * 8);
  for (int w : {3328, 8192}) {
    run<0>("ld.relaxed.gpu.u64", d, o, cyc, w);
    run<1>("ld.global.cg.u64", d, o, cyc, w);
    run<2>("ld.relaxed.gpu.v2.u64", d, o, cyc, w);
    run<3>("ld.volatile.u64", d, o, cyc, w);
  }
  return 0;
}
