// Exhaustive check of the fast fp32 division used by the product kernels
// (rdk::div_fast_f32) against IEEE div.rn (__fdiv_rn) on the reaction's real
// input domain: for EVERY finite fp32 C, a = RN(C - q), b = RN(C + q).
// Counts mismatches inside the guarded range |b| in [2^-60, 2^126] (must be 0)
// and outside it (informational: those inputs are replayed precisely).
#include <cstdio>
#include <cstdlib>
#include "../../paper_1901_06535_b200/csrc/rd_kernels.cuh"

__global__ void check(float q, unsigned long long* bad_in, unsigned long long* bad_out, unsigned long long* tested,
                      unsigned int* first_bad) {
  unsigned long long n_in = 0, n_out = 0, n = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < (1ull << 32);
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const float C = __uint_as_float((unsigned int)i);
    if (!isfinite(C)) continue;
    const float a = __fsub_rn(C, q), b = __fadd_rn(C, q);
    const float f = rdk::div_fast_f32(a, b), r = __fdiv_rn(a, b);
    ++n;
    const bool same = __float_as_uint(f) == __float_as_uint(r) || (isnan(f) && isnan(r));
    if (!same) {
      if (fabsf(b) >= rdk::kFastDivMinB && fabsf(b) <= 0x1p126f) {
        ++n_in;
        atomicMin(first_bad, (unsigned int)i);
      } else {
        ++n_out;
      }
    }
  }
  atomicAdd(bad_in, n_in);
  atomicAdd(bad_out, n_out);
  atomicAdd(tested, n);
}

int main(int argc, char** argv) {
  const float q = argc > 1 ? (float)atof(argv[1]) : (float)0.002;
  unsigned long long* d;
  unsigned int* fb;
  cudaMalloc(&d, 3 * sizeof(unsigned long long));
  cudaMalloc(&fb, sizeof(unsigned int));
  cudaMemset(d, 0, 3 * sizeof(unsigned long long));
  cudaMemset(fb, 0xff, sizeof(unsigned int));
  check<<<148 * 16, 256>>>(q, d, d + 1, d + 2, fb);
  unsigned long long h[3];
  unsigned int hf;
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaMemcpy(&hf, fb, sizeof hf, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("{\"q\": %.9g, \"tested\": %llu, \"mismatch_guarded\": %llu, \"mismatch_unguarded\": %llu, \"first_bad_C_bits\": %u, \"cuda\": \"%s\"}\n",
         q, h[2], h[0], h[1], hf, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
