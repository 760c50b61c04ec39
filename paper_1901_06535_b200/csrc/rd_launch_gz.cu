// gz_kernel instantiations, fp32 and fp64 (see rd_launch.h).
#include "rd_gz.cuh"
#include "rd_launch.h"

namespace rdl {
namespace {

template <typename T, bool REACT, int MODE, int M, bool PROBE, int NT>
cudaError_t go_nt(const rdk::GzArgs<T>& ga, unsigned grid, size_t smem, cudaStream_t st, int* occ) {
  auto fn = rdk::gz_kernel<T, REACT, MODE, M, PROBE, NT>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, NT, smem);
  // cooperative: every tile resident at once (tiles wait on their neighbours)
  void* args[] = {const_cast<rdk::GzArgs<T>*>(&ga)};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(NT), args, smem, st);
}

template <typename T, bool REACT, int MODE, int M, bool PROBE>
cudaError_t go(const rdk::GzArgs<T>& ga, unsigned grid, size_t smem, cudaStream_t st, int* occ) {
  return ga.nt == 256 ? go_nt<T, REACT, MODE, M, PROBE, 256>(ga, grid, smem, st, occ)
                      : go_nt<T, REACT, MODE, M, PROBE, rdk::kGzThreads>(ga, grid, smem, st, occ);
}

template <typename T, bool REACT, int MODE, int M>
cudaError_t by_probe(const rdk::GzArgs<T>& ga, unsigned grid, size_t smem, cudaStream_t st, int* occ) {
  return ga.probe_every ? go<T, REACT, MODE, M, true>(ga, grid, smem, st, occ)
                        : go<T, REACT, MODE, M, false>(ga, grid, smem, st, occ);
}

// m: zone vectors per thread (1 .. kGzMaxSlots)
template <typename T, bool REACT, int MODE>
cudaError_t by_m(const rdk::GzArgs<T>& ga, int m, unsigned grid, size_t smem, cudaStream_t st, int* occ) {
  static_assert(rdk::kGzMaxSlots == 6, "one case per slot count");
  switch (m) {
    case 1: return by_probe<T, REACT, MODE, 1>(ga, grid, smem, st, occ);
    case 2: return by_probe<T, REACT, MODE, 2>(ga, grid, smem, st, occ);
    case 3: return by_probe<T, REACT, MODE, 3>(ga, grid, smem, st, occ);
    case 4: return by_probe<T, REACT, MODE, 4>(ga, grid, smem, st, occ);
    case 5: return by_probe<T, REACT, MODE, 5>(ga, grid, smem, st, occ);
    case 6: return by_probe<T, REACT, MODE, 6>(ga, grid, smem, st, occ);
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t dispatch(const rdk::GzArgs<T>& ga, int mode, bool react, int m, unsigned grid, size_t smem,
                     cudaStream_t st, int* occ) {
  if (!react) return by_m<T, false, rdk::MODE_PRECISE>(ga, m, grid, smem, st, occ);
  if (mode == rdk::MODE_FOLD) return by_m<T, true, rdk::MODE_FOLD>(ga, m, grid, smem, st, occ);
  if constexpr (sizeof(T) == 4) {
    if (mode == rdk::MODE_FOLD_DIV4) return by_m<T, true, rdk::MODE_FOLD_DIV4>(ga, m, grid, smem, st, occ);
    if (mode == rdk::MODE_FOLD_DIV4_NG) return by_m<T, true, rdk::MODE_FOLD_DIV4_NG>(ga, m, grid, smem, st, occ);
  }
  return cudaErrorInvalidValue;  // gz_kernel serves the fast modes only
}

}  // namespace

cudaError_t launch_gz(const rdk::GzArgs<float>& a, int mode, bool react, int m, unsigned grid, size_t smem,
                      cudaStream_t st, int* occ) {
  return dispatch<float>(a, mode, react, m, grid, smem, st, occ);
}

cudaError_t launch_gz(const rdk::GzArgs<double>& a, int mode, bool react, int m, unsigned grid, size_t smem,
                      cudaStream_t st, int* occ) {
  return dispatch<double>(a, mode, react, m, grid, smem, st, occ);
}

}  // namespace rdl

#ifdef RD_GZ_PROF
// measurement build only: copy (and clear) the per-CTA phase cycle counts
extern "C" int rd_gz_prof_dump(unsigned long long* out, int n) {
  if (n > 2048 * 8) n = 2048 * 8;
  if (cudaMemcpyFromSymbol(out, rdk::g_gz_prof, n * sizeof(unsigned long long)) != cudaSuccess) return -1;
  static unsigned long long zero[2048 * 8];
  return cudaMemcpyToSymbol(rdk::g_gz_prof, zero, sizeof zero) == cudaSuccess ? 0 : -1;
}
#endif
