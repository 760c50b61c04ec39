// cr_kernel instantiations, fp32 and fp64 (see rd_launch.h).
#include "rd_launch.h"

namespace rdl {
namespace {

template <typename T, bool REACT, int MODE, bool PAL, bool PROBE>
cudaError_t go_p(const rdk::CrArgs<T>& ca, int cs, unsigned batch, size_t smem, cudaStream_t st, bool query,
                 int* clusters) {
  constexpr int nt = rdk::cr_threads<T>();
  auto fn = rdk::cr_kernel<T, REACT, MODE, nt, PAL, PROBE>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)cs, batch, 1);
  cfg.blockDim = dim3((unsigned)nt, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (query) return cudaOccupancyMaxActiveClusters(clusters, fn, &cfg);
  return cudaLaunchKernelEx(&cfg, fn, ca);
}

// segments with a probe due inside take the variant that evaluates probes in
// its step loop; the others keep the loop without that code (the latency-bound
// small bands pay for every instruction on the step's critical path)
template <typename T, bool REACT, int MODE, bool PAL>
cudaError_t go(const rdk::CrArgs<T>& ca, int cs, unsigned batch, size_t smem, cudaStream_t st, bool query,
               int* clusters) {
  return ca.probe_every ? go_p<T, REACT, MODE, PAL, true>(ca, cs, batch, smem, st, query, clusters)
                        : go_p<T, REACT, MODE, PAL, false>(ca, cs, batch, smem, st, query, clusters);
}

template <typename T, bool PAL>
cudaError_t by_mode(const rdk::CrArgs<T>& ca, int mode, bool react, int cs, unsigned batch, size_t smem,
                    cudaStream_t st, bool query, int* clusters) {
  if (!react) return go<T, false, rdk::MODE_PRECISE, PAL>(ca, cs, batch, smem, st, query, clusters);
  if (mode == rdk::MODE_FOLD) return go<T, true, rdk::MODE_FOLD, PAL>(ca, cs, batch, smem, st, query, clusters);
  if constexpr (sizeof(T) == 4) {
    if (mode == rdk::MODE_FOLD_DIV4)
      return go<T, true, rdk::MODE_FOLD_DIV4, PAL>(ca, cs, batch, smem, st, query, clusters);
    if (mode == rdk::MODE_FOLD_DIV4_NG)
      return go<T, true, rdk::MODE_FOLD_DIV4_NG, PAL>(ca, cs, batch, smem, st, query, clusters);
  }
  return cudaErrorInvalidValue;  // cr_kernel serves the fast modes only
}

template <typename T>
cudaError_t dispatch(const rdk::CrArgs<T>& ca, int mode, bool react, bool pal, int cs, unsigned batch, size_t smem,
                     cudaStream_t st, bool query, int* clusters) {
  return pal ? by_mode<T, true>(ca, mode, react, cs, batch, smem, st, query, clusters)
             : by_mode<T, false>(ca, mode, react, cs, batch, smem, st, query, clusters);
}

}  // namespace

cudaError_t launch_cr(const rdk::CrArgs<float>& a, int mode, bool react, bool pal, int cs, unsigned batch,
                      size_t smem, cudaStream_t st, bool query, int* clusters) {
  return dispatch<float>(a, mode, react, pal, cs, batch, smem, st, query, clusters);
}

cudaError_t launch_cr(const rdk::CrArgs<double>& a, int mode, bool react, bool pal, int cs, unsigned batch,
                      size_t smem, cudaStream_t st, bool query, int* clusters) {
  return dispatch<double>(a, mode, react, pal, cs, batch, smem, st, query, clusters);
}

}  // namespace rdl
