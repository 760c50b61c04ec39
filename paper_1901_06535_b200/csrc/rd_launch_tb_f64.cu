// tb_kernel / lp_kernel instantiations and their occupancy, fp64 (see rd_launch.h).
#include "rd_launch_tb.cuh"

namespace rdl {
cudaError_t launch_tb(const rdk::TBArgs<double>& a, int K, int mode, bool react, bool lp, int var, bool uphi,
                      unsigned grid, cudaStream_t st) {
  return detail::dispatch<double>(a, K, mode, react, lp, var, uphi, grid, st, nullptr);
}
int occupancy_tb_f64(int K, int mode, bool react, bool lp, int var, bool uphi) {
  return detail::occupancy<double>(K, mode, react, lp, var, uphi);
}
}  // namespace rdl
