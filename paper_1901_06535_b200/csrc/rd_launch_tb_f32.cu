// tb_kernel / lp_kernel instantiations and their occupancy, fp32 (see rd_launch.h).
#include "rd_launch_tb.cuh"

namespace rdl {
cudaError_t launch_tb(const rdk::TBArgs<float>& a, int K, int mode, bool react, bool lp, int var, bool uphi,
                      unsigned grid, cudaStream_t st) {
  return detail::dispatch<float>(a, K, mode, react, lp, var, uphi, grid, st, nullptr);
}
int occupancy_tb_f32(int K, int mode, bool react, bool lp, int var, bool uphi) {
  return detail::occupancy<float>(K, mode, react, lp, var, uphi);
}
}  // namespace rdl
