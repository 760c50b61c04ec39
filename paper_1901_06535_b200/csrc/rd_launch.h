// rd_launch.h — the stencil-kernel launchers, instantiated in their own
// translation units (rd_launch_tb_f32.cu, rd_launch_tb_f64.cu,
// rd_launch_cr.cu) so the heavy template instantiations compile in parallel.
// The runtime (rd_runtime.cu) computes the arguments and the launch geometry.
#pragma once
#include <cuda_runtime.h>

#include "rd_gz.cuh"
#include "rd_kernels.cuh"

namespace rdl {

// mode: rdk::MODE_*; react: reaction on (else diffusion only, MODE_PRECISE);
// lp: the level-parallel variant (K <= 4; CTAs of 32*K threads), else
// tb_kernel (one-warp CTAs). An unsupported combination returns
// cudaErrorInvalidValue.
// var: rdk::TB_FULL / TB_LEAN / TB_CHECKED (tb_kernel variants).
// uphi: the uniform-phi tb_kernel (TBArgs::phi_u), only where tb_uphi_ok.
int occupancy_tb_f32(int K, int mode, bool react, bool lp, int var, bool uphi);  // resident CTAs per SM (>= 1)
int occupancy_tb_f64(int K, int mode, bool react, bool lp, int var, bool uphi);
inline int occupancy_tb(bool f32, int K, int mode, bool react, bool lp, int var, bool uphi) {
  return f32 ? occupancy_tb_f32(K, mode, react, lp, var, uphi) : occupancy_tb_f64(K, mode, react, lp, var, uphi);
}
cudaError_t launch_tb(const rdk::TBArgs<float>& a, int K, int mode, bool react, bool lp, int var, bool uphi,
                      unsigned grid, cudaStream_t st);
cudaError_t launch_tb(const rdk::TBArgs<double>& a, int K, int mode, bool react, bool lp, int var, bool uphi,
                      unsigned grid, cudaStream_t st);
// the uniform-phi tb_kernel is instantiated for K <= 4, reaction on, in the
// default fast mode of the precision (fp32: guard-free 4-op division; fp64: FOLD)
constexpr bool tb_uphi_depth(bool f32, int K) { return K <= 4 || (f32 && K <= 7); }
inline bool tb_uphi_ok(bool f32, int K, int mode, bool react, bool lp) {
  return tb_uphi_depth(f32, K) && react && !lp && mode == (f32 ? rdk::MODE_FOLD_DIV4_NG : rdk::MODE_FOLD);
}

// cr_kernel over `batch` clusters of cs CTAs with `smem` dynamic shared memory
// (pal: phi as palette indices). query: return the co-resident cluster count
// in *clusters instead of launching.
cudaError_t launch_cr(const rdk::CrArgs<float>& a, int mode, bool react, bool pal, int cs, unsigned batch,
                      size_t smem, cudaStream_t st, bool query, int* clusters);
cudaError_t launch_cr(const rdk::CrArgs<double>& a, int mode, bool react, bool pal, int cs, unsigned batch,
                      size_t smem, cudaStream_t st, bool query, int* clusters);

// gz_kernel over `grid` tiles (cooperative launch: all resident) with
// `smem` dynamic shared memory, m zone vectors per thread; occ: return the
// resident CTAs per SM in *occ instead of launching.
cudaError_t launch_gz(const rdk::GzArgs<float>& a, int mode, bool react, int m, unsigned grid, size_t smem,
                      cudaStream_t st, int* occ);
cudaError_t launch_gz(const rdk::GzArgs<double>& a, int mode, bool react, int m, unsigned grid, size_t smem,
                      cudaStream_t st, int* occ);

}  // namespace rdl
