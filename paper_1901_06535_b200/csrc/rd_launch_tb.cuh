// rd_launch_tb.cuh — tb_kernel / lp_kernel launch dispatch for one precision
// (included by rd_launch_tb_f32.cu and rd_launch_tb_f64.cu).
#pragma once
#include <map>
#include <mutex>
#include <tuple>

#include "rd_launch.h"

#include <cstdlib>

namespace rdl {
namespace detail {

// RD_TB_DSMEM=bytes: dynamic shared memory added to every tb_kernel launch (and
// to its occupancy query). Measurement only: it caps the resident one-warp
// CTAs per SM without touching the kernel (occupancy sweep).
inline size_t tb_dsmem() {
  static const size_t v = [] {
    const char* e = std::getenv("RD_TB_DSMEM");
    return e ? (size_t)std::strtoul(e, nullptr, 10) : (size_t)0;
  }();
  return v;
}

// the default fast mode of each precision (fp32 Table-1: guard-free 4-op
// division; fp64: FOLD) also has the LEAN / CHECKED tb_kernel variants
template <typename T, int MODE>
constexpr bool has_variants() {
  return sizeof(T) == 4 ? MODE == rdk::MODE_FOLD_DIV4_NG : MODE == rdk::MODE_FOLD;
}

template <typename T, int K, bool REACT, int MODE, int VAR>
cudaError_t go_uphi(const rdk::TBArgs<T>& a, unsigned grid, cudaStream_t st, int* occ) {
  constexpr int V = 16 / (int)sizeof(T);
  if (occ)
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, rdk::tb_kernel<T, K, V, REACT, MODE, VAR, true>, 32,
                                                         tb_dsmem());
  rdk::tb_kernel<T, K, V, REACT, MODE, VAR, true><<<grid, 32, tb_dsmem(), st>>>(a);
  return cudaGetLastError();
}

// uphi: the uniform-phi tb_kernel (TBArgs::phi_u), instantiated for K <= 4 in
// the default fast mode of each precision (rdl::tb_uphi_ok).
template <typename T, int K, bool REACT, int MODE>
cudaError_t go(const rdk::TBArgs<T>& a, bool lp, int var, bool uphi, unsigned grid, cudaStream_t st, int* occ) {
  constexpr int V = 16 / (int)sizeof(T);
  if (uphi) {
    if constexpr (rdl::tb_uphi_depth(sizeof(T) == 4, K) && REACT && has_variants<T, MODE>()) {
      if (lp) return cudaErrorInvalidValue;
      switch (var) {
        case rdk::TB_LEAN: return go_uphi<T, K, REACT, MODE, rdk::TB_LEAN>(a, grid, st, occ);
        case rdk::TB_CHECKED: return go_uphi<T, K, REACT, MODE, rdk::TB_CHECKED>(a, grid, st, occ);
        default: return go_uphi<T, K, REACT, MODE, rdk::TB_FULL>(a, grid, st, occ);
      }
    }
    return cudaErrorInvalidValue;
  }
  if constexpr (REACT && has_variants<T, MODE>()) {
    if (!lp && var == rdk::TB_LEAN) {
      if (occ)
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, rdk::tb_kernel<T, K, V, REACT, MODE, rdk::TB_LEAN>,
                                                             32, tb_dsmem());
      rdk::tb_kernel<T, K, V, REACT, MODE, rdk::TB_LEAN><<<grid, 32, tb_dsmem(), st>>>(a);
      return cudaGetLastError();
    }
    if (!lp && var == rdk::TB_CHECKED) {
      if (occ)
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            occ, rdk::tb_kernel<T, K, V, REACT, MODE, rdk::TB_CHECKED>, 32, tb_dsmem());
      rdk::tb_kernel<T, K, V, REACT, MODE, rdk::TB_CHECKED><<<grid, 32, tb_dsmem(), st>>>(a);
      return cudaGetLastError();
    }
  }
  if (lp) {
    if constexpr (K <= 4) {
      if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, rdk::lp_kernel<T, K, V, REACT, MODE>, 32 * K, 0);
      rdk::lp_kernel<T, K, V, REACT, MODE><<<grid, 32 * K, 0, st>>>(a);
      return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
  }
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, rdk::tb_kernel<T, K, V, REACT, MODE>, 32, tb_dsmem());
  rdk::tb_kernel<T, K, V, REACT, MODE><<<grid, 32, tb_dsmem(), st>>>(a);
  return cudaGetLastError();
}

template <typename T, bool REACT, int MODE>
cudaError_t by_k(const rdk::TBArgs<T>& a, int K, bool lp, int var, bool uphi, unsigned grid, cudaStream_t st,
                 int* occ) {
  switch (K) {
    case 1: return go<T, 1, REACT, MODE>(a, lp, var, uphi, grid, st, occ);
    case 2: return go<T, 2, REACT, MODE>(a, lp, var, uphi, grid, st, occ);
    case 3: return go<T, 3, REACT, MODE>(a, lp, var, uphi, grid, st, occ);
    case 4: return go<T, 4, REACT, MODE>(a, lp, var, uphi, grid, st, occ);
    case 5: return go<T, 5, REACT, MODE>(a, lp, var, uphi, grid, st, occ);
    case 6: return go<T, 6, REACT, MODE>(a, lp, var, uphi, grid, st, occ);
    case 7: return go<T, 7, REACT, MODE>(a, lp, var, uphi, grid, st, occ);
    case 8: return go<T, 8, REACT, MODE>(a, lp, var, uphi, grid, st, occ);
  }
  return cudaErrorInvalidValue;
}

// the (react, mode) pairs a precision supports
// var: rdk::TB_FULL / TB_LEAN / TB_CHECKED (the variants exist for the
// default fast mode only; any other combination runs TB_FULL)
template <typename T>
cudaError_t dispatch(const rdk::TBArgs<T>& a, int K, int mode, bool react, bool lp, int var, bool uphi,
                     unsigned grid, cudaStream_t st, int* occ) {
  if (!react) return by_k<T, false, rdk::MODE_PRECISE>(a, K, lp, var, uphi, grid, st, occ);
  switch (mode) {
    case rdk::MODE_PRECISE: return by_k<T, true, rdk::MODE_PRECISE>(a, K, lp, var, uphi, grid, st, occ);
    case rdk::MODE_FOLD: return by_k<T, true, rdk::MODE_FOLD>(a, K, lp, var, uphi, grid, st, occ);
  }
  if constexpr (sizeof(T) == 4) {
    switch (mode) {
      case rdk::MODE_FOLD_DIV4: return by_k<T, true, rdk::MODE_FOLD_DIV4>(a, K, lp, var, uphi, grid, st, occ);
      case rdk::MODE_FOLD_DIV4_NG: return by_k<T, true, rdk::MODE_FOLD_DIV4_NG>(a, K, lp, var, uphi, grid, st, occ);
    }
  }
  return cudaErrorInvalidValue;
}

template <typename T>
int occupancy(int K, int mode, bool react, bool lp, int var, bool uphi) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, bool, bool, int, bool>, int> cache;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_tuple(K, mode, react, lp, var, uphi);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int occ = 0;
  rdk::TBArgs<T> dummy;
  if (dispatch<T>(dummy, K, mode, react, lp, var, uphi, 0, nullptr, &occ) != cudaSuccess || occ < 1) occ = 1;
  cache[key] = occ;
  return occ;
}

}  // namespace detail
}  // namespace rdl
