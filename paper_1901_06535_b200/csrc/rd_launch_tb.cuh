// rd_launch_tb.cuh — tb_kernel / lp_kernel launch dispatch for one precision
// (included by rd_launch_tb_f32.cu and rd_launch_tb_f64.cu).
#pragma once
#include <map>
#include <mutex>
#include <tuple>

#include "rd_launch.h"

namespace rdl {
namespace detail {

template <typename T, int K, bool REACT, int MODE>
cudaError_t go(const rdk::TBArgs<T>& a, bool lp, unsigned grid, cudaStream_t st, int* occ) {
  constexpr int V = 16 / (int)sizeof(T);
  if (lp) {
    if constexpr (K <= 4) {
      if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, rdk::lp_kernel<T, K, V, REACT, MODE>, 32 * K, 0);
      rdk::lp_kernel<T, K, V, REACT, MODE><<<grid, 32 * K, 0, st>>>(a);
      return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
  }
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, rdk::tb_kernel<T, K, V, REACT, MODE>, 32, 0);
  rdk::tb_kernel<T, K, V, REACT, MODE><<<grid, 32, 0, st>>>(a);
  return cudaGetLastError();
}

template <typename T, bool REACT, int MODE>
cudaError_t by_k(const rdk::TBArgs<T>& a, int K, bool lp, unsigned grid, cudaStream_t st, int* occ) {
  switch (K) {
    case 1: return go<T, 1, REACT, MODE>(a, lp, grid, st, occ);
    case 2: return go<T, 2, REACT, MODE>(a, lp, grid, st, occ);
    case 3: return go<T, 3, REACT, MODE>(a, lp, grid, st, occ);
    case 4: return go<T, 4, REACT, MODE>(a, lp, grid, st, occ);
    case 5: return go<T, 5, REACT, MODE>(a, lp, grid, st, occ);
    case 6: return go<T, 6, REACT, MODE>(a, lp, grid, st, occ);
    case 7: return go<T, 7, REACT, MODE>(a, lp, grid, st, occ);
    case 8: return go<T, 8, REACT, MODE>(a, lp, grid, st, occ);
  }
  return cudaErrorInvalidValue;
}

// the (react, mode) pairs a precision supports
template <typename T>
cudaError_t dispatch(const rdk::TBArgs<T>& a, int K, int mode, bool react, bool lp, unsigned grid, cudaStream_t st,
                     int* occ) {
  if (!react) return by_k<T, false, rdk::MODE_PRECISE>(a, K, lp, grid, st, occ);
  switch (mode) {
    case rdk::MODE_PRECISE: return by_k<T, true, rdk::MODE_PRECISE>(a, K, lp, grid, st, occ);
    case rdk::MODE_FOLD: return by_k<T, true, rdk::MODE_FOLD>(a, K, lp, grid, st, occ);
  }
  if constexpr (sizeof(T) == 4) {
    switch (mode) {
      case rdk::MODE_FOLD_DIV4: return by_k<T, true, rdk::MODE_FOLD_DIV4>(a, K, lp, grid, st, occ);
      case rdk::MODE_FOLD_DIV4_NG: return by_k<T, true, rdk::MODE_FOLD_DIV4_NG>(a, K, lp, grid, st, occ);
    }
  }
  return cudaErrorInvalidValue;
}

template <typename T>
int occupancy(int K, int mode, bool react, bool lp) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, bool, bool>, int> cache;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_tuple(K, mode, react, lp);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int occ = 0;
  rdk::TBArgs<T> dummy;
  if (dispatch<T>(dummy, K, mode, react, lp, 0, nullptr, &occ) != cudaSuccess || occ < 1) occ = 1;
  cache[key] = occ;
  return occ;
}

}  // namespace detail
}  // namespace rdl
