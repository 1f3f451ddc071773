// Launch plumbing shared by fast_rows.cu / fast_cols.cu.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <type_traits>

#include "socs_fast.cuh"

namespace lg {

template <typename F>
inline void with_lg(int lg, F&& f) {
  switch (lg) {
    case 5: f(std::integral_constant<int, 5>()); break;
    case 6: f(std::integral_constant<int, 6>()); break;
    case 7: f(std::integral_constant<int, 7>()); break;
    case 8: f(std::integral_constant<int, 8>()); break;
    case 9: f(std::integral_constant<int, 9>()); break;
    case 10: f(std::integral_constant<int, 10>()); break;
    case 11: f(std::integral_constant<int, 11>()); break;
    case 12: f(std::integral_constant<int, 12>()); break;
    case 13: f(std::integral_constant<int, 13>()); break;
    default: throw std::runtime_error("fast path: unsupported transform length 2^" + std::to_string(lg));
  }
}

// groups of TPR threads per CTA: ~target threads, capped so named barriers fit
template <int LG>
inline int fgroups(int target, int cap = 1 << 30) {
  constexpr int TPR = RPlan<LG>::TPR;
  int gr = target / TPR;
  if (gr < 1) gr = 1;
  if (gr > cap) gr = cap;
  if (TPR > 32 && gr > 15) gr = 15;
  return gr;
}

template <int LG, typename K, typename... A>
inline void flaunch(K kern, dim3 grid, int groups, cudaStream_t s, A... args) {
  const size_t smem = size_t(groups) * rsm_len<LG>() * sizeof(C32);
  static size_t set_bytes = 0;  // per instantiation
  if (smem > 48 * 1024 && smem > set_bytes) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    set_bytes = smem;
  }
  kern<<<grid, groups * RPlan<LG>::TPR, smem, s>>>(args...);
}

inline int cdivi(long long a, long long b) { return int((a + b - 1) / b); }

}  // namespace lg
