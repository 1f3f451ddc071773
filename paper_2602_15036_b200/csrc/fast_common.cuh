// Launch plumbing shared by fast_rows.cu / fast_cols.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <unordered_set>

#ifndef LG_DEFAULT_CARVEOUT
#define LG_DEFAULT_CARVEOUT -1
#endif

#include "socs_fast.cuh"

namespace lg {

template <typename F>
inline void with_len(int len, F&& f) {
  switch (len) {
#define LG_CASE(X) \
  case X:          \
    f(std::integral_constant<int, X>()); \
    break;
    LG_CASE(32) LG_CASE(64) LG_CASE(128) LG_CASE(192) LG_CASE(256) LG_CASE(384) LG_CASE(512)
    LG_CASE(768) LG_CASE(1024) LG_CASE(1536) LG_CASE(2048) LG_CASE(3072) LG_CASE(4096) LG_CASE(8192)
#undef LG_CASE
    default: throw std::runtime_error("fast path: unsupported transform length " + std::to_string(len));
  }
}

// groups of TPR threads per CTA: ~target threads, capped so named barriers fit
template <int L>
inline int fgroups(int target, int cap = 1 << 30) {
  constexpr int TPR = RPlan<L>::TPR;
  int gr = target / TPR;
  if (gr < 1) gr = 1;
  if (gr > cap) gr = cap;
  if (TPR > 32 && gr > 15) gr = 15;
  return gr;
}

// kernel groups per CTA for the (row|column) x kernel-group kernels: the
// largest power of two <= 256/TPR that divides K
template <int L>
inline int kgroups(int K) {
  int kg = 256 / RPlan<L>::TPR;
  if (kg < 1) kg = 1;
  if (RPlan<L>::TPR > 32 && kg > 15) kg = 8;
  while (kg > 1 && K % kg) kg >>= 1;
  return kg;
}

// groups per CTA for low-parallelism transforms: spread `units` row groups
// over the SMs first (>= ~2 CTAs per SM before packing groups together)
template <int L>
inline int spread_groups(long long units, int cap = 8) {
  constexpr int TPR = RPlan<L>::TPR;
  long long gr = units / (2 * 148);
  int g = 1;
  while (g * 2 <= gr && g * 2 <= cap && g * 2 * TPR <= 256) g *= 2;
  return g;
}

// dynamic shared memory above 48 KB, raised once per kernel (keyed on the
// kernel itself: kernels of one signature share a launcher instantiation)
template <typename K>
inline void set_max_smem(K kern, size_t smem) {
  thread_local std::unordered_map<const void*, size_t> set;
  size_t& cur = set[reinterpret_cast<const void*>(kern)];
  if (smem > cur) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cur = smem;
  }
}

// launch with `extra` bytes of shared memory after the row-group buffers
template <int L, typename K, typename... A>
inline void flaunch_x(K kern, dim3 grid, int groups, size_t extra, cudaStream_t s, A... args) {
  const size_t smem = size_t(groups) * rsm_len<L>() * sizeof(C32) + extra;
  if (smem > 32 * 1024) set_max_smem(kern, smem);  // static shared memory counts toward the 48 KB default too
  pdl_launch(kern, grid, dim3(groups * RPlan<L>::TPR), smem, s, args...);
}

template <int L, typename K, typename... A>
inline void flaunch(K kern, dim3 grid, int groups, cudaStream_t s, A... args) {
  flaunch_x<L>(kern, grid, groups, 0, s, args...);
}

// PDL measured: +15% on the forward imaging chain, -8% on the graph-replayed
// ILT loop, so callers switch it per path.
inline bool& pdl_enabled() {
  thread_local bool on = true;
  return on;
}

// Shared-memory carveout applied once per kernel (LITHOGPU_CARVEOUT=percent;
// -1 = driver default).  Kernels of one ILT iteration that ask for different
// L1/shared splits force the SMs to drain and reconfigure between launches.
inline int carveout_pct() {
  static const int pct = [] {
    const char* e = std::getenv("LITHOGPU_CARVEOUT");
    return e ? std::atoi(e) : LG_DEFAULT_CARVEOUT;
  }();
  return pct;
}
template <typename K>
inline void apply_carveout(K kern) {
  const int pct = carveout_pct();
  if (pct < 0) return;
  thread_local std::unordered_set<const void*> done;
  if (done.insert(reinterpret_cast<const void*>(kern)).second)
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

// launch with programmatic stream serialization (PDL; LITHOGPU_NO_PDL=1 disables)
template <typename K, typename... A>
inline void pdl_launch(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, A... args) {
  apply_carveout(kern);
  static const bool env_off = std::getenv("LITHOGPU_NO_PDL") != nullptr;
  const bool on = pdl_enabled() && !env_off;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = on ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

// LITHOGPU_NO_SPARSE=1: dense first / last FFT stages everywhere (A/B)
inline bool sparse_off() {
  static const bool off = std::getenv("LITHOGPU_NO_SPARSE") != nullptr;
  return off;
}

inline int cdivi(long long a, long long b) { return int((a + b - 1) / b); }

}  // namespace lg
