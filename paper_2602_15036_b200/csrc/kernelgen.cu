// SOCS kernel generation on the GPU: the same
// semantics as the host generator lithogpu_socs_kernels (host/socs_kernels.cpp)
// and the reference build_tcc + decompose_tcc (imaging.cpp:113-216), for every
// focus plane of a run in one call.
//
// Abbe-SVD route: TCC = Q Q^H, Q[i][s] = sqrt(w_s) P(f_i + s fc).
//   A = Q^T (Ns x S, column-major)  -- built by k_build_q (fp64 pupil)
//   Gbar = A A^H = conj(Q^H Q)       -- cublasZherk (Ns x Ns)
//   Gbar vbar = l vbar               -- cusolverDnZheevd (ascending)
//   u_k = Q conj(vbar_k) / sqrt(l_k) -- cublasZgemm (S x K), then the
//   reference phase rule: the first largest-|.| component made real positive.
// Eigenvalue ordering / truncation (k_fixed, energy floor, fp64 noise floor)
// is decided on the host from the Ns eigenvalues, exactly as the host path.
#include <cublas_v2.h>
#include <cuComplex.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lithogpu.h"

namespace lg_internal {
cudaStream_t ctx_stream(lithogpu_ctx* ctx);
void ctx_activate(lithogpu_ctx* ctx);
void ctx_count_launch(lithogpu_ctx* ctx);
void set_error(const char* msg);
}  // namespace lg_internal

namespace {

#define KG_CUDA(x)                                                                   \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e_)); \
  } while (0)
#define KG_BLAS(x)                                                                   \
  do {                                                                               \
    if ((x) != CUBLAS_STATUS_SUCCESS) throw std::runtime_error("cuBLAS failure: " #x); \
  } while (0)
#define KG_SOLV(x)                                                                   \
  do {                                                                               \
    if ((x) != CUSOLVER_STATUS_SUCCESS) throw std::runtime_error("cuSOLVER failure: " #x); \
  } while (0)

struct Buf {
  void* p = nullptr;
  ~Buf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* get(size_t n) {
    if (!p) KG_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return static_cast<T*>(p);
  }
};

// pupil (imaging.cpp:72-84), fp64
__device__ cuDoubleComplex d_pupil(double lambda, double na, int high_na, double fx, double fy, double focus) {
  const double f2 = fx * fx + fy * fy;
  const double fc = na / lambda;
  if (f2 > fc * fc) return make_cuDoubleComplex(0.0, 0.0);
  double phase;
  if (high_na) {
    const double s = 1.0 - lambda * lambda * f2;
    phase = (2.0 * M_PI * focus / lambda) * (sqrt(fmax(s, 0.0)) - 1.0);
  } else {
    phase = -M_PI * lambda * focus * f2;
  }
  double sn, cs;
  sincos(phase, &sn, &cs);
  return make_cuDoubleComplex(cs, sn);
}

// A[s + Ns*i] = sqrt(w_s) P(f_i + s fc; focus)
__global__ void k_build_q(int S, int Ns, int nx, int ny, double pitch, double lambda, double na, int high_na,
                          double focus, const int* __restrict__ sup, const double* __restrict__ src,
                          cuDoubleComplex* __restrict__ A) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)S * Ns) return;
  const int i = int(idx / Ns), s = int(idx % Ns);
  const double fc = na / lambda;
  const double fx = double(sup[2 * i]) / (double(nx) * pitch) + src[3 * s] * fc;
  const double fy = double(sup[2 * i + 1]) / (double(ny) * pitch) + src[3 * s + 1] * fc;
  const cuDoubleComplex p = d_pupil(lambda, na, high_na, fx, fy, focus);
  const double w = sqrt(src[3 * s + 2]);
  A[idx] = make_cuDoubleComplex(w * p.x, w * p.y);
}

// Bk[:, k] = conj(vbar[:, col_k]) / sqrt(lam_k)   (Ns x K, column-major)
__global__ void k_pick_vecs(int Ns, int K, const cuDoubleComplex* __restrict__ vbar, const int* __restrict__ cols,
                            const double* __restrict__ scale, cuDoubleComplex* __restrict__ B) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Ns * K) return;
  const int s = idx % Ns, k = idx / Ns;
  const cuDoubleComplex v = vbar[size_t(cols[k]) * Ns + s];
  B[idx] = make_cuDoubleComplex(v.x * scale[k], -v.y * scale[k]);
}

// per kernel: first index of the largest |u| (strict >, as the reference), then
// u *= conj(u_max) / |u_max|; one block per kernel
__global__ void k_phase_fix(int S, cuDoubleComplex* __restrict__ U) {
  cuDoubleComplex* u = U + size_t(blockIdx.x) * S;
  __shared__ double bm[256];
  __shared__ int bi[256];
  double m = -1.0;
  int mi = 0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) {
    const double a = hypot(u[i].x, u[i].y);
    if (a > m) {
      m = a;
      mi = i;
    }
  }
  bm[threadIdx.x] = m;
  bi[threadIdx.x] = mi;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (int(threadIdx.x) < h) {
      const double om = bm[threadIdx.x + h];
      const int oi = bi[threadIdx.x + h];
      if (om > bm[threadIdx.x] || (om == bm[threadIdx.x] && oi < bi[threadIdx.x])) {
        bm[threadIdx.x] = om;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  const cuDoubleComplex um = u[bi[0]];
  const double am = bm[0];
  if (!(am > 0)) return;
  const double pr = um.x / am, pi = -um.y / am;  // conj(u_max) / |u_max|
  for (int i = threadIdx.x; i < S; i += blockDim.x) {
    const cuDoubleComplex x = u[i];
    u[i] = make_cuDoubleComplex(x.x * pr - x.y * pi, x.x * pi + x.y * pr);
  }
}

}  // namespace

extern "C" lithogpu_status lithogpu_socs_kernels_gpu(lithogpu_ctx* ctx, int nx, int ny, double pitch, double lambda,
                                                     double na, int high_na, const double* source_xyw, int n_source,
                                                     int n_focus, const double* focus_nm, int n_support,
                                                     const int32_t* support, int k_fixed, double energy_floor,
                                                     int max_order, int* out_order, double* out_captured,
                                                     double* out_weights, double* out_values) {
  if (!ctx || !source_xyw || !focus_nm || !support || !out_order || !out_weights || !out_values || n_source <= 0 ||
      n_support <= 0 || max_order <= 0 || n_focus <= 0) {
    lg_internal::set_error("lithogpu_socs_kernels_gpu: bad argument");
    return LITHOGPU_ERR_USAGE;
  }
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solv = nullptr;
  try {
    lg_internal::ctx_activate(ctx);
    cudaStream_t st = lg_internal::ctx_stream(ctx);
    const int S = n_support, Ns = n_source;
    KG_BLAS(cublasCreate(&blas));
    KG_BLAS(cublasSetStream(blas, st));
    KG_SOLV(cusolverDnCreate(&solv));
    KG_SOLV(cusolverDnSetStream(solv, st));
    Buf dsup, dsrc, dA, dG, dW, dwork, dinfo, dB, dU, dcols, dscale;
    int* sup = dsup.get<int>(size_t(2) * S);
    double* src = dsrc.get<double>(size_t(3) * Ns);
    cuDoubleComplex* A = dA.get<cuDoubleComplex>(size_t(S) * Ns);
    cuDoubleComplex* G = dG.get<cuDoubleComplex>(size_t(Ns) * Ns);
    double* W = dW.get<double>(Ns);
    int* info = dinfo.get<int>(1);
    cuDoubleComplex* B = dB.get<cuDoubleComplex>(size_t(Ns) * max_order);
    cuDoubleComplex* U = dU.get<cuDoubleComplex>(size_t(S) * max_order);
    int* cols = dcols.get<int>(max_order);
    double* scale = dscale.get<double>(max_order);
    KG_CUDA(cudaMemcpyAsync(sup, support, sizeof(int) * 2 * S, cudaMemcpyHostToDevice, st));
    KG_CUDA(cudaMemcpyAsync(src, source_xyw, sizeof(double) * 3 * Ns, cudaMemcpyHostToDevice, st));
    int lwork = 0;
    KG_SOLV(cusolverDnZheevd_bufferSize(solv, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, Ns, G, Ns, W,
                                        &lwork));
    cuDoubleComplex* work = dwork.get<cuDoubleComplex>(size_t(lwork));
    std::vector<double> lam(Ns);
    for (int f = 0; f < n_focus; ++f) {
      const long long nq = (long long)S * Ns;
      k_build_q<<<int((nq + 255) / 256), 256, 0, st>>>(S, Ns, nx, ny, pitch, lambda, na, high_na, focus_nm[f], sup,
                                                       src, A);
      KG_CUDA(cudaGetLastError());
      lg_internal::ctx_count_launch(ctx);
      const double one = 1.0, zero = 0.0;
      KG_BLAS(cublasZherk(blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, Ns, S, &one, A, Ns, &zero, G, Ns));
      KG_SOLV(cusolverDnZheevd(solv, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, Ns, G, Ns, W, work, lwork,
                               info));
      int hinfo = 0;
      KG_CUDA(cudaMemcpyAsync(lam.data(), W, sizeof(double) * Ns, cudaMemcpyDeviceToHost, st));
      KG_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, st));
      KG_CUDA(cudaStreamSynchronize(st));
      if (hinfo != 0) throw std::runtime_error("decompose_tcc: eigensolver failed");
      // descending order (zheevd is ascending); same truncation rules as the host path
      std::vector<int> order(Ns);
      std::iota(order.begin(), order.end(), 0);
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return lam[x] > lam[y]; });
      double total = 0;
      for (int i = 0; i < Ns; ++i) total += std::max(lam[i], 0.0);
      const double lam_max = std::max(lam[order[0]], 0.0);
      double captured = 0;
      int K = 0;
      std::vector<int> hcols;
      std::vector<double> hscale, hw;
      for (int rank = 0; rank < Ns && K < max_order; ++rank) {
        const double l = std::max(lam[order[rank]], 0.0);
        if (k_fixed > 0) {
          if (rank >= k_fixed) break;
        } else if (total > 0 && captured >= energy_floor * total && rank > 0) {
          break;
        }
        if (l <= 0 && rank > 0) break;
        if (rank > 0 && (rank >= S || l <= 1e-13 * lam_max)) break;
        hcols.push_back(order[rank]);
        hscale.push_back(l > 0 ? 1.0 / std::sqrt(l) : 0.0);
        hw.push_back(l);
        captured += l;
        ++K;
      }
      out_order[f] = K;
      if (out_captured) out_captured[f] = total > 0 ? captured / total : 1.0;
      for (int k = 0; k < K; ++k) out_weights[size_t(f) * max_order + k] = hw[k];
      if (K == 0) continue;
      KG_CUDA(cudaMemcpyAsync(cols, hcols.data(), sizeof(int) * K, cudaMemcpyHostToDevice, st));
      KG_CUDA(cudaMemcpyAsync(scale, hscale.data(), sizeof(double) * K, cudaMemcpyHostToDevice, st));
      k_pick_vecs<<<(Ns * K + 255) / 256, 256, 0, st>>>(Ns, K, G, cols, scale, B);
      KG_CUDA(cudaGetLastError());
      lg_internal::ctx_count_launch(ctx);
      // U (S x K) = A^T (S x Ns) * B (Ns x K)
      const cuDoubleComplex c1 = make_cuDoubleComplex(1.0, 0.0), c0 = make_cuDoubleComplex(0.0, 0.0);
      KG_BLAS(cublasZgemm(blas, CUBLAS_OP_T, CUBLAS_OP_N, S, K, Ns, &c1, A, Ns, B, Ns, &c0, U, S));
      k_phase_fix<<<K, 256, 0, st>>>(S, U);
      KG_CUDA(cudaGetLastError());
      lg_internal::ctx_count_launch(ctx);
      KG_CUDA(cudaMemcpyAsync(out_values + size_t(f) * max_order * S * 2, U, sizeof(cuDoubleComplex) * S * K,
                              cudaMemcpyDeviceToHost, st));
      KG_CUDA(cudaStreamSynchronize(st));
    }
    cublasDestroy(blas);
    cusolverDnDestroy(solv);
    lg_internal::set_error("");
    return LITHOGPU_OK;
  } catch (const std::exception& e) {
    if (blas) cublasDestroy(blas);
    if (solv) cusolverDnDestroy(solv);
    lg_internal::set_error(e.what());
    return LITHOGPU_ERR_DOMAIN;
  }
}
