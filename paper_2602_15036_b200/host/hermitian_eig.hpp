// Cyclic Jacobi eigensolver for small dense Hermitian matrices (host).
// Shared by the Abbe-SVD kernel generator (socs_kernels.cpp) and the C++
// drop-in's decompose_tcc for small supports.
#pragma once

#include <cmath>
#include <complex>
#include <vector>

namespace lg_host {

using cplx = std::complex<double>;

// Cyclic Jacobi eigensolver for a Hermitian matrix (row-major n x n, in place);
// eigenvalues on the diagonal on exit, eigenvectors in columns of V.
inline void hermitian_jacobi(int n, std::vector<cplx>& A, std::vector<cplx>& V) {
  V.assign(size_t(n) * n, cplx{0, 0});
  for (int i = 0; i < n; ++i) V[size_t(i) * n + i] = 1.0;
  auto a = [&](int i, int j) -> cplx& { return A[size_t(i) * n + j]; };
  auto v = [&](int i, int j) -> cplx& { return V[size_t(i) * n + j]; };
  double fro = 0;
  for (const auto& x : A) fro += std::norm(x);
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += std::norm(a(p, q));
    if (off <= 1e-32 * fro || off == 0.0) return;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const cplx apq = a(p, q);
        const double r = std::abs(apq);
        if (r == 0.0 || r * r < 1e-40 * fro) continue;
        const cplx e = apq / r;
        const double th = (a(q, q).real() - a(p, p).real()) / (2.0 * r);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::abs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const cplx up = a(k, p), uq = a(k, q) * std::conj(e);
          a(k, p) = c * up - s * uq;
          a(k, q) = s * up + c * uq;
        }
        for (int k = 0; k < n; ++k) {
          const cplx wp = a(p, k), wq = a(q, k) * e;
          a(p, k) = c * wp - s * wq;
          a(q, k) = s * wp + c * wq;
        }
        a(p, q) = a(q, p) = 0.0;
        a(p, p) = a(p, p).real();
        a(q, q) = a(q, q).real();
        for (int k = 0; k < n; ++k) {
          const cplx up = v(k, p), uq = v(k, q) * std::conj(e);
          v(k, p) = c * up - s * uq;
          v(k, q) = s * up + c * uq;
        }
      }
  }
}


}  // namespace lg_host
