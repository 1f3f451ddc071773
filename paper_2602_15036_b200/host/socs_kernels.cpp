// Host-side SOCS kernel generation (not on the timed path: kernels are
// inputs to the imaging kernels, as in the reference where build_tcc /
// decompose_tcc run before image_socs).
//
// Same semantics as the reference build_tcc + decompose_tcc
// (proj/src/core/imaging.cpp:113-216): TCC(f1,f2;F) = sum_s w_s P(f1+s fc;F)
// P*(f2+s fc;F) on the DFT support |f| <= (1+sigma_max) NA/lambda (same
// support order, :115-129), eigenpairs sorted descending, clamped at zero,
// truncated at k_fixed or at the energy floor, and the largest-magnitude
// component of each eigenvector made real positive (:183-196).
//
// Route ("Abbe-SVD"): TCC = Q Q^H with Q[i][s] = sqrt(w_s) P(f_i + s fc; F), so
// its nonzero eigenpairs follow from the small Ns x Ns Gram matrix
// G = Q^H Q = V L V^H:  TCC (Q v) = Q G v = l (Q v),  u = Q v / sqrt(l).
// Cost O(S Ns^2) instead of the dense O(S^3) eigensolve, which is what makes
// the BASELINE tile sizes (S up to 1e5, above the reference's 6000 budget,
// imaging.cpp:130-134) feasible.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lithogpu.h"
#include "hermitian_eig.hpp"

namespace {

using cplx = std::complex<double>;
thread_local std::string g_err;

// pupil (imaging.cpp:72-84)
cplx pupil(double lambda, double na, bool high_na, double fx, double fy, double focus) {
  const double f2 = fx * fx + fy * fy;
  const double fc = na / lambda;
  if (f2 > fc * fc) return {0.0, 0.0};
  double phase;
  if (high_na) {
    const double s = 1.0 - lambda * lambda * f2;
    phase = (2.0 * M_PI * focus / lambda) * (std::sqrt(std::max(s, 0.0)) - 1.0);
  } else {
    phase = -M_PI * lambda * focus * f2;
  }
  return std::polar(1.0, phase);
}

}  // namespace

extern "C" {

const char* lithogpu_host_last_error(void) { return g_err.c_str(); }

// Annular source (imaging.cpp:50-64); sigma_out <= 0 -> point source.
// out_xyw may be NULL to query the count.
lithogpu_status lithogpu_source_annular(double sigma_in, double sigma_out, int grid_n,
                                        int* count, double* out_xyw) {
  if (!count) return LITHOGPU_ERR_USAGE;
  std::vector<double> pts;
  if (sigma_out <= 0) {
    pts = {0.0, 0.0, 1.0};
  } else {
    if (sigma_out <= sigma_in || grid_n <= 0) {
      g_err = "annular source: need 0 <= sigma_in < sigma_out";
      return LITHOGPU_ERR_DOMAIN;
    }
    for (int iy = 0; iy < grid_n; ++iy)
      for (int ix = 0; ix < grid_n; ++ix) {
        const double sx = -1.0 + (ix + 0.5) * 2.0 / grid_n;
        const double sy = -1.0 + (iy + 0.5) * 2.0 / grid_n;
        const double r = std::hypot(sx, sy);
        if (r >= sigma_in && r <= sigma_out) {
          pts.push_back(sx);
          pts.push_back(sy);
          pts.push_back(1.0);
        }
      }
    double tot = 0;
    for (size_t i = 2; i < pts.size(); i += 3) tot += pts[i];
    for (size_t i = 2; i < pts.size(); i += 3) pts[i] /= tot;
  }
  *count = int(pts.size() / 3);
  if (out_xyw) std::memcpy(out_xyw, pts.data(), sizeof(double) * pts.size());
  return LITHOGPU_OK;
}

// Support of the band-limited TCC (imaging.cpp:115-129), in reference order.
lithogpu_status lithogpu_tcc_support(int nx, int ny, double pitch, double lambda, double na,
                                     double max_source_radius, int* count, int32_t* out_kxky) {
  if (!count || nx <= 0 || ny <= 0 || !(pitch > 0)) return LITHOGPU_ERR_USAGE;
  const double fc = na / lambda;
  const double fmax = (1.0 + max_source_radius) * fc;
  int c = 0;
  for (int ky = 0; ky < ny; ++ky)
    for (int kx = 0; kx < nx; ++kx) {
      const int skx = kx <= nx / 2 ? kx : kx - nx;
      const int sky = ky <= ny / 2 ? ky : ky - ny;
      const double fx = double(skx) / (double(nx) * pitch);
      const double fy = double(sky) / (double(ny) * pitch);
      if (fx * fx + fy * fy <= fmax * fmax * (1.0 + 1e-12)) {
        if (out_kxky) {
          out_kxky[2 * c] = skx;
          out_kxky[2 * c + 1] = sky;
        }
        ++c;
      }
    }
  *count = c;
  return LITHOGPU_OK;
}

// SOCS kernels for one focus plane.  source_xyw: n_source (sx, sy, w) rows,
// pupil-normalized, weights summing to 1.  k_fixed > 0 -> exactly that many
// (fewer if the TCC rank is lower); else truncate at energy_floor.
// support: n_support signed (kx, ky) (from lithogpu_tcc_support).
// out_weights[K], out_values[K][n_support] (re, im); *out_order = K.
// Capacity: max_order kernels.
lithogpu_status lithogpu_socs_kernels(int nx, int ny, double pitch, double lambda, double na,
                                      int high_na, const double* source_xyw, int n_source,
                                      double focus_nm, int n_support, const int32_t* support,
                                      int k_fixed, double energy_floor, int max_order,
                                      int* out_order, double* out_captured, double* out_weights,
                                      double* out_values) {
  if (!source_xyw || !support || !out_order || !out_weights || !out_values || n_source <= 0 ||
      n_support <= 0 || max_order <= 0)
    return LITHOGPU_ERR_USAGE;
  try {
    const int S = n_support, Ns = n_source;
    const double fc = na / lambda;
    // Q[i][s] = sqrt(w_s) P(f_i + s fc)
    std::vector<cplx> Q(size_t(S) * Ns);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < S; ++i) {
      const double fx = double(support[2 * i]) / (double(nx) * pitch);
      const double fy = double(support[2 * i + 1]) / (double(ny) * pitch);
      for (int s = 0; s < Ns; ++s) {
        const double* sp = source_xyw + 3 * s;
        Q[size_t(i) * Ns + s] =
            std::sqrt(sp[2]) * pupil(lambda, na, high_na != 0, fx + sp[0] * fc, fy + sp[1] * fc, focus_nm);
      }
    }
    // G = Q^H Q
    std::vector<cplx> G(size_t(Ns) * Ns, cplx{0, 0});
#pragma omp parallel for schedule(dynamic)
    for (int a = 0; a < Ns; ++a)
      for (int b = a; b < Ns; ++b) {
        cplx acc{0, 0};
        for (int i = 0; i < S; ++i)
          acc += std::conj(Q[size_t(i) * Ns + a]) * Q[size_t(i) * Ns + b];
        G[size_t(a) * Ns + b] = acc;
        G[size_t(b) * Ns + a] = std::conj(acc);
      }
    for (int a = 0; a < Ns; ++a) G[size_t(a) * Ns + a] = G[size_t(a) * Ns + a].real();
    std::vector<cplx> V;
    lg_host::hermitian_jacobi(Ns, G, V);
    std::vector<int> order(Ns);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
      return G[size_t(x) * Ns + x].real() > G[size_t(y) * Ns + y].real();
    });
    double total = 0;
    for (int i = 0; i < Ns; ++i) total += std::max(G[size_t(i) * Ns + i].real(), 0.0);
    double captured = 0;
    int K = 0;
    const double lam_max = std::max(G[size_t(order[0]) * Ns + order[0]].real(), 0.0);
    std::vector<cplx> u(S);
    for (int rank = 0; rank < Ns && K < max_order; ++rank) {
      const double lam = std::max(G[size_t(order[rank]) * Ns + order[rank]].real(), 0.0);
      if (k_fixed > 0) {
        if (rank >= k_fixed) break;
      } else if (total > 0 && captured >= energy_floor * total && rank > 0) {
        break;
      }
      if (lam <= 0 && rank > 0) break;
      // TCC rank <= min(S, Ns): eigenvalues at the fp64 noise floor are not kernels
      if (rank > 0 && (rank >= S || lam <= 1e-13 * lam_max)) break;
      const int col = order[rank];
      const double inv = lam > 0 ? 1.0 / std::sqrt(lam) : 0.0;
      for (int i = 0; i < S; ++i) {
        cplx acc{0, 0};
        for (int s = 0; s < Ns; ++s) acc += Q[size_t(i) * Ns + s] * V[size_t(s) * Ns + col];
        u[i] = acc * inv;
      }
      // deterministic phase: largest-magnitude component real positive (imaging.cpp:192-196)
      int imax = 0;
      for (int i = 1; i < S; ++i)
        if (std::abs(u[i]) > std::abs(u[imax])) imax = i;
      if (std::abs(u[imax]) > 0) {
        const cplx ph = std::conj(u[imax]) / std::abs(u[imax]);
        for (auto& x : u) x *= ph;
      }
      out_weights[K] = lam;
      for (int i = 0; i < S; ++i) {
        out_values[2 * (size_t(K) * S + i)] = u[i].real();
        out_values[2 * (size_t(K) * S + i) + 1] = u[i].imag();
      }
      captured += lam;
      ++K;
    }
    *out_order = K;
    if (out_captured) *out_captured = total > 0 ? captured / total : 1.0;
    return LITHOGPU_OK;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LITHOGPU_ERR_DOMAIN;
  }
}

}  // extern "C"
