// TEST INFRASTRUCTURE ONLY (oracle/_ref). Thin extern "C" veneer over the
// UNMODIFIED reference sources (compiled from /root/reference/proj/src by
// oracle/build_ref.sh) so pytest / bench.py can call the reference itself:
// rasterize_layer (raster.cpp:53-95, heal included), heal (boolean.hpp:40-42),
// build_tcc/decompose_tcc (imaging.cpp:113-216), image_socs (:218-241),
// image_hopkins_direct (:243-285), gaussian_blur (:287-314), pupil (:72-84),
// intensity_gradient (ai.cpp:11-42), z_print/z_round (ai.cpp:76-94),
// marching_squares / measure_epe (contour.cpp:58-201).
//
// The ILT pieces the reference lacks (weighted adjoint, sigmoid resist,
// process-window cost, theta update) are composed
// here from reference calls only (image_socs, gaussian_blur, fft2), following
// intensity_gradient's own structure (ai.cpp:19-41) with W(r) inserted before
// the forward FFT. W == 1 reproduces intensity_gradient exactly.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "core/ai.hpp"
#include "core/boolean.hpp"
#include "core/contour.hpp"
#include "core/io.hpp"
#include "core/imaging.hpp"
#include "core/raster.hpp"

extern "C" {
void oracle_fft_set_threads(int n);
}

using litho::cplx;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_err.clear();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown error";
    return 1;
  }
}

litho::Grid make_grid(int nx, int ny, double pitch, double ox, double oy) {
  return litho::Grid{nx, ny, pitch, ox, oy};
}

litho::Layer make_layer(const int64_t* xy, const int64_t* starts, int npoly) {
  litho::Layer layer;
  for (int p = 0; p < npoly; ++p) {
    litho::Polygon poly;
    for (int64_t v = starts[p]; v < starts[p + 1]; ++v)
      poly.vertices.push_back({litho::coord_t(xy[2 * v]), litho::coord_t(xy[2 * v + 1])});
    layer.polygons.push_back(std::move(poly));
  }
  return layer;
}

litho::OpticalModel make_model(double lambda, double na, double sigma_in, double sigma_out,
                               int grid_n, int high_na) {
  litho::OpticalModel m;
  m.wavelength_nm = lambda;
  m.na = na;
  if (sigma_out <= 0)
    m.source = litho::make_point_source();
  else
    m.source = litho::make_annular_source(sigma_in, sigma_out, grid_n);
  m.high_na_defocus = high_na != 0;
  return m;
}

// band-sparse kernel stack (support S of signed (kx,ky); values K*S complex)
litho::SocsKernelSet expand_kernels(const litho::Grid& g, int K, const double* weights, int S,
                                    const int32_t* support, const double* values) {
  litho::SocsKernelSet set;
  set.grid = g;
  for (int k = 0; k < K; ++k) {
    std::vector<cplx> freq(g.size(), cplx{0, 0});
    for (int s = 0; s < S; ++s) {
      const int kx = (support[2 * s] % g.nx + g.nx) % g.nx;
      const int ky = (support[2 * s + 1] % g.ny + g.ny) % g.ny;
      const double* v = values + 2 * (std::size_t(k) * S + s);
      freq[g.index(kx, ky)] = cplx{v[0], v[1]};
    }
    set.weights.push_back(weights[k]);
    set.kernels_freq.push_back(std::move(freq));
  }
  return set;
}

// restatement of intensity_gradient (ai.cpp:11-42) with a per-pixel weight W
std::vector<double> weighted_gradient(const litho::MaskField& mask,
                                      const litho::SocsKernelSet& kernels, double dose,
                                      const double* W) {
  const litho::Grid& g = mask.grid;
  const std::size_t sz = g.size();
  std::vector<cplx> spectrum = mask.values;
  litho::fft2(spectrum, g.nx, g.ny, false);
  const double inv_n = 1.0 / double(sz);
  for (auto& s : spectrum) s *= inv_n;
  std::vector<double> grad(sz, 0.0);
  std::vector<cplx> field(sz), corr(sz);
  for (std::size_t k = 0; k < kernels.order(); ++k) {
    for (std::size_t i = 0; i < sz; ++i) field[i] = spectrum[i] * kernels.kernels_freq[k][i];
    litho::fft2(field, g.nx, g.ny, true);
    corr = field;
    if (W)
      for (std::size_t i = 0; i < sz; ++i) corr[i] *= W[i];
    litho::fft2(corr, g.nx, g.ny, false);
    for (std::size_t i = 0; i < sz; ++i) corr[i] *= std::conj(kernels.kernels_freq[k][i]) * inv_n;
    litho::fft2(corr, g.nx, g.ny, true);
    const double w = 2.0 * kernels.weights[k] * dose;
    for (std::size_t i = 0; i < sz; ++i) grad[i] += w * corr[i].real();
  }
  return grad;
}

struct RefKernels {
  litho::TccMatrix tcc;
  litho::SocsKernelSet set;
};

double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_set_threads(int n) { oracle_fft_set_threads(n); }

int ref_rasterize(const int64_t* xy, const int64_t* starts, int npoly, int nx, int ny,
                  double pitch, double ox, double oy, double dbu_per_nm, double* out) {
  return guarded([&] {
    const auto pix = litho::rasterize_layer(make_layer(xy, starts, npoly),
                                            make_grid(nx, ny, pitch, ox, oy), dbu_per_nm);
    std::memcpy(out, pix.data(), pix.size() * sizeof(double));
  });
}

// heal: first call with out_xy == nullptr returns counts; second fills.
int ref_heal(const int64_t* xy, const int64_t* starts, int npoly, int64_t* out_npoly,
             int64_t* out_nvert, int64_t* out_xy, int64_t* out_starts) {
  return guarded([&] {
    const litho::Layer healed = litho::heal(make_layer(xy, starts, npoly));
    int64_t nv = 0;
    for (const auto& p : healed.polygons) nv += int64_t(p.vertices.size());
    *out_npoly = int64_t(healed.polygons.size());
    *out_nvert = nv;
    if (!out_xy) return;
    int64_t v = 0;
    for (std::size_t p = 0; p < healed.polygons.size(); ++p) {
      out_starts[p] = v;
      for (const auto& q : healed.polygons[p].vertices) {
        out_xy[2 * v] = q.x;
        out_xy[2 * v + 1] = q.y;
        ++v;
      }
    }
    out_starts[healed.polygons.size()] = v;
  });
}

int ref_pupil(double lambda, double na, int high_na, double fx, double fy, double focus,
              double* out_re_im) {
  return guarded([&] {
    litho::OpticalModel m;
    m.wavelength_nm = lambda;
    m.na = na;
    m.high_na_defocus = high_na != 0;
    const cplx p = m.pupil(fx, fy, focus);
    out_re_im[0] = p.real();
    out_re_im[1] = p.imag();
  });
}

int ref_source(double sigma_in, double sigma_out, int grid_n, int* out_n, double* out_xyw) {
  return guarded([&] {
    const litho::SourceMap s = sigma_out <= 0 ? litho::make_point_source()
                                              : litho::make_annular_source(sigma_in, sigma_out,
                                                                           grid_n);
    *out_n = int(s.points.size());
    if (!out_xyw) return;
    for (std::size_t i = 0; i < s.points.size(); ++i) {
      out_xyw[3 * i] = s.points[i].sx;
      out_xyw[3 * i + 1] = s.points[i].sy;
      out_xyw[3 * i + 2] = s.points[i].weight;
    }
  });
}

// build_tcc + decompose_tcc; handle holds both (TCC needed by Hopkins oracle)
int ref_kernels_build(int nx, int ny, double pitch, double lambda, double na, double sigma_in,
                      double sigma_out, int grid_n, int high_na, double focus,
                      double energy_floor, int k_fixed, int full_rank, void** out) {
  return guarded([&] {
    auto* h = new RefKernels;
    const litho::OpticalModel m = make_model(lambda, na, sigma_in, sigma_out, grid_n, high_na);
    h->tcc = litho::build_tcc(m, make_grid(nx, ny, pitch, 0, 0), focus);
    h->set = litho::decompose_tcc(h->tcc, energy_floor,
                                  full_rank ? int(h->tcc.dim()) : k_fixed);
    *out = h;
  });
}

void ref_kernels_info(void* hv, int* K, int* S, double* captured) {
  auto* h = static_cast<RefKernels*>(hv);
  *K = int(h->set.order());
  *S = int(h->tcc.dim());
  *captured = h->set.captured_energy;
}

// weights[K], support[S*2] (signed kx,ky), values[K*S*2], tcc[S*S*2] (optional)
void ref_kernels_get(void* hv, double* weights, int32_t* support, double* values, double* tcc) {
  auto* h = static_cast<RefKernels*>(hv);
  const litho::Grid& g = h->set.grid;
  const std::size_t S = h->tcc.dim();
  for (std::size_t s = 0; s < S; ++s) {
    support[2 * s] = h->tcc.support[s].kx;
    support[2 * s + 1] = h->tcc.support[s].ky;
  }
  for (std::size_t k = 0; k < h->set.order(); ++k) {
    weights[k] = h->set.weights[k];
    for (std::size_t s = 0; s < S; ++s) {
      const int kx = (h->tcc.support[s].kx + g.nx) % g.nx;
      const int ky = (h->tcc.support[s].ky + g.ny) % g.ny;
      const cplx v = h->set.kernels_freq[k][g.index(kx, ky)];
      values[2 * (k * S + s)] = v.real();
      values[2 * (k * S + s) + 1] = v.imag();
    }
  }
  if (tcc)
    for (std::size_t i = 0; i < S * S; ++i) {
      tcc[2 * i] = h->tcc.m[i].real();
      tcc[2 * i + 1] = h->tcc.m[i].imag();
    }
}

void ref_kernels_free(void* hv) { delete static_cast<RefKernels*>(hv); }

int ref_image_hopkins(void* hv, const double* mask, double dose, double* out) {
  return guarded([&] {
    auto* h = static_cast<RefKernels*>(hv);
    const litho::MaskField mf =
        litho::MaskField::from_real(h->tcc.grid, std::vector<double>(mask, mask + h->tcc.grid.size()));
    const auto img = litho::image_hopkins_direct(mf, h->tcc, dose, 1u << 20);
    std::memcpy(out, img.intensity.data(), img.intensity.size() * sizeof(double));
  });
}

int ref_image_socs(int nx, int ny, double pitch, const double* mask, int K,
                   const double* weights, int S, const int32_t* support, const double* values,
                   double dose, double* out) {
  return guarded([&] {
    const litho::Grid g = make_grid(nx, ny, pitch, 0, 0);
    const auto set = expand_kernels(g, K, weights, S, support, values);
    const auto mf = litho::MaskField::from_real(g, std::vector<double>(mask, mask + g.size()));
    const auto img = litho::image_socs(mf, set, dose);
    std::memcpy(out, img.intensity.data(), img.intensity.size() * sizeof(double));
  });
}

int ref_gaussian_blur(int nx, int ny, double pitch, const double* in, double sigma_nm,
                      double* out) {
  return guarded([&] {
    const litho::Grid g = make_grid(nx, ny, pitch, 0, 0);
    const auto r = litho::gaussian_blur(g, std::vector<double>(in, in + g.size()), sigma_nm);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

int ref_intensity_gradient(int nx, int ny, double pitch, const double* mask, int K,
                           const double* weights, int S, const int32_t* support,
                           const double* values, double dose, double* out) {
  return guarded([&] {
    const litho::Grid g = make_grid(nx, ny, pitch, 0, 0);
    const auto set = expand_kernels(g, K, weights, S, support, values);
    const auto mf = litho::MaskField::from_real(g, std::vector<double>(mask, mask + g.size()));
    const auto r = litho::intensity_gradient(mf, set, dose);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

int ref_weighted_gradient(int nx, int ny, double pitch, const double* mask, int K,
                          const double* weights, int S, const int32_t* support,
                          const double* values, double dose, const double* W, double* out) {
  return guarded([&] {
    const litho::Grid g = make_grid(nx, ny, pitch, 0, 0);
    const auto set = expand_kernels(g, K, weights, S, support, values);
    const auto mf = litho::MaskField::from_real(g, std::vector<double>(mask, mask + g.size()));
    const auto r = weighted_gradient(mf, set, dose, W);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

int ref_z_print(int nx, int ny, double pitch, const double* field, int K,
                const double* weights, int S, const int32_t* support, const double* values,
                double dose, double tau, double* out) {
  return guarded([&] {
    const litho::Grid g = make_grid(nx, ny, pitch, 0, 0);
    const auto set = expand_kernels(g, K, weights, S, support, values);
    const litho::ContinuousMaskField f{g, std::vector<double>(field, field + g.size())};
    const auto r = litho::z_print(f, set, dose, tau);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

int ref_z_round(int nx, int ny, double pitch, const double* raster, double sigma_nm,
                double tau, double* out) {
  return guarded([&] {
    const litho::Grid g = make_grid(nx, ny, pitch, 0, 0);
    const auto r = litho::z_round(g, std::vector<double>(raster, raster + g.size()), sigma_nm, tau);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

// One ILT iteration composed from reference calls.
// kernels: F stacks of K, shared support S; values [F][K][S] complex;
// weights [F][K]; focus_weight [F]. theta updated in place.
// params: {mask_steepness a, resist_beta, threshold, resist_sigma_nm, dose, step}
int ref_ilt_iteration(int nx, int ny, double pitch, int F, int K, const double* weights, int S,
                      const int32_t* support, const double* values, const double* focus_weight,
                      const double* params, const double* target, double* theta,
                      double* cost_out, double* grad_out) {
  return guarded([&] {
    const litho::Grid g = make_grid(nx, ny, pitch, 0, 0);
    const double a = params[0], beta = params[1], thr = params[2], sig = params[3],
                 dose = params[4], step = params[5];
    const std::size_t sz = g.size();
    std::vector<double> m(sz);
    for (std::size_t i = 0; i < sz; ++i) m[i] = sigmoid(a * theta[i]);
    const auto mf = litho::MaskField::from_real(g, m);
    std::vector<double> gm(sz, 0.0);
    double cost = 0;
    for (int f = 0; f < F; ++f) {
      const auto set = expand_kernels(g, K, weights + std::size_t(f) * K, S, support,
                                      values + 2 * std::size_t(f) * K * S);
      const auto img = litho::image_socs(mf, set, dose);
      const auto r = litho::gaussian_blur(g, img.intensity, sig);
      std::vector<double> d(sz);
      for (std::size_t i = 0; i < sz; ++i) {
        const double z = sigmoid(beta * (r[i] - thr));
        const double e = z - target[i];
        cost += focus_weight[f] * e * e;
        d[i] = 2.0 * focus_weight[f] * e * beta * z * (1.0 - z);
      }
      const auto w = litho::gaussian_blur(g, d, sig);
      const auto gf = weighted_gradient(mf, set, dose, w.data());
      for (std::size_t i = 0; i < sz; ++i) gm[i] += gf[i];
    }
    for (std::size_t i = 0; i < sz; ++i) {
      const double gt = gm[i] * a * m[i] * (1.0 - m[i]);
      if (grad_out) grad_out[i] = gt;
      theta[i] -= step * gt;
    }
    *cost_out = cost;
  });
}

// marching_squares (contour.cpp:58-168): the result is kept for ref_ms_get /
// ref_measure_epe (single-threaded test use)
namespace {
litho::ContourSet g_contours;
}

int ref_marching_squares(int nx, int ny, double pitch, double ox, double oy, const double* field, double thr,
                         int64_t* n_loops, int64_t* n_points) {
  return guarded([&] {
    litho::ResistImage r;
    r.grid = make_grid(nx, ny, pitch, ox, oy);
    r.values.assign(field, field + size_t(nx) * ny);
    g_contours = litho::marching_squares(r, thr);
    int64_t np = 0;
    for (const auto& l : g_contours.loops) np += int64_t(l.size());
    *n_loops = int64_t(g_contours.loops.size());
    *n_points = np;
  });
}

void ref_ms_get(int64_t* loop_start, double* xs, double* ys) {
  int64_t o = 0, k = 0;
  for (const auto& l : g_contours.loops) {
    loop_start[k++] = o;
    for (size_t i = 0; i < l.size(); ++i, ++o) {
      xs[o] = l.xs[i];
      ys[o] = l.ys[i];
    }
  }
  loop_start[k] = o;
}

// measure_epe (contour.cpp:181-201) on the last marching_squares result;
// gauges n x {x, y, nx, ny}
int ref_measure_epe(const double* gauges, int64_t n, double radius, double* epe, uint8_t* open) {
  return guarded([&] {
    std::vector<litho::Gauge> gs(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      gs[i].segment_id = uint32_t(i);
      gs[i].x = gauges[4 * i];
      gs[i].y = gauges[4 * i + 1];
      gs[i].nx = gauges[4 * i + 2];
      gs[i].ny = gauges[4 * i + 3];
    }
    const auto recs = litho::measure_epe(g_contours, gs, radius);
    for (int64_t i = 0; i < n; ++i) {
      epe[i] = recs[i].epe_nm;
      open[i] = recs[i].open ? 1 : 0;
    }
  });
}

// write_aimg / read_aimg (io.cpp:317-350)
int ref_write_aimg(const char* path, int nx, int ny, double pitch, const double* values) {
  return guarded([&] {
    litho::write_aimg(path, make_grid(nx, ny, pitch, 0, 0), std::vector<double>(values, values + size_t(nx) * ny));
  });
}

int ref_read_aimg(const char* path, int* nx, int* ny, double* pitch, double* values, int64_t cap) {
  return guarded([&] {
    litho::Grid g;
    std::vector<double> v;
    litho::read_aimg(path, g, v);
    *nx = g.nx;
    *ny = g.ny;
    *pitch = g.pitch_nm;
    if (values && int64_t(v.size()) <= cap) std::memcpy(values, v.data(), v.size() * sizeof(double));
  });
}

}  // extern "C"
