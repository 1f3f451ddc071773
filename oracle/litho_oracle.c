/* TEST INFRASTRUCTURE ONLY — CPU oracle for the SOCS imaging / ILT hot path.
 *
 * A plain-C fp64 restatement of the reference algorithm (arxiv 2602.15036's
 * `litho` C++ toolkit, /root/reference/proj), used only by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg as the CHECKER.
 * It is never linked into or called by the product path.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * reference itself (oracle/_ref/libref_litho.so, the unmodified reference
 * sources compiled by oracle/build_ref.sh) and against the golden vectors in
 * tests/golden/ generated from it. Build: oracle/Makefile (-O2
 * -ffp-contract=off, matching the reference's x86-64 no-FMA arithmetic).
 */
#include "litho_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "fft64.h"

/* ---------------------------------------------------------------------------
 * Rasterization — restates raster.cpp:17-95 (poly_area :17-25, clip_axis
 * :31-49, rasterize_layer :53-95) on an ALREADY HEALED layer: the reference
 * runs heal() (boolean.hpp:40-42) first; healing is a host precondition here.
 * ------------------------------------------------------------------------- */
typedef struct {
  double* x;
  double* y;
  int n, cap;
} dpoly;

static void dp_reserve(dpoly* p, int cap) {
  if (cap <= p->cap) return;
  p->x = (double*)realloc(p->x, sizeof(double) * (size_t)cap);
  p->y = (double*)realloc(p->y, sizeof(double) * (size_t)cap);
  p->cap = cap;
}

static void dp_push(dpoly* p, double x, double y) {
  if (p->n == p->cap) dp_reserve(p, p->cap ? 2 * p->cap : 16);
  p->x[p->n] = x;
  p->y[p->n] = y;
  p->n++;
}

/* raster.cpp:17-25 */
static double poly_area(const dpoly* p) {
  double a = 0;
  for (int i = 0; i < p->n; ++i) {
    const int j = (i + 1) % p->n;
    a += p->x[i] * p->y[j] - p->x[j] * p->y[i];
  }
  return 0.5 * a;
}

/* raster.cpp:31-49: keep sign*(coord - bound) >= 0; crossing pinned to bound */
static void clip_axis(const dpoly* in, int axis, double bound, double sign, dpoly* out) {
  out->n = 0;
  const int n = in->n;
  for (int i = 0; i < n; ++i) {
    const int j = (i + 1) % n;
    const double x0 = in->x[i], y0 = in->y[i], x1 = in->x[j], y1 = in->y[j];
    const double d0 = sign * ((axis == 0 ? x0 : y0) - bound);
    const double d1 = sign * ((axis == 0 ? x1 : y1) - bound);
    if (d0 >= 0) dp_push(out, x0, y0);
    if ((d0 >= 0) != (d1 >= 0)) {
      const double t = d0 / (d0 - d1);
      if (axis == 0)
        dp_push(out, bound, y0 + t * (y1 - y0));
      else
        dp_push(out, x0 + t * (x1 - x0), bound);
    }
  }
}

int orc_rasterize(const int64_t* xy, const int64_t* starts, int npoly, int nx, int ny,
                  double pitch, double ox, double oy, double dbu_per_nm, double* pix) {
  if (pitch <= 0 || nx <= 0 || ny <= 0) return 1;
  memset(pix, 0, sizeof(double) * (size_t)nx * (size_t)ny);
  const double scale = 1.0 / dbu_per_nm; /* raster.cpp:59 */
  dpoly dp = {0}, r1 = {0}, row = {0}, c1 = {0}, cell = {0};
  for (int p = 0; p < npoly; ++p) {
    const int64_t v0 = starts[p], v1 = starts[p + 1];
    if (v1 - v0 < 3) continue;
    dp.n = 0;
    double minx = 1e300, maxx = -1e300, miny = 1e300, maxy = -1e300;
    for (int64_t v = v0; v < v1; ++v) {
      const double x = ((double)xy[2 * v] * scale - ox) / pitch; /* :68-69 */
      const double y = ((double)xy[2 * v + 1] * scale - oy) / pitch;
      dp_push(&dp, x, y);
      minx = fmin(minx, x);
      maxx = fmax(maxx, x);
      miny = fmin(miny, y);
      maxy = fmax(maxy, y);
    }
    int iy0 = (int)floor(miny), iy1 = (int)ceil(maxy); /* :77-80 */
    int ix0 = (int)floor(minx), ix1 = (int)ceil(maxx);
    if (iy0 < 0) iy0 = 0;
    if (ix0 < 0) ix0 = 0;
    if (iy1 > ny - 1) iy1 = ny - 1;
    if (ix1 > nx - 1) ix1 = nx - 1;
    for (int iy = iy0; iy <= iy1; ++iy) {
      clip_axis(&dp, 1, (double)iy, 1.0, &r1);
      clip_axis(&r1, 1, (double)(iy + 1), -1.0, &row);
      if (row.n < 3) continue;
      for (int ix = ix0; ix <= ix1; ++ix) {
        clip_axis(&row, 0, (double)ix, 1.0, &c1);
        clip_axis(&c1, 0, (double)(ix + 1), -1.0, &cell);
        if (cell.n < 3) continue;
        pix[(size_t)iy * nx + ix] += poly_area(&cell); /* :89 */
      }
    }
  }
  for (size_t i = 0; i < (size_t)nx * ny; ++i) /* :93 clamp [0,1] */
    pix[i] = pix[i] < 0.0 ? 0.0 : (pix[i] > 1.0 ? 1.0 : pix[i]);
  dpoly* all[] = {&dp, &r1, &row, &c1, &cell};
  for (int i = 0; i < 5; ++i) {
    free(all[i]->x);
    free(all[i]->y);
  }
  return 0;
}

/* ---------------------------------------------------------------------------
 * SOCS imaging — restates image_socs (imaging.cpp:218-241) with band-sparse
 * kernel spectra (support entries of the full-grid kernels_freq; the rest are
 * exactly zero by decompose_tcc's scatter, imaging.cpp:198-203).
 * ------------------------------------------------------------------------- */
static size_t wrap_index(int kx, int ky, int nx, int ny) {
  const int x = ((kx % nx) + nx) % nx, y = ((ky % ny) + ny) % ny;
  return (size_t)y * nx + x;
}

/* M^ = FFT(mask) / N^2  (imaging.cpp:222-225) */
static double* mask_spectrum(int nx, int ny, const double* mask) {
  const size_t n = (size_t)nx * ny;
  double* s = (double*)malloc(sizeof(double) * 2 * n);
  for (size_t i = 0; i < n; ++i) {
    s[2 * i] = mask[i];
    s[2 * i + 1] = 0.0;
  }
  oracle_fft2(s, nx, ny, -1);
  const double inv = 1.0 / (double)n;
  for (size_t i = 0; i < 2 * n; ++i) s[i] *= inv;
  return s;
}

/* field = IFFT_unnorm(M^ . H_k) on the full grid (imaging.cpp:234-236) */
static void kernel_field(int nx, int ny, const double* spec, int S, const int32_t* support,
                         const double* kv, double* field) {
  memset(field, 0, sizeof(double) * 2 * (size_t)nx * ny);
  for (int s = 0; s < S; ++s) {
    const size_t i = wrap_index(support[2 * s], support[2 * s + 1], nx, ny);
    const double ar = spec[2 * i], ai = spec[2 * i + 1], br = kv[2 * s], bi = kv[2 * s + 1];
    field[2 * i] = ar * br - ai * bi;
    field[2 * i + 1] = ar * bi + ai * br;
  }
  oracle_fft2(field, nx, ny, +1);
}

int orc_image_socs(int nx, int ny, const double* mask, int K, const double* weights, int S,
                   const int32_t* support, const double* values, double dose, double* out) {
  const size_t n = (size_t)nx * ny;
  double* spec = mask_spectrum(nx, ny, mask);
  double* field = (double*)malloc(sizeof(double) * 2 * n);
  memset(out, 0, sizeof(double) * n);
  for (int k = 0; k < K; ++k) {
    kernel_field(nx, ny, spec, S, support, values + 2 * (size_t)k * S, field);
    const double w = weights[k] * dose; /* :237 */
    for (size_t i = 0; i < n; ++i)
      out[i] += w * (field[2 * i] * field[2 * i] + field[2 * i + 1] * field[2 * i + 1]);
  }
  free(field);
  free(spec);
  return 0;
}

/* ---------------------------------------------------------------------------
 * Gaussian blur — restates gaussian_blur (imaging.cpp:287-314): unit-sum
 * truncated Gaussian on the rectangle |dx|<=rx, |dy|<=ry, r = min(N/2,
 * ceil(6 sigma_px)+1), scattered cyclically, applied via 3 FFTs.
 * ------------------------------------------------------------------------- */
int orc_gaussian_blur(int nx, int ny, double pitch, const double* in, double sigma_nm,
                      double* out) {
  const size_t n = (size_t)nx * ny;
  if (sigma_nm < 0) return 1;
  if (sigma_nm == 0) {
    memcpy(out, in, sizeof(double) * n);
    return 0;
  }
  const double sp = sigma_nm / pitch;
  int rx = (int)ceil(6 * sp) + 1, ry = rx;
  if (rx > nx / 2) rx = nx / 2;
  if (ry > ny / 2) ry = ny / 2;
  double* ker = (double*)calloc(2 * n, sizeof(double));
  double sum = 0;
  for (int dy = -ry; dy <= ry; ++dy)
    for (int dx = -rx; dx <= rx; ++dx) {
      const double v = exp(-0.5 * (dx * dx + dy * dy) / (sp * sp));
      ker[2 * wrap_index(dx, dy, nx, ny)] += v;
      sum += v;
    }
  for (size_t i = 0; i < 2 * n; ++i) ker[i] /= sum;
  oracle_fft2(ker, nx, ny, -1);
  double* f = (double*)malloc(sizeof(double) * 2 * n);
  for (size_t i = 0; i < n; ++i) {
    f[2 * i] = in[i];
    f[2 * i + 1] = 0;
  }
  oracle_fft2(f, nx, ny, -1);
  for (size_t i = 0; i < n; ++i) {
    const double kr = ker[2 * i] / (double)n, ki = ker[2 * i + 1] / (double)n;
    const double fr = f[2 * i], fi = f[2 * i + 1];
    f[2 * i] = fr * kr - fi * ki;
    f[2 * i + 1] = fr * ki + fi * kr;
  }
  oracle_fft2(f, nx, ny, +1);
  for (size_t i = 0; i < n; ++i) out[i] = f[2 * i];
  free(f);
  free(ker);
  return 0;
}

/* ---------------------------------------------------------------------------
 * Adjoint — restates intensity_gradient (ai.cpp:11-42):
 *   grad(x) = sum_k 2 dose w_k Re[ IFFT( FFT(W . E_k) . conj(H_k) / N^2 ) ](x)
 * with the ILT generalisation W(r) = dL/dI(r) inserted before the forward FFT
 * (SURVEY.md §8a row A8). W == NULL is the reference's uniform case W == 1.
 * ------------------------------------------------------------------------- */
int orc_weighted_gradient(int nx, int ny, const double* mask, int K, const double* weights,
                          int S, const int32_t* support, const double* values, double dose,
                          const double* W, double* grad) {
  const size_t n = (size_t)nx * ny;
  const double inv = 1.0 / (double)n;
  double* spec = mask_spectrum(nx, ny, mask);
  double* field = (double*)malloc(sizeof(double) * 2 * n);
  double* corr = (double*)calloc(2 * n, sizeof(double));
  memset(grad, 0, sizeof(double) * n);
  for (int k = 0; k < K; ++k) {
    const double* kv = values + 2 * (size_t)k * S;
    kernel_field(nx, ny, spec, S, support, kv, field); /* A_k, ai.cpp:29-31 */
    for (size_t i = 0; i < n; ++i) {
      const double w = W ? W[i] : 1.0;
      field[2 * i] *= w;
      field[2 * i + 1] *= w;
    }
    oracle_fft2(field, nx, ny, -1); /* ai.cpp:34 */
    memset(corr, 0, sizeof(double) * 2 * n);
    for (int s = 0; s < S; ++s) { /* x conj(H_k)/N^2, zero off-support (ai.cpp:35-36) */
      const size_t i = wrap_index(support[2 * s], support[2 * s + 1], nx, ny);
      const double ar = field[2 * i], ai = field[2 * i + 1];
      const double br = kv[2 * s] * inv, bi = -kv[2 * s + 1] * inv;
      corr[2 * i] = ar * br - ai * bi;
      corr[2 * i + 1] = ar * bi + ai * br;
    }
    oracle_fft2(corr, nx, ny, +1); /* ai.cpp:37 */
    const double w = 2.0 * weights[k] * dose;
    for (size_t i = 0; i < n; ++i) grad[i] += w * corr[2 * i];
  }
  free(corr);
  free(field);
  free(spec);
  return 0;
}

/* ---------------------------------------------------------------------------
 * ILT iteration (absent from the reference), composed
 * from the restated primitives above:
 *   M = sigmoid(a theta);  per focus f: I_f = image_socs(M, H_f, dose),
 *   R_f = blur(I_f), Z_f = sigmoid(beta (R_f - t)),
 *   L = sum_f c_f sum_r (Z_f - Z_t)^2,
 *   dL/dR_f = 2 c_f (Z_f - Z_t) beta Z_f (1 - Z_f),  W_f = blur(dL/dR_f),
 *   dL/dM = sum_f weighted_gradient(M, H_f, W_f),  dL/dtheta = dL/dM a M (1-M),
 *   theta <- theta - step dL/dtheta.
 * params = {a, beta, t, sigma_nm, dose, step}.
 * ------------------------------------------------------------------------- */
static double sigm(double x) { return 1.0 / (1.0 + exp(-x)); }

int orc_ilt_iteration(int nx, int ny, double pitch, int F, int K, const double* weights, int S,
                      const int32_t* support, const double* values, const double* focus_weight,
                      const double* params, const double* target, double* theta, double* cost_out,
                      double* grad_out) {
  const size_t n = (size_t)nx * ny;
  const double a = params[0], beta = params[1], thr = params[2], sig = params[3],
               dose = params[4], step = params[5];
  double* m = (double*)malloc(sizeof(double) * n);
  double* img = (double*)malloc(sizeof(double) * n);
  double* r = (double*)malloc(sizeof(double) * n);
  double* d = (double*)malloc(sizeof(double) * n);
  double* w = (double*)malloc(sizeof(double) * n);
  double* gf = (double*)malloc(sizeof(double) * n);
  double* gm = (double*)calloc(n, sizeof(double));
  for (size_t i = 0; i < n; ++i) m[i] = sigm(a * theta[i]);
  double cost = 0;
  for (int f = 0; f < F; ++f) {
    const double* wf = weights + (size_t)f * K;
    const double* vf = values + 2 * (size_t)f * K * S;
    orc_image_socs(nx, ny, m, K, wf, S, support, vf, dose, img);
    orc_gaussian_blur(nx, ny, pitch, img, sig, r);
    for (size_t i = 0; i < n; ++i) {
      const double z = sigm(beta * (r[i] - thr));
      const double e = z - target[i];
      cost += focus_weight[f] * e * e;
      d[i] = 2.0 * focus_weight[f] * e * beta * z * (1.0 - z);
    }
    orc_gaussian_blur(nx, ny, pitch, d, sig, w);
    orc_weighted_gradient(nx, ny, m, K, wf, S, support, vf, dose, w, gf);
    for (size_t i = 0; i < n; ++i) gm[i] += gf[i];
  }
  for (size_t i = 0; i < n; ++i) {
    const double g = gm[i] * a * m[i] * (1.0 - m[i]);
    if (grad_out) grad_out[i] = g;
    theta[i] -= step * g;
  }
  *cost_out = cost;
  free(m);
  free(img);
  free(r);
  free(d);
  free(w);
  free(gf);
  free(gm);
  return 0;
}

void orc_set_threads(int n) { oracle_fft_set_threads(n); }
