/* TEST INFRASTRUCTURE ONLY (oracle/). See fft64.h. */
#include "fft64.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

static int g_threads = 1;
void oracle_fft_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int oracle_fft_get_threads(void) { return g_threads; }

typedef struct plan1d {
  int n, pow2, log2n;
  cplx* tw;  /* n/2 twiddles exp(-2 pi i k / n) (pow2) */
  int* rev;  /* bit reversal (pow2) */
  /* Bluestein */
  int m;
  cplx* chirp;  /* exp(-i pi k^2 / n), k < n            */
  cplx* bhat;   /* FFT_m of conj(chirp) wrapped         */
  struct plan1d* sub;
} plan1d;

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

static plan1d* plan_create(int n);

static void plan_free(plan1d* p) {
  if (!p) return;
  free(p->tw);
  free(p->rev);
  free(p->chirp);
  free(p->bhat);
  plan_free(p->sub);
  free(p);
}

/* forward (sign -1) radix-2 DIT on a power-of-two length */
static void exec_pow2(const plan1d* p, cplx* x, int sign) {
  const int n = p->n;
  for (int i = 0; i < n; ++i) {
    const int j = p->rev[i];
    if (j > i) {
      cplx t = x[i];
      x[i] = x[j];
      x[j] = t;
    }
  }
  for (int len = 2; len <= n; len <<= 1) {
    const int half = len >> 1;
    const int step = n / len;
    for (int i = 0; i < n; i += len) {
      for (int k = 0; k < half; ++k) {
        cplx w = p->tw[k * step];
        if (sign > 0) w = conj(w);
        const cplx a = x[i + k];
        const cplx b = x[i + k + half] * w;
        x[i + k] = a + b;
        x[i + k + half] = a - b;
      }
    }
  }
}

static void exec(const plan1d* p, cplx* x, int sign, cplx* scratch) {
  if (p->n <= 1) return;
  if (p->pow2) {
    exec_pow2(p, x, sign);
    return;
  }
  /* Bluestein: X_m = c_m * sum_k (x_k c_k) conj(c_{m-k}), c_j = exp(s i pi j^2/n) */
  const int n = p->n, m = p->m;
  cplx* a = scratch;
  for (int k = 0; k < n; ++k) {
    const cplx c = sign < 0 ? p->chirp[k] : conj(p->chirp[k]);
    a[k] = x[k] * c;
  }
  for (int k = n; k < m; ++k) a[k] = 0;
  exec_pow2(p->sub, a, -1);
  for (int k = 0; k < m; ++k) {
    /* bhat holds FFT of conj(chirp) for sign -1; for sign +1 the kernel is
     * chirp, whose FFT is conj(bhat) index-reversed: use direct relation */
    a[k] *= sign < 0 ? p->bhat[k] : conj(p->bhat[(m - k) % m]);
  }
  exec_pow2(p->sub, a, +1);
  const double inv = 1.0 / m;
  for (int k = 0; k < n; ++k) {
    const cplx c = sign < 0 ? p->chirp[k] : conj(p->chirp[k]);
    x[k] = a[k] * inv * c;
  }
}

static plan1d* plan_create(int n) {
  plan1d* p = (plan1d*)calloc(1, sizeof(plan1d));
  p->n = n;
  p->pow2 = is_pow2(n);
  if (n <= 1) return p;
  if (p->pow2) {
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    p->log2n = lg;
    p->tw = (cplx*)malloc(sizeof(cplx) * (size_t)(n / 2 > 0 ? n / 2 : 1));
    for (int k = 0; k < n / 2; ++k) {
      const double ang = -2.0 * M_PI * (double)k / (double)n;
      p->tw[k] = cos(ang) + I * sin(ang);
    }
    p->rev = (int*)malloc(sizeof(int) * (size_t)n);
    for (int i = 0; i < n; ++i) {
      int r = 0;
      for (int b = 0; b < lg; ++b)
        if (i & (1 << b)) r |= 1 << (lg - 1 - b);
      p->rev[i] = r;
    }
    return p;
  }
  int m = 1;
  while (m < 2 * n - 1) m <<= 1;
  p->m = m;
  p->sub = plan_create(m);
  p->chirp = (cplx*)malloc(sizeof(cplx) * (size_t)n);
  for (long long k = 0; k < n; ++k) {
    const long long k2 = (k * k) % (2LL * n);
    const double ang = -M_PI * (double)k2 / (double)n;
    p->chirp[k] = cos(ang) + I * sin(ang);
  }
  p->bhat = (cplx*)calloc((size_t)m, sizeof(cplx));
  p->bhat[0] = conj(p->chirp[0]);
  for (int k = 1; k < n; ++k) {
    p->bhat[k] = conj(p->chirp[k]);
    p->bhat[m - k] = conj(p->chirp[k]);
  }
  exec_pow2(p->sub, p->bhat, -1);
  return p;
}

static int scratch_len(const plan1d* p) { return p->pow2 ? 1 : p->m; }

void oracle_fft1(double* data, int n, int sign) {
  plan1d* p = plan_create(n);
  cplx* s = (cplx*)malloc(sizeof(cplx) * (size_t)scratch_len(p));
  exec(p, (cplx*)data, sign, s);
  free(s);
  plan_free(p);
}

void oracle_fft2(double* data, int nx, int ny, int sign) {
  if (nx <= 0 || ny <= 0) return;
  cplx* d = (cplx*)data;
  plan1d* px = plan_create(nx);
  plan1d* py = plan_create(ny);
  const int nth = g_threads;
  /* rows */
#pragma omp parallel num_threads(nth)
  {
    cplx* s = (cplx*)malloc(sizeof(cplx) * (size_t)scratch_len(px));
#pragma omp for schedule(static)
    for (int y = 0; y < ny; ++y) exec(px, d + (size_t)y * nx, sign, s);
    free(s);
  }
  /* columns, gathered in blocks of CB for cache locality */
  enum { CB = 8 };
  const int nblk = (nx + CB - 1) / CB;
#pragma omp parallel num_threads(nth)
  {
    cplx* col = (cplx*)malloc(sizeof(cplx) * (size_t)ny * CB);
    cplx* s = (cplx*)malloc(sizeof(cplx) * (size_t)scratch_len(py));
#pragma omp for schedule(static)
    for (int b = 0; b < nblk; ++b) {
      const int x0 = b * CB;
      const int w = nx - x0 < CB ? nx - x0 : CB;
      for (int y = 0; y < ny; ++y)
        for (int c = 0; c < w; ++c) col[(size_t)c * ny + y] = d[(size_t)y * nx + x0 + c];
      for (int c = 0; c < w; ++c) exec(py, col + (size_t)c * ny, sign, s);
      for (int y = 0; y < ny; ++y)
        for (int c = 0; c < w; ++c) d[(size_t)y * nx + x0 + c] = col[(size_t)c * ny + y];
    }
    free(col);
    free(s);
  }
  plan_free(px);
  plan_free(py);
}
