/* TEST INFRASTRUCTURE ONLY: FFTW3 stand-in implementation (see fftw3.h). */
#include <stdlib.h>
#include <string.h>

#include "../fft64.h"
#include "fftw3.h"

struct oracle_fftw_plan_s {
  int n0, n1, sign;
  fftw_complex *in, *out;
};

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
  (void)flags;
  fftw_plan p = (fftw_plan)malloc(sizeof(*p));
  p->n0 = n0; /* rows (ny) */
  p->n1 = n1; /* contiguous (nx) */
  p->sign = sign;
  p->in = in;
  p->out = out;
  return p;
}

void fftw_execute(const fftw_plan p) {
  if (p->in != p->out) memcpy(p->out, p->in, sizeof(fftw_complex) * (size_t)p->n0 * p->n1);
  oracle_fft2((double*)p->out, p->n1, p->n0, p->sign);
}

void fftw_destroy_plan(fftw_plan p) { free(p); }
