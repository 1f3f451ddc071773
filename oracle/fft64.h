/* TEST INFRASTRUCTURE ONLY (oracle/): fp64 complex DFT used by the CPU oracle
 * and by the FFTW3 stand-in that lets the unmodified reference sources link.
 *
 * Conventions follow the reference's FFT wrapper `fft2` (reference
 * proj/src/core/imaging.cpp:17-31): FFTW_FORWARD = exp(-2*pi*i*k*x/n),
 * FFTW_BACKWARD = exp(+2*pi*i*k*x/n), both unnormalized; 2-D data row-major
 * with x (nx) the contiguous axis, plan dims (ny, nx).
 *
 * FFTW3 itself is an un-vendored, unpinned third-party dependency of the
 * reference (proj/CMakeLists.txt:15, `find_library(FFTW3_LIB fftw3)`), absent
 * from this image. This file restates the published DFT definition: radix-2
 * iterative Cooley-Tukey for powers of two, Bluestein's chirp-z otherwise.
 * Rows / columns are spread over OpenMP threads (oracle_fft_set_threads). */
#ifndef LITHO_ORACLE_FFT64_H
#define LITHO_ORACLE_FFT64_H

#ifdef __cplusplus
extern "C" {
#endif

/* data: interleaved (re, im) doubles, ny rows of nx complex values.
 * sign = -1 forward, +1 backward (unnormalized). */
void oracle_fft2(double* data, int nx, int ny, int sign);
/* 1-D in place on n contiguous complex values */
void oracle_fft1(double* data, int n, int sign);
void oracle_fft_set_threads(int n);
int oracle_fft_get_threads(void);

#ifdef __cplusplus
}
#endif
#endif
