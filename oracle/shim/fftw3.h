/* TEST INFRASTRUCTURE ONLY (oracle/_ref build).
 * Minimal FFTW3 API stand-in exposing exactly the five symbols the reference
 * uses in fft2 (reference proj/src/core/imaging.cpp:17-31): fftw_complex,
 * fftw_plan, fftw_plan_dft_2d, fftw_execute, fftw_destroy_plan and the
 * FFTW_FORWARD / FFTW_BACKWARD / FFTW_ESTIMATE constants. FFTW3 is an
 * un-vendored, unpinned dependency of the reference (CMakeLists.txt:15) and is
 * absent from this image; the arithmetic is the fp64 DFT in ../fft64.c. */
#ifndef LITHO_ORACLE_FFTW3_SHIM_H
#define LITHO_ORACLE_FFTW3_SHIM_H
#ifdef __cplusplus
extern "C" {
#endif
typedef double fftw_complex[2];
typedef struct oracle_fftw_plan_s* fftw_plan;
#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)
fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);
#ifdef __cplusplus
}
#endif
#endif
