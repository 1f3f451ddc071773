/* TEST INFRASTRUCTURE ONLY: route the reference's FFTW3 calls (imaging.cpp:17-31)
 * to NVIDIA cuFFTW, the FFTW-compatible front end of cuFFT (library GPU
 * baseline of the unmodified reference; oracle/build_ref_cufftw.sh). */
#pragma once
#include <cufftw.h>
