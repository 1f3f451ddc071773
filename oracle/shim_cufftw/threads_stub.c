/* TEST INFRASTRUCTURE ONLY: ref_capi.cpp's thread knob of the CPU FFT stand-in;
 * cuFFTW needs none. */
void oracle_fft_set_threads(int n) { (void)n; }
