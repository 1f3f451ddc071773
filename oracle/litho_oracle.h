/* TEST INFRASTRUCTURE ONLY — CPU oracle (see litho_oracle.c for the reference
 * file:line each function restates). Callers: tests/, smoke(), bench.py
 * cpu_baseline. Never linked into the product. */
#ifndef LITHO_ORACLE_H
#define LITHO_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
int orc_rasterize(const int64_t* xy, const int64_t* starts, int npoly, int nx, int ny,
                  double pitch, double ox, double oy, double dbu_per_nm, double* out);
int orc_image_socs(int nx, int ny, const double* mask, int K, const double* weights, int S,
                   const int32_t* support, const double* values, double dose, double* out);
int orc_gaussian_blur(int nx, int ny, double pitch, const double* in, double sigma_nm,
                      double* out);
int orc_weighted_gradient(int nx, int ny, const double* mask, int K, const double* weights,
                          int S, const int32_t* support, const double* values, double dose,
                          const double* W, double* grad);
int orc_ilt_iteration(int nx, int ny, double pitch, int F, int K, const double* weights, int S,
                      const int32_t* support, const double* values, const double* focus_weight,
                      const double* params, const double* target, double* theta, double* cost,
                      double* grad);
void orc_set_threads(int n);
#ifdef __cplusplus
}
#endif
#endif
