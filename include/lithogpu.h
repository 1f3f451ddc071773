/* lithogpu — C ABI of the B200-native SOCS imaging / ILT hot path.
 *
 * Drop-in boundary for the reference `litho` toolkit (arxiv 2602.15036,
 * /root/reference/proj).  Each entry point replaces one reference function
 * on the north-star path; the replaced interface is cited beside it.  The
 * reference's own C ABI conventions are kept (proj/include/litho/litho.h:1-20):
 * every call returns a status, failures leave a thread-local message in
 * lithogpu_last_error(), objects returned through out-parameters are owned by
 * the caller and released with the matching _destroy, and no C++ exception
 * ever crosses this boundary (CUDA failures map to LITHOGPU_ERR_DOMAIN).
 *
 * Buffers are plain pointers.  Each pointer may be HOST memory (pageable or
 * pinned: staged through the context's device scratch, the call returns after
 * the results are back on the host) or DEVICE memory of the context's GPU
 * (stream-ordered on the context stream, no host synchronisation; call
 * lithogpu_ctx_synchronize before reading).  Images are row-major, x fastest,
 * index iy*nx + ix (reference raster.hpp:18).
 *
 * Thread safety: a context (and the objects created from it) is used by one
 * host thread at a time; different contexts are independent (one per GPU /
 * per host thread).  Kernel stacks are read-only after creation.
 */
#ifndef LITHOGPU_H
#define LITHOGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LITHOGPU_OK = 0,
  LITHOGPU_ERR_DOMAIN = 1, /* invalid input data or failed computation (incl. CUDA errors) */
  LITHOGPU_ERR_USAGE = 2   /* bad arguments (null pointers, unknown enums) */
} lithogpu_status;

typedef enum { LITHOGPU_F32 = 0, LITHOGPU_F64 = 1, LITHOGPU_U8 = 2 } lithogpu_dtype;

/* Thread-local message for the last failing call; "" if none.
 * Replaces litho_last_error (litho.h:19-20, litho_c.cpp:22-42). */
const char* lithogpu_last_error(void);

/* Uniform pixel grid; pixel (ix,iy) covers [origin + i*pitch, origin+(i+1)*pitch)
 * (reference Grid, raster.hpp:10-20). */
typedef struct {
  int nx, ny;
  double pitch_nm;
  double origin_x_nm, origin_y_nm;
} lithogpu_grid;

/* ---- context ---------------------------------------------------------- */
typedef struct lithogpu_ctx lithogpu_ctx;
lithogpu_status lithogpu_ctx_create(int device, lithogpu_ctx** out);
void lithogpu_ctx_destroy(lithogpu_ctx* ctx);
/* cudaStream_t to launch on (NULL = the legacy default stream) */
lithogpu_status lithogpu_ctx_set_stream(lithogpu_ctx* ctx, void* stream);
lithogpu_status lithogpu_ctx_synchronize(lithogpu_ctx* ctx);
/* number of kernels this context launched so far (instrumentation) */
long long lithogpu_ctx_launch_count(const lithogpu_ctx* ctx);

/* Per-launch CUDA-event timing of every kernel this context launches
 * (instrumentation for the roofline; adds one event pair per launch). */
lithogpu_status lithogpu_ctx_set_profiling(lithogpu_ctx* ctx, int on);
/* "name count total_ms" lines, aggregated since the last reset */
lithogpu_status lithogpu_ctx_profile_report(lithogpu_ctx* ctx, char* buf, size_t len, int reset);
/* FFMA-pipe peak of the context's GPU, TFLOP/s (microbenchmark, ~1 ms) */
lithogpu_status lithogpu_fp32_peak(lithogpu_ctx* ctx, double* tflops);

/* ---- rasterization ------------------------------------------------------
 * Exact area-weighted coverage in fp64, bit-exact with the reference
 * rasterize_layer (raster.cpp:53-95) on a HEALED layer: polygons must be the
 * output of the reference heal() (boolean.hpp:40-42) — disjoint, CCW outers /
 * CW holes, canonical order.  Vertices are int64 dbu (geometry.hpp:15);
 * polygon p is xy[2*poly_start[p] .. 2*poly_start[p+1]).  out: nx*ny f64. */
lithogpu_status lithogpu_rasterize(lithogpu_ctx* ctx, const lithogpu_grid* grid,
                                   const int64_t* xy, const int64_t* poly_start, int n_poly,
                                   double dbu_per_nm, double* out);

/* ---- SOCS kernel stacks -------------------------------------------------
 * Replaces SocsKernelSet (imaging.hpp:78-87) and build_optics' per-focus
 * stacks (opc.cpp:114-124).  n_focus stacks of `order` kernels share one
 * frequency support of n_support signed DFT indices (kx, ky) (the TCC support,
 * imaging.cpp:120-129); values[f][k][s] = kernels_freq[k] at that index
 * (interleaved re, im).  weights[f][k] >= 0.  precision LITHOGPU_F32 (fast
 * path) or LITHOGPU_F64 (reference-tolerance path). */
typedef struct lithogpu_kernels lithogpu_kernels;
lithogpu_status lithogpu_kernels_create(lithogpu_ctx* ctx, const lithogpu_grid* grid,
                                        lithogpu_dtype precision, int n_focus, int order,
                                        const double* weights, int n_support,
                                        const int32_t* support, const double* values,
                                        lithogpu_kernels** out);
void lithogpu_kernels_destroy(lithogpu_kernels* ks);
/* geometry chosen for the tile: decimated grid and kernel band */
lithogpu_status lithogpu_kernels_info(const lithogpu_kernels* ks, int* nx_sub, int* ny_sub,
                                      int* band_x, int* band_y);
/* transforms per focus stack on the fp32 fast path: K, or ceil(K/2) when the
 * kernels are Hermitian-symmetric and run as pairs; 0 when the
 * stack runs on the generic path */
lithogpu_status lithogpu_kernels_fast_order(const lithogpu_kernels* ks, int* order);
/* focus stacks the fast path computes: F, fewer when a stack is the conjugate
 * mirror of another (paraxial -F / +F under a point-symmetric source; both
 * print the same image) */
lithogpu_status lithogpu_kernels_fast_stacks(const lithogpu_kernels* ks, int* stacks);

/* ---- imaging ------------------------------------------------------------
 * image_socs (imaging.cpp:218-241): I = dose * sum_k w_k |IFFT(FFT(mask)/N^2 H_k)|^2
 * for focus stack `focus`.  mask: nx*ny real (f32/f64); intensity: nx*ny. */
lithogpu_status lithogpu_image_socs(lithogpu_kernels* ks, int focus, const void* mask,
                                    lithogpu_dtype mask_dtype, double dose, void* intensity,
                                    lithogpu_dtype out_dtype);

/* Fused forward: aerial image + resist_filter (imaging.cpp:316-323, Gaussian
 * blur sigma_nm) + threshold map (ResistImage threshold, v >= threshold -> 1).
 * Any of intensity / resist / print may be NULL. */
lithogpu_status lithogpu_image_resist(lithogpu_kernels* ks, int focus, const void* mask,
                                      lithogpu_dtype mask_dtype, double dose, double sigma_nm,
                                      double threshold, void* intensity, void* resist,
                                      lithogpu_dtype out_dtype, unsigned char* print);

/* gaussian_blur (imaging.cpp:287-314): cyclic unit-sum truncated Gaussian,
 * radius min(N/2, ceil(6 sigma_px)+1); sigma 0 = identity. */
lithogpu_status lithogpu_gaussian_blur(lithogpu_ctx* ctx, const lithogpu_grid* grid,
                                       const void* in, lithogpu_dtype dtype, double sigma_nm,
                                       void* out);

/* fft2 (imaging.cpp:17-31): in-place 2-D DFT of ny rows of nx interleaved
 * complex values (dtype F64: complex128, F32: complex64); forward e^{-i},
 * inverse e^{+i}, both unnormalized.  Any sizes. */
lithogpu_status lithogpu_fft2(lithogpu_ctx* ctx, void* data, lithogpu_dtype dtype, int nx, int ny,
                              int inverse);

/* z_print / threshold semantics (ai.cpp:85-94): out[i] = in[i] >= tau ? 1 : 0 */
lithogpu_status lithogpu_threshold(lithogpu_ctx* ctx, size_t n, const void* in,
                                   lithogpu_dtype in_dtype, double tau, void* out,
                                   lithogpu_dtype out_dtype);

/* ---- adjoint --------------------------------------------------------------
 * intensity_gradient (ai.cpp:11-42) generalised with a per-pixel weight W:
 *   grad(x) = sum_r W(r) dI(r)/dM(x)
 *           = sum_k 2 dose w_k Re IFFT(FFT(W E_k) conj(H_k)/N^2)(x).
 * weight == NULL is the reference's uniform case (d sum_r I / dM). */
lithogpu_status lithogpu_intensity_gradient(lithogpu_kernels* ks, int focus, const void* mask,
                                            lithogpu_dtype mask_dtype, const void* weight,
                                            lithogpu_dtype weight_dtype, double dose, void* grad,
                                            lithogpu_dtype grad_dtype);

/* ---- pixel ILT (through-focus) --------------------------------------------
 * Not in the reference.  Per tile:
 *   M = sigmoid(mask_steepness * theta);  for each focus stack f:
 *   R_f = blur(image_socs(M, H_f, dose), resist_sigma_nm),
 *   Z_f = sigmoid(resist_beta * (R_f - threshold)),
 *   cost = sum_f focus_weights[f] * sum_r (Z_f - target)^2,
 *   theta <- theta - step * dcost/dtheta   (exact adjoint, all foci).   */
typedef struct {
  double mask_steepness;
  double resist_beta;
  double threshold;
  double resist_sigma_nm;
  double dose;
  double step;
  const double* focus_weights; /* n_focus entries (host) */
} lithogpu_ilt_params;

typedef struct lithogpu_ilt lithogpu_ilt;
lithogpu_status lithogpu_ilt_create(lithogpu_kernels* ks, const lithogpu_ilt_params* params,
                                    int n_tiles, lithogpu_ilt** out);
void lithogpu_ilt_destroy(lithogpu_ilt* ilt);
/* target: nx*ny in [0,1]; theta0 NULL -> theta0 = (2*target-1)*2/steepness */
lithogpu_status lithogpu_ilt_set_tile(lithogpu_ilt* ilt, int tile, const void* target,
                                      const void* theta0, lithogpu_dtype dtype);
/* all tiles target/theta at once: n_tiles*nx*ny each (theta0 may be NULL) */
lithogpu_status lithogpu_ilt_set_tiles(lithogpu_ilt* ilt, const void* target,
                                       const void* theta0, lithogpu_dtype dtype);
/* Run `iterations` steps on all tiles.  cost (nullable): iterations*n_tiles
 * f64, cost[i*n_tiles+t] = cost of tile t BEFORE update i; gmax (nullable):
 * max |dcost/dtheta| per iteration and tile, same layout. */
lithogpu_status lithogpu_ilt_run(lithogpu_ilt* ilt, int iterations, double* cost,
                                 double* gmax);
/* Cost and exact gradient dcost/dtheta at the CURRENT theta of every tile,
 * without updating theta (one iteration of the same kernels with step 0).
 * cost (nullable): n_tiles f64; grad: n_tiles*nx*ny of `dtype` (F32/F64),
 * host or device.  The oracle twin is orc_ilt_iteration's grad_out
 * (oracle/litho_oracle.c); W = 1 reduces it to intensity_gradient
 * (ai.cpp:11-42) chained through the resist and mask sigmoids. */
lithogpu_status lithogpu_ilt_gradient(lithogpu_ilt* ilt, double* cost, void* grad, lithogpu_dtype dtype);
/* theta and/or mask = sigmoid(steepness*theta) of one tile (nullable outs) */
lithogpu_status lithogpu_ilt_get_tile(lithogpu_ilt* ilt, int tile, void* theta, void* mask,
                                      lithogpu_dtype dtype);
/* Mask window of one tile for chip stitching (only tile
 * cores are kept): out[r*row_stride + c] = sigmoid(steepness*theta) at pixel
 * (x0 + c, y0 + r) of `tile`, r < h, c < w (dtype F32/F64; host or device;
 * e.g. the core [halo, halo+core)^2 written straight into the chip image). */
lithogpu_status lithogpu_ilt_get_window(lithogpu_ilt* ilt, int tile, int x0, int y0, int w, int h, void* mask,
                                        int64_t row_stride, lithogpu_dtype dtype);
/* The same, stream-ordered on the context stream without waiting: `mask` is
 * device memory or PAGE-LOCKED host memory (cudaHostAlloc / pinned), valid
 * once the context stream has passed the copy (lithogpu_ctx_synchronize).
 * Lets a caller pipeline the D2H of one tile batch under the next batch's
 * iterations (e.g. on a second context).  Pageable host memory: USAGE. */
lithogpu_status lithogpu_ilt_get_window_async(lithogpu_ilt* ilt, int tile, int x0, int y0, int w, int h,
                                              void* mask, int64_t row_stride, lithogpu_dtype dtype);
/* all tiles: n_tiles*nx*ny (nullable outs) */
lithogpu_status lithogpu_ilt_get_tiles(lithogpu_ilt* ilt, void* theta, void* mask,
                                       lithogpu_dtype dtype);

/* ---- contours and EPE gauges of a resist image ----
 * marching_squares (contour.cpp:58-168) of an ny x nx f64 field (host or
 * device; node (ix,iy) at the pixel centre origin + (i+0.5)*pitch) at
 * `threshold`.  The loops are bit-identical to the reference ContourSet: same
 * loop order (ascending smallest grid-edge id), same start point, same point
 * order and fp64 values.  Non-finite fields and open (border-crossing)
 * contours fail with LITHOGPU_ERR_DOMAIN, as the reference throws.  The
 * object keeps the crossing graph on the device for lithogpu_measure_epe. */
typedef struct lithogpu_contours lithogpu_contours;
lithogpu_status lithogpu_marching_squares(lithogpu_ctx* ctx, const lithogpu_grid* grid, const double* field,
                                          double threshold, lithogpu_contours** out);
lithogpu_status lithogpu_contours_size(const lithogpu_contours* c, int64_t* n_loops, int64_t* n_points);
/* loop_start[n_loops+1] offsets into xs/ys[n_points] (host or device buffers;
 * the reference ContourLoop::xs/ys, contour.hpp:13-22) */
lithogpu_status lithogpu_contours_get(const lithogpu_contours* c, int64_t* loop_start, double* xs, double* ys);
void lithogpu_contours_destroy(lithogpu_contours* c);
/* measure_epe (contour.cpp:181-201 over SegmentBvh::nearest_crossing,
 * bvh.cpp:241-273): gauges are n x {x, y, nx, ny} f64 (site and unit outward
 * normal, nm; Gauge contour.hpp:30-34, segment ids stay with the caller).
 * epe_nm[i] = signed distance to the nearest crossing along the normal
 * (|t| <= search_radius, ties to +t), open[i] = 1 when there is none
 * (epe 0).  Host or device buffers. */
lithogpu_status lithogpu_measure_epe(lithogpu_contours* c, const double* gauges, int64_t n,
                                     double search_radius_nm, double* epe_nm, uint8_t* open);

/* measure_epe on an arbitrary ContourSet given as loops (loop_start[n_loops+1]
 * offsets into xs/ys, host or device): segments in loop order as the
 * reference build_contour_bvh (contour.cpp:170-178), every segment scanned on
 * the GPU; same records as lithogpu_measure_epe on a marching-squares set. */
lithogpu_status lithogpu_measure_epe_loops(lithogpu_ctx* ctx, const int64_t* loop_start, int64_t n_loops,
                                           const double* xs, const double* ys, const double* gauges,
                                           int64_t n, double search_radius_nm, double* epe_nm,
                                           uint8_t* open);

/* evaluate_epe (opc.cpp:140-151) without leaving the
 * device: n_masks mask rasters (n_masks x ny x nx, host or device, f32/f64;
 * e.g. the MEEF probe batches of estimate_meef, opc.cpp:153-202) are imaged
 * in ONE batched launch sequence on focus stack `focus`, resist-filtered
 * (gaussian blur sigma_nm), contoured at t_eff (marching_squares) and gauged
 * (measure_epe) with the same n_gauges gauges {x, y, nx, ny}.  epe_nm / open:
 * n_masks x n_gauges; resist (nullable): n_masks x ny x nx f64. */
lithogpu_status lithogpu_evaluate_epe(lithogpu_kernels* ks, int focus, int n_masks, const void* masks,
                                      lithogpu_dtype mask_dtype, double dose, double sigma_nm, double t_eff,
                                      const double* gauges, int64_t n_gauges, double search_radius_nm,
                                      double* epe_nm, uint8_t* open, double* resist);

/* ---- host-side kernel generation (precompute, not on the timed path) ----
 * Replaces build_tcc + decompose_tcc (imaging.cpp:113-216) with the same
 * semantics via the TCC = Q Q^H factorisation (no dense S x S eigensolve, so
 * no 6000-frequency budget).  Error text: lithogpu_host_last_error(). */
const char* lithogpu_host_last_error(void);
/* make_annular_source (imaging.cpp:50-64); sigma_out <= 0 -> point source.
 * out_xyw (3*count doubles: sx, sy, weight) may be NULL to query count. */
lithogpu_status lithogpu_source_annular(double sigma_in, double sigma_out, int grid_n, int* count,
                                        double* out_xyw);
/* TCC support (imaging.cpp:115-129), reference order; out may be NULL */
lithogpu_status lithogpu_tcc_support(int nx, int ny, double pitch_nm, double wavelength_nm,
                                     double na, double max_source_radius, int* count,
                                     int32_t* out_kxky);
/* One focus plane's SOCS kernels on `support`: out_weights[K] descending,
 * out_values[K][n_support] interleaved complex, K <= max_order. */
lithogpu_status lithogpu_socs_kernels(int nx, int ny, double pitch_nm, double wavelength_nm,
                                      double na, int high_na, const double* source_xyw,
                                      int n_source, double focus_nm, int n_support,
                                      const int32_t* support, int k_fixed, double energy_floor,
                                      int max_order, int* out_order, double* out_captured,
                                      double* out_weights, double* out_values);

/* ---- AIMG tile I/O --------------------------------
 * write_aimg (io.cpp:317-330), byte-identical files: "AIMG", u32 nx, u32 ny,
 * f64 pitch, row-major f64 payload (origin not stored, io.cpp:346).  values:
 * n_tiles x ny x nx of `dtype` (host or device; F32/U8 become f64), one path
 * per tile.  Device tiles go through a pinned double buffer: the D2H copy of
 * tile t+1 overlaps the file write of tile t. */
lithogpu_status lithogpu_write_aimg(lithogpu_ctx* ctx, const lithogpu_grid* grid, int n_tiles,
                                    const char* const* paths, const void* values, lithogpu_dtype dtype);
/* read_aimg (io.cpp:332-350): header into nx/ny/pitch; values (host or device
 * f64, nx*ny; NULL = header only).  Reference error messages. */
lithogpu_status lithogpu_read_aimg(lithogpu_ctx* ctx, const char* path, int* nx, int* ny, double* pitch_nm,
                                   double* values);

/* ---- layout JSON -> polygon buffers ------------------
 * Reader of the reference layout format (load_layout, io.cpp:53-116): same
 * validation and error messages (LITHOGPU_ERR_DOMAIN + lithogpu_last_error).
 * A layer's polygons come out flattened for lithogpu_rasterize: xy (2 int64
 * per vertex, dbu) and poly_start (n_poly + 1 offsets), into host OR device
 * memory.  Polygons are as stored (the reference heals inside
 * rasterize_layer; the GPU rasterizer takes healed input). */
typedef struct lithogpu_layout lithogpu_layout;
lithogpu_status lithogpu_layout_load(const char* path, lithogpu_layout** out);
void lithogpu_layout_destroy(lithogpu_layout* layout);
lithogpu_status lithogpu_layout_info(const lithogpu_layout* layout, int* n_layers, int64_t* dbu_num,
                                     int64_t* dbu_den);
lithogpu_status lithogpu_layout_layer(const lithogpu_layout* layout, int layer, const char** name,
                                      int64_t* n_poly, int64_t* n_vert);
lithogpu_status lithogpu_layout_get(const lithogpu_layout* layout, int layer, int64_t* xy, int64_t* poly_start);

/* GPU kernel generation: lithogpu_socs_kernels for
 * n_focus focus planes in one call (fp64; cuBLAS Gram + cuSOLVER eigensolve
 * + cuBLAS kernel assembly).  Same support, ordering, truncation and phase
 * rules; eigenvectors of degenerate eigenvalues may differ by a unitary mix,
 * which leaves the full image unchanged.  Outputs per focus f:
 * out_order[f], out_captured[f] (nullable), out_weights[f*max_order + k],
 * out_values[(f*max_order + k)*n_support*2 ..] (re, im).  Error text:
 * lithogpu_last_error(). */
lithogpu_status lithogpu_socs_kernels_gpu(lithogpu_ctx* ctx, int nx, int ny, double pitch_nm,
                                          double wavelength_nm, double na, int high_na,
                                          const double* source_xyw, int n_source, int n_focus,
                                          const double* focus_nm, int n_support, const int32_t* support,
                                          int k_fixed, double energy_floor, int max_order, int* out_order,
                                          double* out_captured, double* out_weights, double* out_values);

#ifdef __cplusplus
}
#endif
#endif
