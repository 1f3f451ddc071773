// Host-side interface of the fp32 fast path (power-of-two tiles): one
// launcher per kernel, each enqueues exactly one kernel on `s`.
// Kernels live in socs_fast.cuh; launchers are split over fast_rows.cu /
// fast_cols.cu so the template instantiations compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include "fft.cuh"
#include "geom.h"

namespace lg {

struct FGeo {
  AxisGeom ax, ay;
  int F, K;
  // per-stage twiddle tables (fftr.cuh layout) for Nx, Ny, nx, ny
  const cx<float>* twNx;
  const cx<float>* twNy;
  const cx<float>* twnx;
  const cx<float>* twny;
  // launch trace (LITHOGPU_TRACE): per-CTA [start, end] %globaltimer of
  // launch `trace_slot`, kTraceCtas CTAs per slot; null = off
  unsigned long long* trace = nullptr;
  int trace_slot = 0;
  // row stride (complex elements) of the per-kernel column spectra T[fk][sy][.]:
  // the band width Bx rounded up to even, so every row is a 16-byte multiple
  // (TMA bulk copies in fk_socs_rows)
  int tld = 0;
  // reverse the tile order (blockIdx.z) of this launch (see tz() in socs_fast.cuh)
  int zrev = 0;
  // mixed kernel pairs (Plan::make_pairs): 0 marks an empty kernel slot that
  // every kernel skips; null = all slots active
  const int* slot_on = nullptr;
};
constexpr int kTraceCtas = 4096;

using C32 = cx<float>;

inline bool fast_len_ok(int L) {
  for (int v : kFastLens)
    if (v == L) return true;
  return false;
}
int fast_tw_len(int len);
void fast_set_pdl(bool on);  // programmatic dependent launch for subsequent fast launches
int fast_tpr(int len);  // threads per row group of the length-len plan
void fast_fill_twiddles(int len, C32* host_out);  // fftr per-stage layout

// ---- row kernels (fast_rows.cu) ----
void fl_real_rows_fwd(const FGeo& g, cudaStream_t s, int tiles, int mode, const float* src,
                      long long src_ts, float steep, int Pout, C32* out, long long out_ts);
// SOCS rows with the fixed-order sum over the K kernels and the intensity row
// transform: T -> Ir[F][P+1][n].  Eo (nullable): keep E_fk[sy][x] for
// fl_adj_rows(from_e)
// wk2 != nullptr: g.K kernel pairs with weights wk (real part) / wk2 (imaginary part)
void fl_socs_rows(const FGeo& g, cudaStream_t s, int tiles, const C32* T, long long t_ts,
                  const float* wk, const float* wk2, float dose, C32* Ir, long long ir_ts, C32* Eo,
                  long long e_ts);
void fl_resist_rows(const FGeo& g, cudaStream_t s, int tiles, const C32* Rc, long long c_ts,
                    const float* target, long long tg_ts, const float* cf, float beta, float thr,
                    C32* Dr, long long d_ts, double* costp, long long cp_ts);
void fl_out_rows(const FGeo& g, cudaStream_t s, int tiles, const C32* Ic, const C32* Rc,
                 long long c_ts, float* Iout, float* Rout, unsigned char* print, long long o_ts,
                 float thr);
void fl_wlp_rows(const FGeo& g, cudaStream_t s, int tiles, int nf, const C32* Wc, long long w_ts,
                 float* Wsub, long long ws_ts);
// from_e: T holds E_fk[sy][x] (fl_socs_rows Eo) instead of the column pass T_fk[sy][cx]
void fl_adj_rows(const FGeo& g, cudaStream_t s, int tiles, int nf, bool uniform, bool from_e,
                 const C32* T, long long t_ts, const float* Wsub, long long ws_ts, C32* U, long long u_ts);
void fl_grad_rows(const FGeo& g, cudaStream_t s, int tiles, bool ilt, const C32* Gc, long long g_ts,
                  float* grad, long long gr_ts, float* theta, long long th_ts, float steep,
                  float step, C32* Mr, long long mr_ts, double* gmaxp, long long gm_ts);

// ---- column kernels (fast_cols.cu) ----
void fl_mask_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* Mr, long long mr_ts,
                  C32* Mhat, long long mh_ts);
void fl_socs_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* Mhat, long long mh_ts,
                  const C32* H, C32* T, long long t_ts);
// column FFT of length Ly (ny or Ny) -> intensity band (optionally x Gaussian)
void fl_band_colfwd(const FGeo& g, cudaStream_t s, int tiles, int nf, bool sub, const C32* in,
                    long long in_ts, const float* gxh, const float* gyb, C32* outR, C32* outI,
                    long long o_ts);
// intensity band -> column IFFT of length Ly (Ny if !sub else ny)
void fl_band_colinv(const FGeo& g, cudaStream_t s, int tiles, int nf, bool sub, const C32* band,
                    long long b_ts, C32* out, long long o_ts);
void fl_adj_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* U, long long u_ts,
                 const C32* H, const float* wk, float dose, C32* Acc, long long a_ts);
// Acc: the per-kernel-group partials of fl_adj_cols, summed in fixed order;
// nsum = F*K (the launcher divides by the groups)
void fl_grad_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* Acc, long long a_ts, int nsum,
                  C32* Gc, long long g_ts, const double* costp, long long cp_ts, int ncost,
                  double* cost_out, long long co_ts);
// fused fl_band_colfwd + fl_band_colinv (false when the plan pair is not
// supported: caller falls back to the two-pass form)
bool fl_band_col2(const FGeo& g, cudaStream_t s, int tiles, int nf, bool sub_in, const C32* in,
                  long long in_ts, const float* gxh, const float* gyb, C32* outR, C32* outI,
                  long long o_ts);

}  // namespace lg
