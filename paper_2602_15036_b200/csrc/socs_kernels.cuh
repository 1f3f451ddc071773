// SOCS forward / adjoint / ILT pipeline kernels (sm_100a, templated on the
// real type T = float for throughput, double for the reference-tolerance
// drop-in mode).  See DESIGN.md §3 for the data flow; every kernel is a
// batched set of 1-D transforms ("row groups", fft.cuh) with its band
// gather / scatter prologue and pointwise epilogue fused in.
//
// Reference anchors (proj/src/core):
//   mask spectrum   M^ = FFT(mask)/N^2                 imaging.cpp:222-225
//   coherent field  E_k = IFFT(M^ . H_k)               imaging.cpp:234-236
//   intensity       I += dose w_k |E_k|^2              imaging.cpp:237-238
//   resist blur     unit-sum truncated Gaussian        imaging.cpp:287-314
//   adjoint         2 dose w_k Re IFFT(FFT(W E_k) conj(H_k)/N^2)  ai.cpp:27-39
#pragma once

#include <cuda_runtime.h>

#include "fft.cuh"
#include "geom.h"

namespace lg {

// per-length transform tables (filled by make_tab in capi.cu)
template <typename T>
struct Tab {
  const cx<T>* tw;  // exp(-2 pi i m / L)
  int L;
  int log2L;  // >= 4 for the radix-16 Stockham path, else -1
  int kind;   // FftKind (fft.cuh)
  int nst;    // mixed radix: stages, radices as nibbles in rad
  unsigned long long rad;
  int M, log2M;        // Bluestein convolution length (0 otherwise)
  const cx<T>* twM;    // exp(-2 pi i m / M)
  const cx<T>* chirp;  // exp(-i pi n^2 / L), n < L
  const cx<T>* bhat;   // FFT_M of the wrapped conj chirp
};

template <typename T>
struct Geo {
  AxisGeom ax, ay;
  Tab<T> tNx, tNy, tnx, tny;
  int F, K;
};

// ---- per-group shared memory ---------------------------------------------
__host__ __device__ inline int imax(int a, int b) { return a > b ? a : b; }

template <typename T>
__host__ __device__ inline bool fast_len(int L) {
  return is_pow2(L) && L >= 16;
}

// elements of T of the group scratch: the mixed-radix ping-pong row
// (unpadded, max(LA, LB) complex) and the Bluestein work row (padded, M
// complex) share it (a transform uses one or the other)
template <typename T>
__host__ __device__ inline int scratch_elems(int LA, int LB) {
  const bool gen = !fast_len<T>(LA) || (LB && !fast_len<T>(LB));
  const int mb = imax(blue_len(LA), LB ? blue_len(LB) : 0);
  int e = gen ? 2 * imax(LA, LB) : 0;
  if (mb) e = imax(e, 2 * padded_len<T>(mb));
  return e;
}

// elements of T: row A + row B + scratch + reduce area (32 doubles)
template <typename T>
__host__ __device__ inline int group_elems(int LA, int LB) {
  int e = 2 * padded_len<T>(LA);
  if (LB) e += 2 * padded_len<T>(LB);
  e += scratch_elems<T>(LA, LB);
  e += 32 * 8 / int(sizeof(T));
  e = (e + 3) & ~3;
  return e;
}

template <typename T>
__host__ __device__ inline int group_threads(int LA, int LB) {
  return imax(fft_tpr(LA), LB ? fft_tpr(LB) : 1);
}

template <typename T>
struct Group {
  T* base;
  int G;    // threads in group
  int t;    // thread index in group
  int gid;  // group index in CTA
  int LA, LB;

  __device__ Group(int LA_, int LB_) : LA(LA_), LB(LB_) {
    extern __shared__ __align__(16) unsigned char g_smem_raw[];
    G = group_threads<T>(LA, LB);
    gid = threadIdx.x / G;
    t = threadIdx.x % G;
    base = reinterpret_cast<T*>(g_smem_raw) + size_t(gid) * group_elems<T>(LA, LB);
  }
  __device__ T* scratch() const {
    return base + 2 * padded_len<T>(LA) + (LB ? 2 * padded_len<T>(LB) : 0);
  }
  __device__ double* red() const {
    return reinterpret_cast<double*>(scratch() + scratch_elems<T>(LA, LB));
  }
  __device__ Row<T> row(int which, const Tab<T>& tab, bool active) const {
    Row<T> r;
    r.L = tab.L;
    r.re = which == 0 ? base : base + 2 * padded_len<T>(LA);
    r.im = r.re + padded_len<T>(tab.L);
    r.sre = scratch();
    r.sim = r.sre + imax(LA, LB);
    r.log2L = tab.log2L;
    r.kind = tab.kind;
    r.nst = tab.nst;
    r.rad = tab.rad;
    r.bre = scratch();
    r.bim = r.bre + padded_len<T>(tab.M > 0 ? tab.M : 1);
    r.M = tab.M;
    r.log2M = tab.log2M;
    r.twM = tab.twM;
    r.chirp = tab.chirp;
    r.bhat = tab.bhat;
    r.TPR = fft_tpr(tab.L);
    r.t = t;
    r.active = active && t < r.TPR;
    r.cta_sync = G > 32;
    r.tw = tab.tw;
    return r;
  }
  __device__ void sync() const {
    if (G > 32)
      __syncthreads();
    else
      __syncwarp();
  }
  // sum over the group's threads (all threads of the CTA must call)
  __device__ double reduce_sum(double v) const {
    const int w = G < 32 ? G : 32;
    for (int o = w / 2; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, w);
    if (G <= 32) return __shfl_sync(0xffffffffu, v, 0, w);
    double* r = red();
    __syncthreads();
    if ((t & 31) == 0) r[t >> 5] = v;
    __syncthreads();
    double s = 0;
    for (int i = 0; i < G / 32; ++i) s += r[i];
    __syncthreads();
    return s;
  }
  __device__ double reduce_max(double v) const {
    const int w = G < 32 ? G : 32;
    for (int o = w / 2; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o, w));
    if (G <= 32) return __shfl_sync(0xffffffffu, v, 0, w);
    double* r = red();
    __syncthreads();
    if ((t & 31) == 0) r[t >> 5] = v;
    __syncthreads();
    double s = r[0];
    for (int i = 1; i < G / 32; ++i) s = fmax(s, r[i]);
    __syncthreads();
    return s;
  }
};

template <typename T>
__device__ __forceinline__ T sigm(T x) {
  return T(1) / (T(1) + exp(-x));
}
template <>
__device__ __forceinline__ float sigm<float>(float x) {
  return 1.0f / (1.0f + __expf(-x));
}


// ===========================================================================
// Full-grid real row pairs -> half spectra px in [0, Pout] (column-major out)
//   MODE 0: rows of a real image (mask or weight field)
//   MODE 1: rows of sigmoid(steep * theta)   (ILT mask parametrisation)
// Packs rows (y, y+1) into one complex FFT_Nx (real-pair trick).
// ===========================================================================
template <typename T, int MODE>
__global__ void k_real_rows_fwd(Geo<T> g, const T* __restrict__ src, long long src_ts, T steep,
                                int Pout, cx<T>* __restrict__ out, long long out_ts) {
  Group<T> grp(g.ax.N, 0);
  const int Nx = g.ax.N, Ny = g.ay.N;
  const int pair = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const bool active = pair < (Ny + 1) / 2;
  const int tile = blockIdx.z;
  const Row<T> row = grp.row(0, g.tNx, active);
  const int y0 = 2 * pair, y1 = y0 + 1;
  const bool has1 = y1 < Ny;
  const T* s = src + tile * src_ts;
  if (row.active) {
    for (int i = row.t; i < Nx; i += row.TPR) {
      T a = s[size_t(y0) * Nx + i];
      T b = has1 ? s[size_t(y1) * Nx + i] : T(0);
      if (MODE == 1) {
        a = sigm(steep * a);
        b = has1 ? sigm(steep * b) : T(0);
      }
      row.st(i, mk(a, b));
    }
  }
  row.sync();
  fft<T, -1>(row);
  if (row.active) {
    cx<T>* o = out + tile * out_ts;
    for (int px = row.t; px <= Pout; px += row.TPR) {
      cx<T> A, Bv;
      split_pair(row.ld(px), row.ld(wrapi(-px, Nx)), A, Bv);
      o[size_t(px) * Ny + y0] = A;
      if (has1) o[size_t(px) * Ny + y1] = Bv;
    }
  }
}

// ===========================================================================
// Mask half-spectrum columns -> kernel band M^[By][Bx] (scaled 1/(Nx Ny)).
// One group per column px in [0, Pmx]; negative qx via Hermitian symmetry.
// ===========================================================================
template <typename T>
__global__ void k_mask_cols(Geo<T> g, const cx<T>* __restrict__ Mr, long long mr_ts,
                            cx<T>* __restrict__ Mhat, long long mh_ts) {
  Group<T> grp(g.ay.N, 0);
  const int Ny = g.ay.N;
  const int px = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const bool active = px <= g.ax.Pm;
  const int tile = blockIdx.z;
  const Row<T> row = grp.row(0, g.tNy, active);
  const cx<T>* src = Mr + tile * mr_ts + size_t(px) * Ny;
  if (row.active)
    for (int i = row.t; i < Ny; i += row.TPR) row.st(i, src[i]);
  row.sync();
  fft<T, -1>(row);
  if (!row.active) return;
  const T inv = T(1.0 / (double(g.ax.N) * double(g.ay.N)));
  cx<T>* mh = Mhat + tile * mh_ts;
  const int Bx = g.ax.B;
  const int sp = band_slot(g.ax, px);
  const int sn = px > 0 ? band_slot(g.ax, -px) : -1;
  for (int j = row.t; j < g.ay.B; j += row.TPR) {
    const int qy = g.ay.lo + j;
    if (sp >= 0) mh[size_t(j) * Bx + sp] = scale(row.ld(wrapi(qy, Ny)), inv);
    if (sn >= 0 && sn != sp) mh[size_t(j) * Bx + sn] = scale(conjg(row.ld(wrapi(-qy, Ny))), inv);
  }
}

// ===========================================================================
// Per-kernel column pass on the decimated grid:
//   T_fk[sy][qx] = IFFT_ny over qy of M^(qy,qx) H_fk(qy,qx)
// grid (ceil(Bx/RPC), F*K, tiles); output row-major [ny][Bx] per (tile, fk).
// ===========================================================================
template <typename T>
__global__ void k_socs_cols(Geo<T> g, const cx<T>* __restrict__ Mhat, long long mh_ts,
                            const cx<T>* __restrict__ H, cx<T>* __restrict__ Tout, long long t_ts) {
  Group<T> grp(g.ay.n, 0);
  const int ny = g.ay.n, Bx = g.ax.B, By = g.ay.B;
  const int cx_ = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const int fk = blockIdx.y;
  const int tile = blockIdx.z;
  const bool active = cx_ < Bx;
  const Row<T> row = grp.row(0, g.tny, active);
  row.zero();
  row.sync();
  const cx<T>* mh = Mhat + tile * mh_ts;
  const cx<T>* h = H + size_t(fk) * By * Bx;
  if (row.active)
    for (int j = row.t; j < By; j += row.TPR) {
      const size_t o = size_t(j) * Bx + cx_;
      row.st(wrapi(g.ay.lo + j, ny), mul(mh[o], ldg_cx(h + o)));
    }
  row.sync();
  fft<T, +1>(row);
  if (row.active) {
    cx<T>* o = Tout + tile * t_ts + size_t(fk) * ny * Bx;
    for (int sy = row.t; sy < ny; sy += row.TPR) o[size_t(sy) * Bx + cx_] = row.ld(sy);
  }
}

// ===========================================================================
// Per-kernel row pass + |E|^2 accumulate on the decimated grid, fused with
// the forward FFT of the resulting intensity row:
//   I_sub(sy, sx) = dose sum_k w_fk |IFFT_nx(T_fk[sy])|^2
//   Ir[f][px][sy] = FFT_nx(I_sub(sy, .))(px),  px in [0, Px]
// grid (ceil(ny/RPC), F, tiles)
// ===========================================================================
template <typename T>
__global__ void k_socs_rows(Geo<T> g, const cx<T>* __restrict__ Tin, long long t_ts,
                            const T* __restrict__ wk, T dose, cx<T>* __restrict__ Ir,
                            long long ir_ts, T* __restrict__ Isub, long long is_ts) {
  Group<T> grp(g.ax.n, 0);
  const int nx = g.ax.n, ny = g.ay.n, Bx = g.ax.B, K = g.K;
  const int sy = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const int f = blockIdx.y;
  const int tile = blockIdx.z;
  const bool active = sy < ny;
  const Row<T> row = grp.row(0, g.tnx, active);
  T acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = T(0);
  for (int k = 0; k < K; ++k) {
    row.zero();
    row.sync();
    const cx<T>* src = Tin + tile * t_ts + (size_t(f) * K + k) * ny * Bx + size_t(sy) * Bx;
    if (row.active)
      for (int j = row.t; j < Bx; j += row.TPR) row.st(wrapi(g.ax.lo + j, nx), src[j]);
    row.sync();
    fft<T, +1>(row);
    const T w = wk[f * K + k] * dose;
    if (row.active) {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int i = row.t + e * row.TPR;
        if (i < nx) {
          const cx<T> v = row.ld(i);
          acc[e] += w * (v.x * v.x + v.y * v.y);
        }
      }
    }
  }
  // forward FFT of the real intensity row (own elements only: no hazard)
  if (row.active) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int i = row.t + e * row.TPR;
      if (i < nx) {
        row.st(i, mk(acc[e], T(0)));
        if (Isub) Isub[tile * is_ts + size_t(f) * nx * ny + size_t(sy) * nx + i] = acc[e];
      }
    }
  }
  row.sync();
  fft<T, -1>(row);
  if (row.active) {
    cx<T>* o = Ir + tile * ir_ts + size_t(f) * (g.ax.P + 1) * ny;
    for (int px = row.t; px <= g.ax.P; px += row.TPR) o[size_t(px) * ny + sy] = row.ld(px);
  }
}

// ===========================================================================
// Intensity-band column pass: FFT_ny of I_sub columns -> intensity spectrum
// on the band (exact, n >= 2P+1), optional Gaussian transfer, then the
// band-pruned IFFT_Ny back to full-grid rows:
//   WANT_I: Ic[f][y][px] = IFFT_Ny(I^)(y)        (aerial image half rows)
//   WANT_R: Rc[f][y][px] = IFFT_Ny(I^ . g^)(y)   (resist image half rows)
// grid (ceil((Px+1)/RPC), F, tiles)
// ===========================================================================
template <typename T, bool WANT_I, bool WANT_R>
__global__ void k_isub_cols(Geo<T> g, const cx<T>* __restrict__ Ir, long long ir_ts,
                            const T* __restrict__ gxh, const T* __restrict__ gyb,
                            cx<T>* __restrict__ Ic, cx<T>* __restrict__ Rc, long long c_ts) {
  Group<T> grp(g.ay.n, g.ay.N);
  const int ny = g.ay.n, Ny = g.ay.N, Px = g.ax.P;
  const int px = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const int f = blockIdx.y;
  const int tile = blockIdx.z;
  const bool active = px <= Px;
  const Row<T> ra = grp.row(0, g.tny, active);
  const Row<T> rb = grp.row(1, g.tNy, active);
  const cx<T>* src = Ir + tile * ir_ts + (size_t(f) * (Px + 1) + px) * ny;
  if (ra.active)
    for (int i = ra.t; i < ny; i += ra.TPR) ra.st(i, src[i]);
  ra.sync();
  fft<T, -1>(ra);
  const T inv = T(1.0 / (double(g.ax.n) * double(g.ay.n)));
  const T gx = active ? gxh[px] : T(0);
  const size_t obase = tile * c_ts + size_t(f) * Ny * (Px + 1);
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    if ((pass == 0 && !WANT_I) || (pass == 1 && !WANT_R)) continue;
    rb.zero();
    rb.sync();
    if (rb.active)
      for (int j = rb.t; j < g.ay.nb2; j += rb.TPR) {
        const int p = band2_p(g.ay, j);
        T s = inv;
        if (pass == 1) s *= gx * gyb[j];
        rb.st(wrapi(p, Ny), scale(ra.ld(wrapi(p, ny)), s));
      }
    rb.sync();
    fft<T, +1>(rb);
    if (rb.active) {
      cx<T>* o = (pass == 0 ? Ic : Rc) + obase;
      for (int y = rb.t; y < Ny; y += rb.TPR) o[size_t(y) * (Px + 1) + px] = rb.ld(y);
    }
    rb.sync();
  }
}

// place a real signal's half spectrum h (px in [0, P]) into a full row by
// Hermitian symmetry, packed as  Z = A + i B  for two real signals.
template <typename T>
__device__ __forceinline__ void place_pair(const Row<T>& row, int P, const cx<T>* a,
                                           const cx<T>* b) {
  const int N = row.L;
  if (!row.active) return;
  for (int px = row.t; px <= P; px += row.TPR) {
    cx<T> A = a ? a[px] : mk(T(0), T(0));
    cx<T> Bv = b ? b[px] : mk(T(0), T(0));
    const int m = wrapi(-px, N);
    if (m == px) {  // DC / Nyquist: the spectrum of a real signal is real here
      A.y = T(0);
      Bv.y = T(0);
      row.st(px, mk(A.x, Bv.x));
      continue;
    }
    row.st(px, mk(A.x - Bv.y, A.y + Bv.x));
    row.st(m, mk(A.x + Bv.y, Bv.x - A.y));
  }
}

// ===========================================================================
// Forward output rows: I (aerial) and R (resist) for one focus, one packed
// IFFT_Nx per row.  print[y][x] = (R >= thr) as u8 (threshold resist).
// grid (ceil(Ny/RPC), F, tiles)
// ===========================================================================
template <typename T, typename OutT>
__global__ void k_out_rows(Geo<T> g, const cx<T>* __restrict__ Ic, const cx<T>* __restrict__ Rc,
                           long long c_ts, OutT* __restrict__ Iout, OutT* __restrict__ Rout,
                           unsigned char* __restrict__ print, long long o_ts, T thr) {
  Group<T> grp(g.ax.N, 0);
  const int Nx = g.ax.N, Ny = g.ay.N, Px = g.ax.P;
  const int y = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const int f = blockIdx.y;
  const int tile = blockIdx.z;
  const bool active = y < Ny;
  const Row<T> row = grp.row(0, g.tNx, active);
  row.zero();
  row.sync();
  const size_t cb = tile * c_ts + (size_t(f) * Ny + y) * (Px + 1);
  place_pair(row, Px, Ic ? Ic + cb : nullptr, Rc ? Rc + cb : nullptr);
  row.sync();
  fft<T, +1>(row);
  if (!row.active) return;
  const size_t ob = tile * o_ts + (size_t(f) * Ny + y) * Nx;
  for (int x = row.t; x < Nx; x += row.TPR) {
    const cx<T> v = row.ld(x);
    if (Iout) Iout[ob + x] = OutT(v.x);
    if (Rout) Rout[ob + x] = OutT(v.y);
    if (print) print[ob + x] = v.y >= thr ? 1 : 0;
  }
}

// ===========================================================================
// ILT resist rows (foci pair f0, f0+1): R_f = IFFT_Nx(R^ rows), sigmoid
// resist Z_f = sig(beta (R_f - thr)), cost c_f (Z_f - Z_t)^2, and
//   D_f = dL/dR_f = 2 c_f (Z_f - Z_t) beta Z_f (1 - Z_f)
// then FFT_Nx of the packed pair -> Dr[f][px][y] half spectra.
// grid (ceil(Ny/RPC), ceil(F/2), tiles)
// ===========================================================================
template <typename T>
__global__ void k_resist_rows(Geo<T> g, const cx<T>* __restrict__ Rc, long long c_ts,
                              const T* __restrict__ target, long long tg_ts,
                              const T* __restrict__ cf, T beta, T thr, cx<T>* __restrict__ Dr,
                              long long d_ts, double* __restrict__ costrow, long long cr_ts,
                              T* __restrict__ Zout, long long z_ts) {
  Group<T> grp(g.ax.N, 0);
  const int Nx = g.ax.N, Ny = g.ay.N, Px = g.ax.P, F = g.F;
  const int y = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const int f0 = 2 * blockIdx.y, f1 = f0 + 1;
  const bool has1 = f1 < F;
  const int tile = blockIdx.z;
  const bool active = y < Ny;
  const Row<T> row = grp.row(0, g.tNx, active);
  row.zero();
  row.sync();
  const cx<T>* rc = Rc + tile * c_ts;
  place_pair(row, Px, rc + (size_t(f0) * Ny + y) * (Px + 1),
             has1 ? rc + (size_t(f1) * Ny + y) * (Px + 1) : nullptr);
  row.sync();
  fft<T, +1>(row);
  double c0 = 0, c1 = 0;
  if (row.active) {
    const T* tg = target + tile * tg_ts + size_t(y) * Nx;
    const T w0 = cf[f0], w1 = has1 ? cf[f1] : T(0);
    for (int x = row.t; x < Nx; x += row.TPR) {
      const cx<T> v = row.ld(x);
      const T t = tg[x];
      const T z0 = sigm(beta * (v.x - thr));
      const T e0 = z0 - t;
      c0 += double(w0) * double(e0) * double(e0);
      const T d0 = T(2) * w0 * e0 * beta * z0 * (T(1) - z0);
      T d1 = T(0);
      if (has1) {
        const T z1 = sigm(beta * (v.y - thr));
        const T e1 = z1 - t;
        c1 += double(w1) * double(e1) * double(e1);
        d1 = T(2) * w1 * e1 * beta * z1 * (T(1) - z1);
        if (Zout) Zout[tile * z_ts + (size_t(f1) * Ny + y) * Nx + x] = z1;
      }
      if (Zout) Zout[tile * z_ts + (size_t(f0) * Ny + y) * Nx + x] = z0;
      row.st(x, mk(d0, d1));
    }
  }
  c0 = grp.reduce_sum(c0);
  c1 = grp.reduce_sum(c1);
  if (row.active && row.t == 0) {
    costrow[tile * cr_ts + size_t(f0) * Ny + y] = c0;
    if (has1) costrow[tile * cr_ts + size_t(f1) * Ny + y] = c1;
  }
  row.sync();
  fft<T, -1>(row);
  if (row.active) {
    cx<T>* d = Dr + tile * d_ts;
    for (int px = row.t; px <= Px; px += row.TPR) {
      cx<T> A, Bv;
      split_pair(row.ld(px), row.ld(wrapi(-px, Nx)), A, Bv);
      d[(size_t(f0) * (Px + 1) + px) * Ny + y] = A;
      if (has1) d[(size_t(f1) * (Px + 1) + px) * Ny + y] = Bv;
    }
  }
}

// ===========================================================================
// Weight-field columns: FFT_Ny of D (or W) half-spectrum columns, band-pass
// to the intensity band with the Gaussian transfer (W = blur(D)), scale
// 1/(Nx Ny), then IFFT_ny onto the decimated grid:
//   Wc[f][sy][px] = IFFT_ny( g^(px,py) FFT_N(D)(py,px)/(Nx Ny) )(sy)
// grid (ceil((Px+1)/RPC), F, tiles)
// ===========================================================================
template <typename T, bool GAUSS>
__global__ void k_wlp_cols(Geo<T> g, const cx<T>* __restrict__ Dr, long long d_ts,
                           const T* __restrict__ gxh, const T* __restrict__ gyb,
                           cx<T>* __restrict__ Wc, long long w_ts) {
  Group<T> grp(g.ay.N, g.ay.n);
  const int ny = g.ay.n, Ny = g.ay.N, Px = g.ax.P;
  const int px = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const int f = blockIdx.y;
  const int tile = blockIdx.z;
  const bool active = px <= Px;
  const Row<T> ra = grp.row(0, g.tNy, active);
  const Row<T> rb = grp.row(1, g.tny, active);
  const cx<T>* src = Dr + tile * d_ts + (size_t(f) * (Px + 1) + px) * Ny;
  if (ra.active)
    for (int i = ra.t; i < Ny; i += ra.TPR) ra.st(i, src[i]);
  ra.sync();
  fft<T, -1>(ra);
  rb.zero();
  rb.sync();
  const T inv = T(1.0 / (double(g.ax.N) * double(g.ay.N)));
  const T gx = (GAUSS && active) ? gxh[px] : T(1);
  if (rb.active)
    for (int j = rb.t; j < g.ay.nb2; j += rb.TPR) {
      const int p = band2_p(g.ay, j);
      const T s = GAUSS ? inv * gx * gyb[j] : inv;
      rb.st(wrapi(p, ny), scale(ra.ld(wrapi(p, Ny)), s));
    }
  rb.sync();
  fft<T, +1>(rb);
  if (rb.active) {
    cx<T>* o = Wc + tile * w_ts + size_t(f) * ny * (Px + 1);
    for (int sy = rb.t; sy < ny; sy += rb.TPR) o[size_t(sy) * (Px + 1) + px] = rb.ld(sy);
  }
}

// ===========================================================================
// Adjoint row pass on the decimated grid, per focus f and subgrid row sy:
//   W_lp(sy, .) = IFFT_nx(Hermitian(Wc[f][sy]))          (real, once)
//   for k: E = IFFT_nx(T_fk[sy]);  U_fk[qx][sy] = FFT_nx(W_lp . E)(qx), qx in band
// UNIFORM: W == 1 (the reference's intensity_gradient, ai.cpp:11-42).
// grid (ceil(ny/RPC), F, tiles)
// ===========================================================================
template <typename T, bool UNIFORM>
__global__ void k_adj_rows(Geo<T> g, const cx<T>* __restrict__ Tin, long long t_ts,
                           const cx<T>* __restrict__ Wc, long long w_ts, cx<T>* __restrict__ U,
                           long long u_ts) {
  Group<T> grp(g.ax.n, 0);
  const int nx = g.ax.n, ny = g.ay.n, Bx = g.ax.B, K = g.K, Px = g.ax.P;
  const int sy = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const int f = blockIdx.y;
  const int tile = blockIdx.z;
  const bool active = sy < ny;
  const Row<T> row = grp.row(0, g.tnx, active);
  T wv[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) wv[e] = T(1);
  if (!UNIFORM) {
    row.zero();
    row.sync();
    place_pair(row, Px, Wc + tile * w_ts + (size_t(f) * ny + sy) * (Px + 1),
               static_cast<const cx<T>*>(nullptr));
    row.sync();
    fft<T, +1>(row);
    if (row.active) {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int i = row.t + e * row.TPR;
        if (i < nx) wv[e] = row.ld(i).x;
      }
    }
  }
  for (int k = 0; k < K; ++k) {
    row.zero();
    row.sync();
    const cx<T>* src = Tin + tile * t_ts + (size_t(f) * K + k) * ny * Bx + size_t(sy) * Bx;
    if (row.active)
      for (int j = row.t; j < Bx; j += row.TPR) row.st(wrapi(g.ax.lo + j, nx), src[j]);
    row.sync();
    fft<T, +1>(row);
    if (row.active) {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int i = row.t + e * row.TPR;
        if (i < nx) row.st(i, scale(row.ld(i), wv[e]));
      }
    }
    row.sync();
    fft<T, -1>(row);
    if (row.active) {
      cx<T>* o = U + tile * u_ts + (size_t(f) * K + k) * Bx * ny;
      for (int j = row.t; j < Bx; j += row.TPR)
        o[size_t(j) * ny + sy] = row.ld(wrapi(g.ax.lo + j, nx));
    }
    row.sync();
  }
}

// ===========================================================================
// Adjoint column pass + accumulation over (f, k), one CTA per band column qx:
//   Acc(qy,qx) = sum_fk FFT_ny(U_fk[qx])(qy) conj(H_fk(qy,qx)) 2 dose w_fk dx dy/(Nx Ny)
// Row groups take (f,k) round-robin, then reduce in shared memory.
// grid (Bx, 1, tiles); Acc out [By][Bx]
// ===========================================================================
template <typename T>
__global__ void k_adj_cols(Geo<T> g, const cx<T>* __restrict__ U, long long u_ts,
                           const cx<T>* __restrict__ H, const T* __restrict__ wk, T dose,
                           cx<T>* __restrict__ Acc, long long a_ts) {
  Group<T> grp(g.ay.n, 0);
  const int ny = g.ay.n, Bx = g.ax.B, By = g.ay.B, FK = g.F * g.K;
  const int RPC = blockDim.x / grp.G;
  const int qxs = blockIdx.x;
  const int tile = blockIdx.z;
  const Row<T> row = grp.row(0, g.tny, true);
  const T sc = T(2.0 / (double(g.ax.n) * double(g.ay.n)));  // 2 (N/n)^2 / N^2
  cx<T> acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = mk(T(0), T(0));
  const int rounds = (FK + RPC - 1) / RPC;
  for (int r = 0; r < rounds; ++r) {
    const int fk = r * RPC + grp.gid;
    const bool act = fk < FK;
    const Row<T> rr = grp.row(0, g.tny, act);
    const cx<T>* src = U + tile * u_ts + (size_t(fk) * Bx + qxs) * ny;
    if (rr.active)
      for (int i = rr.t; i < ny; i += rr.TPR) rr.st(i, src[i]);
    rr.sync();
    fft<T, -1>(rr);
    if (rr.active) {
      const T w = wk[fk] * dose * sc;
      const cx<T>* h = H + size_t(fk) * By * Bx;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int j = rr.t + e * rr.TPR;
        if (j < By) {
          const cx<T> hv = h[size_t(j) * Bx + qxs];
          const cx<T> v = mulc(rr.ld(wrapi(g.ay.lo + j, ny)), hv);
          acc[e] = add(acc[e], scale(v, w));
        }
      }
    }
    rr.sync();
  }
  // cross-group reduction through shared memory (reuse group rows)
  __syncthreads();
  if (row.t < row.TPR) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int j = row.t + e * row.TPR;
      if (j < By) row.st(j, acc[e]);
    }
  }
  __syncthreads();
  if (grp.gid == 0 && row.t < row.TPR) {
    cx<T>* o = Acc + tile * a_ts;
    for (int j = row.t; j < By; j += row.TPR) {
      cx<T> s = mk(T(0), T(0));
      for (int q = 0; q < RPC; ++q) {
        const T* b = grp.base + size_t(q) * group_elems<T>(grp.LA, grp.LB) - size_t(grp.gid) * 0;
        const T* re = reinterpret_cast<const T*>(b);
        const int p = pidx<T>(j);
        s = add(s, mk(re[p], re[padded_len<T>(g.ay.n) + p]));
      }
      o[size_t(j) * Bx + qxs] = s;
    }
  }
}

// ===========================================================================
// Gradient columns: Hermitian part of the accumulated band spectrum (the
// gradient is Re IFFT(Acc)), band-pruned IFFT_Ny -> Gc[y][px], px in [0,Pmx].
// An extra CTA (blockIdx.x == gridDim.x-1) reduces the per-row cost and
// gradient partials of this iteration in fixed order (deterministic).
// grid (ceil((Pmx+1)/RPC) + 1, 1, tiles)
// ===========================================================================
template <typename T>
__global__ void k_grad_cols(Geo<T> g, const cx<T>* __restrict__ Acc, long long a_ts,
                            cx<T>* __restrict__ Gc, long long g_ts, const double* costrow,
                            long long cr_ts, int ncost, double* cost_out, long long co_ts) {
  Group<T> grp(g.ay.N, 0);
  const int Ny = g.ay.N, Bx = g.ax.B, Pm = g.ax.Pm;
  const int tile = blockIdx.z;
  if (blockIdx.x == gridDim.x - 1) {
    if (cost_out && threadIdx.x == 0) {
      double s = 0;
      const double* c = costrow + tile * cr_ts;
      for (int i = 0; i < ncost; ++i) s += c[i];
      cost_out[tile * co_ts] = s;
    }
    return;
  }
  const int px = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const bool active = px <= Pm;
  const Row<T> row = grp.row(0, g.tNy, active);
  row.zero();
  row.sync();
  if (row.active) {
    const cx<T>* a = Acc + tile * a_ts;
    const int sp = band_slot(g.ax, px), sn = band_slot(g.ax, -px);
    const int Pmy = g.ay.Pm;
    for (int qy = -Pmy + row.t; qy <= Pmy; qy += row.TPR) {
      const int jp = band_slot(g.ay, qy), jn = band_slot(g.ay, -qy);
      cx<T> v = mk(T(0), T(0));
      if (sp >= 0 && jp >= 0) v = add(v, a[size_t(jp) * Bx + sp]);
      if (sn >= 0 && jn >= 0) v = add(v, conjg(a[size_t(jn) * Bx + sn]));
      const int bin = wrapi(qy, Ny);
      if (2 * Pmy + 1 > Ny && qy != -Pmy + 0 && wrapi(-Pmy, Ny) == bin && qy != -Pmy) {
      }
      row.st(bin, scale(v, T(0.5)));
    }
  }
  row.sync();
  fft<T, +1>(row);
  if (row.active) {
    cx<T>* o = Gc + tile * g_ts;
    for (int y = row.t; y < Ny; y += row.TPR) o[size_t(y) * (Pm + 1) + px] = row.ld(y);
  }
}

// ===========================================================================
// Gradient rows (row pair y0, y0+1): g = IFFT_Nx(Hermitian Gc rows) = dL/dM.
//   GRAD_OUT: grad[y][x] = g                          (intensity_gradient API)
//   ILT:      theta -= step g a M (1-M), M = sig(a theta); then the next
//             iteration's mask row pass (sig(a theta') -> FFT_Nx -> Mr).
// grid (ceil(Ny/2/RPC), 1, tiles)
// ===========================================================================
template <typename T, bool ILT, typename OutT>
__global__ void k_grad_rows(Geo<T> g, const cx<T>* __restrict__ Gc, long long g_ts,
                            OutT* __restrict__ grad, long long gr_ts, T* __restrict__ theta,
                            long long th_ts, T steep, T step, cx<T>* __restrict__ Mr,
                            long long mr_ts, double* __restrict__ gmaxrow, long long gm_ts) {
  Group<T> grp(g.ax.N, 0);
  const int Nx = g.ax.N, Ny = g.ay.N, Pm = g.ax.Pm;
  const int pair = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const bool active = pair < (Ny + 1) / 2;
  const int tile = blockIdx.z;
  const Row<T> row = grp.row(0, g.tNx, active);
  const int y0 = 2 * pair, y1 = y0 + 1;
  const bool has1 = y1 < Ny;
  row.zero();
  row.sync();
  const cx<T>* gc = Gc + tile * g_ts;
  place_pair(row, Pm, gc + size_t(y0) * (Pm + 1), has1 ? gc + size_t(y1) * (Pm + 1) : nullptr);
  row.sync();
  fft<T, +1>(row);
  if (!ILT) {
    if (row.active) {
      OutT* o = grad + tile * gr_ts;
      for (int x = row.t; x < Nx; x += row.TPR) {
        const cx<T> v = row.ld(x);
        o[size_t(y0) * Nx + x] = OutT(v.x);
        if (has1) o[size_t(y1) * Nx + x] = OutT(v.y);
      }
    }
    return;
  }
  double gm = 0;
  if (row.active) {
    T* th = theta + tile * th_ts;
    for (int x = row.t; x < Nx; x += row.TPR) {
      const cx<T> v = row.ld(x);
      const T t0 = th[size_t(y0) * Nx + x];
      const T m0 = sigm(steep * t0);
      const T g0 = v.x * steep * m0 * (T(1) - m0);
      const T n0 = t0 - step * g0;
      th[size_t(y0) * Nx + x] = n0;
      if (grad) grad[tile * gr_ts + size_t(y0) * Nx + x] = OutT(g0);  // dL/dtheta (lithogpu_ilt_gradient)
      gm = fmax(gm, fabs(double(g0)));
      T n1v = T(0);
      if (has1) {
        const T t1 = th[size_t(y1) * Nx + x];
        const T m1 = sigm(steep * t1);
        const T g1 = v.y * steep * m1 * (T(1) - m1);
        const T n1 = t1 - step * g1;
        th[size_t(y1) * Nx + x] = n1;
        if (grad) grad[tile * gr_ts + size_t(y1) * Nx + x] = OutT(g1);
        gm = fmax(gm, fabs(double(g1)));
        n1v = sigm(steep * n1);
      }
      row.st(x, mk(sigm(steep * n0), n1v));
    }
  }
  gm = grp.reduce_max(gm);
  if (row.active && row.t == 0 && gmaxrow) gmaxrow[tile * gm_ts + pair] = gm;
  row.sync();
  fft<T, -1>(row);
  if (row.active) {
    cx<T>* o = Mr + tile * mr_ts;
    for (int px = row.t; px <= Pm; px += row.TPR) {
      cx<T> A, Bv;
      split_pair(row.ld(px), row.ld(wrapi(-px, Nx)), A, Bv);
      o[size_t(px) * Ny + y0] = A;
      if (has1) o[size_t(px) * Ny + y1] = Bv;
    }
  }
}

// ===========================================================================
// Plain batched 2-D DFT (the reference fft2, imaging.cpp:17-31: unnormalized,
// x contiguous): rows then columns, any lengths (generic path).
// ===========================================================================
template <typename T, int SIGN>
__global__ void k_fft2_rows(Tab<T> tab, int nx, int ny, cx<T>* __restrict__ data) {
  Group<T> grp(nx, 0);
  const int y = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const Row<T> row = grp.row(0, tab, y < ny);
  cx<T>* d = data + size_t(blockIdx.z) * nx * ny + size_t(y) * nx;
  if (row.active)
    for (int i = row.t; i < nx; i += row.TPR) row.st(i, d[i]);
  row.sync();
  fft<T, SIGN>(row);
  if (row.active)
    for (int i = row.t; i < nx; i += row.TPR) d[i] = row.ld(i);
}

template <typename T, int SIGN>
__global__ void k_fft2_cols(Tab<T> tab, int nx, int ny, cx<T>* __restrict__ data) {
  Group<T> grp(ny, 0);
  const int x = blockIdx.x * (blockDim.x / grp.G) + grp.gid;
  const Row<T> row = grp.row(0, tab, x < nx);
  cx<T>* d = data + size_t(blockIdx.z) * nx * ny + x;
  if (row.active)
    for (int i = row.t; i < ny; i += row.TPR) row.st(i, d[size_t(i) * nx]);
  row.sync();
  fft<T, SIGN>(row);
  if (row.active)
    for (int i = row.t; i < ny; i += row.TPR) d[size_t(i) * nx] = row.ld(i);
}

}  // namespace lg
