// Device-side FFT building blocks for the SOCS imaging / ILT kernels (sm_100a).
//
// One "row group" of TPR threads transforms one length-L complex row held in
// shared memory (split re/im arrays, one pad word per 128 B so the strided
// Stockham stores stay bank-conflict free).  Every length is O(L log L):
//   * power-of-two L >= 16: Stockham autosort FFT with radix-16 register
//     butterflies (16 values per thread, TPR = L/16, final radix 8/4/2 stage);
//   * L whose prime factors are all <= 7 (12, 24, 49 = 7*7; not 74 = 2*37 or
//     987 = 3*7*47): mixed-radix Stockham (radices 4, 2, 3, 5, 7),
//     ping-ponging between the row and the group scratch;
//   * any other L (a make_window size like 1234 = 2*617, opc.cpp:108-109):
//     Bluestein's chirp-z, X_k = w_k sum_n (x_n w_n) conj(w_{k-n}),
//     w_n = exp(-i pi n^2 / L), as a cyclic convolution of length
//     M = 2^ceil(log2(2L-1)) on the power-of-two path, with the chirp and the
//     chirp filter's spectrum precomputed in fp64 (n^2 reduced mod 2L exactly).
// The reference's FFTW (imaging.cpp:17-31) is O(L log L) at every size; so is
// this.
//
// Conventions are the reference fft2 (proj/src/core/imaging.cpp:17-31):
// SIGN = -1 forward exp(-2 pi i k x / L), SIGN = +1 backward, unnormalized.
// Twiddle tables hold exp(-2 pi i m / L), m < L, rounded once from fp64.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lg {

template <typename T>
struct alignas(2 * sizeof(T)) cx {
  T x, y;
};

template <typename T>
__device__ __forceinline__ cx<T> mk(T a, T b) {
  cx<T> r;
  r.x = a;
  r.y = b;
  return r;
}
template <typename T>
__device__ __forceinline__ cx<T> add(cx<T> a, cx<T> b) {
  return mk(a.x + b.x, a.y + b.y);
}
template <typename T>
__device__ __forceinline__ cx<T> sub(cx<T> a, cx<T> b) {
  return mk(a.x - b.x, a.y - b.y);
}
template <typename T>
__device__ __forceinline__ cx<T> mul(cx<T> a, cx<T> b) {
  return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename T>
__device__ __forceinline__ cx<T> mulc(cx<T> a, cx<T> b) {
  return mk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename T>
__device__ __forceinline__ cx<T> conjg(cx<T> a) {
  return mk(a.x, -a.y);
}
template <typename T>
__device__ __forceinline__ cx<T> scale(cx<T> a, T s) {
  return mk(a.x * s, a.y * s);
}
// read-only cached load of a complex value
__device__ __forceinline__ cx<float> ldg_cx(const cx<float>* p) {
  const float2 v = __ldg(reinterpret_cast<const float2*>(p));
  return mk(v.x, v.y);
}
__device__ __forceinline__ cx<double> ldg_cx(const cx<double>* p) {
  const double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return mk(v.x, v.y);
}

// Hermitian split of a packed real pair: Z = FFT(a + i b) ->
//   A(p) = (Z(p) + conj Z(-p))/2,  B(p) = (Z(p) - conj Z(-p))/(2i)
template <typename T>
__device__ __forceinline__ void split_pair(cx<T> X, cx<T> Ym, cx<T>& A, cx<T>& Bv) {
  const cx<T> Yc = conjg(Ym);
  A = scale(add(X, Yc), T(0.5));
  const cx<T> D = sub(X, Yc);
  Bv = mk(T(0.5) * D.y, T(-0.5) * D.x);
}

// a * (S * i)
template <int S, typename T>
__device__ __forceinline__ cx<T> mul_si(cx<T> a) {
  return S < 0 ? mk(a.y, -a.x) : mk(-a.y, a.x);
}

// ---- shared-memory row layout -------------------------------------------
template <typename T>
__host__ __device__ constexpr int pad_shift() {
  return sizeof(T) == 4 ? 5 : 4;  // one pad element per 128 bytes
}
template <typename T>
__host__ __device__ __forceinline__ int pidx(int i) {
  return i + (i >> pad_shift<T>());
}
template <typename T>
__host__ __device__ constexpr int padded_len(int L) {
  return L + (L >> pad_shift<T>()) + 1;
}

__host__ __device__ inline bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
__host__ __device__ inline int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}
__host__ __device__ inline int next_pow2(int n) { return 1 << ilog2(n); }
// threads per row group for a length-L transform
__host__ __device__ inline int tpr_for(int L) {
  const int t = next_pow2(L) / 16;
  return t < 1 ? 1 : t;
}

// transform kinds of the generic path (see the header comment)
enum FftKind { kFftPow2 = 0, kFftMixed = 1, kFftBluestein = 2 };
constexpr int kMaxMixedRadix = 7;
__host__ __device__ inline int fft_kind(int L) {
  if (is_pow2(L) && L >= 16) return kFftPow2;
  int r = L;
  for (int p = 2; p <= kMaxMixedRadix; ++p)
    while (r % p == 0) r /= p;
  return r == 1 ? kFftMixed : kFftBluestein;
}
// Bluestein convolution length (0 when L does not use Bluestein)
__host__ __device__ inline int blue_len(int L) {
  if (fft_kind(L) != kFftBluestein) return 0;
  const int m = next_pow2(2 * L - 1);
  return m < 16 ? 16 : m;
}
// threads a row group needs for a length-L transform
__host__ __device__ inline int fft_tpr(int L) { return tpr_for(fft_kind(L) == kFftBluestein ? blue_len(L) : L); }
// mixed-radix plan: radices (4 first, then 2, 3, 5, 7) as 4-bit nibbles
__host__ __device__ inline unsigned long long mixed_radices(int L, int& nst) {
  unsigned long long code = 0;
  nst = 0;
  int r = L;
  auto push = [&](int R) {
    code |= (unsigned long long)R << (4 * nst);
    ++nst;
    r /= R;
  };
  while (r % 4 == 0) push(4);
  while (r % 2 == 0) push(2);
  for (int p = 3; p <= kMaxMixedRadix; p += 2)
    while (r % p == 0) push(p);
  return code;
}

// lengths of the compile-time-planned fp32 fast path (fftr.cuh), ascending
constexpr int kFastLens[] = {32, 64, 128, 192, 256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096, 8192};

// Row-group context: one length-L row in smem, processed by TPR threads.
template <typename T>
struct Row {
  T* re;
  T* im;
  T* sre;  // scratch (generic DFT only), length L unpadded
  T* sim;
  int L;
  int log2L;  // >= 4 iff power-of-two path
  int kind;   // FftKind
  unsigned long long rad;  // mixed radix: radices as 4-bit nibbles, stage 0 lowest
  int nst;                 // mixed radix: number of stages
  // Bluestein: padded work row of length M (power of two) and its tables
  T* bre;
  T* bim;
  int M, log2M;
  const cx<T>* twM;    // exp(-2 pi i m / M)
  const cx<T>* chirp;  // w_n = exp(-i pi n^2 / L), n < L
  const cx<T>* bhat;   // FFT_M(conj w wrapped), k < M
  int t;      // thread index in group
  int TPR;
  bool cta_sync;  // TPR > 32 -> group spans warps
  bool active;
  const cx<T>* tw;  // exp(-2 pi i m / L)

  __device__ __forceinline__ void sync() const {
    if (cta_sync)
      __syncthreads();
    else
      __syncwarp();
  }
  __device__ __forceinline__ cx<T> ld(int i) const {
    const int p = pidx<T>(i);
    return mk(re[p], im[p]);
  }
  __device__ __forceinline__ void st(int i, cx<T> v) const {
    const int p = pidx<T>(i);
    re[p] = v.x;
    im[p] = v.y;
  }
  __device__ __forceinline__ void zero() const {
    if (!active) return;
    for (int i = t; i < L; i += TPR) st(i, mk(T(0), T(0)));
  }
};

// ---- radix-R DFT on registers, natural-order in and out -----------------
template <int S, typename T>
__device__ __forceinline__ void dft2(cx<T>& a, cx<T>& b) {
  const cx<T> t = a;
  a = add(t, b);
  b = sub(t, b);
}

template <int S, typename T>
__device__ __forceinline__ void dft4(cx<T>& v0, cx<T>& v1, cx<T>& v2, cx<T>& v3) {
  const cx<T> t0 = add(v0, v2), t1 = sub(v0, v2), t2 = add(v1, v3);
  const cx<T> t3 = mul_si<S>(sub(v1, v3));
  v0 = add(t0, t2);
  v2 = sub(t0, t2);
  v1 = add(t1, t3);
  v3 = sub(t1, t3);
}

// multiply by W_R^q = exp(S 2 pi i q / R) for R = 8, 16 with cheap special cases
template <int R, int Q, int S, typename T>
__device__ __forceinline__ cx<T> twc(cx<T> a) {
  constexpr int q = Q % R;
  if constexpr (q == 0) {
    return a;
  } else if constexpr (4 * q == R) {
    return mul_si<S>(a);
  } else if constexpr (8 * q == R) {  // (1 + S i)/sqrt2
    const T c = T(0.70710678118654752440);
    return S < 0 ? mk(c * (a.x + a.y), c * (a.y - a.x)) : mk(c * (a.x - a.y), c * (a.y + a.x));
  } else if constexpr (8 * q == 3 * R) {  // (-1 + S i)/sqrt2
    const T c = T(0.70710678118654752440);
    return S < 0 ? mk(c * (a.y - a.x), -c * (a.x + a.y)) : mk(-c * (a.x + a.y), c * (a.x - a.y));
  } else {
    // generic: only R = 16, q in {1,3,5,7}
    constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;
    constexpr double cr = (q == 1) ? C1 : (q == 3) ? S1 : (q == 5) ? -S1 : -C1;
    constexpr double si = (q == 1) ? S1 : (q == 3) ? C1 : (q == 5) ? C1 : S1;
    const cx<T> w = mk(T(cr), T(S * si));
    return mul(a, w);
  }
}

template <int S, typename T>
__device__ __forceinline__ void dft8(cx<T>* v) {
  cx<T> e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  cx<T> o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<S>(e0, e1, e2, e3);
  dft4<S>(o0, o1, o2, o3);
  o1 = twc<8, 1, S>(o1);
  o2 = twc<8, 2, S>(o2);
  o3 = twc<8, 3, S>(o3);
  v[0] = add(e0, o0);
  v[4] = sub(e0, o0);
  v[1] = add(e1, o1);
  v[5] = sub(e1, o1);
  v[2] = add(e2, o2);
  v[6] = sub(e2, o2);
  v[3] = add(e3, o3);
  v[7] = sub(e3, o3);
}

template <int S, typename T>
__device__ __forceinline__ void dft16(cx<T>* v) {
  cx<T> e[8], o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    e[i] = v[2 * i];
    o[i] = v[2 * i + 1];
  }
  dft8<S>(e);
  dft8<S>(o);
  o[1] = twc<16, 1, S>(o[1]);
  o[2] = twc<16, 2, S>(o[2]);
  o[3] = twc<16, 3, S>(o[3]);
  o[4] = twc<16, 4, S>(o[4]);
  o[5] = twc<16, 5, S>(o[5]);
  o[6] = twc<16, 6, S>(o[6]);
  o[7] = twc<16, 7, S>(o[7]);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = add(e[i], o[i]);
    v[i + 8] = sub(e[i], o[i]);
  }
}

// radix 3: y1,2 = x0 - (x1+x2)/2 +- S i sqrt(3)/2 (x1 - x2)
template <int S, typename T>
__device__ __forceinline__ void dft3(cx<T>& x0, cx<T>& x1, cx<T>& x2) {
  const T h = T(0.86602540378443864676);
  const cx<T> s = add(x1, x2);
  const cx<T> d = sub(x1, x2);
  const cx<T> m = mk(x0.x - T(0.5) * s.x, x0.y - T(0.5) * s.y);
  const cx<T> r = S < 0 ? mk(h * d.y, -h * d.x) : mk(-h * d.y, h * d.x);  // (S i h) d
  x0 = add(x0, s);
  x1 = add(m, r);
  x2 = sub(m, r);
}

// multiply by exp(S 2 pi i q / R) for R in {6, 12}
template <int R, int Q, int S, typename T>
__device__ __forceinline__ cx<T> twc3(cx<T> a) {
  constexpr int q = Q % R;
  if constexpr (q == 0) {
    return a;
  } else if constexpr (4 * q == R) {
    return mul_si<S>(a);
  } else {
    constexpr double PI = 3.14159265358979323846;
    // cos/sin of 2 pi q / R for the few angles used (multiples of 30 degrees)
    constexpr int deg = 360 * q / R;
    constexpr double c = deg == 30 ? 0.86602540378443864676 : deg == 60 ? 0.5 : deg == 120 ? -0.5
                       : deg == 150 ? -0.86602540378443864676 : 0.0;
    constexpr double s = deg == 30 ? 0.5 : deg == 60 ? 0.86602540378443864676 : deg == 120
                       ? 0.86602540378443864676 : deg == 150 ? 0.5 : 0.0;
    (void)PI;
    return mul(a, mk(T(c), T(S * s)));
  }
}

template <int S, typename T>
__device__ __forceinline__ void dft6(cx<T>* v) {
  cx<T> e0 = v[0], e1 = v[2], e2 = v[4], o0 = v[1], o1 = v[3], o2 = v[5];
  dft3<S>(e0, e1, e2);
  dft3<S>(o0, o1, o2);
  o1 = twc3<6, 1, S>(o1);
  o2 = twc3<6, 2, S>(o2);
  v[0] = add(e0, o0);
  v[3] = sub(e0, o0);
  v[1] = add(e1, o1);
  v[4] = sub(e1, o1);
  v[2] = add(e2, o2);
  v[5] = sub(e2, o2);
}

template <int S, typename T>
__device__ __forceinline__ void dft12(cx<T>* v) {
  cx<T> e[6], o[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    e[i] = v[2 * i];
    o[i] = v[2 * i + 1];
  }
  dft6<S>(e);
  dft6<S>(o);
  o[1] = twc3<12, 1, S>(o[1]);
  o[2] = twc3<12, 2, S>(o[2]);
  o[3] = twc3<12, 3, S>(o[3]);
  o[4] = twc3<12, 4, S>(o[4]);
  o[5] = twc3<12, 5, S>(o[5]);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    v[i] = add(e[i], o[i]);
    v[i + 6] = sub(e[i], o[i]);
  }
}

template <int R, int S, typename T>
__device__ __forceinline__ void dftR(cx<T>* v) {
  if constexpr (R == 2) {
    dft2<S>(v[0], v[1]);
  } else if constexpr (R == 3) {
    dft3<S>(v[0], v[1], v[2]);
  } else if constexpr (R == 4) {
    dft4<S>(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 6) {
    dft6<S>(v);
  } else if constexpr (R == 8) {
    dft8<S>(v);
  } else if constexpr (R == 12) {
    dft12<S>(v);
  } else {
    static_assert(R == 16, "unsupported radix");
    dft16<S>(v);
  }
}

// One Stockham stage of radix R (Govindaraju et al. formulation): butterfly
// j reads x[j + r L/R], twiddles by W_{Ns R}^{r (j mod Ns)}, transforms, and
// writes to (j - j mod Ns) R + j mod Ns + r Ns.  Each thread owns 16/R
// butterflies (j = t + b TPR), i.e. 16 values per stage.
template <typename T, int R, int S>
__device__ __forceinline__ void stockham_stage(const Row<T>& row, int Ns) {
  constexpr int NB = 16 / R;
  cx<T> v[NB][R];
  const int LR = row.L / R;
  if (row.active) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = row.t + b * row.TPR;
#pragma unroll
      for (int r = 0; r < R; ++r) v[b][r] = row.ld(j + r * LR);
    }
  }
  row.sync();
  if (row.active) {
    const int tstride = row.L / (Ns * R);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = row.t + b * row.TPR;
      const int k = j & (Ns - 1);
      if (Ns > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          cx<T> w = ldg_cx(row.tw + r * k * tstride);
          if (S > 0) w.y = -w.y;
          v[b][r] = mul(v[b][r], w);
        }
      }
      dftR<R, S>(v[b]);
      const int base = (j - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) row.st(base + r * Ns, v[b][r]);
    }
  }
  row.sync();
}

template <typename T, int S>
__device__ __forceinline__ void fft_pow2(const Row<T>& row) {
  int Ns = 1;
  int rem = row.log2L;
  while (rem >= 4) {
    stockham_stage<T, 16, S>(row, Ns);
    Ns <<= 4;
    rem -= 4;
  }
  if (rem == 3)
    stockham_stage<T, 8, S>(row, Ns);
  else if (rem == 2)
    stockham_stage<T, 4, S>(row, Ns);
  else if (rem == 1)
    stockham_stage<T, 2, S>(row, Ns);
}

// ---- mixed radix (prime factors <= 13) ------------------------------------
// direct radix-R DFT with the row's length-L table: W_R^m = tw[m L / R]
template <int R, int S, typename T>
__device__ __forceinline__ void dft_tab(cx<T> (&x)[R], const cx<T>* __restrict__ tw, int LR) {
  if constexpr (R == 2 || R == 3 || R == 4) {
    dftR<R, S>(x);
  } else {
    cx<T> y[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      cx<T> a = x[0];
#pragma unroll
      for (int r = 1; r < R; ++r) {
        cx<T> w = ldg_cx(tw + ((r * q) % R) * LR);
        if (S > 0) w.y = -w.y;
        a = add(a, mul(x[r], w));
      }
      y[q] = a;
    }
#pragma unroll
    for (int q = 0; q < R; ++q) x[q] = y[q];
  }
}

// one out-of-place Stockham stage of radix R: src -> dst (padded = row layout)
template <int R, int S, typename T>
__device__ __forceinline__ void mixed_stage(const Row<T>& row, int Ns, const T* sre, const T* sim, bool spad,
                                            T* dre, T* dim, bool dpad) {
  const int L = row.L, LR = L / R, tstride = L / (Ns * R);
  for (int j = row.t; j < LR; j += row.TPR) {
    const int k = j % Ns;
    cx<T> x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = j + r * LR;
      const int p = spad ? pidx<T>(i) : i;
      x[r] = mk(sre[p], sim[p]);
    }
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        cx<T> w = ldg_cx(row.tw + r * k * tstride);
        if (S > 0) w.y = -w.y;
        x[r] = mul(x[r], w);
      }
    }
    dft_tab<R, S>(x, row.tw, LR);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = base + r * Ns;
      const int p = dpad ? pidx<T>(i) : i;
      dre[p] = x[r].x;
      dim[p] = x[r].y;
    }
  }
}

template <typename T, int S>
__device__ __noinline__ void fft_mixed(const Row<T>& row) {
  // ping-pong row <-> scratch; every thread of the group runs the syncs
  bool in_row = true;
  int Ns = 1;
  for (int s = 0; s < row.nst; ++s) {
    const int R = int((row.rad >> (4 * s)) & 15u);
    const T* sre = in_row ? row.re : row.sre;
    const T* sim = in_row ? row.im : row.sim;
    T* dre = in_row ? row.sre : row.re;
    T* dim = in_row ? row.sim : row.im;
    if (row.active) {
      switch (R) {
        case 2: mixed_stage<2, S>(row, Ns, sre, sim, in_row, dre, dim, !in_row); break;
        case 3: mixed_stage<3, S>(row, Ns, sre, sim, in_row, dre, dim, !in_row); break;
        case 4: mixed_stage<4, S>(row, Ns, sre, sim, in_row, dre, dim, !in_row); break;
        case 5: mixed_stage<5, S>(row, Ns, sre, sim, in_row, dre, dim, !in_row); break;
        default: mixed_stage<7, S>(row, Ns, sre, sim, in_row, dre, dim, !in_row); break;
      }
    }
    row.sync();
    Ns *= R;
    in_row = !in_row;
  }
  if (!in_row) {  // result sits in the scratch: copy back
    if (row.active)
      for (int i = row.t; i < row.L; i += row.TPR) row.st(i, mk(row.sre[i], row.sim[i]));
    row.sync();
  }
}

// ---- Bluestein (any L) -----------------------------------------------------
// forward: X_k = w_k sum_n (x_n w_n) b_{k-n}, b_m = conj(w_m) (cyclic, length
// M >= 2L-1); backward = conj(forward(conj x)).
template <typename T, int S>
__device__ __noinline__ void fft_bluestein(const Row<T>& row) {
  Row<T> m = row;  // the length-M work row (power-of-two Stockham)
  m.re = row.bre;
  m.im = row.bim;
  m.L = row.M;
  m.log2L = row.log2M;
  m.tw = row.twM;
  if (row.active) {
    for (int n = row.t; n < row.M; n += row.TPR) {
      cx<T> v = mk(T(0), T(0));
      if (n < row.L) {
        v = row.ld(n);
        if (S > 0) v.y = -v.y;
        v = mul(v, ldg_cx(row.chirp + n));
      }
      m.st(n, v);
    }
  }
  row.sync();
  fft_pow2<T, -1>(m);
  if (row.active)
    for (int k = row.t; k < row.M; k += row.TPR) m.st(k, mul(m.ld(k), ldg_cx(row.bhat + k)));
  row.sync();
  fft_pow2<T, +1>(m);
  if (row.active) {
    const T inv = T(1) / T(row.M);
    for (int k = row.t; k < row.L; k += row.TPR) {
      cx<T> v = scale(mul(m.ld(k), ldg_cx(row.chirp + k)), inv);
      if (S > 0) v.y = -v.y;
      row.st(k, v);
    }
  }
  row.sync();
}

// In-place transform of the row; callers sync before (data written) and may
// read the result right after (ends with a sync).
template <typename T, int S>
__device__ __forceinline__ void fft(const Row<T>& row) {
  if (row.kind == kFftPow2)
    fft_pow2<T, S>(row);
  else if (row.kind == kFftMixed)
    fft_mixed<T, S>(row);
  else
    fft_bluestein<T, S>(row);
}

}  // namespace lg
