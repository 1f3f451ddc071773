// Register-resident, compile-time-planned Stockham FFT (fp32 fast path).
//
// A row group of TPR = L/E threads transforms one length-L row.  Thread t
// holds the row in the NATURAL distribution v[e] = x[t + e*TPR] (coalesced
// global loads/stores, band gathers/scatters straight from registers).  The
// first Stockham stage reads its butterflies from that distribution and the
// last one writes its outputs back into it, so an S-stage plan needs only
// S-1 shared-memory exchanges.  Stage twiddles come from per-stage tables laid
// out [r-1][k] (k fastest) so a warp's twiddle loads are contiguous; they are
// issued before the exchange barrier so their latency hides behind it.
//
// Plans cover powers of two 32..8192 and 3*2^a (192..3072: the decimated
// imaging grid only has to hold 2P+1 samples), with radices
// 2, 3, 4, 6, 8, 12, 16 (every radix divides E).
//
// Conventions: reference fft2 (proj/src/core/imaging.cpp:17-31), SIGN -1
// forward, +1 backward, unnormalized.
#pragma once

#include <type_traits>
#include <utility>

#include "fft.cuh"

namespace lg {

// Twiddles per butterfly: 1 = load W^k and form W^(rk) by products (the row
// kernels are LSU-bound: C5 -5.3 % per iteration); 2 (default) = W^k from the
// SFU as well (__sincosf, |angle| < 2 pi / R, abs err ~4e-7; another -2.5 %);
// 0 = load every power (round 1).
#ifndef LG_TW_REC
#define LG_TW_REC 2
#endif

template <int L>
struct RPlan;

#define LG_RPLAN(LL, EE, ...)                            \
  template <>                                            \
  struct RPlan<LL> {                                     \
    static constexpr int L = LL;                         \
    static constexpr int E = EE;                         \
    static constexpr int TPR = LL / EE;                  \
    static constexpr int R[] = {__VA_ARGS__};            \
    static constexpr int NS = sizeof(R) / sizeof(int);   \
  };

LG_RPLAN(32, 8, 8, 4)
LG_RPLAN(64, 8, 8, 8)
LG_RPLAN(128, 16, 16, 8)
LG_RPLAN(256, 16, 16, 16)
LG_RPLAN(512, 8, 8, 8, 8)
LG_RPLAN(1024, 16, 16, 8, 8)
// 2048 = 8*4*8*8 on 256 threads: in-graph A/B at C2 against 8*8*8*4 (-1.0 %),
// 4*8*8*8, 8*8*4*8 and the E = 16 plans 16*16*8, 16*8*16, 8*16*16 (+3-6 %)
// 2048: 16*16*8 on 128 threads (two exchanges) since round 2: the row kernels
// are LSU-bound, C5 -6.5 % per iteration against 8*4*8*8 (C2 +3.7 %, tail)
#if !defined(LG_PLAN2048) || LG_PLAN2048 == 4
LG_RPLAN(2048, 16, 16, 16, 8)
#elif LG_PLAN2048 == 0
LG_RPLAN(2048, 8, 8, 4, 8, 8)
#elif LG_PLAN2048 == 1
LG_RPLAN(2048, 8, 8, 8, 8, 4)
#elif LG_PLAN2048 == 2
LG_RPLAN(2048, 8, 8, 8, 4, 8)
#elif LG_PLAN2048 == 3
LG_RPLAN(2048, 8, 4, 8, 8, 8)
#elif LG_PLAN2048 == 5
LG_RPLAN(2048, 16, 8, 16, 16)
#endif
LG_RPLAN(4096, 16, 16, 16, 16)
LG_RPLAN(8192, 16, 16, 16, 16, 2)
LG_RPLAN(192, 12, 12, 4, 4)
// 384 = 4*6*4*4: in-graph A/B at C2 against 12*4*4*2 (-1.5 %), 4*4*4*6,
// 4*4*6*4, 6*4*4*4, 4*4*2*12 and the E = 24 plans 8*6*8 / 6*8*8 (+16-26 %)
#if !defined(LG_PLAN384) || LG_PLAN384 == 0
LG_RPLAN(384, 12, 4, 6, 4, 4)
#elif LG_PLAN384 == 1
LG_RPLAN(384, 24, 8, 6, 8)
#elif LG_PLAN384 == 2
LG_RPLAN(384, 24, 6, 8, 8)
#elif LG_PLAN384 == 3
LG_RPLAN(384, 12, 12, 4, 4, 2)
#elif LG_PLAN384 == 4
LG_RPLAN(384, 12, 4, 4, 6, 4)
#elif LG_PLAN384 == 5
LG_RPLAN(384, 12, 4, 4, 4, 6)
#endif
// 768 = 4*4*4*12: C4 A/B against 12*4*4*4 (+5 % tile-iter/s), 4*12*4*4 (+3 %),
// 8*6*4*4 (E = 24, -1 %)
LG_RPLAN(768, 12, 4, 4, 4, 12)
LG_RPLAN(1536, 12, 12, 4, 4, 4, 2)
LG_RPLAN(3072, 12, 12, 4, 4, 4, 4)
#undef LG_RPLAN


template <int L, int S>
struct Stg {
  static constexpr int R = RPlan<L>::R[S];
  static constexpr int Ns = Stg<L, S - 1>::Ns * Stg<L, S - 1>::R;
  static constexpr int tw_off = Stg<L, S - 1>::tw_off + Stg<L, S - 1>::tw_len;
  static constexpr int tw_len = (R - 1) * Ns;
};
template <int L>
struct Stg<L, 0> {
  static constexpr int R = RPlan<L>::R[0];
  static constexpr int Ns = 1;
  static constexpr int tw_off = 0;
  static constexpr int tw_len = 0;
};

template <int L>
struct TwLen {
  static constexpr int value = Stg<L, RPlan<L>::NS - 1>::tw_off + Stg<L, RPlan<L>::NS - 1>::tw_len;
};

// Shared-memory exchange layouts (policy): where element i of a row lives.
//   Xch2<SW>: one float2 array;  XchS<SW>: split re / im float arrays.
// SW: 0 = i + (i>>4) padding, 1 = i ^ ((i>>3)&15), 2 = i ^ ((i>>4)&31),
//     3 = i ^ ((i>>3)&31), 4 = i + (i>>5) padding.  (XOR variants only for
//     power-of-two lengths.)
template <int SW>
__host__ __device__ __forceinline__ constexpr int swz(int i) {
  if constexpr (SW == 0) return i + (i >> 4);
  else if constexpr (SW == 1) return i ^ ((i >> 3) & 15);
  else if constexpr (SW == 2) return i ^ ((i >> 4) & 31);
  else if constexpr (SW == 3) return i ^ ((i >> 3) & 31);
  else return i + (i >> 5);
}
template <int SW>
__host__ __device__ constexpr int swz_len(int L) {
  return (SW == 0) ? L + (L >> 4) + 1 : (SW == 4) ? L + (L >> 5) + 1 : L;
}

// swz<SW>(i + C) == swz<SW>(i) + lin_delta<SW>(C) for every i >= 0 when
// lin_ok<SW>(C): the exchange addresses of a stage are then one swizzle per
// thread plus compile-time offsets.
template <int SW>
__host__ __device__ constexpr bool lin_ok(int C) {
  return SW == 0 ? C % 16 == 0 : (SW == 1 ? C % 128 == 0 : (SW == 4 ? C % 32 == 0 : false));
}
template <int SW>
__host__ __device__ constexpr int lin_delta(int C) {
  return SW == 0 ? C + C / 16 : (SW == 4 ? C + C / 32 : C);
}

// Exact compile-time linearity test of one exchange access pattern: thread t
// touches a(t) + c for the offsets c = b*cb + r*cr (b < NB, r < R), with
// a(t) = (t - t%Ns)*R + t%Ns for a Stockham store (TPR % Ns == 0, so k = t % Ns
// for every butterfly) or a(t) = t for a load.  Linear when
// swz(a(t) + c) == swz(a(t)) + swz(c) for every t and c: the addresses are then
// one swizzle per thread plus compile-time offsets (no per-element index math).
template <int SW>
__host__ __device__ constexpr bool lin_all(int TPR, int Ns, int R, int NB, int cb, int cr, bool store) {
  if (SW < 0) return false;
  if (store && TPR % Ns != 0) return false;
  for (int t = 0; t < TPR; ++t) {
    const int a = store ? (t - t % Ns) * R + t % Ns : t;
    for (int b = 0; b < NB; ++b)
      for (int r = 0; r < R; ++r) {
        const int c = b * cb + r * cr;
        if (swz<(SW < 0 ? 0 : SW)>(a + c) != swz<(SW < 0 ? 0 : SW)>(a) + swz<(SW < 0 ? 0 : SW)>(c)) return false;
      }
  }
  return true;
}

template <int SW>
struct Xch2 {  // float2 cells
  static constexpr bool soa = false;
  static constexpr int sw = SW;
  template <typename T>
  static __device__ __forceinline__ void st_raw(void* sm, int p, cx<T> v) {
    reinterpret_cast<cx<T>*>(sm)[p] = v;
  }
  template <typename T>
  static __device__ __forceinline__ cx<T> ld_raw(const void* sm, int p) {
    return reinterpret_cast<const cx<T>*>(sm)[p];
  }
  template <int L>
  __host__ __device__ static constexpr int bytes() { return swz_len<SW>(L) * 8; }
  template <typename T>
  static __device__ __forceinline__ void st(void* sm, int L, int i, cx<T> v) {
    reinterpret_cast<cx<T>*>(sm)[swz<SW>(i)] = v;
  }
  template <typename T>
  static __device__ __forceinline__ cx<T> ld(const void* sm, int L, int i) {
    return reinterpret_cast<const cx<T>*>(sm)[swz<SW>(i)];
  }
};
template <int SW>
struct XchS {  // split re / im
  static constexpr bool soa = true;
  static constexpr int sw = -1;  // no linear fast path
  template <int L>
  __host__ __device__ static constexpr int bytes() { return 2 * swz_len<SW>(L) * 4; }
  template <typename T>
  static __device__ __forceinline__ void st(void* sm, int L, int i, cx<T> v) {
    T* r = reinterpret_cast<T*>(sm);
    const int p = swz<SW>(i);
    r[p] = v.x;
    r[swz_len<SW>(L) + p] = v.y;
  }
  template <typename T>
  static __device__ __forceinline__ cx<T> ld(const void* sm, int L, int i) {
    const T* r = reinterpret_cast<const T*>(sm);
    const int p = swz<SW>(i);
    return mk(r[p], r[swz_len<SW>(L) + p]);
  }
};

// default exchange layout per plan (chosen by the on-GPU sweep)
template <int L>
struct XchOf {
  using type = Xch2<0>;
};
template <>
struct XchOf<512> {  // [8,8,8] plan: XOR swizzle measured 29.6 vs 26.1 TFLOP/s for padding
  using type = Xch2<1>;
};
#ifdef LG_XCH2048
template <>
struct XchOf<2048> {
  using type = Xch2<LG_XCH2048>;
};
#endif

// float2 cells of one row buffer (>= the padded natural layout used by to_smem)
template <int L>
__host__ __device__ constexpr int rsm_len() {
  return (XchOf<L>::type::template bytes<L>() + 7) / 8 > L + (L >> 4) + 1
             ? (XchOf<L>::type::template bytes<L>() + 7) / 8
             : L + (L >> 4) + 1;
}
__device__ __forceinline__ int rpad(int i) { return i + (i >> 4); }

// Barrier of one row group: warp-level when the group fits a warp, else a
// named barrier per group (id 1 + gid, <= 15 groups) or the CTA barrier.
struct GSync {
  int id;  // 0: __syncwarp(mask); >0: bar.sync id; <0: __syncthreads
  int n;
  unsigned mask = 0xffffffffu;  // id 0: the group's own lanes only
  __device__ __forceinline__ void operator()() const {
    if (id == 0)
      __syncwarp(mask);
    else if (id > 0)
      asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
    else
      __syncthreads();
  }
};

// Groups narrower than a warp synchronise only their own lanes: groups that
// share a warp run independent work (different kernel slots, some of them
// empty), so a full-warp barrier would couple them.
template <int L>
__device__ __forceinline__ GSync make_gsync(int gid, int groups) {
  constexpr int TPR = RPlan<L>::TPR;
  GSync s;
  s.n = TPR;
  if (TPR <= 32 && (32 % TPR) == 0) {
    s.id = 0;
    s.mask = TPR == 32 ? 0xffffffffu : (((1u << TPR) - 1u) << ((gid * TPR) & 31));
  } else if (groups <= 15 && TPR % 32 == 0) {
    s.id = 1 + gid;
  } else {
    s.id = -1;
  }
  return s;
}

// a * exp(S 2 pi i Q / R), R a power of two <= 16, any Q (compile-time rotations)
template <int R, int Q, int S, typename T>
__device__ __forceinline__ cx<T> rot(cx<T> a) {
  constexpr int q = ((Q % R) + R) % R;
  if constexpr (R >= 2 && 2 * q >= R) {
    const cx<T> b = rot<R, q - R / 2, S>(a);
    return mk(-b.x, -b.y);
  } else if constexpr (R >= 4 && 4 * q >= R) {
    return mul_si<S>(rot<R, q - R / 4, S>(a));
  } else {
    return twc<R, q, S>(a);  // q < R/4: 0, (R=16) 1..3, (R=8) 1
  }
}

// y_q = a + b W^{S q (R-1)}, q < R
template <int R, int SIGN, typename T, int... Q>
__device__ __forceinline__ void sp_in_outputs(cx<T> (&y)[R], cx<T> a, cx<T> b, std::integer_sequence<int, Q...>) {
  ((y[Q] = add(a, rot<R, Q * (R - 1), SIGN>(b))), ...);
}
// output q = R-1 of a radix-R DFT: sum_r x_r W^{S r (R-1)}
template <int R, int SIGN, typename T, int... Q>
__device__ __forceinline__ cx<T> sp_out_last(const cx<T> (&x)[R], std::integer_sequence<int, Q...>) {
  cx<T> y = x[0];
  ((Q > 0 ? (y = add(y, rot<R, Q * (R - 1), SIGN>(x[Q]))) : y), ...);
  return y;
}

__host__ __device__ constexpr bool pow2r(int r) { return r == 2 || r == 4 || r == 8 || r == 16; }

// ---- twiddled radix-2^j butterflies with the first radix-2 layer fused into
// FMAs (LG_FMA_L1).  For the pairs (r, r + R/2) of a twiddled stage:
//   t = x_r W^r,  p = t + x_{r+R/2} W^{r+R/2}  (4 FFMA),  m = 2t - p  (2 FFMA)
// instead of two complex products and two complex adds (-2 instructions per
// pair); the rest of the radix-R DFT takes the (p, m) pairs.
#ifndef LG_FMA_L1
#define LG_FMA_L1 1
#endif
template <typename T>
__device__ __forceinline__ void fma_pair(cx<T> t, cx<T> b, cx<T> wb, cx<T>& p, cx<T>& m) {
  p.x = fma(b.x, wb.x, fma(-b.y, wb.y, t.x));
  p.y = fma(b.x, wb.y, fma(b.y, wb.x, t.y));
  m.x = fma(T(2), t.x, -p.x);
  m.y = fma(T(2), t.y, -p.y);
}
// dft4 of (v0, v1, v2, v3) given p_r = v_r + v_{r+2}, m_r = v_r - v_{r+2}
template <int S, typename T>
__device__ __forceinline__ void dft4_pm(const cx<T>* p, const cx<T>* m, cx<T>* v) {
  const cx<T> t3 = mul_si<S>(m[1]);
  v[0] = add(p[0], p[1]);
  v[2] = sub(p[0], p[1]);
  v[1] = add(m[0], t3);
  v[3] = sub(m[0], t3);
}
template <int S, typename T>
__device__ __forceinline__ void dft8_pm(const cx<T>* p, const cx<T>* m, cx<T>* v) {
  // evens v0, v2, v4, v6: pairs (v0, v4) = (p0, m0), (v2, v6) = (p2, m2)
  cx<T> e[4], o[4];
  const cx<T> pe[2] = {p[0], p[2]}, me[2] = {m[0], m[2]}, po[2] = {p[1], p[3]}, mo[2] = {m[1], m[3]};
  dft4_pm<S>(pe, me, e);
  dft4_pm<S>(po, mo, o);
  o[1] = twc<8, 1, S>(o[1]);
  o[2] = twc<8, 2, S>(o[2]);
  o[3] = twc<8, 3, S>(o[3]);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = add(e[i], o[i]);
    v[i + 4] = sub(e[i], o[i]);
  }
}
template <int S, typename T>
__device__ __forceinline__ void dft16_pm(const cx<T>* p, const cx<T>* m, cx<T>* v) {
  cx<T> pe[4], me[4], po[4], mo[4], e[8], o[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    pe[i] = p[2 * i];
    me[i] = m[2 * i];
    po[i] = p[2 * i + 1];
    mo[i] = m[2 * i + 1];
  }
  dft8_pm<S>(pe, me, e);
  dft8_pm<S>(po, mo, o);
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
// twiddled radix-R butterfly (R = 4, 8, 16): x[r] <- DFT_R(x[r] W^r), w[r] = W^r (w[0] unused)
template <int R, int S, typename T>
__device__ __forceinline__ void dftR_tw_fma(cx<T> (&x)[R], const cx<T> (&w)[R]) {
  constexpr int H = R / 2;
  cx<T> p[H], m[H];
#pragma unroll
  for (int r = 0; r < H; ++r) {
    cx<T> wb = w[r + H];
    if (S > 0) wb.y = -wb.y;
    cx<T> t = x[r];
    if (r > 0) {
      cx<T> wa = w[r];
      if (S > 0) wa.y = -wa.y;
      t = mul(t, wa);
    }
    fma_pair(t, x[r + H], wb, p[r], m[r]);
  }
  if constexpr (R == 4)
    dft4_pm<S>(p, m, x);
  else if constexpr (R == 8)
    dft8_pm<S>(p, m, x);
  else
    dft16_pm<S>(p, m, x);
}

// Sparsity flags of fftr (band-limited rows):
//   kSpIn:  only the slots [0, NB) and [E-NB, E) (NB = butterflies per thread
//           in the first stage, sp_in_slots) are nonzero on entry;
//   kSpOut: only the slots [0, NB) and [E-NB, E) (NB = butterflies per thread
//           in the last stage, sp_out_slots) are needed on exit (the other
//           slots are left undefined).  Each flag is honoured where the stage structure
//           allows it (power-of-two radix, one butterfly per thread in the
//           stage concerned) and ignored otherwise (the dense path is exact).
constexpr int kSpIn = 1, kSpOut = 2;
// slots at each end that a kSpIn transform may hold nonzero
template <int L>
__host__ __device__ constexpr int sp_in_slots() {
  return RPlan<L>::E / RPlan<L>::R[0];
}
// slots at each end that a kSpOut transform defines
template <int L>
__host__ __device__ constexpr int sp_out_slots() {
  return RPlan<L>::E / RPlan<L>::R[RPlan<L>::NS - 1];
}

template <typename T, int L, int SIGN, int S, typename X, int SP = 0>
__device__ __forceinline__ void fftr_stage(cx<T> (&v)[RPlan<L>::E], cx<T>* sm,
                                           const cx<T>* __restrict__ tw, int t, const GSync& sync) {
  using P = RPlan<L>;
  using G = Stg<L, S>;
  constexpr int E = P::E, R = G::R, NB = E / R, TPR = P::TPR, Ns = G::Ns;
  constexpr bool FIRST = S == 0, LAST = S == P::NS - 1;
  // kSpIn: only slots [0, NB) and [E-NB, E) are nonzero on entry, i.e. only
  // inputs r = 0 and r = R-1 of every first-stage butterfly
  constexpr bool SP_IN = FIRST && (SP & kSpIn) && pow2r(R);
  constexpr bool SP_OUT = LAST && (SP & kSpOut) && pow2r(R) && !FIRST;
  cx<T> x[NB][R];
  cx<T> w[NB][R];
  if constexpr (Ns > 1) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int k = (t + b * TPR) % Ns;
#if LG_TW_REC
      // one table load per butterfly, the other powers W^(r k) by products
      // (LSU wavefronts traded for FMA-pipe work)
#if LG_TW_REC == 2
      if constexpr (std::is_same<T, float>::value) {
        float sn, cs;
        __sincosf(float(-2.0 * 3.14159265358979323846 / (Ns * R)) * float(k), &sn, &cs);
        w[b][1] = mk(cs, sn);
      } else {
        w[b][1] = ldg_cx(tw + G::tw_off + k);
      }
#else
      w[b][1] = ldg_cx(tw + G::tw_off + k);
#endif
#pragma unroll
      for (int r = 2; r < R; ++r) w[b][r] = (r % 2 == 0) ? mul(w[b][r / 2], w[b][r / 2]) : mul(w[b][r - 1], w[b][1]);
#else
#pragma unroll
      for (int r = 1; r < R; ++r) w[b][r] = ldg_cx(tw + G::tw_off + (r - 1) * Ns + k);
#endif
    }
  }
  constexpr int SW = X::sw;
  if constexpr (SP_IN) {
    // y_q = x_0 + x_{R-1} W^{S q (R-1)}: one rotation per output, no butterfly
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      cx<T> y[R];
      sp_in_outputs<R, SIGN>(y, v[b], v[b + (R - 1) * NB], std::make_integer_sequence<int, R>{});
#pragma unroll
      for (int r = 0; r < R; ++r) x[b][r] = y[r];
    }
  } else if constexpr (FIRST) {
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int r = 0; r < R; ++r) x[b][r] = v[b + r * NB];
  } else if constexpr (SW >= 0 && lin_all<SW>(TPR, 1, R, NB, TPR, L / R, false)) {
    // one swizzle per thread, compile-time offsets
    constexpr int SWc = SW < 0 ? 0 : SW;
    const int p0 = swz<SWc>(t);
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int r = 0; r < R; ++r)
        x[b][r] = X::template ld_raw<T>(sm, p0 + swz<SWc>(b * TPR + r * (L / R)));
  } else {
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int r = 0; r < R; ++r) x[b][r] = X::template ld<T>(sm, L, t + b * TPR + r * (L / R));
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if constexpr (Ns > 1 && !SP_OUT && LG_FMA_L1 && (R == 4 || R == 8 || R == 16)) {
      dftR_tw_fma<R, SIGN>(x[b], w[b]);  // twiddles fused into the first radix-2 layer
    } else {
      if constexpr (Ns > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          cx<T> ww = w[b][r];
          if (SIGN > 0) ww.y = -ww.y;
          x[b][r] = mul(x[b][r], ww);
        }
      }
      if constexpr (!SP_OUT && !SP_IN) dftR<R, SIGN>(x[b]);
    }
  }
  if constexpr (SP_OUT) {
    // only outputs q = 0 and q = R-1 of every butterfly are needed: slots
    // [0, NB) and [E-NB, E) of the natural distribution
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      cx<T> y0 = x[b][0];
#pragma unroll
      for (int r = 1; r < R; ++r) y0 = add(y0, x[b][r]);
      v[b] = y0;
      v[b + (R - 1) * NB] = sp_out_last<R, SIGN>(x[b], std::make_integer_sequence<int, R>{});
    }
    return;
  }
  if constexpr (LAST) {
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int r = 0; r < R; ++r) v[b + r * NB] = x[b][r];
  } else {
    sync();  // every thread finished reading sm (previous stage / previous use)
    constexpr int SWc = SW < 0 ? 0 : SW;
    if constexpr (SW >= 0 && lin_all<SW>(TPR, Ns, R, NB, TPR * R, Ns, true)) {
      // k = j mod Ns is the same for every butterfly of the thread
      const int k = t % Ns;
      const int p0 = swz<SWc>((t - k) * R + k);
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int r = 0; r < R; ++r)
          X::template st_raw<T>(sm, p0 + swz<SWc>(b * TPR * R + r * Ns), x[b][r]);
    } else {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int j = t + b * TPR;
        const int k = j % Ns;
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) X::template st<T>(sm, L, base + r * Ns, x[b][r]);
      }
    }
    sync();
    fftr_stage<T, L, SIGN, S + 1, X, SP>(v, sm, tw, t, sync);
  }
}

// In-register FFT of the row held in the natural distribution (SP: kSpIn /
// kSpOut sparsity flags, see fftr_stage).
template <typename T, int L, int SIGN, typename X = typename XchOf<L>::type, int SP = 0>
__device__ __forceinline__ void fftr(cx<T> (&v)[RPlan<L>::E], cx<T>* sm,
                                     const cx<T>* __restrict__ tw, int t, const GSync& sync) {
  fftr_stage<T, L, SIGN, 0, X, SP>(v, sm, tw, t, sync);
}
template <typename T, int L, int SIGN, int SP>
__device__ __forceinline__ void fftr_sp(cx<T> (&v)[RPlan<L>::E], cx<T>* sm,
                                        const cx<T>* __restrict__ tw, int t, const GSync& sync) {
  fftr_stage<T, L, SIGN, 0, typename XchOf<L>::type, SP>(v, sm, tw, t, sync);
}

// Store the natural-distribution row into sm (padded) so any element can be
// read by any thread of the group (callers sync before and after).
template <typename T, int L>
__device__ __forceinline__ void to_smem(const cx<T> (&v)[RPlan<L>::E], cx<T>* sm, int t) {
  constexpr int E = RPlan<L>::E, TPR = RPlan<L>::TPR;
#pragma unroll
  for (int e = 0; e < E; ++e) sm[rpad(t + e * TPR)] = v[e];
}

// Host helper: per-stage twiddle table (exp(-2 pi i r k / (Ns R)), [r-1][k])
template <int L, int S = 0, typename F>
void fill_rtwiddles(F&& put) {
  using G = Stg<L, S>;
  for (int r = 1; r < G::R; ++r)
    for (int k = 0; k < G::Ns; ++k) put(G::tw_off + (r - 1) * G::Ns + k, r * k, G::Ns * G::R);
  if constexpr (S + 1 < RPlan<L>::NS) fill_rtwiddles<L, S + 1>(put);
}

}  // namespace lg
