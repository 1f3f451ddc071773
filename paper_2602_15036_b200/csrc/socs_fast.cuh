// fp32 fast-path kernels for power-of-two tiles, built on the register FFT
// (fftr.cuh).  Same data flow and reference anchors as socs_kernels.cuh (the
// generic runtime-length path kept for odd grids and the fp64 mode); here
// every transform length is a template parameter, band gathers/scatters go
// straight between global memory and registers, and the per-kernel work is
// spread over (row, kernel) so a 2048^2 tile fills all 148 SMs.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "fftr.cuh"
#include "socs_fast.h"

namespace lg {

// Programmatic dependent launch (sm_90+): wait for the predecessor's
// completion (and memory flush) before touching its outputs.  No explicit
// launch_dependents: the implicit trigger at CTA exit lets the next grid's
// CTAs take the slots the draining tail frees, without stealing slots from
// this grid's later waves (an early trigger measured slower).
// No-op when the launch did not opt in.
__device__ __forceinline__ void pdl_entry() {
#ifdef LG_PDL_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Tile index of this CTA: launches alternate the tile order (FGeo::zrev, set
// per launch by the host) so each kernel starts on the tiles its predecessor
// finished last, whose outputs are still in L2.
__device__ __forceinline__ unsigned tz(const FGeo& g) {
  return g.zrev ? gridDim.z - 1u - blockIdx.z : blockIdx.z;
}

// ---- launch trace (diagnostic; FGeo::trace) ----
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// CTAs fold onto kTraceCtas cells (batched launches have far more CTAs):
// cell[0] keeps ~min(start) (atomicMax of the complement), cell[1] max(end)
__device__ __forceinline__ unsigned long long* trace_cell(const FGeo& g) {
  const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  return g.trace + (size_t(g.trace_slot) * kTraceCtas + cta % unsigned(kTraceCtas)) * 2;
}
__device__ __forceinline__ void trace_begin(const FGeo& g) {
  if (g.trace && threadIdx.x == 0)
    if (auto* c = trace_cell(g)) atomicMax(c, ~gtimer());
}
__device__ __forceinline__ void trace_end(const FGeo& g) {
  if (g.trace && (threadIdx.x & 31) == 0)
    if (auto* c = trace_cell(g)) atomicMax(c + 1, gtimer());
}
struct TraceScope {  // CTA begin at construction, per-warp end at scope exit
  const FGeo& g;
  __device__ __forceinline__ explicit TraceScope(const FGeo& g_) : g(g_) { trace_begin(g); }
  __device__ __forceinline__ ~TraceScope() { trace_end(g); }
};

template <int L>
struct FGroup {
  static constexpr int TPR = RPlan<L>::TPR;
  static constexpr int E = RPlan<L>::E;
  int gid, t, groups;
  C32* sm;
  GSync sync;
  __device__ __forceinline__ FGroup() {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char fsm_raw[];
    groups = blockDim.x / TPR;
    gid = threadIdx.x / TPR;
    t = threadIdx.x % TPR;
    sm = reinterpret_cast<C32*>(fsm_raw) + gid * rsm_len<L>();
    sync = make_gsync<L>(gid, groups);
  }
  __device__ __forceinline__ int idx(int e) const { return t + e * TPR; }
};

// logistic sigmoid 1/(1+e^-x) on the SFU: ex2.approx.ftz + rcp.approx.ftz
// (|rel err| ~ 2^-22; no denormal fix-up sequences)
__device__ __forceinline__ float fsig(float x) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * -1.4426950408889634f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return r;
}

// kernel-band slot of residue i mod L, or -1
__device__ __forceinline__ int kslot(int i, int lo, int hi, int L) {
  int r = i - lo;  // i in [0, L), lo in (-L, L)
  r += r < 0 ? L : 0;
  r -= r >= L ? L : 0;
  return lo + r <= hi ? r : -1;
}
// Centered kernel band [lo, hi] (lo <= 0 <= hi, hi < L/2, -lo < L/2) of a
// length-L register row in the natural distribution (E even, so L/2 is a
// multiple of TPR): element e of thread t (index i = t + TPR e) lies in the
// lower half when 2e < E and then has slot i - lo if i <= hi; in the upper
// half it has slot i - L - lo if i >= L + lo.  So the slot is
// base + off(e) with a per-thread base and a compile-time offset, and
// validity is one bit per element: no per-element index arithmetic
// (kslot) in the loops over kernels.  centered_band() checks the geometry
// on the host.
template <int L>
struct BandMap {
  static constexpr int E = RPlan<L>::E, TPR = RPlan<L>::TPR;
  unsigned mask;  // bit e: element e is in the band
  int base;       // t - lo
  __host__ __device__ static constexpr int off(int e) { return TPR * e - (2 * e >= E ? L : 0); }
  __device__ __forceinline__ BandMap(int t, int lo, int hi) : mask(0u), base(t - lo) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = t + TPR * e;
      const bool in = (2 * e < E) ? (i <= hi) : (i >= L + lo);
      mask |= in ? (1u << e) : 0u;
    }
  }
  __device__ __forceinline__ bool has(int e) const { return (mask >> e) & 1u; }
};
__host__ __device__ inline bool centered_band(int L, int E, int lo, int hi) {
  return E % 2 == 0 && lo <= 0 && hi >= 0 && 2 * hi < L && -2 * lo < L;
}
// the band [lo, hi] fits the kSpIn / kSpOut slots of the length-L plan
// (centered): sparse first stage (band input) / pruned last stage (band output)
template <int L>
__host__ __device__ inline bool band_fits_sp_in(int lo, int hi) {
  const int w = sp_in_slots<L>() * RPlan<L>::TPR;
  return hi < w && -lo < w;
}
template <int L>
__host__ __device__ inline bool band_fits_sp_out(int lo, int hi) {
  const int w = sp_out_slots<L>() * RPlan<L>::TPR;
  return hi < w && -lo < w;
}
template <int L>
__host__ __device__ inline bool band_fits_sp(int lo, int hi) {
  constexpr int TPR = RPlan<L>::TPR;
  const int w = (sp_in_slots<L>() < sp_out_slots<L>() ? sp_in_slots<L>() : sp_out_slots<L>()) * TPR;
  return hi < w && -lo < w;
}

// intensity-band slot of residue i mod L (band2 layout of geom.h), or -1
__device__ __forceinline__ int islot(const AxisGeom& a, int i, int L) {
  if (a.full) return i;  // full band: L == n == N, slot j = residue
  int r = i + a.P;  // residue of p + P
  r -= r >= L ? L : 0;
  return r <= 2 * a.P ? r : -1;
}

// Build Z = A + iB for the row held in the natural distribution from the
// half spectra a[p*ld], b[p*ld] (p in [0, P]) of two real signals (b may be
// null; ld = 1 for row-major spectra, the column length for column-major).  Element
// e holds indices t + e*TPR, so only e < ceil((P+1)/TPR) can hit [0, P] and
// only e >= E - ceil(P/TPR) can hit the mirror [L-P, L): the other slots are
// zero by a warp-uniform test, without per-element divergent branches.
template <int L, int NSL = 0>
__device__ __forceinline__ void load_herm_pair(C32 (&v)[RPlan<L>::E], const FGroup<L>& g,
                                               const C32* a, const C32* b, int P, int ld) {
  constexpr int E = RPlan<L>::E, TPR = RPlan<L>::TPR;
  if constexpr (NSL > 0) {
    // band P < NSL*TPR: only slots e < NSL (index i = t + e TPR <= P) and
    // e >= E - NSL (mirror m = L - i <= P) can be nonzero (compile-time zero
    // elsewhere).  Rows y0, y0+1 of a column-major spectrum are adjacent
    // (b == a + 1, 16-byte aligned): one 16-byte load per entry.
    const bool adj = b == a + 1 && (ld % 2) == 0 && (reinterpret_cast<size_t>(a) & 15) == 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      C32 A = mk(0.f, 0.f), Bv = mk(0.f, 0.f);
      if (e < NSL || e >= E - NSL) {
        const int i = g.idx(e);
        const bool lo = e < NSL;
        const int m = (i == 0 ? 0 : L - i);
        const int src = lo ? i : m;
        if (src <= P) {
          if (adj) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(a + size_t(src) * ld));
            A = mk(q.x, q.y);
            Bv = mk(q.z, q.w);
          } else {
            A = a[size_t(src) * ld];
            if (b) Bv = b[size_t(src) * ld];
          }
          if (lo) {
            if (m == i) {
              A.y = 0.f;
              Bv.y = 0.f;
            }
          } else {
            A = conjg(A);
            Bv = conjg(Bv);
          }
        }
      }
      v[e] = mk(A.x - Bv.y, A.y + Bv.x);
    }
    return;
  }
  const int nlo = (P + TPR) / TPR, nhi = (P + TPR - 1) / TPR;
  const bool adj = b == a + 1 && (ld % 2) == 0 && (reinterpret_cast<size_t>(a) & 15) == 0;
  auto ld2 = [&](int src, C32& A, C32& Bv) {
    if (adj) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(a + size_t(src) * ld));
      A = mk(q.x, q.y);
      Bv = mk(q.z, q.w);
    } else {
      A = a[size_t(src) * ld];
      if (b) Bv = b[size_t(src) * ld];
    }
  };
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = g.idx(e);
    const int m = (i == 0 ? 0 : L - i);
    C32 A = mk(0.f, 0.f), Bv = mk(0.f, 0.f);
    if (e < nlo && i <= P) {
      ld2(i, A, Bv);
      if (m == i) {
        A.y = 0.f;
        Bv.y = 0.f;
      }
    } else if (e >= E - nhi && m <= P) {
      ld2(m, A, Bv);
      A = conjg(A);
      Bv = conjg(Bv);
    }
    v[e] = mk(A.x - Bv.y, A.y + Bv.x);
  }
}

// Two real rows (L floats each) staged into the group's shared-memory slab
// [2][L] with cp.async (16-byte chunks, L2-only) at kernel entry, so the
// transform runs without holding them in registers.  Reader: stage_wait()
// then a group barrier.
template <int L>
__host__ __device__ constexpr size_t groups_bytes(int groups) {
  return (size_t(groups) * rsm_len<L>() * sizeof(C32) + 15) & ~size_t(15);
}
template <int L>
__device__ __forceinline__ float* row_slab(int groups, int gid) {
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  return reinterpret_cast<float*>(fsm_raw + groups_bytes<L>(groups)) + size_t(gid) * 2 * L;
}
template <int L>
__device__ __forceinline__ void stage_rows_async(float* dst, const float* r0, const float* r1, int t) {
  constexpr int CH = L / 4, TPR = RPlan<L>::TPR;
#pragma unroll
  for (int c = t; c < 2 * CH; c += TPR) {
    const float* src = c < CH ? r0 + 4 * c : r1 + 4 * (c - CH);
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + 4 * c));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void stage_wait() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// The same staging through the TMA engine (cp.async.bulk, one elected
// thread, completion on an mbarrier): the two 4L-byte rows bypass the LSU
// pipe, which the exchange traffic of the row FFTs saturates.
// bar: the group's mbarrier (8 B of shared memory).  Readers call
// stage_wait_tma() after at least one group barrier (orders the init).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
template <int L>
__device__ __forceinline__ void stage_rows_tma(float* dst, const float* r0, const float* r1, int t,
                                               unsigned long long* bar) {
  if (t != 0) return;
  const unsigned b = smem_u32(bar);
  constexpr unsigned bytes = L * sizeof(float);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2 * bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(r0), "r"(bytes), "r"(b) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst + L)), "l"(r1), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void stage_wait_tma_parity(unsigned long long* bar, unsigned parity) {
  const unsigned b = smem_u32(bar);
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(b), "r"(parity) : "memory");
}
__device__ __forceinline__ void stage_wait_tma(unsigned long long* bar) {
  const unsigned b = smem_u32(bar);
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(b) : "memory");
}
#ifndef LG_NO_TMA_STAGE
#define LG_TMA_STAGE 1
#else
#define LG_TMA_STAGE 0
#endif
template <int L>
__host__ __device__ constexpr size_t row_slab_bytes(int groups) {
  return size_t(groups) * 2 * L * sizeof(float);
}

// Transposed store of a CTA's row pairs into a column-major half spectrum
// o[px][y] (px in [0, Pout]): the group's row pair sits in its exchange buffer
// (to_smem, synced); it is split into the two real rows' spectra, staged as
// tile[px][R] (R = 2 * groups rows of the CTA) and written as contiguous runs
// of R rows per column instead of 8-byte scattered stores.  CTA-wide barrier
// inside: every thread of the CTA must call it.  tile_off: byte offset of the
// tile past the row-group buffers.
template <int L>
__device__ __forceinline__ void store_pair_cols(const FGroup<L>& G, size_t tile_off, C32* o, int ld,
                                                int ybase, int nrows, int Pout) {
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  C32* tile = reinterpret_cast<C32*>(fsm_raw + tile_off);
  const int R = 2 * G.groups;
  for (int px = G.t; px <= Pout; px += G.TPR) {
    C32 A, Bv;
    split_pair(G.sm[rpad(px)], G.sm[rpad(px == 0 ? 0 : L - px)], A, Bv);
    tile[px * R + 2 * G.gid] = A;
    tile[px * R + 2 * G.gid + 1] = Bv;
  }
  __syncthreads();
  const int rows = min(R, nrows - ybase);
  for (int idx = threadIdx.x; idx < (Pout + 1) * R; idx += blockDim.x) {
    const int px = idx / R, r = idx - px * R;
    if (r < rows) o[size_t(px) * ld + ybase + r] = tile[idx];
  }
}

// to_smem of the slots a kSpOut transform defines ([0, NB) and [E-NB, E))
template <int L>
__device__ __forceinline__ void to_smem_sp(const C32 (&v)[RPlan<L>::E], C32* sm, int t) {
  constexpr int E = RPlan<L>::E, TPR = RPlan<L>::TPR, NB = sp_out_slots<L>();
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    sm[rpad(t + b * TPR)] = v[b];
    sm[rpad(t + (E - NB + b) * TPR)] = v[E - NB + b];
  }
}

// min resident CTAs for the full-resolution row kernels (64 registers with the
// 2048 = 8*8*8*4 plan)
// (after the twiddle-product change: 3 CTAs/SM, 85 registers, -1.1 % at C5)
#ifndef LG_FULLROW_MINB
#define LG_FULLROW_MINB 3
#endif

// warp-partial (deterministic) reduction: lane 0 of each warp-slice writes
__device__ __forceinline__ float warp_sum(float v, int width) {
  for (int o = width / 2; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, width);
  return v;
}
__device__ __forceinline__ float warp_max(float v, int width) {
  for (int o = width / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_down_sync(0xffffffffu, v, o, width));
  return v;
}

// ===========================================================================
// real row pairs -> half spectra [Pout+1][Ny] (MODE 0 raw, 1 sigmoid(steep x))
// ===========================================================================
template <int L, int MODE, int SPM>
__global__ void __launch_bounds__(256) fk_real_rows_fwd(FGeo g, const float* __restrict__ src,
                                                        long long src_ts, float steep, int Pout,
                                                        C32* __restrict__ out, long long out_ts) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E;
  const int Ny = g.ay.N, npairs = (Ny + 1) / 2;
  const int pair0 = blockIdx.x * G.groups + G.gid;
  const bool act = pair0 < npairs;
  const int pair = act ? pair0 : npairs - 1;
  const int y0 = 2 * pair, y1 = y0 + 1;
  const bool has1 = y1 < Ny;
  const float* s = src + tz(g) * src_ts;
  C32 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = G.idx(e);
    float a = s[size_t(y0) * L + i];
    float b = has1 ? s[size_t(y1) * L + i] : 0.f;
    if (MODE == 1) {
      a = fsig(steep * a);
      b = has1 ? fsig(steep * b) : 0.f;
    }
    v[e] = mk(a, b);
  }
  // kSpOut when the output band fits the first / last slot: the same
  // arithmetic as fk_grad_rows' fused next-iteration mask rows, so both
  // producers of Mr agree bitwise
  fftr_sp<float, L, -1, (SPM & 2) ? kSpOut : 0>(v, G.sm, g.twNx, G.t, G.sync);
  G.sync();
  if constexpr ((SPM & 2) != 0)
    to_smem_sp<L>(v, G.sm, G.t);
  else
    to_smem<float, L>(v, G.sm, G.t);
  G.sync();
  store_pair_cols<L>(G, groups_bytes<L>(G.groups), out + tz(g) * out_ts, Ny,
                     2 * blockIdx.x * G.groups, Ny, Pout);
}

// ===========================================================================
// SOCS rows, CTA = one subgrid row sy of focus f: the groups take the K
// kernels in turn (k = gid, gid + groups, ...), each  E = IFFT_nx(T_fk[sy])
// and accumulates dose w_fk |E|^2 in registers (wk2 != null: K kernel PAIRS,
// dose (w_a Re(E)^2 + w_b Im(E)^2), Plan::make_pairs); the group rows are summed in
// shared memory in fixed group order (deterministic), and group 0 transforms
// the intensity row: Ir[f][px][sy] = FFT_nx(I_sub[sy])(px), px in [0, P].
// Eo (nullable) keeps E_fk[sy][x] for the adjoint rows.
// grid (ny, F, tiles)
// ===========================================================================
// 3 CTAs / SM (80 registers, small spills) keeps all n rows resident: -2 % per
// ILT iteration at C2 against the unbounded 128-register build
#ifndef LG_SOCSROWS_MINB
#define LG_SOCSROWS_MINB 3
#endif
template <int L, bool CB, bool SPF = false>
__global__ void __launch_bounds__(256, LG_SOCSROWS_MINB) fk_socs_rows(FGeo g, const C32* __restrict__ T,
                                                    long long t_ts, const float* __restrict__ wk,
                                                    const float* __restrict__ wk2, float dose,
                                                    C32* __restrict__ Ir, long long ir_ts,
                                                    C32* __restrict__ Eo, long long e_ts) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E;
  const int ny = g.ay.n, lo = g.ax.lo, hi = g.ax.hi, K = g.K, tld = g.tld;
  const int sy = blockIdx.x, f = blockIdx.y;
  float acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  const BandMap<L> bm(G.t, lo, hi);
  // per-kernel row pointers advance by one kernel plane per slot
  const long long tstep = (long long)ny * tld;
  // CB: the group's T rows stream through a TMA double buffer in shared memory
  // (one bulk copy per kernel row, issued one row ahead; fk_socs_rows was
  // latency-bound on these gathers)
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  // 16-byte aligned for the bulk copies (groups_bytes rounds the exchange buffers up)
  C32* rb = reinterpret_cast<C32*>(fsm_raw + groups_bytes<L>(G.groups)) + size_t(G.gid) * 2 * tld;
  __shared__ unsigned long long tbar[16][2];
  const unsigned rbytes = unsigned(tld) * sizeof(C32);
  auto prefetch = [&](const C32* row, int b) {
    if (G.t == 0) {
      const unsigned bar = smem_u32(&tbar[G.gid][b]);
      // the group's generic-proxy reads of this buffer (two slots ago) are
      // ordered before the async-proxy overwrite
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(rbytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(rb + b * tld)), "l"(row), "r"(rbytes), "r"(bar) : "memory");
    }
  };
  // one kernel slot of this group: load its T row (CB: from the TMA buffer),
  // transform, keep E, accumulate w |E|^2
  auto slot = [&](int k, const C32* rowsrc) {
    const int fk = f * K + k;
    C32 v[E];
    if constexpr (CB) {
      const C32* sb = rowsrc + bm.base;
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = bm.has(e) ? sb[BandMap<L>::off(e)] : mk(0.f, 0.f);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int sl = kslot(G.idx(e), lo, hi, L);
        v[e] = sl >= 0 ? rowsrc[sl] : mk(0.f, 0.f);
      }
    }
    fftr_sp<float, L, +1, SPF ? kSpIn : 0>(v, G.sm, g.twnx, G.t, G.sync);
    if (Eo) {  // keep the coherent field for the adjoint (fk_adj_rows<.., FROM_E>)
      C32* eo = Eo + tz(g) * e_ts + (size_t(fk) * ny + sy) * L + G.t;
#pragma unroll
      for (int e = 0; e < E; ++e) eo[e * RPlan<L>::TPR] = v[e];
    }
    const float w = wk[fk] * dose;
    if (wk2) {  // kernel pair: E = E_a + i E_b with real E_a, E_b
      const float w2 = wk2[fk] * dose;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] += w * (v[e].x * v[e].x) + w2 * (v[e].y * v[e].y);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] += w * (v[e].x * v[e].x + v[e].y * v[e].y);
    }
  };
  // this group's ACTIVE slots k = gid, gid + groups, ... (empty slots of mixed
  // pairs skipped): only those are copied and waited for, so between two
  // copies into one buffer every thread of the group passes the FFT's group
  // barriers (a copy can never run a full mbarrier phase ahead of a waiter)
  auto next_k = [&](int k) {
    for (; k < K; k += G.groups)
      if (!g.slot_on || g.slot_on[f * K + k]) return k;
    return K;
  };
  const C32* trow0 = T + tz(g) * t_ts + size_t(f * K) * tstep + size_t(sy) * tld;
  // the TMA buffer only for whole-warp groups (the 384 / 768 plans); narrower
  // groups (short test transforms) gather straight from global memory
  constexpr bool TMA_T = CB && RPlan<L>::TPR >= 32;
  if constexpr (TMA_T) {
    if (G.t == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tbar[G.gid][0])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tbar[G.gid][1])) : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    G.sync();  // barrier inits before any wait
    int k = next_k(G.gid);
    if (k < K) prefetch(trow0 + size_t(k) * tstep, 0);
    for (int j = 0; k < K; ++j) {
      const int kn = next_k(k + G.groups);
      if (kn < K) prefetch(trow0 + size_t(kn) * tstep, (j + 1) & 1);
      const int b = j & 1;
      stage_wait_tma_parity(&tbar[G.gid][b], unsigned(j >> 1) & 1u);
      slot(k, rb + b * tld);
      k = kn;
    }
  } else {
    for (int k = next_k(G.gid); k < K; k = next_k(k + G.groups)) slot(k, trow0 + size_t(k) * tstep);
  }
  (void)rbytes;
  G.sync();  // exchange buffer free: publish the group's partial row
  float* red = reinterpret_cast<float*>(G.sm);
#pragma unroll
  for (int e = 0; e < E; ++e) red[G.idx(e)] = acc[e];
  __syncthreads();
  // the LAST group transforms the summed row: with the kernel slots dealt out
  // round-robin from group 0 it has the fewest of them (mixed pairs: half the
  // slots of a pairing stack are empty), so the CTA's critical path is shortest
  if (G.gid != G.groups - 1) return;
  const float* base = reinterpret_cast<const float*>(fsm_raw);
  constexpr int stride = 2 * rsm_len<L>();
  C32 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    float s = base[G.idx(e)];
    for (int gg = 1; gg < G.groups; ++gg) s += base[gg * stride + G.idx(e)];
    v[e] = mk(s, 0.f);
  }
  G.sync();  // every partial read before this group reuses its buffer
  fftr<float, L, -1>(v, G.sm, g.twnx, G.t, G.sync);
  C32* o = Ir + tz(g) * ir_ts + size_t(f) * (g.ax.P + 1) * ny + sy;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int px = G.idx(e);
    if (px <= g.ax.P) o[size_t(px) * ny] = v[e];
  }
}

// ===========================================================================
// ILT resist rows (row pair y0, y0+1 of focus f): R = IFFT_Nx(R^ half rows),
// Z = sig(beta (R - thr)), cost partial, D = 2 c_f (Z - Zt) beta Z (1 - Z),
// FFT_Nx(D pair) -> Dr[f][px][y].  grid (ceil(Ny/2/groups), F, tiles)
// ===========================================================================
template <int L, int SPM>
__global__ void __launch_bounds__(256, LG_FULLROW_MINB) fk_resist_rows(FGeo g, const C32* __restrict__ Rc,
                                                      long long c_ts, const float* __restrict__ target,
                                                      long long tg_ts, const float* __restrict__ cf,
                                                      float beta, float thr, C32* __restrict__ Dr,
                                                      long long d_ts, double* __restrict__ costp,
                                                      long long cp_ts) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E, TPR = RPlan<L>::TPR;
  constexpr int WPG = TPR >= 32 ? TPR / 32 : 1;
  // SPM bit 0: band inside slot 0 / E-1 (sparse first stage, 1-slot gather);
  // bit 1: band inside the kSpOut slots (pruned last stage)
  constexpr bool SPB = (SPM & 1) != 0, SPO = (SPM & 2) != 0;
  constexpr int NSL = SPB ? 1 : ((SPM & 4) ? 2 : 0);  // band slots at each end of the gather
  constexpr int SP_IN = SPB ? kSpIn : 0, SP_OUT = SPO ? kSpOut : 0;
  const int Ny = g.ay.N, Px = g.ax.P, f = blockIdx.y, npairs = (Ny + 1) / 2;
  const int pair0 = blockIdx.x * G.groups + G.gid;
  const bool act = pair0 < npairs;
  const int pair = act ? pair0 : npairs - 1;
  const int y0 = 2 * pair, y1 = y0 + 1;
  const bool has1 = y1 < Ny;
  const C32* rc = Rc + tz(g) * c_ts + size_t(f) * Ny * (Px + 1);
  // target rows staged into shared memory behind the transform
  const float* tg = target + tz(g) * tg_ts;
  float* tsl = row_slab<L>(G.groups, G.gid);
  __shared__ unsigned long long stage_bar[16];
  if (LG_TMA_STAGE)
    stage_rows_tma<L>(tsl, tg + size_t(y0) * L, tg + size_t(has1 ? y1 : y0) * L, G.t, &stage_bar[G.gid]);
  else
    stage_rows_async<L>(tsl, tg + size_t(y0) * L, tg + size_t(has1 ? y1 : y0) * L, G.t);
  C32 v[E];
  load_herm_pair<L, NSL>(v, G, rc + y0, has1 ? rc + y1 : nullptr, Px, Ny);  // column-major [px][y]
  fftr_sp<float, L, +1, SP_IN>(v, G.sm, g.twNx, G.t, G.sync);
  if (LG_TMA_STAGE) {
    stage_wait_tma(&stage_bar[G.gid]);
  } else {
    stage_wait();
    G.sync();
  }
  // branch-free pointwise resist: an odd last row (no partner) is masked by h1
  const float w = cf[f], h1 = has1 ? 1.f : 0.f;
  const float k2 = 2.f * w * beta;
  float c0 = 0.f, c1 = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const float z0 = fsig(beta * (v[e].x - thr));
    const float z1 = fsig(beta * (v[e].y - thr));
    const float e0 = z0 - tsl[G.idx(e)];
    const float e1 = z1 - tsl[L + G.idx(e)];
    c0 += e0 * e0;
    c1 += e1 * e1;
    v[e] = mk(k2 * e0 * (z0 - z0 * z0), h1 * (k2 * e1 * (z1 - z1 * z1)));
  }
  float c = warp_sum((c0 + h1 * c1) * w, TPR < 32 ? TPR : 32);
  if (act && (G.t & 31) == 0)
    costp[tz(g) * cp_ts + (size_t(f) * npairs + pair) * WPG + (G.t >> 5)] = double(c);
  fftr_sp<float, L, -1, SP_OUT>(v, G.sm, g.twNx, G.t, G.sync);
  G.sync();
  if constexpr (SPO)
    to_smem_sp<L>(v, G.sm, G.t);
  else
    to_smem<float, L>(v, G.sm, G.t);
  G.sync();
  store_pair_cols<L>(G, groups_bytes<L>(G.groups) + row_slab_bytes<L>(G.groups),
                     Dr + tz(g) * d_ts + size_t(f) * (Px + 1) * Ny, Ny, 2 * blockIdx.x * G.groups, Ny, Px);
}

// ===========================================================================
// forward output rows: I = Re, R = Im of IFFT_Nx(I^ + i R^), print = R >= thr
// grid (ceil(Ny/groups), F, tiles)
// ===========================================================================
template <int L>
__global__ void __launch_bounds__(256) fk_out_rows(FGeo g, const C32* __restrict__ Ic,
                                                   const C32* __restrict__ Rc, long long c_ts,
                                                   float* __restrict__ Iout, float* __restrict__ Rout,
                                                   unsigned char* __restrict__ print, long long o_ts,
                                                   float thr) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E;
  const int Ny = g.ay.N, Px = g.ax.P, f = blockIdx.y;
  const int y0 = blockIdx.x * G.groups + G.gid;
  const bool act = y0 < Ny;
  const int y = act ? y0 : Ny - 1;
  const size_t cb = tz(g) * c_ts + size_t(f) * Ny * (Px + 1) + y;  // column-major [f][px][y]
  C32 v[E];
  load_herm_pair<L>(v, G, Ic ? Ic + cb : Rc + cb, (Ic && Rc) ? Rc + cb : nullptr, Px, Ny);
  fftr<float, L, +1>(v, G.sm, g.twNx, G.t, G.sync);
  if (!act) return;
  const size_t ob = tz(g) * o_ts + (size_t(f) * Ny + y) * L;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = G.idx(e);
    const float Iv = v[e].x;
    const float Rv = Ic ? v[e].y : v[e].x;  // R alone sits in the real slot
    if (Iout && Ic) Iout[ob + i] = Iv;
    if (Rout && Rc) Rout[ob + i] = Rv;
    if (print && Rc) print[ob + i] = Rv >= thr ? 1 : 0;
  }
}

// ===========================================================================
// W_lp on the decimated grid: Wsub[f][sy] = IFFT_nx(Hermitian Wc[f][sy]) for
// row pairs.  grid (ceil(ny/2/groups), nf, tiles)
// ===========================================================================
template <int L>
__global__ void __launch_bounds__(256) fk_wlp_rows(FGeo g, const C32* __restrict__ Wc,
                                                   long long w_ts, float* __restrict__ Wsub,
                                                   long long ws_ts) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E;
  const int ny = g.ay.n, Px = g.ax.P, f = blockIdx.y, npairs = (ny + 1) / 2;
  const int pair0 = blockIdx.x * G.groups + G.gid;
  const bool act = pair0 < npairs;
  const int pair = act ? pair0 : npairs - 1;
  const int y0 = 2 * pair, y1 = y0 + 1;
  const bool has1 = y1 < ny;
  const C32* wc = Wc + tz(g) * w_ts + size_t(f) * ny * (Px + 1);
  C32 v[E];
  load_herm_pair<L>(v, G, wc + y0, has1 ? wc + y1 : nullptr, Px, ny);  // column-major [px][sy]
  fftr<float, L, +1>(v, G.sm, g.twnx, G.t, G.sync);
  if (!act) return;
  float* o = Wsub + tz(g) * ws_ts + size_t(f) * ny * L;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = G.idx(e);
    o[size_t(y0) * L + i] = v[e].x;
    if (has1) o[size_t(y1) * L + i] = v[e].y;
  }
}

// ===========================================================================
// adjoint rows, one (sy, f*K+k) per group:
//   U_fk[qx][sy] = FFT_nx(W_lp(sy,.) . IFFT_nx(T_fk[sy]))(qx), qx in band
// grid (ceil(ny/groups), F*K, tiles)
// ===========================================================================
// TMA-prefetched E rows in adj_rows: measured neutral-to-slower at C5 / C4 / C2
// (+0.2-0.6 %), so off by default (A/B switch)
// L2 prefetch of the next slot's E row in adj_rows (A/B switch)
#ifndef LG_ADJ_L2PF
#define LG_ADJ_L2PF 1
#endif
#ifndef LG_ADJ_TMA
#define LG_ADJ_TMA 0
#endif
#ifndef LG_ADJROWS_MINB
// C5 A/B: 4 CTAs/SM (64 regs) was +3.4 % over 2 (profiles/r2_ab1_occupancy.log); after the twiddle-product
// change 3 CTAs/SM (85 regs) is 1.5 % faster than 4
#define LG_ADJROWS_MINB 3
#endif
template <int L, bool UNIFORM, bool FROM_E, bool CB, bool SPF = false>
__global__ void __launch_bounds__(256, LG_ADJROWS_MINB) fk_adj_rows(FGeo g, const C32* __restrict__ T,
                                                      long long t_ts, const float* __restrict__ Wsub,
                                                      long long ws_ts, C32* __restrict__ U,
                                                      long long u_ts, int kc, int nfk) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E, TPR = RPlan<L>::TPR;
  const int ny = g.ay.n, Bx = g.ax.B, K = g.K, lo = g.ax.lo, hi = g.ax.hi;
  const int r0 = blockIdx.x * G.groups;
  const int sy0 = r0 + G.gid;
  const bool act = sy0 < ny;
  const int sy = act ? sy0 : ny - 1;
  const BandMap<L> bm(G.t, lo, hi);
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  C32* tile = reinterpret_cast<C32*>(fsm_raw) + G.groups * rsm_len<L>();
  const int ld = G.groups | 1;
  const int nr = min(G.groups, ny - r0);
  const int lgg = __ffs(G.groups) - 1;  // groups is a power of two (fgroups)
  // kc kernel slots per CTA (amortises the setup over several transforms);
  // empty slots (mixed pairs) are skipped, CTA-uniformly
  const int fk_begin = blockIdx.y * kc, fk_end = min(fk_begin + kc, nfk);
  auto next_active = [&](int x) {
    for (; x < fk_end; ++x)
      if (!g.slot_on || g.slot_on[x]) return x;
    return -1;
  };
  // FROM_E (LG_ADJ_TMA): the group's E row (L complex, contiguous, from HBM)
  // arrives by TMA bulk copy into shared memory, the next slot's copy issued
  // as soon as this one is in registers (after a group barrier, so a copy
  // never runs a phase ahead of a waiter)
  const size_t tile_bytes = (size_t(Bx) * ld * sizeof(C32) + 15) & ~size_t(15);
  C32* eb = reinterpret_cast<C32*>(fsm_raw + groups_bytes<L>(G.groups) + tile_bytes) + size_t(G.gid) * L;
  __shared__ unsigned long long ebar[16];
  auto erow = [&](int fk) { return T + tz(g) * t_ts + (size_t(fk) * ny + sy) * L; };
  auto prefetch = [&](int fk) {
    if (G.t == 0) {
      const unsigned bar = smem_u32(&ebar[G.gid]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(unsigned(L * sizeof(C32)))
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(eb)), "l"(erow(fk)), "r"(unsigned(L * sizeof(C32))), "r"(bar) : "memory");
    }
  };
  constexpr bool TMA_E = FROM_E && LG_ADJ_TMA;
  int cur = next_active(fk_begin);
  if constexpr (TMA_E) {
    if (G.t == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ebar[G.gid])) : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    G.sync();  // barrier init before any wait
    if (cur >= 0) prefetch(cur);
  }
  for (int j = 0; cur >= 0; ++j) {
    const int fk = cur, f = fk / K;
    const int nxt = next_active(fk + 1);
    C32 v[E];
    if constexpr (TMA_E) {
      stage_wait_tma_parity(&ebar[G.gid], unsigned(j) & 1u);
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = eb[G.t + e * TPR];
      G.sync();  // the group's reads of eb done before it is refilled
      if (nxt >= 0) prefetch(nxt);
    } else if (FROM_E) {  // T holds the fields E_fk[sy][x] kept by fk_socs_rows
      const C32* src = erow(fk) + G.t;
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = src[e * TPR];
#if LG_ADJ_L2PF
      // pull the next active slot's E row (from HBM) into L2 while this slot
      // transforms: one 128-byte line per lane
      if (nxt >= 0) {
        constexpr int LINES = (L * int(sizeof(C32)) + 127) / 128;
        const char* nrow = reinterpret_cast<const char*>(erow(nxt));
        for (int ln = G.t; ln < LINES; ln += TPR) asm volatile("prefetch.global.L2 [%0];" ::"l"(nrow + ln * 128));
      }
#endif
    } else if (CB) {
      const C32* sb = T + tz(g) * t_ts + size_t(fk) * ny * g.tld + size_t(sy) * g.tld + bm.base;
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = bm.has(e) ? sb[BandMap<L>::off(e)] : mk(0.f, 0.f);
    } else {
      const C32* src = T + tz(g) * t_ts + size_t(fk) * ny * g.tld + size_t(sy) * g.tld;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int sl = kslot(G.idx(e), lo, hi, L);
        v[e] = sl >= 0 ? src[sl] : mk(0.f, 0.f);
      }
    }
    float wv[E];
    if (!UNIFORM) {
      const float* w = Wsub + tz(g) * ws_ts + (size_t(f) * ny + sy) * L + G.t;
#pragma unroll
      for (int e = 0; e < E; ++e) wv[e] = w[e * TPR];
    }
    if (!FROM_E) fftr_sp<float, L, +1, SPF ? kSpIn : 0>(v, G.sm, g.twnx, G.t, G.sync);
    if (!UNIFORM) {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = scale(v[e], wv[e]);
    }
    fftr_sp<float, L, -1, SPF ? kSpOut : 0>(v, G.sm, g.twnx, G.t, G.sync);
    // stage the band outputs as tile[slot][row] (odd stride: conflict free),
    // then write U[fk][slot][r0 .. r0+groups) as contiguous row segments
    if constexpr (CB) {
      C32* tb = tile + bm.base * ld + G.gid;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (bm.has(e)) tb[BandMap<L>::off(e) * ld] = v[e];
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int sl = kslot(G.idx(e), lo, hi, L);
        if (sl >= 0) tile[sl * ld + G.gid] = v[e];
      }
    }
    __syncthreads();
    {  // fixed lane roles: thread -> row rr, slots sl0, sl0 + step, ...
      const int rr = threadIdx.x & (G.groups - 1), step = blockDim.x >> lgg;
      if (rr < nr) {
        int sl = threadIdx.x >> lgg;
        C32* op = U + tz(g) * u_ts + size_t(fk) * Bx * ny + r0 + size_t(sl) * ny + rr;
        const C32* tp = tile + sl * ld + rr;
        const size_t ostep = size_t(step) * ny;
        const int tstep = step * ld;
        for (; sl < Bx; sl += step, op += ostep, tp += tstep) *op = *tp;
      }
    }
    __syncthreads();  // tile free for the next slot
    cur = nxt;
  }
}

// ===========================================================================
// gradient rows (pair y0, y0+1): g = IFFT_Nx(Hermitian Gc rows) = dL/dM;
// !ILT: write grad; ILT: theta update, then next iteration's mask rows.
// grid (ceil(Ny/2/groups), 1, tiles)
// ===========================================================================
template <int L, bool ILT, int SPM>
__global__ void __launch_bounds__(256, LG_FULLROW_MINB) fk_grad_rows(FGeo g, const C32* __restrict__ Gc,
                                                    long long g_ts, float* __restrict__ grad,
                                                    long long gr_ts, float* __restrict__ theta,
                                                    long long th_ts, float steep, float step,
                                                    C32* __restrict__ Mr, long long mr_ts,
                                                    double* __restrict__ gmaxp, long long gm_ts) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E, TPR = RPlan<L>::TPR;
  constexpr int WPG = TPR >= 32 ? TPR / 32 : 1;
  // SPM bit 0: band inside slot 0 / E-1 (sparse first stage, 1-slot gather);
  // bit 1: band inside the kSpOut slots (pruned last stage)
  constexpr bool SPB = (SPM & 1) != 0, SPO = (SPM & 2) != 0;
  constexpr int NSL = SPB ? 1 : ((SPM & 4) ? 2 : 0);  // band slots at each end of the gather
  constexpr int SP_IN = SPB ? kSpIn : 0, SP_OUT = SPO ? kSpOut : 0;
  const int Ny = g.ay.N, Pm = g.ax.Pm, npairs = (Ny + 1) / 2;
  const int pair0 = blockIdx.x * G.groups + G.gid;
  const bool act = pair0 < npairs;
  const int pair = act ? pair0 : npairs - 1;
  const int y0 = 2 * pair, y1 = y0 + 1;
  const bool has1 = y1 < Ny;
  const C32* gc = Gc + tz(g) * g_ts;
  float* th = theta + tz(g) * th_ts;
  float* tsl = nullptr;  // theta rows staged into shared memory behind the transform
  __shared__ unsigned long long stage_bar[16];
  if (ILT) {
    tsl = row_slab<L>(G.groups, G.gid);
    if (LG_TMA_STAGE)
      stage_rows_tma<L>(tsl, th + size_t(y0) * L, th + size_t(has1 ? y1 : y0) * L, G.t, &stage_bar[G.gid]);
    else
      stage_rows_async<L>(tsl, th + size_t(y0) * L, th + size_t(has1 ? y1 : y0) * L, G.t);
  }
  C32 v[E];
  load_herm_pair<L, NSL>(v, G, gc + y0, has1 ? gc + y1 : nullptr, Pm, Ny);  // column-major [px][y]
  fftr_sp<float, L, +1, SP_IN>(v, G.sm, g.twNx, G.t, G.sync);
  if (ILT) {
    if (LG_TMA_STAGE) {
      stage_wait_tma(&stage_bar[G.gid]);
    } else {
      stage_wait();
      G.sync();
    }
  }
  if (!ILT) {
    if (!act) return;
    float* o = grad + tz(g) * gr_ts;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = G.idx(e);
      o[size_t(y0) * L + i] = v[e].x;
      if (has1) o[size_t(y1) * L + i] = v[e].y;
    }
    return;
  }
  // theta update, dL/dtheta = dL/dM * steep M (1 - M); rows written only by
  // active groups, an odd last row (no partner) only for y0
  float gm = 0.f;
  float* th0 = th + size_t(y0) * L;
  float* th1 = th + size_t(has1 ? y1 : y0) * L;
  float* gr0 = grad ? grad + tz(g) * gr_ts + size_t(y0) * L : nullptr;
  float* gr1 = grad ? grad + tz(g) * gr_ts + size_t(has1 ? y1 : y0) * L : nullptr;
  const bool w1 = act && has1;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = G.idx(e);
    const float t0 = tsl[i];
    const float t1 = tsl[L + i];
    const float m0 = fsig(steep * t0);
    const float m1 = fsig(steep * t1);
    const float g0 = v[e].x * steep * (m0 - m0 * m0);
    const float g1 = v[e].y * steep * (m1 - m1 * m1);
    const float n0 = t0 - step * g0;
    const float n1 = t1 - step * g1;
    gm = fmaxf(gm, fmaxf(fabsf(g0), has1 ? fabsf(g1) : 0.f));
    if (act) th0[i] = n0;
    if (w1) th1[i] = n1;
    if (gr0 && act) gr0[i] = g0;  // dL/dtheta (lithogpu_ilt_gradient)
    if (gr0 && w1) gr1[i] = g1;
    v[e] = mk(fsig(steep * n0), has1 ? fsig(steep * n1) : 0.f);
  }
  gm = warp_max(gm, TPR < 32 ? TPR : 32);
  if (act && gmaxp && (G.t & 31) == 0) gmaxp[tz(g) * gm_ts + size_t(pair) * WPG + (G.t >> 5)] = gm;
  fftr_sp<float, L, -1, SP_OUT>(v, G.sm, g.twNx, G.t, G.sync);
  G.sync();
  if constexpr (SPO)
    to_smem_sp<L>(v, G.sm, G.t);
  else
    to_smem<float, L>(v, G.sm, G.t);
  G.sync();
  store_pair_cols<L>(G, groups_bytes<L>(G.groups) + row_slab_bytes<L>(G.groups), Mr + tz(g) * mr_ts, Ny,
                     2 * blockIdx.x * G.groups, Ny, Pm);
}

// ===========================================================================
// mask half-spectrum columns -> kernel band M^ (Hermitian mirror for qx < 0)
// grid (ceil((Pmx+1)/groups), 1, tiles)
// ===========================================================================
template <int L, bool SPF = false>
__global__ void __launch_bounds__(256) fk_mask_cols(FGeo g, const C32* __restrict__ Mr,
                                                    long long mr_ts, C32* __restrict__ Mhat,
                                                    long long mh_ts) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E;
  const int Pm = g.ax.Pm;
  const int px0 = blockIdx.x * G.groups + G.gid;
  const bool act = px0 <= Pm;
  const int px = act ? px0 : Pm;
  const C32* src = Mr + tz(g) * mr_ts + size_t(px) * L;
  C32 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = src[G.idx(e)];
  fftr_sp<float, L, -1, SPF ? kSpOut : 0>(v, G.sm, g.twNy, G.t, G.sync);  // band (and mirror) outputs only
  if (!act) return;
  const float inv = 1.0f / (float(g.ax.N) * float(L));
  C32* mh = Mhat + tz(g) * mh_ts;  // column-major band [cx][jy]
  const int By = g.ay.B;
  const int sp = band_slot(g.ax, px);
  const int sn = px > 0 ? band_slot(g.ax, -px) : -1;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = G.idx(e);
    if (sp >= 0) {
      const int jy = kslot(i, g.ay.lo, g.ay.hi, L);
      if (jy >= 0) mh[size_t(sp) * By + jy] = scale(v[e], inv);
    }
    if (sn >= 0 && sn != sp) {
      const int jy = kslot((i == 0 ? 0 : L - i), g.ay.lo, g.ay.hi, L);
      if (jy >= 0) mh[size_t(sn) * By + jy] = scale(conjg(v[e]), inv);
    }
  }
}

// ===========================================================================
// per-kernel columns on the decimated grid: T_fk[sy][cx] = IFFT_ny(M^ H_fk);
// the CTA's groups take consecutive columns and stage the result through
// shared memory so T rows are written as contiguous segments.
// grid (ceil(Bx/groups), F*K, tiles)
// ===========================================================================
template <int L, bool CB, bool SPF = false>
__global__ void __launch_bounds__(512) fk_socs_cols(FGeo g, const C32* __restrict__ Mhat,
                                                    long long mh_ts, const C32* __restrict__ H,
                                                    C32* __restrict__ T, long long t_ts) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E;
  const int Bx = g.ax.B, By = g.ay.B, fk = blockIdx.y;
  if (g.slot_on && !g.slot_on[fk]) return;  // empty slot: T never read
  const int c0 = blockIdx.x * G.groups;
  const int cx0 = c0 + G.gid;
  const bool act = cx0 < Bx;
  const int cx_ = act ? cx0 : Bx - 1;
  // M^ and H are column-major [cx][jy]: each group reads contiguous columns
  const C32* mh = Mhat + tz(g) * mh_ts + size_t(cx_) * By;
  const C32* h = H + (size_t(fk) * Bx + cx_) * By;
  C32 v[E];
  if constexpr (CB) {
    const BandMap<L> bm(G.t, g.ay.lo, g.ay.hi);
    const C32* mb = mh + bm.base;
    const C32* hb = h + bm.base;
#pragma unroll
    for (int e = 0; e < E; ++e)
      v[e] = bm.has(e) ? mul(mb[BandMap<L>::off(e)], ldg_cx(hb + BandMap<L>::off(e))) : mk(0.f, 0.f);
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int jy = kslot(G.idx(e), g.ay.lo, g.ay.hi, L);
      v[e] = jy >= 0 ? mul(mh[jy], ldg_cx(h + jy)) : mk(0.f, 0.f);
    }
  }
  fftr_sp<float, L, +1, SPF ? kSpIn : 0>(v, G.sm, g.twny, G.t, G.sync);
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  C32* tile = reinterpret_cast<C32*>(fsm_raw) + G.groups * rsm_len<L>();
  const int ld = G.groups | 1;
#pragma unroll
  for (int e = 0; e < E; ++e) tile[G.idx(e) * ld + G.gid] = v[e];
  __syncthreads();
  const int nc = min(G.groups, Bx - c0);
  const int lgg = __ffs(G.groups) - 1;  // groups is a power of two (fgroups)
  // fixed lane roles: thread -> column cc, rows sy0, sy0 + step, ...
  const int cc = threadIdx.x & (G.groups - 1), step = blockDim.x >> lgg;
  if (cc >= nc) return;
  int sy = threadIdx.x >> lgg;
  C32* op = T + tz(g) * t_ts + size_t(fk) * L * g.tld + c0 + size_t(sy) * g.tld + cc;
  const C32* tp = tile + sy * ld + cc;
  const size_t ostep = size_t(step) * g.tld;
  const int tstep = step * ld;
#pragma unroll 4
  for (; sy < L; sy += step, op += ostep, tp += tstep) *op = *tp;
}

// ===========================================================================
// column FFT -> intensity band: out[f][j][px] = FFT_L(in[f][px])(p_j) s(j,px)
// grid (ceil((Px+1)/groups), nf, tiles).  inv = 1/(Lx L) (grid normalisation)
// ===========================================================================
template <int L>
__global__ void __launch_bounds__(256) fk_band_colfwd(FGeo g, const C32* __restrict__ in,
                                                      long long in_ts, float inv,
                                                      const float* __restrict__ gxh,
                                                      const float* __restrict__ gyb,
                                                      C32* __restrict__ outR, C32* __restrict__ outI,
                                                      long long o_ts) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E;
  const int Px = g.ax.P, f = blockIdx.y, nb2 = g.ay.nb2;
  const int px0 = blockIdx.x * G.groups + G.gid;
  const bool act = px0 <= Px;
  const int px = act ? px0 : Px;
  const C32* src = in + tz(g) * in_ts + (size_t(f) * (Px + 1) + px) * L;
  C32 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = src[G.idx(e)];
  fftr<float, L, -1>(v, G.sm, L == g.ay.N ? g.twNy : g.twny, G.t, G.sync);
  if (!act) return;
  const float gx = gxh ? gxh[px] : 1.f;
  const size_t ob = tz(g) * o_ts + size_t(f) * nb2 * (Px + 1);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = islot(g.ay, G.idx(e), L);
    if (j < 0) continue;
    const C32 c = scale(v[e], inv);
    if (outI) outI[ob + size_t(j) * (Px + 1) + px] = c;
    if (outR) outR[ob + size_t(j) * (Px + 1) + px] = gyb ? scale(c, gx * gyb[j]) : c;
  }
}

// ===========================================================================
// intensity band -> column IFFT of length L: out[f][y][px]
// grid (ceil((Px+1)/groups), nf, tiles)
// ===========================================================================
template <int L>
__global__ void __launch_bounds__(256) fk_band_colinv(FGeo g, const C32* __restrict__ band,
                                                      long long b_ts, C32* __restrict__ out,
                                                      long long o_ts) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E;
  const int Px = g.ax.P, f = blockIdx.y, nb2 = g.ay.nb2;
  const int px0 = blockIdx.x * G.groups + G.gid;
  const bool act = px0 <= Px;
  const int px = act ? px0 : Px;
  const C32* b = band + tz(g) * b_ts + size_t(f) * nb2 * (Px + 1);
  C32 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = islot(g.ay, G.idx(e), L);
    v[e] = j >= 0 ? b[size_t(j) * (Px + 1) + px] : mk(0.f, 0.f);
  }
  fftr<float, L, +1>(v, G.sm, L == g.ay.N ? g.twNy : g.twny, G.t, G.sync);
  if (!act) return;
  C32* o = out + tz(g) * o_ts + (size_t(f) * (Px + 1) + px) * L;  // column-major [f][px][y]
#pragma unroll
  for (int e = 0; e < E; ++e) o[G.idx(e)] = v[e];
}

// ===========================================================================
// fused band resampling column: out[f][y][px] = IFFT_LOUT(band(FFT_LIN(in[f][px]))
// s(j,px)), i.e. fk_band_colfwd + fk_band_colinv without the band round trip.
// One column per group of max(TPR_in, TPR_out) threads; the smaller plan runs
// on the group's leading warps.  outI (optional) gets the unscaled band.
// grid (ceil((Px+1)/groups), nf, tiles)
// ===========================================================================
template <int LIN, int LOUT>
struct Col2 {
  static constexpr int TIN = RPlan<LIN>::TPR, TOUT = RPlan<LOUT>::TPR;
  static constexpr int TPR = TIN > TOUT ? TIN : TOUT;
  static constexpr int SM = rsm_len<LIN>() > rsm_len<LOUT>() ? rsm_len<LIN>() : rsm_len<LOUT>();
  static constexpr int NB = LIN < LOUT ? LIN : LOUT;  // >= nb2
  static constexpr bool ok = TIN % 32 == 0 && TOUT % 32 == 0;
};

__device__ __forceinline__ GSync sub_gsync(int nthreads, int id) {
  GSync s;
  s.n = nthreads;
  s.id = nthreads == 32 ? 0 : id;
  return s;
}

template <int LIN, int LOUT, bool CB, bool SPF = false>
__global__ void __launch_bounds__(256) fk_band_col2(FGeo g, const C32* __restrict__ in,
                                                    long long in_ts, float inv,
                                                    const float* __restrict__ gxh,
                                                    const float* __restrict__ gyb,
                                                    C32* __restrict__ outR, C32* __restrict__ outI,
                                                    long long o_ts) {
  pdl_entry();
  TraceScope trace_(g);
  using CP = Col2<LIN, LOUT>;
  constexpr int EI = RPlan<LIN>::E, EO = RPlan<LOUT>::E;
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  const int groups = blockDim.x / CP::TPR, gid = threadIdx.x / CP::TPR, t = threadIdx.x % CP::TPR;
  C32* sm = reinterpret_cast<C32*>(fsm_raw) + gid * CP::SM;
  C32* bbR = reinterpret_cast<C32*>(fsm_raw) + groups * CP::SM + gid * 2 * CP::NB;
  C32* bbI = bbR + CP::NB;
  // barriers: 1..groups whole group, groups+1.. leading sub-group
  const GSync gsync = groups == 1 ? GSync{-1, CP::TPR} : GSync{1 + gid, CP::TPR};
  const int Px = g.ax.P, f = blockIdx.y;
  const int px0 = blockIdx.x * groups + gid;
  const bool act = px0 <= Px;
  const int px = act ? px0 : Px;
  if (t < CP::TIN) {
    const GSync s1 = CP::TIN == CP::TPR ? gsync : sub_gsync(CP::TIN, 1 + groups + gid);
    const C32* src = in + tz(g) * in_ts + (size_t(f) * (Px + 1) + px) * LIN;
    C32 v[EI];
#pragma unroll
    for (int e = 0; e < EI; ++e) v[e] = src[t + e * CP::TIN];
    fftr_sp<float, LIN, -1, SPF ? kSpOut : 0>(v, sm, LIN == g.ay.N ? g.twNy : g.twny, t, s1);  // band outputs only
    const float gx = gxh ? gxh[px] : 1.f;
    if constexpr (CB) {  // intensity band |p| <= P = centered band [-P, P]
      const BandMap<LIN> bm(t, -g.ay.P, g.ay.P);
#pragma unroll
      for (int e = 0; e < EI; ++e) {
        if (!bm.has(e)) continue;
        const int j = bm.base + BandMap<LIN>::off(e);
        const C32 c = scale(v[e], inv);
        if (outI) bbI[j] = c;
        bbR[j] = gyb ? scale(c, gx * gyb[j]) : c;
      }
    } else {
#pragma unroll
      for (int e = 0; e < EI; ++e) {
        const int j = islot(g.ay, t + e * CP::TIN, LIN);
        if (j < 0) continue;
        const C32 c = scale(v[e], inv);
        if (outI) bbI[j] = c;
        bbR[j] = gyb ? scale(c, gx * gyb[j]) : c;
      }
    }
  }
  gsync();
  if (t >= CP::TOUT) return;
  const GSync s2 = CP::TOUT == CP::TPR ? gsync : sub_gsync(CP::TOUT, 1 + groups + gid);
  const size_t ob = tz(g) * o_ts + (size_t(f) * (Px + 1) + px) * LOUT;  // column-major [f][px][y]
  for (int pass = 0; pass < 2; ++pass) {
    C32* out = pass == 0 ? outR : outI;
    if (!out) continue;
    const C32* bb = pass == 0 ? bbR : bbI;
    C32 v[EO];
    if constexpr (CB) {
      const BandMap<LOUT> bm(t, -g.ay.P, g.ay.P);
      const C32* b0 = bb + bm.base;
#pragma unroll
      for (int e = 0; e < EO; ++e) v[e] = bm.has(e) ? b0[BandMap<LOUT>::off(e)] : mk(0.f, 0.f);
    } else {
#pragma unroll
      for (int e = 0; e < EO; ++e) {
        const int j = islot(g.ay, t + e * CP::TOUT, LOUT);
        v[e] = j >= 0 ? bb[j] : mk(0.f, 0.f);
      }
    }
    fftr<float, LOUT, +1>(v, sm, LOUT == g.ay.N ? g.twNy : g.twny, t, s2);
    if (act) {
#pragma unroll
      for (int e = 0; e < EO; ++e) out[ob + t + e * CP::TOUT] = v[e];
    }
    s2();  // sm reused by the second pass
  }
}

// ===========================================================================
// adjoint columns: CTA = one band column cx x KG consecutive kernels (one per
// group), each FFT_ny(U_fk[cx]) conj(H_fk(.,cx)) 2 dose w_fk (N/n)^2/N^2 over
// the kernel band, summed over the CTA's kernels in fixed group order:
//   Accp[fk/KG][cx][qy]   (fk_grad_cols sums the F*K/KG partials, fixed order)
// grid (Bx, F*K/KG, tiles)
// ===========================================================================
template <int L, bool CB, bool SPF = false>
__global__ void __launch_bounds__(256) fk_adj_cols(FGeo g, const C32* __restrict__ U,
                                                   long long u_ts, const C32* __restrict__ H,
                                                   const float* __restrict__ wk, float dose,
                                                   C32* __restrict__ Accp, long long a_ts, int cc) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E, TPR = RPlan<L>::TPR;
  const int Bx = g.ax.B, By = g.ay.B, fk = blockIdx.y * G.groups + G.gid;
  const float sc = float(2.0 / (double(g.ax.n) * double(g.ay.n)));  // 2 (N/n)^2 / N^2
  const bool on = !g.slot_on || g.slot_on[fk];  // empty slot contributes 0
  const float w = on ? wk[fk] * dose * sc : 0.f;
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  const C32* base = reinterpret_cast<const C32*>(fsm_raw);
  // cc consecutive band columns per CTA; the next column's U row (HBM, written
  // by adj_rows) is pulled into L2 while this one transforms
  const int c0 = blockIdx.x * cc, c1 = min(c0 + cc, Bx);
  for (int cx = c0; cx < c1; ++cx) {
    const C32* src = U + tz(g) * u_ts + (size_t(fk) * Bx + cx) * L;
    C32 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = on ? src[G.idx(e)] : mk(0.f, 0.f);
    if (on && cx + 1 < c1) {
      constexpr int LINES = (L * int(sizeof(C32)) + 127) / 128;
      const char* nrow = reinterpret_cast<const char*>(src + L);
      for (int ln = G.t; ln < LINES; ln += TPR) asm volatile("prefetch.global.L2 [%0];" ::"l"(nrow + ln * 128));
    }
    if (on) fftr_sp<float, L, -1, SPF ? kSpOut : 0>(v, G.sm, g.twny, G.t, G.sync);
    const C32* h = H + (size_t(fk) * Bx + cx) * By;  // column-major [fk][cx][jy]
    G.sync();
    if constexpr (CB) {
      const BandMap<L> bm(G.t, g.ay.lo, g.ay.hi);
      const C32* hb = h + bm.base;
      C32* sb = G.sm + bm.base;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (bm.has(e)) sb[BandMap<L>::off(e)] = scale(mulc(v[e], ldg_cx(hb + BandMap<L>::off(e))), w);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int jy = kslot(G.idx(e), g.ay.lo, g.ay.hi, L);
        if (jy >= 0) G.sm[jy] = scale(mulc(v[e], ldg_cx(h + jy)), w);
      }
    }
    __syncthreads();
    C32* o = Accp + tz(g) * a_ts + (size_t(blockIdx.y) * Bx + cx) * By;
    for (int jy = threadIdx.x; jy < By; jy += blockDim.x) {
      C32 acc = base[jy];
      for (int gg = 1; gg < G.groups; ++gg) acc = add(acc, base[gg * rsm_len<L>() + jy]);
      o[jy] = acc;
    }
    __syncthreads();  // exchange buffers free for the next column
  }
}

// Fixed-order (deterministic) CTA sum of n cost partials into *out: strided
// per-thread sums with 8 loads in flight, then a fixed pairwise tree
// (blockDim a power of two <= 512).
__device__ __forceinline__ void reduce_cost(const double* __restrict__ c, int n, double* out) {
  __shared__ double red[512];
  const int bd = blockDim.x;
  double s = 0;
  int i = threadIdx.x;
  for (; i + 7 * bd < n; i += 8 * bd) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = c[i + j * bd];
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
  }
  for (; i < n; i += bd) s += c[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int h = bd / 2; h > 0; h >>= 1) {
    if (int(threadIdx.x) < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// ===========================================================================
// gradient columns: Hermitian part of Acc, IFFT_Ny -> Gc[y][px], px in [0,Pmx];
// the last CTA reduces this iteration's cost partials (fixed order).
// grid (ceil((Pmx+1)/groups) + 1, 1, tiles)
// ===========================================================================
template <int L, bool SPF = false>
__global__ void __launch_bounds__(256) fk_grad_cols(FGeo g, const C32* __restrict__ Acc,
                                                    long long a_ts, int nsum, C32* __restrict__ Gc,
                                                    long long g_ts, const double* __restrict__ costp,
                                                    long long cp_ts, int ncost,
                                                    double* __restrict__ cost_out, long long co_ts) {
  FGroup<L> G;
  TraceScope trace_(g);
  constexpr int E = RPlan<L>::E;
  if (blockIdx.x == gridDim.x - 1) {
    if (cost_out) reduce_cost(costp + tz(g) * cp_ts, ncost, cost_out + tz(g) * co_ts);
    return;
  }
  const int Pm = g.ax.Pm, Bx = g.ax.B;
  const int px0 = blockIdx.x * G.groups + G.gid;
  const bool act = px0 <= Pm;
  const int px = act ? px0 : Pm;
  // Acc holds nsum partials [.][cx][qy] (fk_adj_cols kernel groups): the
  // group first sums band columns sp and -px (sn) in fixed order into shared
  // memory with all its threads (short code, loads in flight together), then
  // gathers the Hermitian column from there
  const C32* a = Acc + tz(g) * a_ts;
  const int sp = band_slot(g.ax, px), sn = band_slot(g.ax, -px);
  const int By = g.ay.B;
  const size_t plane = size_t(Bx) * By;
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  C32* col = reinterpret_cast<C32*>(fsm_raw) + G.groups * rsm_len<L>() + G.gid * 2 * By;
  // up to 4 entries per thread summed side by side (independent loads in
  // flight), each over the partials in fixed order k = 0..nsum-1
  constexpr int MAXJ = 4;
  if (2 * By <= MAXJ * G.TPR) {
    const C32* src[MAXJ];
    C32 q[MAXJ];
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int idx = G.t + j * G.TPR;
      const int which = idx >= By, jy = idx - which * By, slot = which ? sn : sp;
      src[j] = (idx < 2 * By && slot >= 0) ? a + size_t(slot) * By + jy : nullptr;
      q[j] = mk(0.f, 0.f);
    }
    for (int k = 0; k < nsum; ++k) {
#pragma unroll
      for (int j = 0; j < MAXJ; ++j)
        if (src[j]) q[j] = add(q[j], ldg_cx(src[j] + k * plane));
    }
#pragma unroll
    for (int j = 0; j < MAXJ; ++j)
      if (G.t + j * G.TPR < 2 * By) col[G.t + j * G.TPR] = q[j];
  } else {
    for (int idx = G.t; idx < 2 * By; idx += G.TPR) {
      const int which = idx >= By, jy = idx - which * By, slot = which ? sn : sp;
      C32 q = mk(0.f, 0.f);
      if (slot >= 0) {
#pragma unroll 4
        for (int k = 0; k < nsum; ++k) q = add(q, ldg_cx(a + k * plane + size_t(slot) * By + jy));
      }
      col[idx] = q;
    }
  }
  G.sync();
  C32 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = G.idx(e);
    const int jp = kslot(i, g.ay.lo, g.ay.hi, L);
    const int jn = kslot((i == 0 ? 0 : L - i), g.ay.lo, g.ay.hi, L);
    C32 s = mk(0.f, 0.f);
    if (sp >= 0 && jp >= 0) s = add(s, col[jp]);
    if (sn >= 0 && jn >= 0) s = add(s, conjg(col[By + jn]));
    v[e] = scale(s, 0.5f);
  }
  fftr_sp<float, L, +1, SPF ? kSpIn : 0>(v, G.sm, g.twNy, G.t, G.sync);  // band input
  if (!act) return;
  C32* o = Gc + tz(g) * g_ts + size_t(px) * L;  // column-major [px][y]
#pragma unroll
  for (int e = 0; e < E; ++e) o[G.idx(e)] = v[e];
}

}  // namespace lg
