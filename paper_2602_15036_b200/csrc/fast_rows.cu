// fp32 fast path: row-kernel launchers (see socs_fast.h).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "fast_common.cuh"

namespace lg {

// sparsity mode of a full-resolution row transform pair whose band is
// |p| <= P: bit 0 = the band fits slots 0 / E-1 (sparse first stage, 1-slot
// gather), bit 1 = it fits the kSpOut slots (pruned last stage)
template <int L>
static int spm_of(int P) {
  if (sparse_off()) return 0;
  int m = 0;
  if (P < RPlan<L>::TPR) m |= 1;
  if (P < sp_out_slots<L>() * RPlan<L>::TPR) m |= 2;
  if (!(m & 1) && P < 2 * RPlan<L>::TPR && RPlan<L>::E >= 4) m |= 4;  // 2-slot gather
  return m;
}

// threads per CTA of the full-resolution row kernels (real_rows_fwd,
// resist_rows, grad_rows) for `units` row pairs in the launch: 256 for batched
// launches (C5 -3.6 % against 128), 128 for launches of fewer than 2048 pairs
// 256-thread CTAs (C2, 1024 pairs: 1.8 % faster; C3, 3072: 2 % slower);
// LITHOGPU_ROW_THREADS=<n> (A/B)
static int fullrow_threads(long long units) {
  static const int env = [] {
    const char* e = std::getenv("LITHOGPU_ROW_THREADS");
    return e ? std::max(32, std::atoi(e)) : 0;
  }();
  if (env) return env;
  return units < 2048 ? 128 : 256;
}

int fast_tw_len(int len) {
  int n = 0;
  with_len(len, [&](auto c) { n = TwLen<decltype(c)::value>::value; });
  return n;
}

void fast_set_pdl(bool on) { pdl_enabled() = on; }

int fast_tpr(int len) {
  int n = 0;
  with_len(len, [&](auto c) { n = RPlan<decltype(c)::value>::TPR; });
  return n;
}

void fast_fill_twiddles(int len, C32* out) {
  with_len(len, [&](auto c) {
    fill_rtwiddles<decltype(c)::value>([&](int idx, int rk, int NsR) {
      const double a = 2.0 * M_PI * double(rk) / double(NsR);
      out[idx].x = float(std::cos(a));
      out[idx].y = float(-std::sin(a));
    });
  });
}

void fl_real_rows_fwd(const FGeo& g, cudaStream_t s, int tiles, int mode, const float* src,
                      long long src_ts, float steep, int Pout, C32* out, long long out_ts) {
  with_len(g.ax.N, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = fgroups<L>(fullrow_threads((long long)tiles * ((g.ay.N + 1) / 2)));
    const dim3 grid(cdivi((g.ay.N + 1) / 2, gr), 1, tiles);
    const size_t extra = size_t(Pout + 1) * 2 * gr * sizeof(C32) + 16;  // transposed-store tile
    auto go = [&](auto kern) { flaunch_x<L>(kern, grid, gr, extra, s, g, src, src_ts, steep, Pout, out, out_ts); };
    const bool sp = (spm_of<L>(Pout) & 2) != 0;
    if (mode == 0)
      sp ? go(fk_real_rows_fwd<L, 0, 2>) : go(fk_real_rows_fwd<L, 0, 0>);
    else
      sp ? go(fk_real_rows_fwd<L, 1, 2>) : go(fk_real_rows_fwd<L, 1, 0>);
  });
}

void fl_socs_rows(const FGeo& g, cudaStream_t s, int tiles, const C32* T, long long t_ts,
                  const float* wk, const float* wk2, float dose, C32* Ir, long long ir_ts, C32* Eo,
                  long long e_ts) {
  with_len(g.ax.n, [&](auto c) {
    constexpr int L = decltype(c)::value;
    int gr = fgroups<L>(256);
    if (gr > g.K) gr = g.K;
    auto go = [&](auto kern) {
      // + the TMA double buffer of T rows (2 rows per group)
      const size_t pad = groups_bytes<L>(gr) - size_t(gr) * rsm_len<L>() * sizeof(C32);  // 16-byte alignment
      flaunch_x<L>(kern, dim3(g.ay.n, g.F, tiles), gr, pad + size_t(gr) * 2 * g.tld * sizeof(C32), s, g, T, t_ts, wk,
                   wk2, dose, Ir, ir_ts, Eo, e_ts);
    };
    if (centered_band(L, RPlan<L>::E, g.ax.lo, g.ax.hi) && !sparse_off())
      band_fits_sp<L>(g.ax.lo, g.ax.hi) ? go(fk_socs_rows<L, true, true>) : go(fk_socs_rows<L, true, false>);
    else
      go(fk_socs_rows<L, false>);
  });
}

void fl_resist_rows(const FGeo& g, cudaStream_t s, int tiles, const C32* Rc, long long c_ts,
                    const float* target, long long tg_ts, const float* cf, float beta, float thr,
                    C32* Dr, long long d_ts, double* costp, long long cp_ts) {
  with_len(g.ax.N, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = fgroups<L>(fullrow_threads((long long)tiles * g.F * ((g.ay.N + 1) / 2)));
    auto go = [&](auto kern) {
      flaunch_x<L>(kern, dim3(cdivi((g.ay.N + 1) / 2, gr), g.F, tiles), gr,
                   row_slab_bytes<L>(gr) + size_t(g.ax.P + 1) * 2 * gr * sizeof(C32) + 16, s, g, Rc, c_ts, target,
                   tg_ts, cf, beta, thr, Dr, d_ts, costp, cp_ts);
    };
    // band inside the first / last register slots: sparse first / last FFT stage
    switch (spm_of<L>(g.ax.P)) {
      case 3: go(fk_resist_rows<L, 3>); break;
      case 6: go(fk_resist_rows<L, 6>); break;
      case 2: go(fk_resist_rows<L, 2>); break;
      case 4: go(fk_resist_rows<L, 4>); break;
      default: go(fk_resist_rows<L, 0>); break;
    }
  });
}

void fl_out_rows(const FGeo& g, cudaStream_t s, int tiles, const C32* Ic, const C32* Rc,
                 long long c_ts, float* Iout, float* Rout, unsigned char* print, long long o_ts,
                 float thr) {
  with_len(g.ax.N, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = fgroups<L>(256);
    flaunch<L>(fk_out_rows<L>, dim3(cdivi(g.ay.N, gr), g.F, tiles), gr, s, g, Ic, Rc, c_ts, Iout,
                Rout, print, o_ts, thr);
  });
}

void fl_wlp_rows(const FGeo& g, cudaStream_t s, int tiles, int nf, const C32* Wc, long long w_ts,
                 float* Wsub, long long ws_ts) {
  with_len(g.ax.n, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = spread_groups<L>((long long)tiles * nf * ((g.ay.n + 1) / 2));
    flaunch<L>(fk_wlp_rows<L>, dim3(cdivi((g.ay.n + 1) / 2, gr), nf, tiles), gr, s, g, Wc, w_ts,
                Wsub, ws_ts);
  });
}

void fl_adj_rows(const FGeo& g, cudaStream_t s, int tiles, int nf, bool uniform, bool from_e,
                 const C32* T, long long t_ts, const float* Wsub, long long ws_ts, C32* U, long long u_ts) {
  with_len(g.ax.n, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = fgroups<L>(256);
    const int nfk = nf * g.K;
    // kernel slots per CTA: keep >= ~8 CTAs per SM, amortise setup beyond that
    const long long units = (long long)cdivi(g.ay.n, gr) * nfk * tiles;
    int kc = int(units / (148 * 8));
    kc = kc < 1 ? 1 : (kc > 8 ? 8 : kc);
    if (const char* e = std::getenv("LITHOGPU_ADJ_KC")) kc = std::max(1, std::atoi(e));
    const dim3 grid(cdivi(g.ay.n, gr), cdivi(nfk, kc), tiles);
    // staging tile (16-byte padded) + one E row per group (TMA buffer, FROM_E)
    const size_t pad = groups_bytes<L>(gr) - size_t(gr) * rsm_len<L>() * sizeof(C32);
    const size_t tile_bytes = (size_t(g.ax.B) * (gr | 1) * sizeof(C32) + 15) & ~size_t(15);
    const size_t extra = pad + tile_bytes + ((from_e && LG_ADJ_TMA) ? size_t(gr) * L * sizeof(C32) : 0);
    auto go = [&](auto kern) { flaunch_x<L>(kern, grid, gr, extra, s, g, T, t_ts, Wsub, ws_ts, U, u_ts, kc, nfk); };
    const bool cb = centered_band(L, RPlan<L>::E, g.ax.lo, g.ax.hi) && !sparse_off();
    if (cb && band_fits_sp<L>(g.ax.lo, g.ax.hi)) {
      if (uniform)
        from_e ? go(fk_adj_rows<L, true, true, true, true>) : go(fk_adj_rows<L, true, false, true, true>);
      else
        from_e ? go(fk_adj_rows<L, false, true, true, true>) : go(fk_adj_rows<L, false, false, true, true>);
    } else if (cb) {
      if (uniform)
        from_e ? go(fk_adj_rows<L, true, true, true>) : go(fk_adj_rows<L, true, false, true>);
      else
        from_e ? go(fk_adj_rows<L, false, true, true>) : go(fk_adj_rows<L, false, false, true>);
    } else {
      if (uniform)
        from_e ? go(fk_adj_rows<L, true, true, false>) : go(fk_adj_rows<L, true, false, false>);
      else
        from_e ? go(fk_adj_rows<L, false, true, false>) : go(fk_adj_rows<L, false, false, false>);
    }
  });
}

void fl_grad_rows(const FGeo& g, cudaStream_t s, int tiles, bool ilt, const C32* Gc, long long g_ts,
                  float* grad, long long gr_ts, float* theta, long long th_ts, float steep,
                  float step, C32* Mr, long long mr_ts, double* gmaxp, long long gm_ts) {
  with_len(g.ax.N, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = fgroups<L>(fullrow_threads((long long)tiles * ((g.ay.N + 1) / 2)));
    const dim3 grid(cdivi((g.ay.N + 1) / 2, gr), 1, tiles);
    const size_t extra = row_slab_bytes<L>(gr) + size_t(g.ax.Pm + 1) * 2 * gr * sizeof(C32) + 16;
    const int spm = spm_of<L>(g.ax.Pm);
    auto go = [&](auto kern, size_t ex) {
      flaunch_x<L>(kern, grid, gr, ex, s, g, Gc, g_ts, grad, gr_ts, theta, th_ts, steep, step, Mr, mr_ts, gmaxp,
                   gm_ts);
    };
    if (ilt) {
      switch (spm) {
        case 3: go(fk_grad_rows<L, true, 3>, extra); break;
        case 6: go(fk_grad_rows<L, true, 6>, extra); break;
        case 2: go(fk_grad_rows<L, true, 2>, extra); break;
        case 4: go(fk_grad_rows<L, true, 4>, extra); break;
        default: go(fk_grad_rows<L, true, 0>, extra); break;
      }
    } else {
      // the gradient write path reads every slot of the first transform
      (spm & 1) ? go(fk_grad_rows<L, false, 1>, 0)
                : ((spm & 4) ? go(fk_grad_rows<L, false, 4>, 0) : go(fk_grad_rows<L, false, 0>, 0));
    }
  });
}

}  // namespace lg
