// fp32 fast path: column-kernel launchers (see socs_fast.h).
#include <algorithm>
#include <cstdlib>

#include "fast_common.cuh"

namespace lg {

void fl_mask_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* Mr, long long mr_ts,
                  C32* Mhat, long long mh_ts) {
  with_len(g.ay.N, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = spread_groups<L>((long long)tiles * (g.ax.Pm + 1));
    auto go = [&](auto kern) {
      flaunch<L>(kern, dim3(cdivi(g.ax.Pm + 1, gr), 1, tiles), gr, s, g, Mr, mr_ts, Mhat, mh_ts);
    };
    if (!sparse_off() && band_fits_sp_out<L>(g.ay.lo, g.ay.hi))
      go(fk_mask_cols<L, true>);
    else
      go(fk_mask_cols<L, false>);
  });
}

void fl_socs_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* Mhat, long long mh_ts,
                  const C32* H, C32* T, long long t_ts) {
  with_len(g.ay.n, [&](auto c) {
    constexpr int L = decltype(c)::value;
    int gr = fgroups<L>(4 * RPlan<L>::TPR);  // 4 columns per CTA: -0.7 % vs 8 at C2
    if (const char* e = std::getenv("LITHOGPU_SOCSCOLS_GROUPS")) gr = fgroups<L>(std::atoi(e) * RPlan<L>::TPR);
    const size_t extra = size_t(L) * (gr | 1) * sizeof(C32);  // staging tile
    auto go = [&](auto kern) {
      flaunch_x<L>(kern, dim3(cdivi(g.ax.B, gr), g.F * g.K, tiles), gr, extra, s, g, Mhat, mh_ts, H, T, t_ts);
    };
    if (centered_band(L, RPlan<L>::E, g.ay.lo, g.ay.hi) && !sparse_off())
      band_fits_sp<L>(g.ay.lo, g.ay.hi) ? go(fk_socs_cols<L, true, true>) : go(fk_socs_cols<L, true, false>);
    else
      go(fk_socs_cols<L, false>);
  });
}

void fl_band_colfwd(const FGeo& g, cudaStream_t s, int tiles, int nf, bool sub, const C32* in,
                    long long in_ts, const float* gxh, const float* gyb, C32* outR, C32* outI,
                    long long o_ts) {
  const int Lc = sub ? g.ay.n : g.ay.N;
  const float inv = float(1.0 / (double(sub ? g.ax.n : g.ax.N) * double(sub ? g.ay.n : g.ay.N)));
  with_len(Lc, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = fgroups<L>(256);
    flaunch<L>(fk_band_colfwd<L>, dim3(cdivi(g.ax.P + 1, gr), nf, tiles), gr, s, g, in, in_ts, inv,
                gxh, gyb, outR, outI, o_ts);
  });
}

void fl_band_colinv(const FGeo& g, cudaStream_t s, int tiles, int nf, bool sub, const C32* band,
                    long long b_ts, C32* out, long long o_ts) {
  with_len(sub ? g.ay.n : g.ay.N, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = fgroups<L>(256);
    flaunch<L>(fk_band_colinv<L>, dim3(cdivi(g.ax.P + 1, gr), nf, tiles), gr, s, g, band, b_ts, out,
                o_ts);
  });
}

void fl_adj_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* U, long long u_ts,
                 const C32* H, const float* wk, float dose, C32* Accp, long long a_ts) {
  with_len(g.ay.n, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int kg = kgroups<L>(g.K);  // fl_grad_cols sums F*K/kg partials: keep the two in step
    // band columns per CTA: keep >= ~8 CTAs per SM, amortise beyond that
    const long long units = (long long)g.ax.B * (g.F * g.K / kg) * tiles;
    int cc = int(units / (148 * 8));
    cc = cc < 1 ? 1 : (cc > 4 ? 4 : cc);
    if (const char* e = std::getenv("LITHOGPU_ADJCOLS_CC")) cc = std::max(1, std::atoi(e));
    auto go = [&](auto kern) {
      flaunch<L>(kern, dim3(cdivi(g.ax.B, cc), g.F * g.K / kg, tiles), kg, s, g, U, u_ts, H, wk, dose, Accp, a_ts,
                 cc);
    };
    if (centered_band(L, RPlan<L>::E, g.ay.lo, g.ay.hi) && !sparse_off())
      band_fits_sp<L>(g.ay.lo, g.ay.hi) ? go(fk_adj_cols<L, true, true>) : go(fk_adj_cols<L, true, false>);
    else
      go(fk_adj_cols<L, false>);
  });
}

void fl_grad_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* Acc, long long a_ts, int nsum,
                  C32* Gc, long long g_ts, const double* costp, long long cp_ts, int ncost,
                  double* cost_out, long long co_ts) {
  with_len(g.ay.N, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = 1;  // one column per CTA: Pm+1 is small, spread it over SMs
    with_len(g.ay.n, [&](auto cn) { nsum /= kgroups<decltype(cn)::value>(g.K); });  // fk_adj_cols partials
    const size_t extra = size_t(gr) * 2 * g.ay.B * sizeof(C32);  // summed band columns
    auto go = [&](auto kern) {
      flaunch_x<L>(kern, dim3(cdivi(g.ax.Pm + 1, gr) + 1, 1, tiles), gr, extra, s, g, Acc, a_ts, nsum, Gc, g_ts, costp,
                   cp_ts, ncost, cost_out, co_ts);
    };
    if (!sparse_off() && band_fits_sp_in<L>(g.ay.lo, g.ay.hi))
      go(fk_grad_cols<L, true>);
    else
      go(fk_grad_cols<L, false>);
  });
}

bool fl_band_col2(const FGeo& g, cudaStream_t s, int tiles, int nf, bool sub_in, const C32* in,
                  long long in_ts, const float* gxh, const float* gyb, C32* outR, C32* outI,
                  long long o_ts) {
  // sub_in: n -> N (intensity band -> resist columns); else N -> n (W band)
  const int Lin = sub_in ? g.ay.n : g.ay.N, Lout = sub_in ? g.ay.N : g.ay.n;
  const float inv = float(1.0 / (double(sub_in ? g.ax.n : g.ax.N) * double(Lin)));
  bool done = false;
  with_len(Lin, [&](auto ci) {
    constexpr int LI = decltype(ci)::value;
    with_len(Lout, [&](auto co) {
      constexpr int LO = decltype(co)::value;
      using CP = Col2<LI, LO>;
      constexpr int LBIG = LI > LO ? LI : LO, LSM = LI > LO ? LO : LI;
      constexpr bool pair = (LBIG == 1024 || LBIG == 2048 || LBIG == 4096) && LSM >= 256 && LSM <= 1536;
      if constexpr (pair && CP::ok && CP::TPR <= 256) {
        const int gr = CP::TPR >= 128 ? 1 : 128 / CP::TPR;
        const size_t smem = size_t(gr) * (CP::SM + 2 * CP::NB) * sizeof(C32);
        const bool cb = !g.ay.full && centered_band(LI, RPlan<LI>::E, -g.ay.P, g.ay.P) &&
                        centered_band(LO, RPlan<LO>::E, -g.ay.P, g.ay.P) && !sparse_off();
        auto go = [&](auto kern) {
          if (smem > 32 * 1024) set_max_smem(kern, smem);  // static shared memory counts toward the 48 KB default too
          pdl_launch(kern, dim3(cdivi(g.ax.P + 1, gr), nf, tiles), dim3(gr * CP::TPR), smem, s, g, in, in_ts,
                     inv, gxh, gyb, outR, outI, o_ts);
        };
        // N -> n (W band): only the intensity band of the length-N FFT is read
        const bool spo = cb && !sub_in && band_fits_sp_out<LI>(-g.ay.P, g.ay.P);
        if (spo)
          go(fk_band_col2<LI, LO, true, true>);
        else if (cb)
          go(fk_band_col2<LI, LO, true>);
        else
          go(fk_band_col2<LI, LO, false>);
        done = true;
      }
    });
  });
  return done;
}

}  // namespace lg

