// fp32 fast path: column-kernel launchers (see socs_fast.h).
#include "fast_common.cuh"

namespace lg {

void fl_mask_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* Mr, long long mr_ts,
                  C32* Mhat, long long mh_ts) {
  with_len(g.ay.N, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = fgroups<L>(256);
    flaunch<L>(fk_mask_cols<L>, dim3(cdivi(g.ax.Pm + 1, gr), 1, tiles), gr, s, g, Mr, mr_ts, Mhat,
                mh_ts);
  });
}

void fl_socs_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* Mhat, long long mh_ts,
                  const C32* H, C32* T, long long t_ts) {
  with_len(g.ay.n, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = fgroups<L>(256);
    const size_t extra = size_t(L) * (gr | 1) * sizeof(C32);  // staging tile
    flaunch_x<L>(fk_socs_cols<L>, dim3(cdivi(g.ax.B, gr), g.F * g.K, tiles), gr, extra, s, g, Mhat, mh_ts,
                 H, T, t_ts);
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
    const int gr = fgroups<L>(256);
    flaunch<L>(fk_adj_cols<L>, dim3(cdivi(g.ax.B, gr), g.F * g.K, tiles), gr, s, g, U, u_ts, H, wk, dose,
               Accp, a_ts);
  });
}

void fl_grad_cols(const FGeo& g, cudaStream_t s, int tiles, const C32* Acc, long long a_ts, C32* Gc,
                  long long g_ts, const double* costp, long long cp_ts, int ncost,
                  double* cost_out, long long co_ts) {
  with_len(g.ay.N, [&](auto c) {
    constexpr int L = decltype(c)::value;
    const int gr = 1;  // one column per CTA: Pm+1 is small, spread it over SMs
    flaunch<L>(fk_grad_cols<L>, dim3(cdivi(g.ax.Pm + 1, gr) + 1, 1, tiles), gr, s, g, Acc, a_ts, Gc,
                g_ts, costp, cp_ts, ncost, cost_out, co_ts);
  });
}

}  // namespace lg
