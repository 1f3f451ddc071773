// fp32 fast path: row-kernel launchers (see socs_fast.h).
#include <cmath>

#include "fast_common.cuh"

namespace lg {

int fast_tw_len(int lg) {
  int n = 0;
  with_lg(lg, [&](auto c) { n = TwLen<decltype(c)::value>::value; });
  return n;
}

int fast_tpr(int lg) {
  int n = 0;
  with_lg(lg, [&](auto c) { n = RPlan<decltype(c)::value>::TPR; });
  return n;
}

void fast_fill_twiddles(int lg, C32* out) {
  with_lg(lg, [&](auto c) {
    fill_rtwiddles<decltype(c)::value>([&](int idx, int rk, int NsR) {
      const double a = 2.0 * M_PI * double(rk) / double(NsR);
      out[idx].x = float(std::cos(a));
      out[idx].y = float(-std::sin(a));
    });
  });
}

void fl_real_rows_fwd(const FGeo& g, cudaStream_t s, int tiles, int mode, const float* src,
                      long long src_ts, float steep, int Pout, C32* out, long long out_ts) {
  with_lg(g.lgNx, [&](auto c) {
    constexpr int LG = decltype(c)::value;
    const int gr = fgroups<LG>(256);
    const dim3 grid(cdivi((g.ay.N + 1) / 2, gr), 1, tiles);
    if (mode == 0)
      flaunch<LG>(fk_real_rows_fwd<LG, 0>, grid, gr, s, g, src, src_ts, steep, Pout, out, out_ts);
    else
      flaunch<LG>(fk_real_rows_fwd<LG, 1>, grid, gr, s, g, src, src_ts, steep, Pout, out, out_ts);
  });
}

void fl_socs_rows(const FGeo& g, cudaStream_t s, int tiles, const C32* T, long long t_ts,
                  const float* wk, float dose, C32* Ir, long long ir_ts) {
  with_lg(g.lgnx, [&](auto c) {
    constexpr int LG = decltype(c)::value;
    const int gr = fgroups<LG>(512, g.K);
    flaunch<LG>(fk_socs_rows<LG>, dim3(g.ay.n, g.F, tiles), gr, s, g, T, t_ts, wk, dose, Ir, ir_ts);
  });
}

void fl_resist_rows(const FGeo& g, cudaStream_t s, int tiles, const C32* Rc, long long c_ts,
                    const float* target, long long tg_ts, const float* cf, float beta, float thr,
                    C32* Dr, long long d_ts, double* costp, long long cp_ts) {
  with_lg(g.lgNx, [&](auto c) {
    constexpr int LG = decltype(c)::value;
    const int gr = fgroups<LG>(256);
    flaunch<LG>(fk_resist_rows<LG>, dim3(cdivi((g.ay.N + 1) / 2, gr), g.F, tiles), gr, s, g, Rc,
                c_ts, target, tg_ts, cf, beta, thr, Dr, d_ts, costp, cp_ts);
  });
}

void fl_out_rows(const FGeo& g, cudaStream_t s, int tiles, const C32* Ic, const C32* Rc,
                 long long c_ts, float* Iout, float* Rout, unsigned char* print, long long o_ts,
                 float thr) {
  with_lg(g.lgNx, [&](auto c) {
    constexpr int LG = decltype(c)::value;
    const int gr = fgroups<LG>(256);
    flaunch<LG>(fk_out_rows<LG>, dim3(cdivi(g.ay.N, gr), g.F, tiles), gr, s, g, Ic, Rc, c_ts, Iout,
                Rout, print, o_ts, thr);
  });
}

void fl_wlp_rows(const FGeo& g, cudaStream_t s, int tiles, int nf, const C32* Wc, long long w_ts,
                 float* Wsub, long long ws_ts) {
  with_lg(g.lgnx, [&](auto c) {
    constexpr int LG = decltype(c)::value;
    const int gr = fgroups<LG>(256);
    flaunch<LG>(fk_wlp_rows<LG>, dim3(cdivi((g.ay.n + 1) / 2, gr), nf, tiles), gr, s, g, Wc, w_ts,
                Wsub, ws_ts);
  });
}

void fl_adj_rows(const FGeo& g, cudaStream_t s, int tiles, int nf, bool uniform, const C32* T,
                 long long t_ts, const float* Wsub, long long ws_ts, C32* U, long long u_ts) {
  with_lg(g.lgnx, [&](auto c) {
    constexpr int LG = decltype(c)::value;
    const int gr = fgroups<LG>(256);
    const dim3 grid(cdivi(g.ay.n, gr), nf * g.K, tiles);
    if (uniform)
      flaunch<LG>(fk_adj_rows<LG, true>, grid, gr, s, g, T, t_ts, Wsub, ws_ts, U, u_ts);
    else
      flaunch<LG>(fk_adj_rows<LG, false>, grid, gr, s, g, T, t_ts, Wsub, ws_ts, U, u_ts);
  });
}

void fl_grad_rows(const FGeo& g, cudaStream_t s, int tiles, bool ilt, const C32* Gc, long long g_ts,
                  float* grad, long long gr_ts, float* theta, long long th_ts, float steep,
                  float step, C32* Mr, long long mr_ts, double* gmaxp, long long gm_ts) {
  with_lg(g.lgNx, [&](auto c) {
    constexpr int LG = decltype(c)::value;
    const int gr = fgroups<LG>(256);
    const dim3 grid(cdivi((g.ay.N + 1) / 2, gr), 1, tiles);
    if (ilt)
      flaunch<LG>(fk_grad_rows<LG, true>, grid, gr, s, g, Gc, g_ts, grad, gr_ts, theta, th_ts, steep,
                  step, Mr, mr_ts, gmaxp, gm_ts);
    else
      flaunch<LG>(fk_grad_rows<LG, false>, grid, gr, s, g, Gc, g_ts, grad, gr_ts, theta, th_ts,
                  steep, step, Mr, mr_ts, gmaxp, gm_ts);
  });
}

}  // namespace lg
