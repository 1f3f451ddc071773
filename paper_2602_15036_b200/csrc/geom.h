// Band geometry of one imaging tile (host + device).
//
// The reference stores SOCS kernels full-grid but writes them only on the
// TCC support (proj/src/core/imaging.cpp:198-203), a disk of radius
// (1+sigma_max) NA/lambda: kernel band Q = [lo,hi] per axis, B = hi-lo+1.
// |E_k|^2 then holds only difference frequencies |p| <= B-1 =: P, so the
// aerial image is an exact trigonometric polynomial that is fully determined
// by its samples on a decimated grid n = N/d as long as n >= 2P+1 (no
// aliasing of the intensity band).  All per-kernel work (the K x F coherent
// fields) runs on that n-grid; only the few real-valued mask / resist /
// gradient transforms run at the full N-grid resolution, band-pruned.
// When no decimation satisfies n >= 2P+1 (small or coarse grids) the tile
// runs with d = 1 and a "full" intensity band (all residues), which is the
// reference's own full-grid algorithm.
#pragma once

namespace lg {

struct AxisGeom {
  int N;      // full grid length
  int n;      // decimated grid length (N / d)
  int d;      // decimation factor
  int lo, hi; // kernel band, signed DFT indices, B = hi - lo + 1 <= N
  int B;
  int Pm;     // mask half-spectrum extent max(-lo, hi)
  int P;      // intensity half extent: full ? n/2 : B-1
  int full;   // intensity band covers all n residues (then n == N, d == 1)
  int nb2;    // intensity band entries along the axis: full ? n : 2P+1
};

// signed intensity-band frequency of band slot j in [0, nb2)
__host__ __device__ inline int band2_p(const AxisGeom& a, int j) {
  if (a.full) return j <= a.n / 2 ? j : j - a.n;
  return j - a.P;
}

__host__ __device__ inline int wrapi(int p, int n) {
  int r = p % n;
  return r < 0 ? r + n : r;
}

// kernel-band slot of DFT residue r (mod N), or -1 when outside [lo, hi]
__host__ __device__ inline int band_slot(const AxisGeom& a, int r) {
  int s = wrapi(r, a.N);
  if (s > a.hi) s -= a.N;
  if (s < a.lo || s > a.hi) return -1;
  return s - a.lo;
}

}  // namespace lg
