// Marching-squares contours of a resist image and EPE gauges on the GPU.
//
// Reference: marching_squares (proj/src/core/contour.cpp:58-168) and
// measure_epe (contour.cpp:181-201) over SegmentBvh::nearest_crossing
// (proj/src/core/bvh.cpp:241-273).  The reference walks the cells serially,
// keeps the crossings in a std::map keyed by grid-edge id and stitches loops
// from the smallest edge id.  Here:
//   1. one thread per cell computes the crossings with the reference's fp64
//      arithmetic (explicit round-to-nearest ops: no FMA contraction, as the
//      reference's x86-64 build) and writes succ[from_edge] = to_edge and the
//      crossing point of from_edge (every crossing edge is the "from" side of
//      exactly one cell of a closed contour, so the writes never race);
//   2. the crossing edges are compacted in edge-id order (device scan);
//   3. loops are found by pointer jumping: the minimum edge id of each cycle
//      (its canonical start), then every crossing's distance from that start;
//   4. loops are laid out in ascending start-edge order, points in chain order
//      from the start: exactly the reference's ContourSet, bit for bit.
// EPE: every contour segment lies inside the cell that emitted it, so a gauge
// only has to test the crossing edges of the cells its probe line
// [p - r d, p + r d] can reach (a box of cells, one warp per gauge), with the
// reference's t / u arithmetic and its tie rule (smallest |t|, +t on ties).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lg {

struct CGeo {
  int nx, ny;
  double pitch, ox, oy;
  long long nh;  // horizontal edges (nx-1)*ny; vertical ids follow
};

__device__ __forceinline__ double c_node_x(const CGeo& g, int ix) {
  return __dadd_rn(g.ox, __dmul_rn(__dadd_rn(double(ix), 0.5), g.pitch));
}
__device__ __forceinline__ double c_node_y(const CGeo& g, int iy) {
  return __dadd_rn(g.oy, __dmul_rn(__dadd_rn(double(iy), 0.5), g.pitch));
}
__device__ __forceinline__ long long h_edge(const CGeo& g, int ix, int iy) {
  return (long long)iy * (g.nx - 1) + ix;
}
__device__ __forceinline__ long long v_edge(const CGeo& g, int ix, int iy) {
  return g.nh + (long long)iy * g.nx + ix;
}

// per-block min / max / non-finite flag of the field (reference :62-70)
__global__ void k_field_minmax(const double* __restrict__ f, long long n, double* __restrict__ bmin,
                               double* __restrict__ bmax, int* __restrict__ nonfinite) {
  __shared__ double smin[256], smax[256];
  double lo = f[0], hi = f[0];
  bool bad = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = f[i];
    bad |= !isfinite(v);
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  if (bad) atomicOr(nonfinite, 1);
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (int(threadIdx.x) < h) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + h]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + h]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bmin[blockIdx.x] = smin[0];
    bmax[blockIdx.x] = smax[0];
  }
}

struct CCross {
  long long edge;
  double x, y;    // crossing point
  double ix, iy;  // inside node
};

// final min / max of the block partials: mm[0] = min, mm[1] = max
__global__ void k_field_minmax_final(const double* __restrict__ bmin, const double* __restrict__ bmax, int nblk,
                                     double* __restrict__ mm) {
  if (threadIdx.x != 0) return;
  double lo = bmin[0], hi = bmax[0];
  for (int b = 1; b < nblk; ++b) {
    lo = fmin(lo, bmin[b]);
    hi = fmax(hi, bmax[b]);
  }
  mm[0] = lo;
  mm[1] = hi;
}

// one thread per cell (reference :90-139)
__global__ void k_ms_cells(CGeo g, const double* __restrict__ f, double thr, const double* __restrict__ mm,
                           int* __restrict__ succ, double2* __restrict__ pt, int* __restrict__ dup) {
  const int ix = blockIdx.x * blockDim.x + threadIdx.x, iy = blockIdx.y * blockDim.y + threadIdx.y;
  if (ix + 1 >= g.nx || iy + 1 >= g.ny) return;
  const double vmin = mm[0], vmax = mm[1];
  const double eps = __dmul_rn(fmax(__dadd_rn(vmax, -vmin), 1.0), 1e-12);
  auto val = [&](int x, int y) {
    const double v = f[(size_t)y * g.nx + x];
    return v == thr ? __dadd_rn(v, eps) : v;  // +eps symbolic perturbation (:71-74)
  };
  const double v00 = val(ix, iy), v10 = val(ix + 1, iy), v01 = val(ix, iy + 1), v11 = val(ix + 1, iy + 1);
  const bool i00 = v00 > thr, i10 = v10 > thr, i01 = v01 > thr, i11 = v11 > thr;
  if (i00 == i10 && i10 == i11 && i11 == i01) return;
  const double x0 = c_node_x(g, ix), x1 = c_node_x(g, ix + 1), y0 = c_node_y(g, iy), y1 = c_node_y(g, iy + 1);
  auto cross = [&](double va, double vb, double pax, double pay, double pbx, double pby, bool ina, long long e) {
    const double t = __ddiv_rn(__dadd_rn(thr, -va), __dadd_rn(vb, -va));
    CCross c;
    c.edge = e;
    c.x = __dadd_rn(pax, __dmul_rn(t, __dadd_rn(pbx, -pax)));
    c.y = __dadd_rn(pay, __dmul_rn(t, __dadd_rn(pby, -pay)));
    c.ix = ina ? pax : pbx;
    c.iy = ina ? pay : pby;
    return c;
  };
  CCross side[4];
  bool has[4] = {i00 != i10, i10 != i11, i01 != i11, i00 != i01};
  if (has[0]) side[0] = cross(v00, v10, x0, y0, x1, y0, i00, h_edge(g, ix, iy));
  if (has[1]) side[1] = cross(v10, v11, x1, y0, x1, y1, i10, v_edge(g, ix + 1, iy));
  if (has[2]) side[2] = cross(v01, v11, x0, y1, x1, y1, i01, h_edge(g, ix, iy + 1));
  if (has[3]) side[3] = cross(v00, v01, x0, y0, x0, y1, i00, v_edge(g, ix, iy));
  // direct so the inside node of the source lies on the left (:84-91)
  auto emit = [&](const CCross& a, const CCross& b) {
    const CCross* from = &a;
    const CCross* to = &b;
    const double c = __dadd_rn(__dmul_rn(__dadd_rn(to->x, -from->x), __dadd_rn(from->iy, -from->y)),
                               -__dmul_rn(__dadd_rn(to->y, -from->y), __dadd_rn(from->ix, -from->x)));
    if (c < 0) {
      const CCross* s = from;
      from = to;
      to = s;
    }
    if (atomicExch(succ + from->edge, int(to->edge)) >= 0) atomicOr(dup, 1);
    pt[from->edge] = make_double2(from->x, from->y);
  };
  const int count = has[0] + has[1] + has[2] + has[3];
  if (count == 2) {
    int k[2], m = 0;
    for (int s = 0; s < 4; ++s)
      if (has[s]) k[m++] = s;
    emit(side[k[0]], side[k[1]]);
  } else if (count == 4) {  // saddle (:124-136)
    const double center = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(v00, v10), v01), v11));
    const bool center_in = center == thr ? true : center > thr;
    const bool corner_in[4] = {i00, i10, i11, i01};
    const int cs[4][2] = {{0, 3}, {0, 1}, {2, 1}, {2, 3}};
    for (int corner = 0; corner < 4; ++corner)
      if (corner_in[corner] != center_in) emit(side[cs[corner][0]], side[cs[corner][1]]);
  }
}

__global__ void k_ms_flags(const int* __restrict__ succ, long long ne, int* __restrict__ flag) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ne; e += (long long)gridDim.x * blockDim.x)
    flag[e] = succ[e] >= 0;
}

// compacted crossing list in edge order; idx[e] = compact index (or -1)
__global__ void k_ms_compact(const int* __restrict__ succ, const int* __restrict__ pos, long long ne,
                             int* __restrict__ cedge, int* __restrict__ idx) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ne; e += (long long)gridDim.x * blockDim.x) {
    if (succ[e] >= 0) {
      cedge[pos[e]] = int(e);
      idx[e] = pos[e];
    } else {
      idx[e] = -1;
    }
  }
}

// csucc[i] = compact successor; m[i] = own edge id; broken chains flagged
__global__ void k_ms_link(const int* __restrict__ cedge, const int* __restrict__ succ, const int* __restrict__ idx,
                          int n, int* __restrict__ csucc, int* __restrict__ m, int* __restrict__ broken) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = idx[succ[cedge[i]]];
  if (s < 0) atomicOr(broken, 1);
  csucc[i] = s < 0 ? i : s;
  m[i] = cedge[i];
}

// pointer jumping: cycle minimum of the edge ids
__global__ void k_ms_minjump(const int* __restrict__ m0, const int* __restrict__ j0, int n, int* __restrict__ m1,
                             int* __restrict__ j1) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = j0[i];
  m1[i] = min(m0[i], m0[j]);
  j1[i] = j0[j];
}

// list for ranking: the cycle is cut in front of its start
__global__ void k_ms_rank_init(const int* __restrict__ csucc, const int* __restrict__ cedge, const int* __restrict__ m,
                               int n, int* __restrict__ nxt, int* __restrict__ d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = csucc[i];
  const bool last = cedge[s] == m[i];
  nxt[i] = last ? -1 : s;
  d[i] = last ? 0 : 1;
}

__global__ void k_ms_rank_jump(const int* __restrict__ n0, const int* __restrict__ d0, int n, int* __restrict__ n1,
                               int* __restrict__ d1) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = n0[i];
  if (j < 0) {
    n1[i] = -1;
    d1[i] = d0[i];
  } else {
    n1[i] = n0[j];
    d1[i] = d0[i] + d0[j];
  }
}

// loop starts and their lengths (d[start] = length - 1)
__global__ void k_ms_starts(const int* __restrict__ cedge, const int* __restrict__ m, const int* __restrict__ d,
                            int n, int* __restrict__ isstart, int* __restrict__ len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool st = cedge[i] == m[i];
  isstart[i] = st;
  len[i] = st ? d[i] + 1 : 0;
}

// scatter points: loop of i = loop index of its start, position = d[start] - d[i]
__global__ void k_ms_scatter(const int* __restrict__ cedge, const int* __restrict__ m, const int* __restrict__ idx,
                             const int* __restrict__ d, const long long* __restrict__ pt_off,
                             const double2* __restrict__ pt, int n, double* __restrict__ xs,
                             double* __restrict__ ys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = idx[m[i]];
  const long long o = pt_off[s] + (d[s] - d[i]);
  const double2 p = pt[cedge[i]];
  xs[o] = p.x;
  ys[o] = p.y;
}

// loop offsets (prefix of lengths over starts, in start order)
__global__ void k_ms_offsets(const int* __restrict__ isstart, const int* __restrict__ loop_idx,
                             const long long* __restrict__ pt_off, int n, long long* __restrict__ offsets,
                             long long total) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && isstart[i]) offsets[loop_idx[i]] = pt_off[i];
  if (i == 0) offsets[loop_idx[n - 1] + isstart[n - 1]] = total;
}

// ---- EPE: one warp per gauge ----------------------------------------------
struct Gauge {
  double x, y, nx, ny;
};

__device__ __forceinline__ bool epe_better(double t, double best, bool have) {
  const double at = fabs(t), ab = fabs(best);
  return !have || at < ab || (at == ab && t > best);
}

__global__ void k_epe(CGeo g, const int* __restrict__ succ, const double2* __restrict__ pt, int ncross,
                      const Gauge* __restrict__ gauges, int ng, double r, double* __restrict__ epe,
                      unsigned char* __restrict__ open) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= ng) return;
  const Gauge q = gauges[warp];
  bool have = false;
  double best = 0.0;
  if (ncross > 0 && r > 0.0) {
    // cells whose box can hold a crossing of the probe within |t| <= r
    const double ex = fabs(q.nx) * r, ey = fabs(q.ny) * r;
    const int cx0 = max(0, int(floor((q.x - ex - g.ox) / g.pitch - 0.5)) - 1);
    const int cx1 = min(g.nx - 2, int(floor((q.x + ex - g.ox) / g.pitch - 0.5)) + 1);
    const int cy0 = max(0, int(floor((q.y - ey - g.oy) / g.pitch - 0.5)) - 1);
    const int cy1 = min(g.ny - 2, int(floor((q.y + ey - g.oy) / g.pitch - 0.5)) + 1);
    const int w = cx1 - cx0 + 1, h = cy1 - cy0 + 1;
    if (w > 0 && h > 0) {
      const long long cells = (long long)w * h;
      for (long long c = lane; c < cells; c += 32) {
        const int ix = cx0 + int(c % w), iy = cy0 + int(c / w);
        const long long es[4] = {h_edge(g, ix, iy), v_edge(g, ix + 1, iy), h_edge(g, ix, iy + 1), v_edge(g, ix, iy)};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int to = succ[es[k]];
          if (to < 0) continue;
          const double2 a = pt[es[k]], b = pt[to];
          // reference bvh.cpp:262-270
          const double sx = __dadd_rn(b.x, -a.x), sy = __dadd_rn(b.y, -a.y);
          const double denom = __dadd_rn(__dmul_rn(q.nx, sy), -__dmul_rn(q.ny, sx));
          if (denom == 0.0) continue;
          const double rx = __dadd_rn(a.x, -q.x), ry = __dadd_rn(a.y, -q.y);
          const double t = __ddiv_rn(__dadd_rn(__dmul_rn(rx, sy), -__dmul_rn(ry, sx)), denom);
          const double u = __ddiv_rn(__dadd_rn(__dmul_rn(rx, q.ny), -__dmul_rn(ry, q.nx)), denom);
          if (u < 0.0 || u > 1.0) continue;
          if (fabs(t) > r) continue;
          if (epe_better(t, best, have)) {
            best = t;
            have = true;
          }
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_down_sync(0xffffffffu, best, o);
    const bool oh = __shfl_down_sync(0xffffffffu, have, o);
    if (oh && epe_better(ob, best, have)) {
      best = ob;
      have = true;
    }
  }
  if (lane == 0) {
    epe[warp] = have ? best : 0.0;
    open[warp] = have ? 0 : 1;
  }
}

// EPE against an arbitrary segment list (ContourSet not produced by the GPU
// marching squares): one warp per gauge scans every segment (x0, y0, x1, y1)
// with the same arithmetic and tie rule as k_epe.
__global__ void k_epe_segments(const double4* __restrict__ segs, long long ns, const Gauge* __restrict__ gauges,
                               int ng, double r, double* __restrict__ epe, unsigned char* __restrict__ open) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= ng) return;
  const Gauge q = gauges[warp];
  bool have = false;
  double best = 0.0;
  if (r > 0.0) {
    for (long long k = lane; k < ns; k += 32) {
      const double4 s = segs[k];
      const double sx = __dadd_rn(s.z, -s.x), sy = __dadd_rn(s.w, -s.y);
      const double denom = __dadd_rn(__dmul_rn(q.nx, sy), -__dmul_rn(q.ny, sx));
      if (denom == 0.0) continue;
      const double rx = __dadd_rn(s.x, -q.x), ry = __dadd_rn(s.y, -q.y);
      const double t = __ddiv_rn(__dadd_rn(__dmul_rn(rx, sy), -__dmul_rn(ry, sx)), denom);
      const double u = __ddiv_rn(__dadd_rn(__dmul_rn(rx, q.ny), -__dmul_rn(ry, q.nx)), denom);
      if (u < 0.0 || u > 1.0 || fabs(t) > r) continue;
      if (epe_better(t, best, have)) {
        best = t;
        have = true;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_down_sync(0xffffffffu, best, o);
    const bool oh = __shfl_down_sync(0xffffffffu, have, o);
    if (oh && epe_better(ob, best, have)) {
      best = ob;
      have = true;
    }
  }
  if (lane == 0) {
    epe[warp] = have ? best : 0.0;
    open[warp] = have ? 0 : 1;
  }
}

}  // namespace lg
