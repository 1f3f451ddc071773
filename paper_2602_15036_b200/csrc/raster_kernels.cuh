// Bit-exact fp64 rasterization (sm_100a) of a healed polygon layer.
//
// Reference: rasterize_layer, proj/src/core/raster.cpp:53-95 (poly_area
// :17-25, clip_axis :31-49).  The reference walks polygons in healed order,
// clips each to a pixel row (y >= iy, then y <= iy+1), then to each cell
// (x >= ix, then x <= ix+1) with Sutherland-Hodgman, and adds the shoelace
// area into pix[iy*nx+ix]; finally clamps to [0,1].
//
// GPU formulation: one thread per pixel.  Polygons are binned into 32x32
// pixel bins in polygon order (ordered compaction, no atomics), and each
// pixel thread walks its bin list in order, streaming the polygon through the
// same four clip stages and the shoelace accumulator in registers (identical
// vertex order and arithmetic, so identical rounding), and accumulates the
// per-polygon areas in the reference's polygon order.  All floating-point
// operations are explicit round-to-nearest intrinsics: no FMA contraction
// (the reference's x86-64 build emits none).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lg {

constexpr int kRasterBin = 32;

// --- stage 0: vertices to pixel units + clamped bbox (raster.cpp:62-81) ---
// Axis-aligned rectangles also get their pixel-unit bounds and orientation:
// a pixel box lying inside such a rectangle clips (raster.cpp:31-49) to its
// own four integer corners (every intersection is computed along an
// axis-parallel edge, so it is exact), whose shoelace sum is exactly +-2, i.e.
// the reference adds exactly +-1.0 -- k_raster_pixels adds that directly.
__global__ void k_raster_prep(const int64_t* __restrict__ xy, const int64_t* __restrict__ starts,
                              int npoly, double scale, double ox, double oy, double pitch, int nx,
                              int ny, double* __restrict__ vx, double* __restrict__ vy,
                              int4* __restrict__ bbox, double4* __restrict__ rect,
                              double* __restrict__ rsign) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npoly) return;
  const int64_t v0 = starts[p], v1 = starts[p + 1];
  double sg = 0.0;
  if (v1 - v0 == 4) {
    const int64_t* q = xy + 2 * v0;  // (x0,y0) .. (x3,y3)
    const bool a = q[0] == q[2] && q[3] == q[5] && q[4] == q[6] && q[7] == q[1];
    const bool b = q[1] == q[3] && q[2] == q[4] && q[5] == q[7] && q[6] == q[0];
    if ((a || b) && q[0] != q[4] && q[1] != q[5]) {
      // orientation: sign of the cross product of the first two edges
      const double e1x = double(q[2] - q[0]), e1y = double(q[3] - q[1]);
      const double e2x = double(q[4] - q[2]), e2y = double(q[5] - q[3]);
      sg = (e1x * e2y - e1y * e2x) > 0 ? 1.0 : -1.0;
    }
  }
  int4 bb = make_int4(1, 0, 1, 0);  // empty: ix0 > ix1
  if (v1 - v0 >= 3) {
    double minx = 1e300, maxx = -1e300, miny = 1e300, maxy = -1e300;
    for (int64_t v = v0; v < v1; ++v) {
      const double x = __ddiv_rn(__dsub_rn(__dmul_rn(double(xy[2 * v]), scale), ox), pitch);
      const double y = __ddiv_rn(__dsub_rn(__dmul_rn(double(xy[2 * v + 1]), scale), oy), pitch);
      vx[v] = x;
      vy[v] = y;
      minx = fmin(minx, x);
      maxx = fmax(maxx, x);
      miny = fmin(miny, y);
      maxy = fmax(maxy, y);
    }
    int iy0 = int(floor(miny)), iy1 = int(ceil(maxy));
    int ix0 = int(floor(minx)), ix1 = int(ceil(maxx));
    iy0 = iy0 < 0 ? 0 : iy0;
    ix0 = ix0 < 0 ? 0 : ix0;
    iy1 = iy1 > ny - 1 ? ny - 1 : iy1;
    ix1 = ix1 > nx - 1 ? nx - 1 : ix1;
    bb = make_int4(ix0, ix1, iy0, iy1);
    rect[p] = make_double4(minx, maxx, miny, maxy);
  }
  bbox[p] = bb;
  rsign[p] = sg;
}

__device__ __forceinline__ bool bb_hits_bin(int4 bb, int bx, int by) {
  const int x0 = bx * kRasterBin, x1 = x0 + kRasterBin - 1;
  const int y0 = by * kRasterBin, y1 = y0 + kRasterBin - 1;
  return bb.x <= bb.y && bb.z <= bb.w && bb.x <= x1 && bb.y >= x0 && bb.z <= y1 && bb.w >= y0;
}

// --- stage 1: per-bin ordered polygon lists (count, then fill) ------------
// one CTA (256 threads) per bin; polygons scanned in order in chunks of 256
template <bool FILL>
__global__ void k_raster_bin(const int4* __restrict__ bbox, int npoly, int nbx,
                             int* __restrict__ counts, const int* __restrict__ offsets,
                             int* __restrict__ lists) {
  __shared__ int warp_tot[8];
  const int bin = blockIdx.x;
  const int bx = bin % nbx, by = bin / nbx;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int base = FILL ? offsets[bin] : 0;
  int total = 0;
  for (int c = 0; c < npoly; c += 256) {
    const int p = c + threadIdx.x;
    const bool hit = p < npoly && bb_hits_bin(bbox[p], bx, by);
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) warp_tot[wid] = __popc(m);
    __syncthreads();
    int before = 0, chunk = 0;
    for (int w = 0; w < 8; ++w) {
      if (w < wid) before += warp_tot[w];
      chunk += warp_tot[w];
    }
    if (FILL && hit) lists[base + total + before + __popc(m & ((1u << lane) - 1u))] = p;
    total += chunk;
    __syncthreads();
  }
  if (!FILL && threadIdx.x == 0) counts[bin] = total;
}

// --- stage 2: streaming Sutherland-Hodgman chain + shoelace ---------------
struct ShState {
  double fx, fy, px, py;  // first and previous vertex
  double fd, pd;          // their signed distances
  int n;                  // vertices received
  int out;                // vertices emitted
};

struct AreaState {
  double fx, fy, px, py, a;
  int n;
};

struct ClipChain {
  double b[4];  // bounds: y >= iy, y <= iy+1, x >= ix, x <= ix+1
  ShState s[4];
  AreaState ar;

  __device__ __forceinline__ void init(int ix, int iy) {
    b[0] = double(iy);
    b[1] = double(iy + 1);
    b[2] = double(ix);
    b[3] = double(ix + 1);
#pragma unroll
    for (int i = 0; i < 4; ++i) s[i].n = s[i].out = 0;
    ar.n = 0;
    ar.a = 0.0;
  }

  __device__ __forceinline__ void area_push(double x, double y) {
    if (ar.n == 0) {
      ar.fx = x;
      ar.fy = y;
    } else {
      // raster.cpp:22  a += x0 * y1 - x1 * y0
      ar.a = __dadd_rn(ar.a, __dsub_rn(__dmul_rn(ar.px, y), __dmul_rn(x, ar.py)));
    }
    ar.px = x;
    ar.py = y;
    ++ar.n;
  }
  __device__ __forceinline__ void area_finish() {
    if (ar.n > 0)
      ar.a = __dadd_rn(ar.a, __dsub_rn(__dmul_rn(ar.px, ar.fy), __dmul_rn(ar.fx, ar.py)));
  }

  template <int S>
  __device__ __forceinline__ void emit(double x, double y) {
    if constexpr (S == 4) {
      area_push(x, y);
    } else {
      ++s[S - 1].out;  // count outputs of stage S-1
      push<S>(x, y);
    }
  }

  // raster.cpp:36-47 for edge (prev -> cur); stage S: axis = S < 2 ? y : x,
  // sign = even S ? +1 : -1
  template <int S>
  __device__ __forceinline__ void edge(double x0, double y0, double d0, double x1, double y1,
                                       double d1) {
    if (d0 >= 0) emit<S + 1>(x0, y0);
    if ((d0 >= 0) != (d1 >= 0)) {
      const double t = __ddiv_rn(d0, __dsub_rn(d0, d1));
      if (S >= 2)
        emit<S + 1>(b[S], __dadd_rn(y0, __dmul_rn(t, __dsub_rn(y1, y0))));
      else
        emit<S + 1>(__dadd_rn(x0, __dmul_rn(t, __dsub_rn(x1, x0))), b[S]);
    }
  }

  template <int S>
  __device__ __forceinline__ void push(double x, double y) {
    if constexpr (S == 4) {
      area_push(x, y);
    } else {
      const double sign = (S % 2 == 0) ? 1.0 : -1.0;
      const double d = __dmul_rn(sign, __dsub_rn(S >= 2 ? x : y, b[S]));
      ShState& st = s[S];
      if (st.n == 0) {
        st.fx = x;
        st.fy = y;
        st.fd = d;
      } else {
        edge<S>(st.px, st.py, st.pd, x, y, d);
      }
      st.px = x;
      st.py = y;
      st.pd = d;
      ++st.n;
    }
  }

  template <int S>
  __device__ __forceinline__ void finish() {
    if constexpr (S == 4) {
      area_finish();
    } else {
      ShState& st = s[S];
      if (st.n > 0) edge<S>(st.px, st.py, st.pd, st.fx, st.fy, st.fd);
      finish<S + 1>();
    }
  }
};

// emit<S> counts into s[S-1].out for S in 1..3; stage 3's outputs go to the
// area accumulator (ar.n).  Row polygon size = s[1].out, cell size = ar.n.

// Pixel value: every polygon of the pixel's bin in order (raster.cpp:83-93).
// EXACT_ONLY: only pixels whose polygons all take the exact shortcut (outside
// the bbox, or inside a rectangle) are finished here; the others set
// slow[pix] and are finished by the full clip pass over their compacted list,
// so no warp carries a clip chain for a few edge pixels.
template <bool EXACT_ONLY>
__device__ __forceinline__ bool raster_pixel(int ix, int iy, const double* __restrict__ vx,
                                             const double* __restrict__ vy, const int64_t* __restrict__ starts,
                                             const int4* __restrict__ bbox, const double4* __restrict__ rect,
                                             const double* __restrict__ rsign, const int* __restrict__ offsets,
                                             const int* __restrict__ counts, const int* __restrict__ lists,
                                             int nbx, double& pix) {
  const int bin = (iy / kRasterBin) * nbx + ix / kRasterBin;
  const int o = offsets[bin], c = counts[bin];
  pix = 0.0;
  for (int i = 0; i < c; ++i) {
    const int p = lists[o + i];
    const int4 bb = bbox[p];
    if (ix < bb.x || ix > bb.y || iy < bb.z || iy > bb.w) continue;
    const double sg = rsign[p];
    if (sg != 0.0) {
      const double4 r = rect[p];
      if (r.x <= double(ix) && r.y >= double(ix + 1) && r.z <= double(iy) && r.w >= double(iy + 1)) {
        pix = __dadd_rn(pix, sg);  // == pix + 0.5 * (+-2): the exact clipped unit square
        continue;
      }
    }
    if (EXACT_ONLY) return false;
    ClipChain ch;
    ch.init(ix, iy);
    const int64_t v0 = starts[p], v1 = starts[p + 1];
    for (int64_t v = v0; v < v1; ++v) ch.push<0>(vx[v], vy[v]);
    ch.finish<0>();
    if (ch.s[1].out < 3) continue;  // raster.cpp:85 row polygon degenerate
    if (ch.ar.n < 3) continue;      // raster.cpp:88 cell polygon degenerate
    pix = __dadd_rn(pix, __dmul_rn(0.5, ch.ar.a));  // raster.cpp:24,89
  }
  return true;
}

__device__ __forceinline__ double raster_clamp(double pix) {
  return pix < 0.0 ? 0.0 : (pix > 1.0 ? 1.0 : pix);  // raster.cpp:93
}

// pass 1: all pixels; exact-shortcut pixels are written, the rest flagged
__global__ void k_raster_pixels(const double* __restrict__ vx, const double* __restrict__ vy,
                                const int64_t* __restrict__ starts, const int4* __restrict__ bbox,
                                const double4* __restrict__ rect, const double* __restrict__ rsign,
                                const int* __restrict__ offsets, const int* __restrict__ counts,
                                const int* __restrict__ lists, int nx, int ny, int nbx,
                                double* __restrict__ out, int* __restrict__ slow) {
  const int ix = blockIdx.x * blockDim.x + threadIdx.x;
  const int iy = blockIdx.y * blockDim.y + threadIdx.y;
  if (ix >= nx || iy >= ny) return;
  double pix;
  const bool done = raster_pixel<true>(ix, iy, vx, vy, starts, bbox, rect, rsign, offsets, counts, lists, nbx, pix);
  const size_t o = size_t(iy) * nx + ix;
  slow[o] = done ? 0 : 1;
  if (done) out[o] = raster_clamp(pix);
}

// pass 2: the flagged pixels (compacted list), full ordered clip chain
__global__ void k_raster_pixels_slow(const double* __restrict__ vx, const double* __restrict__ vy,
                                     const int64_t* __restrict__ starts, const int4* __restrict__ bbox,
                                     const double4* __restrict__ rect, const double* __restrict__ rsign,
                                     const int* __restrict__ offsets, const int* __restrict__ counts,
                                     const int* __restrict__ lists, int nx, int nbx,
                                     const int* __restrict__ slow_list, const int* __restrict__ nslow,
                                     double* __restrict__ out) {
  const int n = *nslow;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int q = slow_list[i];
    const int ix = q % nx, iy = q / nx;
    double pix;
    raster_pixel<false>(ix, iy, vx, vy, starts, bbox, rect, rsign, offsets, counts, lists, nbx, pix);
    out[q] = raster_clamp(pix);
  }
}

}  // namespace lg
