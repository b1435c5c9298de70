// Device helpers of the image kernels (raster.cu, composite.cu):
//  * raster_triangle: one triangle into the packed depth|scalar key buffer
//    (the raster step of K2, one thread per triangle) -- 16.8 fixed-point
//    edge functions with a top-left rule, sampling at pixel centres, depth
//    clipped to [0, 1], order-independent atomicMin;
//  * dec_ordered / cmap_channel: the colour-range decoding and the colormap.
// oracle/sem_oracle.c restates them operation for operation.
#pragma once

#include "checked.cuh"

#include <cuda_runtime.h>
#include <math.h>

#include "nkb_internal.h"

namespace nkb {
namespace rdev {

// inverse of the order-preserving encoding of doubles used by the colour-range words
__device__ __forceinline__ double dec_ordered(unsigned long long u) {
  unsigned long long b = (u & 0x8000000000000000ULL) ? (u & 0x7fffffffffffffffULL) : ~u;
  return __longlong_as_double((long long)b);
}

// np.interp on clipped t, then floor(v + 0.5) -> uint8 (sinks.py:201-209);
// shared by K3 resolve, the structured renderer and the P2P composite
__device__ __forceinline__ unsigned char cmap_channel(const Colormap& cm, double t, int ch) {
  if (t != t) return 0;
  const int n = cm.n;
  double v;
  if (t >= cm.t[n - 1]) {
    v = cm.rgb[n - 1][ch];
  } else {
    int j = 0;
    for (int k = 1; k < n - 1; ++k)
      if (t >= cm.t[k]) j = k;
    if (t == cm.t[j]) {
      v = cm.rgb[j][ch];
    } else {
      const double slope = cm.slope[j][ch];      // host-precomputed, same IEEE division
      v = __dadd_rn(__dmul_rn(slope, __dsub_rn(t, cm.t[j])), cm.rgb[j][ch]);
    }
  }
  return (unsigned char)floor(__dadd_rn(v, 0.5));
}


// all three channels with one anchor search (the per-channel arithmetic of
// cmap_channel, unchanged)
__device__ __forceinline__ uchar4 cmap_rgba(const Colormap& cm, double t) {
  if (t != t) return make_uchar4(0, 0, 0, 255);
  const int n = cm.n;
  unsigned char o[3];
  if (t >= cm.t[n - 1]) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) o[ch] = (unsigned char)floor(__dadd_rn(cm.rgb[n - 1][ch], 0.5));
  } else {
    int j = 0;
    for (int k = 1; k < n - 1; ++k)
      if (t >= cm.t[k]) j = k;
    const double tj = cm.t[j];
    const bool at = t == tj;
    const double dt = __dsub_rn(t, tj);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const double v = at ? cm.rgb[j][ch] : __dadd_rn(__dmul_rn(cm.slope[j][ch], dt), cm.rgb[j][ch]);
      o[ch] = (unsigned char)floor(__dadd_rn(v, 0.5));
    }
  }
  return make_uchar4(o[0], o[1], o[2], 255);
}

constexpr double kGuard = 32768.0;   // |screen coordinate| bound in pixels

__device__ __forceinline__ void xform(const double* V, double x, double y, double z, double& sx,
                                      double& sy, double& sz) {
  sx = __dadd_rn(__fma_rn(V[2], z, __fma_rn(V[1], y, __dmul_rn(V[0], x))), V[3]);
  sy = __dadd_rn(__fma_rn(V[6], z, __fma_rn(V[5], y, __dmul_rn(V[4], x))), V[7]);
  sz = __dadd_rn(__fma_rn(V[10], z, __fma_rn(V[9], y, __dmul_rn(V[8], x))), V[11]);
}

__device__ __forceinline__ long long floordiv(long long a, long long b) {  // b > 0
  long long q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}


// sub / nsub: this thread draws rows py0 + sub, py0 + sub + nsub, ... (nsub
// threads share a triangle; the edge values stay exact integers)
__device__ __forceinline__ void raster_triangle(const double* view, int W, int H, const float4* tri,
                                                unsigned long long* zbuf, int sub = 0, int nsub = 1) {
  long long X[3], Y[3];
  double Z[3], C[3];
  bool ok = true;
  const bool persp = view[12] != 0.0 || view[13] != 0.0 || view[14] != 0.0 || view[15] != 0.0;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const float4 v = tri[q];
    double sx, sy, sz;
    xform(view, (double)v.x, (double)v.y, (double)v.z, sx, sy, sz);
    if (persp) {                                   // perspective divide (w > 0 in front)
      const double* P = view + 12;
      const double w = __dadd_rn(__fma_rn(P[2], (double)v.z, __fma_rn(P[1], (double)v.y, __dmul_rn(P[0], (double)v.x))),
                                 P[3]);
      if (!(w > 0.0)) ok = false;
      sx = __ddiv_rn(sx, w);
      sy = __ddiv_rn(sy, w);
      sz = __ddiv_rn(sz, w);
    }
    if (!(fabs(sx) <= kGuard && fabs(sy) <= kGuard && sz == sz && v.w == v.w)) ok = false;
    X[q] = __double2ll_rn(__dmul_rn(sx, 256.0));
    Y[q] = __double2ll_rn(__dmul_rn(sy, 256.0));
    Z[q] = sz;
    C[q] = (double)v.w;
  }
  if (!ok) return;
  // the pixel-centre box first: most triangles of a fine mesh cover no pixel
  // centre and leave here, before the area, the edge set-up and 1 / area
  const long long xmin = min(X[0], min(X[1], X[2])), xmax = max(X[0], max(X[1], X[2]));
  const long long ymin = min(Y[0], min(Y[1], Y[2])), ymax = max(Y[0], max(Y[1], Y[2]));
  long long px0 = -floordiv(-(xmin - 128), 256), px1 = floordiv(xmax - 128, 256);
  long long py0 = -floordiv(-(ymin - 128), 256), py1 = floordiv(ymax - 128, 256);
  if (px0 < 0) px0 = 0;
  if (py0 < 0) py0 = 0;
  if (px1 > W - 1) px1 = W - 1;
  if (py1 > H - 1) py1 = H - 1;
  if (px0 > px1 || py0 > py1) return;
  long long area = (X[1] - X[0]) * (Y[2] - Y[0]) - (Y[1] - Y[0]) * (X[2] - X[0]);
  if (area == 0) return;
  if (area < 0) {
    long long tx = X[1]; X[1] = X[2]; X[2] = tx;
    long long ty = Y[1]; Y[1] = Y[2]; Y[2] = ty;
    double tz = Z[1]; Z[1] = Z[2]; Z[2] = tz;
    double tc = C[1]; C[1] = C[2]; C[2] = tc;
    area = -area;
  }
  // edge (a->b) opposite vertex i: w_i(P) = (Xb-Xa)(Py-Ya) - (Yb-Ya)(Px-Xa)
  const int ea[3] = {1, 2, 0}, eb[3] = {2, 0, 1};
  long long bias[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const long long dy = Y[eb[i]] - Y[ea[i]], dx = X[eb[i]] - X[ea[i]];
    bias[i] = (dy > 0 || (dy == 0 && dx < 0)) ? 0 : -1;   // inclusive (top-left) edges
  }
  const double inv = __drcp_rn((double)area);     // == 1.0 / area: one IEEE division per triangle
  // edge functions stepped incrementally: w_i(cx + 256) = w_i(cx) - 256 (Yb - Ya),
  // w_i(cy + 256) = w_i(cy) + 256 (Xb - Xa) -- exact int64, the same values as
  // evaluating w_i at every pixel centre
  long long dwx[3], dwy[3], wrow[3];
  {
    const long long cy0 = py0 * 256 + 128, cx0 = px0 * 256 + 128;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      dwx[i] = -(Y[eb[i]] - Y[ea[i]]) * 256;
      dwy[i] = (X[eb[i]] - X[ea[i]]) * 256;
      wrow[i] = (X[eb[i]] - X[ea[i]]) * (cy0 - Y[ea[i]]) - (Y[eb[i]] - Y[ea[i]]) * (cx0 - X[ea[i]]);
    }
  }
  if (nsub > 1) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      wrow[i] += (long long)sub * dwy[i];
      dwy[i] *= nsub;
    }
  }
  for (long long py = py0 + sub; py <= py1; py += nsub) {
    long long w[3] = {wrow[0], wrow[1], wrow[2]};
    for (long long px = px0; px <= px1; ++px) {
      if (w[0] + bias[0] >= 0 && w[1] + bias[1] >= 0 && w[2] + bias[2] >= 0) {
        double d = __dmul_rn(__fma_rn((double)w[2], Z[2],
                                      __fma_rn((double)w[1], Z[1], __dmul_rn((double)w[0], Z[0]))),
                             inv);
        if (d >= 0.0 && d <= 1.0) {
          d = __dadd_rn(d, 0.0);
          const double c = __dmul_rn(__fma_rn((double)w[2], C[2],
                                              __fma_rn((double)w[1], C[1], __dmul_rn((double)w[0], C[0]))),
                                     inv);
          const unsigned long long key =
              ((unsigned long long)__float_as_uint(__double2float_rn(d)) << 32) |
              (unsigned long long)__float_as_uint(__double2float_rn(c));
          NKB_DCHECK(px >= 0 && px < W && py >= 0 && py < H);
          atomicMin(zbuf + py * W + px, key);
        }
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) w[i] += dwx[i];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) wrow[i] += dwy[i];
  }
}

}  // namespace rdev
}  // namespace nkb
