// Device helpers shared by the owner-computes kernels (cmax_owner.cu,
// cmax_cells.cu): compressed splat records, warp-collective list/range utilities.
#pragma once

#include <cstdint>

#include "cmax_device.cuh"
#include "cmax_owner.h"

namespace evcm_b200 {
namespace owner_dev {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kDead = 0xffffffffu;
constexpr int kOwnPx = kOwnW * kOwnH;

// Bilinear fractions compressed to one float each with full relative precision
// on the smaller of (w, 1-w): f = w if w < 0.5 else -(1-w) (the sign bit marks
// the second form, so -0.0 encodes w = 1).
__device__ __forceinline__ float compress_frac(double w) {
  return w < 0.5 ? (float)w : -(float)(1.0 - w);
}
__device__ __forceinline__ void expand_frac(float f, double& w, double& a) {
  if (signbit(f)) {
    a = -(double)f;
    w = 1.0 - a;
  } else {
    w = (double)f;
    a = 1.0 - w;
  }
}

struct CellW {
  int x0, y0;
  double wx, wy, ax, ay;  // ax = 1 - wx, ay = 1 - wy
};

__device__ __forceinline__ CellW decode(const FwdRec& r) {
  CellW c;
  c.x0 = (int)(r.cell & 0xffffu);
  c.y0 = (int)((r.cell >> 16) & 0x7fffu);
  expand_frac(r.fx, c.wx, c.ax);
  expand_frac(r.fy, c.wy, c.ay);
  return c;
}



__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ int sort_tile_of(double x, double y, const WinParams& P,
                                            const TileParams& TP) {
  const double xm = (double)(P.W - 1), ym = (double)(P.H - 1);
  const double cx = x < 0.0 ? 0.0 : (xm < x ? xm : x);  // also maps NaN to 0 via the casts below
  const double cy = y < 0.0 ? 0.0 : (ym < y ? ym : y);
  int ix = (int)cx, iy = (int)cy;
  ix = ix < 0 ? 0 : (ix >= P.W ? P.W - 1 : ix);
  iy = iy < 0 ? 0 : (iy >= P.H ? P.H - 1 : iy);
  return (iy / kSortTile) * TP.ntx + ix / kSortTile;
}



// Warp-collective exclusive scan of per-entry lengths: pre[l] (l <= n), rng[l] =
// first slot of entry l, for entries [l0, l0 + n) of a concatenated list whose
// running total starts at `carry`. lohi(l) -> (first, end) slot of entry l.
template <typename F>
__device__ __forceinline__ uint32_t warp_ranges(int l0, int n, uint32_t carry, uint32_t* pre,
                                                uint32_t* rng, F&& lohi) {
  const int lane = threadIdx.x & 31;
  for (int b = 0; b < n; b += 32) {
    const int l = b + lane;
    uint32_t lo = 0, len = 0;
    if (l < n) {
      const uint2 r = lohi(l0 + l);
      lo = r.x;
      len = r.y - r.x;
    }
    uint32_t x = len;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (l < n) {
      pre[l0 + l] = carry + x - len;
      rng[l0 + l] = lo;
    }
    carry += __shfl_sync(kFull, x, 31);
  }
  if (lane == 0) pre[l0 + n] = carry;
  __syncwarp();
  return carry;
}


}  // namespace owner_dev

}  // namespace evcm_b200
