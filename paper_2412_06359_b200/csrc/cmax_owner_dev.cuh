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

__device__ __forceinline__ double corner_w(const CellW& c, int q) {
  return (q == 0) ? c.ax * c.ay : (q == 1) ? c.wx * c.ay : (q == 2) ? c.ax * c.wy : c.wx * c.wy;
}

// Lane-ordered accumulation of (v0, v1) into a warp-private shared tile: lanes
// sharing `key` are summed in lane order by the lowest of them, which then does
// a plain read-modify-write. key < 0: no contribution. Warp-collective.
__device__ __forceinline__ void warp_accumulate2(double* base, int key, double v0, double v1) {
  const unsigned act = __ballot_sync(kFull, key >= 0);
  if (key >= 0) {
    const unsigned peers = __match_any_sync(act, key);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    if (peers == (1u << lane)) {  // common case: no other lane on this pixel
      base[2 * key] += v0;
      base[2 * key + 1] += v1;
    } else {
      double s0 = 0.0, s1 = 0.0;
      if (lane == leader) {
        s0 = base[2 * key];
        s1 = base[2 * key + 1];
      }
      unsigned m = peers;
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const double a = __shfl_sync(peers, v0, src);
        const double b = __shfl_sync(peers, v1, src);
        s0 += a;
        s1 += b;
      }
      if (lane == leader) {
        base[2 * key] = s0;
        base[2 * key + 1] = s1;
      }
    }
  }
  __syncwarp();
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

// Scan every box of one slot (sort tiles, increasing) and call fn(S) for those
// whose cells can touch the owner rectangle [ox0, ox0+kOwnW) x [oy0, oy0+kOwnH).
// The slow path for overflowed owner lists. Warp-collective.
template <typename Fn>
__device__ __forceinline__ void scan_sources(const uint4* __restrict__ bbox, int nT, int ox0,
                                             int oy0, uint16_t* list, int cap, Fn&& fn) {
  const int lane = threadIdx.x & 31;
  const int lx = ox0 - 1, hx = ox0 + kOwnW - 1, ly = oy0 - 1, hy = oy0 + kOwnH - 1;
  int fill = 0;
  for (int s0 = 0; s0 < nT; s0 += 32) {
    const int S = s0 + lane;
    bool hit = false;
    if (S < nT) {
      const uint4 b = __ldg(bbox + S);
      if (b.x != 0xffffffffu) {
        const int mnx = (int)b.x, mny = (int)b.y;
        const int mxx = 0xffff - (int)b.z, mxy = 0xffff - (int)b.w;
        hit = !(mxx < lx || mnx > hx || mxy < ly || mny > hy);
      }
    }
    const unsigned hits = __ballot_sync(kFull, hit);
    if (hit) list[fill + __popc(hits & ((1u << lane) - 1u))] = (uint16_t)S;
    fill += __popc(hits);
    if (fill > cap - 32 || s0 + 32 >= nT) {
      __syncwarp();
      for (int i = 0; i < fill; ++i) fn((int)list[i]);
      __syncwarp();
      fill = 0;
    }
  }
}

// Sorted source list of one (window, slot, owner tile) into `list`; returns its
// length, or -1 when the precomputed list overflowed (the caller then scans).
// Warp-collective version: rank-sort the (unique) sources in parallel.
__device__ __forceinline__ int warp_load_sorted_list(const uint32_t* __restrict__ lcount,
                                                     const uint16_t* __restrict__ lists,
                                                     size_t slotT, uint16_t* list) {
  const int lane = threadIdx.x & 31;
  const uint32_t cnt = lcount[slotT];
  if (cnt > (uint32_t)kListCapO) return -1;
  const uint16_t* src = lists + slotT * kListCapO;
  for (uint32_t e = lane; e < cnt; e += 32) {
    const uint16_t v = src[e];
    int rank = 0;
    for (uint32_t q = 0; q < cnt; ++q) rank += src[q] < v ? 1 : 0;
    list[rank] = v;
  }
  __syncwarp();
  return (int)cnt;
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

// Virtual concatenation of event ranges: pre[l] = sum of earlier lengths,
// rng[l] = first slot of range l. Returns the slot of virtual index v.
__device__ __forceinline__ uint32_t virt_slot(const uint32_t* pre, const uint32_t* rng, int nl,
                                              uint32_t v, int* which) {
  int lo = 0, hi = nl - 1;  // largest l with pre[l] <= v
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= v) lo = mid; else hi = mid - 1;
  }
  *which = lo;
  return rng[lo] + (v - pre[lo]);
}

}  // namespace owner_dev

}  // namespace evcm_b200
