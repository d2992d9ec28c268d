// Device primitives of the CMax loss path (sm_100a).
//
// Every position / weight / flow expression uses explicit round-to-nearest
// fp64 intrinsics (__dadd_rn, __dmul_rn, ...) in the reference's evaluation
// order, which forbids FMA contraction: trajectories, bilinear weights, the
// motion field, bin indices and the alive mask are therefore BIT-IDENTICAL to
// the reference (warp.hpp, geometry.hpp), and only the scatter-add order of
// the IWE stack and the gradient buffer differs (atomics / tiles vs the
// reference's event order).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace evcm_b200 {

constexpr int kMaxBins = 32;
constexpr int kMaxRefs = kMaxBins + 1;
constexpr double kLossEps = 1e-9;  // warp.hpp:26

// Window geometry shared by every window of a batch (kernel parameter).
struct WinParams {
  int W, H, B;       // sensor size, number of flow bins
  int HW;            // W*H
  int n_windows;
  double window_s;   // edges_s[B] (engine.hpp:380)
  double inv_window; // 1 / window_s: owner kernels form tb = |t - e_r| * inv_window in the
                     // forward AND the backward, so count/tsum cancel exactly as in fp64
  double es[kMaxRefs];      // edge times on the window clock, s (engine.hpp:244-249)
  uint32_t erel[kMaxRefs];  // edges_us[i] - edges_us[0]
  uint64_t t0, t_end;       // slice window [t0, t_end) of window 0
  uint64_t stride_us;       // window w spans [t0, t_end) + w * stride_us
};

// Packed event, 8 B: x = (t_us - t0) | (negative polarity << 31), y = x | y << 16.
__device__ __forceinline__ uint32_t ev_dt(uint2 e) { return e.x & 0x7fffffffu; }
__device__ __forceinline__ int ev_pol(uint2 e) { return (int)(e.x >> 31); }  // polarity_index
__device__ __forceinline__ int ev_x(uint2 e) { return (int)(e.y & 0xffffu); }
__device__ __forceinline__ int ev_y(uint2 e) { return (int)(e.y >> 16); }

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }

// bin_of (warp.hpp:284-288) in integer form: largest j with edges_us[j] <= t,
// clamped to [0, B-1]. Exact: (t - t0)*1e-6 is monotone and injective on
// the microsecond integers involved.
__device__ __forceinline__ int bin_of(uint32_t dt, const uint32_t* erel, int B) {
  int j = 0;
  for (int i = 1; i < B; ++i) j += (erel[i] <= dt) ? 1 : 0;
  return j;
}

// bilin_cell (warp.hpp:42-53). `i00` is the flat index of (x0, y0); `ox` and
// `oy` are the flat offsets to x1 and y1 (0 when the sensor is 1 px wide/high).
struct Cell {
  int i00, ox, oy;
  int x0, y0;
  double wx, wy;
};

__device__ __forceinline__ Cell bilin_cell(double x, double y, int W, int H) {
  const double xm = (double)(W - 1), ym = (double)(H - 1);
  // std::clamp(v, lo, hi) == v < lo ? lo : (hi < v ? hi : v)
  const double cx = x < 0.0 ? 0.0 : (xm < x ? xm : x);
  const double cy = y < 0.0 ? 0.0 : (ym < y ? ym : y);
  int x0 = 0, y0 = 0;
  if (W >= 2) { x0 = (int)floor(cx); x0 = x0 < W - 2 ? x0 : W - 2; }
  if (H >= 2) { y0 = (int)floor(cy); y0 = y0 < H - 2 ? y0 : H - 2; }
  Cell c;
  c.x0 = x0;
  c.y0 = y0;
  c.i00 = y0 * W + x0;
  c.ox = (x0 + 1 < W - 1 ? x0 + 1 : W - 1) - x0;
  c.oy = ((y0 + 1 < H - 1 ? y0 + 1 : H - 1) - y0) * W;
  c.wx = ds(cx, (double)x0);
  c.wy = ds(cy, (double)y0);
  return c;
}

// in_bounds (warp.hpp:55-57)
__device__ __forceinline__ bool in_bounds(double x, double y, int W, int H) {
  return x >= 0.0 && x <= (double)(W - 1) && y >= 0.0 && y <= (double)(H - 1);
}

// Bilinear weights w00, w10, w01, w11 (warp.hpp:36-39).
struct Weights {
  double w00, w10, w01, w11;
};
__device__ __forceinline__ Weights weights(const Cell& c) {
  const double ax = ds(1.0, c.wx), ay = ds(1.0, c.wy);
  return {dm(ax, ay), dm(c.wx, ay), dm(ax, c.wy), dm(c.wx, c.wy)};
}

// sample_flow (warp.hpp:61-68) on an interleaved (u, v) plane.
__device__ __forceinline__ double2 sample_flow(const double2* __restrict__ f, const Cell& c) {
  const Weights w = weights(c);
  const double2 a = __ldg(f + c.i00);
  const double2 b = __ldg(f + c.i00 + c.ox);
  const double2 d = __ldg(f + c.i00 + c.oy);
  const double2 e = __ldg(f + c.i00 + c.oy + c.ox);
  double2 r;
  r.x = da(da(da(dm(w.w00, a.x), dm(w.w10, b.x)), dm(w.w01, d.x)), dm(w.w11, e.x));
  r.y = da(da(da(dm(w.w00, a.y), dm(w.w10, b.y)), dm(w.w01, d.y)), dm(w.w11, e.y));
  return r;
}

// sample_flow_jacobian (warp.hpp:76-88): {dux, duy, dvx, dvy}. Precision of
// the Jacobian only enters gradients (tolerance-checked), so FMA is allowed.
struct Jac {
  double dux, duy, dvx, dvy;
};
__device__ __forceinline__ Jac sample_jacobian(const double2* __restrict__ f, const Cell& c) {
  const double2 a = __ldg(f + c.i00);
  const double2 b = __ldg(f + c.i00 + c.ox);
  const double2 d = __ldg(f + c.i00 + c.oy);
  const double2 e = __ldg(f + c.i00 + c.oy + c.ox);
  const double ax = 1.0 - c.wx, ay = 1.0 - c.wy;
  Jac j;
  j.dux = ay * (b.x - a.x) + c.wy * (e.x - d.x);
  j.duy = ax * (d.x - a.x) + c.wx * (e.x - b.x);
  j.dvx = ay * (b.y - a.y) + c.wy * (e.y - d.y);
  j.dvy = ax * (d.y - a.y) + c.wx * (e.y - b.y);
  return j;
}

// Event trajectory (build_trajectory, warp.hpp:257-281) with the two legs
// interleaved into one loop of B-1 chained steps, so that every lane of a warp
// runs the same number of samples whatever its bin j. The two partial steps of
// the reference both sample u_j(x0); it is sampled once here (same bits).
// pos[r * stride] receives the position at reference r (shared memory).
// Returns alive (all B+1 positions in bounds).
__device__ __forceinline__ bool trajectory(double x0, double y0, double t, int j,
                                           const double2* __restrict__ flows,
                                           const WinParams& P, const double* es, double2* pos,
                                           int stride) {
  const int W = P.W, H = P.H, B = P.B, HW = P.HW;
  const Cell c0 = bilin_cell(x0, y0, W, H);
  const double2 u0 = sample_flow(flows + (size_t)j * HW, c0);
  const double db = ds(es[j], t), df = ds(es[j + 1], t);
  double2 pb = make_double2(da(x0, dm(db, u0.x)), da(y0, dm(db, u0.y)));
  double2 pf = make_double2(da(x0, dm(df, u0.x)), da(y0, dm(df, u0.y)));
  pos[j * stride] = pb;
  pos[(j + 1) * stride] = pf;
  bool ok = in_bounds(pb.x, pb.y, W, H) && in_bounds(pf.x, pf.y, W, H);
  for (int s = 0; s < B - 1; ++s) {
    const bool back = s < j;
    // backward leg: bin i = j-1-s sampled at pos[i+1], writes pos[i]
    // forward leg:  bin i = s+1     sampled at pos[i],   writes pos[i+1]
    const int i = back ? j - 1 - s : s + 1;
    const double2 p = back ? pb : pf;
    const double dt = back ? ds(es[i], es[i + 1]) : ds(es[i + 1], es[i]);
    const Cell c = bilin_cell(p.x, p.y, W, H);
    const double2 u = sample_flow(flows + (size_t)i * HW, c);
    const double2 q = make_double2(da(p.x, dm(dt, u.x)), da(p.y, dm(dt, u.y)));
    pos[(back ? i : i + 1) * stride] = q;
    ok = ok && in_bounds(q.x, q.y, W, H);
    if (back) pb = q; else pf = q;
  }
  return ok;
}

}  // namespace evcm_b200
