// Predictor decode chain on the device: the caller of
// the CMax path in predictor_loss_and_gradients (optimize.hpp:205-241).
//
//   k_decode          depth = upsample_bilinear(softplus(params), f)
//                     (predictor.hpp:25-27, 40-66, 126-131)
//   k_decode_adjoint  d_params = upsample_bilinear_adjoint(d_depth) * softplus_grad(params)
//                     (predictor.hpp:30-34, 69-96, 156-162); a GATHER per source
//                     pixel over the output pixels whose bilinear stencil holds it
//                     (fixed order: deterministic), instead of the reference's scatter
//   k_adam            Adam::step (optimize.hpp:115-134), element-wise
//
// Arithmetic follows the reference's expression order with explicit
// round-to-nearest intrinsics (no FMA contraction): the upsampling weights and
// products, and Adam, are bit-identical to the reference given the same inputs;
// softplus uses the device's exp/log1p (within an ulp of the host libm).
#include <cstdint>

#include "cmax_device.cuh"
#include "cmax_kernels.h"

namespace evcm_b200 {

namespace {

__device__ __forceinline__ double softplus(double x) {  // predictor.hpp:25-27
  return x > 0.0 ? da(x, log1p(exp(-x))) : log1p(exp(x));
}

__device__ __forceinline__ double softplus_grad(double x) {  // predictor.hpp:30-34
  if (x >= 0.0) return dd(1.0, da(1.0, exp(-x)));
  const double e = exp(x);
  return dd(e, da(1.0, e));
}

// upsample_src_coord (predictor.hpp:40-44): output centres map to
// (o + 0.5) / factor - 0.5 on the source grid, clamped to the border
__device__ __forceinline__ double src_coord(int o, int factor, int src_size) {
  const double s = ds(dd(da((double)o, 0.5), (double)factor), 0.5);
  const double hi = (double)(src_size - 1);
  return s < 0.0 ? 0.0 : (hi < s ? hi : s);
}

struct Tap {
  int i0, i1;
  double w;  // weight of i1; i0 gets 1 - w
};
__device__ __forceinline__ Tap tap(int o, int factor, int src_size) {
  const double s = src_coord(o, factor, src_size);
  Tap t;
  t.i0 = min((int)floor(s), src_size - 1);
  t.i1 = min(t.i0 + 1, src_size - 1);
  t.w = ds(s, (double)t.i0);
  return t;
}

__global__ void k_decode(const double* __restrict__ params, int sw, int sh, int factor,
                         double* __restrict__ depth) {
  const int W = sw * factor, H = sh * factor;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < W * H; q += gridDim.x * blockDim.x) {
    const int y = q / W, x = q - y * W;
    const Tap ty = tap(y, factor, sh), tx = tap(x, factor, sw);
    const double a00 = softplus(params[ty.i0 * sw + tx.i0]);
    const double a10 = softplus(params[ty.i0 * sw + tx.i1]);
    const double a01 = softplus(params[ty.i1 * sw + tx.i0]);
    const double a11 = softplus(params[ty.i1 * sw + tx.i1]);
    const double ax = ds(1.0, tx.w), ay = ds(1.0, ty.w);
    // (1-wx)(1-wy) s00 + wx(1-wy) s10 + (1-wx) wy s01 + wx wy s11, left to right
    depth[q] = da(da(da(dm(dm(ax, ay), a00), dm(dm(tx.w, ay), a10)), dm(dm(ax, ty.w), a01)),
                  dm(dm(tx.w, ty.w), a11));
  }
}

// Output range [lo, hi) whose taps can reference source index p along one axis.
__device__ __forceinline__ void out_range(int p, int factor, int src_size, int out_size, int& lo,
                                          int& hi) {
  lo = max(0, (p - 1) * factor - factor);
  hi = min(out_size, (p + 2) * factor + factor);
  (void)src_size;
}

__global__ void k_decode_adjoint(const double* __restrict__ params, const double* __restrict__ d_depth,
                                 int sw, int sh, int factor, double* __restrict__ d_params) {
  const int W = sw * factor, H = sh * factor;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < sw * sh; p += gridDim.x * blockDim.x) {
    const int py = p / sw, px = p - py * sw;
    int x_lo, x_hi, y_lo, y_hi;
    out_range(px, factor, sw, W, x_lo, x_hi);
    out_range(py, factor, sh, H, y_lo, y_hi);
    double acc = 0.0;
    for (int y = y_lo; y < y_hi; ++y) {
      const Tap ty = tap(y, factor, sh);
      // weight of source row py in output row y (both taps may coincide at the border)
      const double ay = ds(1.0, ty.w);
      const bool r0 = ty.i0 == py, r1 = ty.i1 == py;
      if (!r0 && !r1) continue;
      for (int x = x_lo; x < x_hi; ++x) {
        const Tap tx = tap(x, factor, sw);
        const bool c0 = tx.i0 == px, c1 = tx.i1 == px;
        if (!c0 && !c1) continue;
        const double ax = ds(1.0, tx.w);
        const double g = d_depth[(size_t)y * W + x];
        // the reference's four corner products (predictor.hpp:91-94), those landing on p
        if (r0 && c0) acc = da(acc, dm(dm(ax, ay), g));
        if (r0 && c1) acc = da(acc, dm(dm(tx.w, ay), g));
        if (r1 && c0) acc = da(acc, dm(dm(ax, ty.w), g));
        if (r1 && c1) acc = da(acc, dm(dm(tx.w, ty.w), g));
      }
    }
    d_params[p] = dm(acc, softplus_grad(params[p]));  // predictor.hpp:161-162
  }
}

__global__ void k_adam(double* __restrict__ slots, const double* __restrict__ grads,
                       double* __restrict__ m, double* __restrict__ v, size_t n, double lr,
                       double b1, double b2, double eps, double c1, double c2) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double g = grads[i];
    // optimize.hpp:125-128, same association
    m[i] = da(dm(b1, m[i]), dm(ds(1.0, b1), g));
    v[i] = da(dm(b2, v[i]), dm(dm(ds(1.0, b2), g), g));
    slots[i] = ds(slots[i], dd(dm(lr, dd(m[i], c1)), da(__dsqrt_rn(dd(v[i], c2)), eps)));
  }
}

}  // namespace

void launch_decode(cudaStream_t s, const double* params, int sw, int sh, int factor, double* depth) {
  const int n = sw * factor * sh * factor;
  count_launch();
  k_decode<<<(n + 255) / 256, 256, 0, s>>>(params, sw, sh, factor, depth);
}

void launch_decode_adjoint(cudaStream_t s, const double* params, const double* d_depth, int sw,
                           int sh, int factor, double* d_params) {
  count_launch();
  k_decode_adjoint<<<(sw * sh + 127) / 128, 128, 0, s>>>(params, d_depth, sw, sh, factor, d_params);
}

void launch_adam(cudaStream_t s, double* slots, const double* grads, double* m, double* v, size_t n,
                 double lr, double b1, double b2, double eps, double c1, double c2) {
  if (n == 0) return;
  count_launch();
  k_adam<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(slots, grads, m, v, n,
                                                                            lr, b1, b2, eps, c1, c2);
}

}  // namespace evcm_b200
