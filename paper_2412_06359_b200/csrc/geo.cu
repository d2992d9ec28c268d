// Geometry-consistency loss L_geo on the device:
// geometry_consistency_loss[_backward] (geometry.hpp:329-534) for n_poses poses
// of one depth pair at once (grid.y = pose), as predictor_loss_and_gradients
// calls it once per bin with d0 = d1 = the decoded depth (optimize.hpp:219-236).
//
//   k_geo_project   reproject every usable source pixel (geometry.hpp:157-166, the
//                   motion-field expressions: bit-identical pixel and z), nearest
//                   target cell by lround, z-min per cell as an atomicMin on the
//                   bits of z (z > 0, so the u64 order is the fp64 order)
//   k_geo_winner    among the pixels whose z equals the cell minimum, the smallest
//                   source index wins (atomicMin): exactly the reference's
//                   sequential scan with a strict "<" (project_with_zmin, :359-390)
//   k_geo_terms     per winner: bilinear target depth (sample_target_depth,
//                   :394-409, bit-identical), the term |a-b|/(a+b), and with
//                   gradients the per-pixel d_d0, the gb weight for d_d1 and the
//                   pose contributions (:479-516); block partials in fixed order
//   k_geo_finalize  per pose: value = sum / n_valid, scale = upstream / n_valid,
//                   d_pose (optionally added onto the CMax pose gradients), and
//                   l_geo / total for the predictor (optimize.hpp:232-238)
//   k_geo_gather    d_d1 as a GATHER: the winners whose landing pixel's bilinear
//                   cell can touch target cell c sit at nearest cells c +- 1, so
//                   each cell reads its 3x3 neighbourhood of winners (fixed
//                   order: deterministic, no atomics); then d_d0, d_d1 scaled and
//                   the predictor's extra depth term sum_i (d_d0_i + d_d1_i),
//                   optionally added onto the CMax depth gradient.
//
// Everything that decides membership (pixel, z, winner, target depth, validity)
// is bit-identical to the reference; sums over pixels (the loss, d_pose, d_d1)
// differ from the reference's sequential order only by rounding.
#include <cstdint>

#include "cmax_device.cuh"
#include "cmax_kernels.h"

namespace evcm_b200 {

namespace {

constexpr int kGeoBlock = 256;
constexpr int kGeoParts = 8;  // sum, n_valid, d_omega[3], d_trans[3]

struct GeoCam {
  double fx, fy, cx, cy;
};

// reproject (geometry.hpp:157-166) with backproject (:147-149): same expressions
// as k_motion_field. Returns valid (z > 0).
__device__ __forceinline__ bool reproject(int x, int y, double d, const double* t, const GeoCam& k,
                                          double& ux, double& uy, double& z) {
  const double bx = dd(dm(d, ds((double)x, k.cx)), k.fx);
  const double by = dd(dm(d, ds((double)y, k.cy)), k.fy);
  const double px = da(da(da(dm(t[0], bx), dm(t[1], by)), dm(t[2], d)), t[36]);
  const double py = da(da(da(dm(t[3], bx), dm(t[4], by)), dm(t[5], d)), t[37]);
  z = da(da(da(dm(t[6], bx), dm(t[7], by)), dm(t[8], d)), t[38]);
  if (!(z > 0.0)) return false;
  ux = da(dd(dm(k.fx, px), z), k.cx);
  uy = da(dd(dm(k.fy, py), z), k.cy);
  return true;
}

// A usable, in-view source pixel: its nearest target cell, else -1.
__device__ __forceinline__ int project_cell(const double* __restrict__ d0,
                                            const uint8_t* __restrict__ m0, int q, int W, int H,
                                            const double* t, const GeoCam& k, double& ux,
                                            double& uy, double& z) {
  if (m0 && !m0[q]) return -1;
  const double d = d0[q];
  if (!(d > 0.0)) return -1;
  const int y = q / W, x = q - y * W;
  if (!reproject(x, y, d, t, k, ux, uy, z)) return -1;
  if (!in_bounds(ux, uy, W, H)) return -1;
  const int nx = (int)lround(ux), ny = (int)lround(uy);  // std::lround
  return ny * W + nx;
}

__global__ void k_geo_project(const double* __restrict__ d0, const uint8_t* __restrict__ m0, int W,
                              int H, const double* __restrict__ tab, GeoCam k,
                              unsigned long long* __restrict__ zkey) {
  const int i = blockIdx.y, HW = W * H;
  const double* t = tab + (size_t)i * kPoseTab;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < HW; q += gridDim.x * blockDim.x) {
    double ux, uy, z;
    const int c = project_cell(d0, m0, q, W, H, t, k, ux, uy, z);
    if (c >= 0) atomicMin(zkey + (size_t)i * HW + c, (unsigned long long)__double_as_longlong(z));
  }
}

__global__ void k_geo_winner(const double* __restrict__ d0, const uint8_t* __restrict__ m0, int W,
                             int H, const double* __restrict__ tab, GeoCam k,
                             const unsigned long long* __restrict__ zkey,
                             unsigned* __restrict__ winner) {
  const int i = blockIdx.y, HW = W * H;
  const double* t = tab + (size_t)i * kPoseTab;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < HW; q += gridDim.x * blockDim.x) {
    double ux, uy, z;
    const int c = project_cell(d0, m0, q, W, H, t, k, ux, uy, z);
    if (c >= 0 && zkey[(size_t)i * HW + c] == (unsigned long long)__double_as_longlong(z))
      atomicMin(winner + (size_t)i * HW + c, (unsigned)q);
  }
}

// Fixed-order block sum of kGeoParts doubles (butterfly in the warp, then warps in
// order); thread 0 writes the block's partials.
__device__ __forceinline__ void block_parts(double (&v)[kGeoParts], double* __restrict__ out) {
  __shared__ double sh[kGeoBlock / 32][kGeoParts];
#pragma unroll
  for (int j = 0; j < kGeoParts; ++j)
    for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0)
    for (int j = 0; j < kGeoParts; ++j) sh[wid][j] = v[j];
  __syncthreads();
  if (threadIdx.x < kGeoParts) {
    double s = 0.0;
    for (int w = 0; w < kGeoBlock / 32; ++w) s += sh[w][threadIdx.x];
    out[threadIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kGeoBlock) k_geo_terms(
    const double* __restrict__ d0, const uint8_t* __restrict__ m0, const double* __restrict__ d1,
    const uint8_t* __restrict__ m1, int W, int H, const double* __restrict__ tab, GeoCam k,
    const unsigned* __restrict__ winner, int want_grad, double* __restrict__ projected,
    double* __restrict__ interpolated, uint8_t* __restrict__ valid, double* __restrict__ dd0_raw,
    double* __restrict__ gb_src, double2* __restrict__ land, double* __restrict__ parts) {
  const int i = blockIdx.y, HW = W * H;
  const double* t = tab + (size_t)i * kPoseTab;
  const size_t base = (size_t)i * HW;
  double acc[kGeoParts] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < HW; q += gridDim.x * blockDim.x) {
    double ux = 0.0, uy = 0.0, a = 0.0, b = 0.0, d_d0 = 0.0, gb = 0.0;
    bool ok = false;
    const int c = project_cell(d0, m0, q, W, H, t, k, ux, uy, a);
    Cell cl;
    double v00 = 0, v10 = 0, v01 = 0, v11 = 0;
    if (c >= 0 && winner[base + c] == (unsigned)q) {
      cl = bilin_cell(ux, uy, W, H);  // sample_target_depth (geometry.hpp:394-409)
      const int i00 = cl.i00;
      if (!m1 || (m1[i00] && m1[i00 + cl.ox] && m1[i00 + cl.oy] && m1[i00 + cl.oy + cl.ox])) {
        v00 = d1[i00];
        v10 = d1[i00 + cl.ox];
        v01 = d1[i00 + cl.oy];
        v11 = d1[i00 + cl.oy + cl.ox];
        const Weights w = weights(cl);
        b = da(da(da(dm(w.w00, v00), dm(w.w10, v10)), dm(w.w01, v01)), dm(w.w11, v11));
        ok = b > 0.0;
      }
    }
    if (projected) projected[base + q] = ok ? a : 0.0;
    if (interpolated) interpolated[base + q] = ok ? b : 0.0;
    if (valid) valid[base + q] = ok ? 1 : 0;
    if (ok) {
      acc[0] += dd(fabs(ds(a, b)), da(a, b));
      acc[1] += 1.0;
    }
    if (want_grad) {
      if (ok) {
        // geometry.hpp:486-516 with reproject_with_grads (:185-209)
        const double dbx = (1.0 - cl.wy) * (v10 - v00) + cl.wy * (v11 - v01);
        const double dby = (1.0 - cl.wx) * (v01 - v00) + cl.wx * (v11 - v10);
        const double s = (a > b) ? 1.0 : (a < b ? -1.0 : 0.0);
        const double inv_ab = 1.0 / ((a + b) * (a + b));
        const double ga = 2.0 * s * b * inv_ab;
        gb = -2.0 * s * a * inv_ab;
        const int y = q / W, x = q - y * W;
        const double d = d0[q];
        const double ray[3] = {(x - k.cx) / k.fx, (y - k.cy) / k.fy, 1.0};
        double rr[3];
        for (int r = 0; r < 3; ++r) rr[r] = t[3 * r] * ray[0] + t[3 * r + 1] * ray[1] + t[3 * r + 2] * ray[2];
        const double p0 = d * rr[0] + t[36], p1 = d * rr[1] + t[37], p2 = d * rr[2] + t[38];
        const double iz = 1.0 / p2;
        const double ju[3] = {k.fx * iz, 0.0, -k.fx * p0 * iz * iz};
        const double jv[3] = {0.0, k.fy * iz, -k.fy * p1 * iz * iz};
        const double dpx = ju[0] * rr[0] + ju[1] * rr[1] + ju[2] * rr[2];
        const double dpy = jv[0] * rr[0] + jv[1] * rr[1] + jv[2] * rr[2];
        d_d0 = ga * rr[2] + gb * (dbx * dpx + dby * dpy);
        for (int cc = 0; cc < 3; ++cc) {
          const double* dR = t + 9 + 9 * cc;
          double qv[3];
          for (int r = 0; r < 3; ++r)
            qv[r] = d * (dR[3 * r] * ray[0] + dR[3 * r + 1] * ray[1] + dR[3 * r + 2] * ray[2]);
          const double pox = ju[0] * qv[0] + ju[1] * qv[1] + ju[2] * qv[2];
          const double poy = jv[0] * qv[0] + jv[1] * qv[1] + jv[2] * qv[2];
          acc[2 + cc] += ga * qv[2] + gb * (dbx * pox + dby * poy);
          acc[5 + cc] += ga * (cc == 2 ? 1.0 : 0.0) + gb * (dbx * ju[cc] + dby * jv[cc]);
        }
        land[base + q] = make_double2(ux, uy);
      }
      dd0_raw[base + q] = d_d0;
      gb_src[base + q] = gb;
    }
  }
  block_parts(acc, parts + ((size_t)i * gridDim.x + blockIdx.x) * kGeoParts);
}

// One block: per pose the fixed-order sum of the block partials, then the
// per-pose value / scale / d_pose and the predictor's l_geo and total.
__global__ void k_geo_finalize(const double* __restrict__ parts, int n_parts, int n_poses,
                               double upstream, double* __restrict__ value,
                               long long* __restrict__ n_valid, double* __restrict__ scale,
                               double* __restrict__ d_poses, const double* __restrict__ add_poses,
                               const double* __restrict__ l_cm, double lambda,
                               double* __restrict__ losses) {
  __shared__ double sh[kGeoBlock];
  __shared__ double tot[kGeoParts];
  for (int i = 0; i < n_poses; ++i) {
    for (int j = 0; j < kGeoParts; ++j) {
      double s = 0.0;
      for (int b = threadIdx.x; b < n_parts; b += blockDim.x)
        s += parts[((size_t)i * n_parts + b) * kGeoParts + j];
      sh[threadIdx.x] = s;
      __syncthreads();
      for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
      }
      if (threadIdx.x == 0) tot[j] = sh[0];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const double n = tot[1];
      const double v = n > 0.0 ? tot[0] / n : 0.0;  // geometry.hpp:521-531
      const double sc = n > 0.0 ? upstream / n : 0.0;
      value[i] = v;
      n_valid[i] = (long long)n;
      scale[i] = sc;
      if (d_poses)
        for (int c = 0; c < 6; ++c) {
          const double g = sc * tot[2 + c];
          // accumulate_gradients adds the extra pose term (predictor.hpp:166-171)
          d_poses[6 * i + c] = add_poses ? add_poses[6 * i + c] + g : g;
        }
    }
    __syncthreads();
  }
  if (losses && threadIdx.x == 0) {
    double geo_sum = 0.0;  // optimize.hpp:223-236
    for (int i = 0; i < n_poses; ++i) geo_sum += value[i];
    const double l_geo = geo_sum / (double)n_poses;
    losses[0] = *l_cm;
    losses[1] = l_geo;
    losses[2] = *l_cm + lambda * l_geo;  // optimize.hpp:238
  }
}

__global__ void k_geo_gather(int W, int H, int n_poses, const unsigned* __restrict__ winner,
                             const double* __restrict__ gb_src, const double2* __restrict__ land,
                             const double* __restrict__ dd0_raw, const double* __restrict__ scale,
                             double* __restrict__ d_d0, double* __restrict__ d_d1,
                             double* __restrict__ d_depth_sum, const double* __restrict__ add_depth) {
  const int HW = W * H;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < HW; c += gridDim.x * blockDim.x) {
    const int cy = c / W, cx = c - cy * W;
    double extra = 0.0;
    for (int i = 0; i < n_poses; ++i) {
      const size_t base = (size_t)i * HW;
      double acc = 0.0;
      for (int ny = max(cy - 1, 0); ny <= min(cy + 1, H - 1); ++ny)
        for (int nx = max(cx - 1, 0); nx <= min(cx + 1, W - 1); ++nx) {
          const unsigned s = winner[base + ny * W + nx];
          if (s == 0xffffffffu) continue;
          const double gb = gb_src[base + s];
          if (gb == 0.0) continue;
          const double2 p = land[base + s];
          const Cell cl = bilin_cell(p.x, p.y, W, H);
          const Weights w = weights(cl);
          // geometry.hpp:502-506: the four corners (coincident corners add twice)
          if (cl.i00 == c) acc += gb * w.w00;
          if (cl.i00 + cl.ox == c) acc += gb * w.w10;
          if (cl.i00 + cl.oy == c) acc += gb * w.w01;
          if (cl.i00 + cl.oy + cl.ox == c) acc += gb * w.w11;
        }
      const double sc = scale[i];
      const double a0 = dd0_raw[base + c] * sc, a1 = acc * sc;
      if (d_d0) d_d0[base + c] = a0;
      if (d_d1) d_d1[base + c] = a1;
      extra += a0 + a1;  // optimize.hpp:229-230
    }
    if (d_depth_sum) d_depth_sum[c] = add_depth ? add_depth[c] + extra : extra;  // predictor.hpp:153-155
  }
}

__global__ void k_geo_losses_off(const double* __restrict__ l_cm, double lambda,
                                 double* __restrict__ losses) {
  losses[0] = *l_cm;
  losses[1] = 0.0;
  losses[2] = *l_cm + lambda * 0.0;  // optimize.hpp:238 with the term switched off
}

}  // namespace

void launch_geo_losses_off(cudaStream_t s, const double* l_cm, double lambda, double* losses) {
  count_launch();
  k_geo_losses_off<<<1, 1, 0, s>>>(l_cm, lambda, losses);
}

int geo_parts(int W, int H) { return std::min((W * H + kGeoBlock - 1) / kGeoBlock, 148 * 8); }

void launch_geo(cudaStream_t s, const GeoArgs& g) {
  const int HW = g.W * g.H;
  const GeoCam k{g.K[0], g.K[1], g.K[2], g.K[3]};
  const int nb = geo_parts(g.W, g.H);
  const dim3 grid(nb, g.n_poses);
  cudaMemsetAsync(g.zkey, 0xff, sizeof(unsigned long long) * HW * g.n_poses, s);
  cudaMemsetAsync(g.winner, 0xff, sizeof(unsigned) * HW * g.n_poses, s);
  count_launch();
  k_geo_project<<<grid, kGeoBlock, 0, s>>>(g.d0, g.m0, g.W, g.H, g.tab, k, g.zkey);
  count_launch();
  k_geo_winner<<<grid, kGeoBlock, 0, s>>>(g.d0, g.m0, g.W, g.H, g.tab, k, g.zkey, g.winner);
  count_launch();
  k_geo_terms<<<grid, kGeoBlock, 0, s>>>(g.d0, g.m0, g.d1, g.m1, g.W, g.H, g.tab, k, g.winner,
                                         g.want_grad, g.projected, g.interpolated, g.valid,
                                         g.dd0_raw, g.gb_src, g.land, g.parts);
  count_launch();
  k_geo_finalize<<<1, kGeoBlock, 0, s>>>(g.parts, nb, g.n_poses, g.upstream, g.value, g.n_valid,
                                         g.scale, g.want_grad ? g.d_poses : nullptr, g.add_poses,
                                         g.l_cm, g.lambda, g.losses);
  if (g.want_grad) {
    count_launch();
    k_geo_gather<<<(HW + kGeoBlock - 1) / kGeoBlock, kGeoBlock, 0, s>>>(
        g.W, g.H, g.n_poses, g.winner, g.gb_src, g.land, g.dd0_raw, g.scale, g.d_d0, g.d_d1,
        g.d_depth_sum, g.add_depth);
  }
}

}  // namespace evcm_b200
