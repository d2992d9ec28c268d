// CUDA kernels of the CMax loss path for B200 (sm_100a).
//
// Stage map:
//   k_stage          events AoS (evcm::Event) -> packed 8 B records + window
//                    validation (EventSlice::validate, types.hpp:135-159)
//   k_motion_field   K1  depth_pose_to_flows          geometry.hpp:229-264
//   k_fwd_splat      K2+K3 build_trajectory + splat   warp.hpp:257-281, engine.hpp:365-374
//   k_loss_reduce    K3b refresh_active + reference_loss + coefficient planes
//                    warp.hpp:186-192, 299-312, 345-350
//   k_loss_finalize  reduce_loss                      engine.hpp:442-468
//   k_bwd            K4  backward_event               engine.hpp:475-504
//   k_flows_bwd      K5  depth_pose_to_flows_backward geometry.hpp:279-325
//
// Data layout in HBM (per window w of a batch; HW = W*H, R = B+1):
//   packed events  uint2 [n]                         8 B / event
//   flows          double2 [w][B][HW]   (u, v) interleaved, 16 B / px / bin
//   stack          S2 [w][R][2][HW]     (count, tsum) interleaved, S2 = float2|double2
//   coef           S2 [w][R][2][HW]     (a = S/(C+eps), q = a/(C+eps))
//   grad           G2 [w][B][HW]        (gu, gv) interleaved, G2 = float2|double2
#include <cstdint>
#include <cstdio>

#include "cmax_device.cuh"
#include "cmax_kernels.h"

namespace evcm_b200 {

static thread_local int g_launches = 0;
void reset_launch_count() { g_launches = 0; }
void count_launch() { ++g_launches; }
int launch_count() { return g_launches; }

// --------------------------------------------------------------------------
// helpers

template <typename T> struct Vec2Of;
template <> struct Vec2Of<float> { using type = float2; };
template <> struct Vec2Of<double> { using type = double2; };

__device__ __forceinline__ void red_add2(float2* p, double a, double b) {
  atomicAdd(p, make_float2((float)a, (float)b));  // REDG.E.ADD.F32x2
}
__device__ __forceinline__ void red_add2(double2* p, double a, double b) {
  atomicAdd(&p->x, a);  // REDG.E.ADD.F64
  atomicAdd(&p->y, b);
}
__device__ __forceinline__ double2 ld2(const float2* p) {
  const float2 v = __ldg(p);
  return make_double2(v.x, v.y);
}
__device__ __forceinline__ double2 ld2(const double2* p) { return __ldg(p); }
__device__ __forceinline__ void store2(float2* p, double a, double b) {
  *p = make_float2((float)a, (float)b);
}
__device__ __forceinline__ void store2(double2* p, double a, double b) { *p = make_double2(a, b); }

__device__ __forceinline__ void load_edges(const WinParams& P, double* es, uint32_t* erel) {
  for (int i = threadIdx.x; i <= P.B; i += blockDim.x) {
    es[i] = P.es[i];
    erel[i] = P.erel[i];
  }
}

// --------------------------------------------------------------------------
// K0: staging + validation

// Error key per window: (index << 4 | code), minimum wins = first violation in
// event order, and for that event the first failing check in the order of
// EventSlice::validate (types.hpp:143-155).
__global__ void k_stage(const evcm_event* __restrict__ ev, const uint64_t* __restrict__ ev_off,
                        WinParams P, uint2* __restrict__ packed,
                        unsigned long long* __restrict__ err) {
  const int w = blockIdx.y;
  const uint64_t base = ev_off[w];
  const uint64_t n = ev_off[w + 1] - base;
  const uint64_t t0 = P.t0 + (uint64_t)w * P.stride_us, t_end = P.t_end + (uint64_t)w * P.stride_us;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const evcm_event e = ev[base + k];
    unsigned code = 0;
    if (e.x >= P.W || e.y >= P.H) code = 3;
    else if (e.p != 1 && e.p != -1) code = 4;
    else if (k > 0 && e.t_us < ev[base + k - 1].t_us) code = 5;
    else if (e.t_us < t0 || e.t_us >= t_end) code = 6;
    if (code) {
      atomicMin(err + w, ((unsigned long long)k << 4) | code);
      continue;
    }
    const uint32_t dt = (uint32_t)(e.t_us - t0);
    packed[base + k] = make_uint2(dt | (e.p > 0 ? 0u : 0x80000000u),
                                  (uint32_t)e.x | ((uint32_t)e.y << 16));
  }
}

// flows [B][2][HW] f64 planes -> interleaved double2 [B][HW]
// (out32: optional fp32 copy, the owner backward's flow-Jacobian operand)
__global__ void k_interleave_flows(const double* __restrict__ uv, int B, int HW,
                                   double2* __restrict__ out, float2* __restrict__ out32) {
  const size_t total = (size_t)B * HW;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / HW, p = i % HW;
    const double2 f = make_double2(uv[(2 * b) * HW + p], uv[(2 * b + 1) * HW + p]);
    out[i] = f;
    if (out32) out32[i] = make_float2((float)f.x, (float)f.y);
  }
}

// --------------------------------------------------------------------------
// Pose tables on the device (for device-resident poses: no host round trip).
// Same expression order as rodrigues / rodrigues_jacobian (geometry.hpp:94-135);
// the device sin/cos may differ from the host libm by an ulp, so flows from
// device poses match the reference to ~1e-16 relative instead of bit for bit.
// Pose validation (types.hpp:362-368) sets *bad = 1.

__device__ void m3mul(const double* a, const double* b, double* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}
__device__ void m3skew(double x, double y, double z, double* s) {
  s[0] = 0; s[1] = -z; s[2] = y; s[3] = z; s[4] = 0; s[5] = -x; s[6] = -y; s[7] = x; s[8] = 0;
}
__device__ void rodrigues_dev(const double* w, double* R) {
  const double t2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  const double t = sqrt(t2);
  double a, b;
  if (t < 1e-8) {
    a = 1.0 - t2 / 6.0;
    b = 0.5 - t2 / 24.0;
  } else {
    a = sin(t) / t;
    b = (1.0 - cos(t)) / t2;
  }
  double S[9], S2[9];
  m3skew(w[0], w[1], w[2], S);
  m3mul(S, S, S2);
  for (int i = 0; i < 9; ++i) R[i] = ((i % 4 == 0 ? 1.0 : 0.0) + a * S[i]) + b * S2[i];
}

// One (window, bin) entry of the pose table: R[9], dR[27], t[3], inv_dt.
// Returns true when the pose fails PoseStep::validate (types.hpp:362-368).
__device__ bool pose_entry(const double* __restrict__ p, double inv_dt, double* __restrict__ t) {
  const double pi = 3.14159265358979323846;
  const bool bad = !(sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]) < pi) || !isfinite(p[0]) ||
                   !isfinite(p[1]) || !isfinite(p[2]) || !isfinite(p[3]) || !isfinite(p[4]) ||
                   !isfinite(p[5]);
  double R[9], S[9];
  rodrigues_dev(p, R);
  for (int q = 0; q < 9; ++q) t[q] = R[q];
  const double t2 = p[0] * p[0] + p[1] * p[1] + p[2] * p[2];
  m3skew(p[0], p[1], p[2], S);
  if (sqrt(t2) < 1e-4) {
    for (int kk = 0; kk < 3; ++kk) {
      double ek[9], a[9], b[9];
      m3skew(kk == 0, kk == 1, kk == 2, ek);
      m3mul(ek, S, a);
      m3mul(S, ek, b);
      for (int q = 0; q < 9; ++q) t[9 + 9 * kk + q] = ek[q] + 0.5 * (a[q] + b[q]);
    }
  } else {
    double IR[9];
    for (int q = 0; q < 9; ++q) IR[q] = (q % 4 == 0 ? 1.0 : 0.0) - R[q];
    for (int kk = 0; kk < 3; ++kk) {
      const double c0 = IR[kk], c1 = IR[3 + kk], c2 = IR[6 + kk];
      double sc[9], m[9], pr[9];
      m3skew(p[1] * c2 - p[2] * c1, p[2] * c0 - p[0] * c2, p[0] * c1 - p[1] * c0, sc);
      for (int q = 0; q < 9; ++q) m[q] = p[kk] * S[q] + sc[q];
      m3mul(m, R, pr);
      for (int q = 0; q < 9; ++q) t[9 + 9 * kk + q] = (1.0 / t2) * pr[q];
    }
  }
  t[36] = p[3];
  t[37] = p[4];
  t[38] = p[5];
  t[39] = inv_dt;
  return bad;
}

__global__ void k_pose_table(const double* __restrict__ poses, int n, int B,
                             const double* __restrict__ inv_dt, double* __restrict__ tab,
                             int* __restrict__ bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (window, bin)
  if (i >= n) return;
  if (pose_entry(poses + 6 * (size_t)i, inv_dt[i % B], tab + (size_t)i * kPoseTab)) atomicExch(bad, 1);
}

void launch_pose_table(cudaStream_t s, const double* poses, int n_windows, int B,
                       const double* inv_dt, double* tab, int* bad) {
  const int n = n_windows * B;
  ++g_launches;
  k_pose_table<<<(n + 63) / 64, 64, 0, s>>>(poses, n, B, inv_dt, tab, bad);
}

// Packed window sums [sum_w loss, sum_w d_depth, sum_w d_poses], each entry
// summed over the windows in window order (deterministic).
__global__ void k_window_sums(const double* __restrict__ loss, const double* __restrict__ d_depth,
                              const double* __restrict__ d_poses, int nw, int HW, int B6,
                              double* __restrict__ out) {
  const int n = 1 + HW + B6;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double* src;
    size_t stride;
    if (i == 0) {
      src = loss;
      stride = 1;
    } else if (i <= HW) {
      src = d_depth + (i - 1);
      stride = HW;
    } else {
      src = d_poses + (i - 1 - HW);
      stride = B6;
    }
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += src[(size_t)w * stride];
    out[i] = s;
  }
}

void launch_window_sums(cudaStream_t s, const double* loss, const double* d_depth,
                        const double* d_poses, int nw, int HW, int B6, double* out) {
  ++g_launches;
  const int n = 1 + HW + B6;
  k_window_sums<<<(n + 255) / 256, 256, 0, s>>>(loss, d_depth, d_poses, nw, HW, B6, out);
}

// The chain's prologue in one launch (instead of two host->device copies, two
// memsets and the pose-table kernel): the window offsets (kernel parameters)
// into device memory, the per-window validation words to "no error", and --
// for device poses -- the pose table with FlowSequence::zeros bin durations
// (types.hpp:303-304, the host expression) and the validation flag in word nw.
__global__ void __launch_bounds__(256) k_chain_init(ChainInit a, WinParams P) {
  const int tid = threadIdx.x, nw = a.nw, B = a.B;
  for (int i = tid; i <= nw; i += blockDim.x) a.ev_off[i] = a.off[i];
  for (int i = tid; i < nw; i += blockDim.x) a.err[i] = ~0ull;
  int bad = 0;
  if (a.poses)
    for (int i = tid; i < nw * B; i += blockDim.x) {
      const int b = i % B;
      const double dur = dm(ds((double)(P.t0 + P.erel[b + 1]), (double)(P.t0 + P.erel[b])), 1e-6);
      bad |= pose_entry(a.poses + 6 * (size_t)i, dd(1.0, dur), a.tab + (size_t)i * kPoseTab) ? 1 : 0;
    }
  bad = __syncthreads_or(bad);
  if (tid == 0) a.err[nw] = bad ? 1ull : 0ull;
}

void launch_chain_init(cudaStream_t s, const ChainInit& a, const WinParams& P) {
  ++g_launches;
  k_chain_init<<<1, 256, 0, s>>>(a, P);
}

// --------------------------------------------------------------------------
// K1: motion field (depth_pose_to_flows, geometry.hpp:229-264)

// pose table per (window, bin): R[9], dR[27], t[3], inv_dt  -> 40 doubles
// One thread per pixel, bins in a loop: the back-projection (two IEEE fp64
// divisions) is bin-independent and computed once; same expressions as the
// reference, so the flows stay bit-identical.
__global__ void k_motion_field(const double* __restrict__ depth, const uint8_t* __restrict__ mask,
                               const double* __restrict__ pose_tab, WinParams P, double fx,
                               double fy, double cx, double cy, double2* __restrict__ flows,
                               uint8_t* __restrict__ valid, float2* __restrict__ flows32) {
  const int w = blockIdx.y;
  const int HW = P.HW, B = P.B;
  const double* dep = depth + (size_t)w * HW;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < HW; q += gridDim.x * blockDim.x) {
    const double d = dep[q];
    const bool dv = (!mask || mask[(size_t)w * HW + q]) && d > 0.0;
    const int y = q / P.W, x = q - y * P.W;
    double bx = 0.0, by = 0.0;
    if (dv) {  // backproject (geometry.hpp:147-149)
      bx = dd(dm(d, ds((double)x, cx)), fx);
      by = dd(dm(d, ds((double)y, cy)), fy);
    }
    const double bz = d;
    for (int b = 0; b < B; ++b) {
      const double* pt = pose_tab + ((size_t)w * B + b) * kPoseTab;
      double2 f = make_double2(0.0, 0.0);
      uint8_t ok = 0;
      if (dv) {
        const double* Rm = pt;
        const double* tr = pt + 36;
        // rot * v + trans (geometry.hpp:77-81, 159)
        const double px = da(da(da(dm(Rm[0], bx), dm(Rm[1], by)), dm(Rm[2], bz)), tr[0]);
        const double py = da(da(da(dm(Rm[3], bx), dm(Rm[4], by)), dm(Rm[5], bz)), tr[1]);
        const double pz = da(da(da(dm(Rm[6], bx), dm(Rm[7], by)), dm(Rm[8], bz)), tr[2]);
        if (pz > 0.0) {
          const double inv_dt = pt[39];
          const double ux = da(dd(dm(fx, px), pz), cx);
          const double uy = da(dd(dm(fy, py), pz), cy);
          f = make_double2(dm(ds(ux, (double)x), inv_dt), dm(ds(uy, (double)y), inv_dt));
          ok = 1;
        }
      }
      flows[((size_t)w * B + b) * HW + q] = f;
      if (flows32) flows32[((size_t)w * B + b) * HW + q] = make_float2((float)f.x, (float)f.y);
      if (valid) valid[((size_t)w * B + b) * HW + q] = ok;
    }
  }
}

// --------------------------------------------------------------------------
// K2+K3: per-event trajectory + bilinear splat into the per-reference stack

template <typename S2>
__global__ void __launch_bounds__(kEvBlock) k_fwd_splat(const uint2* __restrict__ packed,
                                                        const uint64_t* __restrict__ ev_off,
                                                        WinParams P,
                                                        const double2* __restrict__ flows,
                                                        S2* __restrict__ stack) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* es = reinterpret_cast<double*>(smem);
  uint32_t* erel = reinterpret_cast<uint32_t*>(es + kMaxRefs);
  double2* pos = reinterpret_cast<double2*>(smem + kEvSmemHeader) + threadIdx.x;
  load_edges(P, es, erel);
  __syncthreads();
  const int w = blockIdx.y;
  const uint64_t base = ev_off[w];
  const uint64_t n = ev_off[w + 1] - base;
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint2 e = packed[base + k];
  const uint32_t dt = ev_dt(e);
  const double t = dm((double)dt, 1e-6);  // engine.hpp:270
  const int j = bin_of(dt, erel, P.B);
  const double2* fl = flows + (size_t)w * P.B * P.HW;
  if (!trajectory((double)ev_x(e), (double)ev_y(e), t, j, fl, P, es, pos, blockDim.x)) return;
  const int pol = ev_pol(e);
  S2* st = stack + (size_t)w * (P.B + 1) * 2 * P.HW;
  for (int r = 0; r <= P.B; ++r) {
    const double2 p = pos[r * blockDim.x];
    const Cell c = bilin_cell(p.x, p.y, P.W, P.H);
    const Weights wt = weights(c);
    const double tb = dd(fabs(ds(t, es[r])), P.window_s);  // engine.hpp:370
    S2* plane = st + (size_t)(r * 2 + pol) * P.HW + c.i00;
    red_add2(plane, wt.w00, dm(wt.w00, tb));
    red_add2(plane + c.ox, wt.w10, dm(wt.w10, tb));
    red_add2(plane + c.oy, wt.w01, dm(wt.w01, tb));
    red_add2(plane + c.oy + c.ox, wt.w11, dm(wt.w11, tb));
  }
}

// --------------------------------------------------------------------------
// K3b: n_active + per-reference loss partial sums + coefficient planes

template <typename S2>
__global__ void __launch_bounds__(kPxBlock) k_loss_reduce(const S2* __restrict__ stack,
                                                          WinParams P,
                                                          S2* __restrict__ coef,
                                                          double* __restrict__ part_acc,
                                                          unsigned long long* __restrict__ part_act) {
  const int w = blockIdx.z, r = blockIdx.y;
  const int HW = P.HW;
  const size_t plane0 = ((size_t)w * (P.B + 1) + r) * 2 * HW;
  double acc = 0.0;
  unsigned act = 0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < HW; q += gridDim.x * blockDim.x) {
    const double2 v0 = ld2(stack + plane0 + q);
    const double2 v1 = ld2(stack + plane0 + HW + q);
    act += (v0.x + v1.x > 0.0) ? 1u : 0u;  // refresh_active (warp.hpp:190)
    // reference_loss (warp.hpp:306-309)
    const double a0 = v0.y / (v0.x + kLossEps), a1 = v1.y / (v1.x + kLossEps);
    acc += a0 * a0 + a1 * a1;
    // splat_position_grad's per-pixel factors (warp.hpp:346-349)
    const double i0 = __drcp_rn(v0.x + kLossEps), i1 = __drcp_rn(v1.x + kLossEps);  // == 1.0 / x
    const double b0 = v0.y * i0, b1 = v1.y * i1;
    store2(coef + plane0 + q, b0, b0 * i0);
    store2(coef + plane0 + HW + q, b1, b1 * i1);
  }
  // block reduction
  __shared__ double s_acc[kPxBlock / 32];
  __shared__ unsigned s_act[kPxBlock / 32];
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    act += __shfl_xor_sync(0xffffffffu, act, o);
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_acc[wid] = acc;
    s_act[wid] = act;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    unsigned long long c = 0;
    for (int i = 0; i < kPxBlock / 32; ++i) {
      a += s_acc[i];
      c += s_act[i];
    }
    const size_t slot = ((size_t)w * (P.B + 1) + r) * gridDim.x + blockIdx.x;
    part_acc[slot] = a;
    part_act[slot] = c;
  }
}

// reduce_loss (engine.hpp:442-468): fixed-order sum of the block partials.
// One CTA per window, one warp per reference: lanes take parts lane, lane+32, ...
// and reduce with a fixed shuffle tree, so the result is bit-stable.
// out per window: loss, no_survivors, n_active[R], scale[R] = 2/((n_a+eps) R)
__global__ void __launch_bounds__(1024) k_loss_finalize(const double* __restrict__ part_acc,
                                                        const unsigned long long* __restrict__ part_act,
                                                        int n_parts, WinParams P,
                                                        double* __restrict__ loss,
                                                        int* __restrict__ no_surv,
                                                        long long* __restrict__ n_active,
                                                        double* __restrict__ scale) {
  __shared__ double s_term[kMaxRefs];
  __shared__ unsigned long long s_na[kMaxRefs];
  const int w = blockIdx.x, R = P.B + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int r = wid; r < R; r += nwarps) {
    const size_t s0 = ((size_t)w * R + r) * n_parts;
    double acc = 0.0;
    unsigned long long na = 0;
    for (int i = lane; i < n_parts; i += 32) {
      acc += part_acc[s0 + i];
      na += part_act[s0 + i];
    }
    for (int o = 16; o > 0; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      na += __shfl_xor_sync(0xffffffffu, na, o);
    }
    if (lane == 0) {
      s_term[r] = acc / ((double)na + kLossEps);
      s_na[r] = na;
      n_active[(size_t)w * R + r] = (long long)na;
      scale[(size_t)w * R + r] = 2.0 / (((double)na + kLossEps) * (double)R);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long total = 0;
    double sum = 0.0;
    for (int r = 0; r < R; ++r) {
      total += (long long)s_na[r];
      sum += s_term[r];
    }
    no_surv[w] = total == 0 ? 1 : 0;
    loss[w] = total == 0 ? 0.0 : sum / (double)R;
  }
}

// --------------------------------------------------------------------------
// K4: per-event backward (backward_event, engine.hpp:475-504)

// dL/dpos at reference r (splat_position_grad, warp.hpp:334-358), from the
// coefficient planes: corner g = scale * q * (tb - a).
template <typename C2>
__device__ __forceinline__ double2 pos_grad(const C2* __restrict__ cp, const Cell& c,
                                            double tb, double scale) {
  const double2 k00 = ld2(cp + c.i00), k10 = ld2(cp + c.i00 + c.ox);
  const double2 k01 = ld2(cp + c.i00 + c.oy), k11 = ld2(cp + c.i00 + c.oy + c.ox);
  const double g00 = scale * k00.y * (tb - k00.x);
  const double g10 = scale * k10.y * (tb - k10.x);
  const double g01 = scale * k01.y * (tb - k01.x);
  const double g11 = scale * k11.y * (tb - k11.x);
  const double ax = 1.0 - c.wx, ay = 1.0 - c.wy;
  return make_double2(-ay * g00 + ay * g10 - c.wy * g01 + c.wy * g11,
                      -ax * g00 - c.wx * g10 + ax * g01 + c.wx * g11);
}

// BufferGradSink::add (warp.hpp:394-406) as vector atomics.
template <typename G2>
__device__ __forceinline__ void sink_add(G2* __restrict__ g, const Cell& c, double gx, double gy) {
  const Weights w = weights(c);
  red_add2(g + c.i00, w.w00 * gx, w.w00 * gy);
  red_add2(g + c.i00 + c.ox, w.w10 * gx, w.w10 * gy);
  red_add2(g + c.i00 + c.oy, w.w01 * gx, w.w01 * gy);
  red_add2(g + c.i00 + c.oy + c.ox, w.w11 * gx, w.w11 * gy);
}

template <typename C2, typename G2>
__global__ void __launch_bounds__(kEvBlock) k_bwd(const uint2* __restrict__ packed,
                                                  const uint64_t* __restrict__ ev_off,
                                                  WinParams P, const double2* __restrict__ flows,
                                                  const C2* __restrict__ coef,
                                                  const double* __restrict__ scale_tab,
                                                  const int* __restrict__ no_surv,
                                                  G2* __restrict__ grad) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* es = reinterpret_cast<double*>(smem);
  uint32_t* erel = reinterpret_cast<uint32_t*>(es + kMaxRefs);
  double2* pos = reinterpret_cast<double2*>(smem + kEvSmemHeader) + threadIdx.x;
  load_edges(P, es, erel);
  __syncthreads();
  const int w = blockIdx.y;
  if (no_surv[w]) return;  // engine.hpp:196
  const uint64_t base = ev_off[w];
  const uint64_t n = ev_off[w + 1] - base;
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int B = P.B, R = B + 1, HW = P.HW, W = P.W, H = P.H;
  const uint2 e = packed[base + k];
  const uint32_t dt_us = ev_dt(e);
  const double t = dm((double)dt_us, 1e-6);
  const int j = bin_of(dt_us, erel, B);
  const double2* fl = flows + (size_t)w * B * HW;
  const double x0 = (double)ev_x(e), y0 = (double)ev_y(e);
  const int stride = blockDim.x;
  if (!trajectory(x0, y0, t, j, fl, P, es, pos, stride)) return;
  const int pol = ev_pol(e);
  const C2* cw = coef + (size_t)w * R * 2 * HW + (size_t)pol * HW;  // + r*2*HW
  const double* sc = scale_tab + (size_t)w * R;
  G2* gw = grad + (size_t)w * B * HW;
  const double inv_win = 1.0 / P.window_s;
  (void)inv_win;

  // d[0] and d[B] start the two adjoint legs.
  double2 gb, gf;
  {
    const double2 p = pos[0];
    const Cell c = bilin_cell(p.x, p.y, W, H);
    gb = pos_grad(cw, c, fabs(t - es[0]) / P.window_s, sc[0]);
  }
  {
    const double2 p = pos[B * stride];
    const Cell c = bilin_cell(p.x, p.y, W, H);
    gf = pos_grad(cw + (size_t)B * 2 * HW, c, fabs(t - es[B]) / P.window_s, sc[B]);
  }
  // Interleaved reverse sweep: step s < j is backward-leg step i = s (position
  // r = i+1); otherwise forward-leg step i = B-1-(s-j) (position r = i).
  for (int s = 0; s < B - 1; ++s) {
    const bool back = s < j;
    const int i = back ? s : B - 1 - (s - j);
    const int r = back ? i + 1 : i;
    const double dt = back ? es[i] - es[i + 1] : es[i + 1] - es[i];
    const double2 p = pos[r * stride];
    const Cell c = bilin_cell(p.x, p.y, W, H);
    double2 g = back ? gb : gf;
    sink_add(gw + (size_t)i * HW, c, dt * g.x, dt * g.y);
    const Jac J = sample_jacobian(fl + (size_t)i * HW, c);
    // apply_step_transpose (warp.hpp:91-94), then + d[r]
    const double2 d = pos_grad(cw + (size_t)r * 2 * HW, c, fabs(t - es[r]) / P.window_s, sc[r]);
    const double nx = g.x * (1.0 + dt * J.dux) + g.y * dt * J.dvx + d.x;
    const double ny = g.y * (1.0 + dt * J.dvy) + g.x * dt * J.duy + d.y;
    if (back) gb = make_double2(nx, ny); else gf = make_double2(nx, ny);
  }
  // Both legs end with a partial step sampled at the source pixel in bin j;
  // x0 is integral, so its cell has a single nonzero weight (= 1).
  const double cb = es[j] - t, cf = es[j + 1] - t;
  const Cell c = bilin_cell(x0, y0, W, H);
  const int q = c.i00 + (c.wx > 0.5 ? c.ox : 0) + (c.wy > 0.5 ? c.oy : 0);
  red_add2(gw + (size_t)j * HW + q, cb * gb.x + cf * gf.x, cb * gb.y + cf * gf.y);
}

// --------------------------------------------------------------------------
// K5: flows backward (depth_pose_to_flows_backward, geometry.hpp:279-325)

// Each thread owns kK5Px pixels (stride blockDim.x); bins are the outer loop so
// the 6 pose partials of a bin stay in registers and are reduced once per warp
// per bin; d_depth accumulates over bins in registers (bin order, as the
// reference's outer loop, geometry.hpp:293-323).
constexpr int kK5Px = 2;  // pixels per thread (1 when that leaves SMs idle)

template <typename G2, int kPx>
__global__ void __launch_bounds__(kPxBlock) k_flows_bwd(const double* __restrict__ depth,
                                                        const uint8_t* __restrict__ mask,
                                                        const double* __restrict__ pose_tab,
                                                        WinParams P, double fx, double fy,
                                                        double cx, double cy,
                                                        const G2* __restrict__ grad,
                                                        double* __restrict__ d_depth,
                                                        double* __restrict__ pose_part) {
  __shared__ double s_pose[kMaxBins * kPoseTab];
  __shared__ double s_red[kPxBlock / 32][kMaxBins][kPoseSums];
  const int w = blockIdx.y;
  const int B = P.B, HW = P.HW;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < B * kPoseTab; i += blockDim.x)
    s_pose[i] = pose_tab[(size_t)w * B * kPoseTab + i];
  __syncthreads();
  const int q0 = blockIdx.x * blockDim.x * kPx + threadIdx.x;
  double dd[kPx], dep[kPx], rx[kPx], ry[kPx];
  bool ok[kPx];
#pragma unroll
  for (int m = 0; m < kPx; ++m) {
    const int q = q0 + m * blockDim.x;
    dd[m] = 0.0;
    ok[m] = false;
    dep[m] = rx[m] = ry[m] = 0.0;
    if (q < HW) {
      dep[m] = depth[(size_t)w * HW + q];
      ok[m] = (!mask || mask[(size_t)w * HW + q]) && dep[m] > 0.0;
      const int y = q / P.W, x = q - y * P.W;
      rx[m] = 1.0 * ((double)x - cx) / fx;  // backproject(x, 1.0, k)
      ry[m] = 1.0 * ((double)y - cy) / fy;
    }
  }
  const G2* gw = grad + (size_t)w * B * HW;
  for (int b = 0; b < B; ++b) {
    const double* pt = s_pose + b * kPoseTab;
    double c6[16];  // pose moments (k_bwd_cells): N = sum d v r^T (0..8), v (9..11)
#pragma unroll
    for (int k = 0; k < 16; ++k) c6[k] = 0.0;
#pragma unroll
    for (int m = 0; m < kPx; ++m) {
      const int q = q0 + m * blockDim.x;
      if (!ok[m]) continue;
      const auto gg = gw[(size_t)b * HW + q];
      const double gu = gg.x, gv = gg.y;
      if (gu == 0.0 && gv == 0.0) continue;
      const double d = dep[m];
      const double rr0 = pt[0] * rx[m] + pt[1] * ry[m] + pt[2];
      const double rr1 = pt[3] * rx[m] + pt[4] * ry[m] + pt[5];
      const double rr2 = pt[6] * rx[m] + pt[7] * ry[m] + pt[8];
      const double p0 = d * rr0 + pt[36], p1 = d * rr1 + pt[37], p2 = d * rr2 + pt[38];
      if (!(p2 > 0.0)) continue;
      const double inv_dt = pt[39];
      const double iz = __drcp_rn(p2);  // == 1.0 / p2 (correctly rounded)
      // the Jacobian folded into the adjoint, as in k_bwd_cells: v = d_t of this pixel
      const double sc = iz * inv_dt;
      const double v0 = gu * fx * sc, v1 = gv * fy * sc;
      const double v2 = -(v0 * p0 + v1 * p1) * iz;
      dd[m] += v0 * rr0 + v1 * rr1 + v2 * rr2;
      const double dv[3] = {d * v0, d * v1, d * v2};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        c6[3 * a] += dv[a] * rx[m];
        c6[3 * a + 1] += dv[a] * ry[m];
        c6[3 * a + 2] += dv[a];
      }
      c6[9] += v0;
      c6[10] += v1;
      c6[11] += v2;
    }
    // transposed warp sums (fixed order), lane 2c holds moment c
#pragma unroll
    for (int h = 8, off = 16; h >= 1; h >>= 1, off >>= 1) {
      const bool up = lane & off;
#pragma unroll
      for (int k = 0; k < h; ++k) {
        const double mine = up ? c6[h + k] : c6[k], other = up ? c6[k] : c6[h + k];
        c6[k] = mine + __shfl_xor_sync(0xffffffffu, other, off);
      }
    }
    const double v = c6[0] + __shfl_xor_sync(0xffffffffu, c6[0], 1);
    const int comp = ((lane & 16) ? 8 : 0) + ((lane & 8) ? 4 : 0) + ((lane & 4) ? 2 : 0) +
                     ((lane & 2) ? 1 : 0);
    if ((lane & 1) == 0 && comp < kPoseSums) s_red[wid][b][comp] = v;
  }
#pragma unroll
  for (int m = 0; m < kPx; ++m) {
    const int q = q0 + m * blockDim.x;
    if (q < HW) d_depth[(size_t)w * HW + q] = dd[m];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < B * kPoseSums; i += blockDim.x) {
    const int b = i / kPoseSums, a = i % kPoseSums;
    double v = 0.0;
    for (int q = 0; q < kPxBlock / 32; ++q) v += s_red[q][b][a];  // warp order
    pose_part[(((size_t)w * B + b) * kPoseSums + a) * gridDim.x + blockIdx.x] = v;  // [w][bin][moment][part]
  }
}

// Owner backward pose gradients: one block per (window, bin); warp c sums moment
// c over the parts (lane-strided + shuffle tree, fixed order), then
// d_omega_a = sum_ij dR_a[i][j] N[i][j] and d_t = v (see k_bwd_cells).
__global__ void k_pose_contract(const double* __restrict__ pose_part, int n_parts, int B,
                                const double* __restrict__ pose_tab, double* __restrict__ d_poses) {
  __shared__ double s[kPoseSums];
  const int wb = blockIdx.x;  // window * B + bin
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  if (c < kPoseSums) {
    double v = 0.0;
    const double* src = pose_part + ((size_t)wb * kPoseSums + c) * n_parts;  // contiguous parts
    for (int p = lane; p < n_parts; p += 32) v += src[p];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s[c] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int a = threadIdx.x;
    double r;
    if (a < 3) {
      const double* dR = pose_tab + (size_t)wb * kPoseTab + 9 + 9 * a;
      r = 0.0;
      for (int k = 0; k < 9; ++k) r += dR[k] * s[k];
    } else {
      r = s[9 + a - 3];
    }
    d_poses[(size_t)wb * 6 + a] = r;
  }
}

// --------------------------------------------------------------------------
// products / format conversion

template <typename S2>
__global__ void k_unpack_stack(const S2* __restrict__ stack, size_t planes, int HW,
                               double* __restrict__ count, double* __restrict__ tsum) {
  const size_t total = planes * HW;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = ld2(stack + i);
    count[i] = v.x;
    tsum[i] = v.y;
  }
}

template <typename G2>
__global__ void k_unpack_grad(const G2* __restrict__ g, int B, int HW, double* __restrict__ out) {
  const size_t total = (size_t)B * HW;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / HW, p = i % HW;
    const double2 v = ld2(g + i);
    out[(2 * b) * HW + p] = v.x;
    out[(2 * b + 1) * HW + p] = v.y;
  }
}

// Trajectories products in original event order (pos optional).
__global__ void __launch_bounds__(kEvBlock) k_traj_products(const uint2* __restrict__ packed,
                                                            uint64_t n, WinParams P,
                                                            const double2* __restrict__ flows,
                                                            uint8_t* __restrict__ alive,
                                                            int32_t* __restrict__ bin,
                                                            double* __restrict__ pos_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* es = reinterpret_cast<double*>(smem);
  uint32_t* erel = reinterpret_cast<uint32_t*>(es + kMaxRefs);
  double2* pos = reinterpret_cast<double2*>(smem + kEvSmemHeader) + threadIdx.x;
  load_edges(P, es, erel);
  __syncthreads();
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint2 e = packed[k];
  const uint32_t dt = ev_dt(e);
  const double t = dm((double)dt, 1e-6);
  const int j = bin_of(dt, erel, P.B);
  const bool ok = trajectory((double)ev_x(e), (double)ev_y(e), t, j, flows, P, es, pos, blockDim.x);
  alive[k] = ok ? 1 : 0;
  bin[k] = j;
  if (pos_out)
    for (int r = 0; r <= P.B; ++r) {
      const double2 p = pos[r * blockDim.x];
      pos_out[(k * (P.B + 1) + r) * 2] = p.x;
      pos_out[(k * (P.B + 1) + r) * 2 + 1] = p.y;
    }
}

// --------------------------------------------------------------------------
// host launchers

size_t ev_smem_bytes(const WinParams& P) {
  return kEvSmemHeader + sizeof(double2) * (size_t)(P.B + 1) * kEvBlock;
}

// Opt every per-event kernel into the dynamic shared memory its largest
// window (B = kMaxBins) needs; done once per process.
static void ensure_smem_attrs() {
  static bool done = false;
  if (done) return;
  const int bytes = (int)(kEvSmemHeader + sizeof(double2) * (size_t)kMaxRefs * kEvBlock);
  cudaFuncSetAttribute(k_fwd_splat<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_fwd_splat<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_bwd<float2, float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_bwd<float2, double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_bwd<double2, float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_bwd<double2, double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_traj_products, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done = true;
}

void launch_stage(cudaStream_t s, const evcm_event* ev, const uint64_t* ev_off, const WinParams& P,
                  uint64_t max_n, uint2* packed, unsigned long long* err) {
  const int blocks = (int)std::min<uint64_t>((max_n + 255) / 256, 148 * 16);
  if (blocks == 0) return;
  ++g_launches;
  k_stage<<<dim3(blocks, P.n_windows), 256, 0, s>>>(ev, ev_off, P, packed, err);
}

void launch_interleave_flows(cudaStream_t s, const double* uv, int B, int HW, double2* out,
                             float2* out32) {
  const size_t total = (size_t)B * HW;
  const int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 16);
  ++g_launches;
  k_interleave_flows<<<blocks, 256, 0, s>>>(uv, B, HW, out, out32);
}

void launch_motion_field(cudaStream_t s, const double* depth, const uint8_t* mask,
                         const double* pose_tab, const WinParams& P, const double* K,
                         double2* flows, uint8_t* valid, float2* flows32) {
  const int bx = (P.HW + 255) / 256;
  ++g_launches;
  k_motion_field<<<dim3(bx, P.n_windows), 256, 0, s>>>(depth, mask, pose_tab, P, K[0], K[1], K[2],
                                                      K[3], flows, valid, flows32);
}

template <typename S2>
void launch_fwd_splat(cudaStream_t s, const uint2* packed, const uint64_t* ev_off,
                      const WinParams& P, uint64_t max_n, const double2* flows, S2* stack) {
  if (max_n == 0) return;
  ensure_smem_attrs();
  const unsigned blocks = (unsigned)((max_n + kEvBlock - 1) / kEvBlock);
  ++g_launches;
  k_fwd_splat<S2><<<dim3(blocks, P.n_windows), kEvBlock, ev_smem_bytes(P), s>>>(packed, ev_off, P,
                                                                             flows, stack);
}

void launch_loss_finalize(cudaStream_t s, const double* part_acc, const unsigned long long* part_act,
                          int n_parts, const WinParams& P, double* loss, int* no_surv,
                          long long* n_active, double* scale) {
  ++g_launches;
  k_loss_finalize<<<P.n_windows, 32 * std::min(P.B + 1, 32), 0, s>>>(part_acc, part_act, n_parts,
                                                                     P, loss, no_surv, n_active,
                                                                     scale);
}

void launch_pose_contract(cudaStream_t s, const double* pose_part, int n_parts, int B, int n_windows,
                          const double* pose_tab, double* d_poses) {
  ++g_launches;
  k_pose_contract<<<n_windows * B, 32 * kPoseSums, 0, s>>>(pose_part, n_parts, B, pose_tab, d_poses);
}

int loss_parts(const WinParams& P) { return std::max(1, std::min((P.HW + kPxBlock - 1) / kPxBlock, 64)); }

template <typename S2>
void launch_loss(cudaStream_t s, const S2* stack, const WinParams& P, S2* coef,
                 double* part_acc, unsigned long long* part_act, double* loss, int* no_surv,
                 long long* n_active, double* scale) {
  const int parts = loss_parts(P);
  ++g_launches;
  k_loss_reduce<S2><<<dim3(parts, P.B + 1, P.n_windows), kPxBlock, 0, s>>>(stack, P, coef,
                                                                          part_acc, part_act);
  ++g_launches;
  k_loss_finalize<<<P.n_windows, 32 * std::min(P.B + 1, 32), 0, s>>>(part_acc, part_act, parts, P,
                                                                     loss, no_surv, n_active, scale);
}

template <typename C2, typename G2>
void launch_bwd(cudaStream_t s, const uint2* packed, const uint64_t* ev_off, const WinParams& P,
                uint64_t max_n, const double2* flows, const C2* coef, const double* scale,
                const int* no_surv, G2* grad) {
  if (max_n == 0) return;
  ensure_smem_attrs();
  const unsigned blocks = (unsigned)((max_n + kEvBlock - 1) / kEvBlock);
  ++g_launches;
  k_bwd<C2, G2><<<dim3(blocks, P.n_windows), kEvBlock, ev_smem_bytes(P), s>>>(
      packed, ev_off, P, flows, coef, scale, no_surv, grad);
}

// parts at kK5Px pixels per thread, or at one when that fills fewer than two
// blocks per SM; flows_bwd_parts is the allocation bound (the larger count)
static int flows_bwd_px(const WinParams& P) {
  const int parts2 = (P.HW + kPxBlock * kK5Px - 1) / (kPxBlock * kK5Px);
  return (long)parts2 * P.n_windows < 2L * 148 ? 1 : kK5Px;
}
int flows_bwd_parts(const WinParams& P) { return (P.HW + kPxBlock - 1) / kPxBlock; }

template <typename G2>
void launch_flows_bwd(cudaStream_t s, const double* depth, const uint8_t* mask,
                      const double* pose_tab, const WinParams& P, const double* K, const G2* grad,
                      double* d_depth, double* pose_part, double* d_poses) {
  const int px = flows_bwd_px(P);
  const int parts = (P.HW + kPxBlock * px - 1) / (kPxBlock * px);
  ++g_launches;
  if (px == 1)
    k_flows_bwd<G2, 1><<<dim3(parts, P.n_windows), kPxBlock, 0, s>>>(
        depth, mask, pose_tab, P, K[0], K[1], K[2], K[3], grad, d_depth, pose_part);
  else
    k_flows_bwd<G2, kK5Px><<<dim3(parts, P.n_windows), kPxBlock, 0, s>>>(
        depth, mask, pose_tab, P, K[0], K[1], K[2], K[3], grad, d_depth, pose_part);
  launch_pose_contract(s, pose_part, parts, P.B, P.n_windows, pose_tab, d_poses);
}

template <typename S2>
void launch_unpack_stack(cudaStream_t s, const S2* stack, size_t planes, int HW, double* count,
                         double* tsum) {
  const size_t total = planes * HW;
  const int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 16);
  if (blocks) k_unpack_stack<S2><<<blocks, 256, 0, s>>>(stack, planes, HW, count, tsum);
}

template <typename G2>
void launch_unpack_grad(cudaStream_t s, const G2* g, int B, int HW, double* out) {
  const size_t total = (size_t)B * HW;
  const int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 16);
  if (blocks) k_unpack_grad<G2><<<blocks, 256, 0, s>>>(g, B, HW, out);
}

void launch_traj_products(cudaStream_t s, const uint2* packed, uint64_t n, const WinParams& P,
                          const double2* flows, uint8_t* alive, int32_t* bin, double* pos) {
  if (n == 0) return;
  ensure_smem_attrs();
  const unsigned blocks = (unsigned)((n + kEvBlock - 1) / kEvBlock);
  ++g_launches;
  k_traj_products<<<blocks, kEvBlock, ev_smem_bytes(P), s>>>(packed, n, P, flows, alive, bin, pos);
}

#define INST_S(S2)                                                                              \
  template void launch_fwd_splat<S2>(cudaStream_t, const uint2*, const uint64_t*,                \
                                     const WinParams&, uint64_t, const double2*, S2*);          \
  template void launch_loss<S2>(cudaStream_t, const S2*, const WinParams&, S2*, double*,        \
                                unsigned long long*, double*, int*, long long*, double*);       \
  template void launch_unpack_stack<S2>(cudaStream_t, const S2*, size_t, int, double*, double*);
#define INST_B(C2, G2)                                                                          \
  template void launch_bwd<C2, G2>(cudaStream_t, const uint2*, const uint64_t*, const WinParams&, \
                                   uint64_t, const double2*, const C2*, const double*,          \
                                   const int*, G2*);
INST_B(float2, float2)
INST_B(float2, double2)
INST_B(double2, float2)
INST_B(double2, double2)
#define INST_G(G2)                                                                              \
  template void launch_flows_bwd<G2>(cudaStream_t, const double*, const uint8_t*, const double*, \
                                     const WinParams&, const double*, const G2*, double*,       \
                                     double*, double*);                                         \
  template void launch_unpack_grad<G2>(cudaStream_t, const G2*, int, int, double*);
INST_S(float2)
INST_S(double2)
INST_G(float2)
INST_G(double2)

}  // namespace evcm_b200
