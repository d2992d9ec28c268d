// evcm_cuda_backend.hpp — reference-side binding of the B200 CMax path.
//
// Header-only C++20 adapter a maintainer of the reference (evcm,
// /root/reference/proj/include/evcm) includes to get a `cuda` backend with the
// reference's own types and error classes. It only talks to the C-ABI of
// include/evcm_cuda.h (libevcm_cuda.so); no CUDA or torch types appear here.
//
//   evcm::cuda::Engine            ~ evcm::Engine              (engine.hpp:134-213)
//   evcm::cuda::depth_pose_to_flows / _backward               (geometry.hpp:229-325)
//   evcm::cuda::contrast_loss_backward / build_iwe_stack / rsat (engine.hpp:606-631)
//   evcm::cuda::geometry_consistency_loss[_backward]            (geometry.hpp:416-534)
//   evcm::cuda::predictor_loss_and_gradients                    (optimize.hpp:205-241)
//
// Requires the reference headers on the include path (it reuses EventSlice,
// FlowSequence, ForwardResult, ... from evcm).
#pragma once

#include <cstring>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "evcm/engine.hpp"
#include "evcm/geometry.hpp"
#include "evcm/optimize.hpp"
#include "evcm/predictor.hpp"
#include "evcm_cuda.h"

namespace evcm::cuda {

// Status -> the reference's exception taxonomy (types.hpp:18-76).
[[noreturn]] inline void raise(int rc) {
  const std::string msg = std::string("cuda backend: ") + evcm_cuda_last_error();
  switch (rc) {
    case EVCM_ERR_CONFIG:
    case EVCM_ERR_STATE: throw ConfigError(msg);
    case EVCM_ERR_DIMENSION: throw DimensionMismatchError(msg);
    case EVCM_ERR_COORDINATE: throw CoordinateRangeError(msg);
    case EVCM_ERR_POLARITY: throw InvalidPolarityError(msg);
    case EVCM_ERR_UNSORTED: throw UnsortedEventsError(msg);
    case EVCM_ERR_TIME_RANGE: throw TimeRangeError(msg);
    case EVCM_ERR_EMPTY: throw EmptySliceError(msg);
    default: throw Error(msg);
  }
}
inline void check(int rc) {
  if (rc != EVCM_OK) raise(rc);
}

// FlowSequence -> contiguous [B][2][H][W] (types.hpp:228-253).
inline std::vector<double> pack_flows(const FlowSequence& f) {
  const std::size_t HW = f.fields.empty() ? 0 : f.fields[0].u.size();
  std::vector<double> uv(static_cast<std::size_t>(f.n_bins()) * 2 * HW);
  for (int b = 0; b < f.n_bins(); ++b) {
    std::memcpy(uv.data() + (2 * b) * HW, &f.fields[b].u[0], HW * sizeof(double));
    std::memcpy(uv.data() + (2 * b + 1) * HW, &f.fields[b].v[0], HW * sizeof(double));
  }
  return uv;
}

inline evcm_flows c_flows(const FlowSequence& f, const std::vector<double>& uv) {
  return evcm_flows{f.n_bins(), f.edges_us.data(), uv.data(), f.width(), f.height()};
}

inline evcm_slice c_slice(const EventSlice& s) {
  static_assert(sizeof(Event) == sizeof(evcm_event), "evcm::Event layout");
  return evcm_slice{s.width, s.height, s.t_start_us, s.t_end_us,
                    reinterpret_cast<const evcm_event*>(s.events.data()), s.events.size()};
}

// EngineOptions of the reference plus the cuda-only knobs.
struct CudaOptions {
  int device = 0;
  bool deterministic = true;  // engine.hpp:60 default
  int algo = 2;               // 0 owner, 1 atomic, 2 auto
};

class Engine {
 public:
  explicit Engine(CudaOptions o = {}) {
    evcm_cuda_options co;
    evcm_cuda_default_options(&co);
    co.device = o.device;
    co.deterministic = o.deterministic ? 1 : 0;
    co.algo = o.algo;
    evcm_cuda_engine* h = nullptr;
    check(evcm_cuda_create(&co, &h));
    h_.reset(h);
  }

  // Engine::forward (engine.hpp:145-183): stack, trajectories, loss and the
  // per-phase PhaseStats (engine.hpp:154,169,179).
  ForwardResult forward(const EventSlice& slice, const FlowSequence& flows) const {
    const std::vector<double> uv = pack_flows(flows);
    const evcm_slice s = c_slice(slice);
    const evcm_flows f = c_flows(flows, uv);
    evcm_loss loss{};
    check(evcm_cuda_forward(h_.get(), &s, &f, EVCM_MEM_HOST, &loss));
    last_fwd_ = Fingerprint{loss.forward_id, loss.value, loss.no_survivors != 0};
    ForwardResult res;
    const int W = slice.width, H = slice.height, R = flows.n_bins() + 1;
    const std::size_t HW = static_cast<std::size_t>(W) * H, n = slice.events.size();
    res.stack = IweStack(W, H, R);
    std::vector<double> count(R * 2 * HW), tsum(R * 2 * HW), pos(n * R * 2);
    res.traj.resize(n, R);
    std::size_t n_alive = 0;
    check(evcm_cuda_forward_products(h_.get(), count.data(), tsum.data(),
                                     res.stack.n_active.data(), res.traj.alive.data(),
                                     res.traj.bin.data(), pos.data(), &n_alive));
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < 2; ++c) {
        std::memcpy(&res.stack.count[r][c][0], count.data() + (r * 2 + c) * HW, HW * sizeof(double));
        std::memcpy(&res.stack.tsum[r][c][0], tsum.data() + (r * 2 + c) * HW, HW * sizeof(double));
      }
    std::memcpy(res.traj.pos.data(), pos.data(), pos.size() * sizeof(double));
    res.traj.n_alive = n_alive;
    res.loss.value = loss.value;
    res.loss.no_survivors = loss.no_survivors != 0;
    double t_us[4];
    std::size_t bytes[4];
    check(evcm_cuda_phase_stats(h_.get(), t_us, bytes));
    res.warp_stats = PhaseStats{t_us[0], bytes[0]};
    res.splat_stats = PhaseStats{t_us[1], bytes[1]};
    res.loss_stats = PhaseStats{t_us[2], bytes[2]};
    return res;
  }

  // Engine::backward (engine.hpp:185-205) for the window of the last forward.
  // The device keeps the state of the engine's LAST forward only: `fwd` must be
  // that forward's result (matched by its loss), otherwise ConfigError.
  BackwardResult backward(const EventSlice& slice, const FlowSequence& flows,
                          const ForwardResult& fwd) const {
    const std::vector<double> uv = pack_flows(flows);
    const evcm_slice s = c_slice(slice);
    const evcm_flows f = c_flows(flows, uv);
    const std::size_t HW = static_cast<std::size_t>(slice.width) * slice.height;
    std::vector<double> g(static_cast<std::size_t>(flows.n_bins()) * 2 * HW);
    const bool same = std::memcmp(&fwd.loss.value, &last_fwd_.value, sizeof(double)) == 0 &&
                      fwd.loss.no_survivors == last_fwd_.no_survivors;
    check(evcm_cuda_backward_of(h_.get(), &s, &f, same ? last_fwd_.id : 0, EVCM_MEM_HOST,
                                g.data()));
    BackwardResult res;
    res.grad = GradientBuffer(slice.width, slice.height, flows.n_bins());
    for (int b = 0; b < flows.n_bins(); ++b) {
      std::memcpy(&res.grad.gu[b][0], g.data() + (2 * b) * HW, HW * sizeof(double));
      std::memcpy(&res.grad.gv[b][0], g.data() + (2 * b + 1) * HW, HW * sizeof(double));
    }
    double t_us[4];
    std::size_t bytes[4];
    check(evcm_cuda_phase_stats(h_.get(), t_us, bytes));
    res.stats = PhaseStats{t_us[3], bytes[3]};
    return res;
  }

  std::pair<ForwardResult, BackwardResult> loss_and_grad(const EventSlice& slice,
                                                         const FlowSequence& flows) const {
    ForwardResult f = forward(slice, flows);
    BackwardResult b = backward(slice, flows, f);
    return {std::move(f), std::move(b)};
  }

  evcm_cuda_engine* handle() const { return h_.get(); }

 private:
  struct Fingerprint {
    std::uint64_t id = 0;
    double value = 0.0;
    bool no_survivors = false;
  };
  mutable Fingerprint last_fwd_;
  struct Del {
    void operator()(evcm_cuda_engine* e) const { evcm_cuda_destroy(e); }
  };
  std::unique_ptr<evcm_cuda_engine, Del> h_;
};

inline std::vector<double> pack_poses(const std::vector<PoseStep>& poses) {
  std::vector<double> p(poses.size() * 6);
  for (std::size_t i = 0; i < poses.size(); ++i) {
    const double v[6] = {poses[i].omega.x, poses[i].omega.y, poses[i].omega.z,
                         poses[i].trans.x, poses[i].trans.y, poses[i].trans.z};
    std::memcpy(p.data() + 6 * i, v, sizeof v);
  }
  return p;
}

// depth_pose_to_flows (geometry.hpp:229-264).
inline GeometryFlows depth_pose_to_flows(const Engine& e, const DepthMap& depth,
                                         const std::vector<PoseStep>& poses,
                                         const CameraIntrinsics& k, std::uint64_t t0,
                                         std::uint64_t t1) {
  const int W = depth.width(), H = depth.height(), B = static_cast<int>(poses.size());
  const std::size_t HW = static_cast<std::size_t>(W) * H;
  const std::vector<double> p = pack_poses(poses);
  const double K[4] = {k.fx, k.fy, k.cx, k.cy};
  std::vector<double> uv(static_cast<std::size_t>(B) * 2 * HW);
  std::vector<std::uint8_t> valid(static_cast<std::size_t>(B) * HW);
  std::vector<std::uint64_t> edges(static_cast<std::size_t>(B) + 1);
  check(evcm_cuda_depth_pose_to_flows(e.handle(), W, H, &depth.d[0],
                                      depth.has_mask() ? &depth.valid[0] : nullptr, B, p.data(),
                                      K, t0, t1, EVCM_MEM_HOST, uv.data(), valid.data(),
                                      edges.data()));
  GeometryFlows out;
  out.flows = FlowSequence::zeros(W, H, t0, t1, B);
  for (int b = 0; b < B; ++b) {
    std::memcpy(&out.flows.fields[b].u[0], uv.data() + (2 * b) * HW, HW * sizeof(double));
    std::memcpy(&out.flows.fields[b].v[0], uv.data() + (2 * b + 1) * HW, HW * sizeof(double));
    Image<std::uint8_t> m(W, H, 0);
    std::memcpy(&m[0], valid.data() + b * HW, HW);
    out.valid.push_back(std::move(m));
  }
  return out;
}

// depth_pose_to_flows_backward (geometry.hpp:279-325).
inline FlowsBackwardResult depth_pose_to_flows_backward(const Engine& e, const DepthMap& depth,
                                                        const std::vector<PoseStep>& poses,
                                                        const CameraIntrinsics& k,
                                                        const FlowSequence& flows,
                                                        const GradientBuffer& grad) {
  const int W = depth.width(), H = depth.height(), B = static_cast<int>(poses.size());
  if (flows.n_bins() != B || grad.n_bins() != B)
    throw ConfigError("flows backward: bins, poses, and gradients must align");
  if (grad.width() != W || grad.height() != H)
    throw DimensionMismatchError("flows backward: grids must match the depth map");
  const std::size_t HW = static_cast<std::size_t>(W) * H;
  std::vector<double> g(static_cast<std::size_t>(B) * 2 * HW);
  for (int b = 0; b < B; ++b) {
    std::memcpy(g.data() + (2 * b) * HW, &grad.gu[b][0], HW * sizeof(double));
    std::memcpy(g.data() + (2 * b + 1) * HW, &grad.gv[b][0], HW * sizeof(double));
  }
  const std::vector<double> p = pack_poses(poses);
  const double K[4] = {k.fx, k.fy, k.cx, k.cy};
  FlowsBackwardResult out;
  out.d_depth = Image<double>(W, H, 0.0);
  std::vector<double> dp(static_cast<std::size_t>(B) * 6);
  check(evcm_cuda_depth_pose_to_flows_backward(e.handle(), W, H, &depth.d[0],
                                               depth.has_mask() ? &depth.valid[0] : nullptr, B,
                                               p.data(), K, flows.edges_us.data(), g.data(),
                                               EVCM_MEM_HOST, &out.d_depth[0], dp.data()));
  out.d_poses.resize(static_cast<std::size_t>(B));
  for (int b = 0; b < B; ++b)
    out.d_poses[b] = PoseGrad{{dp[6 * b], dp[6 * b + 1], dp[6 * b + 2]},
                              {dp[6 * b + 3], dp[6 * b + 4], dp[6 * b + 5]}};
  return out;
}

// Module-level helpers (engine.hpp:606-631).
inline ForwardResult build_iwe_stack(const EventSlice& s, const FlowSequence& f,
                                     CudaOptions o = {}) {
  return Engine(o).forward(s, f);
}
inline GradientBuffer contrast_loss_backward(const EventSlice& s, const FlowSequence& f,
                                             CudaOptions o = {}) {
  const Engine e(o);
  const ForwardResult fw = e.forward(s, f);
  return e.backward(s, f, fw).grad;
}
inline double rsat(const EventSlice& s, const FlowSequence& f, CudaOptions o = {}) {
  if (s.events.empty()) throw EmptySliceError("rsat: no events in slice");
  const Engine e(o);
  const double with_flow = e.forward(s, f).loss.value;
  const LossResult base = e.forward(s, f.zeros_like()).loss;
  if (base.no_survivors || base.value == 0.0) throw EmptySliceError("rsat: zero-flow loss is zero");
  return with_flow / base.value;
}

// geometry_consistency_loss_backward (geometry.hpp:458-534); want_grad = false
// gives geometry_consistency_loss (:416-453) with zero gradients.
inline GeoLossGrad geometry_consistency_loss_backward(const Engine& e, const DepthMap& d0,
                                                      const DepthMap& d1, const PoseStep& pose,
                                                      const CameraIntrinsics& k,
                                                      double upstream = 1.0,
                                                      bool want_grad = true) {
  if (!d0.d.same_shape(d1.d))
    throw DimensionMismatchError("depth consistency: depth maps must share a shape");
  const int W = d0.width(), H = d0.height();
  const double p[6] = {pose.omega.x, pose.omega.y, pose.omega.z,
                       pose.trans.x, pose.trans.y, pose.trans.z};
  const double K[4] = {k.fx, k.fy, k.cx, k.cy};
  GeoLossGrad out;
  out.terms.projected = Image<double>(W, H, 0.0);
  out.terms.interpolated = Image<double>(W, H, 0.0);
  out.terms.valid = Image<std::uint8_t>(W, H, 0);
  out.d_d0 = Image<double>(W, H, 0.0);
  out.d_d1 = Image<double>(W, H, 0.0);
  double value = 0.0, dp[6] = {0, 0, 0, 0, 0, 0};
  std::int64_t n_valid = 0;
  evcm_geo_out o{&value, &n_valid, &out.terms.projected[0], &out.terms.interpolated[0],
                 &out.terms.valid[0], want_grad ? &out.d_d0[0] : nullptr,
                 want_grad ? &out.d_d1[0] : nullptr, want_grad ? dp : nullptr, nullptr};
  check(evcm_cuda_geometry_consistency_loss(
      e.handle(), W, H, &d0.d[0], d0.has_mask() ? &d0.valid[0] : nullptr, &d1.d[0],
      d1.has_mask() ? &d1.valid[0] : nullptr, 1, p, K, upstream, want_grad ? 1 : 0,
      EVCM_MEM_HOST, &o));
  out.terms.value = value;
  out.terms.n_valid = n_valid;
  out.terms.empty_valid_set = n_valid == 0;
  out.d_omega = Vec3{dp[0], dp[1], dp[2]};
  out.d_trans = Vec3{dp[3], dp[4], dp[5]};
  return out;
}

inline GeoLossTerms geometry_consistency_loss(const Engine& e, const DepthMap& d0,
                                              const DepthMap& d1, const PoseStep& pose,
                                              const CameraIntrinsics& k) {
  return geometry_consistency_loss_backward(e, d0, d1, pose, k, 1.0, false).terms;
}

// predictor_loss_and_gradients (optimize.hpp:205-241) as one device call:
// decode -> depth_pose_to_flows -> forward -> backward -> [L_geo] -> adjoint.
inline WindowGradients predictor_loss_and_gradients(const Engine& e, const DirectPredictor& pred,
                                                    const EventSlice& slice,
                                                    const CameraIntrinsics& k,
                                                    double lambda_geo) {
  pred.validate();
  const int pw = pred.depth_params.width(), ph = pred.depth_params.height();
  const std::vector<double> p = pack_poses(pred.poses);
  const double K[4] = {k.fx, k.fy, k.cx, k.cy};
  const evcm_slice cs = c_slice(slice);
  double losses[3];
  WindowGradients out;
  out.grads.d_depth_params = Image<double>(pw, ph, 0.0);
  std::vector<double> dp(6 * pred.poses.size());
  check(evcm_cuda_predictor_loss_and_gradients_geo(
      e.handle(), pw, ph, pred.upsample, &pred.depth_params[0], pred.n_bins(), p.data(), K, &cs,
      lambda_geo, EVCM_MEM_HOST, losses, &out.grads.d_depth_params[0], dp.data()));
  out.l_cm = losses[0];
  out.l_geo = losses[1];
  out.total = losses[2];
  for (std::size_t b = 0; b < pred.poses.size(); ++b)
    out.grads.d_poses.push_back(PoseGrad{{dp[6 * b], dp[6 * b + 1], dp[6 * b + 2]},
                                         {dp[6 * b + 3], dp[6 * b + 4], dp[6 * b + 5]}});
  return out;
}

}  // namespace evcm::cuda
