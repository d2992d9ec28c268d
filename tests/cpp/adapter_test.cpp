// GPU test (built against the reference headers by oracle/Makefile `adapter`,
// run by tests/test_cpp_adapter.py on the GPU box): the C++ binding
// include/evcm_cuda_backend.hpp used exactly as a reference maintainer would,
// checked against the reference's own Engine on the reference's own fixtures.
// Prints "OK <n checks>" on success, exits 1 on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "evcm/fdcheck.hpp"
#include "evcm/geometry.hpp"
#include "chain_support.hpp"
#include "evcm_cuda_backend.hpp"

using namespace evcm;

static int g_checks = 0;
#define CHECK(cond, ...)                          \
  do {                                            \
    ++g_checks;                                   \
    if (!(cond)) {                                \
      std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);                   \
      std::printf("\n");                          \
      std::exit(1);                               \
    }                                             \
  } while (0)

static double rel_inf_grad(const GradientBuffer& a, const GradientBuffer& b) {
  double num = 0, den = 0;
  for (int k = 0; k < a.n_bins(); ++k)
    for (std::size_t i = 0; i < a.gu[k].size(); ++i) {
      num = std::max({num, std::abs(a.gu[k][i] - b.gu[k][i]), std::abs(a.gv[k][i] - b.gv[k][i])});
      den = std::max({den, std::abs(b.gu[k][i]), std::abs(b.gv[k][i])});
    }
  return den > 0 ? num / den : num;
}

int main() {
  EngineOptions ro;
  ro.backend = Backend::naive;
  const Engine ref(ro);
  for (bool det : {true, false}) {
    cuda::CudaOptions co;
    co.deterministic = det;
    const cuda::Engine gpu(co);
    for (std::uint64_t seed : {100ull, 7ull, 503ull, 1300ull, 1701ull, 2500ull}) {
      const FdInstance inst = random_fd_instance(seed);
      const auto [rf, rb] = ref.loss_and_grad(inst.slice, inst.flows);
      const auto [gf, gb] = gpu.loss_and_grad(inst.slice, inst.flows);
      CHECK(std::abs(gf.loss.value - rf.loss.value) <= 1e-5 * std::abs(rf.loss.value),
            "loss seed %llu", (unsigned long long)seed);
      CHECK(gf.traj.n_alive == rf.traj.n_alive, "n_alive");
      for (std::size_t k = 0; k < inst.slice.events.size(); ++k) {
        CHECK(gf.traj.alive[k] == rf.traj.alive[k] && gf.traj.bin[k] == rf.traj.bin[k], "alive/bin");
        for (int r = 0; r < rf.traj.n_refs; ++r)
          CHECK(gf.traj.position(k, r) == rf.traj.position(k, r), "position bit-exact");
      }
      for (int r = 0; r < rf.stack.n_refs; ++r)
        CHECK(gf.stack.n_active[r] == rf.stack.n_active[r], "n_active");
      CHECK(rel_inf_grad(gb.grad, rb.grad) <= 1e-5, "grad rel %g", rel_inf_grad(gb.grad, rb.grad));
    }
    // errors map onto the reference taxonomy
    FdInstance bad = random_fd_instance(42);
    bad.slice.events[0].x = bad.slice.width;
    bool threw = false;
    try {
      gpu.forward(bad.slice, bad.flows);
    } catch (const CoordinateRangeError&) {
      threw = true;
    }
    CHECK(threw, "CoordinateRangeError");
    // flow grid of the wrong size: DimensionMismatchError (engine.hpp:218-219)
    FdInstance small = random_fd_instance(43);
    const FlowSequence other = FlowSequence::zeros(small.slice.width + 1, small.slice.height,
                                                   small.slice.t_start_us, small.slice.t_end_us,
                                                   small.flows.n_bins());
    threw = false;
    try {
      gpu.forward(small.slice, other);
    } catch (const DimensionMismatchError&) {
      threw = true;
    }
    CHECK(threw, "DimensionMismatchError on a flow/sensor size mismatch");
    // PhaseStats are filled (engine.hpp:63-66, 226-242)
    const FdInstance a = random_fd_instance(101), b = random_fd_instance(102);
    const ForwardResult fa = gpu.forward(a.slice, a.flows);
    CHECK(fa.warp_stats.time_us > 0 && fa.splat_stats.time_us > 0 && fa.loss_stats.time_us > 0 &&
              fa.splat_stats.peak_bytes > 0,
          "forward PhaseStats");
    const BackwardResult ba = gpu.backward(a.slice, a.flows, fa);
    CHECK(ba.stats.time_us > 0 && ba.stats.peak_bytes > 0, "backward PhaseStats");
    // a backward of an earlier forward is refused (the device holds the last one)
    const ForwardResult fb = gpu.forward(b.slice, b.flows);
    threw = false;
    try {
      gpu.backward(a.slice, a.flows, fa);
    } catch (const ConfigError&) {
      threw = true;
    }
    CHECK(threw, "stale forward refused");
    (void)fb;
  }
  // motion field and its backward
  const cuda::Engine gpu;
  Image<double> dimg(17, 11, 0.0);
  for (std::size_t i = 0; i < dimg.size(); ++i) dimg[i] = 1.0 + 0.01 * static_cast<double>(i % 37);
  const DepthMap depth(dimg);
  const CameraIntrinsics k{20.0, 21.0, 8.0, 5.0};
  const std::vector<PoseStep> poses{{{0.01, -0.02, 0.005}, {0.05, 0.02, -0.01}},
                                    {{-0.003, 0.004, 0.001}, {-0.02, 0.01, 0.03}}};
  const GeometryFlows rf = depth_pose_to_flows(depth, poses, k, 0, 100000);
  const GeometryFlows gf = cuda::depth_pose_to_flows(gpu, depth, poses, k, 0, 100000);
  for (int b = 0; b < 2; ++b)
    CHECK(rf.flows.fields[b].u == gf.flows.fields[b].u && rf.flows.fields[b].v == gf.flows.fields[b].v &&
              rf.valid[b] == gf.valid[b],
          "motion field bit-exact");
  GradientBuffer g(17, 11, 2);
  for (int b = 0; b < 2; ++b)
    for (std::size_t i = 0; i < g.gu[b].size(); ++i) {
      g.gu[b][i] = std::sin(0.1 * i + b);
      g.gv[b][i] = std::cos(0.07 * i - b);
    }
  const FlowsBackwardResult rb = depth_pose_to_flows_backward(depth, poses, k, rf.flows, g);
  const FlowsBackwardResult gb = cuda::depth_pose_to_flows_backward(gpu, depth, poses, k, rf.flows, g);
  double dmax = 0, dref = 0;
  for (std::size_t i = 0; i < rb.d_depth.size(); ++i) {
    dmax = std::max(dmax, std::abs(gb.d_depth[i] - rb.d_depth[i]));
    dref = std::max(dref, std::abs(rb.d_depth[i]));
  }
  CHECK(dmax <= 1e-12 * dref, "d_depth");
  for (int b = 0; b < 2; ++b)
    CHECK(std::abs(gb.d_poses[b].trans.x - rb.d_poses[b].trans.x) <=
              1e-10 * (1 + std::abs(rb.d_poses[b].trans.x)),
          "d_pose");
  // L_geo: membership bit-exact, sums within rounding
  {
    Image<double> d1img = dimg;
    for (std::size_t i = 0; i < d1img.size(); ++i) d1img[i] *= 1.0 + 0.02 * std::sin(0.3 * i);
    const DepthMap d1(d1img);
    const PoseStep pose{{0.01, -0.015, 0.02}, {0.12, -0.05, 0.03}};
    const GeoLossGrad r = geometry_consistency_loss_backward(depth, d1, pose, k, 0.7);
    const GeoLossGrad c = cuda::geometry_consistency_loss_backward(gpu, depth, d1, pose, k, 0.7);
    CHECK(r.terms.n_valid == c.terms.n_valid && r.terms.valid == c.terms.valid &&
              r.terms.projected == c.terms.projected && r.terms.interpolated == c.terms.interpolated,
          "L_geo membership");
    CHECK(std::abs(r.terms.value - c.terms.value) <= 1e-13 * r.terms.value, "L_geo value");
    double m = 0, mr = 0;
    for (std::size_t i = 0; i < r.d_d0.size(); ++i) {
      m = std::max({m, std::abs(r.d_d0[i] - c.d_d0[i]), std::abs(r.d_d1[i] - c.d_d1[i])});
      mr = std::max({mr, std::abs(r.d_d0[i]), std::abs(r.d_d1[i])});
    }
    CHECK(m <= 1e-10 * mr, "L_geo depth gradients %g", m / mr);
    CHECK(std::abs(r.d_trans.x - c.d_trans.x) <= 1e-10 * (1 + std::abs(r.d_trans.x)), "L_geo pose");
  }
  // predictor_loss_and_gradients with L_geo on the reference's chain fixture
  {
    evcm_test::ChainParams cp;
    cp.sensor_w = 32;
    cp.sensor_h = 24;
    cp.factor = 8;
    cp.n_bins = 3;
    cp.n_events = 60;
    const evcm_test::ChainInstance inst = evcm_test::make_chain_instance(3, cp);
    const Engine eng{EngineOptions{}};
    const WindowGradients r = predictor_loss_and_gradients(inst.pred, inst.slice, inst.k, 0.05, eng);
    const WindowGradients c = cuda::predictor_loss_and_gradients(gpu, inst.pred, inst.slice, inst.k, 0.05);
    CHECK(std::abs(r.total - c.total) <= 1e-5 * std::abs(r.total), "predictor total");
    CHECK(std::abs(r.l_geo - c.l_geo) <= 1e-12 * std::abs(r.l_geo), "predictor l_geo");
    double m = 0, mr = 0;
    for (std::size_t i = 0; i < r.grads.d_depth_params.size(); ++i) {
      m = std::max(m, std::abs(r.grads.d_depth_params[i] - c.grads.d_depth_params[i]));
      mr = std::max(mr, std::abs(r.grads.d_depth_params[i]));
    }
    CHECK(m <= 1e-5 * mr, "predictor d_params %g", m / mr);
  }
  std::printf("OK %d\n", g_checks);
  return 0;
}
