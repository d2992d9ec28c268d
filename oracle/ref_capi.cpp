// TEST INFRASTRUCTURE ONLY — builds the UNMODIFIED reference (evcm, header-only
// C++20, /root/reference/proj/include) into oracle/_ref/libevcm_ref.so behind a
// small C-ABI so the Python tests and bench.py's reference arm can drive it.
// Nothing here re-implements the algorithm: every entry point calls the
// reference's own functions (engine.hpp, geometry.hpp, fdcheck.hpp, bench.hpp,
// synth.hpp, tests/chain_support.hpp). Built with -fvisibility=hidden so only
// the ref_* symbols leave the library (no ODR clash with anything else).
//
// Layouts are the ones documented in oracle/cmax_oracle.h.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "evcm/bench.hpp"
#include "evcm/engine.hpp"
#include "evcm/fdcheck.hpp"
#include "evcm/geometry.hpp"
#include "evcm/io.hpp"
#include "evcm/optimize.hpp"
#include "evcm/predictor.hpp"
#include "evcm/synth.hpp"
#include "chain_support.hpp"
#include "test_support.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

using namespace evcm;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& ex) {
  // Order: most-derived first. Codes match oracle/cmax_oracle.h ORC_*.
  if (dynamic_cast<const ConfigError*>(&ex)) return 1;
  if (dynamic_cast<const DimensionMismatchError*>(&ex)) return 2;
  if (dynamic_cast<const CoordinateRangeError*>(&ex)) return 3;
  if (dynamic_cast<const InvalidPolarityError*>(&ex)) return 4;
  if (dynamic_cast<const UnsortedEventsError*>(&ex)) return 5;
  if (dynamic_cast<const TimeRangeError*>(&ex)) return 6;
  if (dynamic_cast<const EmptySliceError*>(&ex)) return 7;
  if (dynamic_cast<const BadMagicError*>(&ex)) return 10;
  if (dynamic_cast<const TruncatedFileError*>(&ex)) return 11;
  if (dynamic_cast<const IoError*>(&ex)) return 12;
  return 99;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return code_of(ex);
  }
}

struct RefEvent {  // byte-identical to evcm::Event
  std::uint64_t t_us;
  std::uint16_t x, y;
  std::int8_t p;
  std::uint8_t pad[3];
};
static_assert(sizeof(RefEvent) == sizeof(Event), "event layout");

EventSlice make_slice(int W, int H, std::uint64_t t0, std::uint64_t t1, const void* ev,
                      std::size_t n) {
  EventSlice s;
  s.width = static_cast<std::uint16_t>(W);
  s.height = static_cast<std::uint16_t>(H);
  s.t_start_us = t0;
  s.t_end_us = t1;
  s.events.resize(n);
  if (n) std::memcpy(s.events.data(), ev, n * sizeof(Event));
  return s;
}

FlowSequence make_flows(int W, int H, int B, const std::uint64_t* edges, const double* flows) {
  FlowSequence f;
  f.edges_us.assign(edges, edges + B + 1);
  const std::size_t HW = static_cast<std::size_t>(W) * H;
  for (int b = 0; b < B; ++b) {
    const double d = (static_cast<double>(edges[b + 1]) - static_cast<double>(edges[b])) * 1e-6;
    FlowField ff(W, H, d);
    for (std::size_t i = 0; i < HW; ++i) {
      ff.u[i] = flows[(static_cast<std::size_t>(b) * 2) * HW + i];
      ff.v[i] = flows[(static_cast<std::size_t>(b) * 2 + 1) * HW + i];
    }
    f.fields.push_back(std::move(ff));
  }
  return f;
}

void dump_flows(const FlowSequence& f, double* out) {
  const std::size_t HW = f.fields.empty() ? 0 : f.fields[0].u.size();
  for (int b = 0; b < f.n_bins(); ++b)
    for (std::size_t i = 0; i < HW; ++i) {
      out[(static_cast<std::size_t>(b) * 2) * HW + i] = f.fields[static_cast<std::size_t>(b)].u[i];
      out[(static_cast<std::size_t>(b) * 2 + 1) * HW + i] = f.fields[static_cast<std::size_t>(b)].v[i];
    }
}

EngineOptions make_opts(int backend, int n_workers, int deterministic) {
  EngineOptions o;
  o.backend = backend == 0 ? Backend::naive : backend == 1 ? Backend::padded : Backend::parallel;
  o.n_workers = n_workers;
  o.deterministic = deterministic != 0;
  if (backend == 1) o.batch_size = 16;
  return o;
}

std::vector<PoseStep> make_poses(int B, const double* p) {
  std::vector<PoseStep> v(static_cast<std::size_t>(B));
  for (int i = 0; i < B; ++i)
    v[static_cast<std::size_t>(i)] = PoseStep{{p[6 * i], p[6 * i + 1], p[6 * i + 2]},
                                              {p[6 * i + 3], p[6 * i + 4], p[6 * i + 5]}};
  return v;
}

DepthMap make_depth(int W, int H, const double* d, const std::uint8_t* mask) {
  Image<double> img(W, H, 0.0);
  for (std::size_t i = 0; i < img.size(); ++i) img[i] = d[i];
  if (!mask) return DepthMap(std::move(img));
  Image<std::uint8_t> m(W, H, 0);
  for (std::size_t i = 0; i < m.size(); ++i) m[i] = mask[i];
  return DepthMap(std::move(img), std::move(m));
}

}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// read_events / write_events (io.hpp:115-172). ref_read_events fills at most
// `cap` records; *n receives the file's count.
REF_API int ref_read_events(const char* path, int* W, int* H, std::uint64_t* t0, std::uint64_t* t1,
                            void* ev, std::size_t cap, std::size_t* n) {
  return guarded([&] {
    const EventSlice s = read_events(path);
    *W = s.width;
    *H = s.height;
    *t0 = s.t_start_us;
    *t1 = s.t_end_us;
    *n = s.events.size();
    if (ev && s.events.size() <= cap && !s.events.empty())
      std::memcpy(ev, s.events.data(), s.events.size() * sizeof(Event));
  });
}

REF_API int ref_write_events(const char* path, int W, int H, std::uint64_t t0, std::uint64_t t1,
                             const void* ev, std::size_t n) {
  return guarded([&] { write_events(make_slice(W, H, t0, t1, ev, n), path); });
}

// evcm_test::random_slice (tests/test_support.hpp:36-58) with std::mt19937_64(seed):
// the generator of the reference's Evt1.RandomRoundTrip10kEvents test.
REF_API int ref_random_slice(std::uint64_t seed, std::size_t n, int* W, int* H, std::uint64_t* t0,
                             std::uint64_t* t1, void* ev) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    const EventSlice s = evcm_test::random_slice(rng, n);
    *W = s.width;
    *H = s.height;
    *t0 = s.t_start_us;
    *t1 = s.t_end_us;
    if (n) std::memcpy(ev, s.events.data(), n * sizeof(Event));
  });
}

REF_API int ref_validate_slice(int W, int H, std::uint64_t t0, std::uint64_t t1, const void* ev,
                               std::size_t n) {
  return guarded([&] { make_slice(W, H, t0, t1, ev, n).validate(); });
}

REF_API unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// Engine::forward + optional Engine::backward through the reference's own
// backends. Any output pointer may be NULL.
REF_API int ref_loss_and_grad(int W, int H, int B, const std::uint64_t* edges, const void* ev,
                              std::size_t n, const double* flows, int backend, int n_workers,
                              int deterministic, int do_backward, double* count, double* tsum,
                              std::int64_t* n_active, std::uint8_t* alive, std::int32_t* bin,
                              double* pos, double* loss, int* no_survivors, double* grad) {
  return guarded([&] {
    const EventSlice s = make_slice(W, H, edges[0], edges[B], ev, n);
    const FlowSequence f = make_flows(W, H, B, edges, flows);
    const Engine eng(make_opts(backend, n_workers, deterministic));
    const ForwardResult fw = eng.forward(s, f);
    const std::size_t HW = static_cast<std::size_t>(W) * H;
    const int R = B + 1;
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < 2; ++c) {
        const std::size_t o = (static_cast<std::size_t>(r) * 2 + c) * HW;
        if (count)
          std::memcpy(count + o, &fw.stack.count[r][c][0], HW * sizeof(double));
        if (tsum) std::memcpy(tsum + o, &fw.stack.tsum[r][c][0], HW * sizeof(double));
      }
    if (n_active) std::memcpy(n_active, fw.stack.n_active.data(), R * sizeof(std::int64_t));
    if (alive && n) std::memcpy(alive, fw.traj.alive.data(), n);
    if (bin && n) std::memcpy(bin, fw.traj.bin.data(), n * sizeof(std::int32_t));
    if (pos && n) std::memcpy(pos, fw.traj.pos.data(), n * R * 2 * sizeof(double));
    if (loss) *loss = fw.loss.value;
    if (no_survivors) *no_survivors = fw.loss.no_survivors ? 1 : 0;
    if (do_backward && grad) {
      const BackwardResult bw = eng.backward(s, f, fw);
      for (int b = 0; b < B; ++b) {
        std::memcpy(grad + (static_cast<std::size_t>(b) * 2) * HW, &bw.grad.gu[b][0],
                    HW * sizeof(double));
        std::memcpy(grad + (static_cast<std::size_t>(b) * 2 + 1) * HW, &bw.grad.gv[b][0],
                    HW * sizeof(double));
      }
    }
  });
}

REF_API int ref_warp_event(int W, int H, int B, const std::uint64_t* edges, const double* flows,
                           double x, double y, double t_from, double t_to, double* out) {
  return guarded([&] {
    const FlowSequence f = make_flows(W, H, B, edges, flows);
    const Vec2 p = warp_event({x, y}, t_from, t_to, f);
    out[0] = p.x;
    out[1] = p.y;
  });
}

REF_API int ref_rsat(int W, int H, int B, const std::uint64_t* edges, const void* ev,
                     std::size_t n, const double* flows, double* out) {
  return guarded([&] {
    const EventSlice s = make_slice(W, H, edges[0], edges[B], ev, n);
    const FlowSequence f = make_flows(W, H, B, edges, flows);
    *out = rsat(s, f);
  });
}

REF_API int ref_depth_pose_to_flows(int W, int H, const double* depth, const std::uint8_t* mask,
                                    int B, const double* poses, const double* K,
                                    std::uint64_t t0, std::uint64_t t1, double* flows,
                                    std::uint8_t* valid, std::uint64_t* edges_out) {
  return guarded([&] {
    const DepthMap d = make_depth(W, H, depth, mask);
    const CameraIntrinsics k{K[0], K[1], K[2], K[3]};
    const GeometryFlows g = depth_pose_to_flows(d, make_poses(B, poses), k, t0, t1);
    dump_flows(g.flows, flows);
    const std::size_t HW = static_cast<std::size_t>(W) * H;
    if (valid)
      for (int b = 0; b < B; ++b) std::memcpy(valid + b * HW, &g.valid[b][0], HW);
    if (edges_out) std::memcpy(edges_out, g.flows.edges_us.data(), (B + 1) * sizeof(std::uint64_t));
  });
}

REF_API int ref_depth_pose_to_flows_backward(int W, int H, const double* depth,
                                             const std::uint8_t* mask, int B, const double* poses,
                                             const double* K, const std::uint64_t* edges,
                                             const double* grad, double* d_depth,
                                             double* d_poses) {
  return guarded([&] {
    const DepthMap d = make_depth(W, H, depth, mask);
    const CameraIntrinsics k{K[0], K[1], K[2], K[3]};
    std::vector<double> zero(static_cast<std::size_t>(B) * 2 * W * H, 0.0);
    const FlowSequence f = make_flows(W, H, B, edges, zero.data());
    GradientBuffer g(W, H, B);
    const std::size_t HW = static_cast<std::size_t>(W) * H;
    for (int b = 0; b < B; ++b)
      for (std::size_t i = 0; i < HW; ++i) {
        g.gu[b][i] = grad[(static_cast<std::size_t>(b) * 2) * HW + i];
        g.gv[b][i] = grad[(static_cast<std::size_t>(b) * 2 + 1) * HW + i];
      }
    const FlowsBackwardResult r = depth_pose_to_flows_backward(d, make_poses(B, poses), k, f, g);
    std::memcpy(d_depth, &r.d_depth[0], HW * sizeof(double));
    for (int b = 0; b < B; ++b) {
      const PoseGrad& pg = r.d_poses[b];
      const double v[6] = {pg.omega.x, pg.omega.y, pg.omega.z, pg.trans.x, pg.trans.y, pg.trans.z};
      std::memcpy(d_poses + 6 * b, v, sizeof v);
    }
  });
}

// ---- the reference's own fixture generators ---------------------------------

// random_fd_instance (fdcheck.hpp:94-146). Two-call protocol: with ev == NULL
// only the shape is reported.
REF_API int ref_random_fd_instance(std::uint64_t seed, int max_events, int max_dim,
                                   int want_masked, int* W, int* H, int* B, std::size_t* n,
                                   std::uint64_t* edges, void* ev, double* flows,
                                   std::size_t* n_masked) {
  return guarded([&] {
    FdInstanceParams p;
    if (max_events > 0) p.max_events = max_events;
    if (max_dim > 0) p.max_dim = max_dim;
    p.want_masked = want_masked != 0;
    const FdInstance inst = random_fd_instance(seed, p);
    *W = inst.slice.width;
    *H = inst.slice.height;
    *B = inst.flows.n_bins();
    *n = inst.slice.events.size();
    if (n_masked) *n_masked = inst.n_masked;
    if (!ev) return;
    std::memcpy(edges, inst.flows.edges_us.data(), (*B + 1) * sizeof(std::uint64_t));
    if (*n) std::memcpy(ev, inst.slice.events.data(), *n * sizeof(Event));
    dump_flows(inst.flows, flows);
  });
}

// detail::bench_window (bench.hpp:112-141): constant per-bin flows.
REF_API int ref_bench_window(int W, int H, int B, double window_s, std::uint64_t seed,
                             std::size_t n_events, std::uint64_t* edges, void* ev,
                             double* flows) {
  return guarded([&] {
    BenchConfig cfg;
    cfg.width = W;
    cfg.height = H;
    cfg.bins = B;
    cfg.window_s = window_s;
    cfg.seed = seed;
    FlowSequence f;
    const EventSlice s = detail::bench_window(cfg, n_events, f);
    std::memcpy(edges, f.edges_us.data(), (B + 1) * sizeof(std::uint64_t));
    if (n_events) std::memcpy(ev, s.events.data(), n_events * sizeof(Event));
    dump_flows(f, flows);
  });
}

// generate_scene (synth.hpp:81-135) with the two-plane chain config of
// SURVEY.md §8(d). Two-call protocol on the event count.
REF_API int ref_generate_scene(int W, int H, int B, const double* poses, const double* K,
                               double event_rate, std::uint64_t seed, std::size_t* n,
                               void* ev, double* depth, std::uint8_t* mask) {
  return guarded([&] {
    SceneSpec spec;
    spec.width = W;
    spec.height = H;
    spec.k = CameraIntrinsics{K[0], K[1], K[2], K[3]};
    spec.event_rate = event_rate;
    spec.seed = seed;
    spec.trajectory = make_poses(B, poses);
    spec.planes.push_back(PlaneSpec{1.0, 0, 0, W / 2, H, 0.05});
    spec.planes.push_back(PlaneSpec{3.0, W / 2, 0, W, H, 0.05});
    const SceneData sd = generate_scene(spec);
    *n = sd.events.events.size();
    if (!ev) return;
    if (*n) std::memcpy(ev, sd.events.events.data(), *n * sizeof(Event));
    for (std::size_t i = 0; i < sd.depth.d.size(); ++i) {
      depth[i] = sd.depth.d[i];
      mask[i] = sd.depth.valid[i];
    }
  });
}

// make_chain_instance (tests/chain_support.hpp:119-184) decoded to full
// resolution: depth (all valid), poses, intrinsics, events.
REF_API int ref_chain_instance(std::uint64_t seed, int sensor_w, int sensor_h, int factor,
                               int n_bins, int n_events, std::size_t* n, void* ev, double* depth,
                               double* poses, double* K) {
  return guarded([&] {
    evcm_test::ChainParams cp;
    cp.sensor_w = sensor_w;
    cp.sensor_h = sensor_h;
    cp.factor = factor;
    cp.n_bins = n_bins;
    cp.n_events = n_events;
    const evcm_test::ChainInstance inst = evcm_test::make_chain_instance(seed, cp);
    *n = inst.slice.events.size();
    if (!ev) return;
    if (*n) std::memcpy(ev, inst.slice.events.data(), *n * sizeof(Event));
    const DecodedPredictor dec = decode(inst.pred);
    for (std::size_t i = 0; i < dec.depth.d.size(); ++i) depth[i] = dec.depth.d[i];
    for (int b = 0; b < n_bins; ++b) {
      const PoseStep& p = dec.poses[b];
      const double v[6] = {p.omega.x, p.omega.y, p.omega.z, p.trans.x, p.trans.y, p.trans.z};
      std::memcpy(poses + 6 * b, v, sizeof v);
    }
    K[0] = inst.k.fx;
    K[1] = inst.k.fy;
    K[2] = inst.k.cx;
    K[3] = inst.k.cy;
  });
}

// ---- CPU baseline: the reference's own chain, window by window -------------
// Per window: depth_pose_to_flows (geometry.hpp:229) → Engine::loss_and_grad
// (engine.hpp:208, default EngineOptions except n_workers) →
// depth_pose_to_flows_backward (geometry.hpp:279); the composition of
// predictor_loss_and_gradients (optimize.hpp:205-241) minus decode and L_geo.
// Events are concatenated across windows; ev_off has n_windows+1 entries.
// Returns wall seconds in *seconds and the summed loss in *loss_sum.
REF_API int ref_chain_batch(int W, int H, int B, int n_windows, const double* depth,
                            const double* poses, const double* K, std::uint64_t t0,
                            std::uint64_t t1, const void* ev, const std::size_t* ev_off,
                            int n_workers, double* loss_sum, double* d_depth_out,
                            double* d_poses_out, double* seconds) {
  return guarded([&] {
    const CameraIntrinsics k{K[0], K[1], K[2], K[3]};
    const std::size_t HW = static_cast<std::size_t>(W) * H;
    EngineOptions o;
    o.n_workers = n_workers;
    const Engine eng(o);
    double ls = 0.0;
    const auto start = std::chrono::steady_clock::now();
    for (int w = 0; w < n_windows; ++w) {
      const DepthMap d = make_depth(W, H, depth + static_cast<std::size_t>(w) * HW, nullptr);
      const std::vector<PoseStep> ps = make_poses(B, poses + static_cast<std::size_t>(w) * 6 * B);
      const GeometryFlows g = depth_pose_to_flows(d, ps, k, t0, t1);
      const EventSlice s =
          make_slice(W, H, t0, t1, static_cast<const Event*>(ev) + ev_off[w], ev_off[w + 1] - ev_off[w]);
      const auto [fw, bw] = eng.loss_and_grad(s, g.flows);
      const FlowsBackwardResult r = depth_pose_to_flows_backward(d, ps, k, g.flows, bw.grad);
      ls += fw.loss.value;
      if (d_depth_out)
        std::memcpy(d_depth_out + static_cast<std::size_t>(w) * HW, &r.d_depth[0], HW * sizeof(double));
      if (d_poses_out)
        for (int b = 0; b < B; ++b) {
          const PoseGrad& pg = r.d_poses[b];
          const double v[6] = {pg.omega.x, pg.omega.y, pg.omega.z, pg.trans.x, pg.trans.y, pg.trans.z};
          std::memcpy(d_poses_out + (static_cast<std::size_t>(w) * B + b) * 6, v, sizeof v);
        }
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    *loss_sum = ls;
  });
}

// ---- predictor decode chain (predictor.hpp, optimize.hpp) --------------------

namespace {
DirectPredictor make_pred(int pw, int ph, int factor, const double* params, int B,
                          const double* poses) {
  DirectPredictor p;
  p.depth_params = Image<double>(pw, ph, 0.0);
  for (int i = 0; i < pw * ph; ++i) p.depth_params[i] = params[i];
  p.upsample = factor;
  p.poses.resize(B);
  for (int b = 0; b < B; ++b) {
    const double* q = poses + 6 * b;
    p.poses[b].omega = {q[0], q[1], q[2]};
    p.poses[b].trans = {q[3], q[4], q[5]};
  }
  return p;
}
}  // namespace

// decode (predictor.hpp:126-131)
REF_API int ref_decode(int pw, int ph, int factor, const double* params, double* depth) {
  return guarded([&] {
    const double zero_pose[6] = {0, 0, 0, 0, 0, 0};
    const DecodedPredictor d = decode(make_pred(pw, ph, factor, params, 1, zero_pose));
    for (std::size_t i = 0; i < d.depth.d.size(); ++i) depth[i] = d.depth.d[i];
  });
}

// upsample_bilinear_adjoint * softplus_grad: the depth half of
// accumulate_gradients (predictor.hpp:156-162)
REF_API int ref_decode_backward(int pw, int ph, int factor, const double* params,
                                const double* d_depth, double* d_params) {
  return guarded([&] {
    Image<double> g(pw * factor, ph * factor, 0.0);
    for (std::size_t i = 0; i < g.size(); ++i) g[i] = d_depth[i];
    const Image<double> low = upsample_bilinear_adjoint(g, pw, ph, factor);
    for (int i = 0; i < pw * ph; ++i) d_params[i] = low[i] * softplus_grad(params[i]);
  });
}

// Adam::step (optimize.hpp:115-134), t steps from zero state on the same grads
REF_API int ref_adam_steps(std::size_t n, double* slots, const double* grads, int t, double lr,
                           double beta1, double beta2, double eps) {
  return guarded([&] {
    OptimizerConfig cfg;
    cfg.learning_rate = lr;
    cfg.adam_beta1 = beta1;
    cfg.adam_beta2 = beta2;
    cfg.adam_eps = eps;
    Adam adam(n);
    std::vector<double*> s(n);
    for (std::size_t i = 0; i < n; ++i) s[i] = slots + i;
    const std::vector<double> g(grads, grads + n);
    for (int k = 0; k < t; ++k) adam.step(s, g, cfg);
  });
}

// predictor_loss_and_gradients (optimize.hpp:205-241), lambda_geo = 0, on the
// reference's own chain fixture (tests/chain_support.hpp:119-184): returns the
// raw predictor (low-res params, poses), intrinsics, events, and the reference's
// loss and parameter gradients. n_workers: Engine parallel backend workers.
REF_API int ref_predictor_instance(std::uint64_t seed, int sensor_w, int sensor_h, int factor,
                                   int n_bins, int n_events, std::size_t* n, void* ev,
                                   double* params, double* poses, double* K, double* loss,
                                   double* d_params, double* d_poses) {
  return guarded([&] {
    evcm_test::ChainParams cp;
    cp.sensor_w = sensor_w;
    cp.sensor_h = sensor_h;
    cp.factor = factor;
    cp.n_bins = n_bins;
    cp.n_events = n_events;
    const evcm_test::ChainInstance inst = evcm_test::make_chain_instance(seed, cp);
    *n = inst.slice.events.size();
    if (!ev) return;
    if (*n) std::memcpy(ev, inst.slice.events.data(), *n * sizeof(Event));
    const DirectPredictor& p = inst.pred;
    for (std::size_t i = 0; i < p.depth_params.size(); ++i) params[i] = p.depth_params[i];
    for (int b = 0; b < n_bins; ++b) {
      const PoseStep& q = p.poses[b];
      const double v[6] = {q.omega.x, q.omega.y, q.omega.z, q.trans.x, q.trans.y, q.trans.z};
      std::memcpy(poses + 6 * b, v, sizeof v);
    }
    K[0] = inst.k.fx;
    K[1] = inst.k.fy;
    K[2] = inst.k.cx;
    K[3] = inst.k.cy;
    const Engine engine{EngineOptions{}};
    const WindowGradients wg = predictor_loss_and_gradients(p, inst.slice, inst.k, 0.0, engine);
    *loss = wg.l_cm;
    for (std::size_t i = 0; i < wg.grads.d_depth_params.size(); ++i)
      d_params[i] = wg.grads.d_depth_params[i];
    for (int b = 0; b < n_bins; ++b) {
      const PoseGrad& q = wg.grads.d_poses[b];
      const double v[6] = {q.omega.x, q.omega.y, q.omega.z, q.trans.x, q.trans.y, q.trans.z};
      std::memcpy(d_poses + 6 * b, v, sizeof v);
    }
  });
}

// geometry_consistency_loss (want_grad = 0) / _backward (geometry.hpp:416-534) for
// one pose. Output pointers may be NULL (d_pose = {omega, trans}).
REF_API int ref_geo_loss(int W, int H, const double* d0, const std::uint8_t* m0, const double* d1,
                         const std::uint8_t* m1, const double* pose, const double* K,
                         double upstream, int want_grad, double* value, std::int64_t* n_valid,
                         int* empty, double* projected, double* interpolated, std::uint8_t* valid,
                         double* d_d0, double* d_d1, double* d_pose) {
  return guarded([&] {
    const DepthMap a = make_depth(W, H, d0, m0), b = make_depth(W, H, d1, m1);
    const PoseStep ps = make_poses(1, pose)[0];
    const CameraIntrinsics k{K[0], K[1], K[2], K[3]};
    auto dump_terms = [&](const GeoLossTerms& t) {
      *value = t.value;
      *n_valid = t.n_valid;
      *empty = t.empty_valid_set ? 1 : 0;
      for (std::size_t i = 0; i < static_cast<std::size_t>(W) * H; ++i) {
        if (projected) projected[i] = t.projected[i];
        if (interpolated) interpolated[i] = t.interpolated[i];
        if (valid) valid[i] = t.valid[i];
      }
    };
    if (!want_grad) {
      dump_terms(geometry_consistency_loss(a, b, ps, k));
      return;
    }
    const GeoLossGrad g = geometry_consistency_loss_backward(a, b, ps, k, upstream);
    dump_terms(g.terms);
    for (std::size_t i = 0; i < static_cast<std::size_t>(W) * H; ++i) {
      if (d_d0) d_d0[i] = g.d_d0[i];
      if (d_d1) d_d1[i] = g.d_d1[i];
    }
    if (d_pose) {
      const double v[6] = {g.d_omega.x, g.d_omega.y, g.d_omega.z,
                           g.d_trans.x, g.d_trans.y, g.d_trans.z};
      std::memcpy(d_pose, v, sizeof v);
    }
  });
}

// predictor_loss_and_gradients (optimize.hpp:205-241) of a DirectPredictor with
// any lambda_geo: losses = {l_cm, l_geo, total}.
REF_API int ref_predictor_loss(int pw, int ph, int factor, const double* params, int n_bins,
                               const double* poses, const double* K, std::uint64_t t0,
                               std::uint64_t t1, const void* ev, std::size_t n, double lambda_geo,
                               double* losses, double* d_params, double* d_poses) {
  return guarded([&] {
    DirectPredictor p;
    p.depth_params = Image<double>(pw, ph, 0.0);
    for (std::size_t i = 0; i < p.depth_params.size(); ++i) p.depth_params[i] = params[i];
    p.poses = make_poses(n_bins, poses);
    p.upsample = factor;
    const EventSlice s = make_slice(pw * factor, ph * factor, t0, t1, ev, n);
    const Engine engine{EngineOptions{}};
    const WindowGradients wg = predictor_loss_and_gradients(
        p, s, CameraIntrinsics{K[0], K[1], K[2], K[3]}, lambda_geo, engine);
    losses[0] = wg.l_cm;
    losses[1] = wg.l_geo;
    losses[2] = wg.total;
    for (std::size_t i = 0; i < wg.grads.d_depth_params.size(); ++i)
      d_params[i] = wg.grads.d_depth_params[i];
    for (int b = 0; b < n_bins; ++b) {
      const PoseGrad& q = wg.grads.d_poses[b];
      const double v[6] = {q.omega.x, q.omega.y, q.omega.z, q.trans.x, q.trans.y, q.trans.z};
      std::memcpy(d_poses + 6 * b, v, sizeof v);
    }
  });
}

// save_predictor / load_predictor (predictor.hpp:178-218) and the PFM codec
// (io.hpp:178-236) for the checkpoint fixtures.
REF_API int ref_save_predictor(int pw, int ph, int factor, const double* params, int n_bins,
                               const double* poses, const char* pfm, const char* csv) {
  return guarded([&] {
    DirectPredictor p;
    p.depth_params = Image<double>(pw, ph, 0.0);
    for (std::size_t i = 0; i < p.depth_params.size(); ++i) p.depth_params[i] = params[i];
    p.poses = make_poses(n_bins, poses);
    p.upsample = factor;
    save_predictor(p, pfm, csv);
  });
}

REF_API int ref_load_predictor(const char* pfm, const char* csv, int* pw, int* ph, int* factor,
                               int* n_bins, double* params, std::size_t cap_params, double* poses,
                               int cap_bins) {
  return guarded([&] {
    const DirectPredictor p = load_predictor(pfm, csv);
    *pw = p.depth_params.width();
    *ph = p.depth_params.height();
    *factor = p.upsample;
    *n_bins = static_cast<int>(p.poses.size());
    if (params && p.depth_params.size() <= cap_params)
      for (std::size_t i = 0; i < p.depth_params.size(); ++i) params[i] = p.depth_params[i];
    if (poses && *n_bins <= cap_bins)
      for (int b = 0; b < *n_bins; ++b) {
        const PoseStep& q = p.poses[b];
        const double v[6] = {q.omega.x, q.omega.y, q.omega.z, q.trans.x, q.trans.y, q.trans.z};
        std::memcpy(poses + 6 * b, v, sizeof v);
      }
  });
}

REF_API int ref_read_pfm(const char* path, int* w, int* h, float* out, std::size_t cap) {
  return guarded([&] {
    const Image<float> img = read_pfm(path);
    *w = img.width();
    *h = img.height();
    if (out && img.size() <= cap)
      for (std::size_t i = 0; i < img.size(); ++i) out[i] = img[i];
  });
}

// format_number (io.hpp:295-299) into buf (>= 64 bytes).
REF_API void ref_format_number(double v, char* buf) {
  const std::string s = format_number(v);
  std::memcpy(buf, s.c_str(), s.size() + 1);
}

// run_window (optimize.hpp:297-375) over nw windows (events concatenated,
// window w = events[offs[w], offs[w+1]) on [t01[2w], t01[2w+1])). Returns the
// trained params / poses and per record {l_cm, l_geo, total, rsat, gnd, gnp}.
REF_API int ref_run_window(int nw, const std::uint64_t* t01, const void* ev,
                           const std::uint64_t* offs, int pw, int ph, int factor,
                           const double* params, int n_bins, const double* poses, const double* K,
                           double lr, int steps_per_update, int max_updates, double lambda_geo,
                           double* params_out, double* poses_out, double* rec, int* n_rec) {
  return guarded([&] {
    std::vector<EventSlice> wins;
    const auto* e = static_cast<const Event*>(ev);
    for (int w = 0; w < nw; ++w)
      wins.push_back(make_slice(pw * factor, ph * factor, t01[2 * w], t01[2 * w + 1], e + offs[w],
                                offs[w + 1] - offs[w]));
    DirectPredictor p;
    p.depth_params = Image<double>(pw, ph, 0.0);
    for (std::size_t i = 0; i < p.depth_params.size(); ++i) p.depth_params[i] = params[i];
    p.poses = make_poses(n_bins, poses);
    p.upsample = factor;
    OptimizerConfig cfg;
    cfg.learning_rate = lr;
    cfg.steps_per_update = steps_per_update;
    cfg.bins = n_bins;
    cfg.max_updates = max_updates;
    cfg.lambda_geo = lambda_geo;
    const RunResult r = run_window(wins, p, CameraIntrinsics{K[0], K[1], K[2], K[3]}, cfg);
    for (std::size_t i = 0; i < r.predictor.depth_params.size(); ++i)
      params_out[i] = r.predictor.depth_params[i];
    for (int b = 0; b < n_bins; ++b) {
      const PoseStep& q = r.predictor.poses[b];
      const double v[6] = {q.omega.x, q.omega.y, q.omega.z, q.trans.x, q.trans.y, q.trans.z};
      std::memcpy(poses_out + 6 * b, v, sizeof v);
    }
    *n_rec = static_cast<int>(r.log.records.size());
    for (std::size_t i = 0; i < r.log.records.size(); ++i) {
      const TrainRecord& t = r.log.records[i];
      const double v[6] = {t.l_cm, t.l_geo, t.total, t.rsat, t.grad_norm_depth, t.grad_norm_pose};
      std::memcpy(rec + 6 * i, v, sizeof v);
    }
  });
}

// optimize_flow_only (optimize.hpp:385-487): final (best) flows [B][2][H][W] and
// the per-update l_cm / rsat / grad_norm_depth of the log.
REF_API int ref_optimize_flow_only(int W, int H, std::uint64_t t0, std::uint64_t t1, const void* ev,
                                   std::size_t n, int n_bins, double lr, int max_updates,
                                   double* flows_out, double* l_cm, double* rsat, double* gnorm,
                                   int* n_records) {
  return guarded([&] {
    EventSlice s;
    s.width = W;
    s.height = H;
    s.t_start_us = t0;
    s.t_end_us = t1;
    s.events.resize(n);
    if (n) std::memcpy(s.events.data(), ev, n * sizeof(Event));
    OptimizerConfig cfg;
    cfg.learning_rate = lr;
    cfg.max_updates = max_updates;
    const FlowOnlyResult r = optimize_flow_only(s, n_bins, cfg);
    const std::size_t HW = static_cast<std::size_t>(W) * H;
    for (int b = 0; b < n_bins; ++b)
      for (std::size_t i = 0; i < HW; ++i) {
        flows_out[(2 * b) * HW + i] = r.flows.fields[b].u[i];
        flows_out[(2 * b + 1) * HW + i] = r.flows.fields[b].v[i];
      }
    *n_records = static_cast<int>(r.log.records.size());
    for (std::size_t i = 0; i < r.log.records.size(); ++i) {
      l_cm[i] = r.log.records[i].l_cm;
      rsat[i] = r.log.records[i].rsat;
      gnorm[i] = r.log.records[i].grad_norm_depth;
    }
  });
}
