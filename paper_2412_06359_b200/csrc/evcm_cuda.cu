// C-ABI implementation of include/evcm_cuda.h: validation with the reference's
// error taxonomy, workspace management, host<->device staging, and the stage
// sequencing of Engine::forward / backward, the motion field and the batched
// chain. Kernels live in cmax_kernels.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/evcm_cuda.h"
#include "cmax_kernels.h"
#include "cmax_owner.h"

using namespace evcm_b200;

namespace {

thread_local std::string g_err;

struct Failure {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, std::string msg) { throw Failure{code, std::move(msg)}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(EVCM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return EVCM_OK;
  } catch (const Failure& x) {
    g_err = x.msg;
    return x.code;
  } catch (const std::exception& x) {
    g_err = x.what();
    return EVCM_ERR_CUDA;
  }
}

// ---- host-side rigid geometry (geometry.hpp:21-135), used to build the
// per-(window, bin) pose table. Same expression order as the reference so
// that R is bit-identical (the motion field then matches bit for bit).
struct M3 {
  double m[9];
};
M3 mul(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.m[3 * i + j] = a.m[3 * i] * b.m[j] + a.m[3 * i + 1] * b.m[3 + j] + a.m[3 * i + 2] * b.m[6 + j];
  return r;
}
M3 skew(double x, double y, double z) { return {{0, -z, y, z, 0, -x, -y, x, 0}}; }

M3 rodrigues(const double* w) {  // geometry.hpp:94-107
  const double t2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  const double t = std::sqrt(t2);
  double a, b;
  if (t < 1e-8) {
    a = 1.0 - t2 / 6.0;
    b = 0.5 - t2 / 24.0;
  } else {
    a = std::sin(t) / t;
    b = (1.0 - std::cos(t)) / t2;
  }
  const M3 S = skew(w[0], w[1], w[2]);
  const M3 S2 = mul(S, S);
  static const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  M3 R;
  for (int i = 0; i < 9; ++i) R.m[i] = (I[i] + a * S.m[i]) + b * S2.m[i];
  return R;
}

void rodrigues_jacobian(const double* w, M3 out[3]) {  // geometry.hpp:114-135
  const double t2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  const double t = std::sqrt(t2);
  const M3 S = skew(w[0], w[1], w[2]);
  static const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  if (t < 1e-4) {
    for (int k = 0; k < 3; ++k) {
      const M3 ek = skew(k == 0, k == 1, k == 2);
      const M3 a = mul(ek, S), b = mul(S, ek);
      for (int i = 0; i < 9; ++i) out[k].m[i] = ek.m[i] + 0.5 * (a.m[i] + b.m[i]);
    }
    return;
  }
  const M3 R = rodrigues(w);
  M3 IR;
  for (int i = 0; i < 9; ++i) IR.m[i] = I[i] - R.m[i];
  for (int k = 0; k < 3; ++k) {
    const double c0 = IR.m[k], c1 = IR.m[3 + k], c2 = IR.m[6 + k];
    const M3 sc = skew(w[1] * c2 - w[2] * c1, w[2] * c0 - w[0] * c2, w[0] * c1 - w[1] * c0);
    M3 m;
    for (int i = 0; i < 9; ++i) m.m[i] = w[k] * S.m[i] + sc.m[i];
    const M3 p = mul(m, R);
    for (int i = 0; i < 9; ++i) out[k].m[i] = (1.0 / t2) * p.m[i];
  }
}

void validate_pose(const double* p) {  // PoseStep::validate (types.hpp:362-368)
  const double pi = 3.14159265358979323846;
  if (!(std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]) < pi))
    fail(EVCM_ERR_CONFIG, "pose step: rotation angle must stay below pi");
  for (int i = 0; i < 6; ++i)
    if (!std::isfinite(p[i])) fail(EVCM_ERR_CONFIG, "pose step: non-finite component");
}

// FlowSequence::zeros edge rule (types.hpp:293-300)
std::vector<uint64_t> zeros_edges(uint64_t t0, uint64_t t1, int B) {
  if (B < 1 || t1 <= t0) fail(EVCM_ERR_CONFIG, "flow sequence: need n_bins >= 1 and a nonempty window");
  std::vector<uint64_t> e(B + 1);
  const double span = static_cast<double>(t1 - t0);
  for (int i = 0; i <= B; ++i)
    e[i] = (i == B) ? t1 : t0 + static_cast<uint64_t>(std::llround(span * i / B));
  return e;
}

// ---- workspace ----------------------------------------------------------------

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
};

}  // namespace

struct evcm_cuda_engine {
  evcm_cuda_options opt{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::unordered_map<std::string, Buf> bufs;
  std::unordered_map<std::string, Buf> pins;  // pinned host staging
  int stage_nw = 0;
  bool check_pose_flag = false;  // device pose tables: validation result pending
  // CUDA graphs of the device-resident chain, keyed by the call signature
  // (shapes, pointers, event offsets, options): the first call of a signature
  // runs eagerly, the second is captured, later ones replay. A few signatures
  // are kept (e.g. double-buffered inputs of a pipelined caller); every entry
  // is dropped when a workspace buffer is reallocated (alloc_gen), since its
  // graph would reference the freed memory.
  struct GraphEntry {
    std::vector<uint64_t> sig;
    cudaGraphExec_t exec = nullptr;
    bool failed = false;  // capture failed for this signature: run eagerly
    int launches = 0;
    uint64_t gen = 0, last_use = 0;
  };
  static constexpr size_t kGraphCache = 4;
  std::vector<GraphEntry> graphs;
  uint64_t alloc_gen = 0, use_clock = 0;
  // asynchronous chain calls (evcm_cuda_chain_batch_async): each of kSlots
  // slots has its own pinned error words, completion event and pending checks,
  // so a caller can keep the next batch queued while it waits for this one
  static constexpr int kSlots = 4;
  int slot = 0;
  struct Pending {
    bool active = false;
    int nw = 0;
    bool pose = false;
    cudaEvent_t done = nullptr;
  } pending[kSlots];
  std::string slot_name(const char* base) const {
    return slot ? std::string(base) + "#" + std::to_string(slot) : std::string(base);
  }
  // owner pipeline state
  TileParams TP{};
  uint64_t n_total = 0, max_n = 0;
  // resolved per call in stage_events: opt.algo 0 owner, 1 atomic, 2 auto
  bool use_owner = true;
  bool owner() const { return use_owner; }
  // state of the last forward (Engine::forward -> backward hand-off)
  bool have_fwd = false;
  WinParams P{};
  uint64_t n_events = 0;
  int last_launches = 0;
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  std::vector<double> stage_ms;

  template <typename T>
  T* get(const std::string& name, size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    Buf& b = bufs[name];
    if (b.cap < bytes) {
      if (b.p) ck(cudaFree(b.p), "cudaFree");
      b.p = nullptr;
      ck(cudaMalloc(&b.p, bytes), "cudaMalloc");
      b.cap = bytes;
      ++alloc_gen;
    }
    return static_cast<T*>(b.p);
  }

  template <typename T>
  T* pinned(const std::string& name, size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    Buf& b = pins[name];
    if (b.cap < bytes) {
      if (b.p) ck(cudaFreeHost(b.p), "cudaFreeHost");
      b.p = nullptr;
      ck(cudaMallocHost(&b.p, bytes), "cudaMallocHost");
      b.cap = bytes;
      ++alloc_gen;  // captured graphs may copy from / into the old buffer
    }
    return static_cast<T*>(b.p);
  }

  // PhaseStats of the last forward / backward (evcm_cuda_phase_stats)
  double phase_us[4] = {0, 0, 0, 0};
  size_t phase_bytes[4] = {0, 0, 0, 0};
  size_t ws_at_mark[16] = {};
  uint64_t fwd_id = 0;  // id of the forward whose state the engine holds (0: none)
  uint64_t fwd_counter = 0;
  cudaEvent_t order_ev = nullptr;  // evcm_cuda_stream_wait / signal
  size_t ws_bytes() const {
    size_t t = 0;
    for (auto& kv : bufs) t += kv.second.cap;
    return t;
  }
  // NVTX markers at the stage boundaries (host side; visible to nsys / ncu
  // --nvtx): instantaneous marks, so a forward-only call leaves nothing open
  void nvtx_stage(int i) {
    static const char* kOwner[] = {"evcm: staging", "evcm: motion_field", "evcm: sort",
                                   "evcm: traj_records+lists", "evcm: fwd_owner",
                                   "evcm: loss_finalize", "evcm: bwd_event", "evcm: bwd_owner",
                                   "evcm: pose_contract", "evcm: end"};
    if (i >= 0 && i < 10) nvtxMarkA(use_owner || i < 2 ? kOwner[i] : "evcm: atomic stage");
  }
  void mark(int i) {
    nvtx_stage(i);
    if (i >= 0 && i < 16) ws_at_mark[i] = ws_bytes();
    if (!timing) return;
    while ((int)ev.size() <= i) {
      cudaEvent_t e;
      ck(cudaEventCreate(&e), "cudaEventCreate");
      ev.push_back(e);
    }
    ck(cudaEventRecord(ev[i], stream), "cudaEventRecord");
  }
  // stage_ms[i] = time between marks i and i+1, for lo <= i < hi (others 0)
  void collect_range(int lo, int hi) {
    stage_ms.assign(9, 0.0);
    if (!timing) return;
    ck(cudaEventSynchronize(ev[hi]), "cudaEventSynchronize");
    for (int i = lo; i < hi; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      stage_ms[i] = ms;
    }
  }
};

namespace {

// Stage marks (CUDA events on the engine stream), see evcm_cuda_stage_times:
// 0 start | staging | 1 | motion field | 2 | stack memset | 3 | warp+splat | 4 |
// loss reduce | 5 | grad memset | 6 | backward | 7 | flows backward | 8
constexpr int M_FWD0 = 2;

void set_device(evcm_cuda_engine* e) { ck(cudaSetDevice(e->opt.device), "cudaSetDevice"); }

// Copy `bytes` from a host or device pointer into a device buffer (or return
// the device pointer itself).
template <typename T>
const T* to_device(evcm_cuda_engine* e, const char* name, const T* src, size_t count, int mem) {
  if (mem == EVCM_MEM_DEVICE || count == 0) return src;
  T* d = e->get<T>(name, count);
  ck(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, e->stream), "H2D");
  return d;
}

void from_device(evcm_cuda_engine* e, void* dst, const void* src, size_t bytes, int mem) {
  if (bytes == 0) return;
  ck(cudaMemcpyAsync(dst, src, bytes,
                     mem == EVCM_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     e->stream),
     "copy out");
}

// Window parameters from (W, H, edges): Engine::edge_seconds (engine.hpp:244-249)
WinParams make_params(int W, int H, const uint64_t* edges, int B, int n_windows, uint64_t t0,
                      uint64_t t_end) {
  if (B > kMaxBins)
    fail(EVCM_ERR_CONFIG, "cuda backend: at most " + std::to_string(kMaxBins) + " bins");
  WinParams P{};
  P.W = W;
  P.H = H;
  P.B = B;
  P.HW = W * H;
  P.n_windows = n_windows;
  for (int i = 0; i <= B; ++i) {
    P.es[i] = (static_cast<double>(edges[i]) - static_cast<double>(edges[0])) * 1e-6;
    P.erel[i] = static_cast<uint32_t>(edges[i] - edges[0]);
  }
  P.window_s = P.es[B];
  P.inv_window = 1.0 / P.window_s;
  P.t0 = t0;
  P.t_end = t_end;
  P.stride_us = 0;
  return P;
}

void check_slice_header(const evcm_slice* s) {  // EventSlice::validate (types.hpp:136-139)
  if (s->width == 0 || s->height == 0)
    fail(EVCM_ERR_DIMENSION, "event slice: width and height must be positive");
  if (s->t_end_us < s->t_start_us) fail(EVCM_ERR_TIME_RANGE, "event slice: t_end precedes t_start");
}

// Engine::validate_window after slice.validate() (engine.hpp:215-222): FlowSequence::validate
// (types.hpp:268-284), then the sensor shape, then the window span.
void check_flows(const evcm_slice* s, const evcm_flows* f) {
  if (f->n_bins < 1 || !f->edges_us)
    fail(EVCM_ERR_CONFIG, "flow sequence: need B >= 1 fields and B+1 edges");
  for (int i = 0; i < f->n_bins; ++i)
    if (f->edges_us[i] >= f->edges_us[i + 1])
      fail(EVCM_ERR_CONFIG, "flow sequence: edges must be strictly increasing");
  if (f->width <= 0 || f->height <= 0 || !f->uv)
    fail(EVCM_ERR_DIMENSION, "flow field: u and v must share a nonempty shape");
  if (f->width != (int)s->width || f->height != (int)s->height)
    fail(EVCM_ERR_DIMENSION, "engine: flow shape differs from sensor shape");
  if (f->edges_us[0] != s->t_start_us || f->edges_us[f->n_bins] != s->t_end_us)
    fail(EVCM_ERR_CONFIG, "engine: flow bin edges do not span the slice window");
  if (s->t_end_us - s->t_start_us >= (1ull << 31))
    fail(EVCM_ERR_CONFIG, "cuda backend: window longer than 2^31 us");
}

const char* code_name(int c) {
  switch (c) {
    case EVCM_OK: return "OK";
    case EVCM_ERR_CONFIG: return "ConfigError";
    case EVCM_ERR_DIMENSION: return "DimensionMismatchError";
    case EVCM_ERR_COORDINATE: return "CoordinateRangeError";
    case EVCM_ERR_POLARITY: return "InvalidPolarityError";
    case EVCM_ERR_UNSORTED: return "UnsortedEventsError";
    case EVCM_ERR_TIME_RANGE: return "TimeRangeError";
    case EVCM_ERR_EMPTY: return "EmptySliceError";
    case EVCM_ERR_STATE: return "ConfigError";
    default: return "Error";
  }
}

// Stage + validate events of n_windows windows (offsets on host). Asynchronous:
// the per-window first-violation keys land in pinned host memory and are
// checked by check_stage_errors() after the call's final stream sync.
// prepared: k_chain_init already wrote the device offsets ("ev_off") and reset
// the validation words ("stage_err", nw + 1 words); the caller copies them back.
void stage_events(evcm_cuda_engine* e, const evcm_event* ev, const uint64_t* off_h, const WinParams& P,
                  int mem, bool prepared = false) {
  const int nw = P.n_windows;
  const uint64_t total = off_h[nw];
  uint64_t max_n = 0;
  for (int w = 0; w < nw; ++w) max_n = std::max<uint64_t>(max_n, off_h[w + 1] - off_h[w]);
  const evcm_event* dev = to_device(e, "events_aos", ev, total, mem);
  uint64_t* off_d = e->get<uint64_t>("ev_off", nw + 1);
  unsigned long long* err = e->get<unsigned long long>("stage_err", nw + 1);
  if (!prepared) {
    uint64_t* off_pin = e->pinned<uint64_t>("ev_off_h", nw + 1);
    std::memcpy(off_pin, off_h, (nw + 1) * sizeof(uint64_t));
    ck(cudaMemcpyAsync(off_d, off_pin, (nw + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, e->stream),
       "H2D offsets");
    ck(cudaMemsetAsync(err, 0xff, nw * sizeof(unsigned long long), e->stream), "memset");
  }
  uint2* packed = e->get<uint2>("packed", total);
  e->n_total = (total + 1) & ~1ull;  // even plane stride (16 B-aligned 8 B sub-arrays)
  e->max_n = max_n;
  // algo auto: the owner pipeline (deterministic, fixed-point) ties the atomic one
  // at ~1 event per pixel and window and wins above, once the call carries
  // ~2.5e5 events (below, its fixed per-stage latency dominates; measured,
  // DESIGN.md)
  if (e->opt.algo == 2)
    e->use_owner = e->opt.deterministic ||
                   ((double)total >= 1.0 * (double)P.HW * nw && total >= kOwnerMinEvents);
  else
    e->use_owner = e->opt.algo == 0 || e->opt.deterministic;
  if (e->owner()) {
    // validation + packing; the sort needs the flows and runs in the forward
    const TileParams TP = make_tiles(P, max_n);
    if (TP.nT > kMaxTiles)
      fail(EVCM_ERR_CONFIG, "cuda backend: sensor too large (more than " +
                                std::to_string(kMaxTiles) + " 8x8 sort tiles)");
    if ((uint64_t)TP.nchunks > 0xffffu)
      fail(EVCM_ERR_CONFIG, "cuda backend: too many events in one window");
    e->TP = TP;
    launch_stage_pack(e->stream, dev, off_d, P, max_n, packed, err);
  } else {
    launch_stage(e->stream, dev, off_d, P, max_n, packed, err);
  }
  // one read-back: the window words and, after them, the chain's pose flag
  const int nwords = nw + 1;
  unsigned long long* err_h = e->pinned<unsigned long long>(e->slot_name("stage_err_h"), nw + 1);
  ck(cudaMemcpyAsync(err_h, err, nwords * sizeof(unsigned long long), cudaMemcpyDeviceToHost, e->stream),
     "D2H err");
  e->stage_nw = nw;
}

// After the stream sync: raise the reference's error for the first invalid
// event of the first bad window (EventSlice::validate order, types.hpp:143-155).
void check_stage_errors(evcm_cuda_engine* e) {
  const unsigned long long* h = e->pinned<unsigned long long>(e->slot_name("stage_err_h"), e->stage_nw);
  for (int w = 0; w < e->stage_nw; ++w) {
    if (h[w] == ~0ull) continue;
    const int code = static_cast<int>(h[w] & 0xf);
    const uint64_t k = h[w] >> 4;
    std::string msg;
    switch (code) {
      case 3: msg = "event slice: coordinate outside the sensor"; break;
      case 4: msg = "event slice: polarity must be +1 or -1"; break;
      case 5: msg = "event slice: timestamps must be non-decreasing"; break;
      default: msg = "event slice: timestamp outside the window"; break;
    }
    fail(code, msg + " (window " + std::to_string(w) + ", event " + std::to_string(k) + ")");
  }
}

void sync_and_check(evcm_cuda_engine* e, const char* what) {
  ck(cudaStreamSynchronize(e->stream), what);
  // depth_pose_to_flows validates poses before Engine::forward validates events
  // (optimize.hpp:211-213), so a bad pose wins over a bad event.
  if (e->check_pose_flag) {
    e->check_pose_flag = false;
    if (e->pinned<unsigned long long>(e->slot_name("stage_err_h"), e->stage_nw + 1)[e->stage_nw])
      fail(EVCM_ERR_CONFIG, "pose step: rotation angle must stay below pi and components finite");
  }
  check_stage_errors(e);
  ck(cudaGetLastError(), what);
}

// Pose table per (window, bin): R[9], dR[27], t[3], inv_dt, built on the host
// with the reference's rodrigues / rodrigues_jacobian (bit-identical R) and
// copied from a pinned staging buffer (no sync needed: every API call ends
// with a stream sync before the buffer is rewritten).
const double* upload_pose_table(evcm_cuda_engine* e, const double* poses_h, int nw, int B,
                                const uint64_t* edges, bool validate) {
  const size_t n = static_cast<size_t>(nw) * B * kPoseTab;
  double* tab = e->pinned<double>("pose_tab_h", n);
  for (int w = 0; w < nw; ++w)
    for (int b = 0; b < B; ++b) {
      const double* p = poses_h + (static_cast<size_t>(w) * B + b) * 6;
      if (validate) validate_pose(p);
      double* t = tab + (static_cast<size_t>(w) * B + b) * kPoseTab;
      const M3 R = rodrigues(p);
      M3 dR[3];
      rodrigues_jacobian(p, dR);
      std::memcpy(t, R.m, sizeof R.m);
      for (int k = 0; k < 3; ++k) std::memcpy(t + 9 + 9 * k, dR[k].m, sizeof dR[k].m);
      t[36] = p[3];
      t[37] = p[4];
      t[38] = p[5];
      const double dur = (static_cast<double>(edges[b + 1]) - static_cast<double>(edges[b])) * 1e-6;
      t[39] = 1.0 / dur;
    }
  double* d = e->get<double>("pose_tab", n);
  ck(cudaMemcpyAsync(d, tab, n * sizeof(double), cudaMemcpyHostToDevice, e->stream), "H2D pose table");
  return d;
}

// Workspace of the L_geo kernels (geo.cu) for g.n_poses poses of a W x H pair.
void geo_workspace(evcm_cuda_engine* e, GeoArgs& g) {
  const size_t n = (size_t)g.W * g.H * g.n_poses;
  g.zkey = e->get<unsigned long long>("geo_zkey", n);
  g.winner = e->get<unsigned>("geo_winner", n);
  if (g.want_grad) {
    g.dd0_raw = e->get<double>("geo_dd0_raw", n);
    g.gb_src = e->get<double>("geo_gb", n);
    g.land = e->get<double2>("geo_land", n);
  }
  g.parts = e->get<double>("geo_parts", (size_t)geo_parts(g.W, g.H) * g.n_poses * 8);
  g.scale = e->get<double>("geo_scale", (size_t)g.n_poses);
  g.value = e->get<double>("geo_value_ws", (size_t)g.n_poses);
  g.n_valid = (long long*)e->get<int64_t>("geo_nvalid_ws", (size_t)g.n_poses);
}

template <typename S2>
void run_forward_t(evcm_cuda_engine* e, const WinParams& P, uint64_t max_n, const double2* flows) {
  const size_t R = P.B + 1;
  S2* stack = e->get<S2>("stack", (size_t)P.n_windows * R * 2 * P.HW);
  e->mark(M_FWD0);
  ck(cudaMemsetAsync(stack, 0, (size_t)P.n_windows * R * 2 * P.HW * sizeof(S2), e->stream), "memset");
  e->mark(M_FWD0 + 1);
  launch_fwd_splat<S2>(e->stream, e->get<uint2>("packed", 1), e->get<uint64_t>("ev_off", 1), P, max_n,
                       flows, stack);
  e->mark(M_FWD0 + 2);
  const int parts = loss_parts(P);
  const size_t np = (size_t)P.n_windows * R * parts;
  launch_loss<S2>(e->stream, stack, P, e->get<S2>("coef", (size_t)P.n_windows * R * 2 * P.HW),
                  e->get<double>("part_acc", np), e->get<unsigned long long>("part_act", np),
                  e->get<double>("loss", P.n_windows), e->get<int>("no_surv", P.n_windows),
                  e->get<long long>("n_active", (size_t)P.n_windows * R),
                  e->get<double>("scale", (size_t)P.n_windows * R));
  e->mark(M_FWD0 + 3);
}

// Owner-computes forward (cmax_owner.cu): sort by the position at the middle
// reference, trajectory records + source lists, per-tile stack + loss partials +
// coefficient planes, loss finalize. Marks 2..6.
void run_forward_owner(evcm_cuda_engine* e, const WinParams& P, const double2* flows,
                       bool want_stack) {
  const TileParams& TP = e->TP;
  const int nw = P.n_windows, R = P.B + 1, NS = 2 * P.B + 1;
  const uint64_t total = e->n_total;
  const uint64_t* ev_off = e->get<uint64_t>("ev_off", 1);
  uint2* sorted = e->get<uint2>("sorted", total);
  uint32_t* tile_ptr = e->get<uint32_t>("tile_ptr", (size_t)nw * (TP.nT + 1));
  e->mark(2);
  // keys: unsorted + sorted keys, per-tile totals, then the coarse flow map (double2)
  uint32_t* keys = e->get<uint32_t>("sort_keys", 2 * total + (((size_t)nw * TP.nT + 3) & ~(size_t)3) +
                                                     (size_t)nw * P.B * TP.nT * 4);
  uint4* bbox = e->get<uint4>("bbox", (size_t)nw * NS * TP.nT);
  const size_t nl = (size_t)nw * NS * TP.oT;
  uint32_t* lcount = e->get<uint32_t>("lcount", nl);
  // the sort's first kernel also resets the cell boxes and list counts
  // the engine-level forward (want_stack) also keeps the sort permutation for
  // evcm_cuda_sort_products; the batched chain does not write it
  launch_sort(e->stream, e->get<uint2>("packed", 1), ev_off, P, TP, flows, total, keys,
              e->get<uint32_t>("sort_counts", (size_t)nw * TP.nT * TP.nchunks), tile_ptr, sorted,
              want_stack ? e->get<uint32_t>("perm", total) : nullptr,
              e->get<uint32_t>("bin_ptr", (size_t)nw * TP.nT * (P.B + 1)),
              e->get<uint32_t>("srcbase", (size_t)nw * P.B * TP.nT), bbox,
              (size_t)nw * NS * TP.nT, lcount, nl);
  e->mark(3);
  FwdRec* recs = e->get<FwdRec>("recs", (size_t)R * total);
  uint16_t* lists = e->get<uint16_t>("lists", nl * kListCapO);
  launch_traj_records(e->stream, sorted, ev_off, P, TP, tile_ptr, keys + total, e->max_n, flows,
                      total, recs, bbox, lcount, lists);
  uint2* ranges = e->get<uint2>("ranges", nl * (kListCapO + 2));
  launch_ranges(e->stream, lcount, lists, tile_ptr, e->get<uint32_t>("bin_ptr", 1),
                e->get<uint32_t>("srcbase", 1), P, TP, ranges);
  e->mark(4);
  const size_t np = (size_t)nw * R * TP.oT;
  double2* stack = want_stack ? e->get<double2>("stack", (size_t)nw * R * 2 * P.HW) : nullptr;
  // fixed-point accumulation: bit-deterministic in both modes
  launch_fwd_cells(e->stream, ev_off, P, TP, tile_ptr, recs, total, bbox, lcount, lists, ranges,
                   e->get<double2>("coef", (size_t)nw * R * 2 * P.HW), stack,
                   e->get<double>("part_acc", np), e->get<unsigned long long>("part_act", np),
                   owner_groups(TP, P, false));
  e->mark(5);
  launch_loss_finalize(e->stream, e->get<double>("part_acc", np),
                       e->get<unsigned long long>("part_act", np), TP.oT, P,
                       e->get<double>("loss", nw), e->get<int>("no_surv", nw),
                       e->get<long long>("n_active", (size_t)nw * R),
                       e->get<double>("scale", (size_t)nw * R));
  e->mark(6);
}

// Owner-computes backward: per-event adjoint -> per-bin (gx, gy), then the
// per-tile gradient gather with the fused flows backward (when depth is given)
// and/or the f64 gradient planes (grad_out, [w][B][2][HW]). Marks 7..9.
// flows32: fp32 copy of the window's flows (the flow-Jacobian operand of k_bwd_event)
void run_backward_owner(evcm_cuda_engine* e, const WinParams& P, const float2* flows32,
                        const double* depth, const uint8_t* mask, const double* pose_tab,
                        const double* K, double* d_depth, double* d_poses, double* grad_out) {
  const TileParams& TP = e->TP;
  const int nw = P.n_windows, R = P.B + 1;
  const uint64_t total = e->n_total;
  const uint64_t* ev_off = e->get<uint64_t>("ev_off", 1);
  const uint2* sorted = e->get<uint2>("sorted", 1);
  const uint32_t* tile_ptr = e->get<uint32_t>("tile_ptr", 1);
  const FwdRec* recs = e->get<FwdRec>("recs", (size_t)R * total);
  float2* bwd = e->get<float2>("bwdrec", (size_t)std::max(1, P.B - 1) * total);  // record-sink values
  uint32_t* gmax = e->get<uint32_t>("gmax", (size_t)nw);
  // source-pixel sinks with their packed events, (bin, tile, time) order
  uint4* srcrec = e->get<uint4>("srcrec", total);
  launch_bwd_event(e->stream, sorted, ev_off, P, TP, tile_ptr, e->max_n, flows32, recs, total,
                   e->get<double2>("coef", 1), e->get<double>("scale", 1), e->get<int>("no_surv", 1),
                   e->get<uint32_t>("sort_keys", 1) + total, e->get<uint32_t>("bin_ptr", 1),
                   e->get<uint32_t>("srcbase", 1), srcrec, bwd, gmax);
  e->mark(7);
  double* pose_part =
      depth ? e->get<double>("pose_part_owner", (size_t)nw * TP.oT * P.B * kPoseSums) : nullptr;
  const int bgroups = owner_groups(TP, P, true);
  launch_bwd_cells(e->stream, sorted, ev_off, P, TP, tile_ptr, e->get<uint32_t>("bin_ptr", 1), recs,
                   bwd, total, gmax, e->get<uint4>("bbox", 1), e->get<uint32_t>("lcount", 1),
                   e->get<uint16_t>("lists", 1), e->get<uint2>("ranges", 1),
                   e->get<uint32_t>("srcbase", 1), srcrec, e->get<int>("no_surv", 1),
                   depth, mask, pose_tab,
                   K, depth ? d_depth : nullptr, pose_part, grad_out, bgroups,
                   bgroups > 1 && depth ? e->get<double>("dbin", (size_t)nw * P.B * P.HW) : nullptr);
  e->mark(8);
  if (depth) launch_pose_contract(e->stream, pose_part, TP.oT, P.B, nw, pose_tab, d_poses);
  e->mark(9);
}

void run_forward(evcm_cuda_engine* e, const WinParams& P, uint64_t max_n, const double2* flows,
                 bool want_stack = false) {
  if (e->owner()) run_forward_owner(e, P, flows, want_stack);
  else if (e->opt.stack_f64) run_forward_t<double2>(e, P, max_n, flows);
  else run_forward_t<float2>(e, P, max_n, flows);
}

template <typename C2, typename G2>
void* run_backward_t(evcm_cuda_engine* e, const WinParams& P, uint64_t max_n, const double2* flows) {
  G2* grad = e->get<G2>("grad", (size_t)P.n_windows * P.B * P.HW);
  ck(cudaMemsetAsync(grad, 0, (size_t)P.n_windows * P.B * P.HW * sizeof(G2), e->stream), "memset");
  e->mark(M_FWD0 + 4);
  launch_bwd<C2, G2>(e->stream, e->get<uint2>("packed", 1), e->get<uint64_t>("ev_off", 1), P, max_n,
                     flows, e->get<C2>("coef", 1), e->get<double>("scale", 1),
                     e->get<int>("no_surv", 1), grad);
  e->mark(M_FWD0 + 5);
  return grad;
}

void* run_backward(evcm_cuda_engine* e, const WinParams& P, uint64_t max_n, const double2* flows) {
  if (e->opt.stack_f64)
    return e->opt.grad_f64 ? run_backward_t<double2, double2>(e, P, max_n, flows)
                           : run_backward_t<double2, float2>(e, P, max_n, flows);
  return e->opt.grad_f64 ? run_backward_t<float2, double2>(e, P, max_n, flows)
                         : run_backward_t<float2, float2>(e, P, max_n, flows);
}

// Shared front half of forward(): validation, staging, flows.
const double2* prepare_window(evcm_cuda_engine* e, const evcm_slice* s, const evcm_flows* f, int mem,
                              WinParams* P_out) {
  if (!s || !f) fail(EVCM_ERR_CONFIG, "null slice or flows");
  check_slice_header(s);
  // per-event validation (device) happens before the flow checks, as in
  // Engine::validate_window (slice.validate() first, engine.hpp:216)
  WinParams P0{};
  P0.W = s->width;
  P0.H = s->height;
  P0.HW = s->width * s->height;
  P0.n_windows = 1;
  P0.t0 = s->t_start_us;
  P0.t_end = s->t_end_us;
  const uint64_t off[2] = {0, s->n_events};
  if (s->n_events >= (1ull << 32)) fail(EVCM_ERR_CONFIG, "cuda backend: more than 2^32 events");
  stage_events(e, s->events, off, P0, mem);
  try {
    check_flows(s, f);
  } catch (const Failure&) {
    sync_and_check(e, "stage");  // event errors take precedence (engine.hpp:216-217)
    throw;
  }
  WinParams P = make_params(s->width, s->height, f->edges_us, f->n_bins, 1, s->t_start_us, s->t_end_us);
  const size_t nf = (size_t)f->n_bins * 2 * P.HW;
  const double* uv = to_device(e, "flows_planar", f->uv, nf, mem);
  double2* flows = e->get<double2>("flows", (size_t)f->n_bins * P.HW);
  launch_interleave_flows(e->stream, uv, f->n_bins, P.HW, flows);
  *P_out = P;
  return flows;
}

}  // namespace

// ============================================================================
// C-ABI

extern "C" {

int evcm_cuda_abi_version(void) { return EVCM_CUDA_ABI_VERSION; }

const char* evcm_cuda_last_error(void) { return g_err.c_str(); }

const char* evcm_cuda_error_name(int status) { return code_name(status); }

void evcm_cuda_default_options(evcm_cuda_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->device = 0;
  o->deterministic = 1;  // engine.hpp:60
  o->stack_f64 = 1;  // parity precision
  o->grad_f64 = 0;
  o->stream = nullptr;
  o->algo = 2;  // auto
}

int evcm_cuda_create(const evcm_cuda_options* opts, evcm_cuda_engine** out) {
  return guarded([&] {
    if (!out) fail(EVCM_ERR_CONFIG, "null output handle");
    evcm_cuda_options o;
    evcm_cuda_default_options(&o);
    if (opts) o = *opts;
    int n = 0;
    ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (o.device < 0 || o.device >= n) fail(EVCM_ERR_CONFIG, "engine: no such CUDA device");
    if (o.algo < 0 || o.algo > 2) fail(EVCM_ERR_CONFIG, "engine: unknown algo (0 owner, 1 atomic, 2 auto)");
    if (o.algo == 1 && o.deterministic)
      fail(EVCM_ERR_CONFIG, "deterministic mode needs algo owner or auto");
    auto* e = new evcm_cuda_engine();
    e->opt = o;
    set_device(e);
    if (o.stream) {
      e->stream = static_cast<cudaStream_t>(o.stream);
    } else {
      ck(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking), "cudaStreamCreate");
      e->own_stream = true;
    }
    *out = e;
  });
}

void evcm_cuda_destroy(evcm_cuda_engine* e) {
  if (!e) return;
  cudaSetDevice(e->opt.device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  for (auto& kv : e->bufs)
    if (kv.second.p) cudaFree(kv.second.p);
  for (auto& kv : e->pins)
    if (kv.second.p) cudaFreeHost(kv.second.p);
  for (cudaEvent_t ev : e->ev) cudaEventDestroy(ev);
  if (e->order_ev) cudaEventDestroy(e->order_ev);
  for (auto& g : e->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto& q : e->pending)
    if (q.done) cudaEventDestroy(q.done);
  if (e->own_stream) cudaStreamDestroy(e->stream);
  delete e;
}

int evcm_cuda_set_timing(evcm_cuda_engine* e, int enabled) {
  return guarded([&] {
    if (!e) fail(EVCM_ERR_CONFIG, "null engine");
    e->timing = enabled != 0;
  });
}

int evcm_cuda_stage_times(evcm_cuda_engine* e, double* ms, int max_stages) {
  if (!e) return 0;
  const int n = std::min<int>(max_stages, (int)e->stage_ms.size());
  for (int i = 0; i < n; ++i) ms[i] = e->stage_ms[i];
  return n;
}

int evcm_cuda_last_launch_count(evcm_cuda_engine* e) { return e ? e->last_launches : 0; }

int evcm_cuda_last_algo(evcm_cuda_engine* e) { return e ? (e->owner() ? 0 : 1) : -1; }

size_t evcm_cuda_workspace_bytes(evcm_cuda_engine* e) {
  size_t s = 0;
  if (e)
    for (auto& kv : e->bufs) s += kv.second.cap;
  return s;
}

// The API forward/backward always time their phases (PhaseStats, engine.hpp:226-242):
// the stage marks are CUDA events on the engine stream, read after the call's sync.
struct ForceTiming {
  evcm_cuda_engine* e;
  bool saved;
  explicit ForceTiming(evcm_cuda_engine* x) : e(x), saved(x->timing) { e->timing = true; }
  ~ForceTiming() { e->timing = saved; }
};

int evcm_cuda_forward(evcm_cuda_engine* e, const evcm_slice* s, const evcm_flows* f, int mem,
                      evcm_loss* loss) {
  return guarded([&] {
    if (!e) fail(EVCM_ERR_CONFIG, "null engine");
    set_device(e);
    reset_launch_count();
    ForceTiming ft(e);
    e->have_fwd = false;
    e->fwd_id = 0;
    e->mark(0);
    WinParams P;
    const double2* flows = prepare_window(e, s, f, mem, &P);
    e->mark(1);
    run_forward(e, P, s->n_events, flows, /*want_stack=*/true);
    double l = 0;
    int ns = 0;
    ck(cudaMemcpyAsync(&l, e->get<double>("loss", 1), sizeof l, cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaMemcpyAsync(&ns, e->get<int>("no_surv", 1), sizeof ns, cudaMemcpyDeviceToHost, e->stream), "D2H");
    sync_and_check(e, "forward");
    const int last = e->owner() ? 6 : M_FWD0 + 3;
    e->collect_range(0, last);
    // phases: warp = staging + sort + trajectory records (owner) | staging + memset
    // (atomic, whose warp is fused into the splat kernel); splat; loss
    const int splat = e->owner() ? 4 : M_FWD0 + 1;
    double warp = 0;
    for (int i = 0; i < splat; ++i) warp += e->stage_ms[i];
    e->phase_us[0] = 1e3 * warp;
    e->phase_us[1] = 1e3 * e->stage_ms[splat];
    e->phase_us[2] = 1e3 * e->stage_ms[splat + 1];
    e->phase_bytes[0] = e->ws_at_mark[splat];
    e->phase_bytes[1] = e->ws_at_mark[splat + 1];
    e->phase_bytes[2] = e->ws_at_mark[last];
    e->P = P;
    e->n_events = s->n_events;
    e->have_fwd = true;
    e->fwd_id = ++e->fwd_counter;
    if (loss) {
      loss->value = l;
      loss->no_survivors = ns;
      loss->forward_id = e->fwd_id;
    }
    e->last_launches = launch_count();
  });
}

int evcm_cuda_forward_products(evcm_cuda_engine* e, double* count, double* tsum, int64_t* n_active,
                               uint8_t* alive, int32_t* bin, double* pos, size_t* n_alive) {
  return guarded([&] {
    if (!e || !e->have_fwd) fail(EVCM_ERR_STATE, "engine: no forward result to read");
    set_device(e);
    const WinParams& P = e->P;
    const size_t R = P.B + 1, HW = P.HW, n = e->n_events;
    if (count || tsum) {
      double* c = e->get<double>("prod_count", R * 2 * HW);
      double* t = e->get<double>("prod_tsum", R * 2 * HW);
      if (e->owner() || e->opt.stack_f64)
        launch_unpack_stack<double2>(e->stream, e->get<double2>("stack", 1), R * 2, P.HW, c, t);
      else
        launch_unpack_stack<float2>(e->stream, e->get<float2>("stack", 1), R * 2, P.HW, c, t);
      if (count) from_device(e, count, c, R * 2 * HW * sizeof(double), EVCM_MEM_HOST);
      if (tsum) from_device(e, tsum, t, R * 2 * HW * sizeof(double), EVCM_MEM_HOST);
    }
    if (n_active)
      from_device(e, n_active, e->get<long long>("n_active", R), R * sizeof(int64_t), EVCM_MEM_HOST);
    if (alive || bin || pos || n_alive) {
      uint8_t* a = e->get<uint8_t>("prod_alive", n);
      int32_t* b = e->get<int32_t>("prod_bin", n);
      double* p = pos ? e->get<double>("prod_pos", n * R * 2) : nullptr;
      launch_traj_products(e->stream, e->get<uint2>("packed", 1), n, P, e->get<double2>("flows", 1), a, b, p);
      std::vector<uint8_t> tmp;
      uint8_t* ah = alive;
      if (!ah && n_alive) {
        tmp.resize(n);
        ah = tmp.data();
      }
      if (ah) from_device(e, ah, a, n, EVCM_MEM_HOST);
      if (bin) from_device(e, bin, b, n * sizeof(int32_t), EVCM_MEM_HOST);
      if (pos) from_device(e, pos, p, n * R * 2 * sizeof(double), EVCM_MEM_HOST);
      ck(cudaStreamSynchronize(e->stream), "products");
      if (n_alive) {
        size_t c = 0;
        for (size_t k = 0; k < n; ++k) c += ah[k];
        *n_alive = c;
      }
    }
    ck(cudaStreamSynchronize(e->stream), "products");
  });
}

namespace {
void backward_impl(evcm_cuda_engine* e, const evcm_slice* s, const evcm_flows* f, int mem,
                   double* grad, uint64_t want_id) {
  if (!e) fail(EVCM_ERR_CONFIG, "null engine");
  if (!s || !f) fail(EVCM_ERR_CONFIG, "null slice or flows");
  set_device(e);
  reset_launch_count();
  ForceTiming ft(e);
  check_slice_header(s);
  check_flows(s, f);
  if (!e->have_fwd || e->n_events != s->n_events || e->P.W != s->width || e->P.H != s->height ||
      e->P.B != f->n_bins || (want_id && want_id != e->fwd_id))
    fail(EVCM_ERR_STATE, "engine: backward needs the forward of the same window");
  const WinParams& P = e->P;
  const int m0 = e->owner() ? 6 : M_FWD0 + 3;
  e->mark(m0);
  // the flow Jacobians come from the flows given here (engine.hpp:185-205); the
  // trajectories from the forward (its records / packed events)
  const double* uv = to_device(e, "flows_planar", f->uv, (size_t)f->n_bins * 2 * P.HW, mem);
  double2* flows = e->get<double2>("flows", (size_t)f->n_bins * P.HW);
  float2* flows32 = e->owner() ? e->get<float2>("flows32", (size_t)f->n_bins * P.HW) : nullptr;
  launch_interleave_flows(e->stream, uv, f->n_bins, P.HW, flows, flows32);
  double* out = e->get<double>("grad_f64", (size_t)P.B * 2 * P.HW);
  if (e->owner()) {
    run_backward_owner(e, P, flows32, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, out);
  } else {
    void* g = run_backward(e, P, s->n_events, flows);
    if (e->opt.grad_f64)
      launch_unpack_grad<double2>(e->stream, static_cast<double2*>(g), P.B, P.HW, out);
    else
      launch_unpack_grad<float2>(e->stream, static_cast<float2*>(g), P.B, P.HW, out);
  }
  from_device(e, grad, out, (size_t)P.B * 2 * P.HW * sizeof(double), mem);
  const int m1 = e->owner() ? 9 : M_FWD0 + 5;
  e->mark(m1);
  ck(cudaStreamSynchronize(e->stream), "backward");
  e->collect_range(m0, m1);
  double t = 0;
  for (int i = m0; i < m1; ++i) t += e->stage_ms[i];
  e->phase_us[3] = 1e3 * t;
  e->phase_bytes[3] = e->ws_at_mark[m1];
  ck(cudaGetLastError(), "backward kernels");
  e->last_launches = launch_count();
}
}  // namespace

int evcm_cuda_backward(evcm_cuda_engine* e, const evcm_slice* s, const evcm_flows* f, int mem,
                       double* grad) {
  return guarded([&] { backward_impl(e, s, f, mem, grad, 0); });
}

int evcm_cuda_backward_of(evcm_cuda_engine* e, const evcm_slice* s, const evcm_flows* f,
                          uint64_t forward_id, int mem, double* grad) {
  return guarded([&] {
    if (forward_id == 0) fail(EVCM_ERR_STATE, "engine: backward needs the forward of the same window");
    backward_impl(e, s, f, mem, grad, forward_id);
  });
}

int evcm_cuda_sort_products(evcm_cuda_engine* e, uint32_t* keys, uint32_t* perm, uint32_t* sorted_keys,
                            size_t* n_sorted) {
  return guarded([&] {
    if (!e || !e->have_fwd) fail(EVCM_ERR_STATE, "engine: no forward result to read");
    if (!e->owner()) fail(EVCM_ERR_STATE, "engine: the last forward did not sort (algo atomic)");
    set_device(e);
    const size_t n = e->n_events, total = e->n_total;
    const uint32_t* kd = e->get<uint32_t>("sort_keys", 1);
    uint32_t nv = 0;
    from_device(e, &nv, e->get<uint32_t>("tile_ptr", 1) + e->TP.nT, sizeof nv, EVCM_MEM_HOST);
    if (keys) from_device(e, keys, kd, n * sizeof(uint32_t), EVCM_MEM_HOST);
    if (sorted_keys) from_device(e, sorted_keys, kd + total, n * sizeof(uint32_t), EVCM_MEM_HOST);
    if (perm) from_device(e, perm, e->get<uint32_t>("perm", total), n * sizeof(uint32_t), EVCM_MEM_HOST);
    ck(cudaStreamSynchronize(e->stream), "sort products");
    if (n_sorted) *n_sorted = nv;
  });
}

int evcm_cuda_phase_stats(evcm_cuda_engine* e, double* time_us, size_t* peak_bytes) {
  return guarded([&] {
    if (!e) fail(EVCM_ERR_CONFIG, "null engine");
    for (int i = 0; i < 4; ++i) {
      if (time_us) time_us[i] = e->phase_us[i];
      if (peak_bytes) peak_bytes[i] = e->phase_bytes[i];
    }
  });
}

int evcm_cuda_stream_wait(evcm_cuda_engine* e, void* stream) {
  return guarded([&] {
    if (!e) fail(EVCM_ERR_CONFIG, "null engine");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (st == e->stream) return;
    set_device(e);
    if (!e->order_ev) ck(cudaEventCreateWithFlags(&e->order_ev, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(e->order_ev, st), "event record");
    ck(cudaStreamWaitEvent(e->stream, e->order_ev, 0), "stream wait");
  });
}

int evcm_cuda_stream_signal(evcm_cuda_engine* e, void* stream) {
  return guarded([&] {
    if (!e) fail(EVCM_ERR_CONFIG, "null engine");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (st == e->stream) return;
    set_device(e);
    if (!e->order_ev) ck(cudaEventCreateWithFlags(&e->order_ev, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(e->order_ev, e->stream), "event record");
    ck(cudaStreamWaitEvent(st, e->order_ev, 0), "stream wait");
  });
}

int evcm_cuda_loss_and_grad(evcm_cuda_engine* e, const evcm_slice* s, const evcm_flows* f, int mem,
                            evcm_loss* loss, double* grad) {
  int rc = evcm_cuda_forward(e, s, f, mem, loss);
  if (rc) return rc;
  const int l1 = e->last_launches;
  rc = evcm_cuda_backward(e, s, f, mem, grad);
  if (!rc) e->last_launches += l1;
  return rc;
}

int evcm_cuda_depth_pose_to_flows(evcm_cuda_engine* e, int W, int H, const double* depth,
                                  const uint8_t* mask, int B, const double* poses, const double* K,
                                  uint64_t t0, uint64_t t1, int mem, double* flows_out,
                                  uint8_t* valid, uint64_t* edges_out) {
  return guarded([&] {
    if (!e) fail(EVCM_ERR_CONFIG, "null engine");
    set_device(e);
    reset_launch_count();
    if (B < 1) fail(EVCM_ERR_CONFIG, "depth_pose_to_flows: need one pose per bin");
    if (W <= 0 || H <= 0 || !depth) fail(EVCM_ERR_DIMENSION, "depth_pose_to_flows: empty depth");
    const std::vector<uint64_t> edges = zeros_edges(t0, t1, B);
    WinParams P = make_params(W, H, edges.data(), B, 1, t0, t1);
    std::vector<double> ph(poses, poses + (mem == EVCM_MEM_HOST ? 6 * B : 0));
    if (mem == EVCM_MEM_DEVICE) {
      ph.resize(6 * B);
      ck(cudaMemcpy(ph.data(), poses, 6 * B * sizeof(double), cudaMemcpyDeviceToHost), "D2H poses");
    }
    const double* tab = upload_pose_table(e, ph.data(), 1, B, edges.data(), true);
    const double* dd = to_device(e, "depth", depth, (size_t)P.HW, mem);
    const uint8_t* md = mask ? to_device(e, "mask", mask, (size_t)P.HW, mem) : nullptr;
    // its own buffer: the forward's flows stay intact for a following backward
    double2* fl = e->get<double2>("mf_flows", (size_t)B * P.HW);
    uint8_t* vd = valid ? e->get<uint8_t>("valid", (size_t)B * P.HW) : nullptr;
    launch_motion_field(e->stream, dd, md, tab, P, K, fl, vd);
    double* planar = e->get<double>("flows_planar_out", (size_t)B * 2 * P.HW);
    launch_unpack_grad<double2>(e->stream, fl, B, P.HW, planar);  // same [B][2][HW] unpack
    from_device(e, flows_out, planar, (size_t)B * 2 * P.HW * sizeof(double), mem);
    if (valid) from_device(e, valid, vd, (size_t)B * P.HW, mem);
    if (edges_out) std::memcpy(edges_out, edges.data(), (B + 1) * sizeof(uint64_t));
    e->stage_nw = 0;
    sync_and_check(e, "depth_pose_to_flows");
    e->last_launches = launch_count();
  });
}

int evcm_cuda_depth_pose_to_flows_backward(evcm_cuda_engine* e, int W, int H, const double* depth,
                                           const uint8_t* mask, int B, const double* poses,
                                           const double* K, const uint64_t* edges,
                                           const double* grad, int mem, double* d_depth,
                                           double* d_poses) {
  return guarded([&] {
    if (!e) fail(EVCM_ERR_CONFIG, "null engine");
    set_device(e);
    reset_launch_count();
    if (B < 1 || !edges) fail(EVCM_ERR_CONFIG, "flows backward: bins, poses, and gradients must align");
    if (W <= 0 || H <= 0) fail(EVCM_ERR_DIMENSION, "flows backward: grids must match the depth map");
    WinParams P = make_params(W, H, edges, B, 1, edges[0], edges[B]);
    std::vector<double> ph(6 * B);
    if (mem == EVCM_MEM_DEVICE)
      ck(cudaMemcpy(ph.data(), poses, 6 * B * sizeof(double), cudaMemcpyDeviceToHost), "D2H poses");
    else
      std::memcpy(ph.data(), poses, 6 * B * sizeof(double));
    // geometry.hpp:293-296 does not re-validate poses, so neither do we.
    const double* tab_d = upload_pose_table(e, ph.data(), 1, B, edges, false);
    const double* dd = to_device(e, "depth", depth, (size_t)P.HW, mem);
    const uint8_t* md = mask ? to_device(e, "mask", mask, (size_t)P.HW, mem) : nullptr;
    const double* gp = to_device(e, "grad_planar_in", grad, (size_t)B * 2 * P.HW, mem);
    double2* g2 = e->get<double2>("grad_in", (size_t)B * P.HW);
    launch_interleave_flows(e->stream, gp, B, P.HW, g2);
    double* ddo = e->get<double>("d_depth", (size_t)P.HW);
    double* pp = e->get<double>("pose_part", (size_t)flows_bwd_parts(P) * B * kPoseSums);
    double* dpo = e->get<double>("d_poses", (size_t)B * 6);
    launch_flows_bwd<double2>(e->stream, dd, md, tab_d, P, K, g2, ddo, pp, dpo);
    from_device(e, d_depth, ddo, (size_t)P.HW * sizeof(double), mem);
    from_device(e, d_poses, dpo, (size_t)B * 6 * sizeof(double), mem);
    e->stage_nw = 0;
    sync_and_check(e, "flows backward");
    e->last_launches = launch_count();
  });
}

}  // extern "C"

namespace {
// The batched chain; depth_dev (device, [n_windows][H][W]) replaces bt->depth
// when given (the predictor path decodes the depth on the device).
void chain_enqueue(evcm_cuda_engine* e, const evcm_chain_batch* bt, int in_mem, int out_mem,
                   evcm_chain_out* out, const double* depth_dev) {
  {
    reset_launch_count();
    const int nw = bt->n_windows, B = bt->n_bins, W = bt->width, H = bt->height;
    if (nw < 1) fail(EVCM_ERR_CONFIG, "chain: need at least one window");
    if (W <= 0 || H <= 0 || W > 65535 || H > 65535) fail(EVCM_ERR_DIMENSION, "chain: bad sensor size");
    if (bt->t_end_us <= bt->t_start_us || bt->t_end_us - bt->t_start_us >= (1ull << 31))
      fail(EVCM_ERR_CONFIG, "chain: window must be nonempty and shorter than 2^31 us");
    // event offsets: n_windows + 1 host entries from 0, non-decreasing
    if (bt->ev_offsets[0] != 0) fail(EVCM_ERR_CONFIG, "chain: ev_offsets[0] must be 0");
    for (int w = 0; w < nw; ++w)
      if (bt->ev_offsets[w + 1] < bt->ev_offsets[w])
        fail(EVCM_ERR_CONFIG, "chain: ev_offsets must be non-decreasing");
    if (bt->ev_offsets[nw] >= (1ull << 32)) fail(EVCM_ERR_CONFIG, "chain: more than 2^32 events");
    const std::vector<uint64_t> edges = zeros_edges(bt->t_start_us, bt->t_end_us, B);
    WinParams P = make_params(W, H, edges.data(), B, nw, bt->t_start_us, bt->t_end_us);
    P.stride_us = bt->window_stride_us;
    e->have_fwd = false;
    e->fwd_id = 0;
    e->mark(0);
    // Rotation tables: host poses -> built on the host with the reference's own
    // expression order (bit-identical flows); device poses -> k_pose_table (no
    // host round trip; validation reported through a device flag).
    const double* tab;
    const bool prepared = nw <= kInitMaxWin;
    if (prepared) {
      // offsets, validation words and (device poses) the pose table in one launch
      ChainInit a;
      for (int w = 0; w <= nw; ++w) a.off[w] = bt->ev_offsets[w];
      a.nw = nw;
      a.B = B;
      a.ev_off = e->get<uint64_t>("ev_off", nw + 1);
      a.err = e->get<unsigned long long>("stage_err", nw + 1);
      a.poses = in_mem == EVCM_MEM_DEVICE ? bt->poses : nullptr;
      a.tab = e->get<double>("pose_tab", (size_t)nw * B * kPoseTab);
      if (in_mem != EVCM_MEM_DEVICE) {  // host poses: host-built table (bit-identical R)
        const size_t np = (size_t)nw * B * 6;
        double* ph = e->pinned<double>("poses_h", np);
        std::memcpy(ph, bt->poses, np * sizeof(double));
        tab = upload_pose_table(e, ph, nw, B, edges.data(), true);
      } else {
        tab = a.tab;
        e->check_pose_flag = true;
      }
      launch_chain_init(e->stream, a, P);
    } else if (in_mem == EVCM_MEM_DEVICE) {
      double* inv = e->pinned<double>("inv_dt_h", B);
      for (int b = 0; b < B; ++b)
        inv[b] = 1.0 / ((static_cast<double>(edges[b + 1]) - static_cast<double>(edges[b])) * 1e-6);
      double* inv_d = e->get<double>("inv_dt", B);
      ck(cudaMemcpyAsync(inv_d, inv, B * sizeof(double), cudaMemcpyHostToDevice, e->stream), "H2D");
      // the pose flag lives in validation word nw (copied back by stage_events)
      unsigned long long* errw = e->get<unsigned long long>("stage_err", nw + 1);
      ck(cudaMemsetAsync(errw + nw, 0, sizeof(unsigned long long), e->stream), "memset");
      double* tab_d = e->get<double>("pose_tab", (size_t)nw * B * kPoseTab);
      launch_pose_table(e->stream, bt->poses, nw, B, inv_d, tab_d,
                        reinterpret_cast<int*>(errw + nw));
      e->check_pose_flag = true;
      tab = tab_d;
    } else {
      const size_t np = (size_t)nw * B * 6;
      double* ph = e->pinned<double>("poses_h", np);
      std::memcpy(ph, bt->poses, np * sizeof(double));
      tab = upload_pose_table(e, ph, nw, B, edges.data(), true);
    }
    uint64_t max_n = 0;
    for (int w = 0; w < nw; ++w) max_n = std::max<uint64_t>(max_n, bt->ev_offsets[w + 1] - bt->ev_offsets[w]);
    stage_events(e, bt->events, bt->ev_offsets, P, in_mem, prepared);
    const double* depth =
        depth_dev ? depth_dev : to_device(e, "depth", bt->depth, (size_t)nw * P.HW, in_mem);
    double2* flows = e->get<double2>("flows", (size_t)nw * B * P.HW);
    float2* flows32 = e->owner() ? e->get<float2>("flows32", (size_t)nw * B * P.HW) : nullptr;
    e->mark(1);
    launch_motion_field(e->stream, depth, nullptr, tab, P, bt->K, flows, nullptr, flows32);
    run_forward(e, P, max_n, flows);
    const bool direct = out_mem == EVCM_MEM_DEVICE;
    double* ddo = (direct && out->d_depth) ? out->d_depth : e->get<double>("d_depth", (size_t)nw * P.HW);
    double* dpo = (direct && out->d_poses) ? out->d_poses : e->get<double>("d_poses", (size_t)nw * B * 6);
    if (e->owner()) {
      run_backward_owner(e, P, flows32, depth, nullptr, tab, bt->K, ddo, dpo, nullptr);
    } else {
      void* g = run_backward(e, P, max_n, flows);
      double* pp = e->get<double>("pose_part", (size_t)nw * flows_bwd_parts(P) * B * kPoseSums);
      if (e->opt.grad_f64)
        launch_flows_bwd<double2>(e->stream, depth, nullptr, tab, P, bt->K, static_cast<double2*>(g), ddo, pp, dpo);
      else
        launch_flows_bwd<float2>(e->stream, depth, nullptr, tab, P, bt->K, static_cast<float2*>(g), ddo, pp, dpo);
      e->mark(M_FWD0 + 6);
    }
    if (out->sums) {  // the data-parallel payload, summed in window order
      const size_t ns = 1 + (size_t)P.HW + (size_t)B * 6;
      double* sd = direct ? out->sums : e->get<double>("sums", ns);
      launch_window_sums(e->stream, e->get<double>("loss", nw), ddo, dpo, nw, P.HW, B * 6, sd);
      if (!direct) from_device(e, out->sums, sd, ns * sizeof(double), out_mem);
    }
    if (out->loss) from_device(e, out->loss, e->get<double>("loss", nw), nw * sizeof(double), out_mem);
    if (out->no_survivors) from_device(e, out->no_survivors, e->get<int>("no_surv", nw), nw * sizeof(int), out_mem);
    if (out->d_depth && ddo != out->d_depth) from_device(e, out->d_depth, ddo, (size_t)nw * P.HW * sizeof(double), out_mem);
    if (out->d_poses && dpo != out->d_poses) from_device(e, out->d_poses, dpo, (size_t)nw * B * 6 * sizeof(double), out_mem);
  }
}

// Signature of a graph-replayable chain call (device inputs and outputs only:
// host buffers would be read at capture time, not at replay time).
std::vector<uint64_t> chain_signature(const evcm_cuda_engine* e, const evcm_chain_batch* bt,
                                      const evcm_chain_out* out, const double* depth_dev) {
  std::vector<uint64_t> g;
  auto u = [&](uint64_t v) { g.push_back(v); };
  auto d = [&](double v) {
    uint64_t b;
    std::memcpy(&b, &v, 8);
    g.push_back(b);
  };
  u((uint64_t)e->slot);  // the slot's pinned error words are baked into the graph
  u((uint64_t)bt->n_windows); u((uint64_t)bt->width); u((uint64_t)bt->height); u((uint64_t)bt->n_bins);
  u(bt->t_start_us); u(bt->t_end_us); u(bt->window_stride_us);
  for (double k : bt->K) d(k);
  u((uint64_t)(uintptr_t)bt->events); u((uint64_t)(uintptr_t)(depth_dev ? depth_dev : bt->depth));
  u((uint64_t)(uintptr_t)bt->poses); u((uint64_t)(uintptr_t)out->loss);
  u((uint64_t)(uintptr_t)out->no_survivors); u((uint64_t)(uintptr_t)out->d_depth);
  u((uint64_t)(uintptr_t)out->d_poses); u((uint64_t)(uintptr_t)out->sums);
  u((uint64_t)e->opt.algo); u((uint64_t)e->opt.deterministic); u((uint64_t)e->opt.stack_f64);
  u((uint64_t)e->opt.grad_f64);
  for (int w = 0; w <= bt->n_windows; ++w) u(bt->ev_offsets[w]);
  return g;
}

void chain_impl(evcm_cuda_engine* e, const evcm_chain_batch* bt, int in_mem, int out_mem,
                evcm_chain_out* out, const double* depth_dev, bool async = false) {
  if (!e || !bt || !out || !bt->ev_offsets) fail(EVCM_ERR_CONFIG, "null argument");
  set_device(e);
  // graphs only where every host-side input of the enqueue is baked into kernel
  // parameters: device inputs and outputs, and offsets that fit k_chain_init
  const bool graphable = in_mem == EVCM_MEM_DEVICE && out_mem == EVCM_MEM_DEVICE && !e->timing &&
                         bt->n_windows <= kInitMaxWin;
  std::vector<uint64_t> sig;
  if (graphable) sig = chain_signature(e, bt, out, depth_dev);
  using GE = evcm_cuda_engine::GraphEntry;
  GE* g = nullptr;
  if (graphable) {
    for (GE& x : e->graphs)
      if (x.sig == sig) g = &x;
    if (g && g->gen != e->alloc_gen) {  // workspace moved since the capture
      if (g->exec) cudaGraphExecDestroy(g->exec);
      g->exec = nullptr;
      g->failed = false;
      g->gen = e->alloc_gen;
      g->last_use = ++e->use_clock;
      g = nullptr;  // this call runs eagerly (and re-sizes nothing); the next captures
      for (GE& x : e->graphs)
        if (x.sig == sig) x.gen = e->alloc_gen;
      goto eager;
    }
  }
  if (g && g->exec) {
    // replay: the state the eager path leaves behind is unchanged (same signature)
    g->last_use = ++e->use_clock;
    ck(cudaGraphLaunch(g->exec, e->stream), "graph launch");
    e->have_fwd = false;
    e->fwd_id = 0;
    e->last_launches = g->launches;
    if (async) {  // checked by evcm_cuda_chain_wait(slot)
      auto& q = e->pending[e->slot];
      if (!q.done) ck(cudaEventCreateWithFlags(&q.done, cudaEventDisableTiming), "event");
      ck(cudaEventRecord(q.done, e->stream), "event record");
      q.active = true;
      q.nw = bt->n_windows;
      q.pose = true;  // graphs only exist for device inputs: device pose tables
      return;
    }
    e->stage_nw = bt->n_windows;
    e->check_pose_flag = true;
    sync_and_check(e, "chain");
    return;
  }
  if (graphable && !g) {  // first call of this signature: remember it, run eagerly
    if (e->graphs.size() >= evcm_cuda_engine::kGraphCache) {
      auto lru = std::min_element(e->graphs.begin(), e->graphs.end(),
                                  [](const GE& x, const GE& y) { return x.last_use < y.last_use; });
      if (lru->exec) cudaGraphExecDestroy(lru->exec);
      e->graphs.erase(lru);
    }
    GE ne;
    ne.sig = sig;
    ne.last_use = ++e->use_clock;
    e->graphs.push_back(ne);
    // sized by this eager run; the capture of the next identical call must not
    // see a reallocation, so the entry's generation is taken after it
    chain_enqueue(e, bt, in_mem, out_mem, out, depth_dev);
    sync_and_check(e, "chain");
    e->graphs.back().gen = e->alloc_gen;
    for (GE& x : e->graphs)  // earlier entries survive only if nothing moved
      if (x.gen != e->alloc_gen && x.exec) {
        cudaGraphExecDestroy(x.exec);
        x.exec = nullptr;
        x.gen = e->alloc_gen;
      }
    e->collect_range(0, e->owner() ? 9 : M_FWD0 + 6);
    e->last_launches = launch_count();
    return;
  }
  if (g && !g->failed) {
    // second identical call: capture the enqueue into a graph, then replay it
    g->last_use = ++e->use_clock;
    cudaGraph_t graph = nullptr;
    ck(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    bool ok = true;
    try {
      chain_enqueue(e, bt, in_mem, out_mem, out, depth_dev);
    } catch (...) {
      ok = false;
      cudaStreamEndCapture(e->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    if (cudaStreamEndCapture(e->stream, &graph) != cudaSuccess ||
        cudaGraphInstantiate(&g->exec, graph, 0) != cudaSuccess) {
      ok = false;
      g->exec = nullptr;
      cudaGetLastError();
    }
    if (graph) cudaGraphDestroy(graph);
    if (ok && g->gen == e->alloc_gen) {
      g->launches = launch_count();
      ck(cudaGraphLaunch(g->exec, e->stream), "graph launch");
      sync_and_check(e, "chain");
      e->last_launches = g->launches;
      return;
    }
    if (ok) {  // a buffer moved during the capture: the graph is stale
      cudaGraphExecDestroy(g->exec);
      g->exec = nullptr;
      g->gen = e->alloc_gen;
    } else {
      g->failed = true;  // fall through: eager run
    }
  }
eager:
  chain_enqueue(e, bt, in_mem, out_mem, out, depth_dev);
  sync_and_check(e, "chain");
  e->collect_range(0, e->owner() ? 9 : M_FWD0 + 6);
  e->last_launches = launch_count();
}

void check_grid(int pw, int ph, int factor, const void* params) {  // DirectPredictor::validate
  if (pw <= 0 || ph <= 0 || !params) fail(EVCM_ERR_CONFIG, "predictor: empty depth grid");
  if (factor < 1) fail(EVCM_ERR_CONFIG, "upsample: factor must be at least 1");
  if ((int64_t)pw * factor > 65535 || (int64_t)ph * factor > 65535)
    fail(EVCM_ERR_DIMENSION, "predictor: decoded size too large");
}
}  // namespace

extern "C" {

int evcm_cuda_chain_batch2(evcm_cuda_engine* e, const evcm_chain_batch* bt, int in_mem, int out_mem,
                           evcm_chain_out* out) {
  return guarded([&] { chain_impl(e, bt, in_mem, out_mem, out, nullptr); });
}

int evcm_cuda_chain_batch(evcm_cuda_engine* e, const evcm_chain_batch* bt, int mem, evcm_chain_out* out) {
  return evcm_cuda_chain_batch2(e, bt, mem, mem, out);
}

int evcm_cuda_chain_batch_async(evcm_cuda_engine* e, const evcm_chain_batch* bt, int in_mem,
                                int out_mem, evcm_chain_out* out, int slot) {
  return guarded([&] {
    if (!e) fail(EVCM_ERR_CONFIG, "null engine");
    if (slot < 0 || slot >= evcm_cuda_engine::kSlots) fail(EVCM_ERR_CONFIG, "chain: slot out of range");
    if (e->pending[slot].active) fail(EVCM_ERR_STATE, "chain: slot still pending (call evcm_cuda_chain_wait)");
    struct Restore {
      evcm_cuda_engine* e;
      ~Restore() { e->slot = 0; }
    } restore{e};
    e->slot = slot;
    chain_impl(e, bt, in_mem, out_mem, out, nullptr, true);
  });
}

int evcm_cuda_chain_wait(evcm_cuda_engine* e, int slot) {
  return guarded([&] {
    if (!e) fail(EVCM_ERR_CONFIG, "null engine");
    if (slot < 0 || slot >= evcm_cuda_engine::kSlots) fail(EVCM_ERR_CONFIG, "chain: slot out of range");
    auto& q = e->pending[slot];
    if (!q.active) return;  // the call already completed synchronously
    q.active = false;
    set_device(e);
    ck(cudaEventSynchronize(q.done), "chain wait");
    struct Restore {
      evcm_cuda_engine* e;
      ~Restore() { e->slot = 0; }
    } restore{e};
    e->slot = slot;
    if (q.pose && e->pinned<unsigned long long>(e->slot_name("stage_err_h"), q.nw + 1)[q.nw])
      fail(EVCM_ERR_CONFIG, "pose step: rotation angle must stay below pi and components finite");
    e->stage_nw = q.nw;
    check_stage_errors(e);
    ck(cudaGetLastError(), "chain wait");
  });
}

int evcm_cuda_validate_slice(evcm_cuda_engine* e, const evcm_slice* sl, int check_window, int mem,
                             uint64_t* first_bad) {
  return guarded([&] {
    if (!e || !sl || (sl->n_events && !sl->events)) fail(EVCM_ERR_CONFIG, "null argument");
    const std::string what = check_window ? "event slice: " : "EVT1: ";
    if (sl->width == 0 || sl->height == 0) fail(EVCM_ERR_DIMENSION, what + "zero sensor dimension");
    if (check_window && sl->t_end_us < sl->t_start_us)
      fail(EVCM_ERR_TIME_RANGE, "event slice: t_end precedes t_start");
    set_device(e);
    reset_launch_count();
    const size_t n = sl->n_events;
    if (n == 0) {
      e->last_launches = 0;
      return;
    }
    const evcm_event* d = to_device(e, "ingest_events", sl->events, n, mem);
    unsigned long long* first = e->get<unsigned long long>("ingest_first", 1);
    ck(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), e->stream), "memset");
    launch_validate_events(e->stream, d, n, sl->width, sl->height, check_window, sl->t_start_us,
                           sl->t_end_us, first);
    unsigned long long* h = e->pinned<unsigned long long>("ingest_first_h", 1);
    ck(cudaMemcpyAsync(h, first, sizeof(unsigned long long), cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaStreamSynchronize(e->stream), "validate_slice");
    e->last_launches = launch_count();
    if (*h == ~0ull) return;
    const uint64_t k = *h >> 4;
    const int code = (int)(*h & 0xf);
    if (first_bad) *first_bad = k;
    const std::string rec = what + "record " + std::to_string(k);
    if (code == EVCM_ERR_COORDINATE) fail(code, rec + " coordinate out of range");
    if (code == EVCM_ERR_POLARITY) fail(code, rec + " bad polarity");
    if (code == EVCM_ERR_UNSORTED) fail(code, rec + " breaks timestamp order");
    fail(code, rec + " timestamp outside [t_start, t_end)");
  });
}

int evcm_cuda_window_offsets(evcm_cuda_engine* e, const evcm_event* events, size_t n, uint64_t t0,
                             uint64_t window_us, int n_windows, int mem, uint64_t* offsets) {
  return guarded([&] {
    if (!e || !offsets || (n && !events)) fail(EVCM_ERR_CONFIG, "null argument");
    if (n_windows < 1 || window_us == 0) fail(EVCM_ERR_CONFIG, "windows: need n_windows >= 1 and a nonzero length");
    set_device(e);
    reset_launch_count();
    const evcm_event* d = to_device(e, "ingest_events", events, n, mem);
    uint64_t* od = e->get<uint64_t>("ingest_offsets", (size_t)n_windows + 1);
    launch_window_offsets(e->stream, d, n, t0, window_us, n_windows, od);
    ck(cudaMemcpyAsync(offsets, od, ((size_t)n_windows + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                       e->stream), "D2H offsets");
    ck(cudaStreamSynchronize(e->stream), "window_offsets");
    e->last_launches = launch_count();
  });
}

int evcm_cuda_decode(evcm_cuda_engine* e, int pw, int ph, int factor, const double* params, int mem,
                     double* depth_out) {
  return guarded([&] {
    if (!e || !depth_out) fail(EVCM_ERR_CONFIG, "null argument");
    check_grid(pw, ph, factor, params);
    set_device(e);
    reset_launch_count();
    const double* pd = to_device(e, "pred_params", params, (size_t)pw * ph, mem);
    const size_t n = (size_t)pw * factor * ph * factor;
    double* dd = mem == EVCM_MEM_DEVICE ? depth_out : e->get<double>("pred_depth", n);
    launch_decode(e->stream, pd, pw, ph, factor, dd);
    if (dd != depth_out) from_device(e, depth_out, dd, n * sizeof(double), mem);
    sync_and_check(e, "decode");
    e->last_launches = launch_count();
  });
}

int evcm_cuda_decode_backward(evcm_cuda_engine* e, int pw, int ph, int factor, const double* params,
                              const double* d_depth, int mem, double* d_params_out) {
  return guarded([&] {
    if (!e || !d_depth || !d_params_out) fail(EVCM_ERR_CONFIG, "null argument");
    check_grid(pw, ph, factor, params);
    set_device(e);
    reset_launch_count();
    const size_t n = (size_t)pw * factor * ph * factor;
    const double* pd = to_device(e, "pred_params", params, (size_t)pw * ph, mem);
    const double* gd = to_device(e, "pred_d_depth", d_depth, n, mem);
    double* out = mem == EVCM_MEM_DEVICE ? d_params_out : e->get<double>("pred_d_params", (size_t)pw * ph);
    launch_decode_adjoint(e->stream, pd, gd, pw, ph, factor, out);
    if (out != d_params_out) from_device(e, d_params_out, out, (size_t)pw * ph * sizeof(double), mem);
    sync_and_check(e, "decode_backward");
    e->last_launches = launch_count();
  });
}

int evcm_cuda_adam_step(evcm_cuda_engine* e, size_t n, double* params, const double* grads, double* m,
                        double* v, int t, double lr, double beta1, double beta2, double eps, int mem) {
  return guarded([&] {
    if (!e || (n && (!params || !grads || !m || !v))) fail(EVCM_ERR_CONFIG, "null argument");
    if (t < 1) fail(EVCM_ERR_CONFIG, "adam: step count must be >= 1");
    set_device(e);
    reset_launch_count();
    const double c1 = 1.0 - std::pow(beta1, t), c2 = 1.0 - std::pow(beta2, t);  // optimize.hpp:121-122
    if (mem == EVCM_MEM_DEVICE) {
      launch_adam(e->stream, params, grads, m, v, n, lr, beta1, beta2, eps, c1, c2);
    } else {
      double* pd = e->get<double>("adam_p", n);
      double* gd = e->get<double>("adam_g", n);
      double* md = e->get<double>("adam_m", n);
      double* vd = e->get<double>("adam_v", n);
      const size_t b = n * sizeof(double);
      ck(cudaMemcpyAsync(pd, params, b, cudaMemcpyHostToDevice, e->stream), "H2D");
      ck(cudaMemcpyAsync(gd, grads, b, cudaMemcpyHostToDevice, e->stream), "H2D");
      ck(cudaMemcpyAsync(md, m, b, cudaMemcpyHostToDevice, e->stream), "H2D");
      ck(cudaMemcpyAsync(vd, v, b, cudaMemcpyHostToDevice, e->stream), "H2D");
      launch_adam(e->stream, pd, gd, md, vd, n, lr, beta1, beta2, eps, c1, c2);
      ck(cudaMemcpyAsync(params, pd, b, cudaMemcpyDeviceToHost, e->stream), "D2H");
      ck(cudaMemcpyAsync(m, md, b, cudaMemcpyDeviceToHost, e->stream), "D2H");
      ck(cudaMemcpyAsync(v, vd, b, cudaMemcpyDeviceToHost, e->stream), "D2H");
    }
    sync_and_check(e, "adam_step");
    e->last_launches = launch_count();
  });
}

int evcm_cuda_predictor_loss_and_gradients_geo(evcm_cuda_engine* e, int pw, int ph, int factor,
                                               const double* params, int n_bins,
                                               const double* poses, const double K[4],
                                               const evcm_slice* slice, double lambda_geo, int mem,
                                               double* losses, double* d_params, double* d_poses) {
  return guarded([&] {
    if (!e || !slice || !K || !poses) fail(EVCM_ERR_CONFIG, "null argument");
    check_grid(pw, ph, factor, params);
    if (n_bins < 1) fail(EVCM_ERR_CONFIG, "predictor: need one pose per bin");
    if ((int)slice->width != pw * factor || (int)slice->height != ph * factor)
      fail(EVCM_ERR_DIMENSION, "predictor: decoded depth does not match the slice sensor");
    set_device(e);
    const int W = pw * factor, H = ph * factor;
    const size_t HW = (size_t)W * H;
    // decode on the device (predictor.hpp:126-131); the chain resets the launch count
    const double* pd = to_device(e, "pred_params", params, (size_t)pw * ph, mem);
    double* depth = e->get<double>("pred_depth", HW);
    launch_decode(e->stream, pd, pw, ph, factor, depth);
    // the fused chain: flows -> Engine::forward -> Engine::backward -> flows backward
    evcm_chain_batch bt{};
    bt.n_windows = 1;
    bt.width = W;
    bt.height = H;
    bt.n_bins = n_bins;
    bt.t_start_us = slice->t_start_us;
    bt.t_end_us = slice->t_end_us;
    for (int i = 0; i < 4; ++i) bt.K[i] = K[i];
    bt.events = slice->events;
    const uint64_t offs[2] = {0, (uint64_t)slice->n_events};
    bt.ev_offsets = offs;
    bt.poses = poses;
    double* ld = e->get<double>("pred_loss", 1);
    double* dd = e->get<double>("pred_dd", HW);
    double* dp = mem == EVCM_MEM_DEVICE ? d_poses : e->get<double>("pred_dp", (size_t)n_bins * 6);
    evcm_chain_out co{};
    co.loss = ld;
    co.d_depth = dd;
    co.d_poses = dp;
    chain_impl(e, &bt, mem, EVCM_MEM_DEVICE, &co, depth);
    int launches = launch_count() + 1;  // + the decode before the chain's reset
    double* lo = e->get<double>("pred_losses", 3);
    if (lambda_geo > 0.0) {
      // optimize.hpp:219-236: L_geo per bin on (depth, depth), upstream lambda / B;
      // both halves of the depth gradient and the pose gradient add onto the
      // CMax gradients before the decode adjoint (predictor.hpp:153-171)
      GeoArgs g{};
      g.W = W;
      g.H = H;
      g.n_poses = n_bins;
      g.want_grad = 1;
      g.d0 = g.d1 = depth;
      g.tab = e->get<double>("pose_tab", (size_t)n_bins * kPoseTab);  // built by the chain
      for (int i = 0; i < 4; ++i) g.K[i] = K[i];
      g.upstream = lambda_geo / (double)n_bins;
      geo_workspace(e, g);
      g.d_poses = dp;
      g.add_poses = dp;
      g.d_depth_sum = dd;
      g.add_depth = dd;
      g.l_cm = ld;
      g.lambda = lambda_geo;
      g.losses = lo;
      reset_launch_count();
      launch_geo(e->stream, g);
      launches += launch_count();
    } else {
      launch_geo_losses_off(e->stream, ld, lambda_geo, lo);
      ++launches;
    }
    // accumulate_gradients, depth half (predictor.hpp:156-162)
    double* dpar = mem == EVCM_MEM_DEVICE ? d_params : e->get<double>("pred_d_params", (size_t)pw * ph);
    launch_decode_adjoint(e->stream, pd, dd, pw, ph, factor, dpar);
    ++launches;
    if (losses) from_device(e, losses, lo, 3 * sizeof(double), mem);
    if (d_params && dpar != d_params) from_device(e, d_params, dpar, (size_t)pw * ph * sizeof(double), mem);
    if (d_poses && dp != d_poses) from_device(e, d_poses, dp, (size_t)n_bins * 6 * sizeof(double), mem);
    sync_and_check(e, "predictor_loss_and_gradients");
    e->last_launches = launches;
  });
}

int evcm_cuda_predictor_loss_and_gradients(evcm_cuda_engine* e, int pw, int ph, int factor,
                                           const double* params, int n_bins, const double* poses,
                                           const double K[4], const evcm_slice* slice, int mem,
                                           double* loss, double* d_params, double* d_poses) {
  double l3[3];
  double* dl = nullptr;
  if (loss && mem == EVCM_MEM_DEVICE) {
    // device losses land in a scratch triple; the caller's scalar receives l_cm
    const int rc = guarded([&] { dl = e ? e->get<double>("pred_losses_user", 3) : nullptr; });
    if (rc) return rc;
  }
  const int rc = evcm_cuda_predictor_loss_and_gradients_geo(e, pw, ph, factor, params, n_bins, poses,
                                                           K, slice, 0.0, mem,
                                                           loss ? (dl ? dl : l3) : nullptr,
                                                           d_params, d_poses);
  if (rc || !loss) return rc;
  if (dl)
    return guarded([&] {
      ck(cudaMemcpyAsync(loss, dl, sizeof(double), cudaMemcpyDeviceToDevice, e->stream), "loss");
      ck(cudaStreamSynchronize(e->stream), "loss");
    });
  *loss = l3[0];
  return rc;
}

int evcm_cuda_geometry_consistency_loss(evcm_cuda_engine* e, int W, int H, const double* d0,
                                        const uint8_t* mask0, const double* d1,
                                        const uint8_t* mask1, int n_poses, const double* poses,
                                        const double K[4], double upstream, int want_grad, int mem,
                                        evcm_geo_out* out) {
  return guarded([&] {
    if (!e || !out || !K || !poses || !d0 || !d1) fail(EVCM_ERR_CONFIG, "null argument");
    if (W <= 0 || H <= 0) fail(EVCM_ERR_DIMENSION, "depth consistency: depth maps must share a shape");
    if (n_poses < 1) fail(EVCM_ERR_CONFIG, "depth consistency: need at least one pose");
    set_device(e);
    reset_launch_count();
    const size_t HW = (size_t)W * H, nP = (size_t)n_poses;
    std::vector<double> ph(6 * nP);
    if (mem == EVCM_MEM_DEVICE)
      ck(cudaMemcpy(ph.data(), poses, ph.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H poses");
    else
      std::memcpy(ph.data(), poses, ph.size() * sizeof(double));
    std::vector<uint64_t> unit_edges(nP + 1);  // inv_dt is not used by L_geo
    for (size_t i = 0; i <= nP; ++i) unit_edges[i] = i;
    GeoArgs g{};
    g.W = W;
    g.H = H;
    g.n_poses = n_poses;
    g.want_grad = want_grad ? 1 : 0;
    // geometry_consistency_loss does not validate the pose (geometry.hpp:423)
    g.tab = upload_pose_table(e, ph.data(), 1, n_poses, unit_edges.data(), false);
    g.d0 = to_device(e, "geo_d0", d0, HW, mem);
    g.m0 = mask0 ? to_device(e, "geo_m0", mask0, HW, mem) : nullptr;
    g.d1 = d1 == d0 ? g.d0 : to_device(e, "geo_d1", d1, HW, mem);
    g.m1 = !mask1 ? nullptr : mask1 == mask0 ? g.m0 : to_device(e, "geo_m1", mask1, HW, mem);
    for (int i = 0; i < 4; ++i) g.K[i] = K[i];
    g.upstream = upstream;
    geo_workspace(e, g);
    const bool dev = mem == EVCM_MEM_DEVICE;
    auto outp = [&](auto* user, const char* name, size_t n) {
      using T = std::remove_pointer_t<decltype(user)>;
      return (T*)(user == nullptr ? nullptr : dev ? user : e->get<T>(name, n));
    };
    g.value = outp(out->value, "geo_value", nP);
    if (!g.value) g.value = e->get<double>("geo_value", nP);
    g.n_valid = (long long*)outp((int64_t*)out->n_valid, "geo_nvalid", nP);
    if (!g.n_valid) g.n_valid = (long long*)e->get<int64_t>("geo_nvalid", nP);
    g.projected = outp(out->projected, "geo_proj", nP * HW);
    g.interpolated = outp(out->interpolated, "geo_interp", nP * HW);
    g.valid = outp(out->valid, "geo_valid", nP * HW);
    if (want_grad) {
      g.d_d0 = outp(out->d_d0, "geo_dd0", nP * HW);
      g.d_d1 = outp(out->d_d1, "geo_dd1", nP * HW);
      g.d_poses = outp(out->d_poses, "geo_dposes", nP * 6);
      g.d_depth_sum = outp(out->d_depth_sum, "geo_dsum", HW);
    }
    launch_geo(e->stream, g);
    if (!dev) {
      auto back = [&](void* user, const void* d, size_t bytes) {
        if (user) from_device(e, user, d, bytes, mem);
      };
      back(out->value, g.value, nP * sizeof(double));
      back(out->n_valid, g.n_valid, nP * sizeof(int64_t));
      back(out->projected, g.projected, nP * HW * sizeof(double));
      back(out->interpolated, g.interpolated, nP * HW * sizeof(double));
      back(out->valid, g.valid, nP * HW);
      if (want_grad) {
        back(out->d_d0, g.d_d0, nP * HW * sizeof(double));
        back(out->d_d1, g.d_d1, nP * HW * sizeof(double));
        back(out->d_poses, g.d_poses, nP * 6 * sizeof(double));
        back(out->d_depth_sum, g.d_depth_sum, HW * sizeof(double));
      }
    }
    e->stage_nw = 0;
    sync_and_check(e, "geometry_consistency_loss");
    e->last_launches = launch_count();
  });
}

}  // extern "C"
