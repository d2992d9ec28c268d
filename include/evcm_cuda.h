/*
 * evcm_cuda.h — C-ABI of the B200 (sm_100a) CMax loss path.
 *
 * This is the drop-in boundary a maintainer of the reference (evcm, a
 * header-only C++20 library) binds to add a `cuda` execution backend next to
 * naive/padded/parallel (engine.hpp:37). Plain C: opaque handle, plain
 * pointers and sizes, int status codes, no CUDA or torch types.
 *
 * Reference interfaces replaced (paths under /root/reference/proj/include/evcm):
 *   evcm_cuda_create / destroy          Engine(EngineOptions)           engine.hpp:136-141, 54-61
 *   evcm_cuda_forward                   Engine::forward                 engine.hpp:145-183
 *   evcm_cuda_forward_products          ForwardResult members           engine.hpp:99-105
 *                                       (IweStack, Trajectories)        warp.hpp:167-220
 *   evcm_cuda_backward                  Engine::backward                engine.hpp:185-205
 *   evcm_cuda_loss_and_grad             Engine::loss_and_grad           engine.hpp:208-213
 *   evcm_cuda_depth_pose_to_flows       depth_pose_to_flows             geometry.hpp:229-264
 *   evcm_cuda_depth_pose_to_flows_backward
 *                                       depth_pose_to_flows_backward    geometry.hpp:279-325
 *   evcm_cuda_chain_batch               predictor_loss_and_gradients's  optimize.hpp:205-241
 *                                       flows→forward→backward→flows-backward composition, over a
 *                                       batch of windows (the reference runs them one at a time,
 *                                       optimize.hpp:327-371)
 *   evcm_cuda_last_error / error_name   evcm::Error taxonomy            types.hpp:18-76
 *
 * Memory: every call states where its array arguments live (EVCM_MEM_HOST or
 * EVCM_MEM_DEVICE, device = the engine's CUDA device). Host inputs are staged
 * through pinned buffers owned by the engine. Calls are synchronous with
 * respect to the host unless documented otherwise.
 *
 * Layouts are the reference's own, flattened row-major (idx = y*W + x,
 * Image<T>::idx, types.hpp:199-202):
 *   events   evcm_event[n]          == evcm::Event, 16 B, time-sorted (types.hpp:106-113)
 *   flows    f64 [B][2][H][W]       == FlowSequence.fields[b].{u,v}   (types.hpp:228-253)
 *   stack    f64 [B+1][2][H][W]     == IweStack.count / tsum [ref][pol] (warp.hpp:167-172)
 *   grad     f64 [B][2][H][W]       == GradientBuffer.gu[b] / gv[b]  (warp.hpp:223-224)
 *   pos      f64 [n][B+1][2]        == Trajectories.pos              (warp.hpp:196-199)
 *   poses    f64 [B][6]             == PoseStep {omega.xyz, trans.xyz} (types.hpp:356-358)
 *   K        f64 [4]                == CameraIntrinsics {fx, fy, cx, cy} (types.hpp:164-168)
 */
#ifndef EVCM_CUDA_H
#define EVCM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define EVCM_API __attribute__((visibility("default")))
#else
#define EVCM_API
#endif

#define EVCM_CUDA_ABI_VERSION 2
#define EVCM_CUDA_MAX_BINS 32

/* Status codes; the C++ adapter maps them onto the evcm::Error subclasses. */
enum evcm_status {
  EVCM_OK = 0,
  EVCM_ERR_CONFIG = 1,      /* ConfigError */
  EVCM_ERR_DIMENSION = 2,   /* DimensionMismatchError */
  EVCM_ERR_COORDINATE = 3,  /* CoordinateRangeError */
  EVCM_ERR_POLARITY = 4,    /* InvalidPolarityError */
  EVCM_ERR_UNSORTED = 5,    /* UnsortedEventsError */
  EVCM_ERR_TIME_RANGE = 6,  /* TimeRangeError */
  EVCM_ERR_EMPTY = 7,       /* EmptySliceError */
  EVCM_ERR_CUDA = 20,       /* device / driver failure (evcm::Error) */
  EVCM_ERR_STATE = 21       /* backward without a matching forward (ConfigError analog,
                               engine.hpp:191-193) */
};

enum evcm_mem { EVCM_MEM_HOST = 0, EVCM_MEM_DEVICE = 1 };

/* Byte-identical to evcm::Event. */
typedef struct {
  uint64_t t_us;
  uint16_t x;
  uint16_t y;
  int8_t p;
  uint8_t pad_[3];
} evcm_event;

/* EngineOptions (engine.hpp:54-61) for the cuda backend. Fields the cuda
 * backend does not need (n_workers, batch_size, padding_fraction) have no
 * counterpart; `deterministic` keeps its meaning and its default (1:
 * run-to-run bit-stable results, engine.hpp:60). */
typedef struct {
  int device;          /* CUDA device ordinal */
  int deterministic;   /* 1 (default, as engine.hpp:60): the owner-computes pipeline, exact
                          fixed-point accumulation, bit-stable run to run; 0 allows algo 1 */
  int stack_f64;       /* 1 (default, parity): fp64 IWE stack + loss coefficients;
                          0: fp32 ("fast": loss/IWE within 1e-6, gradients NOT within
                          1e-5 on sparse windows — see DESIGN.md "Numerics") */
  int grad_f64;        /* algo 1 only: fp64 flow-gradient accumulators (default 0: fp32,
                          which keeps gradients within ~1e-7 of the reference). With
                          stack_f64 this is the path that tracks the reference through
                          long optimisation loops (run_window: ~1e-11 after 12 updates;
                          DESIGN.md §3) */
  void* stream;        /* cudaStream_t to run on; NULL = engine-owned stream */
  int algo;            /* 0: owner-computes tiles (no global atomics; the product path);
                          1: per-event global atomics, an independent cross-check kept
                          for tests (needs deterministic = 0; honours stack_f64 /
                          grad_f64); 2 (default): auto -- the owner pipeline when
                          deterministic, else owner from >= 1 event per pixel per window
                          and >= 2.5e5 events per call (measured crossover) */
} evcm_cuda_options;

/* EventSlice (types.hpp:121-126). */
typedef struct {
  uint16_t width;
  uint16_t height;
  uint64_t t_start_us;
  uint64_t t_end_us; /* exclusive */
  const evcm_event* events;
  size_t n_events;
} evcm_slice;

/* FlowSequence (types.hpp:251-253): B+1 edges and B fields of width x height
 * (FlowSequence::width()/height(); a size that differs from the slice's sensor
 * raises DimensionMismatchError, engine.hpp:218-219). */
typedef struct {
  int n_bins;
  const uint64_t* edges_us; /* host pointer, B+1 entries */
  const double* uv;         /* [B][2][height][width], contiguous f64 */
  int width, height;
} evcm_flows;

/* LossResult (warp.hpp:292-295) + the id of the forward that produced it:
 * evcm_cuda_backward_of checks it, so a backward never pairs with the device
 * state of a different (later) forward. */
typedef struct {
  double value;
  int no_survivors;
  uint64_t forward_id;
} evcm_loss;

typedef struct evcm_cuda_engine evcm_cuda_engine;

/* ---- lifecycle / errors -------------------------------------------------- */
EVCM_API void evcm_cuda_default_options(evcm_cuda_options* opts);
EVCM_API int evcm_cuda_create(const evcm_cuda_options* opts, evcm_cuda_engine** out);
EVCM_API void evcm_cuda_destroy(evcm_cuda_engine* e);
/* Message of the last failing call on this thread ("" if none). */
EVCM_API const char* evcm_cuda_last_error(void);
/* "ConfigError", "DimensionMismatchError", ... for a status code. */
EVCM_API const char* evcm_cuda_error_name(int status);
EVCM_API int evcm_cuda_abi_version(void);

/* ---- Engine ---------------------------------------------------------------- */

/* Engine::forward. Validates the window exactly like Engine::validate_window
 * (engine.hpp:215-222) and keeps the IWE stack on the device for a following
 * backward. `mem` applies to slice->events and flows->uv. */
EVCM_API int evcm_cuda_forward(evcm_cuda_engine* e, const evcm_slice* slice, const evcm_flows* flows,
                      int mem, evcm_loss* loss);

/* Copies ForwardResult members of the last forward to HOST buffers; any
 * pointer may be NULL. count/tsum [B+1][2][H][W] f64; n_active [B+1];
 * alive u8 [n]; bin i32 [n]; pos f64 [n][B+1][2]; n_alive scalar. */
EVCM_API int evcm_cuda_forward_products(evcm_cuda_engine* e, double* count, double* tsum,
                               int64_t* n_active, uint8_t* alive, int32_t* bin, double* pos,
                               size_t* n_alive);

/* The tile sort of the last forward (owner pipeline; the reference's
 * determinism analog, engine.hpp:584-598): keys[n] the 8x8 sort-tile key of
 * every event (0xffffffff: masked), perm[n_sorted] the window-local index of
 * the event at each sorted slot, sorted_keys[n_sorted] the keys in sorted order;
 * HOST arrays, any may be NULL. The sort is stable: perm equals a stable argsort
 * of the valid keys. */
EVCM_API int evcm_cuda_sort_products(evcm_cuda_engine* e, uint32_t* keys, uint32_t* perm,
                                     uint32_t* sorted_keys, size_t* n_sorted);

/* Engine::backward for the window of the last forward (same slice). The
 * trajectories come from that forward (ForwardResult.traj, engine.hpp:196,
 * 564-567) and the flow Jacobians from `flows` (engine.hpp:185-205).
 * grad: [B][2][H][W] f64, in `mem` space. */
EVCM_API int evcm_cuda_backward(evcm_cuda_engine* e, const evcm_slice* slice, const evcm_flows* flows,
                       int mem, double* grad);
/* Same, checked against the forward it belongs to: fails with EVCM_ERR_STATE
 * unless forward_id is the id the engine's last forward returned. */
EVCM_API int evcm_cuda_backward_of(evcm_cuda_engine* e, const evcm_slice* slice,
                                   const evcm_flows* flows, uint64_t forward_id, int mem,
                                   double* grad);

/* Engine::loss_and_grad. */
EVCM_API int evcm_cuda_loss_and_grad(evcm_cuda_engine* e, const evcm_slice* slice,
                            const evcm_flows* flows, int mem, evcm_loss* loss, double* grad);

/* ---- motion field ------------------------------------------------------------- */

/* depth_pose_to_flows: depth f64 [H][W], mask u8 [H][W] or NULL (all valid),
 * poses [B][6], K [4]. Writes flows [B][2][H][W], valid u8 [B][H][W] (may be
 * NULL) and, if edges_out != NULL (host), the B+1 FlowSequence::zeros edges. */
EVCM_API int evcm_cuda_depth_pose_to_flows(evcm_cuda_engine* e, int width, int height,
                                  const double* depth, const uint8_t* mask, int n_bins,
                                  const double* poses, const double* K, uint64_t t_start_us,
                                  uint64_t t_end_us, int mem, double* flows, uint8_t* valid,
                                  uint64_t* edges_out);

/* depth_pose_to_flows_backward: grad [B][2][H][W] -> d_depth [H][W], d_poses [B][6]. */
EVCM_API int evcm_cuda_depth_pose_to_flows_backward(evcm_cuda_engine* e, int width, int height,
                                           const double* depth, const uint8_t* mask, int n_bins,
                                           const double* poses, const double* K,
                                           const uint64_t* edges_us, const double* grad,
                                           int mem, double* d_depth, double* d_poses);

/* ---- batched chain (the hot path, one call per batch of windows) ---------------- */

/* n_windows windows sharing sensor size, intrinsics and time window
 * [t_start_us, t_end_us) split into n_bins FlowSequence::zeros bins. For each
 * window w: depth_pose_to_flows(depth[w], poses[w]) -> Engine::forward ->
 * Engine::backward -> depth_pose_to_flows_backward, i.e. the
 * predictor_loss_and_gradients composition without decode / L_geo.
 *   events   concatenated, window w = events[ev_offsets[w] .. ev_offsets[w+1])
 *   depth    f64 [n_windows][H][W] (all pixels valid, as DecodedPredictor)
 *   poses    f64 [n_windows][B][6]
 * Outputs (in `mem` space): loss f64 [n_windows], no_survivors i32 [n_windows]
 * (may be NULL), d_depth f64 [n_windows][H][W], d_poses f64 [n_windows][B][6].
 * ev_offsets is always a HOST array of n_windows+1 entries. Window w's clock
 * starts at t_start_us + w * window_stride_us (see the field). */
typedef struct {
  int n_windows;
  int width, height, n_bins;
  uint64_t t_start_us, t_end_us;
  double K[4];
  const evcm_event* events;
  const uint64_t* ev_offsets;
  const double* depth;
  const double* poses;
  /* window w's clock is shifted by w * window_stride_us: its events lie in
   * [t_start_us + w*stride, t_end_us + w*stride). 0 (zero-initialised) = all
   * windows on one clock; window_us = consecutive windows of one event stream
   * (evcm_cuda_window_offsets). */
  uint64_t window_stride_us;
} evcm_chain_batch;

typedef struct {
  double* loss;
  int32_t* no_survivors;
  double* d_depth;
  double* d_poses;
  /* optional (may be NULL): the batch's data-parallel payload [sum_w loss,
   * sum_w d_depth (H*W), sum_w d_poses (B*6)], summed over the windows in window
   * order (deterministic) inside the chain -- the buffer a multi-GPU caller
   * all-reduces */
  double* sums;
} evcm_chain_out;

EVCM_API int evcm_cuda_chain_batch(evcm_cuda_engine* e, const evcm_chain_batch* batch, int mem,
                          evcm_chain_out* out);
/* Same, with separate memory spaces for the inputs and the outputs (e.g. host
 * inputs staged in, device outputs kept for a following NCCL all-reduce). */
EVCM_API int evcm_cuda_chain_batch2(evcm_cuda_engine* e, const evcm_chain_batch* batch, int in_mem,
                                    int out_mem, evcm_chain_out* out);

/* Asynchronous form for pipelined callers: enqueues the batch on the engine's
 * stream and returns; when the call replays a captured graph (device inputs and
 * outputs, third and later calls of a signature) it does not wait, and the
 * batch's validation result is delivered by evcm_cuda_chain_wait(slot). Slots
 * 0..3 carry separate error words, so batch i+1 can be queued before batch i
 * is waited for. Calls that run eagerly complete (and report) synchronously. */
EVCM_API int evcm_cuda_chain_batch_async(evcm_cuda_engine* e, const evcm_chain_batch* batch,
                                         int in_mem, int out_mem, evcm_chain_out* out, int slot);
/* Waits for the batch queued on `slot` and raises its validation errors (the
 * same codes a synchronous call returns). No-op for a slot with nothing pending. */
EVCM_API int evcm_cuda_chain_wait(evcm_cuda_engine* e, int slot);

/* ---- predictor decode chain ------------------------------- */

/* decode (predictor.hpp:126-131): depth[ph*f][pw*f] =
 * upsample_bilinear(softplus(params[ph][pw]), f) (predictor.hpp:25-27, 46-66).
 * Throws ConfigError for f < 1 or an empty grid. */
EVCM_API int evcm_cuda_decode(evcm_cuda_engine* e, int pw, int ph, int factor, const double* params,
                              int mem, double* depth_out);
/* The depth half of accumulate_gradients (predictor.hpp:156-162):
 * d_params = upsample_bilinear_adjoint(d_depth) * softplus_grad(params). */
EVCM_API int evcm_cuda_decode_backward(evcm_cuda_engine* e, int pw, int ph, int factor,
                                       const double* params, const double* d_depth, int mem,
                                       double* d_params_out);
/* Adam::step (optimize.hpp:115-134) over n slots: the caller keeps the step
 * counter t (already incremented, t >= 1) and the moment buffers m, v. */
EVCM_API int evcm_cuda_adam_step(evcm_cuda_engine* e, size_t n, double* params, const double* grads,
                                 double* m, double* v, int t, double lr, double beta1, double beta2,
                                 double eps, int mem);
/* predictor_loss_and_gradients (optimize.hpp:205-241) with lambda_geo = 0 for
 * one window: decode -> depth_pose_to_flows -> Engine::forward -> Engine::backward
 * -> accumulate_gradients. params f64 [ph][pw] (slice is ph*f x pw*f), poses f64
 * [n_bins][6]; outputs: loss (l_cm), d_params [ph][pw], d_poses [n_bins][6]. */
EVCM_API int evcm_cuda_predictor_loss_and_gradients(evcm_cuda_engine* e, int pw, int ph, int factor,
                                                    const double* params, int n_bins,
                                                    const double* poses, const double K[4],
                                                    const evcm_slice* slice, int mem, double* loss,
                                                    double* d_params, double* d_poses);

/* predictor_loss_and_gradients (optimize.hpp:205-241) with the depth-consistency
 * term: losses[3] = {l_cm, l_geo, total = l_cm + lambda_geo * l_geo}; with
 * lambda_geo > 0, L_geo runs per bin on (depth, depth) with upstream
 * lambda_geo / B and its gradients add onto the CMax ones (optimize.hpp:219-236,
 * predictor.hpp:153-171); lambda_geo <= 0 switches the term off, as in the
 * reference (total = l_cm + lambda_geo * 0). */
EVCM_API int evcm_cuda_predictor_loss_and_gradients_geo(
    evcm_cuda_engine* e, int pw, int ph, int factor, const double* params, int n_bins,
    const double* poses, const double K[4], const evcm_slice* slice, double lambda_geo, int mem,
    double* losses, double* d_params, double* d_poses);

/* ---- geometry-consistency loss L_geo ---------------------- */

/* Outputs of evcm_cuda_geometry_consistency_loss, all in `mem` space; any may be
 * NULL. Per-pose arrays are [n_poses][...]; d_poses rows are {omega xyz, trans xyz}. */
typedef struct {
  double* value;         /* [n_poses] GeoLossTerms::value (0 when the valid set is empty) */
  int64_t* n_valid;      /* [n_poses] GeoLossTerms::n_valid */
  double* projected;     /* [n_poses][H][W] GeoLossTerms::projected */
  double* interpolated;  /* [n_poses][H][W] GeoLossTerms::interpolated */
  uint8_t* valid;        /* [n_poses][H][W] GeoLossTerms::valid */
  double* d_d0;          /* [n_poses][H][W] GeoLossGrad::d_d0 (want_grad) */
  double* d_d1;          /* [n_poses][H][W] GeoLossGrad::d_d1 (want_grad) */
  double* d_poses;       /* [n_poses][6]    GeoLossGrad::d_omega, d_trans (want_grad) */
  double* d_depth_sum;   /* [H][W] sum_i (d_d0_i + d_d1_i), the predictor's extra depth
                            term (optimize.hpp:229-230) (want_grad) */
} evcm_geo_out;

/* geometry_consistency_loss (want_grad = 0, geometry.hpp:416-453) or
 * geometry_consistency_loss_backward (want_grad = 1, :458-534, scaled by
 * `upstream`) of depth maps d0 -> d1 (masks may be NULL = all valid) for each of
 * n_poses poses {omega, trans}. Membership (projection, z-min winners, target
 * depth, valid set) is bit-identical to the reference; sums over pixels differ
 * only by rounding order. */
EVCM_API int evcm_cuda_geometry_consistency_loss(evcm_cuda_engine* e, int W, int H, const double* d0,
                                                 const uint8_t* mask0, const double* d1,
                                                 const uint8_t* mask1, int n_poses,
                                                 const double* poses, const double K[4],
                                                 double upstream, int want_grad, int mem,
                                                 evcm_geo_out* out);

/* ---- event ingestion -------------------------------------- */

/* Slice validation on the device. check_window = 1: EventSlice::validate
 * (types.hpp:137-161) -- dimensions, t_end >= t_start, then per record coordinate,
 * polarity, timestamp order, [t_start, t_end). check_window = 0: the record checks
 * of read_events (io.hpp:123-144) on a freshly read EVT1 payload (window ignored).
 * Returns the error of the first violating record (its index in *first_bad when
 * non-null), EVCM_OK otherwise. */
EVCM_API int evcm_cuda_validate_slice(evcm_cuda_engine* e, const evcm_slice* slice,
                                      int check_window, int mem, uint64_t* first_bad);
/* Window boundaries of time-sorted events for the batched chain:
 * offsets[w] = first event with t_us >= t0 + w * window_us, w = 0..n_windows
 * (offsets is a HOST array of n_windows + 1 entries). */
EVCM_API int evcm_cuda_window_offsets(evcm_cuda_engine* e, const evcm_event* events, size_t n,
                                      uint64_t t0, uint64_t window_us, int n_windows, int mem,
                                      uint64_t* offsets);

/* ---- instrumentation (PhaseStats analog, engine.hpp:63-66,226-242) --------------- */

/* Per-stage device times (ms, CUDA events on the engine stream) of the last
 * chain / forward / backward call when timing is enabled. Stage order:
 * 0 staging (H2D + validation), 1 motion field, 2 stack memset, 3 warp+splat,
 * 4 loss reduce, 5 grad memset, 6 backward, 7 flows backward (0 if the call
 * did not run the stage). Returns the number of stages written (8). */
EVCM_API int evcm_cuda_set_timing(evcm_cuda_engine* e, int enabled);
EVCM_API int evcm_cuda_stage_times(evcm_cuda_engine* e, double* ms, int max_stages);
/* Pipeline the last call ran: 0 owner-computes, 1 per-event atomics. Stage
 * order of evcm_cuda_stage_times for the atomic pipeline: staging, motion field,
 * stack memset, warp+splat, loss reduce, grad memset, backward, flows backward;
 * for the owner pipeline: staging, motion field, sort, trajectory records +
 * source lists, forward owner, loss finalize, per-event backward, backward
 * owner (+ fused flows backward), pose finalize. */
EVCM_API int evcm_cuda_last_algo(evcm_cuda_engine* e);
/* Number of kernels launched by the last API call (for bench gpu_launches). */
EVCM_API int evcm_cuda_last_launch_count(evcm_cuda_engine* e);
/* Device memory currently held by the engine's workspaces, in bytes (the
 * PhaseStats.peak_bytes analog, memtrack.hpp:72-102). */
EVCM_API size_t evcm_cuda_workspace_bytes(evcm_cuda_engine* e);
/* PhaseStats (engine.hpp:63-66, 226-242) of the last evcm_cuda_forward /
 * evcm_cuda_backward, always recorded (CUDA events on the engine stream):
 * phases 0 warp (staging + sort + trajectories), 1 splat, 2 loss, 3 backward.
 * time_us[4]: device time of the phase; peak_bytes[4]: device workspace held by
 * the engine when the phase ended (the engine's buffers only grow, so this is
 * the phase's peak). Either pointer may be NULL. */
EVCM_API int evcm_cuda_phase_stats(evcm_cuda_engine* e, double* time_us, size_t* peak_bytes);

/* ---- stream ordering ---------------------------------------------------------------- */

/* Orders the engine's stream after the work already enqueued on `stream` (a
 * cudaStream_t of the caller, e.g. the producer of device inputs): the
 * engine's next kernels wait for it. No-op when stream is the engine's own. */
EVCM_API int evcm_cuda_stream_wait(evcm_cuda_engine* e, void* stream);
/* The converse: `stream` waits for the work enqueued on the engine's stream
 * (e.g. a consumer of an asynchronous chain's outputs). */
EVCM_API int evcm_cuda_stream_signal(evcm_cuda_engine* e, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EVCM_CUDA_H */
