"""CPU ORACLE loader — TEST INFRASTRUCTURE ONLY.

ctypes bindings for
  * ``liboracle.so``         — the plain-C fp64 restatement (cmax_oracle.c), and
  * ``_ref/libevcm_ref.so``  — the UNMODIFIED reference compiled from
                               /root/reference by ``make ref`` (ref_capi.cpp).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline legs import this module. The product package never does.

Array conventions match oracle/cmax_oracle.h: flows [B,2,H,W] f64,
stack [B+1,2,H,W] f64, grads [B,2,H,W] f64, poses [B,6] f64, K [4] f64.
Events are numpy structured arrays with the 16-byte evcm::Event layout.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libevcm_ref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")

# evcm::Event (types.hpp:106-113), 16 bytes.
EVENT_DTYPE = np.dtype(
    {"names": ["t_us", "x", "y", "p"], "formats": ["<u8", "<u2", "<u2", "i1"],
     "offsets": [0, 8, 10, 12], "itemsize": 16})

ERR_NAMES = {1: "ConfigError", 2: "DimensionMismatchError", 3: "CoordinateRangeError",
             4: "InvalidPolarityError", 5: "UnsortedEventsError", 6: "TimeRangeError",
             7: "EmptySliceError", 10: "BadMagicError", 11: "TruncatedFileError",
             12: "IoError", 99: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        self.code = code
        self.kind = ERR_NAMES.get(code, "Error")
        super().__init__(f"{self.kind}: {msg}")


def build(ref: bool = True) -> None:
    """Compile liboracle.so (always) and _ref/libevcm_ref.so (when the reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if ref and os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
        lib = os.path.join(HERE, "..", "paper_2412_06359_b200", "_lib", "libevcm_cuda.so")
        if os.path.exists(lib):  # the C++ binding test links the product library
            subprocess.run(["make", "-s", "-C", HERE, "adapter"], check=True)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        vp, i32, sz, u64 = C.c_void_p, C.c_int, C.c_size_t, C.c_uint64
        L.orc_forward.argtypes = [i32, i32, i32, vp, vp, sz, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_backward.argtypes = [i32, i32, i32, vp, vp, sz, vp, vp, vp, vp, vp, vp, i32, vp]
        L.orc_depth_pose_to_flows.argtypes = [i32, i32, vp, vp, i32, vp, vp, u64, u64, vp, vp]
        L.orc_depth_pose_to_flows_backward.argtypes = [i32, i32, vp, vp, i32, vp, vp, vp, vp, vp, vp]
        L.orc_make_edges.argtypes = [u64, u64, i32, vp]
        L.orc_make_edges.restype = None
        L.orc_rodrigues.argtypes = [vp, vp]
        L.orc_rodrigues.restype = None
        L.orc_rodrigues_jacobian.argtypes = [vp, vp]
        L.orc_rodrigues_jacobian.restype = None
        L.orc_validate_window.argtypes = [i32, i32, i32, vp, u64, u64, vp, sz, vp]
        f64 = C.c_double
        L.orc_softplus.argtypes = [f64]
        L.orc_softplus.restype = f64
        L.orc_softplus_grad.argtypes = [f64]
        L.orc_softplus_grad.restype = f64
        L.orc_decode.argtypes = [i32, i32, i32, vp, vp]
        L.orc_decode_backward.argtypes = [i32, i32, i32, vp, vp, vp]
        L.orc_adam_step.argtypes = [sz, vp, vp, vp, vp, i32, f64, f64, f64, f64]
        L.orc_adam_step.restype = None
        L.orc_geo_loss.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, f64, i32, vp, vp, vp, vp, vp,
                                   vp, vp, vp]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build(ref=True)
        L = C.CDLL(REF_SO)
        vp, i32, sz, u64, f64 = C.c_void_p, C.c_int, C.c_size_t, C.c_uint64, C.c_double
        L.ref_last_error.restype = C.c_char_p
        L.ref_hardware_concurrency.restype = C.c_uint
        L.ref_loss_and_grad.argtypes = [i32, i32, i32, vp, vp, sz, vp, i32, i32, i32, i32,
                                        vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.ref_warp_event.argtypes = [i32, i32, i32, vp, vp, f64, f64, f64, f64, vp]
        L.ref_rsat.argtypes = [i32, i32, i32, vp, vp, sz, vp, vp]
        L.ref_depth_pose_to_flows.argtypes = [i32, i32, vp, vp, i32, vp, vp, u64, u64, vp, vp, vp]
        L.ref_depth_pose_to_flows_backward.argtypes = [i32, i32, vp, vp, i32, vp, vp, vp, vp, vp, vp]
        L.ref_random_fd_instance.argtypes = [u64, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp]
        L.ref_bench_window.argtypes = [i32, i32, i32, f64, u64, sz, vp, vp, vp]
        L.ref_generate_scene.argtypes = [i32, i32, i32, vp, vp, f64, u64, vp, vp, vp, vp]
        L.ref_chain_instance.argtypes = [u64, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp]
        L.ref_chain_batch.argtypes = [i32, i32, i32, i32, vp, vp, vp, u64, u64, vp, vp, i32,
                                      vp, vp, vp, vp]
        L.ref_decode.argtypes = [i32, i32, i32, vp, vp]
        L.ref_decode_backward.argtypes = [i32, i32, i32, vp, vp, vp]
        L.ref_adam_steps.argtypes = [sz, vp, vp, i32, f64, f64, f64, f64]
        L.ref_predictor_instance.argtypes = [u64, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp,
                                             vp, vp]
        L.ref_optimize_flow_only.argtypes = [i32, i32, u64, u64, vp, sz, i32, f64, i32, vp, vp, vp,
                                             vp, vp]
        L.ref_read_events.argtypes = [C.c_char_p, vp, vp, vp, vp, vp, sz, vp]
        L.ref_write_events.argtypes = [C.c_char_p, i32, i32, u64, u64, vp, sz]
        L.ref_validate_slice.argtypes = [i32, i32, u64, u64, vp, sz]
        L.ref_random_slice.argtypes = [u64, sz, vp, vp, vp, vp, vp]
        L.ref_save_predictor.argtypes = [i32, i32, i32, vp, i32, vp, C.c_char_p, C.c_char_p]
        L.ref_load_predictor.argtypes = [C.c_char_p, C.c_char_p, vp, vp, vp, vp, vp, sz, vp, i32]
        L.ref_read_pfm.argtypes = [C.c_char_p, vp, vp, vp, sz]
        L.ref_format_number.argtypes = [f64, C.c_char_p]
        L.ref_format_number.restype = None
        L.ref_run_window.argtypes = [i32, vp, vp, vp, i32, i32, i32, vp, i32, vp, vp, f64, i32, i32,
                                     f64, vp, vp, vp, vp]
        L.ref_geo_loss.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, f64, i32, vp, vp, vp, vp, vp,
                                   vp, vp, vp, vp]
        L.ref_predictor_loss.argtypes = [i32, i32, i32, vp, i32, vp, vp, u64, u64, vp, sz, f64, vp,
                                         vp, vp]
        _ref = L
    return _ref


def _check(rc, L, which="oracle"):
    if rc != 0:
        msg = L.ref_last_error().decode() if which == "ref" else ""
        raise OracleError(rc, msg)


# ---------------------------------------------------------------------------
# Window containers


class Window:
    """One event window + flows: the (EventSlice, FlowSequence) pair."""

    def __init__(self, W, H, edges, events, flows):
        self.W, self.H = int(W), int(H)
        self.edges = np.ascontiguousarray(edges, dtype=np.uint64)
        self.B = len(self.edges) - 1
        self.events = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
        self.flows = np.ascontiguousarray(flows, dtype=np.float64).reshape(self.B, 2, self.H, self.W)

    @property
    def n(self):
        return len(self.events)


def make_edges(t0, t1, B):
    e = np.zeros(B + 1, np.uint64)
    lib().orc_make_edges(t0, t1, B, _p(e))
    return e


def make_events(t, x, y, p):
    ev = np.zeros(len(t), EVENT_DTYPE)
    ev["t_us"], ev["x"], ev["y"], ev["p"] = t, x, y, p
    return ev


# ---------------------------------------------------------------------------
# C restatement


def forward(w: Window, want_pos=False):
    R = w.B + 1
    HW = w.W * w.H
    out = dict(count=np.zeros((R, 2, w.H, w.W)), tsum=np.zeros((R, 2, w.H, w.W)),
               n_active=np.zeros(R, np.int64), alive=np.zeros(w.n, np.uint8),
               bin=np.zeros(w.n, np.int32))
    pos = np.zeros((w.n, R, 2)) if want_pos else None
    loss = C.c_double()
    ns = C.c_int()
    rc = lib().orc_forward(w.W, w.H, w.B, _p(w.edges), _p(w.events), w.n, _p(w.flows),
                           _p(out["count"]), _p(out["tsum"]), _p(out["n_active"]),
                           _p(out["alive"]), _p(out["bin"]), _p(pos), C.byref(loss), C.byref(ns))
    _check(rc, lib())
    out["loss"] = loss.value
    out["no_survivors"] = bool(ns.value)
    out["n_alive"] = int(out["alive"].sum())
    if want_pos:
        out["pos"] = pos
    del HW
    return out


def backward(w: Window, fwd=None):
    if fwd is None:
        fwd = forward(w)
    g = np.zeros((w.B, 2, w.H, w.W))
    rc = lib().orc_backward(w.W, w.H, w.B, _p(w.edges), _p(w.events), w.n, _p(w.flows),
                            _p(fwd["count"]), _p(fwd["tsum"]), _p(fwd["n_active"]),
                            _p(fwd["alive"]), _p(fwd["bin"]), int(fwd["no_survivors"]), _p(g))
    _check(rc, lib())
    return g


def depth_pose_to_flows(depth, poses, K, t0, t1, mask=None):
    depth = np.ascontiguousarray(depth, np.float64)
    H, W = depth.shape
    poses = np.ascontiguousarray(poses, np.float64).reshape(-1, 6)
    B = poses.shape[0]
    K = np.ascontiguousarray(K, np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    flows = np.zeros((B, 2, H, W))
    valid = np.zeros((B, H, W), np.uint8)
    rc = lib().orc_depth_pose_to_flows(W, H, _p(depth), _p(m), B, _p(poses), _p(K), t0, t1,
                                       _p(flows), _p(valid))
    _check(rc, lib())
    return flows, valid


def depth_pose_to_flows_backward(depth, poses, K, edges, grad, mask=None):
    depth = np.ascontiguousarray(depth, np.float64)
    H, W = depth.shape
    poses = np.ascontiguousarray(poses, np.float64).reshape(-1, 6)
    B = poses.shape[0]
    K = np.ascontiguousarray(K, np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    edges = np.ascontiguousarray(edges, np.uint64)
    grad = np.ascontiguousarray(grad, np.float64)
    dd = np.zeros((H, W))
    dp = np.zeros((B, 6))
    rc = lib().orc_depth_pose_to_flows_backward(W, H, _p(depth), _p(m), B, _p(poses), _p(K),
                                                _p(edges), _p(grad), _p(dd), _p(dp))
    _check(rc, lib())
    return dd, dp


# ---------------------------------------------------------------------------
# predictor decode chain (predictor.hpp:25-173, optimize.hpp:115-134)


def softplus(x):
    return lib().orc_softplus(float(x))


def softplus_grad(x):
    return lib().orc_softplus_grad(float(x))


def decode(params, factor):
    """depth = upsample_bilinear(softplus(params), factor) (predictor.hpp:126-131)."""
    params = np.ascontiguousarray(params, np.float64)
    ph, pw = params.shape
    depth = np.zeros((ph * factor, pw * factor))
    _check(lib().orc_decode(pw, ph, factor, _p(params), _p(depth)), lib())
    return depth


def decode_backward(params, factor, d_depth):
    """upsample_bilinear_adjoint(d_depth) * softplus_grad(params) (predictor.hpp:156-162)."""
    params = np.ascontiguousarray(params, np.float64)
    ph, pw = params.shape
    d_depth = np.ascontiguousarray(d_depth, np.float64)
    out = np.zeros((ph, pw))
    _check(lib().orc_decode_backward(pw, ph, factor, _p(params), _p(d_depth), _p(out)), lib())
    return out


def adam_step(slots, grads, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """Adam::step (optimize.hpp:115-134) in place; t is the incremented step count."""
    lib().orc_adam_step(slots.size, _p(slots), _p(np.ascontiguousarray(grads, np.float64)), _p(m),
                        _p(v), int(t), lr, beta1, beta2, eps)


def ref_decode(params, factor):
    params = np.ascontiguousarray(params, np.float64)
    ph, pw = params.shape
    depth = np.zeros((ph * factor, pw * factor))
    _check(ref().ref_decode(pw, ph, factor, _p(params), _p(depth)), ref(), "ref")
    return depth


def ref_decode_backward(params, factor, d_depth):
    params = np.ascontiguousarray(params, np.float64)
    ph, pw = params.shape
    d_depth = np.ascontiguousarray(d_depth, np.float64)
    out = np.zeros((ph, pw))
    _check(ref().ref_decode_backward(pw, ph, factor, _p(params), _p(d_depth), _p(out)), ref(), "ref")
    return out


def ref_adam_steps(slots, grads, t, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """t Adam steps of the reference from zero moments on fixed grads; returns the slots."""
    s = np.array(slots, np.float64)
    g = np.ascontiguousarray(grads, np.float64)
    _check(ref().ref_adam_steps(s.size, _p(s), _p(g), int(t), lr, beta1, beta2, eps), ref(), "ref")
    return s


def ref_predictor_instance(seed, sensor_w=16, sensor_h=12, factor=4, n_bins=2, n_events=24):
    """The reference's chain fixture (tests/chain_support.hpp:119-184) as a raw
    predictor, with the reference's predictor_loss_and_gradients (lambda_geo = 0)."""
    L = ref()
    n = C.c_size_t()
    args = (seed, sensor_w, sensor_h, factor, n_bins, n_events)
    _check(L.ref_predictor_instance(*args, C.byref(n), None, None, None, None, None, None, None),
           L, "ref")
    pw, ph = sensor_w // factor, sensor_h // factor
    ev = np.zeros(n.value, EVENT_DTYPE)
    params = np.zeros((ph, pw))
    poses = np.zeros((n_bins, 6))
    K = np.zeros(4)
    loss = np.zeros(1)
    dparams = np.zeros((ph, pw))
    dposes = np.zeros((n_bins, 6))
    _check(L.ref_predictor_instance(*args, C.byref(n), _p(ev), _p(params), _p(poses), _p(K),
                                    _p(loss), _p(dparams), _p(dposes)), L, "ref")
    return dict(events=ev, params=params, poses=poses, K=K, loss=float(loss[0]),
                d_params=dparams, d_poses=dposes)


def ref_optimize_flow_only(W, H, t0, t1, events, n_bins, lr, max_updates):
    """The reference's optimize_flow_only (optimize.hpp:385-487): (flows [B,2,H,W],
    l_cm, rsat, grad_norm_depth per logged update)."""
    L = ref()
    ev = np.ascontiguousarray(events, EVENT_DTYPE)
    flows = np.zeros((n_bins, 2, H, W))
    l_cm, rsat, gn = np.zeros(max_updates), np.zeros(max_updates), np.zeros(max_updates)
    nrec = C.c_int()
    _check(L.ref_optimize_flow_only(W, H, t0, t1, _p(ev), len(ev), n_bins, lr, max_updates,
                                    _p(flows), _p(l_cm), _p(rsat), _p(gn), C.byref(nrec)), L, "ref")
    k = nrec.value
    return flows, l_cm[:k], rsat[:k], gn[:k]


def rodrigues(omega):
    o = np.ascontiguousarray(omega, np.float64)
    R = np.zeros(9)
    lib().orc_rodrigues(_p(o), _p(R))
    return R.reshape(3, 3)


def rodrigues_jacobian(omega):
    o = np.ascontiguousarray(omega, np.float64)
    dR = np.zeros(27)
    lib().orc_rodrigues_jacobian(_p(o), _p(dR))
    return dR.reshape(3, 3, 3)


# ---------------------------------------------------------------------------
# The reference itself (oracle/_ref)


def ref_loss_and_grad(w: Window, backend="parallel", n_workers=0, deterministic=True,
                      backward=True, want_pos=False):
    L = ref()
    R = w.B + 1
    be = {"naive": 0, "padded": 1, "parallel": 2}[backend]
    out = dict(count=np.zeros((R, 2, w.H, w.W)), tsum=np.zeros((R, 2, w.H, w.W)),
               n_active=np.zeros(R, np.int64), alive=np.zeros(w.n, np.uint8),
               bin=np.zeros(w.n, np.int32))
    pos = np.zeros((w.n, R, 2)) if want_pos else None
    g = np.zeros((w.B, 2, w.H, w.W)) if backward else None
    loss = C.c_double()
    ns = C.c_int()
    rc = L.ref_loss_and_grad(w.W, w.H, w.B, _p(w.edges), _p(w.events), w.n, _p(w.flows), be,
                             n_workers, int(deterministic), int(backward), _p(out["count"]),
                             _p(out["tsum"]), _p(out["n_active"]), _p(out["alive"]),
                             _p(out["bin"]), _p(pos), C.byref(loss), C.byref(ns), _p(g))
    _check(rc, L, "ref")
    out["loss"] = loss.value
    out["no_survivors"] = bool(ns.value)
    out["n_alive"] = int(out["alive"].sum())
    if want_pos:
        out["pos"] = pos
    if backward:
        out["grad"] = g
    return out


def ref_warp_event(w: Window, x, y, t_from, t_to):
    o = np.zeros(2)
    _check(ref().ref_warp_event(w.W, w.H, w.B, _p(w.edges), _p(w.flows), x, y, t_from, t_to,
                                _p(o)), ref(), "ref")
    return o


def ref_rsat(w: Window):
    o = C.c_double()
    _check(ref().ref_rsat(w.W, w.H, w.B, _p(w.edges), _p(w.events), w.n, _p(w.flows),
                          C.byref(o)), ref(), "ref")
    return o.value


def ref_depth_pose_to_flows(depth, poses, K, t0, t1, mask=None):
    depth = np.ascontiguousarray(depth, np.float64)
    H, W = depth.shape
    poses = np.ascontiguousarray(poses, np.float64).reshape(-1, 6)
    B = poses.shape[0]
    K = np.ascontiguousarray(K, np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    flows = np.zeros((B, 2, H, W))
    valid = np.zeros((B, H, W), np.uint8)
    edges = np.zeros(B + 1, np.uint64)
    _check(ref().ref_depth_pose_to_flows(W, H, _p(depth), _p(m), B, _p(poses), _p(K), t0, t1,
                                         _p(flows), _p(valid), _p(edges)), ref(), "ref")
    return flows, valid, edges


def ref_depth_pose_to_flows_backward(depth, poses, K, edges, grad, mask=None):
    depth = np.ascontiguousarray(depth, np.float64)
    H, W = depth.shape
    poses = np.ascontiguousarray(poses, np.float64).reshape(-1, 6)
    B = poses.shape[0]
    K = np.ascontiguousarray(K, np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    edges = np.ascontiguousarray(edges, np.uint64)
    grad = np.ascontiguousarray(grad, np.float64)
    dd = np.zeros((H, W))
    dp = np.zeros((B, 6))
    _check(ref().ref_depth_pose_to_flows_backward(W, H, _p(depth), _p(m), B, _p(poses), _p(K),
                                                  _p(edges), _p(grad), _p(dd), _p(dp)),
           ref(), "ref")
    return dd, dp


def ref_fd_instance(seed, max_events=0, max_dim=0, want_masked=False) -> Window:
    L = ref()
    W, H, B = C.c_int(), C.c_int(), C.c_int()
    n, nm = C.c_size_t(), C.c_size_t()
    _check(L.ref_random_fd_instance(seed, max_events, max_dim, int(want_masked), C.byref(W),
                                    C.byref(H), C.byref(B), C.byref(n), None, None, None,
                                    C.byref(nm)), L, "ref")
    edges = np.zeros(B.value + 1, np.uint64)
    ev = np.zeros(n.value, EVENT_DTYPE)
    flows = np.zeros((B.value, 2, H.value, W.value))
    _check(L.ref_random_fd_instance(seed, max_events, max_dim, int(want_masked), C.byref(W),
                                    C.byref(H), C.byref(B), C.byref(n), _p(edges), _p(ev),
                                    _p(flows), C.byref(nm)), L, "ref")
    w = Window(W.value, H.value, edges, ev, flows)
    w.n_masked = nm.value
    return w


def ref_bench_window(W, H, B, n_events, seed=1, window_s=0.1) -> Window:
    edges = np.zeros(B + 1, np.uint64)
    ev = np.zeros(n_events, EVENT_DTYPE)
    flows = np.zeros((B, 2, H, W))
    _check(ref().ref_bench_window(W, H, B, window_s, seed, n_events, _p(edges), _p(ev),
                                  _p(flows)), ref(), "ref")
    return Window(W, H, edges, ev, flows)


def ref_generate_scene(W, H, poses, K, event_rate, seed):
    L = ref()
    poses = np.ascontiguousarray(poses, np.float64).reshape(-1, 6)
    B = poses.shape[0]
    K = np.ascontiguousarray(K, np.float64)
    n = C.c_size_t()
    _check(L.ref_generate_scene(W, H, B, _p(poses), _p(K), event_rate, seed, C.byref(n), None,
                                None, None), L, "ref")
    ev = np.zeros(n.value, EVENT_DTYPE)
    depth = np.zeros((H, W))
    mask = np.zeros((H, W), np.uint8)
    _check(L.ref_generate_scene(W, H, B, _p(poses), _p(K), event_rate, seed, C.byref(n),
                                _p(ev), _p(depth), _p(mask)), L, "ref")
    return ev, depth, mask


def ref_chain_instance(seed, sensor_w=16, sensor_h=12, factor=4, n_bins=2, n_events=24):
    L = ref()
    n = C.c_size_t()
    _check(L.ref_chain_instance(seed, sensor_w, sensor_h, factor, n_bins, n_events, C.byref(n),
                                None, None, None, None), L, "ref")
    ev = np.zeros(n.value, EVENT_DTYPE)
    depth = np.zeros((sensor_h, sensor_w))
    poses = np.zeros((n_bins, 6))
    K = np.zeros(4)
    _check(L.ref_chain_instance(seed, sensor_w, sensor_h, factor, n_bins, n_events, C.byref(n),
                                _p(ev), _p(depth), _p(poses), _p(K)), L, "ref")
    return ev, depth, poses, K


def ref_chain_batch(depth, poses, K, t0, t1, events, ev_off, n_workers=0, want_grads=False):
    """Reference chain (flows → loss_and_grad → flows backward), window by window."""
    L = ref()
    depth = np.ascontiguousarray(depth, np.float64)
    nw, H, W = depth.shape
    poses = np.ascontiguousarray(poses, np.float64)
    B = poses.shape[1]
    K = np.ascontiguousarray(K, np.float64)
    events = np.ascontiguousarray(events, EVENT_DTYPE)
    ev_off = np.ascontiguousarray(ev_off, np.uint64)
    dd = np.zeros((nw, H, W)) if want_grads else None
    dp = np.zeros((nw, B, 6)) if want_grads else None
    ls, sec = C.c_double(), C.c_double()
    _check(L.ref_chain_batch(W, H, B, nw, _p(depth), _p(poses), _p(K), t0, t1, _p(events),
                             _p(ev_off), n_workers, C.byref(ls), _p(dd), _p(dp), C.byref(sec)),
           L, "ref")
    return dict(loss_sum=ls.value, seconds=sec.value, d_depth=dd, d_poses=dp)


# ---------------------------------------------------------------------------
# EVT1 event files (io.hpp:106-172): numpy restatement + the reference itself


def read_events(path):
    """read_events (io.hpp:115-154) restated: returns (W, H, t0, t1, events) or
    raises OracleError with the reference's error code. Checks in the
    reference's order: header length, magic, zero dims, count vs payload,
    trailing bytes, then per record coordinate -> polarity -> order."""
    data = open(path, "rb").read()
    if len(data) < 16:  # io.hpp:120-121
        raise OracleError(11, "EVT1: file shorter than the 16-byte header")
    if data[:4] != b"EVT1":  # io.hpp:122-123
        raise OracleError(10, "EVT1: bad magic")
    W = int.from_bytes(data[4:6], "little")
    H = int.from_bytes(data[6:8], "little")
    count = int.from_bytes(data[8:16], "little")
    if W == 0 or H == 0:  # io.hpp:128-129
        raise OracleError(2, "EVT1: zero sensor dimension")
    payload = len(data) - 16
    if count > payload // 16:  # io.hpp:131-132
        raise OracleError(11, "EVT1: header count exceeds payload size")
    if payload != count * 16:  # io.hpp:133-134
        raise OracleError(12, "EVT1: trailing bytes after last record")
    src = np.frombuffer(data, EVENT_DTYPE, count, 16)
    ev = np.zeros(count, EVENT_DTYPE)
    for n in EVENT_DTYPE.names:
        ev[n] = src[n]
    code = first_violation(ev, W, H)  # io.hpp:137-150
    if code:
        raise OracleError(code[1], f"EVT1: record {code[0]}")
    t0 = int(ev["t_us"][0]) if count else 0  # io.hpp:152-153
    t1 = int(ev["t_us"][-1]) + 1 if count else 0
    return W, H, t0, t1, ev


def first_violation(ev, W, H, window=None):
    """First record failing read_events' / EventSlice::validate's checks, as
    (index, code), or None (io.hpp:141-149, types.hpp:146-158)."""
    if len(ev) == 0:
        return None
    bad_xy = (ev["x"] >= W) | (ev["y"] >= H)
    bad_p = (ev["p"] != 1) & (ev["p"] != -1)
    bad_s = np.zeros(len(ev), bool)
    bad_s[1:] = ev["t_us"][1:] < ev["t_us"][:-1]
    bad_t = np.zeros(len(ev), bool)
    if window is not None:
        bad_t = (ev["t_us"] < window[0]) | (ev["t_us"] >= window[1])
    idx = np.flatnonzero(bad_xy | bad_p | bad_s | bad_t)
    if len(idx) == 0:
        return None
    k = int(idx[0])
    return k, 3 if bad_xy[k] else 4 if bad_p[k] else 5 if bad_s[k] else 6


def write_events(path, W, H, t0, t1, ev):
    """write_events (io.hpp:156-172) restated (after EventSlice::validate)."""
    if W == 0 or H == 0:
        raise OracleError(2, "event slice: width and height must be positive")
    if t1 < t0:
        raise OracleError(6, "event slice: t_end precedes t_start")
    code = first_violation(ev, W, H, (t0, t1))
    if code:
        raise OracleError(code[1], f"event slice: record {code[0]}")
    rec = np.zeros(len(ev), EVENT_DTYPE)
    for n in EVENT_DTYPE.names:
        rec[n] = ev[n]
    with open(path, "wb") as f:
        f.write(b"EVT1" + int(W).to_bytes(2, "little") + int(H).to_bytes(2, "little")
                + len(ev).to_bytes(8, "little") + rec.tobytes())


def window_offsets(ev, t0, window_us, n_windows):
    """offsets[w] = first event with t >= t0 + w * window_us."""
    b = np.uint64(t0) + np.arange(n_windows + 1, dtype=np.uint64) * np.uint64(window_us)
    return np.searchsorted(ev["t_us"], b, side="left").astype(np.uint64)


def ref_read_events(path):
    L = ref()
    W, H, n = C.c_int(), C.c_int(), C.c_size_t()
    t0, t1 = C.c_uint64(), C.c_uint64()
    _check(L.ref_read_events(os.fspath(path).encode(), C.byref(W), C.byref(H), C.byref(t0),
                             C.byref(t1), None, 0, C.byref(n)), L, "ref")
    ev = np.zeros(n.value, EVENT_DTYPE)
    _check(L.ref_read_events(os.fspath(path).encode(), C.byref(W), C.byref(H), C.byref(t0),
                             C.byref(t1), _p(ev), len(ev), C.byref(n)), L, "ref")
    return W.value, H.value, t0.value, t1.value, ev


def ref_write_events(path, W, H, t0, t1, ev):
    L = ref()
    ev = np.ascontiguousarray(ev, EVENT_DTYPE)
    _check(L.ref_write_events(os.fspath(path).encode(), W, H, t0, t1, _p(ev), len(ev)), L, "ref")


def ref_validate_slice(W, H, t0, t1, ev):
    L = ref()
    ev = np.ascontiguousarray(ev, EVENT_DTYPE)
    return L.ref_validate_slice(W, H, t0, t1, _p(ev), len(ev))


def ref_random_slice(seed, n):
    """evcm_test::random_slice(std::mt19937_64(seed), n) -> (W, H, t0, t1, events)."""
    L = ref()
    W, H = C.c_int(), C.c_int()
    t0, t1 = C.c_uint64(), C.c_uint64()
    ev = np.zeros(n, EVENT_DTYPE)
    _check(L.ref_random_slice(seed, n, C.byref(W), C.byref(H), C.byref(t0), C.byref(t1), _p(ev)),
           L, "ref")
    return W.value, H.value, t0.value, t1.value, ev


# ---------------------------------------------------------------------------
# geometry-consistency loss L_geo (geometry.hpp:329-543)


def _geo_outputs(H, W):
    return dict(value=np.zeros(1), n_valid=np.zeros(1, np.int64), projected=np.zeros((H, W)),
                interpolated=np.zeros((H, W)), valid=np.zeros((H, W), np.uint8),
                d_d0=np.zeros((H, W)), d_d1=np.zeros((H, W)), d_pose=np.zeros(6))


def geo_loss(d0, d1, pose, K, m0=None, m1=None, upstream=1.0, want_grad=True):
    """orc_geo_loss: the restatement (one pose). Returns a dict of the terms and,
    with want_grad, d_d0 / d_d1 / d_pose (omega, trans)."""
    L = lib()
    H, W = d0.shape
    o = _geo_outputs(H, W)
    c = lambda a, t=np.float64: None if a is None else np.ascontiguousarray(a, t)  # noqa: E731
    d0, d1, pose, K = c(d0), c(d1), c(pose), c(K)
    m0, m1 = c(m0, np.uint8), c(m1, np.uint8)
    _check(L.orc_geo_loss(W, H, _p(d0), _p(m0), _p(d1), _p(m1), _p(pose), _p(K), upstream,
                          int(want_grad), _p(o["value"]), _p(o["n_valid"]), _p(o["projected"]),
                          _p(o["interpolated"]), _p(o["valid"]), _p(o["d_d0"]), _p(o["d_d1"]),
                          _p(o["d_pose"])), L)
    o["value"], o["n_valid"] = float(o["value"][0]), int(o["n_valid"][0])
    o["empty"] = o["n_valid"] == 0
    return o


def ref_geo_loss(d0, d1, pose, K, m0=None, m1=None, upstream=1.0, want_grad=True):
    """The reference's geometry_consistency_loss[_backward] (one pose)."""
    L = ref()
    H, W = d0.shape
    o = _geo_outputs(H, W)
    empty = np.zeros(1, np.int32)
    c = lambda a, t=np.float64: None if a is None else np.ascontiguousarray(a, t)  # noqa: E731
    d0, d1, pose, K = c(d0), c(d1), c(pose), c(K)
    m0, m1 = c(m0, np.uint8), c(m1, np.uint8)
    _check(L.ref_geo_loss(W, H, _p(d0), _p(m0), _p(d1), _p(m1), _p(pose), _p(K), upstream,
                          int(want_grad), _p(o["value"]), _p(o["n_valid"]), _p(empty),
                          _p(o["projected"]), _p(o["interpolated"]), _p(o["valid"]),
                          _p(o["d_d0"]), _p(o["d_d1"]), _p(o["d_pose"])), L, "ref")
    o["value"], o["n_valid"] = float(o["value"][0]), int(o["n_valid"][0])
    o["empty"] = bool(empty[0])
    return o


def ref_predictor_loss(params, factor, poses, K, t0, t1, events, lambda_geo):
    """The reference's predictor_loss_and_gradients with any lambda_geo:
    ((l_cm, l_geo, total), d_params, d_poses)."""
    L = ref()
    ph, pw = params.shape
    B = poses.shape[0]
    losses = np.zeros(3)
    dpar = np.zeros((ph, pw))
    dpo = np.zeros((B, 6))
    params = np.ascontiguousarray(params, np.float64)
    poses = np.ascontiguousarray(poses, np.float64)
    K = np.ascontiguousarray(K, np.float64)
    ev = np.ascontiguousarray(events, EVENT_DTYPE)
    _check(L.ref_predictor_loss(pw, ph, factor, _p(params), B, _p(poses), _p(K), t0, t1, _p(ev),
                                len(ev), lambda_geo, _p(losses), _p(dpar), _p(dpo)), L, "ref")
    return tuple(losses), dpar, dpo


def ref_format_number(v):
    buf = C.create_string_buffer(64)
    ref().ref_format_number(float(v), buf)
    return buf.value.decode()


def ref_run_window(windows, params, factor, poses, K, lr, steps_per_update, max_updates,
                   lambda_geo):
    """The reference's run_window; windows = [(t0, t1, events), ...]. Returns
    (params, poses, records [n, 6] = l_cm, l_geo, total, rsat, gnd, gnp)."""
    L = ref()
    nw = len(windows)
    t01 = np.array([[w[0], w[1]] for w in windows], np.uint64).reshape(-1)
    evs = [np.ascontiguousarray(w[2], EVENT_DTYPE) for w in windows]
    offs = np.zeros(nw + 1, np.uint64)
    offs[1:] = np.cumsum([len(e) for e in evs])
    ev = np.concatenate(evs).astype(EVENT_DTYPE) if nw else np.zeros(0, EVENT_DTYPE)
    ph, pw = params.shape
    B = poses.shape[0]
    po, qo = np.zeros((ph, pw)), np.zeros((B, 6))
    rec = np.zeros((max(max_updates, 1), 6))
    n = C.c_int()
    params = np.ascontiguousarray(params, np.float64)
    poses = np.ascontiguousarray(poses, np.float64)
    K = np.ascontiguousarray(K, np.float64)
    _check(L.ref_run_window(nw, _p(t01), _p(ev), _p(offs), pw, ph, factor, _p(params), B, _p(poses),
                            _p(K), lr, steps_per_update, max_updates, lambda_geo, _p(po), _p(qo),
                            _p(rec), C.byref(n)), L, "ref")
    return po, qo, rec[: n.value]


def ref_save_predictor(params, factor, poses, pfm, csv):
    L = ref()
    ph, pw = params.shape
    params = np.ascontiguousarray(params, np.float64)
    poses = np.ascontiguousarray(poses, np.float64)
    _check(L.ref_save_predictor(pw, ph, factor, _p(params), poses.shape[0], _p(poses),
                                os.fspath(pfm).encode(), os.fspath(csv).encode()), L, "ref")


def ref_load_predictor(pfm, csv):
    """-> (params [ph, pw], factor, poses [B, 6]) or OracleError."""
    L = ref()
    pw, ph, f, nb = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    args = (os.fspath(pfm).encode(), os.fspath(csv).encode())
    _check(L.ref_load_predictor(*args, C.byref(pw), C.byref(ph), C.byref(f), C.byref(nb), None, 0,
                                None, 0), L, "ref")
    params = np.zeros((ph.value, pw.value))
    poses = np.zeros((nb.value, 6))
    _check(L.ref_load_predictor(*args, C.byref(pw), C.byref(ph), C.byref(f), C.byref(nb),
                                _p(params), params.size, _p(poses), nb.value), L, "ref")
    return params, f.value, poses


def ref_read_pfm(path):
    L = ref()
    w, h = C.c_int(), C.c_int()
    _check(L.ref_read_pfm(os.fspath(path).encode(), C.byref(w), C.byref(h), None, 0), L, "ref")
    out = np.zeros((h.value, w.value), np.float32)
    _check(L.ref_read_pfm(os.fspath(path).encode(), C.byref(w), C.byref(h), _p(out), out.size),
           L, "ref")
    return out
