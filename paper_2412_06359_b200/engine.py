"""Host-side mirror of the reference operator API for the CMax loss path.

The reference (evcm, C++20) exposes the path through ``evcm::Engine``
(engine.hpp:134-213), the free functions ``depth_pose_to_flows`` /
``depth_pose_to_flows_backward`` (geometry.hpp:229-325) and the module-level
helpers ``build_iwe_stack`` / ``contrast_loss_backward`` / ``rsat``
(engine.hpp:606-631). This module keeps those names, argument meanings and
the error taxonomy (types.hpp:18-76), and forwards every call through the
C-ABI of ``libevcm_cuda.so`` (include/evcm_cuda.h) to the sm_100a kernels.
There is no CPU fallback: if the shared library or a CUDA device is missing,
construction fails loudly.

Host arrays are numpy; device-resident arrays are torch CUDA tensors (passed
by pointer, no copies).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _build

# ---------------------------------------------------------------------------
# error taxonomy (types.hpp:18-76)


class Error(RuntimeError):
    pass


class IoError(Error):
    pass


class BadMagicError(IoError):
    """File does not start with the expected format magic (types.hpp:28-31)."""


class TruncatedFileError(IoError):
    """File ends mid-header or mid-record (types.hpp:33-36)."""


class UnsortedEventsError(Error):
    pass


class CoordinateRangeError(Error):
    pass


class InvalidPolarityError(Error):
    pass


class TimeRangeError(Error):
    pass


class DimensionMismatchError(Error):
    pass


class EmptySliceError(Error):
    pass


class ConfigError(Error):
    pass


class DivergenceError(Error):
    pass


_ERRORS = {1: ConfigError, 2: DimensionMismatchError, 3: CoordinateRangeError,
           4: InvalidPolarityError, 5: UnsortedEventsError, 6: TimeRangeError,
           7: EmptySliceError, 20: Error, 21: ConfigError}

# evcm::Event, 16 bytes (types.hpp:106-113)
EVENT_DTYPE = np.dtype(
    {"names": ["t_us", "x", "y", "p"], "formats": ["<u8", "<u2", "<u2", "i1"],
     "offsets": [0, 8, 10, 12], "itemsize": 16})

MEM_HOST, MEM_DEVICE = 0, 1
KLOSS_EPS = 1e-9  # warp.hpp:26

# ---------------------------------------------------------------------------
# C-ABI binding


class _Options(C.Structure):
    _fields_ = [("device", C.c_int), ("deterministic", C.c_int), ("stack_f64", C.c_int),
                ("grad_f64", C.c_int), ("stream", C.c_void_p), ("algo", C.c_int)]


class _Slice(C.Structure):
    _fields_ = [("width", C.c_uint16), ("height", C.c_uint16), ("t_start_us", C.c_uint64),
                ("t_end_us", C.c_uint64), ("events", C.c_void_p), ("n_events", C.c_size_t)]


class _Flows(C.Structure):
    _fields_ = [("n_bins", C.c_int), ("edges_us", C.c_void_p), ("uv", C.c_void_p),
                ("width", C.c_int), ("height", C.c_int)]


class _Loss(C.Structure):
    _fields_ = [("value", C.c_double), ("no_survivors", C.c_int), ("forward_id", C.c_uint64)]


class _ChainBatch(C.Structure):
    _fields_ = [("n_windows", C.c_int), ("width", C.c_int), ("height", C.c_int),
                ("n_bins", C.c_int), ("t_start_us", C.c_uint64), ("t_end_us", C.c_uint64),
                ("K", C.c_double * 4), ("events", C.c_void_p), ("ev_offsets", C.c_void_p),
                ("depth", C.c_void_p), ("poses", C.c_void_p), ("window_stride_us", C.c_uint64)]


class _ChainOut(C.Structure):
    _fields_ = [("loss", C.c_void_p), ("no_survivors", C.c_void_p), ("d_depth", C.c_void_p),
                ("d_poses", C.c_void_p), ("sums", C.c_void_p)]


_lib = None


def library_path() -> str:
    return _build.LIB


def load_library(build_if_missing: bool = True):
    """Loads libevcm_cuda.so (in-tree). Raises if it is absent and cannot be built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_build.LIB):
        if not build_if_missing:
            raise Error(f"libevcm_cuda.so missing at {_build.LIB}; run __graft_entry__.build()")
        _build.build()
    L = C.CDLL(_build.LIB)
    vp, i32, u64, sz = C.c_void_p, C.c_int, C.c_uint64, C.c_size_t
    L.evcm_cuda_last_error.restype = C.c_char_p
    L.evcm_cuda_error_name.restype = C.c_char_p
    L.evcm_cuda_create.argtypes = [vp, vp]
    L.evcm_cuda_destroy.argtypes = [vp]
    L.evcm_cuda_destroy.restype = None
    L.evcm_cuda_default_options.argtypes = [vp]
    L.evcm_cuda_default_options.restype = None
    L.evcm_cuda_forward.argtypes = [vp, vp, vp, i32, vp]
    L.evcm_cuda_forward_products.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
    L.evcm_cuda_backward.argtypes = [vp, vp, vp, i32, vp]
    L.evcm_cuda_backward_of.argtypes = [vp, vp, vp, u64, i32, vp]
    L.evcm_cuda_phase_stats.argtypes = [vp, vp, vp]
    L.evcm_cuda_sort_products.argtypes = [vp, vp, vp, vp, vp]
    L.evcm_cuda_stream_wait.argtypes = [vp, vp]
    L.evcm_cuda_stream_signal.argtypes = [vp, vp]
    L.evcm_cuda_abi_version.restype = i32
    L.evcm_cuda_loss_and_grad.argtypes = [vp, vp, vp, i32, vp, vp]
    L.evcm_cuda_depth_pose_to_flows.argtypes = [vp, i32, i32, vp, vp, i32, vp, vp, u64, u64,
                                                i32, vp, vp, vp]
    L.evcm_cuda_depth_pose_to_flows_backward.argtypes = [vp, i32, i32, vp, vp, i32, vp, vp, vp,
                                                         vp, i32, vp, vp]
    L.evcm_cuda_chain_batch.argtypes = [vp, vp, i32, vp]
    L.evcm_cuda_chain_batch2.argtypes = [vp, vp, i32, i32, vp]
    L.evcm_cuda_chain_batch_async.argtypes = [vp, vp, i32, i32, vp, i32]
    L.evcm_cuda_chain_wait.argtypes = [vp, i32]
    L.evcm_cuda_set_timing.argtypes = [vp, i32]
    L.evcm_cuda_stage_times.argtypes = [vp, vp, i32]
    L.evcm_cuda_last_launch_count.argtypes = [vp]
    L.evcm_cuda_last_algo.argtypes = [vp]
    L.evcm_cuda_workspace_bytes.argtypes = [vp]
    L.evcm_cuda_workspace_bytes.restype = sz
    f64 = C.c_double
    L.evcm_cuda_decode.argtypes = [vp, i32, i32, i32, vp, i32, vp]
    L.evcm_cuda_decode_backward.argtypes = [vp, i32, i32, i32, vp, vp, i32, vp]
    L.evcm_cuda_adam_step.argtypes = [vp, sz, vp, vp, vp, vp, i32, f64, f64, f64, f64, i32]
    L.evcm_cuda_predictor_loss_and_gradients_geo.argtypes = [vp, i32, i32, i32, vp, i32, vp, vp,
                                                             vp, f64, i32, vp, vp, vp]
    L.evcm_cuda_geometry_consistency_loss.argtypes = [vp, i32, i32, vp, vp, vp, vp, i32, vp, vp,
                                                      f64, i32, i32, vp]
    L.evcm_cuda_validate_slice.argtypes = [vp, vp, i32, i32, vp]
    L.evcm_cuda_window_offsets.argtypes = [vp, vp, sz, u64, u64, i32, i32, vp]
    L.evcm_cuda_predictor_loss_and_gradients.argtypes = [vp, i32, i32, i32, vp, i32, vp, vp, vp,
                                                         i32, vp, vp, vp]
    _lib = L
    return L


def _raise(rc: int):
    if rc == 0:
        return
    msg = load_library().evcm_cuda_last_error().decode()
    raise _ERRORS.get(rc, Error)(msg)


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _mem_of(*arrays) -> int:
    kinds = {(_is_torch(a) and a.is_cuda) for a in arrays if a is not None}
    if len(kinds) > 1:
        raise ConfigError("inputs must all be host (numpy) or all device (torch cuda)")
    return MEM_DEVICE if kinds == {True} else MEM_HOST


# ---------------------------------------------------------------------------
# reference data types (types.hpp)


@dataclass
class CameraIntrinsics:
    fx: float = 1.0
    fy: float = 1.0
    cx: float = 0.0
    cy: float = 0.0

    def as_array(self):
        return np.array([self.fx, self.fy, self.cx, self.cy], np.float64)


@dataclass
class EventSlice:
    """EventSlice (types.hpp:121-160): sensor size, [t_start, t_end) window, events."""
    width: int
    height: int
    t_start_us: int
    t_end_us: int
    events: object = None  # numpy EVENT_DTYPE array or torch uint8 cuda tensor [n,16]

    def __post_init__(self):
        if self.events is None:
            self.events = np.zeros(0, EVENT_DTYPE)

    @property
    def n_events(self) -> int:
        if _is_torch(self.events):
            return self.events.numel() // 16
        return len(self.events)

    def duration_s(self) -> float:
        return (float(self.t_end_us) - float(self.t_start_us)) * 1e-6

    def _c(self):
        ev = self.events
        if not _is_torch(ev):
            ev = np.ascontiguousarray(ev, dtype=EVENT_DTYPE)
            self.events = ev
        return _Slice(self.width, self.height, self.t_start_us, self.t_end_us, _ptr(ev),
                      self.n_events)


def make_edges(t_start_us: int, t_end_us: int, n_bins: int) -> np.ndarray:
    """FlowSequence::zeros edge rule (types.hpp:293-300)."""
    if n_bins < 1 or t_end_us <= t_start_us:
        raise ConfigError("flow sequence: need n_bins >= 1 and a nonempty window")
    span = float(t_end_us - t_start_us)
    e = np.zeros(n_bins + 1, np.uint64)
    for i in range(n_bins + 1):
        # std::llround(span * i / B): round half away from zero
        v = span * i / n_bins
        r = int(v) + (1 if v - int(v) >= 0.5 else 0)  # std::llround, v >= 0
        e[i] = t_end_us if i == n_bins else t_start_us + r
    return e


@dataclass
class FlowSequence:
    """FlowSequence (types.hpp:251-319): B+1 edges, B (u, v) fields in px/s.

    ``uv`` is [B, 2, H, W] float64 (numpy on the host or a torch cuda tensor)."""
    edges_us: np.ndarray
    uv: object

    @property
    def n_bins(self) -> int:
        return len(self.edges_us) - 1

    @property
    def width(self) -> int:
        return int(self.uv.shape[-1])

    @property
    def height(self) -> int:
        return int(self.uv.shape[-2])

    def t_start_us(self):
        return int(self.edges_us[0])

    def t_end_us(self):
        return int(self.edges_us[-1])

    def bin_duration_s(self, i: int) -> float:
        return (float(self.edges_us[i + 1]) - float(self.edges_us[i])) * 1e-6

    @staticmethod
    def zeros(width, height, t_start_us, t_end_us, n_bins) -> "FlowSequence":
        e = make_edges(t_start_us, t_end_us, n_bins)
        return FlowSequence(e, np.zeros((n_bins, 2, height, width)))

    def zeros_like(self) -> "FlowSequence":
        if _is_torch(self.uv):
            import torch
            return FlowSequence(self.edges_us.copy(), torch.zeros_like(self.uv))
        return FlowSequence(self.edges_us.copy(), np.zeros_like(self.uv))

    def _c(self):
        self.edges_us = np.ascontiguousarray(self.edges_us, np.uint64)
        if _is_torch(self.uv):
            import torch
            if self.uv.dtype != torch.float64 or not self.uv.is_contiguous():
                raise DimensionMismatchError("flow sequence: uv must be a contiguous float64 "
                                             "[B, 2, H, W] tensor")
        else:
            self.uv = np.ascontiguousarray(self.uv, np.float64)
        if self.uv.ndim != 4 or self.uv.shape[0] != self.n_bins or self.uv.shape[1] != 2:
            raise DimensionMismatchError("flow sequence: uv must be [B, 2, H, W]")
        return _Flows(self.n_bins, _ptr(self.edges_us), _ptr(self.uv), self.width, self.height)


@dataclass
class LossResult:
    value: float = 0.0
    no_survivors: bool = False


@dataclass
class IweStack:
    """IweStack (warp.hpp:167-193): count/tsum [B+1, 2, H, W], n_active [B+1]."""
    width: int
    height: int
    n_refs: int
    count: np.ndarray
    tsum: np.ndarray
    n_active: np.ndarray


@dataclass
class Trajectories:
    """Trajectories (warp.hpp:196-220)."""
    n_events: int
    n_refs: int
    alive: np.ndarray
    bin: np.ndarray
    n_alive: int
    pos: Optional[np.ndarray] = None

    def position(self, k: int, r: int):
        return self.pos[k, r]


@dataclass
class PhaseStats:
    time_us: float = 0.0
    peak_bytes: int = 0


class ForwardResult:
    """ForwardResult (engine.hpp:99-105). The stack and trajectories stay on the
    device; ``stack`` / ``traj`` copy them back on first access."""

    def __init__(self, engine: "Engine", generation: int, loss: LossResult, dims,
                 forward_id: int = 0, stats=None):
        self._engine = engine
        self._gen = generation
        self._id = forward_id
        self.loss = loss
        self._dims = dims  # (W, H, B, n)
        self._stack = None
        self._traj = None
        st = stats or [PhaseStats()] * 3
        self.warp_stats, self.splat_stats, self.loss_stats = st[0], st[1], st[2]

    def _check_live(self):
        if self._engine._generation != self._gen:
            raise ConfigError("forward result is stale: the engine ran another forward since")

    @property
    def stack(self) -> IweStack:
        if self._stack is None:
            self._check_live()
            W, H, B, n = self._dims
            R = B + 1
            count = np.zeros((R, 2, H, W))
            tsum = np.zeros((R, 2, H, W))
            na = np.zeros(R, np.int64)
            _raise(load_library().evcm_cuda_forward_products(
                self._engine._h, _ptr(count), _ptr(tsum), _ptr(na), None, None, None, None))
            self._stack = IweStack(W, H, R, count, tsum, na)
        return self._stack

    def alive_bin(self):
        """(alive u8 [n], bin i32 [n], n_alive) without the positions (which are
        (B+1) x 16 B per event)."""
        self._check_live()
        n = self._dims[3]
        alive = np.zeros(n, np.uint8)
        bins = np.zeros(n, np.int32)
        na = C.c_size_t()
        _raise(load_library().evcm_cuda_forward_products(
            self._engine._h, None, None, None, _ptr(alive), _ptr(bins), None, C.byref(na)))
        return alive, bins, int(na.value)

    def sort_products(self):
        """(keys [n], perm [n_sorted], sorted_keys [n_sorted]) of the forward's
        stable tile sort (owner pipeline), uint32."""
        self._check_live()
        n = self._dims[3]
        keys = np.zeros(n, np.uint32)
        perm = np.zeros(n, np.uint32)
        sk = np.zeros(n, np.uint32)
        ns = C.c_size_t()
        _raise(load_library().evcm_cuda_sort_products(self._engine._h, _ptr(keys), _ptr(perm),
                                                      _ptr(sk), C.byref(ns)))
        return keys, perm[: ns.value], sk[: ns.value]

    @property
    def traj(self) -> Trajectories:
        if self._traj is None:
            self._check_live()
            W, H, B, n = self._dims
            alive = np.zeros(n, np.uint8)
            bins = np.zeros(n, np.int32)
            pos = np.zeros((n, B + 1, 2))
            na = C.c_size_t()
            _raise(load_library().evcm_cuda_forward_products(
                self._engine._h, None, None, None, _ptr(alive), _ptr(bins), _ptr(pos),
                C.byref(na)))
            self._traj = Trajectories(n, B + 1, alive, bins, int(na.value), pos)
        return self._traj


@dataclass
class BackwardResult:
    """BackwardResult (engine.hpp:107-110): grad [B, 2, H, W] = (gu, gv) per bin."""
    grad: object
    stats: PhaseStats = field(default_factory=PhaseStats)


# ---------------------------------------------------------------------------
# Engine (engine.hpp:134-213)

BACKENDS = ("cuda",)


def backend_from_name(name: str) -> str:
    """backend_from_name (engine.hpp:39-44) for this build: only "cuda"."""
    if name in BACKENDS:
        return name
    raise ConfigError(f"unknown backend '{name}' (cuda)")


@dataclass
class EngineOptions:
    """EngineOptions (engine.hpp:54-61) for the cuda backend."""
    backend: str = "cuda"
    device: int = 0
    deterministic: bool = True  # engine.hpp:60
    stack_f64: bool = True   # parity precision; False = fp32 "fast" stack
    grad_f64: bool = False
    stream: Optional[int] = None  # raw cudaStream_t handle, None = engine-owned
    algo: str = "auto"  # "owner" (tiles) | "atomic" (per-event atomics) | "auto"


class Engine:
    """evcm::Engine with the cuda backend."""

    def __init__(self, opts: Optional[EngineOptions] = None):
        self.opts = opts or EngineOptions()
        backend_from_name(self.opts.backend)
        L = load_library()
        algos = {"owner": 0, "atomic": 1, "auto": 2}
        if self.opts.algo not in algos:
            raise ConfigError(f"unknown algo '{self.opts.algo}' (owner|atomic|auto)")
        if self.opts.deterministic and self.opts.algo == "atomic":
            raise ConfigError("deterministic mode needs algo='owner' or 'auto'")
        o = _Options(self.opts.device, int(self.opts.deterministic), int(self.opts.stack_f64),
                     int(self.opts.grad_f64), self.opts.stream, algos[self.opts.algo])
        h = C.c_void_p()
        _raise(L.evcm_cuda_create(C.byref(o), C.byref(h)))
        self._h = h
        self._generation = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.evcm_cuda_destroy(h)
            self._h = None

    def options(self) -> EngineOptions:
        return self.opts

    def _order_after(self, *arrays) -> None:
        """Device inputs produced on the caller's current torch stream: the
        engine's stream waits for that work before its kernels read them."""
        for a in arrays:
            if a is not None and _is_torch(a) and a.is_cuda:
                import torch
                cur = torch.cuda.current_stream(a.device).cuda_stream
                _raise(load_library().evcm_cuda_stream_wait(self._h, C.c_void_p(cur)))
                return

    def phase_stats(self):
        """PhaseStats (engine.hpp:63-66) of the last forward's warp / splat / loss
        and the last backward's phases."""
        t = (C.c_double * 4)()
        b = (C.c_size_t * 4)()
        _raise(load_library().evcm_cuda_phase_stats(self._h, t, b))
        return [PhaseStats(float(t[i]), int(b[i])) for i in range(4)]

    # -- Engine::forward (engine.hpp:145-183)
    def forward(self, slice_: EventSlice, flows: FlowSequence) -> ForwardResult:
        s, f = slice_._c(), flows._c()
        mem = _mem_of(slice_.events if slice_.n_events else None, flows.uv)
        self._order_after(slice_.events, flows.uv)
        loss = _Loss()
        self._generation += 1
        _raise(load_library().evcm_cuda_forward(self._h, C.byref(s), C.byref(f), mem,
                                                C.byref(loss)))
        return ForwardResult(self, self._generation,
                             LossResult(loss.value, bool(loss.no_survivors)),
                             (slice_.width, slice_.height, flows.n_bins, slice_.n_events),
                             int(loss.forward_id), self.phase_stats()[:3])

    # -- Engine::backward (engine.hpp:185-205)
    def backward(self, slice_: EventSlice, flows: FlowSequence, fwd: ForwardResult,
                 out=None) -> BackwardResult:
        fwd._check_live()
        s, f = slice_._c(), flows._c()
        mem = _mem_of(slice_.events if slice_.n_events else None, flows.uv)
        self._order_after(slice_.events, flows.uv, out)
        if out is None:
            if mem == MEM_DEVICE:
                import torch
                out = torch.empty((flows.n_bins, 2, slice_.height, slice_.width),
                                  dtype=torch.float64, device=flows.uv.device)
            else:
                out = np.zeros((flows.n_bins, 2, slice_.height, slice_.width))
        if _is_torch(out):
            import torch
            if out.dtype != torch.float64 or not out.is_contiguous() or \
                    tuple(out.shape) != (flows.n_bins, 2, slice_.height, slice_.width):
                raise DimensionMismatchError("backward: out must be a contiguous float64 "
                                             "[B, 2, H, W] tensor")
        _raise(load_library().evcm_cuda_backward_of(self._h, C.byref(s), C.byref(f), fwd._id, mem,
                                                    _ptr(out)))
        return BackwardResult(out, self.phase_stats()[3])

    # -- Engine::loss_and_grad (engine.hpp:208-213)
    def loss_and_grad(self, slice_: EventSlice, flows: FlowSequence):
        f = self.forward(slice_, flows)
        b = self.backward(slice_, flows, f)
        return f, b

    @staticmethod
    def validate_window(slice_: EventSlice, flows: FlowSequence) -> None:
        """Engine::validate_window (engine.hpp:215-222) on the host."""
        if slice_.width == 0 or slice_.height == 0:
            raise DimensionMismatchError("event slice: width and height must be positive")
        if slice_.t_end_us < slice_.t_start_us:
            raise TimeRangeError("event slice: t_end precedes t_start")
        ev = np.asarray(slice_.events)
        if len(ev):
            bad_xy = (ev["x"] >= slice_.width) | (ev["y"] >= slice_.height)
            bad_p = (ev["p"] != 1) & (ev["p"] != -1)
            bad_s = np.zeros(len(ev), bool)
            bad_s[1:] = ev["t_us"][1:] < ev["t_us"][:-1]
            bad_t = (ev["t_us"] < slice_.t_start_us) | (ev["t_us"] >= slice_.t_end_us)
            for k in np.flatnonzero(bad_xy | bad_p | bad_s | bad_t)[:1]:
                if bad_xy[k]:
                    raise CoordinateRangeError("event slice: coordinate outside the sensor")
                if bad_p[k]:
                    raise InvalidPolarityError("event slice: polarity must be +1 or -1")
                if bad_s[k]:
                    raise UnsortedEventsError("event slice: timestamps must be non-decreasing")
                raise TimeRangeError("event slice: timestamp outside the window")
        e = np.asarray(flows.edges_us)
        if flows.n_bins < 1:
            raise ConfigError("flow sequence: need B >= 1 fields and B+1 edges")
        if np.any(e[1:] <= e[:-1]):
            raise ConfigError("flow sequence: edges must be strictly increasing")
        if flows.width != slice_.width or flows.height != slice_.height:
            raise DimensionMismatchError("engine: flow shape differs from sensor shape")
        if int(e[0]) != slice_.t_start_us or int(e[-1]) != slice_.t_end_us:
            raise ConfigError("engine: flow bin edges do not span the slice window")

    # -- event ingestion (io.py)
    def validate_slice(self, slice_: EventSlice, check_window: bool = True) -> None:
        """EventSlice::validate (types.hpp:137-161) on the device; with
        ``check_window=False`` only read_events' record checks (io.hpp:123-144)."""
        s = slice_._c()
        mem = _mem_of(slice_.events if slice_.n_events else None)
        self._order_after(slice_.events)
        _raise(load_library().evcm_cuda_validate_slice(self._h, C.byref(s), int(check_window),
                                                       mem, None))

    def window_offsets(self, events, t0_us: int, window_us: int, n_windows: int) -> np.ndarray:
        """offsets[w] = first event with t_us >= t0 + w * window_us (w = 0..n_windows)
        over time-sorted events (numpy EVENT_DTYPE or a torch cuda [n, 16] uint8
        tensor): the ev_offsets of ``chain_batch``."""
        if not _is_torch(events):
            events = np.ascontiguousarray(events, EVENT_DTYPE)
        n = events.numel() // 16 if _is_torch(events) else len(events)
        self._order_after(events)
        offs = np.zeros(int(n_windows) + 1, np.uint64)
        _raise(load_library().evcm_cuda_window_offsets(
            self._h, _ptr(events) if n else None, n, int(t0_us), int(window_us), int(n_windows),
            _mem_of(events if n else None), offs.ctypes.data_as(C.c_void_p)))
        return offs

    # -- instrumentation
    def set_timing(self, on: bool = True):
        _raise(load_library().evcm_cuda_set_timing(self._h, int(on)))

    def stage_times_ms(self):
        buf = (C.c_double * 16)()
        n = load_library().evcm_cuda_stage_times(self._h, buf, 16)
        return list(buf[:n])

    def last_launch_count(self) -> int:
        return int(load_library().evcm_cuda_last_launch_count(self._h))

    def last_algo(self) -> str:
        return {0: "owner", 1: "atomic"}.get(load_library().evcm_cuda_last_algo(self._h), "?")

    def workspace_bytes(self) -> int:
        return int(load_library().evcm_cuda_workspace_bytes(self._h))

    # -- motion field (geometry.hpp:229-325)
    def depth_pose_to_flows(self, depth, poses, k, t_start_us, t_end_us, mask=None):
        return depth_pose_to_flows(depth, poses, k, t_start_us, t_end_us, mask=mask, engine=self)

    def depth_pose_to_flows_backward(self, depth, poses, k, flows, grad, mask=None):
        return depth_pose_to_flows_backward(depth, poses, k, flows, grad, mask=mask, engine=self)

    # -- batched chain (optimize.hpp:205-241 composition over many windows)
    def chain_batch(self, depth, poses, k, t_start_us, t_end_us, events, ev_offsets, out=None,
                    out_device=None, window_stride_us: int = 0, sums=None):
        """Per window w: depth_pose_to_flows(depth[w], poses[w]) -> forward ->
        backward -> depth_pose_to_flows_backward (the predictor_loss_and_gradients
        composition, optimize.hpp:205-241, without decode / L_geo).

        depth [n, H, W] f64, poses [n, B, 6] f64, events concatenated (evcm::Event
        records), ev_offsets [n+1] (host). Returns (loss [n], d_depth [n, H, W],
        d_poses [n, B, 6]). Inputs may be host (numpy / pinned torch) or device
        (torch cuda); outputs live on the device when ``out_device`` (default:
        same side as the inputs). Window w spans [t_start_us, t_end_us) +
        w * window_stride_us (0: one clock for all windows; the window length:
        consecutive windows of one stream, see io.slice_windows). ``sums`` (optional,
        same side as the outputs, 1 + H*W + B*6 float64): receives [sum_w loss,
        sum_w d_depth, sum_w d_poses] computed inside the chain (dist.py's payload)."""
        out, args = self._chain_args(depth, poses, k, t_start_us, t_end_us, events, ev_offsets,
                                     out, out_device, window_stride_us, sums)
        _raise(load_library().evcm_cuda_chain_batch2(self._h, *args))
        return out

    def chain_batch_async(self, depth, poses, k, t_start_us, t_end_us, events, ev_offsets, out,
                          slot: int, window_stride_us: int = 0, sums=None):
        """chain_batch that does not wait when it replays a captured graph (device
        inputs/outputs): the batch is queued on the engine's stream and its
        validation result is raised by ``chain_wait(slot)``. ``out`` (device
        tensors) must be given; slots 0..3 may be in flight together."""
        out, args = self._chain_args(depth, poses, k, t_start_us, t_end_us, events, ev_offsets,
                                     out, True, window_stride_us, sums)
        _raise(load_library().evcm_cuda_chain_batch_async(self._h, *args, int(slot)))
        return out

    def chain_wait(self, slot: int) -> None:
        """Waits for the batch queued on ``slot`` and raises its errors."""
        _raise(load_library().evcm_cuda_chain_wait(self._h, int(slot)))

    def _chain_args(self, depth, poses, k, t_start_us, t_end_us, events, ev_offsets, out,
                    out_device, window_stride_us, sums=None):
        nw, H, W = depth.shape
        B = poses.shape[1]
        in_mem = _mem_of(depth, poses, events)
        if out_device is None:
            out_device = in_mem == MEM_DEVICE
        out_mem = MEM_DEVICE if out_device else MEM_HOST
        K = k.as_array() if isinstance(k, CameraIntrinsics) else np.asarray(k, np.float64)
        offs = np.ascontiguousarray(ev_offsets, np.uint64)
        n_ev = events.numel() // 16 if _is_torch(events) else len(events)
        if offs.ndim != 1 or len(offs) != nw + 1:
            raise ConfigError(f"chain: ev_offsets needs n_windows + 1 = {nw + 1} entries")
        if offs[0] != 0 or np.any(offs[1:] < offs[:-1]):
            raise ConfigError("chain: ev_offsets must start at 0 and be non-decreasing")
        if int(offs[-1]) > n_ev:
            raise DimensionMismatchError(f"chain: ev_offsets end at {int(offs[-1])} but only "
                                         f"{n_ev} events were given")
        if tuple(poses.shape) != (nw, poses.shape[1], 6):
            raise DimensionMismatchError("chain: poses must be [n_windows, B, 6]")
        self._order_after(depth, poses, events)
        if out is None:
            if out_mem == MEM_DEVICE:
                import torch
                dev = depth.device if in_mem == MEM_DEVICE else torch.device("cuda", self.opts.device)
                out = (torch.empty(nw, dtype=torch.float64, device=dev),
                       torch.empty((nw, H, W), dtype=torch.float64, device=dev),
                       torch.empty((nw, B, 6), dtype=torch.float64, device=dev))
            else:
                out = (np.zeros(nw), np.zeros((nw, H, W)), np.zeros((nw, B, 6)))
        if in_mem == MEM_HOST:
            if not _is_torch(depth):
                depth = np.ascontiguousarray(depth, np.float64)
            if not _is_torch(poses):
                poses = np.ascontiguousarray(poses, np.float64)
            if not _is_torch(events):
                events = np.ascontiguousarray(events, EVENT_DTYPE)
        bt = _ChainBatch(nw, W, H, B, int(t_start_us), int(t_end_us), (C.c_double * 4)(*K),
                         _ptr(events), offs.ctypes.data_as(C.c_void_p), _ptr(depth), _ptr(poses),
                         int(window_stride_us))
        if sums is not None and (sums.shape[0] != 1 + H * W + B * 6 or
                                 _mem_of(sums) != out_mem):
            raise ConfigError("chain: sums must hold 1 + H*W + B*6 values on the output side")
        co = _ChainOut(_ptr(out[0]), None, _ptr(out[1]), _ptr(out[2]), _ptr(sums))
        # keep the (possibly converted) inputs alive until the call has enqueued them
        self._keep = (bt, co, offs, depth, poses, events, K, sums)
        return out, (C.byref(bt), in_mem, out_mem, C.byref(co))


# ---------------------------------------------------------------------------
# free functions (geometry.hpp, engine.hpp:606-631)

_default_engine = None


def default_engine() -> Engine:
    global _default_engine
    if _default_engine is None:
        _default_engine = Engine()
    return _default_engine


@dataclass
class GeometryFlows:
    flows: FlowSequence
    valid: object


def _k_array(k):
    return k.as_array() if isinstance(k, CameraIntrinsics) else np.ascontiguousarray(k, np.float64)


def depth_pose_to_flows(depth, poses, k, t_start_us, t_end_us, mask=None, engine=None):
    """depth_pose_to_flows (geometry.hpp:229-264). depth [H, W], poses [B, 6]."""
    e = engine or default_engine()
    mem = _mem_of(depth, poses, mask)
    e._order_after(depth, poses, mask)
    H, W = depth.shape
    B = poses.shape[0] if len(poses.shape) == 2 else len(poses) // 6
    if mem == MEM_HOST:
        depth = np.ascontiguousarray(depth, np.float64)
        poses = np.ascontiguousarray(poses, np.float64).reshape(-1, 6)
        mask = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        flows = np.zeros((B, 2, H, W))
        valid = np.zeros((B, H, W), np.uint8)
    else:
        import torch
        flows = torch.empty((B, 2, H, W), dtype=torch.float64, device=depth.device)
        valid = torch.empty((B, H, W), dtype=torch.uint8, device=depth.device)
    edges = np.zeros(B + 1, np.uint64)
    _raise(load_library().evcm_cuda_depth_pose_to_flows(
        e._h, W, H, _ptr(depth), _ptr(mask), B, _ptr(poses), _ptr(_k_array(k)), int(t_start_us),
        int(t_end_us), mem, _ptr(flows), _ptr(valid), _ptr(edges)))
    return GeometryFlows(FlowSequence(edges, flows), valid)


def depth_pose_to_flows_backward(depth, poses, k, flows: FlowSequence, grad, mask=None,
                                 engine=None):
    """depth_pose_to_flows_backward (geometry.hpp:279-325) -> (d_depth [H, W], d_poses [B, 6])."""
    e = engine or default_engine()
    mem = _mem_of(depth, poses, grad, mask)
    e._order_after(depth, poses, grad, mask)
    H, W = depth.shape
    B = flows.n_bins
    if grad.shape[0] != B or (len(poses.shape) == 2 and poses.shape[0] != B):
        raise ConfigError("flows backward: bins, poses, and gradients must align")
    if tuple(grad.shape[-2:]) != (H, W) or flows.width != W or flows.height != H:
        raise DimensionMismatchError("flows backward: grids must match the depth map")
    if mem == MEM_HOST:
        depth = np.ascontiguousarray(depth, np.float64)
        poses = np.ascontiguousarray(poses, np.float64).reshape(-1, 6)
        grad = np.ascontiguousarray(grad, np.float64)
        mask = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        dd, dp = np.zeros((H, W)), np.zeros((B, 6))
    else:
        import torch
        dd = torch.empty((H, W), dtype=torch.float64, device=depth.device)
        dp = torch.empty((B, 6), dtype=torch.float64, device=depth.device)
    edges = np.ascontiguousarray(flows.edges_us, np.uint64)
    _raise(load_library().evcm_cuda_depth_pose_to_flows_backward(
        e._h, W, H, _ptr(depth), _ptr(mask), B, _ptr(poses), _ptr(_k_array(k)), _ptr(edges),
        _ptr(grad), mem, _ptr(dd), _ptr(dp)))
    return dd, dp


def build_iwe_stack(slice_: EventSlice, flows: FlowSequence, opts: Optional[EngineOptions] = None):
    """build_iwe_stack (engine.hpp:606-609)."""
    return Engine(opts).forward(slice_, flows) if opts else default_engine().forward(slice_, flows)


def contrast_loss_backward(slice_: EventSlice, flows: FlowSequence,
                           opts: Optional[EngineOptions] = None):
    """contrast_loss_backward (engine.hpp:611-617) -> grad [B, 2, H, W]."""
    e = Engine(opts) if opts else default_engine()
    f = e.forward(slice_, flows)
    return e.backward(slice_, flows, f).grad


def rsat(slice_: EventSlice, flows: FlowSequence, opts: Optional[EngineOptions] = None) -> float:
    """rsat (engine.hpp:621-631)."""
    if slice_.n_events == 0:
        raise EmptySliceError("rsat: no events in slice")
    e = Engine(opts) if opts else default_engine()
    with_flow = e.forward(slice_, flows).loss.value
    base = e.forward(slice_, flows.zeros_like()).loss
    if base.no_survivors or base.value == 0.0:
        raise EmptySliceError("rsat: zero-flow loss is zero")
    return with_flow / base.value
