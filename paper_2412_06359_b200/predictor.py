"""The predictor decode chain on the device — the caller
of the CMax path — mirroring the reference's names and semantics:

  DirectPredictor, DecodedPredictor, decode          predictor.hpp:100-131
  PredictorGrads, accumulate_gradients               predictor.hpp:133-173
  save_predictor, load_predictor (checkpoints)      predictor.hpp:175-218
  OptimizerConfig (Adam fields), Adam                optimize.hpp:25-75, 115-134
  WindowGradients, predictor_loss_and_gradients      optimize.hpp:195-241 (with L_geo)

Everything runs through libevcm_cuda.so (evcm_cuda_decode / _decode_backward /
_adam_step / _predictor_loss_and_gradients_geo); there is no CPU fallback. Arrays
may be numpy (host) or torch CUDA tensors (device, kept on the device)."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from .engine import (MEM_DEVICE, MEM_HOST, CameraIntrinsics, ConfigError, Engine, EventSlice,
                     FlowSequence, _is_torch, _k_array, _mem_of, _ptr, _raise, default_engine,
                     depth_pose_to_flows_backward, load_library)


def _zeros_like_side(ref, shape):
    if _is_torch(ref) and ref.is_cuda:
        import torch
        return torch.zeros(shape, dtype=torch.float64, device=ref.device)
    return np.zeros(shape)


def _f64(a):
    return a if _is_torch(a) else np.ascontiguousarray(a, np.float64)


@dataclass
class DirectPredictor:
    """predictor.hpp:100-120: low-resolution unconstrained depth parameters
    [ph][pw] decoded through softplus and x`upsample` bilinear upsampling, plus
    one 6-dof pose {omega, trans} per flow bin [B][6]."""
    depth_params: object
    poses: object
    upsample: int = 8

    @property
    def full_width(self) -> int:
        return int(self.depth_params.shape[1]) * self.upsample

    @property
    def full_height(self) -> int:
        return int(self.depth_params.shape[0]) * self.upsample

    @property
    def n_bins(self) -> int:
        return int(self.poses.shape[0])

    @property
    def n_parameters(self) -> int:
        return int(self.depth_params.shape[0] * self.depth_params.shape[1]) + 6 * self.n_bins

    def validate(self) -> None:  # predictor.hpp:109-119 (pose checks: PoseStep::validate)
        if self.depth_params.shape[0] == 0 or self.depth_params.shape[1] == 0:
            raise ConfigError("predictor: empty depth grid")
        if self.n_bins == 0:
            raise ConfigError("predictor: need one pose per bin")
        if self.upsample < 1:
            raise ConfigError("predictor: upsample factor must be >= 1")
        p = self.depth_params.cpu().numpy() if _is_torch(self.depth_params) else self.depth_params
        if not np.all(np.isfinite(p)):
            raise ConfigError("predictor: non-finite depth parameter")
        q = self.poses.cpu().numpy() if _is_torch(self.poses) else np.asarray(self.poses)
        for row in np.asarray(q, np.float64).reshape(-1, 6):  # PoseStep::validate (types.hpp:362-368)
            if not (np.sqrt(row[0] * row[0] + row[1] * row[1] + row[2] * row[2]) < np.pi):
                raise ConfigError("pose step: rotation angle must stay below pi")
            if not np.all(np.isfinite(row)):
                raise ConfigError("pose step: non-finite component")


@dataclass
class DecodedPredictor:
    depth: object  # [H][W], all valid
    poses: object


@dataclass
class PredictorGrads:
    d_depth_params: object
    d_poses: object


@dataclass
class WindowGradients:
    grads: PredictorGrads
    l_cm: float = 0.0
    l_geo: float = 0.0
    total: float = 0.0


def decode(pred: DirectPredictor, engine: Engine | None = None) -> DecodedPredictor:
    """decode (predictor.hpp:126-131) on the device."""
    pred.validate()
    e = engine or default_engine()
    params = _f64(pred.depth_params)
    ph, pw = params.shape
    mem = _mem_of(params)
    depth = _zeros_like_side(params, (ph * pred.upsample, pw * pred.upsample))
    e._order_after(params)
    _raise(load_library().evcm_cuda_decode(e._h, pw, ph, pred.upsample, _ptr(params), mem,
                                           _ptr(depth)))
    return DecodedPredictor(depth, pred.poses)


def accumulate_gradients(pred: DirectPredictor, decoded_depth, k, flows: FlowSequence, flow_grads,
                         extra_d_depth=None, extra_d_poses=None,
                         engine: Engine | None = None) -> PredictorGrads:
    """accumulate_gradients (predictor.hpp:143-173): flow-cell gradients through
    depth_pose_to_flows_backward, optional extra depth / pose terms, then the
    upsampling transpose and softplus derivative (on the device)."""
    e = engine or default_engine()
    d_depth, d_poses = depth_pose_to_flows_backward(decoded_depth, pred.poses, k, flows, flow_grads,
                                                    engine=e)
    if extra_d_depth is not None:
        if tuple(extra_d_depth.shape) != tuple(d_depth.shape):
            from .engine import DimensionMismatchError
            raise DimensionMismatchError("gradients: extra depth term shape mismatch")
        d_depth = d_depth + extra_d_depth
    params = _f64(pred.depth_params)
    ph, pw = params.shape
    mem = _mem_of(params, d_depth)
    out = _zeros_like_side(params, (ph, pw))
    e._order_after(params, d_depth)
    _raise(load_library().evcm_cuda_decode_backward(e._h, pw, ph, pred.upsample, _ptr(params),
                                                    _ptr(_f64(d_depth)), mem, _ptr(out)))
    if extra_d_poses is not None:
        if extra_d_poses.shape[0] != d_poses.shape[0]:
            raise ConfigError("gradients: extra pose term count mismatch")
        d_poses = d_poses + extra_d_poses
    return PredictorGrads(out, d_poses)


def predictor_loss_and_gradients(pred: DirectPredictor, slice_: EventSlice, k, lambda_geo=0.0,
                                 engine: Engine | None = None) -> WindowGradients:
    """predictor_loss_and_gradients (optimize.hpp:205-241) in one fused device
    call: decode -> depth_pose_to_flows -> Engine::forward -> Engine::backward ->
    [lambda_geo > 0: L_geo per bin on (depth, depth), upstream lambda_geo / B] ->
    accumulate_gradients."""
    pred.validate()
    e = engine or default_engine()
    params = _f64(pred.depth_params)
    poses = _f64(pred.poses)
    ph, pw = params.shape
    if slice_.width != pw * pred.upsample or slice_.height != ph * pred.upsample:
        from .engine import DimensionMismatchError
        raise DimensionMismatchError("predictor: decoded depth does not match the slice sensor")
    mem = _mem_of(params, poses, slice_.events)
    losses = _zeros_like_side(params, (3,))
    dpar = _zeros_like_side(params, (ph, pw))
    dpos = _zeros_like_side(params, (pred.n_bins, 6))
    sl = slice_._c()
    e._order_after(params, poses, slice_.events)
    _raise(load_library().evcm_cuda_predictor_loss_and_gradients_geo(
        e._h, pw, ph, pred.upsample, _ptr(params), pred.n_bins, _ptr(poses),
        _ptr(_k_array(k)), C.byref(sl), float(lambda_geo), mem, _ptr(losses), _ptr(dpar),
        _ptr(dpos)))
    l = [float(v) for v in losses.tolist()]
    return WindowGradients(PredictorGrads(dpar, dpos), l[0], l[1], l[2])


@dataclass
class OptimizerConfig:
    """OptimizerConfig (optimize.hpp:25-75): the fields the device loops use
    (Adam, stopping, divergence and FD spot-check controls)."""
    learning_rate: float = 1e-4
    steps_per_update: int = 10
    bins: int = 10
    max_updates: int = 100
    lambda_geo: float = 0.05  # kGeoWeightDefault (geometry.hpp:538)
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    seed: int = 1
    fd_check_every: int = 0
    fd_check_tolerance: float = 0.05
    divergence_factor: float = 10.0
    grad_stop_tolerance: float = 1e-10

    def validate(self) -> None:  # optimize.hpp:43-61
        if not (self.learning_rate > 0.0) or not math.isfinite(self.learning_rate):
            raise ConfigError("optimizer: learning_rate must be positive")
        if self.steps_per_update < 1:
            raise ConfigError("optimizer: steps_per_update must be >= 1")
        if self.bins < 1:
            raise ConfigError("optimizer: bins must be >= 1")
        if self.max_updates < 0:
            raise ConfigError("optimizer: max_updates must be >= 0")
        if not (self.lambda_geo >= 0.0) or not math.isfinite(self.lambda_geo):
            raise ConfigError("optimizer: lambda_geo must be >= 0")
        if not (0.0 <= self.adam_beta1 < 1.0) or not (0.0 <= self.adam_beta2 < 1.0):
            raise ConfigError("optimizer: adam betas must lie in [0, 1)")
        if not self.adam_eps > 0.0:
            raise ConfigError("optimizer: adam_eps must be positive")
        if self.fd_check_every < 0:
            raise ConfigError("optimizer: fd_check_every must be >= 0")
        if not self.divergence_factor > 1.0:
            raise ConfigError("optimizer: divergence_factor must exceed 1")
        if not self.grad_stop_tolerance >= 0.0:
            raise ConfigError("optimizer: grad_stop_tolerance must be >= 0")


class Adam:
    """Adam (optimize.hpp:115-134) on the device: moment buffers live next to the
    parameters (host numpy or device torch), state persists across steps."""

    def __init__(self, n: int, like=None):
        self.t = 0
        self.m = _zeros_like_side(like, (n,)) if like is not None else np.zeros(n)
        self.v = _zeros_like_side(like, (n,)) if like is not None else np.zeros(n)

    def step(self, slots, grads, cfg: OptimizerConfig, engine: Engine | None = None) -> None:
        """slots -= lr * m_hat / (sqrt(v_hat) + eps), in place (flat f64 vectors)."""
        cfg.validate()
        e = engine or default_engine()
        self.t += 1
        n = int(slots.shape[0])
        mem = _mem_of(slots, grads, self.m)
        e._order_after(slots, grads)
        _raise(load_library().evcm_cuda_adam_step(
            e._h, n, _ptr(slots), _ptr(_f64(grads)), _ptr(self.m), _ptr(self.v), self.t,
            cfg.learning_rate, cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps, mem))


# ---- checkpoints (predictor.hpp:175-218): depth parameters as PFM (float32), poses
# and the upsample factor as CSV; host files, nothing on the device


def save_predictor(pred: DirectPredictor, params_pfm, poses_csv) -> None:
    """save_predictor (predictor.hpp:178-193)."""
    from .io import format_number, write_pfm
    pred.validate()
    params = pred.depth_params.cpu().numpy() if _is_torch(pred.depth_params) else pred.depth_params
    poses = pred.poses.cpu().numpy() if _is_torch(pred.poses) else np.asarray(pred.poses)
    write_pfm(np.asarray(params, np.float64).astype(np.float32), params_pfm)
    lines = ["bin,upsample,wx,wy,wz,tx,ty,tz"]
    for i, p in enumerate(np.asarray(poses, np.float64).reshape(-1, 6)):
        lines.append(",".join([str(i), str(pred.upsample)] + [format_number(v) for v in p]))
    try:
        with open(poses_csv, "w", newline="") as f:
            f.write("\n".join(lines) + "\n")
    except OSError as e:
        from .engine import IoError
        raise IoError(f"cannot open {poses_csv} for writing: {e}") from None


def _stoi(tok: str) -> int:  # std::stoi: leading whitespace, sign, digits prefix
    import re
    m = re.match(r"\s*[+-]?[0-9]+", tok)
    if not m:
        from .engine import Error
        raise Error(f"stoi: no conversion of '{tok}'")
    return int(m.group(0))


def _stod(tok: str) -> float:  # std::stod: the longest valid prefix
    from .io import _strtod
    import re
    if not re.match(r"\s*[+-]?(?:[0-9]|\.[0-9]|inf|nan)", tok, re.IGNORECASE):
        from .engine import Error
        raise Error(f"stod: no conversion of '{tok}'")
    return _strtod(tok.lstrip())


def load_predictor(params_pfm, poses_csv) -> DirectPredictor:
    """load_predictor (predictor.hpp:195-218)."""
    from .io import read_csv, read_pfm
    params = read_pfm(params_pfm).astype(np.float64)
    rows = read_csv(poses_csv)
    if len(rows) < 2 or len(rows[0]) != 8:
        raise ConfigError("predictor checkpoint: malformed pose table")
    upsample = 0
    poses = []
    for r in rows[1:]:
        if len(r) != 8:
            raise ConfigError("predictor checkpoint: malformed pose row")
        factor = _stoi(r[1])
        if upsample == 0:
            upsample = factor
        elif factor != upsample:
            raise ConfigError("predictor checkpoint: inconsistent upsample factor")
        poses.append([_stod(c) for c in r[2:8]])
    pred = DirectPredictor(params, np.array(poses, np.float64), upsample)
    pred.validate()
    return pred
