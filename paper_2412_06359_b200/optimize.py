"""Device-resident optimization loops over the CMax path,
mirroring optimize.hpp:

  TrainRecord, TrainLog            optimize.hpp:77-111
  predictor_total_loss             optimize.hpp:177-193
  RunResult, run_window            optimize.hpp:288-375: Adam over the predictor's
                                   parameters across a sequence of windows
  FlowOnlyResult,
  optimize_flow_only               optimize.hpp:376-487: Adam over the dense per-bin
                                   flow field from zero flow, best iterate kept

The parameters, their gradients and the Adam moments stay on the GPU for the
whole run; each update is one fused device call (predictor_loss_and_gradients,
or Engine::forward + Engine::backward for flow-only) and one device Adam step.
Only the per-update scalars come back to the host."""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .engine import (ConfigError, DimensionMismatchError, DivergenceError, EmptySliceError, Engine,
                     EngineOptions, Error, EventSlice, FlowSequence, _is_torch, depth_pose_to_flows,
                     make_edges)
from .geo import geometry_consistency_loss_batch
from .io import format_number
from .predictor import Adam, DirectPredictor, OptimizerConfig, decode, predictor_loss_and_gradients


@dataclass
class TrainRecord:
    update: int = 0
    l_cm: float = 0.0
    l_geo: float = 0.0
    total: float = 0.0
    rsat: float = 0.0
    grad_norm_depth: float = 0.0  # flow-field gradient norm in flow-only runs
    grad_norm_pose: float = 0.0
    wall_ms: float = 0.0


@dataclass
class TrainLog:
    records: List[TrainRecord] = field(default_factory=list)

    def write_csv(self, path, include_timings: bool = False) -> None:
        """TrainLog::write_csv (optimize.hpp:92-110): format_number cells, timings opt-in."""
        cols = ["update", "l_cm", "l_geo", "total", "rsat", "grad_norm_depth", "grad_norm_pose"]
        if include_timings:
            cols.append("wall_ms")
        try:
            with open(path, "w", newline="") as f:
                f.write(",".join(cols) + "\n")
                for r in self.records:
                    row = [str(r.update)] + [format_number(x) for x in (
                        r.l_cm, r.l_geo, r.total, r.rsat, r.grad_norm_depth, r.grad_norm_pose)]
                    if include_timings:
                        row.append(format_number(r.wall_ms))
                    f.write(",".join(row) + "\n")
        except OSError as e:
            from .engine import IoError
            raise IoError(f"cannot open {path} for writing: {e}") from None


@dataclass
class RunResult:
    predictor: DirectPredictor
    log: TrainLog


@dataclass
class FlowOnlyResult:
    flows: FlowSequence
    log: TrainLog


def _fmt(x: float) -> str:
    return repr(float(x))


def predictor_total_loss(pred: DirectPredictor, slice_: EventSlice, k, lambda_geo: float,
                         engine: Engine) -> float:
    """predictor_total_loss (optimize.hpp:177-193): the contrast loss under the
    decoded flows plus lambda_geo times the mean per-bin L_geo (all on the device)."""
    dec = decode(pred, engine)
    geo = depth_pose_to_flows(dec.depth, dec.poses, k, slice_.t_start_us, slice_.t_end_us,
                              engine=engine)
    total = engine.forward(slice_, geo.flows).loss.value
    if lambda_geo > 0.0:
        b = geometry_consistency_loss_batch(dec.depth, dec.depth, dec.poses, k, want_grad=False,
                                            engine=engine)
        s = 0.0
        for v in b.value.tolist():  # sequential, as the reference sums
            s += v
        total += lambda_geo * s / float(pred.n_bins)
    return total


def _window_zero_flow_loss(slice_: EventSlice, bins: int, engine: Engine) -> float:
    """detail::window_zero_flow_loss (optimize.hpp:278-284)."""
    zero = FlowSequence.zeros(slice_.width, slice_.height, slice_.t_start_us, slice_.t_end_us, bins)
    if _is_torch(slice_.events):
        import torch
        zero = FlowSequence(zero.edges_us, torch.zeros(zero.uv.shape, dtype=torch.float64,
                                                       device=slice_.events.device))
    base = engine.forward(slice_, zero).loss
    return 0.0 if (base.no_survivors or not base.value > 0.0) else base.value


def run_window(windows, pred: DirectPredictor, k, cfg: OptimizerConfig,
               engine: Engine | None = None) -> RunResult:
    """run_window (optimize.hpp:297-375) on the device: the stream advances one
    window after every max(1, bins / steps_per_update) updates; once exhausted,
    the final window keeps receiving updates until the budget runs out.
    Parameters and Adam state carry across windows (warm start). The returned
    predictor holds numpy arrays when the input did, torch CUDA tensors otherwise.

    The FD spot check (fd_check_every > 0) probes 3 random parameters per check
    like detail::spot_check_predictor_gradients (optimize.hpp:247-276); the
    probed indices come from numpy's generator, not std::mt19937_64."""
    import torch

    cfg.validate()
    pred.validate()
    if pred.n_bins != cfg.bins:
        raise ConfigError("optimizer: predictor must carry exactly one pose per bin")
    e = engine or Engine(EngineOptions())
    dev = torch.device("cuda", e.opts.device)
    live = []
    for w in windows:
        if w.n_events == 0:
            continue  # nothing to learn from; never triggers an update
        e.validate_slice(w)
        if w.width != pred.full_width or w.height != pred.full_height:
            raise DimensionMismatchError("optimizer: window resolution must match the predictor")
        ev = w.events
        if not (_is_torch(ev) and ev.is_cuda):  # each window's events uploaded once
            ev = torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).copy()).to(dev)
        live.append(EventSlice(w.width, w.height, w.t_start_us, w.t_end_us, ev))
    host_in = not _is_torch(pred.depth_params)

    def result(p_params, p_poses):
        if host_in:
            return DirectPredictor(np.asarray(p_params.cpu().numpy() if _is_torch(p_params)
                                              else p_params, np.float64).copy(),
                                   np.asarray(p_poses.cpu().numpy() if _is_torch(p_poses)
                                              else p_poses, np.float64).copy(), pred.upsample)
        return DirectPredictor(p_params.clone(), p_poses.clone(), pred.upsample)

    if not live or cfg.max_updates == 0:
        return RunResult(result(pred.depth_params, pred.poses), TrainLog())

    # one flat parameter vector in predictor_slots order (optimize.hpp:138-151):
    # depth params row-major, then per pose omega xyz, trans xyz
    ph, pw = pred.depth_params.shape
    n_depth = ph * pw
    src_p = torch.as_tensor(pred.depth_params, dtype=torch.float64)
    src_q = torch.as_tensor(pred.poses, dtype=torch.float64)
    slots = torch.cat([src_p.reshape(-1).to(dev), src_q.reshape(-1).to(dev)])
    cur = DirectPredictor(slots[:n_depth].view(ph, pw), slots[n_depth:].view(-1, 6), pred.upsample)
    adam = Adam(slots.numel(), like=slots)
    updates_per_window = max(1, cfg.bins // cfg.steps_per_update)
    window_index = 0
    spent = 0
    zero_loss = _window_zero_flow_loss(live[0], cfg.bins, e)
    initial_total = 0.0
    log = TrainLog()
    for u in range(cfg.max_updates):
        if spent >= updates_per_window and window_index + 1 < len(live):
            window_index += 1
            spent = 0
            zero_loss = _window_zero_flow_loss(live[window_index], cfg.bins, e)
        sl = live[window_index]
        t0 = time.perf_counter()
        wg = predictor_loss_and_gradients(cur, sl, k, cfg.lambda_geo, e)
        if not math.isfinite(wg.total):
            raise DivergenceError(f"optimizer: non-finite loss at update {u}")
        if u == 0:
            initial_total = wg.total
        elif initial_total > 0.0 and wg.total > cfg.divergence_factor * initial_total:
            raise DivergenceError(f"optimizer: loss {format_number(wg.total)} exceeds "
                                  f"{format_number(cfg.divergence_factor)}x initial "
                                  f"{format_number(initial_total)} at update {u}")
        flat = torch.cat([wg.grads.d_depth_params.reshape(-1), wg.grads.d_poses.reshape(-1)])
        norms = torch.stack([flat.abs().max(), torch.linalg.vector_norm(flat[:n_depth]),
                             torch.linalg.vector_norm(flat[n_depth:])]).tolist()
        if norms[0] < cfg.grad_stop_tolerance:
            break  # converged to machine precision
        if cfg.fd_check_every > 0 and u % cfg.fd_check_every == 0:
            _spot_check(cur, slots, flat, n_depth, sl, k, cfg, e, u)
        adam.step(slots, flat, cfg, e)
        t1 = time.perf_counter()
        log.records.append(TrainRecord(
            update=u, l_cm=wg.l_cm, l_geo=wg.l_geo, total=wg.total,
            rsat=wg.l_cm / zero_loss if zero_loss > 0.0 else 1.0,
            grad_norm_depth=norms[1], grad_norm_pose=norms[2], wall_ms=(t1 - t0) * 1e3))
        spent += 1
    return RunResult(result(cur.depth_params, cur.poses), log)


def _spot_check(cur, slots, analytic, n_depth, sl, k, cfg, e, u):
    """detail::spot_check_predictor_gradients (optimize.hpp:247-276)."""
    rng = np.random.default_rng(cfg.seed * 31 + u)
    for _ in range(3):
        i = int(rng.integers(0, slots.numel()))
        h = 1e-5 if i < n_depth else 1e-6
        saved = float(slots[i])
        slots[i] = saved + h
        lp = predictor_total_loss(cur, sl, k, cfg.lambda_geo, e)
        slots[i] = saved - h
        lm = predictor_total_loss(cur, sl, k, cfg.lambda_geo, e)
        slots[i] = saved
        fd = (lp - lm) / (2.0 * h)
        a = float(analytic[i])
        scale = max(1.0, abs(fd), abs(a))
        if abs(a - fd) > cfg.fd_check_tolerance * scale:
            raise Error(f"gradient spot check failed at update {u}, parameter {i}: analytic "
                        f"{format_number(a)} vs finite difference {format_number(fd)}")


def optimize_flow_only(slice_: EventSlice, n_bins: int, cfg: OptimizerConfig,
                       engine: Engine | None = None) -> FlowOnlyResult:
    """optimize_flow_only (optimize.hpp:385-487) on the device."""
    import torch

    cfg.validate()
    if slice_.n_events == 0:
        raise EmptySliceError("flow optimization: slice has no events")
    Engine.validate_window(slice_, FlowSequence.zeros(slice_.width, slice_.height,
                                                      slice_.t_start_us, slice_.t_end_us, n_bins))
    e = engine or Engine(EngineOptions())
    dev = torch.device("cuda", e.opts.device)
    ev = slice_.events
    if not (hasattr(ev, "is_cuda") and ev.is_cuda):  # events uploaded once for the run
        ev = torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).copy()).to(dev)
    sl = EventSlice(slice_.width, slice_.height, slice_.t_start_us, slice_.t_end_us, ev)
    edges = make_edges(slice_.t_start_us, slice_.t_end_us, n_bins)
    uv = torch.zeros((n_bins, 2, slice_.height, slice_.width), dtype=torch.float64, device=dev)
    flows = FlowSequence(edges, uv)
    grad = torch.empty_like(uv)
    flat, gflat = uv.view(-1), grad.view(-1)  # slot order of optimize.hpp:398-401: per bin u then v
    adam = Adam(flat.numel(), like=flat)

    best = uv.clone()  # the zero-flow iterate is the starting best
    best_loss = math.inf
    zero_loss = 0.0
    initial_total = 0.0
    log = TrainLog()
    for u in range(cfg.max_updates):
        t0 = time.perf_counter()
        fwd = e.forward(sl, flows)
        loss = fwd.loss.value
        if not math.isfinite(loss):
            raise DivergenceError(f"flow optimization: non-finite loss at update {u}")
        if u == 0:
            initial_total = loss
            zero_loss = 0.0 if (fwd.loss.no_survivors or not loss > 0.0) else loss
        elif initial_total > 0.0 and loss > cfg.divergence_factor * initial_total:
            raise DivergenceError(f"flow optimization: loss {_fmt(loss)} exceeds "
                                  f"{_fmt(cfg.divergence_factor)}x initial {_fmt(initial_total)} "
                                  f"at update {u}")
        if loss < best_loss:
            best_loss = loss
            best.copy_(uv)
        e.backward(sl, flows, fwd, out=grad)
        grad_inf = float(gflat.abs().max())
        if grad_inf < cfg.grad_stop_tolerance:
            break  # converged to machine precision
        if cfg.fd_check_every > 0 and u % cfg.fd_check_every == 0:
            rng = np.random.default_rng(cfg.seed * 31 + u)
            for _ in range(3):
                i = int(rng.integers(0, flat.numel()))
                h = 1e-4
                saved = float(flat[i])
                flat[i] = saved + h
                lp = e.forward(sl, flows).loss.value
                flat[i] = saved - h
                lm = e.forward(sl, flows).loss.value
                flat[i] = saved
                fd = (lp - lm) / (2.0 * h)
                gi = float(gflat[i])
                scale = max(1.0, abs(fd), abs(gi))
                if abs(gi - fd) > cfg.fd_check_tolerance * scale:
                    raise Error(f"gradient spot check failed at update {u}, flow cell {i}: "
                                f"analytic {_fmt(gi)} vs finite difference {_fmt(fd)}")
        adam.step(flat, gflat, cfg, e)
        t1 = time.perf_counter()
        log.records.append(TrainRecord(
            update=u, l_cm=loss, l_geo=0.0, total=loss,
            rsat=loss / zero_loss if zero_loss > 0.0 else 1.0,
            grad_norm_depth=float(torch.linalg.vector_norm(gflat)), grad_norm_pose=0.0,
            wall_ms=(t1 - t0) * 1e3))
    if cfg.max_updates > 0:  # the loop logs pre-step losses only
        last = e.forward(sl, flows).loss.value
        if math.isfinite(last) and last < best_loss:
            best.copy_(uv)
    return FlowOnlyResult(FlowSequence(edges, best), log)
