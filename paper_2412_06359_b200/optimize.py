"""Device-resident optimization loops over the CMax path,
mirroring optimize.hpp:

  TrainRecord, TrainLog            optimize.hpp:77-111
  FlowOnlyResult,
  optimize_flow_only               optimize.hpp:376-487: Adam over the dense per-bin
                                   flow field from zero flow, best iterate kept

The flow field, its gradient and the Adam moments stay on the GPU for the whole
run; each update is Engine::forward + Engine::backward (C-ABI) and one device
Adam step. Only the per-update scalars come back to the host."""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .engine import (DivergenceError, EmptySliceError, Engine, EngineOptions, Error, EventSlice,
                     FlowSequence, make_edges)
from .predictor import Adam, OptimizerConfig


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


@dataclass
class FlowOnlyResult:
    flows: FlowSequence
    log: TrainLog


def _fmt(x: float) -> str:
    return repr(float(x))


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
