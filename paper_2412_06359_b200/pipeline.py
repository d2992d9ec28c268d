"""Pipelined host -> device feeding of the batched chain (Engine.chain_batch).

A training or serving loop that receives its event batches in host memory pays
the PCIe copy of every batch (16 B per event plus the depth maps and poses).
``ChainPipeline`` hides it behind the compute of the previous batch: two device
input buffer sets, a copy stream that stages batch i+1 (pinned host -> device)
while the engine stream runs batch i, and an event that makes batch i+1's
compute wait for its own copy. Each batch still returns its result to the host
(the caller's ``post`` reduction, read back every step). The engine caches one
CUDA graph per input buffer set, so both alternating calls replay graphs, and
the calls are asynchronous (Engine.chain_batch_async): batch i+1 is already
queued on the GPU while the host waits for batch i's result, so the device
never idles between batches.
"""
from __future__ import annotations

from typing import Callable, Iterable, Iterator, Optional

import numpy as np

from .engine import ConfigError, Engine, _is_torch


class ChainPipeline:
    """Double-buffered ``chain_batch`` over a stream of host batches.

    ``engine`` must run on an explicit CUDA stream (EngineOptions(stream=...));
    ``compute_stream`` (default: that stream wrapped for torch) must be the
    engine's stream: it carries the waits for the staged copies and the result
    read-back."""

    def __init__(self, engine: Engine, compute_stream=None):
        import torch
        self.engine = engine
        self.dev = torch.device("cuda", engine.opts.device)
        if engine.opts.stream is None:
            raise ConfigError("ChainPipeline: the engine needs an explicit stream "
                              "(EngineOptions(stream=torch_stream.cuda_stream))")
        if compute_stream is None:
            compute_stream = torch.cuda.ExternalStream(engine.opts.stream, device=self.dev)
        elif compute_stream.cuda_stream != engine.opts.stream:
            # the engine's kernels must wait for the staged copies: one stream
            raise ConfigError("ChainPipeline: compute_stream must be the engine's stream")
        self.compute = compute_stream
        self.copy = torch.cuda.Stream(self.dev)
        self.sets = [None, None]
        self.copied = [torch.cuda.Event(), torch.cuda.Event()]
        self.out = None

    def _stage(self, slot: int, depth, poses, events):
        import torch
        cur = self.sets[slot]
        if cur is None or cur[0].shape != depth.shape or cur[1].shape != poses.shape or \
                cur[2].shape != events.shape:
            cur = (torch.empty(depth.shape, dtype=torch.float64, device=self.dev),
                   torch.empty(poses.shape, dtype=torch.float64, device=self.dev),
                   torch.empty(events.shape, dtype=torch.uint8, device=self.dev))
            self.sets[slot] = cur
        with torch.cuda.stream(self.copy):
            cur[0].copy_(depth, non_blocking=True)
            cur[1].copy_(poses, non_blocking=True)
            cur[2].copy_(events, non_blocking=True)
            self.copied[slot].record(self.copy)
        return cur

    def run(self, batches: Iterable, k, t_start_us: int, t_end_us: int,
            post: Optional[Callable] = None,
            window_stride_us: int = 0, window_sums: bool = False) -> Iterator:
        """For each host batch ``(depth [n,H,W] f64, poses [n,B,6] f64, events
        uint8 [N,16], ev_offsets [n+1])`` -- pinned torch CPU tensors -- run the
        chain and yield the host result: ``post(loss, d_depth, d_poses)`` (a
        device tensor, e.g. a data-parallel reduction) copied into a pinned host
        buffer owned by the pipeline (valid until two batches later), or the
        three outputs copied to the host when ``post`` is None. With
        ``window_sums`` the chain also writes the packed [sum loss, sum d_depth,
        sum d_poses] payload (Engine.chain_batch ``sums``) and ``post(sums)``
        (default: the payload itself) is what comes back. A batch's validation
        error is raised when its result is collected."""
        import torch
        it = iter(batches)
        cur = next(it, None)
        if cur is None:
            return
        for a in cur[:3]:
            if not (_is_torch(a) and not a.is_cuda):
                raise ConfigError("ChainPipeline: batches must be host (pinned) torch tensors")
        if not hasattr(self, "consumed"):
            self.consumed = [torch.cuda.Event(), torch.cuda.Event()]
            self.done = [torch.cuda.Event(), torch.cuda.Event()]
            self.host = [None, None]
        staged = self._stage(0, *cur[:3])
        slot = 0
        prev = None  # (slot, host result) of the batch queued before this one

        def finish(p):
            self.engine.chain_wait(p[0])  # raises the batch's validation errors
            self.done[p[0]].synchronize()  # its result is in host memory
            return p[1]

        queued = []  # slots with a batch in flight
        try:
            while cur is not None:
                nxt = next(it, None)
                if nxt is not None:  # batch i+1 copies while batch i computes
                    self.copy.wait_event(self.consumed[1 - slot])  # batch i-1 read that set
                    staged_next = self._stage(1 - slot, *nxt[:3])
                self.compute.wait_event(self.copied[slot])
                nw = staged[0].shape[0]
                if self.out is None or self.out[1].shape != staged[0].shape or \
                        self.out[2].shape != staged[1].shape:
                    self.out = (torch.empty(nw, dtype=torch.float64, device=self.dev),
                                torch.empty(tuple(staged[0].shape), dtype=torch.float64,
                                            device=self.dev),
                                torch.empty(tuple(staged[1].shape), dtype=torch.float64,
                                            device=self.dev))
                if window_sums:
                    H, W, B = staged[0].shape[1], staged[0].shape[2], staged[1].shape[1]
                    n_s = 1 + H * W + B * 6
                    if getattr(self, "sums", None) is None or self.sums.shape[0] != n_s:
                        self.sums = torch.empty(n_s, dtype=torch.float64, device=self.dev)
                with torch.cuda.stream(self.compute):
                    self.engine.chain_batch_async(staged[0], staged[1], k, t_start_us, t_end_us,
                                                  staged[2], np.asarray(cur[3], np.uint64),
                                                  self.out, slot,
                                                  window_stride_us=window_stride_us,
                                                  sums=self.sums if window_sums else None)
                    queued.append(slot)
                    self.consumed[slot].record(self.compute)
                    if window_sums or post is not None:
                        if window_sums:
                            r = post(self.sums) if post is not None else self.sums
                        else:
                            r = post(*self.out)
                        h = self.host[slot]
                        if h is None or h.shape != r.shape or h.dtype != r.dtype:
                            h = torch.empty(r.shape, dtype=r.dtype).pin_memory()
                            self.host[slot] = h
                        dst = h
                        dst.copy_(r, non_blocking=True)
                    else:
                        dst = tuple(o.to("cpu", non_blocking=True) for o in self.out)
                    self.done[slot].record(self.compute)
                if prev is not None:
                    queued.remove(prev[0])
                    yield finish(prev)
                prev = (slot, dst)
                cur = nxt
                if nxt is not None:
                    staged, slot = staged_next, 1 - slot
            queued.remove(prev[0])
            yield finish(prev)
        finally:
            # an error or an early stop leaves batches in flight: collect them so
            # the engine's slots are free for the next run (their errors, if any,
            # are secondary to the one being raised)
            for q in queued:
                try:
                    self.engine.chain_wait(q)
                except Exception:
                    pass
