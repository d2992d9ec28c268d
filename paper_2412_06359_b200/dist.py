"""Data-parallel plumbing for batches of event windows.

Windows are independent units: a batch is split into contiguous shards, one per
rank (one process per GPU); each rank runs the chain on its shard, reduces its
windows locally, and the only exchange is one all-reduce of the packed buffer
[sum loss, sum_w d_depth, sum_w d_poses] (NCCL over NVLink on GPUs; gloo in the
CPU tests).
"""
from __future__ import annotations


def shard_windows(n_windows: int, world: int, rank: int) -> range:
    """Contiguous shard of [0, n_windows) for `rank` (sizes differ by at most 1)."""
    base, extra = divmod(n_windows, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def pack_window_sums(loss, d_depth, d_poses, out=None):
    """[sum loss, sum over windows of d_depth (H*W), of d_poses (B*6)] as one flat
    float64 tensor (the all-reduce payload)."""
    import torch
    n = 1 + d_depth[0].numel() + d_poses[0].numel()
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=loss.device)
    out[0:1].copy_(loss.sum().reshape(1))
    out[1:1 + d_depth[0].numel()].copy_(d_depth.sum(0).reshape(-1))
    out[1 + d_depth[0].numel():].copy_(d_poses.sum(0).reshape(-1))
    return out


def allreduce_window_sums(buf, group=None):
    """Sum the packed buffer over ranks (no-op when torch.distributed is not
    initialised or the world has one rank)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


class OverlappedAllReduce:
    """Double-buffered all-reduce of the packed window sums:
    step i's chain writes buffer i % 2 and its reduction is issued asynchronously
    (on NCCL's internal stream, ordered after the chain on the caller's stream),
    so it runs while step i+1 computes into the other buffer. ``buffer(i)``
    makes the caller's stream wait for the reduction of step i-2 before the
    buffer is reused; ``drain()`` waits for every outstanding reduction. With one
    rank (or no process group) it only hands out the buffers."""

    def __init__(self, n: int, device, group=None):
        import torch
        import torch.distributed as dist
        self.bufs = [torch.zeros(n, dtype=torch.float64, device=device) for _ in range(2)]
        self.work = [None, None]
        self.group = group
        self.active = dist.is_available() and dist.is_initialized() and \
            dist.get_world_size(group) > 1

    def _wait(self, slot: int) -> None:
        w = self.work[slot]
        if w is not None:
            w.wait()  # NCCL: the current stream waits; gloo: the host waits
            self.work[slot] = None

    def buffer(self, i: int):
        self._wait(i % 2)
        return self.bufs[i % 2]

    def submit(self, i: int):
        """Starts the reduction of step i's buffer; returns the buffer."""
        import torch.distributed as dist
        b = self.bufs[i % 2]
        if self.active:
            self.work[i % 2] = dist.all_reduce(b, op=dist.ReduceOp.SUM, group=self.group,
                                               async_op=True)
        return b

    def drain(self) -> None:
        for s in (0, 1):
            self._wait(s)
