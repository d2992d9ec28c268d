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
