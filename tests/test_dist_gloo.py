"""CPU, world size 2 over gloo: window sharding + the packed loss/gradient
all-reduce reproduce the single-process batch sums (chain computed by the oracle)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_06359_b200.dist import allreduce_window_sums, pack_window_sums, shard_windows


def _oracle_chain(depth, poses, K, ev, offs, windows):
    from oracle import oracle as O
    W, H, B = depth.shape[2], depth.shape[1], poses.shape[1]
    L, DD, DP = [], [], []
    for w in windows:
        fl, _ = O.depth_pose_to_flows(depth[w], poses[w], K, 0, 100000)
        win = O.Window(W, H, O.make_edges(0, 100000, B), ev[int(offs[w]):int(offs[w + 1])], fl)
        f = O.forward(win)
        g = O.backward(win, f)
        dd, dp = O.depth_pose_to_flows_backward(depth[w], poses[w], K, win.edges, g)
        L.append(f["loss"])
        DD.append(dd)
        DP.append(dp)
    return (torch.tensor(L, dtype=torch.float64), torch.from_numpy(np.array(DD)),
            torch.from_numpy(np.array(DP)))


def _inputs():
    from tests.helpers import chain_inputs
    return chain_inputs(24, 16, 3, 5, 300, seed=4)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    depth, poses, K, ev, offs = _inputs()
    mine = shard_windows(depth.shape[0], world, rank)
    buf = pack_window_sums(*_oracle_chain(depth, poses, K, ev, offs, mine))
    allreduce_window_sums(buf)
    if rank == 0:
        q.put(buf.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,world", [(5, 2), (8, 3), (2, 2), (1, 2)])
def test_shard_windows_partition(n, world):
    shards = [shard_windows(n, world, r) for r in range(world)]
    assert sum(len(s) for s in shards) == n
    assert [i for s in shards for i in s] == list(range(n))
    assert max(len(s) for s in shards) - min(len(s) for s in shards) <= 1


def test_gloo_world2_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    depth, poses, K, ev, offs = _inputs()
    want = pack_window_sums(*_oracle_chain(depth, poses, K, ev, offs, range(depth.shape[0])))
    np.testing.assert_allclose(got, want.numpy(), rtol=1e-12, atol=1e-15)
