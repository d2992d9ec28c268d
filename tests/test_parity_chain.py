"""GPU parity of the batched chain (motion field -> forward -> backward ->
flows backward) against the oracle composition, window by window."""
import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.helpers import chain_inputs, rel_inf

pytestmark = pytest.mark.gpu


def _oracle_chain(depth, poses, K, ev, offs, t0=0, t1=100000):
    out = []
    for w in range(depth.shape[0]):
        fl, _ = O.depth_pose_to_flows(depth[w], poses[w], K, t0, t1)
        win = O.Window(depth.shape[2], depth.shape[1], O.make_edges(t0, t1, poses.shape[1]),
                       ev[int(offs[w]):int(offs[w + 1])], fl)
        f = O.forward(win)
        g = O.backward(win, f)
        dd, dp = O.depth_pose_to_flows_backward(depth[w], poses[w], K, win.edges, g)
        out.append((f["loss"], dd, dp))
    return out


@pytest.mark.parametrize("W,H,B,nw,n", [(64, 48, 10, 3, 3000), (128, 96, 4, 2, 20000),
                                        (346, 260, 10, 2, 100000)])
def test_chain_batch_host(engine, W, H, B, nw, n):
    depth, poses, K, ev, offs = chain_inputs(W, H, B, nw, n, seed=W)
    loss, dd, dp = engine.chain_batch(depth, poses, K, 0, 100000, ev, offs)
    ref = _oracle_chain(depth, poses, K, ev, offs)
    for w in range(nw):
        assert abs(loss[w] - ref[w][0]) <= 1e-5 * abs(ref[w][0])
        assert rel_inf(dd[w], ref[w][1]) <= 1e-5, rel_inf(dd[w], ref[w][1])
        assert rel_inf(dp[w], ref[w][2]) <= 1e-5, rel_inf(dp[w], ref[w][2])


def test_chain_batch_device_matches_host(engine):
    import torch
    depth, poses, K, ev, offs = chain_inputs(64, 48, 10, 4, 5000, seed=1)
    lh, ddh, dph = engine.chain_batch(depth, poses, K, 0, 100000, ev, offs)
    dev = torch.device("cuda:0")
    td = torch.from_numpy(depth).to(dev)
    tp = torch.from_numpy(poses).to(dev)
    te = torch.from_numpy(ev.view(np.uint8)).to(dev)
    ld, ddd, dpd = engine.chain_batch(td, tp, K, 0, 100000, te, offs)
    torch.cuda.synchronize()
    assert rel_inf(ld.cpu().numpy(), lh) <= 1e-12
    assert rel_inf(ddd.cpu().numpy(), ddh) <= 1e-6
    assert rel_inf(dpd.cpu().numpy(), dph) <= 1e-6


def test_chain_graph_replay():
    """Device-resident repeated calls: the first runs eagerly, the second is
    captured into a CUDA graph, later ones replay it. Results must be bit-identical
    (fixed-point accumulation is order-independent), and the replay must read the
    CURRENT contents of the (same) input buffers."""
    import torch
    eng = P.Engine(P.EngineOptions(algo="owner"))  # deterministic pipeline
    W, H, B, nw, n = 96, 64, 6, 3, 8000
    depth, poses, K, ev, offs = chain_inputs(W, H, B, nw, n, seed=3)
    d_depth = torch.from_numpy(depth).cuda()
    d_poses = torch.from_numpy(poses).cuda()
    d_ev = torch.from_numpy(ev.view(np.uint8).copy()).cuda()
    out = (torch.empty(nw, dtype=torch.float64, device="cuda"),
           torch.empty((nw, H, W), dtype=torch.float64, device="cuda"),
           torch.empty((nw, B, 6), dtype=torch.float64, device="cuda"))
    runs = []
    for _ in range(4):
        eng.chain_batch(d_depth, d_poses, K, 0, 100000, d_ev, offs, out=out)
        torch.cuda.synchronize()
        runs.append([o.cpu().numpy().copy() for o in out])
    for r in runs[1:]:
        for a, b in zip(r, runs[0]):
            np.testing.assert_array_equal(a, b)
    ref = _oracle_chain(depth, poses, K, ev, offs)
    for w in range(nw):
        assert abs(runs[-1][0][w] - ref[w][0]) <= 1e-5 * abs(ref[w][0])
    # new data in the same buffers: the replayed graph must see it
    depth2 = depth * 1.5
    d_depth.copy_(torch.from_numpy(depth2))
    eng.chain_batch(d_depth, d_poses, K, 0, 100000, d_ev, offs, out=out)
    torch.cuda.synchronize()
    ref2 = _oracle_chain(depth2, poses, K, ev, offs)
    for w in range(nw):
        assert abs(float(out[0][w]) - ref2[w][0]) <= 1e-5 * abs(ref2[w][0])
        assert rel_inf(out[1][w].cpu().numpy(), ref2[w][1]) <= 1e-5


def test_graph_cache_survives_reallocation():
    """Two alternating signatures keep their graphs; a larger call in between
    reallocates the workspace, which must invalidate (not replay) the old graphs.
    The owner pipeline is bit-deterministic, so every call must match bit for bit."""
    import torch
    eng = P.Engine(P.EngineOptions(deterministic=True))
    dev = torch.device("cuda:0")

    def batch(W, H, nw, n, seed):
        depth, poses, K, ev, offs = chain_inputs(W, H, 6, nw, n, seed=seed)
        return (torch.from_numpy(depth).to(dev), torch.from_numpy(poses).to(dev),
                torch.from_numpy(ev.view(np.uint8)).to(dev), K, offs)

    a, b, big = batch(64, 48, 2, 3000, 1), batch(64, 48, 2, 3000, 2), batch(160, 120, 4, 60000, 3)

    def run(x):
        d, p, e, K, offs = x
        r = eng.chain_batch(d, p, K, 0, 100000, e, offs)
        torch.cuda.synchronize()
        return [t.cpu().numpy().copy() for t in r]

    first_a, first_b = run(a), run(b)
    for _ in range(3):  # eager, capture, replay for both signatures
        for x, ref in ((a, first_a), (b, first_b)):
            got = run(x)
            assert all(np.array_equal(g, r) for g, r in zip(got, ref))
    run(big)  # grows the workspace
    for _ in range(3):
        for x, ref in ((a, first_a), (b, first_b)):
            got = run(x)
            assert all(np.array_equal(g, r) for g, r in zip(got, ref))


def test_chain_window_sums_match_torch():
    """The chain's packed window sums equal dist.pack_window_sums of its outputs
    (window-order sums vs torch's reduction: rounding only), host and device."""
    import torch
    from paper_2412_06359_b200.dist import pack_window_sums
    eng = P.Engine(P.EngineOptions(deterministic=True))
    depth, poses, K, ev, offs = chain_inputs(64, 48, 5, 4, 6000, seed=9)
    n_s = 1 + 64 * 48 + 5 * 6
    sums_h = np.zeros(n_s)
    out = eng.chain_batch(depth, poses, K, 0, 100000, ev, offs, sums=sums_h)
    ref = pack_window_sums(*(torch.from_numpy(np.ascontiguousarray(o)) for o in out)).numpy()
    assert rel_inf(sums_h, ref) <= 1e-14
    dev = torch.device("cuda:0")
    sums_d = torch.empty(n_s, dtype=torch.float64, device=dev)
    outd = eng.chain_batch(torch.from_numpy(depth).to(dev), torch.from_numpy(poses).to(dev), K, 0,
                           100000, torch.from_numpy(ev.view(np.uint8)).to(dev), offs, sums=sums_d)
    refd = pack_window_sums(*outd).cpu().numpy()
    assert rel_inf(sums_d.cpu().numpy(), refd) <= 1e-14
    with pytest.raises(P.ConfigError):
        eng.chain_batch(depth, poses, K, 0, 100000, ev, offs, sums=np.zeros(5))


def test_chain_many_windows_and_async_host_inputs():
    """More windows than the chain prologue's parameter block holds (offsets
    copied from pinned memory, no graph) and an asynchronous call with host
    inputs (runs eagerly, its slot has nothing pending) give the per-window
    results of small batches."""
    import torch
    eng = P.Engine(P.EngineOptions(deterministic=True))
    nw = 300
    depth, poses, K, ev, offs = chain_inputs(16, 12, 3, nw, 40, seed=3)
    loss, dd, dp = eng.chain_batch(depth, poses, K, 0, 100000, ev, offs)
    for w in (0, 137, 299):
        o = np.array([0, offs[w + 1] - offs[w]], np.uint64)
        l1, d1, p1 = eng.chain_batch(depth[w:w + 1], poses[w:w + 1], K, 0, 100000,
                                     ev[int(offs[w]):int(offs[w + 1])], o)
        assert np.array_equal(l1, loss[w:w + 1])
        assert np.array_equal(d1[0], dd[w]) and rel_inf(p1[0], dp[w]) <= 1e-12
    out = (torch.empty(nw, dtype=torch.float64, device="cuda"),
           torch.empty((nw, 12, 16), dtype=torch.float64, device="cuda"),
           torch.empty((nw, 3, 6), dtype=torch.float64, device="cuda"))
    eng.chain_batch_async(depth, poses, K, 0, 100000, ev, offs, out, 1)
    eng.chain_wait(1)
    assert np.array_equal(out[0].cpu().numpy(), loss)
    with pytest.raises(P.ConfigError):
        eng.chain_wait(7)


@pytest.mark.parametrize("B", [1, 32])
def test_chain_bin_extremes_and_ragged_batch(engine_det, B):
    """B = 1 and B = 32 (the cuda backend's limit), a batch with an empty window
    and windows of very different sizes, against the oracle composition."""
    W, H = 48, 36
    depth, poses, K, ev, offs = chain_inputs(W, H, B, 4, 3000, seed=40 + B)
    # ragged: window 1 empty, window 2 keeps 40 events, window 3 all of its own
    keep = np.concatenate([np.arange(int(offs[0]), int(offs[1])),
                           np.arange(int(offs[2]), int(offs[2]) + 40),
                           np.arange(int(offs[3]), int(offs[4]))])
    ev2 = ev[keep].copy()
    offs2 = np.array([0, 3000, 3000, 3040, 6040], np.uint64)
    loss, dd, dp = engine_det.chain_batch(depth, poses, K, 0, 100000, ev2, offs2)
    ref = _oracle_chain(depth, poses, K, ev2, offs2)
    for w in range(4):
        assert abs(loss[w] - ref[w][0]) <= 1e-5 * max(abs(ref[w][0]), 1e-300)
        assert rel_inf(dd[w], ref[w][1]) <= 1e-5
        assert rel_inf(dp[w], ref[w][2]) <= 1e-5
    assert loss[1] == 0.0 and not np.any(dd[1]) and not np.any(dp[1])  # empty window


def test_chain_batch_many_tiles():
    """640 x 480 (4800 sort tiles > 2048): the counting sort takes its 4-warp,
    hand-pipelined scatter; parity against the oracle composition, and the
    owner pipeline is bit-stable run to run."""
    eng = P.Engine(P.EngineOptions(algo="owner"))
    depth, poses, K, ev, offs = chain_inputs(640, 480, 10, 2, 150000, seed=21)
    loss, dd, dp = eng.chain_batch(depth, poses, K, 0, 100000, ev, offs)
    ref = _oracle_chain(depth, poses, K, ev, offs)
    for w in range(2):
        assert abs(loss[w] - ref[w][0]) <= 1e-5 * abs(ref[w][0])
        assert rel_inf(dd[w], ref[w][1]) <= 1e-5, rel_inf(dd[w], ref[w][1])
        assert rel_inf(dp[w], ref[w][2]) <= 1e-5, rel_inf(dp[w], ref[w][2])
    l2, dd2, dp2 = eng.chain_batch(depth, poses, K, 0, 100000, ev, offs)
    assert np.array_equal(l2, loss) and np.array_equal(dd2, dd) and np.array_equal(dp2, dp)


def test_chain_batch_large_sensor():
    """1280 x 720 (14400 sort tiles, beyond round 1's 12000 limit): the batched
    chain with the fused flows backward against the oracle composition."""
    eng = P.Engine()
    depth, poses, K, ev, offs = chain_inputs(1280, 720, 10, 2, 500000, seed=33)
    loss, dd, dp = eng.chain_batch(depth, poses, K, 0, 100000, ev, offs)
    assert eng.last_algo() == "owner"
    ref = _oracle_chain(depth, poses, K, ev, offs)
    for w in range(2):
        assert abs(loss[w] - ref[w][0]) <= 1e-5 * abs(ref[w][0])
        assert rel_inf(dd[w], ref[w][1]) <= 1e-5, rel_inf(dd[w], ref[w][1])
        assert rel_inf(dp[w], ref[w][2]) <= 1e-5, rel_inf(dp[w], ref[w][2])
