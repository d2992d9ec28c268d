"""GPU: the operator contract around the kernels -- shape / dtype checks of the
flow grids (engine.hpp:215-222), the forward -> backward hand-off (engine.hpp:
185-205: trajectories from the forward, Jacobians from the flows given), chain
offset validation, stream ordering of torch-produced inputs, PhaseStats
(engine.hpp:63-66, 226-242) and the reference's default determinism
(engine.hpp:60)."""
import numpy as np
import pytest
import torch

import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.helpers import chain_inputs, rel_inf, smooth_window

pytestmark = pytest.mark.gpu


def _slice_flows(w):
    return P.EventSlice(w.W, w.H, 0, int(w.edges[-1]), w.events), P.FlowSequence(w.edges, w.flows)


def test_default_engine_is_deterministic_owner():
    e = P.Engine()
    assert e.opts.deterministic
    w = smooth_window(40, 30, 4, 2000, seed=3)
    sl, fl = _slice_flows(w)
    f1, b1 = e.loss_and_grad(sl, fl)
    assert e.last_algo() == "owner"
    f2, b2 = e.loss_and_grad(sl, fl)
    assert f1.loss.value == f2.loss.value
    assert np.array_equal(b1.grad, b2.grad)  # bit-stable run to run


def test_atomic_needs_nondeterministic():
    with pytest.raises(P.ConfigError):
        P.Engine(P.EngineOptions(algo="atomic"))
    P.Engine(P.EngineOptions(algo="atomic", deterministic=False))


def test_flow_grid_must_match_sensor(engine):
    w = smooth_window(24, 16, 3, 500, seed=5)
    sl, fl = _slice_flows(w)
    bad = P.FlowSequence(w.edges, np.zeros((3, 2, 16, 25)))
    with pytest.raises(P.DimensionMismatchError):
        engine.forward(sl, bad)
    f = engine.forward(sl, fl)
    with pytest.raises(P.DimensionMismatchError):
        engine.backward(sl, bad, f)
    dev = torch.from_numpy(w.flows).cuda()
    with pytest.raises(P.DimensionMismatchError):  # fp32 device flows
        engine.forward(sl, P.FlowSequence(w.edges, dev.float()))
    with pytest.raises(P.DimensionMismatchError):  # strided device flows
        engine.forward(sl, P.FlowSequence(w.edges, dev.transpose(2, 3).contiguous().transpose(2, 3)))


def test_backward_after_motion_field_call(engine):
    """depth_pose_to_flows between forward and backward leaves the forward's
    device state intact (its own output buffer)."""
    w = smooth_window(32, 24, 4, 3000, seed=8)
    sl, fl = _slice_flows(w)
    f = engine.forward(sl, fl)
    want = engine.backward(sl, fl, f).grad.copy()
    f = engine.forward(sl, fl)
    depth = np.full((24, 32), 2.0)
    engine.depth_pose_to_flows(depth, np.full((4, 6), 1e-3), [20.0, 20.0, 15.5, 11.5], 0,
                               int(w.edges[-1]))
    got = engine.backward(sl, fl, f).grad
    assert np.array_equal(got, want)


def test_backward_uses_the_flows_it_is_given(engine):
    """Reference semantics (engine.hpp:185-205, 475-504): the backward's flow
    Jacobians come from its own `flows` argument, the trajectories from the
    forward. The same flows reproduce the oracle; other flows change the result."""
    w = smooth_window(32, 24, 4, 3000, seed=9)
    sl, fl = _slice_flows(w)
    f = engine.forward(sl, fl)
    same = engine.backward(sl, fl, f).grad.copy()
    want = O.backward(O.Window(w.W, w.H, w.edges, w.events, w.flows))
    assert rel_inf(same, want) <= 1e-5
    uv2 = (w.flows * 1.5).astype(np.float32).astype(np.float64)
    other = engine.backward(sl, P.FlowSequence(w.edges, uv2), f).grad
    assert not np.array_equal(other, same)


def test_stale_forward_is_refused(engine):
    a = smooth_window(20, 16, 3, 400, seed=1)
    b = smooth_window(20, 16, 3, 400, seed=2)
    sa, fa = _slice_flows(a)
    sb, fb = _slice_flows(b)
    ra = engine.forward(sa, fa)
    engine.forward(sb, fb)
    with pytest.raises(P.ConfigError):
        engine.backward(sa, fa, ra)


def test_phase_stats_filled(engine):
    w = smooth_window(64, 48, 5, 20000, seed=4)
    sl, fl = _slice_flows(w)
    f, b = engine.loss_and_grad(sl, fl)
    for st in (f.warp_stats, f.splat_stats, f.loss_stats, b.stats):
        assert st.time_us > 0 and st.peak_bytes > 0
    assert b.stats.peak_bytes >= f.loss_stats.peak_bytes


def test_chain_offsets_validated(engine):
    depth, poses, K, ev, offs = chain_inputs(24, 16, 3, 2, 300, seed=4)
    with pytest.raises(P.ConfigError):
        engine.chain_batch(depth, poses, K, 0, 100000, ev, offs[:-1])
    with pytest.raises(P.ConfigError):
        engine.chain_batch(depth, poses, K, 0, 100000, ev, np.array([0, 400, 300], np.uint64))
    with pytest.raises(P.DimensionMismatchError):
        engine.chain_batch(depth, poses, K, 0, 100000, ev, np.array([0, 300, 601], np.uint64))
    with pytest.raises(P.ConfigError):
        engine.chain_batch(depth, poses, K, 0, 100000, ev, np.array([1, 300, 600], np.uint64))


def test_engine_waits_for_the_producer_stream():
    """Inputs written by a torch kernel on a side stream right before the call:
    the engine (own non-blocking stream) must see the final values."""
    e = P.Engine()
    w = smooth_window(64, 48, 4, 20000, seed=6)
    sl, fl = _slice_flows(w)
    want = e.forward(sl, fl).loss.value
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        big = torch.randn(4096, 4096, device="cuda")
        for _ in range(8):
            big = big @ big * 1e-3  # keep the side stream busy
        uv = torch.zeros(w.flows.shape, dtype=torch.float64, device="cuda")
        uv.copy_(torch.from_numpy(w.flows), non_blocking=False)
        uv.add_(big.sum() * 0.0)  # last writer of uv runs after the matmuls
        ev = torch.from_numpy(w.events.view(np.uint8).copy()).cuda()
        got = e.forward(P.EventSlice(w.W, w.H, 0, int(w.edges[-1]), ev),
                        P.FlowSequence(w.edges, uv)).loss.value
    assert got == want


def test_pipeline_rejects_foreign_compute_stream():
    s = torch.cuda.Stream()
    e = P.Engine(P.EngineOptions(stream=s.cuda_stream))
    with pytest.raises(P.ConfigError):
        P.ChainPipeline(e, compute_stream=torch.cuda.Stream())
    P.ChainPipeline(e, compute_stream=s)
