"""GPU parity of Engine::forward / Engine::backward (C-ABI) against the CPU
oracle (oracle/cmax_oracle.c, pinned bit-exact to the reference).

Tolerances (north_star): bit-exact for bin, alive, n_alive,
n_active and trajectory positions; <= 1e-5 relative for the loss, the IWE
stack (||d||_inf/||ref||_inf) and the flow gradients (same norm)."""
import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.helpers import rel_inf, smooth_window

pytestmark = pytest.mark.gpu

TOL = 1e-5

FD_SEEDS = list(range(100, 110)) + [42, 7] + list(range(500, 508)) + list(range(1300, 1306)) + \
    list(range(1700, 1704)) + [2500]


def _slice(w):
    return P.EventSlice(w.W, w.H, int(w.edges[0]), int(w.edges[-1]), w.events)


def _flows(w):
    return P.FlowSequence(w.edges.copy(), w.flows.copy())


def _check(engine, w, grad_tol=TOL):
    sl, fl = _slice(w), _flows(w)
    fwd = engine.forward(sl, fl)
    ref = O.forward(w, want_pos=True)
    assert fwd.loss.no_survivors == ref["no_survivors"]
    np.testing.assert_array_equal(fwd.stack.n_active, ref["n_active"])
    np.testing.assert_array_equal(fwd.traj.alive, ref["alive"])
    np.testing.assert_array_equal(fwd.traj.bin, ref["bin"])
    assert fwd.traj.n_alive == ref["n_alive"]
    np.testing.assert_array_equal(fwd.traj.pos, ref["pos"])
    if ref["loss"] == 0.0:
        assert fwd.loss.value == 0.0
    else:
        assert abs(fwd.loss.value - ref["loss"]) <= TOL * abs(ref["loss"])
    assert rel_inf(fwd.stack.count, ref["count"]) <= TOL
    assert rel_inf(fwd.stack.tsum, ref["tsum"]) <= TOL
    g = engine.backward(sl, fl, fwd).grad
    og = O.backward(w, ref)
    assert rel_inf(g, og) <= grad_tol, rel_inf(g, og)
    return fwd, g, ref, og


@pytest.mark.parametrize("seed", FD_SEEDS)
def test_fd_instances(engine, seed):
    """The reference suite's own margin-screened instances (fdcheck.hpp:94-146)."""
    w = O.ref_fd_instance(seed) if O.ref_available() else None
    if w is None:
        pytest.skip("reference fixture generator not built")
    _check(engine, w)


def test_fd_instances_masked(engine):
    if not O.ref_available():
        pytest.skip("reference fixture generator not built")
    for seed in range(900, 904):
        w = O.ref_fd_instance(seed, max_events=24, want_masked=True)
        fwd, *_ = _check(engine, w)
        assert fwd.traj.n_alive < w.n


@pytest.mark.parametrize("W,H,B,n", [(64, 48, 10, 5000), (128, 128, 10, 20000),
                                     (346, 260, 10, 100000), (37, 23, 3, 3000),
                                     (50, 40, 1, 2000), (64, 48, 32, 4000), (33, 17, 16, 3000)])
def test_smooth_windows(engine, W, H, B, n):
    w = smooth_window(W, H, B, n, seed=W + n)
    _check(engine, w)


@pytest.mark.parametrize("W,H,B,n", [(64, 48, 10, 5000), (346, 260, 10, 100000), (64, 48, 32, 4000)])
def test_smooth_windows_deterministic(engine_det, W, H, B, n):
    _check(engine_det, smooth_window(W, H, B, n, seed=W + 2 * n))


def test_fp64_accumulators(engine_f64):
    w = smooth_window(346, 260, 10, 100000, seed=3)
    _check(engine_f64, w, grad_tol=1e-12)


@pytest.mark.parametrize("W,H,B,n", [(64, 48, 10, 5000), (346, 260, 10, 100000)])
def test_atomic_path(engine_atomic, W, H, B, n):
    """The per-event atomic pipeline (algo='atomic') as an independent cross-check."""
    _check(engine_atomic, smooth_window(W, H, B, n, seed=W * 3 + n))


def test_owner_deterministic(engine_det):
    """Owner-computes path, deterministic mode: bit-identical loss, stack and
    gradients run to run."""
    engine = engine_det
    w = smooth_window(346, 260, 10, 200000, seed=21)
    a = engine.forward(_slice(w), _flows(w))
    sa, la = a.stack.count.copy(), a.loss.value
    ga = engine.backward(_slice(w), _flows(w), a).grad.copy()
    b = engine.forward(_slice(w), _flows(w))
    assert b.loss.value == la
    np.testing.assert_array_equal(b.stack.count, sa)
    np.testing.assert_array_equal(engine.backward(_slice(w), _flows(w), b).grad, ga)


def test_fast_mode_forward(engine_fast):
    """fp32 stack ("fast" mode of the atomic path): loss and IWE within 1e-6;
    gradients are not parity-grade on sparse windows."""
    w = smooth_window(346, 260, 10, 100000, seed=4)
    fwd = engine_fast.forward(_slice(w), _flows(w))
    ref = O.forward(w)
    np.testing.assert_array_equal(fwd.stack.n_active, ref["n_active"])
    assert abs(fwd.loss.value - ref["loss"]) <= 1e-6 * ref["loss"]
    assert rel_inf(fwd.stack.count, ref["count"]) <= 1e-6


def test_empty_slice(engine):
    """IweStack.EmptySliceGivesZeroStackAndWarningLoss (test_warp.cpp:78-94)."""
    w = O.Window(8, 8, O.make_edges(0, 1000, 2), np.zeros(0, O.EVENT_DTYPE), np.zeros((2, 2, 8, 8)))
    fwd = engine.forward(_slice(w), _flows(w))
    assert fwd.loss.no_survivors and fwd.loss.value == 0.0
    assert not fwd.stack.count.any() and not fwd.stack.n_active.any()
    g = engine.backward(_slice(w), _flows(w), fwd).grad
    assert not np.any(g)


def test_single_event_loss_quarter(engine):
    """IweStack.SingleMidWindowEventUnderZeroFlow (test_warp.cpp:96-113)."""
    ev = O.make_events([500000], [3], [4], [1])
    w = O.Window(8, 8, O.make_edges(0, 1000000, 1), ev, np.zeros((1, 2, 8, 8)))
    fwd = engine.forward(_slice(w), _flows(w))
    assert not fwd.loss.no_survivors
    for r in range(2):
        assert fwd.stack.count[r, 0, 4, 3] == 1.0
        assert abs(fwd.stack.tsum[r, 0, 4, 3] - 0.5) <= 1e-7
        assert fwd.stack.n_active[r] == 1
    assert abs(fwd.loss.value - 0.25) <= 1e-6


def test_exit_at_last_reference(engine):
    """IweStack.EventExitingAtLastReferenceIsExcludedEverywhere (test_warp.cpp:115-129)."""
    ev = O.make_events([0], [6], [2], [1])
    uv = np.zeros((1, 2, 8, 8))
    uv[0, 0] = 2.0
    w = O.Window(8, 8, O.make_edges(0, 1000000, 1), ev, uv)
    fwd = engine.forward(_slice(w), _flows(w))
    assert fwd.loss.no_survivors
    assert fwd.traj.n_alive == 0
    assert not fwd.stack.n_active.any()


def test_mass_conservation(engine):
    """IweStack.MassConservationPerReference (test_warp.cpp:131-145), at scale."""
    w = smooth_window(346, 260, 10, 200000, seed=11)
    fwd = engine.forward(_slice(w), _flows(w))
    mass = fwd.stack.count.sum(axis=(1, 2, 3))
    n_alive = fwd.traj.n_alive
    assert np.all(np.abs(mass - n_alive) <= 1e-5 * n_alive)


def test_true_flow_beats_zero_flow(engine):
    """ContrastLoss.TrueFlowBeatsZeroFlowOnLinearTrajectory (test_warp.cpp:164-186)."""
    ev = O.make_events([k * 20000 for k in range(5)], [2 + (80 * k) // 100 for k in range(5)],
                       [4] * 5, [1] * 5)
    uv = np.zeros((2, 2, 8, 12))
    uv[:, 0] = 40.0
    sl = P.EventSlice(12, 8, 0, 100000, ev)
    truth = P.FlowSequence(O.make_edges(0, 100000, 2), uv)
    zero = truth.zeros_like()
    assert engine.forward(sl, truth).loss.value < engine.forward(sl, zero).loss.value
    assert P.rsat(sl, truth) < 1.0
    assert P.rsat(sl, zero) == 1.0


def test_gradient_support_limited_to_stencils(engine):
    """Backward.GradientSupportLimitedToTrajectoryStencils (test_warp.cpp:211-247):
    exact zeros outside the sampled cells."""
    w = smooth_window(40, 30, 4, 50, seed=5)
    fwd, g, ref, og = _check(engine, w)
    np.testing.assert_array_equal(g == 0.0, og == 0.0)


def test_repeatability(engine):
    w = smooth_window(128, 96, 10, 30000, seed=9)
    a = engine.forward(_slice(w), _flows(w))
    la = a.loss.value
    ga = engine.backward(_slice(w), _flows(w), a).grad.copy()
    b = engine.forward(_slice(w), _flows(w))
    gb = engine.backward(_slice(w), _flows(w), b).grad
    assert abs(la - b.loss.value) <= 1e-9 * abs(la)
    assert rel_inf(ga, gb) <= 1e-6


def test_hot_pixel_dense(engine):
    """A hot pixel: 20k events on one pixel (plus a sparse background) under a
    small smooth flow, so one pixel's per-reference weight sum exceeds 2^14 --
    the fixed-point accumulators must choose their headroom from the candidate
    count (cmax_cells.cu) and still match the oracle."""
    rng = np.random.default_rng(5)
    W, H, B = 64, 48, 4
    n_hot, n_bg = 20000, 3000
    t = np.sort(rng.integers(0, 100000, n_hot + n_bg))
    x = np.concatenate([np.full(n_hot, 20), rng.integers(0, W, n_bg)])
    y = np.concatenate([np.full(n_hot, 30), rng.integers(0, H, n_bg)])
    pol = np.concatenate([np.ones(n_hot, int), np.where(rng.random(n_bg) < 0.5, 1, -1)])
    perm = rng.permutation(n_hot + n_bg)
    ev = O.make_events(t, x[perm], y[perm], pol[perm])
    xs, ys = np.arange(W)[None, :], np.arange(H)[:, None]
    uv = np.zeros((B, 2, H, W))
    for b in range(B):
        uv[b, 0] = 0.5 * np.sin(0.1 * xs + b) + 0 * ys
        uv[b, 1] = 0.5 * np.cos(0.1 * ys - b) + 0 * xs
    uv = uv.astype(np.float32).astype(np.float64)
    w = O.Window(W, H, O.make_edges(0, 100000, B), ev, uv)
    fwd, *_ = _check(engine, w)
    assert fwd.stack.count.max() > 2 ** 14


@pytest.mark.parametrize("factor", [0.5, 0.15])
def test_overflowing_owner_lists(factor):
    """Strong contraction: owner tiles near the centre gather from more sort tiles
    than their precomputed lists hold; the box-scan path must give the same parity."""
    from tests.helpers import contraction_window
    w = contraction_window(256, 192, 6, 40000, factor=factor)
    _check(P.Engine(P.EngineOptions(algo="owner")), w)


@pytest.mark.parametrize("W,H,n", [(1280, 720, 400_000), (1280, 1024, 300_000)])
def test_large_sensor(engine, W, H, n):
    """Sensors beyond 12000 sort tiles (1280x720: 14400, 1280x1024: 20480), the
    owner pipeline's 4-warp scatter at up to 28000 tiles, against the oracle."""
    w = smooth_window(W, H, 10, n, seed=W + H)
    _check(engine, w)
    assert engine.last_algo() == "owner"


def test_sensor_above_tile_limit_raises(engine):
    """More than 28000 8x8 sort tiles (1920x1080 = 32400): ConfigError, as the
    reference raises for invalid configurations (types.hpp:18-76)."""
    w = smooth_window(1920, 1080, 2, 1000, seed=3)
    with pytest.raises(P.ConfigError):
        engine.forward(_slice(w), _flows(w))
