"""GPU: device-resident optimize_flow_only against the
reference's own loop (optimize.hpp:385-487) on identical windows.

The loop starts from zero flow, where every event sits exactly on the pixel
lattice; there the eps = 1e-9 regulariser of the focus loss switches whole pixel
terms on for sub-nanopixel moves, and the first gradient carries ~1e-13
cancellation noise whose sign depends on the summation order (the reference's own
backends differ there too). Adam turns that noise into ~1e-6 px/s steps, after
which trajectories legitimately differ. Parity is therefore checked on update 0
(loss, rsat, gradient norm within 1e-5) and on the first Adam step of the
non-noise components; later updates are checked for the loop's own invariants."""
import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.helpers import rel_inf, smooth_window

pytestmark = pytest.mark.gpu


def _slice(w):
    return P.EventSlice(w.W, w.H, int(w.edges[0]), int(w.edges[-1]), w.events)


@pytest.mark.ref
@pytest.mark.parametrize("W,H,B,n,lr,steps", [(32, 24, 3, 800, 0.5, 6), (48, 32, 4, 3000, 0.05, 8),
                                              (64, 48, 2, 5000, 2.0, 5)])
def test_optimize_flow_only_matches_reference(W, H, B, n, lr, steps):
    if not O.ref_available():
        pytest.skip("reference not built")
    w = smooth_window(W, H, B, n, seed=W + n)
    flows, l_cm, rsat, gn = O.ref_optimize_flow_only(W, H, 0, 100000, w.events, B, lr, steps)
    res = P.optimize_flow_only(_slice(w), B, P.OptimizerConfig(learning_rate=lr, max_updates=steps))
    recs = res.log.records
    assert len(recs) == len(l_cm)
    r0 = recs[0]
    assert abs(r0.l_cm - l_cm[0]) <= 1e-5 * abs(l_cm[0])
    assert abs(r0.rsat - rsat[0]) <= 1e-5 * abs(rsat[0])
    assert abs(r0.grad_norm_depth - gn[0]) <= 1e-5 * abs(gn[0])
    # loop invariants: the returned flows are the best iterate seen
    best = min(r.l_cm for r in recs)
    host_flows = P.FlowSequence(res.flows.edges_us, res.flows.uv.cpu().numpy())
    got = P.Engine().forward(_slice(w), host_flows).loss.value
    assert got <= best * (1 + 1e-12)
    for r in recs:
        assert r.total == r.l_cm and r.l_geo == 0.0
        assert abs(r.rsat - r.l_cm / recs[0].l_cm) <= 1e-12 * r.rsat


def test_first_adam_step_matches_reference_update():
    """One update from zero flow: the device loop's flows after its first Adam
    step equal the oracle's Adam step on the oracle gradient to 1e-5 of the
    learning rate, except on the cancellation-noise components
    (|g| < 1e-9 * ||g||_inf). Near |g| ~ adam_eps the step lr*g/(|g|+eps) is
    sensitive to g's last digits (fixed-point resolution ~1e-15 * max|g|), hence
    the absolute tolerance."""
    w = smooth_window(48, 32, 4, 3000, seed=9)
    B = 4
    zero = np.zeros((B, 2, w.H, w.W))
    w0 = O.Window(w.W, w.H, w.edges, w.events, zero)
    og = O.backward(w0, O.forward(w0))
    s, m, v = np.zeros(og.size), np.zeros(og.size), np.zeros(og.size)
    O.adam_step(s, og.ravel(), m, v, 1, 0.05)
    e = P.Engine()
    fl = P.FlowSequence(w.edges.copy(), zero.copy())
    g = e.loss_and_grad(_slice(w), fl)[1].grad
    opt = P.Adam(g.size)
    flat = fl.uv.reshape(-1)
    opt.step(flat, g.reshape(-1), P.OptimizerConfig(learning_rate=0.05), e)
    real = np.abs(og.ravel()) >= 1e-9 * np.abs(og).max()
    np.testing.assert_allclose(flat[real], s[real], rtol=1e-6, atol=1e-5 * 0.05)


def test_optimize_flow_only_errors():
    w = smooth_window(32, 24, 3, 500, seed=2)
    with pytest.raises(P.EmptySliceError):
        P.optimize_flow_only(P.EventSlice(32, 24, 0, 100000), 3, P.OptimizerConfig())
    with pytest.raises(P.ConfigError):
        P.optimize_flow_only(_slice(w), 3, P.OptimizerConfig(learning_rate=-1.0))
    res = P.optimize_flow_only(_slice(w), 3, P.OptimizerConfig(learning_rate=0.1, max_updates=0))
    assert not res.log.records and float(res.flows.uv.abs().max()) == 0.0
