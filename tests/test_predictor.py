"""GPU: the predictor decode chain through the C-ABI
against the oracle (bit-exact restatement of predictor.hpp / optimize.hpp) and
against the reference's own predictor_loss_and_gradients on its chain fixture
(tests/chain_support.hpp:119-184).

Tolerances: decode / transpose 1e-13 relative (the device's exp/log1p are not
the host libm: softplus may differ in the last bit); Adam bit-exact; the full
predictor loss and gradients 1e-5 (north_star), gradients as ||d||_inf / ||ref||_inf."""
import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.golden_io import events_of, load
from tests.helpers import rel_inf

pytestmark = pytest.mark.gpu


def _engine():
    return P.Engine()


@pytest.mark.parametrize("shape,f", [((5, 7), 8), ((3, 4), 1), ((6, 9), 3), ((1, 1), 8)])
def test_decode_matches_oracle(shape, f):
    rng = np.random.default_rng(shape[0] * 10 + f)
    p = rng.normal(scale=2.0, size=shape)
    d = P.decode(P.DirectPredictor(p, np.zeros((2, 6)), f), _engine()).depth
    o = O.decode(p, f)
    assert d.shape == o.shape
    assert rel_inf(d, o) <= 1e-13


@pytest.mark.parametrize("shape,f", [((5, 7), 8), ((3, 4), 1), ((6, 9), 3)])
def test_decode_backward_matches_oracle(shape, f):
    rng = np.random.default_rng(shape[1] * 10 + f)
    p = rng.normal(size=shape)
    g = rng.normal(size=(shape[0] * f, shape[1] * f))
    e = _engine()
    from paper_2412_06359_b200 import engine as E
    out = np.zeros(shape)
    E._raise(E.load_library().evcm_cuda_decode_backward(e._h, shape[1], shape[0], f, E._ptr(p),
                                                        E._ptr(g), E.MEM_HOST, E._ptr(out)))
    assert rel_inf(out, O.decode_backward(p, f, g)) <= 1e-13


def test_adam_bit_exact_host_and_device():
    g = load("adam")
    cfg = P.OptimizerConfig(learning_rate=float(g["lr"]))
    s = g["slots"].copy()
    opt = P.Adam(s.size)
    for _ in range(int(g["steps"])):
        opt.step(s, g["grads"], cfg, _engine())
    np.testing.assert_array_equal(s, g["out"])
    import torch
    sd = torch.tensor(g["slots"], dtype=torch.float64, device="cuda")
    gd = torch.tensor(g["grads"], dtype=torch.float64, device="cuda")
    optd = P.Adam(sd.shape[0], like=sd)
    for _ in range(int(g["steps"])):
        optd.step(sd, gd, cfg, _engine())
    np.testing.assert_array_equal(sd.cpu().numpy(), g["out"])


def _slice(ev, W, H):
    return P.EventSlice(W, H, 0, 100000, ev)


@pytest.mark.parametrize("name", ["predictor_3", "predictor_11"])
def test_predictor_loss_and_gradients_golden(name):
    g = load(name)
    f = int(g["factor"])
    ph, pw = g["params"].shape
    pred = P.DirectPredictor(g["params"], g["poses"], f)
    wg = P.predictor_loss_and_gradients(pred, _slice(events_of(g), pw * f, ph * f), g["K"],
                                        engine=_engine())
    assert abs(wg.l_cm - float(g["loss"])) <= 1e-5 * abs(float(g["loss"]))
    assert rel_inf(wg.grads.d_depth_params, g["d_params"]) <= 1e-5
    assert rel_inf(wg.grads.d_poses, g["d_poses"]) <= 1e-5


@pytest.mark.ref
@pytest.mark.parametrize("seed", [1, 2, 7, 20])
def test_predictor_matches_reference(seed):
    if not O.ref_available():
        pytest.skip("reference fixture generator not built")
    r = O.ref_predictor_instance(seed, sensor_w=48, sensor_h=32, factor=8, n_bins=4, n_events=200)
    ph, pw = r["params"].shape
    pred = P.DirectPredictor(r["params"], r["poses"], 8)
    wg = P.predictor_loss_and_gradients(pred, _slice(r["events"], pw * 8, ph * 8), r["K"],
                                        engine=_engine())
    assert abs(wg.l_cm - r["loss"]) <= 1e-5 * abs(r["loss"])
    assert rel_inf(wg.grads.d_depth_params, r["d_params"]) <= 1e-5
    assert rel_inf(wg.grads.d_poses, r["d_poses"]) <= 1e-5


def test_predictor_device_resident_and_composition():
    """Device-resident params (torch) give the host result; the fused call equals
    decode -> depth_pose_to_flows -> loss_and_grad -> accumulate_gradients."""
    import torch
    g = load("predictor_3")
    f = int(g["factor"])
    ph, pw = g["params"].shape
    e = _engine()
    sl = _slice(events_of(g), pw * f, ph * f)
    host = P.predictor_loss_and_gradients(P.DirectPredictor(g["params"], g["poses"], f), sl, g["K"],
                                          engine=e)
    pd = torch.tensor(g["params"], device="cuda")
    qd = torch.tensor(g["poses"], device="cuda")
    evd = torch.from_numpy(events_of(g).view(np.uint8).copy()).cuda()
    sld = P.EventSlice(pw * f, ph * f, 0, 100000, evd)
    dev = P.predictor_loss_and_gradients(P.DirectPredictor(pd, qd, f), sld, g["K"], engine=e)
    assert abs(float(dev.l_cm) - host.l_cm) <= 1e-12 * abs(host.l_cm)
    assert rel_inf(dev.grads.d_depth_params.cpu().numpy(), host.grads.d_depth_params) <= 1e-12
    # composition through the separate entry points
    dec = P.decode(P.DirectPredictor(g["params"], g["poses"], f), e)
    gf = e.depth_pose_to_flows(dec.depth, g["poses"], g["K"], 0, 100000)
    fwd, bwd = e.loss_and_grad(sl, gf.flows)
    pg = P.accumulate_gradients(P.DirectPredictor(g["params"], g["poses"], f), dec.depth, g["K"],
                                gf.flows, bwd.grad, engine=e)
    assert abs(fwd.loss.value - host.l_cm) <= 1e-12 * abs(host.l_cm)
    assert rel_inf(pg.d_depth_params, host.grads.d_depth_params) <= 1e-6
    assert rel_inf(pg.d_poses, host.grads.d_poses) <= 1e-6


def test_predictor_errors():
    g = load("predictor_3")
    f = int(g["factor"])
    ph, pw = g["params"].shape
    pred = P.DirectPredictor(g["params"], g["poses"], f)
    with pytest.raises(P.DimensionMismatchError):
        P.predictor_loss_and_gradients(pred, _slice(events_of(g), pw * f + 1, ph * f), g["K"])
    with pytest.raises(P.ConfigError):
        P.decode(P.DirectPredictor(np.zeros((2, 2)), np.zeros((1, 6)), 0))
