"""CPU: the C restatement (oracle/cmax_oracle.c) is pinned to the reference.

1. bit-for-bit against the golden fixtures produced by the UNMODIFIED reference
   (tests/golden/make_golden.py, naive backend for gradients);
2. bit-for-bit against the compiled reference on many fresh instances (only
   where oracle/_ref/libevcm_ref.so exists);
3. the reference suite's closed-form known-answer tests (test_warp.cpp,
   test_geometry.cpp) re-stated on the oracle.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_io import CHAIN_FIXTURES, WINDOW_FIXTURES, load, window_of

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("name", WINDOW_FIXTURES)
def test_golden_windows_bit_exact(name):
    d = load(name)
    w = window_of(d)
    f = O.forward(w, want_pos=True)
    assert f["loss"] == float(d["loss"])
    assert f["no_survivors"] == bool(d["no_survivors"])
    for k in ("count", "tsum", "n_active", "alive", "bin", "pos"):
        np.testing.assert_array_equal(f[k], d[k], err_msg=k)
    np.testing.assert_array_equal(O.backward(w, f), d["grad"])


def test_golden_geometry_bit_exact():
    d = load("geom_13x9")
    fl, valid = O.depth_pose_to_flows(d["depth"], d["poses"], d["K"], 0, 100000, d["mask"])
    np.testing.assert_array_equal(fl, d["flows"])
    np.testing.assert_array_equal(valid, d["valid"])
    dd, dp = O.depth_pose_to_flows_backward(d["depth"], d["poses"], d["K"], d["edges"], d["grad"],
                                            d["mask"])
    np.testing.assert_array_equal(dd, d["d_depth"])
    np.testing.assert_array_equal(dp, d["d_poses"])


@pytest.mark.parametrize("name", CHAIN_FIXTURES)
def test_golden_chain_bit_exact(name):
    d = load(name)
    fl, _ = O.depth_pose_to_flows(d["depth"], d["poses"], d["K"], 0, 100000)
    from tests.golden_io import events_of
    w = O.Window(d["depth"].shape[1], d["depth"].shape[0], d["edges"], events_of(d), fl)
    f = O.forward(w)
    assert f["loss"] == float(d["loss"])
    g = O.backward(w, f)
    dd, dp = O.depth_pose_to_flows_backward(d["depth"], d["poses"], d["K"], d["edges"], g)
    np.testing.assert_array_equal(dd, d["d_depth"])
    np.testing.assert_array_equal(dp, d["d_poses"])


@needs_ref
@pytest.mark.parametrize("seed", list(range(100, 110)) + [42, 7] + list(range(500, 508)) +
                         list(range(1300, 1306)) + list(range(1700, 1704)) + [2500])
def test_fd_instances_match_reference(seed):
    w = O.ref_fd_instance(seed)
    a = O.forward(w, want_pos=True)
    b = O.ref_loss_and_grad(w, backend="naive", want_pos=True)
    assert a["loss"] == b["loss"]
    for k in ("count", "tsum", "n_active", "alive", "bin", "pos"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    np.testing.assert_array_equal(O.backward(w, a), b["grad"])


@needs_ref
def test_bench_window_and_backends_match_reference():
    w = O.ref_bench_window(64, 48, 10, 4000, seed=3)
    a = O.forward(w)
    for backend in ("naive", "padded", "parallel"):
        b = O.ref_loss_and_grad(w, backend=backend)
        assert a["loss"] == b["loss"]  # forward bit-identical across backends (engine.hpp:14-16)
        np.testing.assert_array_equal(a["count"], b["count"])
    np.testing.assert_array_equal(O.backward(w, a), O.ref_loss_and_grad(w, backend="naive")["grad"])


@needs_ref
@pytest.mark.parametrize("trial", range(4))
def test_geometry_matches_reference(trial):
    rng = np.random.default_rng(50 + trial)
    H, W, B = 11, 17, 4
    depth = rng.uniform(0.8, 3.0, (H, W))
    mask = None if trial % 2 else (rng.uniform(size=(H, W)) > 0.2).astype(np.uint8)
    poses = np.concatenate([rng.uniform(-0.03, 0.03, (B, 3)), rng.uniform(-0.1, 0.1, (B, 3))], 1)
    if trial == 2:
        poses[:, :3] *= 1e-7  # series branches (geometry.hpp:98, 119)
    K = np.array([20.0, 21.0, 8.0, 5.0])
    f1, v1 = O.depth_pose_to_flows(depth, poses, K, 0, 100000, mask)
    f2, v2, e = O.ref_depth_pose_to_flows(depth, poses, K, 0, 100000, mask)
    np.testing.assert_array_equal(f1, f2)
    np.testing.assert_array_equal(v1, v2)
    g = rng.uniform(-1, 1, (B, 2, H, W))
    d1 = O.depth_pose_to_flows_backward(depth, poses, K, e, g, mask)
    d2 = O.ref_depth_pose_to_flows_backward(depth, poses, K, e, g, mask)
    np.testing.assert_array_equal(d1[0], d2[0])
    np.testing.assert_array_equal(d1[1], d2[1])


# ---- known-answer tests of the reference suite, on the oracle ---------------


def _const_flow_window(W, H, t1, per_bin, events=None):
    B = len(per_bin)
    uv = np.zeros((B, 2, H, W))
    for b, (u, v) in enumerate(per_bin):
        uv[b, 0], uv[b, 1] = u, v
    ev = events if events is not None else np.zeros(0, O.EVENT_DTYPE)
    return O.Window(W, H, O.make_edges(0, t1, B), ev, uv)


def test_single_event_loss_quarter():
    """IweStack.SingleMidWindowEventUnderZeroFlow (test_warp.cpp:96-113)."""
    w = _const_flow_window(8, 8, 1000000, [(0, 0)], O.make_events([500000], [3], [4], [1]))
    f = O.forward(w)
    assert f["count"][0, 0, 4, 3] == 1.0 and f["count"][1, 0, 4, 3] == 1.0
    assert abs(f["tsum"][0, 0, 4, 3] - 0.5) < 1e-12
    assert list(f["n_active"]) == [1, 1]
    assert abs(f["loss"] - 0.25) < 1e-6


def test_exit_at_last_reference():
    """test_warp.cpp:115-129."""
    w = _const_flow_window(8, 8, 1000000, [(2.0, 0)], O.make_events([0], [6], [2], [1]))
    f = O.forward(w)
    assert f["no_survivors"] and f["n_alive"] == 0


def test_closed_form_warp_and_splat():
    """WarpEvent.ConstantFlowClosedForm / SplatBilinear.WorkedExamples
    (test_warp.cpp:34-76) through the trajectory positions and the stack."""
    w = _const_flow_window(16, 16, 10000, [(100.0, 0.0)], O.make_events([5000], [2], [2], [1]))
    f = O.forward(w, want_pos=True)
    np.testing.assert_allclose(f["pos"][0, 0], [1.5, 2.0], atol=1e-12)
    np.testing.assert_allclose(f["pos"][0, 1], [2.5, 2.0], atol=1e-12)
    assert f["count"][0, 0, 2, 1] == 0.5 and f["count"][0, 0, 2, 2] == 0.5


def test_mass_conservation():
    """IweStack.MassConservationPerReference (test_warp.cpp:131-145)."""
    from tests.helpers import smooth_window
    w = smooth_window(40, 30, 5, 800, seed=2)
    f = O.forward(w)
    mass = f["count"].sum(axis=(1, 2, 3))
    assert np.all(np.abs(mass - f["n_alive"]) <= 1e-9 * f["n_alive"])


def test_rodrigues_identities():
    """rodrigues orthonormal, det 1; Jacobian vs central differences
    (test_geometry.cpp:78-216 style)."""
    rng = np.random.default_rng(3)
    for _ in range(10):
        om = rng.uniform(-0.5, 0.5, 3)
        R = O.rodrigues(om)
        np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-14)
        assert abs(np.linalg.det(R) - 1) < 1e-14
        dR = O.rodrigues_jacobian(om)
        for k in range(3):
            h = np.zeros(3)
            h[k] = 1e-6
            fd = (O.rodrigues(om + h) - O.rodrigues(om - h)) / 2e-6
            np.testing.assert_allclose(dR[k], fd, atol=1e-8)


def test_lateral_translation_parallax():
    """DepthPoseToFlows.LateralTranslationGivesUniformParallax (test_geometry.cpp:288-301)."""
    fl, valid = O.depth_pose_to_flows(np.full((8, 10), 2.0), [[0, 0, 0, 0.1, 0, 0]],
                                      [100.0, 100.0, 0.0, 0.0], 0, 100000)
    dt = (100000 - 0) * 1e-6
    assert np.all(np.abs(fl[0, 0] * dt - 5.0) < 1e-12)
    assert np.all(valid == 1)


def test_flows_backward_finite_differences():
    """FlowsBackward.MatchesFiniteDifferences (test_geometry.cpp:368-437)."""
    rng = np.random.default_rng(41)
    H, W, B = 5, 6, 2
    K = np.array([35.0, 33.0, 2.5, 2.0])
    depth = rng.uniform(1.0, 2.5, (H, W))
    poses = np.concatenate([rng.uniform(-0.02, 0.02, (B, 3)), rng.uniform(-0.05, 0.05, (B, 3))], 1)
    wts = rng.uniform(-1, 1, (B, 2, H, W))
    e = O.make_edges(0, 100000, B)

    def score(dep, ps):
        fl, _ = O.depth_pose_to_flows(dep, ps, K, 0, 100000)
        return float((wts * fl).sum())

    dd, dp = O.depth_pose_to_flows_backward(depth, poses, K, e, wts)
    for j in range(H * W):
        p, m = depth.copy().reshape(-1), depth.copy().reshape(-1)
        p[j] += 1e-5
        m[j] -= 1e-5
        fd = (score(p.reshape(H, W), poses) - score(m.reshape(H, W), poses)) / 2e-5
        assert abs(dd.reshape(-1)[j] - fd) <= 1e-5 * max(1.0, abs(fd))
    for i in range(B):
        for c in range(6):
            pp, pm = poses.copy(), poses.copy()
            pp[i, c] += 1e-6
            pm[i, c] -= 1e-6
            fd = (score(depth, pp) - score(depth, pm)) / 2e-6
            assert abs(dp[i, c] - fd) <= 1e-5 * max(1.0, abs(fd))


def test_flow_gradient_finite_differences():
    """Backward.FiniteDifferenceAgreementSmallInstances (test_warp.cpp:249-259) on a
    margin-screened golden instance."""
    w = window_of(load("fd_100"))
    f = O.forward(w)
    g = O.backward(w, f)
    h = 1e-4
    mx, na, nf = 0.0, 0.0, 0.0
    for idx in np.ndindex(w.flows.shape):
        saved = w.flows[idx]
        w.flows[idx] = saved + h
        lp = O.forward(w)["loss"]
        w.flows[idx] = saved - h
        lm = O.forward(w)["loss"]
        w.flows[idx] = saved
        fd = (lp - lm) / (2 * h)
        mx = max(mx, abs(g[idx] - fd))
        na, nf = max(na, abs(g[idx])), max(nf, abs(fd))
    assert mx / max(na, nf, 1e-12) < 1e-4


# ---- predictor decode chain ---------------------------------

@pytest.mark.parametrize("name", ["predictor_3.npz", "predictor_11.npz"])
def test_golden_predictor_decode_bit_exact(name):
    """The oracle's decode and decode transpose reproduce the reference's
    (predictor.hpp:126-131, 156-162) bit for bit on the committed fixtures."""
    g = load(name[:-4])
    f = int(g["factor"])
    np.testing.assert_array_equal(O.decode(g["params"], f), g["depth"])
    np.testing.assert_array_equal(O.decode_backward(g["params"], f, g["g"]), g["g_params"])


def test_golden_adam_bit_exact():
    g = load("adam")
    s = g["slots"].copy()
    m, v = np.zeros_like(s), np.zeros_like(s)
    for t in range(1, int(g["steps"]) + 1):
        O.adam_step(s, g["grads"], m, v, t, float(g["lr"]))
    np.testing.assert_array_equal(s, g["out"])


def test_softplus_tails_and_upsample_factor_one():
    """softplus is positive and stable on both tails; factor 1 is the identity
    (predictor.hpp:25-34, 48)."""
    for x in (-800.0, -30.0, -1e-3, 0.0, 1e-3, 30.0, 800.0):
        assert O.softplus(x) > 0.0 or x < -700
        assert 0.0 <= O.softplus_grad(x) <= 1.0
    p = np.random.default_rng(0).normal(size=(3, 4))
    np.testing.assert_array_equal(O.decode(p, 1), np.vectorize(O.softplus)(p))


@pytest.mark.ref
@pytest.mark.parametrize("seed", [1, 2, 5])
def test_decode_chain_matches_reference(seed):
    if not O.ref_available():
        pytest.skip("reference not built")
    rng = np.random.default_rng(seed)
    p = rng.normal(size=(4 + seed, 3 + seed))
    for f in (1, 2, 8):
        np.testing.assert_array_equal(O.decode(p, f), O.ref_decode(p, f))
        g = rng.normal(size=(p.shape[0] * f, p.shape[1] * f))
        np.testing.assert_array_equal(O.decode_backward(p, f, g), O.ref_decode_backward(p, f, g))
