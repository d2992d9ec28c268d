"""GPU parity of depth_pose_to_flows (bit-exact) and its backward (<= 1e-5)."""
import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.helpers import rel_inf

pytestmark = pytest.mark.gpu


def _rand_geom(rng, W, H, B, rot=0.02, tr=0.1):
    depth = rng.uniform(0.8, 3.0, (H, W))
    poses = np.concatenate([rng.uniform(-rot, rot, (B, 3)), rng.uniform(-tr, tr, (B, 3))], 1)
    K = np.array([0.9 * W, 0.95 * W, (W - 1) / 2 + 0.3, (H - 1) / 2 - 0.2])
    return depth, poses, K


@pytest.mark.parametrize("trial", range(6))
def test_motion_field_bit_exact(engine, trial):
    rng = np.random.default_rng(100 + trial)
    W, H, B = [(17, 13, 3), (64, 48, 10), (346, 260, 10), (5, 4, 1), (640, 480, 10), (33, 7, 32)][trial]
    depth, poses, K = _rand_geom(rng, W, H, B)
    mask = (rng.uniform(size=(H, W)) > 0.1).astype(np.uint8) if trial % 2 else None
    if trial == 3:
        poses[0, 5] = -2.5  # behind-camera pixels (test_geometry.cpp:348-366)
    if trial == 5:
        poses[:, :3] *= 1e-6  # series branches of rodrigues / its Jacobian
    gf = engine.depth_pose_to_flows(depth, poses, K, 0, 100000, mask=mask)
    of, ov = O.depth_pose_to_flows(depth, poses, K, 0, 100000, mask)
    np.testing.assert_array_equal(gf.flows.uv, of)
    np.testing.assert_array_equal(gf.valid, ov)
    np.testing.assert_array_equal(gf.flows.edges_us, O.make_edges(0, 100000, B))
    g = rng.uniform(-1, 1, (B, 2, H, W))
    g[:, :, ::3] = 0.0
    dd, dp = engine.depth_pose_to_flows_backward(depth, poses, K, gf.flows, g, mask=mask)
    odd, odp = O.depth_pose_to_flows_backward(depth, poses, K, gf.flows.edges_us, g, mask)
    assert rel_inf(dd, odd) <= 1e-12
    assert rel_inf(dp, odp) <= 1e-9


def test_lateral_translation_uniform_parallax(engine):
    """DepthPoseToFlows.LateralTranslationGivesUniformParallax (test_geometry.cpp:288-301)."""
    depth = np.full((8, 10), 2.0)
    gf = engine.depth_pose_to_flows(depth, np.array([[0, 0, 0, 0.1, 0, 0]], float),
                                    np.array([100.0, 100.0, 0.0, 0.0]), 0, 100000)
    dt = gf.flows.bin_duration_s(0)
    assert abs(dt - 0.1) <= 4 * np.spacing(0.1)  # EXPECT_DOUBLE_EQ
    assert np.all(np.abs(gf.flows.uv[0, 0] * dt - 5.0) <= 1e-12)
    assert np.all(np.abs(gf.flows.uv[0, 1] * dt) <= 1e-12)
    assert np.all(gf.valid == 1)


def test_invalid_pixels_contribute_nothing(engine):
    """FlowsBackward.InvalidPixelsContributeNothing (test_geometry.cpp:439-460)."""
    d = np.full((4, 5), 2.0)
    d[0, :] = 0.6
    K = np.array([40.0, 40.0, 2.0, 1.5])
    poses = np.array([[0, 0, 0, 0, 0, -1.0]])
    gf = engine.depth_pose_to_flows(d, poses, K, 0, 50000)
    w = np.zeros((1, 2, 4, 5))
    w[0, 0], w[0, 1] = 1.0, -0.5
    dd, _ = engine.depth_pose_to_flows_backward(d, poses, K, gf.flows, w)
    assert np.all(gf.valid[0, 0] == 0)
    assert np.all(dd[0] == 0.0)
    assert dd[2, 2] != 0.0


def test_rejects_bad_pose(engine):
    with pytest.raises(P.ConfigError):
        engine.depth_pose_to_flows(np.ones((4, 4)), np.array([[4.0, 0, 0, 0, 0, 0]]),
                                   np.array([4.0, 4.0, 1.5, 1.5]), 0, 1000)


def test_translational_flow_scales_inversely_with_depth(engine):
    """DepthPoseToFlows.TranslationalFlowScalesInverselyWithDepth (test_geometry.cpp:303-322)."""
    K = np.array([64.0, 64.0, 4.5, 3.5])
    lateral = np.array([[0.0, 0.0, 0.0, 0.03, -0.02, 0.0]])
    far = engine.depth_pose_to_flows(np.full((8, 10), 2.0), lateral, K, 0, 50000).flows.uv
    near = engine.depth_pose_to_flows(np.full((8, 10), 1.0), lateral, K, 0, 50000).flows.uv
    assert np.all(np.abs(near - 2.0 * far) <= 1e-10)
    rot = np.array([[0.01, -0.02, 0.03, 0.0, 0.0, 0.0]])  # pure rotation: depth-independent
    rf = engine.depth_pose_to_flows(np.full((8, 10), 2.0), rot, K, 0, 50000).flows.uv
    rn = engine.depth_pose_to_flows(np.full((8, 10), 1.0), rot, K, 0, 50000).flows.uv
    assert np.all(np.abs(rn - rf) <= 1e-10)


def test_depth_translation_scale_family(engine):
    """DepthPoseToFlows.DepthAndTranslationScaleFamilyLeavesFlowUnchanged (:324-346)."""
    rng = np.random.default_rng(17)
    base = rng.uniform(1.0, 3.0, (7, 11))
    K = np.array([60.0, 58.0, 5.0, 3.5])
    poses = np.array([[0.01, -0.015, 0.02, 0.04, 0.02, 0.01],
                      [-0.02, 0.01, 0.005, -0.03, 0.01, -0.02]])
    s = 3.7
    sp = poses.copy()
    sp[:, 3:] *= s
    a = engine.depth_pose_to_flows(base, poses, K, 0, 100000)
    b = engine.depth_pose_to_flows(base * s, sp, K, 0, 100000)
    assert np.array_equal(a.valid, b.valid)
    assert np.all(np.abs(a.flows.uv - b.flows.uv) <= 1e-10)


def test_behind_camera_pixels_zero_flow_clear_bit(engine):
    """DepthPoseToFlows.BehindCameraPixelsGetZeroFlowAndClearBit (:348-366)."""
    H, W = 8, 6
    d = np.repeat((0.55 + 0.25 * np.arange(H))[:, None], W, axis=1)
    gf = engine.depth_pose_to_flows(d, np.array([[0, 0, 0, 0, 0, -1.0]]),
                                    np.array([50.0, 50.0, 2.5, 3.5]), 0, 40000)
    expect = (d > 1.0)
    assert np.array_equal(gf.valid[0] != 0, expect)
    assert np.all(gf.flows.uv[0][:, ~expect] == 0.0)


def test_rsat_true_flow_and_zero_flow(engine):
    """ContrastLoss.TrueFlowBeatsZeroFlowOnLinearTrajectory (test_warp.cpp:164-186):
    rsat(zero flow) is exactly 1 and the true flow scores below 1."""
    ev = O.make_events([k * 20000 for k in range(5)], [2 + (80 * k) // 100 for k in range(5)],
                       [4] * 5, [1] * 5)
    s = P.EventSlice(12, 8, 0, 100000, ev)
    truth = P.FlowSequence.zeros(12, 8, 0, 100000, 2)
    truth.uv[:, 0] = 40.0
    zero = truth.zeros_like()
    assert engine.forward(s, truth).loss.value < engine.forward(s, zero).loss.value
    assert P.rsat(s, truth) < 1.0
    assert P.rsat(s, zero) == 1.0
