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
