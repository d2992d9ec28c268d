"""Geometry-consistency loss L_geo (geometry.hpp:329-543).

Pinning: the oracle restatement (orc_geo_loss) reproduces the reference's
golden fixtures bit for bit (CPU tests). The GPU tests check the device path:
membership (projected / interpolated / valid / n_valid) bit-identical, the loss
and the gradients within rounding of the reference's sequential sums.
"""
import os

import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.golden_io import GOLDEN, events_of, load
from tests.helpers import rel_inf

CASES = ["masked", "occlusion", "ties", "empty"]
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
GRAD_TOL = 1e-10  # sums over pixels in another order; everything else bit-exact


def _case(name):
    g = load("geo_" + name)
    return g, g.get("m0"), g.get("m1")


# ---------------------------------------------------------------------------
# CPU: the restatement against the reference


@pytest.mark.parametrize("name", CASES)
def test_oracle_geo_matches_golden(name):
    g, m0, m1 = _case(name)
    r = O.geo_loss(g["d0"], g["d1"], g["pose"], g["K"], m0, m1, upstream=float(g["upstream"]))
    assert r["value"] == float(g["value"]) and r["n_valid"] == int(g["n_valid"])
    for k in ["projected", "interpolated", "valid", "d_d0", "d_d1", "d_pose"]:
        assert np.array_equal(r[k], g[k]), k


@needs_ref
def test_oracle_geo_matches_reference_random():
    rng = np.random.default_rng(17)
    for it in range(40):
        H, W = int(rng.integers(1, 20)), int(rng.integers(1, 24))
        K = np.array([rng.uniform(0.5, 1.5) * W, rng.uniform(0.5, 1.5) * W, (W - 1) / 2,
                      (H - 1) / 2])
        d0 = rng.uniform(0.5, 3, (H, W))
        d0[rng.uniform(size=(H, W)) < 0.05] = -1.0  # non-positive depths are skipped
        d1 = d0 * rng.uniform(0.9, 1.1, (H, W)) if it % 2 else rng.uniform(0.5, 3, (H, W))
        m0 = (rng.uniform(size=(H, W)) > 0.2).astype(np.uint8) if it % 3 == 0 else None
        m1 = (rng.uniform(size=(H, W)) > 0.2).astype(np.uint8) if it % 4 == 0 else None
        pose = np.concatenate([rng.uniform(-0.1, 0.1, 3), rng.uniform(-0.5, 0.5, 3)])
        up = float(rng.uniform(0.1, 2))
        for want in (False, True):
            a = O.geo_loss(d0, d1, pose, K, m0, m1, up, want)
            b = O.ref_geo_loss(d0, d1, pose, K, m0, m1, up, want)
            assert a["value"] == b["value"] and a["n_valid"] == b["n_valid"]
            assert a["empty"] == b["empty"]
            keys = ["projected", "interpolated", "valid"] + (["d_d0", "d_d1", "d_pose"] if want else [])
            for k in keys:
                assert np.array_equal(a[k], b[k]), (it, k)


def test_total_loss_and_weight():
    assert P.GEO_WEIGHT_DEFAULT == 0.05
    assert P.total_loss(1.0, 2.0) == 1.0 + 0.05 * 2.0
    assert P.total_loss(1.0, 2.0, 0.5) == 2.0


# ---------------------------------------------------------------------------
# GPU


def _check(out, ref, value_tol=1e-13):
    assert out["n_valid"] == ref["n_valid"]
    assert abs(out["value"] - ref["value"]) <= value_tol * max(abs(ref["value"]), 1e-300)
    for k in ["projected", "interpolated", "valid"]:
        assert np.array_equal(out[k], ref[k]), k
    for k in ["d_d0", "d_d1", "d_pose"]:
        if k in out:
            assert rel_inf(out[k], ref[k]) <= GRAD_TOL, (k, rel_inf(out[k], ref[k]))


def _np(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


@pytest.mark.gpu
@pytest.mark.parametrize("device", [False, True])
@pytest.mark.parametrize("name", CASES)
def test_geo_backward_matches_reference(name, device):
    import torch
    g, m0, m1 = _case(name)
    conv = (lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()) \
        if device else (lambda a: a)
    r = P.geometry_consistency_loss_backward(conv(g["d0"]), conv(g["d1"]), conv(g["pose"]), g["K"],
                                             float(g["upstream"]), conv(m0), conv(m1))
    out = dict(value=r.terms.value, n_valid=r.terms.n_valid, projected=_np(r.terms.projected),
               interpolated=_np(r.terms.interpolated), valid=_np(r.terms.valid), d_d0=_np(r.d_d0),
               d_d1=_np(r.d_d1), d_pose=np.concatenate([_np(r.d_omega), _np(r.d_trans)]))
    _check(out, {k: g[k] for k in g})
    assert r.terms.empty_valid_set == bool(g["empty"])
    t = P.geometry_consistency_loss(conv(g["d0"]), conv(g["d1"]), conv(g["pose"]), g["K"],
                                    conv(m0), conv(m1))
    assert t.n_valid == int(g["n_valid"]) and np.array_equal(_np(t.valid), g["valid"])


@pytest.mark.gpu
def test_geo_batch_full_size_matches_oracle():
    """640 x 480, 10 poses in one call (the predictor's use), against the
    restatement pose by pose; the summed depth gradient is the predictor's extra
    term sum_i (d_d0_i + d_d1_i) (optimize.hpp:229-230)."""
    rng = np.random.default_rng(8)
    H, W, B = 480, 640, 10
    d = np.full((H, W), 3.0)
    d[:, : W // 2] = 1.2
    d = d * rng.uniform(0.97, 1.03, (H, W))
    K = np.array([0.9 * W, 0.9 * W, (W - 1) / 2, (H - 1) / 2])
    poses = np.concatenate([rng.uniform(-0.01, 0.01, (B, 3)), rng.uniform(-0.05, 0.05, (B, 3))], 1)
    up = 0.05 / B
    b = P.geometry_consistency_loss_batch(d, d, poses, K, upstream=up)
    extra = np.zeros((H, W))
    for i in range(B):
        r = O.geo_loss(d, d, poses[i], K, upstream=up)
        _check(dict(value=b.value[i], n_valid=int(b.n_valid[i]), projected=b.projected[i],
                    interpolated=b.interpolated[i], valid=b.valid[i], d_d0=b.d_d0[i],
                    d_d1=b.d_d1[i], d_pose=b.d_poses[i]), r, value_tol=1e-12)
        extra += r["d_d0"] + r["d_d1"]
    assert rel_inf(b.d_depth_sum, extra) <= GRAD_TOL
    b2 = P.geometry_consistency_loss_batch(d, d, poses, K, upstream=up)
    assert np.array_equal(b2.d_depth_sum, b.d_depth_sum)  # fixed-order: run-to-run identical
    assert np.array_equal(b2.d_poses, b.d_poses) and np.array_equal(b2.value, b.value)


@pytest.mark.gpu
@pytest.mark.parametrize("lam", [0.05, 0.5])
def test_predictor_with_geo_matches_reference(lam):
    g = load("predictor_3")
    gg = load("predictor_geo_3")
    key = str(lam).replace(".", "p")
    f = int(g["factor"])
    ph, pw = g["params"].shape
    pred = P.DirectPredictor(g["params"], g["poses"], f)
    sl = P.EventSlice(pw * f, ph * f, 0, 100000, events_of(g))
    wg = P.predictor_loss_and_gradients(pred, sl, g["K"], lambda_geo=lam)
    l_cm, l_geo, total = gg[f"losses_{key}"]
    assert abs(wg.l_cm - l_cm) <= 1e-5 * abs(l_cm)
    assert abs(wg.l_geo - l_geo) <= 1e-12 * abs(l_geo)
    assert abs(wg.total - total) <= 1e-5 * abs(total)
    assert rel_inf(wg.grads.d_depth_params, gg[f"d_params_{key}"]) <= 1e-5
    assert rel_inf(wg.grads.d_poses, gg[f"d_poses_{key}"]) <= 1e-5
    # composition: lambda = 0 gradients + the L_geo batch through accumulate_gradients
    w0 = P.predictor_loss_and_gradients(pred, sl, g["K"], lambda_geo=0.0)
    assert w0.l_geo == 0.0 and w0.total == w0.l_cm
    dec = P.decode(pred)
    b = P.geometry_consistency_loss_batch(dec.depth, dec.depth, g["poses"], g["K"],
                                          upstream=lam / g["poses"].shape[0])
    assert abs(float(np.mean(b.value)) - wg.l_geo) <= 1e-15 * max(wg.l_geo, 1.0)


@pytest.mark.gpu
def test_predictor_geo_device_resident():
    import torch
    g = load("predictor_3")
    f = int(g["factor"])
    ph, pw = g["params"].shape
    host = P.predictor_loss_and_gradients(
        P.DirectPredictor(g["params"], g["poses"], f),
        P.EventSlice(pw * f, ph * f, 0, 100000, events_of(g)), g["K"], lambda_geo=0.05)
    evd = torch.from_numpy(events_of(g).view(np.uint8).copy()).cuda()
    dev = P.predictor_loss_and_gradients(
        P.DirectPredictor(torch.tensor(g["params"], device="cuda"),
                          torch.tensor(g["poses"], device="cuda"), f),
        P.EventSlice(pw * f, ph * f, 0, 100000, evd), g["K"], lambda_geo=0.05)
    assert abs(dev.l_geo - host.l_geo) <= 1e-15
    assert rel_inf(dev.grads.d_depth_params.cpu().numpy(), host.grads.d_depth_params) <= 1e-12


@pytest.mark.gpu
def test_geo_errors():
    d = np.ones((4, 5))
    with pytest.raises(P.DimensionMismatchError):
        P.geometry_consistency_loss(d, np.ones((5, 4)), np.zeros(6), [1, 1, 0, 0])
    with pytest.raises(P.DimensionMismatchError):
        P.geometry_consistency_loss(d, d, np.zeros(6), [1, 1, 0, 0], mask0=np.ones((3, 3)))
