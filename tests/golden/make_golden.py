"""Generates the golden fixtures in tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libevcm_ref.so, compiled from /root/reference by
oracle/Makefile). Run in the dev container (the reference tree is not on the GPU
box):  python tests/golden/make_golden.py

Each fixture is an .npz with the inputs and the reference outputs:
  fd_<seed>.npz      random_fd_instance (fdcheck.hpp:94-146) -> Engine (naive backend)
  smooth_32x24.npz   smooth-flow window (bench_window semantics + spatial variation)
  geom_13x9.npz      depth_pose_to_flows / _backward on a masked depth map
  chain_<seed>.npz   make_chain_instance (tests/chain_support.hpp:119-184) decoded
  predictor_<seed>.npz  make_chain_instance as a raw DirectPredictor + the reference's
                     decode and predictor_loss_and_gradients (optimize.hpp:205-241)
  adam.npz           Adam::step (optimize.hpp:115-134), 3 steps on fixed gradients
  evt1/*.evt1        EVT1 files written by the reference's write_events (io.hpp:156-172),
                     plus the byte-patched variants of tests/test_core_io.cpp:73-137;
  evt1.npz           the reference's read_events outcome for each (error code or
                     W, H, t0, t1, events)
  geo_<case>.npz     geometry_consistency_loss_backward (geometry.hpp:458-534) on
                     masked / occluding / tied / empty cases
  predictor_geo_3.npz  predictor_loss_and_gradients with lambda_geo = 0.05 and 0.5
  run_window.npz     run_window (optimize.hpp:297-375) over 3 windows, 12 updates
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402
from tests.helpers import smooth_window  # noqa: E402


def save(name, **arrs):
    np.savez_compressed(os.path.join(HERE, name), **arrs)


def window_fixture(name, w):
    r = O.ref_loss_and_grad(w, backend="naive", want_pos=True)
    save(name, W=w.W, H=w.H, edges=w.edges, events=w.events.view(np.uint8).reshape(-1, 16),
         flows=w.flows, loss=r["loss"], no_survivors=r["no_survivors"], count=r["count"],
         tsum=r["tsum"], n_active=r["n_active"], alive=r["alive"], bin=r["bin"], pos=r["pos"],
         grad=r["grad"])


def predictor_fixtures():
    for seed in (3, 11):
        r = O.ref_predictor_instance(seed, sensor_w=32, sensor_h=24, factor=8, n_bins=3,
                                     n_events=60)
        depth = O.ref_decode(r["params"], 8)
        rng = np.random.default_rng(seed)
        g = rng.uniform(-1, 1, depth.shape)
        save(f"predictor_{seed}.npz", events=r["events"].view(np.uint8).reshape(-1, 16),
             params=r["params"], poses=r["poses"], K=r["K"], factor=8, loss=r["loss"],
             d_params=r["d_params"], d_poses=r["d_poses"], depth=depth, g=g,
             g_params=O.ref_decode_backward(r["params"], 8, g))
    rng = np.random.default_rng(2)
    s, g = rng.normal(size=40), rng.normal(size=40)
    save("adam.npz", slots=s, grads=g, lr=0.01, steps=3, out=O.ref_adam_steps(s, g, 3, 0.01))


GEO_CASES = ["masked", "occlusion", "ties", "empty"]


def geo_inputs(case):
    """Inputs of the L_geo fixtures (also used by the tests for the restatement)."""
    rng = np.random.default_rng({"masked": 1, "occlusion": 2, "ties": 3, "empty": 4}[case])
    H, W = 24, 32
    K = np.array([0.9 * W, 0.9 * W, (W - 1) / 2, (H - 1) / 2])
    m0 = m1 = None
    if case == "masked":
        d0 = rng.uniform(1, 3, (H, W))
        d1 = d0 * rng.uniform(0.95, 1.05, (H, W))
        m0 = (rng.uniform(size=(H, W)) > 0.1).astype(np.uint8)
        m1 = (rng.uniform(size=(H, W)) > 0.1).astype(np.uint8)
        pose = np.array([0.01, -0.02, 0.015, 0.05, -0.03, 0.02])
    elif case == "occlusion":  # near plane slides over the far one
        d0 = np.full((H, W), 4.0)
        d0[:, W // 3: W // 2] = 1.0
        d0 *= rng.uniform(0.99, 1.01, (H, W))
        d1 = d0.copy()
        pose = np.array([0.0, 0.03, 0.0, 0.25, 0.0, 0.0])
    elif case == "ties":  # constant depth, forward motion: equal z in every cell
        d0 = np.full((H, W), 2.0)
        d1 = np.full((H, W), 2.0)
        pose = np.array([0.0, 0.0, 0.0, 0.0, 0.0, 0.3])
    else:  # everything leaves the view
        d0 = rng.uniform(1, 2, (H, W))
        d1 = d0.copy()
        pose = np.array([0.0, 0.0, 0.0, 50.0, 0.0, 0.0])
    return d0, d1, m0, m1, pose, K


def geo_fixtures():
    for case in GEO_CASES:
        d0, d1, m0, m1, pose, K = geo_inputs(case)
        r = O.ref_geo_loss(d0, d1, pose, K, m0, m1, upstream=0.7)
        extra = {} if m0 is None else dict(m0=m0, m1=m1)
        save(f"geo_{case}.npz", d0=d0, d1=d1, pose=pose, K=K, upstream=0.7, value=r["value"],
             n_valid=r["n_valid"], empty=r["empty"], projected=r["projected"],
             interpolated=r["interpolated"], valid=r["valid"], d_d0=r["d_d0"], d_d1=r["d_d1"],
             d_pose=r["d_pose"], **extra)
    g = np.load(os.path.join(HERE, "predictor_3.npz"))
    ev = np.ascontiguousarray(g["events"]).view(O.EVENT_DTYPE).reshape(-1)
    out = {}
    for lam in (0.05, 0.5):
        losses, dpar, dpo = O.ref_predictor_loss(g["params"], int(g["factor"]), g["poses"], g["K"],
                                                 0, 100000, ev, lam)
        key = str(lam).replace(".", "p")
        out.update({f"losses_{key}": np.array(losses), f"d_params_{key}": dpar,
                    f"d_poses_{key}": dpo})
    save("predictor_geo_3.npz", **out)


def run_window_fixture():
    base = O.ref_predictor_instance(3, sensor_w=32, sensor_h=24, factor=8, n_bins=3, n_events=60)
    wins = []
    for w, seed in enumerate([3, 4, 5]):
        rr = O.ref_predictor_instance(seed, sensor_w=32, sensor_h=24, factor=8, n_bins=3,
                                      n_events=60)
        ev = rr["events"].copy()
        ev["t_us"] += np.uint64(w * 100000)
        wins.append((w * 100000, (w + 1) * 100000, ev))
    out = {}
    for lam in (0.0, 0.05):
        po, qo, rec = O.ref_run_window(wins, base["params"], 8, base["poses"], base["K"], 1e-3, 1,
                                       12, lam)
        key = str(lam).replace(".", "p")
        out.update({f"params_{key}": po, f"poses_{key}": qo, f"rec_{key}": rec})
    ev = np.concatenate([w[2] for w in wins]).astype(O.EVENT_DTYPE)
    offs = np.cumsum([0] + [len(w[2]) for w in wins]).astype(np.uint64)
    save("run_window.npz", events=ev.view(np.uint8).reshape(-1, 16), offs=offs,
         t01=np.array([[w[0], w[1]] for w in wins], np.uint64), params=base["params"],
         poses=base["poses"], K=base["K"], factor=8, lr=1e-3, steps_per_update=1, max_updates=12,
         **out)


EVT1_FILES = ["empty", "three", "random_2k", "bad_magic", "trunc_record", "trunc_header",
              "unsorted", "coord_at_width", "zero_polarity", "trailing", "zero_width"]


def evt1_fixtures():
    """The reference's EVT1 tests (tests/test_core_io.cpp:45-150) as files."""
    d = os.path.join(HERE, "evt1")
    os.makedirs(d, exist_ok=True)
    f = lambda n: os.path.join(d, n + ".evt1")  # noqa: E731
    three = O.make_events([100, 250, 400], [1, 3, 9], [2, 4, 7], [1, -1, 1])  # :33-41
    O.ref_write_events(f("empty"), 32, 24, 0, 0, np.zeros(0, O.EVENT_DTYPE))
    O.ref_write_events(f("three"), 10, 8, 100, 401, three)
    W, H, t0, t1, ev = O.ref_random_slice(7, 2000)
    O.ref_write_events(f("random_2k"), W, H, t0, t1, ev)
    base = open(f("three"), "rb").read()

    def patched(name, fn):
        b = bytearray(base)
        b = fn(b) or b
        open(f(name), "wb").write(bytes(b))

    patched("bad_magic", lambda b: b.__setitem__(0, ord("X")))
    patched("trunc_record", lambda b: b[:-7])
    patched("trunc_header", lambda b: b[:10])
    patched("unsorted", lambda b: b.__setitem__(slice(16, 19), b"\xff\xff\xff"))
    patched("coord_at_width", lambda b: b.__setitem__(slice(24, 26), b"\x0a\x00"))
    patched("zero_polarity", lambda b: b.__setitem__(28, 0))
    patched("trailing", lambda b: b + b"\x00")
    patched("zero_width", lambda b: b.__setitem__(slice(4, 6), b"\x00\x00"))
    out = {}
    for n in EVT1_FILES:
        try:
            W, H, t0, t1, ev = O.ref_read_events(f(n))
            out[n + "_code"] = 0
            out[n + "_hdr"] = np.array([W, H, t0, t1], np.uint64)
            out[n + "_events"] = ev.view(np.uint8).reshape(-1, 16)
        except O.OracleError as e:
            out[n + "_code"] = e.code
    save("evt1.npz", **out)


def main():
    if not O.ref_available():
        O.build(ref=True)
    evt1_fixtures()
    predictor_fixtures()
    geo_fixtures()
    run_window_fixture()
    for seed in (100, 7, 503, 1300):
        window_fixture(f"fd_{seed}.npz", O.ref_fd_instance(seed))
    window_fixture("fd_masked_900.npz", O.ref_fd_instance(900, max_events=24, want_masked=True))
    window_fixture("smooth_32x24.npz", smooth_window(32, 24, 4, 600, seed=5))
    rng = np.random.default_rng(11)
    H, W, B = 9, 13, 3
    depth = rng.uniform(0.8, 3.0, (H, W)).astype(np.float32).astype(np.float64)
    mask = (rng.uniform(size=(H, W)) > 0.15).astype(np.uint8)
    poses = np.concatenate([rng.uniform(-0.02, 0.02, (B, 3)), rng.uniform(-0.1, 0.1, (B, 3))], 1)
    poses[1, 5] = -2.5  # some pixels behind the camera
    K = np.array([0.9 * W, 0.95 * W, (W - 1) / 2 + 0.3, (H - 1) / 2 - 0.2])
    flows, valid, edges = O.ref_depth_pose_to_flows(depth, poses, K, 0, 100000, mask)
    g = rng.uniform(-1, 1, (B, 2, H, W))
    dd, dp = O.ref_depth_pose_to_flows_backward(depth, poses, K, edges, g, mask)
    save("geom_13x9.npz", depth=depth, mask=mask, poses=poses, K=K, flows=flows, valid=valid,
         edges=edges, grad=g, d_depth=dd, d_poses=dp)
    for seed in (1, 20):
        ev, depth, poses, K = O.ref_chain_instance(seed)
        fl, _, edges = O.ref_depth_pose_to_flows(depth, poses, K, 0, 100000)
        w = O.Window(depth.shape[1], depth.shape[0], edges, ev, fl)
        r = O.ref_loss_and_grad(w, backend="naive")
        dd, dp = O.ref_depth_pose_to_flows_backward(depth, poses, K, edges, r["grad"])
        save(f"chain_{seed}.npz", depth=depth, poses=poses, K=K, edges=edges,
             events=ev.view(np.uint8).reshape(-1, 16), loss=r["loss"], d_depth=dd, d_poses=dp)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
