"""GPU parity at the event densities the benchmark runs.

* configs C / S: the exact ``bench.py`` batches (640x480 windows of 1M events,
  two-plane depth, per-bin ego-motion) through the batched chain and through
  Engine::forward / backward;
* the SURVEY §8(d) sweep's dense points (346x260, 3e6 and 1e7 events per
  window), where the owner kernels' fixed-point stack drops below 50 fraction
  bits (cmax_cells.cu: fb = min(50, 63 - bits(T)));
* the tile sort: its permutation equals a stable argsort of the same integer
  keys (bit-exact, the std::stable_sort analog).

The truth is the reference itself (oracle/_ref/libevcm_ref.so: depth_pose_to_flows,
Engine::loss_and_grad with the parallel deterministic backend,
depth_pose_to_flows_backward), multi-threaded so the 1e7-event window stays in
seconds. Tolerances: bit-exact for bin / alive / n_alive / n_active; <= 1e-5
relative (||d||_inf / ||ref||_inf, fdcheck.hpp:184) for loss, IWE and gradients.
"""
import os
import sys

import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.helpers import rel_inf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]
TOL = 1e-5


def _engine_window(eng, depth, poses, K, ev, t1, B):
    """Engine-level forward / backward of one window on the reference's own
    motion field, checked against Engine::loss_and_grad of the reference."""
    H, W = depth.shape
    flows = O.ref_depth_pose_to_flows(depth, poses, K, 0, t1)[0]
    w = O.Window(W, H, O.make_edges(0, t1, B), ev, flows)
    sl = P.EventSlice(W, H, 0, t1, ev)
    fl = P.FlowSequence(w.edges.copy(), flows.copy())
    fwd = eng.forward(sl, fl)
    ref = O.ref_loss_and_grad(w, backend="parallel", deterministic=True)
    np.testing.assert_array_equal(fwd.stack.n_active, ref["n_active"])
    alive, bins, n_alive = fwd.alive_bin()
    np.testing.assert_array_equal(alive, ref["alive"])
    np.testing.assert_array_equal(bins, ref["bin"])
    assert n_alive == ref["n_alive"]
    assert abs(fwd.loss.value - ref["loss"]) <= TOL * abs(ref["loss"])
    assert rel_inf(fwd.stack.count, ref["count"]) <= TOL
    assert rel_inf(fwd.stack.tsum, ref["tsum"]) <= TOL
    g = eng.backward(sl, fl, fwd).grad
    err = rel_inf(g, ref["grad"])
    assert err <= TOL, err
    return fwd, err


def _chain_vs_reference(eng, depth, poses, K, ev, offs, t1):
    loss, dd, dp = eng.chain_batch(depth, poses, K, 0, t1, ev, offs)
    errs = []
    for w in range(depth.shape[0]):
        one = np.array([0, int(offs[w + 1] - offs[w])], np.uint64)
        r = O.ref_chain_batch(depth[w:w + 1], poses[w:w + 1], K, 0, t1,
                              ev[int(offs[w]):int(offs[w + 1])], one, want_grads=True)
        assert abs(loss[w] - r["loss_sum"]) <= TOL * abs(r["loss_sum"])
        e_dd, e_dp = rel_inf(dd[w], r["d_depth"][0]), rel_inf(dp[w], r["d_poses"][0])
        assert e_dd <= TOL and e_dp <= TOL, (e_dd, e_dp)
        errs.append((e_dd, e_dp))
    return errs


@pytest.fixture(scope="module")
def eng():
    return P.Engine()  # defaults: deterministic -> the owner pipeline the bench runs


@pytest.mark.parametrize("workload", ["C", "S"])
def test_bench_batches_chain(eng, workload):
    """Two windows of the bench's own batch (C: rank 0; S: the first rank's
    first windows) through the batched chain, window by window vs the reference."""
    wl = bench.WORKLOADS[workload]
    depth, poses, K, ev, offs = bench.make_inputs(wl, 0, 2)
    _chain_vs_reference(eng, depth, poses, K, ev, offs, wl["window_us"])
    assert eng.last_algo() == "owner"


def test_bench_window_engine_level(eng):
    wl = bench.WORKLOADS["C"]
    depth, poses, K, ev, offs = bench.make_inputs(wl, 0, 1)
    _engine_window(eng, depth[0], poses[0], K, ev, wl["window_us"], wl["B"])


@pytest.mark.parametrize("n", [3_000_000, 10_000_000])
def test_sweep_dense_windows(eng, n):
    """346x260 at 3e6 / 1e7 events per window (~33 / ~111 events per pixel)."""
    wl = dict(bench.WORKLOADS["B"], n_events=n)
    depth, poses, K, ev, offs = bench.make_inputs(wl, 0, 1)
    _engine_window(eng, depth[0], poses[0], K, ev, wl["window_us"], wl["B"])
    _chain_vs_reference(eng, depth, poses, K, ev, offs, wl["window_us"])


@pytest.mark.parametrize("W,H,n", [(346, 260, 100_000), (640, 480, 1_000_000), (37, 23, 3000)])
def test_sort_permutation_is_stable_argsort(eng, W, H, n):
    wl = dict(bench.WORKLOADS["B"], W=W, H=H, n_events=n)
    depth, poses, K, ev, offs = bench.make_inputs(wl, 0, 1)
    flows = O.ref_depth_pose_to_flows(depth[0], poses[0], K, 0, wl["window_us"])[0]
    edges = O.make_edges(0, wl["window_us"], wl["B"])
    fwd = eng.forward(P.EventSlice(W, H, 0, wl["window_us"], ev), P.FlowSequence(edges, flows))
    keys, perm, sorted_keys = fwd.sort_products()
    valid = np.flatnonzero(keys != 0xFFFFFFFF)
    want = valid[np.argsort(keys[valid], kind="stable")]
    np.testing.assert_array_equal(perm, want.astype(np.uint32))
    np.testing.assert_array_equal(sorted_keys, keys[want])
    # every key is a tile of the sensor, and the sort is a permutation
    n_tiles = ((W + 7) // 8) * ((H + 7) // 8)
    assert keys[valid].max() < n_tiles
    assert len(np.unique(perm)) == len(perm) == n
