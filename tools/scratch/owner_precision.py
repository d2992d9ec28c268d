"""Max relative errors of the default (owner, deterministic) engine vs the oracle:
loss / IWE count / flow gradient per window, and the chain's loss / d_depth / d_poses."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.helpers import rel_inf, smooth_window, chain_inputs

e = P.Engine(P.EngineOptions())
wins = [("fd%d" % s, O.ref_fd_instance(s)) for s in list(range(100, 110)) + list(range(500, 508))]
wins += [("sm%dx%d_%d" % (W, H, n), smooth_window(W, H, B, n, seed=W + n)) for W, H, B, n in
         [(64, 48, 10, 5000), (128, 128, 10, 20000), (346, 260, 10, 100000), (346, 260, 10, 300000),
          (640, 480, 10, 1000000)]]
worst = [0, 0, 0]
for name, w in wins:
    ref = O.forward(w)
    og = O.backward(w, ref)
    sl = P.EventSlice(w.W, w.H, int(w.edges[0]), int(w.edges[-1]), w.events)
    fl = P.FlowSequence(w.edges.copy(), w.flows.copy())
    f = e.forward(sl, fl)
    g = e.backward(sl, fl, f).grad
    le = abs(f.loss.value - ref["loss"]) / max(abs(ref["loss"]), 1e-300)
    ie = rel_inf(f.stack.count, ref["count"])
    ge = rel_inf(g, og)
    worst = [max(a, b) for a, b in zip(worst, [le, ie, ge])]
    print("%-22s L%.1e I%.1e G%.1e" % (name, le, ie, ge), flush=True)
print("WORST L%.1e I%.1e G%.1e" % tuple(worst))
for W, H, B, nw, n in [(346, 260, 10, 2, 100000), (640, 480, 10, 2, 1000000)]:
    depth, poses, K, ev, offs = chain_inputs(W, H, B, nw, n, seed=W)
    loss, dd, dp = e.chain_batch(depth, poses, K, 0, 100000, ev, offs)
    for w in range(nw):
        fl, _ = O.depth_pose_to_flows(depth[w], poses[w], K, 0, 100000)
        win = O.Window(W, H, O.make_edges(0, 100000, B), ev[int(offs[w]):int(offs[w + 1])], fl)
        f = O.forward(win); g = O.backward(win, f)
        odd, odp = O.depth_pose_to_flows_backward(depth[w], poses[w], K, win.edges, g)
        print("chain %dx%d n=%d w%d L%.1e D%.1e P%.1e" % (W, H, n, w, abs(loss[w] - f["loss"]) / f["loss"],
              rel_inf(dd[w], odd), rel_inf(dp[w], odp)), flush=True)
