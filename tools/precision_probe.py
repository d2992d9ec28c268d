"""Max relative errors of the CUDA path vs the oracle per accumulator precision mode."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.helpers import rel_inf, smooth_window, chain_inputs

modes = {"s32g32": P.EngineOptions(), "s64g32": P.EngineOptions(stack_f64=True),
         "s64g64": P.EngineOptions(stack_f64=True, grad_f64=True)}
engines = {k: P.Engine(v) for k, v in modes.items()}
wins = [("fd%d" % s, O.ref_fd_instance(s)) for s in list(range(100, 110)) + list(range(500, 508)) + list(range(1300, 1306)) + list(range(1700, 1704))]
wins += [("fdm%d" % s, O.ref_fd_instance(s, max_events=24, want_masked=True)) for s in range(900, 904)]
wins += [("sm%dx%d_%d" % (W, H, n), smooth_window(W, H, B, n, seed=W + n)) for W, H, B, n in
         [(64, 48, 10, 5000), (128, 128, 10, 20000), (346, 260, 10, 100000), (640, 480, 10, 1000000), (346, 260, 10, 3000000)]]
worst = {k: [0, 0, 0] for k in modes}
for name, w in wins:
    ref = O.forward(w)
    og = O.backward(w, ref)
    row = [name]
    for k, e in engines.items():
        sl = P.EventSlice(w.W, w.H, int(w.edges[0]), int(w.edges[-1]), w.events)
        fl = P.FlowSequence(w.edges.copy(), w.flows.copy())
        f = e.forward(sl, fl)
        g = e.backward(sl, fl, f).grad
        le = abs(f.loss.value - ref["loss"]) / max(abs(ref["loss"]), 1e-300)
        ie = rel_inf(f.stack.count, ref["count"])
        ge = rel_inf(g, og)
        worst[k] = [max(a, b) for a, b in zip(worst[k], [le, ie, ge])]
        row.append("%s L%.1e I%.1e G%.1e" % (k, le, ie, ge))
    print("  ".join(row), flush=True)
print("WORST", worst)
# chain
for W, H, B, nw, n in [(346, 260, 10, 2, 100000), (640, 480, 10, 1, 1000000)]:
    depth, poses, K, ev, offs = chain_inputs(W, H, B, nw, n, seed=W)
    for k, e in engines.items():
        loss, dd, dp = e.chain_batch(depth, poses, K, 0, 100000, ev, offs)
        errs = []
        for w in range(nw):
            fl, _ = O.depth_pose_to_flows(depth[w], poses[w], K, 0, 100000)
            win = O.Window(W, H, O.make_edges(0, 100000, B), ev[int(offs[w]):int(offs[w + 1])], fl)
            f = O.forward(win); g = O.backward(win, f)
            odd, odp = O.depth_pose_to_flows_backward(depth[w], poses[w], K, win.edges, g)
            errs.append((abs(loss[w] - f["loss"]) / f["loss"], rel_inf(dd[w], odd), rel_inf(dp[w], odp)))
        print("chain", W, H, n, k, ["L%.1e D%.1e P%.1e" % x for x in errs], flush=True)
