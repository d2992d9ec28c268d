import sys, numpy as np
sys.path.insert(0, '.')
import paper_2412_06359_b200 as P
from tests.helpers import chain_inputs, smooth_window
eng = P.Engine(P.EngineOptions(algo="owner"))
out = {}
for (W, H, B, nw, n, seed) in [(346, 260, 10, 2, 100000, 1), (200, 150, 7, 3, 60000, 2)]:
    depth, poses, K, ev, offs = chain_inputs(W, H, B, nw, n, seed=seed)
    l, dd, dp = eng.chain_batch(depth, poses, K, 0, 100000, ev, offs)
    out[f"c{seed}"] = np.concatenate([np.ravel(l), np.ravel(dd), np.ravel(dp)])
w = smooth_window(160, 120, 10, 30000, seed=5)
sl = P.EventSlice(w.W, w.H, int(w.edges[0]), int(w.edges[-1]), w.events)
fl = P.FlowSequence(w.edges.copy(), w.flows.copy())
f = eng.forward(sl, fl)
out["stack"] = np.concatenate([np.ravel(f.stack.count), np.ravel(f.stack.tsum)])
out["grad"] = np.ravel(eng.backward(sl, fl, f).grad)
np.savez(sys.argv[1], **out)
