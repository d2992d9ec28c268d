import numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.helpers import rel_inf, smooth_window
eng = P.Engine(P.EngineOptions(algo="owner"))
for seed in [100, 7, 503]:
    w = O.ref_fd_instance(seed)
    sl = P.EventSlice(w.W, w.H, int(w.edges[0]), int(w.edges[-1]), w.events)
    fl = P.FlowSequence(w.edges.copy(), w.flows.copy())
    fwd = eng.forward(sl, fl)
    g = eng.backward(sl, fl, fwd).grad
    ref = O.forward(w)
    og = O.backward(w, ref)
    print("seed", seed, "W,H,B,n", w.W, w.H, len(w.edges)-1, len(w.events), "rel", rel_inf(g, og))
    B = g.shape[0]
    den = np.abs(og).max()
    for b in range(B):
        d = np.abs(g[b]-og[b]).max()/den
        if d > 1e-6:
            idx = np.unravel_index(np.argmax(np.abs(g[b]-og[b])), g[b].shape)
            print("  bin", b, "err", d, "at", idx, "gpu", g[b][idx], "ref", og[b][idx])
for (W,H,B,n) in [(32,24,10,2000),(346,260,10,100000)]:
    w = smooth_window(W,H,B,n)
    sl = P.EventSlice(w.W, w.H, int(w.edges[0]), int(w.edges[-1]), w.events)
    fl = P.FlowSequence(w.edges.copy(), w.flows.copy())
    fwd = eng.forward(sl, fl); g = eng.backward(sl, fl, fwd).grad
    ref = O.forward(w); og = O.backward(w, ref)
    print("smooth", W, H, "rel", rel_inf(g, og))
