import sys
import numpy as np
sys.path.insert(0, '/root/repo')
import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.helpers import rel_inf, smooth_window

w = smooth_window(32, 24, 3, 800, seed=32 + 800)
B = 3
zero = np.zeros((B, 2, w.H, w.W))
w0 = O.Window(w.W, w.H, w.edges, w.events, zero)
f = O.forward(w0); og = O.backward(w0, f)
e = P.Engine()
sl = P.EventSlice(w.W, w.H, 0, 100000, w.events)
fl = P.FlowSequence(w.edges.copy(), zero.copy())
fw, bw = e.loss_and_grad(sl, fl)
g = bw.grad
print("loss", fw.loss.value, f["loss"], "grad rel", rel_inf(g, og))
nz_ref = og != 0; nz = g != 0
print("nonzero mismatch", int((nz_ref != nz).sum()), "of", g.size)
idx = np.argsort(-np.abs(g - og).ravel())[:5]
print("worst", [(float(g.ravel()[i]), float(og.ravel()[i])) for i in idx])
# one Adam step each
s1 = np.zeros(g.size); m = np.zeros(g.size); v = np.zeros(g.size)
O.adam_step(s1, og.ravel(), m, v, 1, 0.5)
s2 = np.zeros(g.size); m2 = np.zeros(g.size); v2 = np.zeros(g.size)
O.adam_step(s2, g.ravel(), m2, v2, 1, 0.5)
d = np.abs(s1 - s2)
print("step diff max", d.max(), "at", int(d.argmax()), "g", float(g.ravel()[d.argmax()]), "og", float(og.ravel()[d.argmax()]))
# loss at the stepped flows
w1 = O.Window(w.W, w.H, w.edges, w.events, s1.reshape(zero.shape))
w2 = O.Window(w.W, w.H, w.edges, w.events, s2.reshape(zero.shape))
print("oracle loss after step: ref-grad", O.forward(w1)["loss"], "gpu-grad", O.forward(w2)["loss"])
