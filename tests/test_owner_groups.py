"""Owner kernels split over CTA groups (references in the forward, bins in the
backward, cmax_cells.cu) when tiles x windows alone leave SMs idle. The split
must not change a single bit: every tile sums the same fixed-point terms, and
d_depth is re-formed in bin order. Each run is a fresh process, the group
counts forced through EVCM_FWD_GROUPS / EVCM_BWD_GROUPS."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2412_06359_b200 as P
from tests.helpers import chain_inputs, contraction_window, smooth_window
out = {{}}
eng = P.Engine(P.EngineOptions(algo="owner"))
for (W, H, B, nw, n, seed) in [(128, 128, 10, 1, 20000, 1), (200, 150, 7, 3, 60000, 2),
                               (64, 48, 3, 2, 0, 3), (96, 64, 2, 2, 9000, 4)]:
    depth, poses, K, ev, offs = chain_inputs(W, H, B, nw, n, seed=seed) if n else \
        chain_inputs(W, H, B, nw, 1, seed=seed)
    if not n:
        ev, offs = ev[:0], np.zeros(nw + 1, dtype=np.uint64)
    l, dd, dp = eng.chain_batch(depth, poses, K, 0, 100000, ev, offs)
    out[f"c{{seed}}"] = np.concatenate([np.ravel(l), np.ravel(dd), np.ravel(dp)])
w = smooth_window(160, 120, 10, 30000, seed=5)
sl = P.EventSlice(w.W, w.H, int(w.edges[0]), int(w.edges[-1]), w.events)
fl = P.FlowSequence(w.edges.copy(), w.flows.copy())
f = eng.forward(sl, fl)
g = eng.backward(sl, fl, f)
out["loss"] = np.array([f.loss.value])
out["stack"] = np.concatenate([np.ravel(f.stack.count), np.ravel(f.stack.tsum)])
out["grad"] = np.ravel(g.grad)
w = contraction_window(256, 192, 6, 40000, factor=0.15)  # overflowed owner lists
sl = P.EventSlice(w.W, w.H, int(w.edges[0]), int(w.edges[-1]), w.events)
fl = P.FlowSequence(w.edges.copy(), w.flows.copy())
f = eng.forward(sl, fl)
out["c_loss"] = np.array([f.loss.value])
out["c_grad"] = np.ravel(eng.backward(sl, fl, f).grad)
np.savez(sys.argv[1], **out)
"""


def _run(tmp_path, fwd, bwd):
    path = str(tmp_path / f"g_{fwd}_{bwd}.npz")
    env = dict(os.environ, EVCM_FWD_GROUPS=str(fwd), EVCM_BWD_GROUPS=str(bwd))
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), path], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(path))


def test_groups_are_bit_identical(tmp_path):
    base = _run(tmp_path, 1, 1)
    for fwd, bwd in [(2, 2), (4, 3), (11, 10), (3, 6)]:
        other = _run(tmp_path, fwd, bwd)
        assert base.keys() == other.keys()
        for k in base:
            np.testing.assert_array_equal(base[k], other[k], err_msg=f"{k} fwd={fwd} bwd={bwd}")
