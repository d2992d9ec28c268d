"""run_window drift vs the reference for several engine configurations."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2412_06359_b200 as P
from tests.golden_io import load
from tests.helpers import rel_inf
from tests.test_run_window import _windows, _cfg

g = load("run_window")
confs = {"owner_f32": dict(), "atomic_f32": dict(algo="atomic", deterministic=False),
         "atomic_f64": dict(algo="atomic", deterministic=False, grad_f64=True)}
confs["owner_f64"] = dict(grad_f64=True)
for lam in (0.0, 0.05):
    key = str(lam).replace(".", "p")
    ref = g[f"rec_{key}"]
    for name, o in confs.items():
        e = P.Engine(P.EngineOptions(**o))
        pred = P.DirectPredictor(g["params"].copy(), g["poses"].copy(), int(g["factor"]))
        r = P.run_window(_windows(g), pred, g["K"], _cfg(g, lam), engine=e)
        rec = np.array([[x.l_cm, x.l_geo, x.total, x.rsat, x.grad_norm_depth, x.grad_norm_pose]
                        for x in r.log.records])
        errs = [rel_inf(rec[u], ref[u]) for u in range(len(ref))]
        print(lam, name, " ".join(f"{x:.1e}" for x in errs),
              "params", f"{rel_inf(r.predictor.depth_params, g[f'params_{key}']):.1e}")
