"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
the batched chain (owner and atomic pipelines), forward/backward, L_geo,
ingestion and the predictor chain on tiny inputs. Usage:
compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_06359_b200 as P  # noqa: E402
from tests.helpers import chain_inputs  # noqa: E402

for algo in ("owner", "atomic"):
    eng = P.Engine(P.EngineOptions(algo=algo, deterministic=algo != "atomic"))
    depth, poses, K, ev, offs = chain_inputs(40, 30, 4, 3, 2500, seed=1)
    loss, dd, dp = eng.chain_batch(depth, poses, K, 0, 100000, ev, offs)
    gf = eng.depth_pose_to_flows(depth[0], poses[0], K, 0, 100000)
    sl = P.EventSlice(40, 30, 0, 100000, ev[: int(offs[1])])
    f, b = eng.loss_and_grad(sl, gf.flows)
    _ = f.stack, f.traj
    print(algo, float(loss[0]), f.loss.value)
b = P.geometry_consistency_loss_batch(depth[0], depth[0], poses[0], K)
print("geo", b.value.tolist()[:2])
e = P.Engine()
print("offsets", e.window_offsets(ev[: int(offs[1])], 0, 25000, 4).tolist())
e.validate_slice(sl)
pred = P.DirectPredictor(np.zeros((3, 4)), poses[0], 10)
wg = P.predictor_loss_and_gradients(pred, sl, K, lambda_geo=0.05)
print("predictor", wg.total)
torch.cuda.synchronize()
print("sanitize smoke done")
