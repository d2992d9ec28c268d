"""Does the pipelined H2D copy slow the chain down? Device-resident S-size chain
steps timed alone and with a concurrent 1.18 GB pinned H2D copy per step on a
side stream (what ChainPipeline does)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import bench
import paper_2412_06359_b200 as P

wl = bench.WORKLOADS["S"]
depth, poses, K, ev, offs = bench.make_inputs(wl, 0, 64)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
eng = P.Engine(P.EngineOptions(stream=stream.cuda_stream))
with torch.cuda.stream(stream):
    d_depth = torch.from_numpy(depth).to(dev)
    d_poses = torch.from_numpy(poses).to(dev)
    d_ev = torch.from_numpy(ev.view(np.uint8)).to(dev)
    out = (torch.empty(64, dtype=torch.float64, device=dev),
           torch.empty((64, wl["H"], wl["W"]), dtype=torch.float64, device=dev),
           torch.empty((64, wl["B"], 6), dtype=torch.float64, device=dev))
h_ev = torch.from_numpy(ev.view(np.uint8)).pin_memory()
h_depth = torch.from_numpy(depth).pin_memory()
dst_ev = torch.empty_like(d_ev)
dst_depth = torch.empty_like(d_depth)
copy = torch.cuda.Stream(dev)
for _ in range(3):
    eng.chain_batch(d_depth, d_poses, K, 0, wl["window_us"], d_ev, offs, out=out)
torch.cuda.synchronize()
for mode in ("alone", "with H2D", "alone", "with H2D"):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for i in range(5):
        if mode != "alone":
            with torch.cuda.stream(copy):
                dst_ev.copy_(h_ev, non_blocking=True)
                dst_depth.copy_(h_depth, non_blocking=True)
        eng.chain_batch(d_depth, d_poses, K, 0, wl["window_us"], d_ev, offs, out=out)
    b.record(stream)
    torch.cuda.synchronize()
    print(f"{mode:9s}: {a.elapsed_time(b) / 5:.2f} ms per step")
