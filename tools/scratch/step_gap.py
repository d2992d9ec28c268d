"""Per-step device time of the S chain: sync chain_batch vs the bench's async
two-slot loop (chain_batch_async + chain_wait, packed window sums)."""
import os, sys
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
    sums = [torch.zeros(1 + wl["H"] * wl["W"] + wl["B"] * 6, dtype=torch.float64, device=dev) for _ in range(2)]
torch.cuda.synchronize()


def run(mode, n=6):
    with torch.cuda.stream(stream):
        for i in range(4):
            if mode == "sync":
                eng.chain_batch(d_depth, d_poses, K, 0, wl["window_us"], d_ev, offs, out=out)
            else:
                if i >= 2:
                    eng.chain_wait(i % 2)
                eng.chain_batch_async(d_depth, d_poses, K, 0, wl["window_us"], d_ev, offs, out, i % 2,
                                      sums=sums[i % 2] if mode == "async+sums" else None)
        if mode != "sync":
            for s in range(2):
                eng.chain_wait(s)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(n):
            if mode == "sync":
                eng.chain_batch(d_depth, d_poses, K, 0, wl["window_us"], d_ev, offs, out=out)
            else:
                if i >= 2:
                    eng.chain_wait(i % 2)
                eng.chain_batch_async(d_depth, d_poses, K, 0, wl["window_us"], d_ev, offs, out, i % 2,
                                      sums=sums[i % 2] if mode == "async+sums" else None)
        b.record(stream)
        if mode != "sync":
            for s in range(2):
                eng.chain_wait(s)
        torch.cuda.synchronize()
        print(f"{mode:11s}: {a.elapsed_time(b) / n:.2f} ms per step, launches {eng.last_launch_count()}")


for mode in ("sync", "async", "async+sums", "sync", "async", "async+sums"):
    run(mode)
import subprocess
p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                      "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
print("with nvidia-smi -lms 100:")
run("async+sums")
run("async+sums")
p.terminate(); p.communicate()
