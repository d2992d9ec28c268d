"""Benchmark of the B200 CMax loss path (DESIGN.md §6 Measurement).

One step = one pass of the hot path over one batch of synthetic windows:
motion field (depth + poses -> flows) -> warp + splat -> focus loss ->
per-event backward -> flows backward (d_depth, d_poses), i.e. the
predictor_loss_and_gradients composition (optimize.hpp:205-241) without decode
and L_geo, followed by the data-parallel reduction of [loss, d_depth, d_poses]
(NCCL all-reduce across ranks when N > 1, overlapped with the next batch).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload S|C|B|A]
    python bench.py --impl reference ...   # the reference CPU path on this host

The default workload is S, the configuration BASELINE.json's metric is quoted
on ("... at 1/2/4/8 B200" = configs[4]: 64 DSEC-shape windows of 1M events,
split over the GPUs). ``--gpus N`` without a torchrun environment re-launches
this script under ``torch.distributed.run`` with N ranks (one process per GPU).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

EVENT_DTYPE = np.dtype({"names": ["t_us", "x", "y", "p"], "formats": ["<u8", "<u2", "<u2", "i1"],
                        "offsets": [0, 8, 10, 12], "itemsize": 16})

WORKLOADS = {
    # BASELINE.json configs[0]: the reference's own CPU-runnable case, one window
    "A": dict(W=128, H=128, B=10, n_events=20_000, batch=1, window_us=100_000,
              name="128x128 window (drone-downsampled), 20k events, batch 1, "
                   "10 bins (11 refs), 0.1 s windows"),
    # BASELINE.json configs[1]: MVSEC-shape windows, ~100k events each, batch 8, 1 B200
    "B": dict(W=346, H=260, B=10, n_events=100_000, batch=8, window_us=100_000,
              name="MVSEC-shape 346x260 windows, 100k events/window, batch 8 per GPU, "
                   "10 bins (11 refs), 0.1 s windows"),
    # BASELINE.json configs[2]: DSEC-shape windows, ~1M events each, batch 16, 1 B200
    "C": dict(W=640, H=480, B=10, n_events=1_000_000, batch=16, window_us=100_000,
              name="DSEC-shape 640x480 windows, 1M events/window, batch 16 per GPU, "
                   "10 bins (11 refs), 0.1 s windows"),
    # BASELINE.json configs[4] (the metric's "at 1/2/4/8 B200" configuration):
    # a fixed batch of 64 DSEC-shape windows split over the GPUs (strong scaling)
    "S": dict(W=640, H=480, B=10, n_events=1_000_000, batch_total=64, window_us=100_000,
              name="configs[4]: batch 64 x DSEC-shape 640x480 windows, 1M events/window, "
                   "split over the GPUs, 10 bins (11 refs), 0.1 s windows"),
}
# SURVEY.md §8(d) sweep: one 346x260 window, N events
SWEEP_N = (10_000, 30_000, 100_000, 300_000, 1_000_000, 3_000_000, 10_000_000)

HBM_PEAK_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback
L2_BYTES = 126 * 1024 * 1024
METRIC = "CMax loss fwd+bwd throughput"


def measured_traffic(workload, kernel, world):
    """DRAM bytes (read + write) per launch of `kernel` from one committed
    `ncu --set full` capture of this workload on 1 GPU (profiles/traffic.json);
    None when not captured (or for N > 1, where the capture was not repeated)."""
    if world != 1:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload, {}).get(kernel)
    except Exception:
        return None


def measured_ceilings(workload, kernel, world):
    """Utilisation of the candidate ceilings (shared-memory / L1 data pipe,
    shared atomics, L1 writeback, fp64 pipe, issue, DRAM; % of peak) of
    `kernel` from the committed `ncu --set full` capture of this workload on
    1 GPU (profiles/ceilings.json, tools/ncu_ceilings_json.py); `binding` names
    the busiest one. This path is gather/atomic work, so the HBM roofline alone
    does not say what bounds a kernel (SURVEY.md §8(d) secondary ceilings)."""
    if world != 1:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "ceilings.json")) as f:
            return json.load(f).get(workload, {}).get(kernel)
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# synthetic inputs (SURVEY.md §8(d) chain-level input)


def make_inputs(wl, rank, n_windows):
    """Two fronto-parallel planes (depth 1.0 | 3.0), per-bin ego-motion
    omega=(0.001,-0.002,0.003), t=(0.02,0.01,0.005), K=(0.9W,0.9W,(W-1)/2,(H-1)/2);
    events uniform in (t, x, y) with alternating polarity (bench_window semantics,
    bench.hpp:112-141). All values fp32-representable. The depth map and poses
    are shared by every window (data-parallel batch over one parameter set)."""
    W, H, B, n = wl["W"], wl["H"], wl["B"], wl["n_events"]
    rng = np.random.default_rng(1000 + rank)
    depth = np.empty((H, W))
    depth[:, : W // 2] = 1.0
    depth[:, W // 2:] = 3.0
    depth = np.broadcast_to(depth, (n_windows, H, W)).copy()
    poses = np.tile(np.array([0.001, -0.002, 0.003, 0.02, 0.01, 0.005]), (n_windows, B, 1))
    poses = poses.astype(np.float32).astype(np.float64)
    K = np.array([0.9 * W, 0.9 * W, (W - 1) / 2, (H - 1) / 2]).astype(np.float32).astype(np.float64)
    ev = np.zeros(n * n_windows, EVENT_DTYPE)
    for w in range(n_windows):
        s = slice(w * n, (w + 1) * n)
        ev["t_us"][s] = np.sort(rng.integers(0, wl["window_us"], n))
        ev["x"][s] = rng.integers(0, W, n)
        ev["y"][s] = rng.integers(0, H, n)
        ev["p"][s] = np.where(np.arange(n) % 2 == 0, 1, -1)
    offs = np.arange(n_windows + 1, dtype=np.uint64) * n
    return depth, poses, K, ev, offs


# SURVEY.md §8(d) precisions: canonical parity precision (depth f32, flows f64,
# stack f32, gradients f32) -> b_px = 1180 B at B = 10; this build's own
# precisions (depth f64, flows f64, stack f64, gradients f32) -> 1720 B.
CANONICAL = dict(sd=4, sf=8, ss=4, sg=4)
BUILD_PRECISION = dict(sd=8, sf=8, ss=8, sg=4)


def algorithmic_bytes(wl, n_windows, algo="owner", prec=CANONICAL):
    """bytes = N*b_ev + HW*b_px per window, b_ev = 18 B,
    b_px = 3 s_d + 6B s_f + 12(B+1) s_s + 4B s_g. Returns the total and the
    per-kernel split used by the roofline object: each model term is attributed
    to the kernel implementing that stage of the reference (fused kernels carry
    the terms of every stage they absorb)."""
    B, HW, n = wl["B"], wl["W"] * wl["H"], wl["n_events"]
    sd, sf, ss, sg = prec["sd"], prec["sf"], prec["ss"], prec["sg"]
    if algo == "owner":
        per = {
            "motion_field": HW * (sd + 2 * B * sf),                       # K1: depth read, flow write
            "traj_records": n * 9 + HW * 2 * B * sf,                      # K2: events, flow gather
            "fwd_owner": HW * 8 * (B + 1) * ss,                           # K3 write + K3b read
            "bwd_event": n * 9 + HW * (2 * B * sf + 4 * (B + 1) * ss),    # K4 gathers
            "bwd_owner": HW * (4 * B * sg + 2 * sd),                      # K4 grad write+read, K5
        }
    else:
        per = {
            "motion_field": HW * (sd + 2 * B * sf),
            "warp_splat": n * 9 + HW * (2 * B * sf + 4 * (B + 1) * ss),
            "loss_reduce": HW * 4 * (B + 1) * ss,
            "backward": n * 9 + HW * (2 * B * sf + 4 * (B + 1) * ss + 2 * B * sg),
            "flows_backward": HW * (2 * B * sg + 2 * sd),
        }
    per = {k: v * n_windows for k, v in per.items()}
    return sum(per.values()), per


# evcm_cuda_stage_times order per pipeline (include/evcm_cuda.h)
STAGES_BY_ALGO = {
    "owner": ["staging", "motion_field", "sort", "traj_records", "fwd_owner", "loss_finalize",
              "bwd_event", "bwd_owner", "pose_contract"],
    "atomic": ["staging", "motion_field", "stack_memset", "warp_splat", "loss_reduce",
               "grad_memset", "backward", "flows_backward", "unused"],
}
# the reference's four PhaseStats phases (bench.hpp:64) over the owner stages
PHASES = {"warp": ["staging", "motion_field", "sort", "traj_records"], "splat": ["fwd_owner"],
          "loss": ["loss_finalize"], "backward": ["bwd_event", "bwd_owner", "pose_contract"]}
CSV_HEADER = ["backend", "phase", "n_events", "time_us", "peak_bytes", "loss",  # bench.hpp:98
              "gpus", "mevents_per_s", "windows_per_s", "hbm_gbs", "roofline_frac", "cpu_cores"]


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.idx = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# multi-rank plumbing


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_ranks(n):
    """`--gpus N` outside torchrun: one process per GPU under
    torch.distributed.run (rendezvous on 127.0.0.1); rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    return subprocess.call(cmd, env=env)


def rank_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def windows_per_rank(wl, world):
    if "batch_total" in wl:  # strong scaling: the fixed batch is split over the ranks
        if wl["batch_total"] % world:
            raise SystemExit(f"workload needs a GPU count dividing {wl['batch_total']}")
        return wl["batch_total"] // world
    return wl["batch"]


def max_over_ranks(value, world, device=None):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# reference arm / cpu baseline


def run_reference_chain(wl, depth, poses, K, ev, offs, windows, n_workers=0):
    from oracle import oracle as O
    d = np.ascontiguousarray(depth[windows])
    p = np.ascontiguousarray(poses[windows])
    evs = [ev[int(offs[w]):int(offs[w + 1])] for w in windows]
    o = np.zeros(len(windows) + 1, np.uint64)
    o[1:] = np.cumsum([len(x) for x in evs])
    r = O.ref_chain_batch(d, p, K, 0, wl["window_us"], np.concatenate(evs).astype(EVENT_DTYPE), o,
                          n_workers=n_workers)
    return r["seconds"], int(o[-1])


def cpu_baseline(wl, depth, poses, K, ev, offs, budget_s=12.0):
    """The reference itself (oracle/_ref/libevcm_ref.so, built from /root/reference
    with its Release flags) on this host's cores: one warm-up window, then
    windows until ~budget_s of CPU work (>= 2 windows)."""
    from oracle import oracle as O
    if not O.ref_available():
        return {"value": None, "unit": "Mevents/s", "cores": os.cpu_count(), "kind": "reference",
                "sample": "unavailable: oracle/_ref/libevcm_ref.so not built"}
    cores = int(O.ref().ref_hardware_concurrency())
    run_reference_chain(wl, depth, poses, K, ev, offs, [0])
    secs, evs, nwin = 0.0, 0, 0
    while (secs < budget_s or nwin < 2) and nwin < 64:
        s, n = run_reference_chain(wl, depth, poses, K, ev, offs, [nwin % depth.shape[0]])
        secs += s
        evs += n
        nwin += 1
    return {"value": evs / secs / 1e6, "unit": "Mevents/s", "cores": cores, "kind": "reference",
            "sample": f"{nwin} windows of the workload (window by window, as optimize.hpp:327-371), "
                      f"{secs:.1f} s, depth_pose_to_flows + Engine::loss_and_grad (parallel, "
                      f"deterministic, n_workers=0) + depth_pose_to_flows_backward",
            "windows_per_s": nwin / secs}


def reference_arm(args, wl):
    world, rank, _ = rank_env()
    if rank != 0:
        return
    nb = min(wl.get("batch", wl.get("batch_total", 4)), 4)  # distinct windows sampled
    depth, poses, K, ev, offs = make_inputs(wl, 0, nb)
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libevcm_ref.so not built"}))
        return
    cores = int(O.ref().ref_hardware_concurrency())
    for i in range(args.warmup):
        run_reference_chain(wl, depth, poses, K, ev, offs, [i % nb])
    times, n_ev = [], 0
    for i in range(args.steps):
        s, n = run_reference_chain(wl, depth, poses, K, ev, offs, [i % nb])
        times.append(s)
        n_ev += n
    total = sum(times)
    value = n_ev / total / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "Mevents/s", "n_gpus": max(args.gpus, world), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong" if "batch_total" in wl else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["name"], "step": "one window per step (bounded sample of the "
                   "workload; the reference runs windows one at a time, optimize.hpp:327-371)",
                   "events_per_window": wl["n_events"]},
        "windows_per_s": args.steps / total,
        "cpu_baseline": {"value": value, "unit": "Mevents/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} windows, one per step"},
        "e2e": {"value": value, "unit": "Mevents/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if args.csv:
        with open(args.csv, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(CSV_HEADER)
            w.writerow(["reference-parallel", "total", wl["n_events"], 1e6 * total / args.steps, 0,
                        "", 1, value, args.steps / total, "", "", cores])
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# CUDA arm


def cuda_arm(args, wl):
    import torch
    import torch.distributed as dist

    world, rank, local = rank_env()
    # one process per GPU; --dist-backend gloo + device sharing only for smoke-testing
    # the multi-rank path on a single-GPU box
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    dev = torch.device("cuda", local)

    import paper_2412_06359_b200 as P
    from paper_2412_06359_b200.dist import OverlappedAllReduce

    nwin = windows_per_rank(wl, world)
    depth, poses, K, ev, offs = make_inputs(wl, rank, nwin)
    stream = torch.cuda.Stream(dev)
    # default options: deterministic (engine.hpp:60) -> the owner-computes pipeline
    eng = P.Engine(P.EngineOptions(device=local, stream=stream.cuda_stream, algo=args.algo,
                                   deterministic=args.algo != "atomic"))
    HW, B = wl["W"] * wl["H"], wl["B"]
    n_sums = 1 + HW + B * 6

    # device-resident inputs / outputs
    with torch.cuda.stream(stream):
        d_depth = torch.from_numpy(depth).to(dev)
        d_poses = torch.from_numpy(poses).to(dev)
        d_ev = torch.from_numpy(ev.view(np.uint8)).to(dev)
        out = (torch.empty(nwin, dtype=torch.float64, device=dev),
               torch.empty((nwin, wl["H"], wl["W"]), dtype=torch.float64, device=dev),
               torch.empty((nwin, wl["B"], 6), dtype=torch.float64, device=dev))
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream.synchronize()
    red = OverlappedAllReduce(n_sums, dev)

    # L2 policy: a step whose algorithmic traffic is far above the 126 MB L2 needs
    # no flush (its inputs cannot stay resident), and the whole loop is timed in
    # one bracket so the overlapped all-reduces are inside it; small steps get an
    # untimed 256 MB flush before each individually timed step
    step_bytes, _ = algorithmic_bytes(wl, nwin)
    flush_each = step_bytes < 4 * L2_BYTES

    def launch(i):
        slot = i % 2
        if i >= 2:
            eng.chain_wait(slot)  # step i-2's validation result (host wait)
        buf = red.buffer(i)  # the stream waits for step i-2's all-reduce
        eng.chain_batch_async(d_depth, d_poses, K, 0, wl["window_us"], d_ev, offs, out, slot,
                              sums=buf)
        red.submit(i)

    with torch.cuda.stream(stream):
        # >= 4 launches: each slot's signature runs eagerly once, is captured into a
        # CUDA graph on its second call, and replays from then on
        for i in range(max(args.warmup, 4)):
            launch(i)
        red.drain()
        for slot in range(2):
            eng.chain_wait(slot)
        stream.synchronize()
        launches_per_step = eng.last_launch_count()
        algo_ran = eng.last_algo()
        STAGES = STAGES_BY_ALGO[algo_ran]

        # timed steps replay the engine's captured CUDA graph of the chain
        eng.set_timing(False)
        clocks = ClockSampler(local)
        flush.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        clocks.start()
        time.sleep(0.3)
        if flush_each:
            starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            for i in range(args.steps):
                flush.zero_()  # untimed L2 flush
                starts[i].record(stream)
                launch(i)
                red.drain()
                ends[i].record(stream)
            for slot in range(2):
                eng.chain_wait(slot)
            torch.cuda.synchronize(dev)
            total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
        else:
            t0e = torch.cuda.Event(enable_timing=True)
            t1e = torch.cuda.Event(enable_timing=True)
            t0e.record(stream)
            for i in range(args.steps):
                launch(i)
            red.drain()
            t1e.record(stream)
            for slot in range(2):
                eng.chain_wait(slot)
            torch.cuda.synchronize(dev)
            total_ms = t0e.elapsed_time(t1e)
        clk = clocks.stop()
        if world > 1:
            dist.barrier()
        reduced = red.bufs[(args.steps - 1) % 2].clone()
        step_loss = float(out[0].sum().item())

        # per-stage breakdown: separate untimed pass, eager launches with CUDA
        # events between the stages on the engine's stream
        eng.set_timing(True)
        n_stage = min(args.steps, 3)
        stage_ms = np.zeros(len(STAGES))
        for i in range(n_stage):
            flush.zero_()
            eng.chain_batch(d_depth, d_poses, K, 0, wl["window_us"], d_ev, offs, out=out)
            stage_ms += np.array((eng.stage_times_ms() + [0.0] * len(STAGES))[: len(STAGES)])
        torch.cuda.synchronize(dev)
        eng.set_timing(False)
        stage_ms /= n_stage
        if world > 1:
            dist.barrier()
    total_ms = max_over_ranks(total_ms, world, dev)
    ms_per_step = total_ms / args.steps
    events_per_step = wl["n_events"] * nwin * world
    value = events_per_step * args.steps / (total_ms * 1e-3) / 1e6
    windows_per_s = nwin * world * args.steps / (total_ms * 1e-3)

    # ---- roofline of the dominant kernel (per-launch algorithmic bytes / its
    # average CUDA-event duration on the launching stream)
    peak, peak_kind = peaks()
    total_bytes, per_kernel = algorithmic_bytes(wl, nwin, algo_ran)
    total_bytes_bp, _ = algorithmic_bytes(wl, nwin, algo_ran, BUILD_PRECISION)
    kern = {k: stage_ms[STAGES.index(k)] for k in per_kernel}
    dom = max(kern, key=kern.get)
    achieved = per_kernel[dom] / (kern[dom] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                "traffic": measured_traffic(args.workload, dom, world),
                "ceilings": measured_ceilings(args.workload, dom, world),
                "algorithmic_bytes_per_launch": per_kernel[dom], "launch_ms": kern[dom],
                "bytes_model": "SURVEY.md §8(d) canonical parity precision (b_ev 18 B, "
                               "b_px 1180 B at B=10), per-kernel split of bench.py "
                               "algorithmic_bytes"}
    step_gbs = total_bytes / (ms_per_step * 1e-3) / 1e9 * world
    step_roofline = {"algorithmic_bytes_per_step_per_gpu": total_bytes,
                     "achieved_GBps_per_gpu": step_gbs / world,
                     "frac": step_gbs / world / peak,
                     "frac_build_precision": total_bytes_bp / (ms_per_step * 1e-3) / 1e9 / peak,
                     "stage_ms": {s: round(float(m), 4) for s, m in zip(STAGES, stage_ms)}}

    # ---- e2e: public API with pinned host buffers, H2D and D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        h_depth = torch.from_numpy(depth).pin_memory()
        h_poses = torch.from_numpy(poses).pin_memory()
        h_ev = torch.from_numpy(ev.view(np.uint8)).pin_memory()
        # the public pipelined feed (paper_2412_06359_b200/pipeline.py): batch
        # i+1's pinned host -> device copy overlaps batch i's compute; every
        # batch's reduced result is read back by the host
        pipe = P.ChainPipeline(eng, compute_stream=stream)
        flush160 = flush[: 160 * 1024 * 1024 // 4]
        from paper_2412_06359_b200.dist import allreduce_window_sums

        def post(sums):  # the chain's packed window sums; all-reduce over ranks
            allreduce_window_sums(sums)
            if flush_each:
                flush160.zero_()
            return sums

        def batches(n):
            for _ in range(n):
                yield (h_depth, h_poses, h_ev, offs)

        for _ in pipe.run(batches(max(4, args.warmup)), K, 0, wl["window_us"], post=post,
                          window_sums=True):
            pass
        t0e = torch.cuda.Event(enable_timing=True)
        t1e = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0e.record(stream)
        pipe.copy.wait_event(t0e)  # the first batch's copy is inside the timed region
        n_done, d2h = 0, 0
        for res in pipe.run(batches(args.steps), K, 0, wl["window_us"], post=post,
                            window_sums=True):
            n_done += 1
            d2h = res.numel() * res.element_size()
        t1e.record(stream)
        torch.cuda.synchronize(dev)
        assert n_done == args.steps
        e2e_ms = max_over_ranks(t0e.elapsed_time(t1e), world, dev)
        e2e = {"value": events_per_step * args.steps / (e2e_ms * 1e-3) / 1e6, "unit": "Mevents/s",
               "h2d_bytes_per_step": int(h_depth.numel() * 8 + h_poses.numel() * 8 + h_ev.numel()),
               "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_ms / args.steps,
               "api": "ChainPipeline.run (double-buffered H2D overlapping compute; the reduced "
                      "[loss, d_depth, d_poses] of every batch read back to the host)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, depth, poses, K, ev, offs, budget_s=args.cpu_budget_s)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mevents/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if "batch_total" in wl else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["name"], "windows_per_gpu_per_step": nwin,
                       "events_per_window": wl["n_events"], "sensor": [wl["W"], wl["H"]],
                       "bins": wl["B"],
                       "numerics": "fp64 trajectories, positions, weights, flows and loss "
                                   "(bit-exact trajectories); bilinear fractions stored as "
                                   "fp32 (full relative precision of the smaller side); IWE "
                                   "stack and flow-gradient tiles as exact 64-bit fixed point "
                                   "(2^-50 weight resolution); per-event adjoint sink values "
                                   "fp32; fp64 coefficient planes and pose/depth gradients",
                       "l2": ("untimed 256 MB flush before every timed step" if flush_each else
                              f"no flush: the step's algorithmic traffic "
                              f"({step_bytes / 1e9:.1f} GB per GPU) is far above the 126 MB L2; "
                              f"the K steps are timed as one bracket"),
                       "mode": f"deterministic={eng.opts.deterministic} (algo {args.algo} -> "
                               f"{algo_ran})",
                       "inputs": "two-plane depth + per-bin ego-motion, uniform events",
                       "parallelism": f"dp{world} (windows sharded, NCCL all-reduce of "
                                      "loss/d_depth/d_poses overlapped with the next batch)"},
            "windows_per_s": windows_per_s,
            "hbm_GBps_step": step_gbs,
            "roofline": roofline,
            "step_roofline": step_roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
            "check": {"sum_loss_last_step": step_loss, "reduced_loss": float(reduced[0].item())},
        }
        if args.csv:
            ws = eng.workspace_bytes()
            with open(args.csv, "w", newline="") as f:
                w = csv.writer(f)
                w.writerow(CSV_HEADER)
                for ph, stages in PHASES.items():
                    t_us = 1e3 * sum(stage_ms[STAGES.index(s)] for s in stages if s in STAGES)
                    w.writerow(["cuda", ph, events_per_step // world, t_us, ws, step_loss, world,
                                value, windows_per_s, step_gbs, step_roofline["frac"],
                                (cpu or {}).get("cores", "")])
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU self-test of the rank path (gloo): sharding, overlapped all-reduce,
# max-over-ranks timing, rank-0 line -- with a stub step in place of the chain


def cpu_harness(args, wl):
    import torch
    import torch.distributed as dist
    from paper_2412_06359_b200.dist import OverlappedAllReduce, shard_windows
    world, rank, _ = rank_env()
    if world > 1:
        dist.init_process_group("gloo")
    total_windows = wl.get("batch_total", wl.get("batch", 1) * world)
    mine = shard_windows(total_windows, world, rank)
    if "batch_total" in wl:
        assert len(mine) == windows_per_rank(wl, world)
    red = OverlappedAllReduce(4, "cpu")
    t0 = time.perf_counter()
    for i in range(args.steps):
        buf = red.buffer(i)
        # stub chain: window w contributes (1, w, w^2, step) to the packed sums
        buf.zero_()
        for w in mine:
            buf += torch.tensor([1.0, float(w), float(w * w), float(i)], dtype=torch.float64)
        red.submit(i)
    red.drain()
    ms = max_over_ranks(1e3 * (time.perf_counter() - t0), world)
    last = red.bufs[(args.steps - 1) % 2]
    if rank == 0:
        print(json.dumps({"harness": "cpu-stub", "n_gpus": world, "steps": args.steps,
                          "windows_per_rank": len(mine), "ms_per_step": ms / args.steps,
                          "reduced": [float(x) for x in last]}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def sweep(args):
    """SURVEY.md §8(d) sweep: one 346x260 window with N events, device-resident
    chain (graph replay), L2 flushed between steps; one JSON line per N."""
    import torch
    import paper_2412_06359_b200 as P
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    eng = P.Engine(P.EngineOptions(stream=stream.cuda_stream, algo=args.algo,
                                   deterministic=args.algo != "atomic"))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for n in SWEEP_N:
        wl = dict(WORKLOADS["B"], n_events=n)
        depth, poses, K, ev, offs = make_inputs(wl, 0, 1)
        with torch.cuda.stream(stream):
            d_depth = torch.from_numpy(depth).to(dev)
            d_poses = torch.from_numpy(poses).to(dev)
            d_ev = torch.from_numpy(ev.view(np.uint8)).to(dev)
            out = (torch.empty(1, dtype=torch.float64, device=dev),
                   torch.empty((1, wl["H"], wl["W"]), dtype=torch.float64, device=dev),
                   torch.empty((1, wl["B"], 6), dtype=torch.float64, device=dev))
            for _ in range(max(3, args.warmup)):
                eng.chain_batch(d_depth, d_poses, K, 0, wl["window_us"], d_ev, offs, out=out)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for a, b in evs:
                flush.zero_()
                a.record(stream)
                eng.chain_batch(d_depth, d_poses, K, 0, wl["window_us"], d_ev, offs, out=out)
                b.record(stream)
        torch.cuda.synchronize(dev)
        ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
        print(json.dumps({"sweep": "346x260, 1 window, 10 bins", "n_events": n,
                          "ms_per_window": ms, "Mevents_per_s": n / (ms * 1e-3) / 1e6,
                          "algo": eng.last_algo(), "steps": args.steps}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--workload", default="S", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--algo", default="auto", choices=["auto", "owner", "atomic"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    ap.add_argument("--csv", default="", help="also write the phase CSV (bench.hpp:94-104 schema "
                                              "+ gpus, mevents_per_s, windows_per_s, hbm_gbs, "
                                              "roofline_frac, cpu_cores)")
    ap.add_argument("--dist-backend", default="nccl", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-harness", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--sweep", action="store_true",
                    help="SURVEY §8(d) sweep (346x260, 1 window, 1e4..1e7 events); not the contract line")
    ap.add_argument("--events", type=int, default=0, help="override events per window (exploration)")
    ap.add_argument("--batch", type=int, default=0, help="override windows per GPU (exploration)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_ranks(args.gpus))
    if args.sweep:
        sweep(args)
        return
    wl = dict(WORKLOADS[args.workload])
    if args.events:
        wl.update(n_events=args.events, name=wl["name"] + f" [events/window overridden: {args.events}]")
    if args.batch:
        wl.pop("batch_total", None)
        wl.update(batch=args.batch, name=wl["name"] + f" [batch overridden: {args.batch}]")
    if args.cpu_harness:
        cpu_harness(args, wl)
    elif args.impl == "reference":
        reference_arm(args, wl)
    else:
        cuda_arm(args, wl)


if __name__ == "__main__":
    main()
