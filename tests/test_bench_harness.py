"""CPU: bench.py's multi-rank path. ``--gpus 2`` outside torchrun re-launches
the script under torch.distributed.run (2 ranks, gloo here); the ranks shard the
64-window S batch, reduce the packed sums with the double-buffered overlapped
all-reduce (paper_2412_06359_b200/dist.py OverlappedAllReduce), time with a
max over ranks, and rank 0 alone prints one JSON line. A stub step stands in
for the chain (no GPU here)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    return lines


def test_gpus2_spawns_two_ranks_and_reduces():
    lines = _run("--gpus", "2", "--cpu-harness", "--steps", "3")
    assert len(lines) == 1  # rank 0 only
    d = lines[0]
    assert d["n_gpus"] == 2 and d["windows_per_rank"] == 32
    # sum over the 64 windows of (1, w, w^2) and the last step index times 64 windows
    assert d["reduced"] == [64.0, 2016.0, 85344.0, 128.0]


def test_single_rank_harness():
    d = _run("--cpu-harness", "--steps", "2")[0]
    assert d["n_gpus"] == 1 and d["windows_per_rank"] == 64
    assert d["reduced"] == [64.0, 2016.0, 85344.0, 64.0]


def test_default_workload_is_the_metric_config():
    sys.path.insert(0, ROOT)
    import bench
    wl = bench.WORKLOADS["S"]
    assert (wl["W"], wl["H"], wl["n_events"], wl["batch_total"]) == (640, 480, 1_000_000, 64)
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'ap.add_argument("--workload", default="S"' in src
    # the canonical SURVEY §8(d) byte model: b_px = 1180 B at B = 10, 18 B/event
    tot, _ = bench.algorithmic_bytes(dict(W=1, H=1, B=10, n_events=0), 1)
    assert tot == 1180
    tot, _ = bench.algorithmic_bytes(dict(W=0, H=0, B=10, n_events=1), 1)
    assert tot == 18
