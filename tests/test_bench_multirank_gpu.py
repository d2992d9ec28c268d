"""GPU: bench.py's multi-rank path on one B200 -- `--gpus 2` re-launches itself
under torch.distributed.run, the two ranks (sharing the GPU; gloo, because NCCL
needs one GPU per rank) each run the chain on their half of the batch, the
overlapped all-reduce sums the packed [loss, d_depth, d_poses] over ranks, the
time is the max over ranks, and rank 0 alone prints the line. The reduced loss
must equal the sum of the per-window losses of the two ranks' shards."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_ranks_on_one_gpu():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--dist-backend", "gloo", "--workload", "B", "--batch", "2",
                        "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["windows_per_gpu_per_step"] == 2
    # the all-reduced loss sums both ranks' windows; rank 0's own sum is smaller
    assert d["check"]["reduced_loss"] > d["check"]["sum_loss_last_step"] > 0


def test_bench_line_contract():
    """One rank, small workload: the JSON line carries the contract's keys --
    roofline (bound/achieved/peak/unit/frac/traffic + the ceilings entry),
    cpu_baseline (the reference compiled here, on this box's cores), e2e with the
    copied bytes, gpu_launches, clocks -- and the values are consistent."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "B",
                        "--steps", "3", "--warmup", "3", "--cpu-budget-s", "2"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"] * 10  # the owner chain's kernels, every step
    assert d["value"] > 100 * d["cpu_baseline"]["value"]
