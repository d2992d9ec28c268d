#!/bin/bash
# One GPU session: smoke, the GPU test suite, the default bench line.
# Usage (from the repo root, via gpurun): bash tools/gpu_check.sh [tag]
tag=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.txt
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
tail -n 3 gpurun_out/${tag}_smoke.txt gpurun_out/${tag}_pytest.txt gpurun_out/${tag}_bench.err
