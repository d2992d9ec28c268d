#!/bin/bash
# GPU test suite only: bash tools/gpu_tests.sh [tag] [pytest args...]
tag=${1:-run}; shift
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 "$@" > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
tail -n 5 gpurun_out/${tag}_pytest.txt
