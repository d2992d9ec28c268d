# quick A/B loop: stage split of workloads B and C (device-resident bench, no e2e / CPU baseline)
python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', d['ms_per_step'], d['step_roofline']['stage_ms'])"
python bench.py --workload C --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C', d['ms_per_step'], d['step_roofline']['stage_ms'])"
