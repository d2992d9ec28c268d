# bench queue depth A/B: ab_depth.sh WORKLOAD d1 d2 ...
WL=$1; shift
for round in 1 2 3; do for x in "$@"; do
  EVCM_BENCH_DEPTH=$x timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['step_roofline']['stage_ms']; print('depth=$x $WL', round(d['ms_per_step'],3), 'stages', round(sum(s.values()),3))"
done; done
