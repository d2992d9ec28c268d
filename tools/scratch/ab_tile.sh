# A/B of EVCM_BWD_TILE=0/1 on library variants: ab_tile.sh WORKLOAD lib...
WL=$1; shift
for round in 1 2; do for v in "$@"; do for t in 0 1; do
  cp _variants/$v paper_2412_06359_b200/_lib/libevcm_cuda.so
  EVCM_BWD_TILE=$t timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['step_roofline']['stage_ms']; print('$v tile=$t $WL', round(d['ms_per_step'],3), 'bev', s['bwd_event'], 'bwd', s['bwd_owner'])"
done; done; done
