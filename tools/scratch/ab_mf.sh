# same-box A/B of library variants in _variants/: ab_libs.sh WORKLOAD lib1 lib2 ...
WL=$1; shift
for round in 1 2; do for v in "$@"; do
  cp _variants/$v paper_2412_06359_b200/_lib/libevcm_cuda.so
  timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['step_roofline']['stage_ms']; print('$v $WL', round(d['ms_per_step'],3), 'mf', s['motion_field'], 'bwd', s['bwd_owner'])"
done; done
