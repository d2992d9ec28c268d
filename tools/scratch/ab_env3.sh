# same-box A/B of an env switch with the full stage print: ab_env3.sh VAR WORKLOAD v1 v2 ...
V=$1; WL=$2; shift; shift
for round in 1 2; do for x in "$@"; do
  env $V=$x timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['step_roofline']['stage_ms']; print('$V=$x $WL', round(d['ms_per_step'],3), {k: s[k] for k in ('motion_field','traj_records','bwd_event')})"
done; done
