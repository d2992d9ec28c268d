# same-box A/B of an environment switch on one workload: ab_stage.sh VAR A B [WORKLOAD]
# prints ms/step and the stage split per run (device-resident bench, no e2e / CPU baseline)
V=$1; A=$2; B=$3; WL=${4:-C}
for round in 1 2; do for x in $A $B; do
  env $V=$x python bench.py --workload $WL --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V=$x $WL', round(d['ms_per_step'],3), d['step_roofline']['stage_ms'])"
done; done
