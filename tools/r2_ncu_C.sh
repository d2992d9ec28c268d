# ncu --set full of the five stage kernels at workload C (one launch each) + the
# launch list of the default (S) bench command. Usage: bash tools/r2_ncu_C.sh TAG
tag=${1:-r2}
O=gpurun_out
mkdir -p $O
K='regex:k_(motion_field|traj_records|fwd_cells|bwd_event|bwd_cells)'
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -c 5 -f -o $O/${tag}_fullC \
    python bench.py --workload C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/${tag}_fullC.log 2>&1
echo "fullC rc=$?"
if [ "${2:-}" = "launches" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${tag}_launches_S.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/${tag}_launches_S.log 2>&1
echo "launches rc=$?"
fi
