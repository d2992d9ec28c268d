# round-end measurement refresh (one GPU): bench lines, reference arm, launch list, ncu full captures
set -x
O=gpurun_out
python bench.py > $O/fB.json 2> $O/fB.err
python bench.py --workload C > $O/fC.json 2> $O/fC.err
python bench.py --workload S > $O/fS.json 2> $O/fS.err
python bench.py --workload A > $O/fA.json 2> $O/fA.err
python bench.py --impl reference > $O/fRef.json 2> $O/fRef.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fl.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/fl.log 2>&1
K='regex:k_(motion_field|traj_records|fwd_cells|bwd_event|bwd_cells)'
ncu --set full --clock-control none --import-source on -k "$K" -c 5 -f -o $O/fullB \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/fullB.log 2>&1
ncu --set full --clock-control none --import-source on -k "$K" -c 5 -f -o $O/fullC \
    python bench.py --workload C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/fullC.log 2>&1
