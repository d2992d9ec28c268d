# Copy a tools/refresh_r02.sh run from gpurun_out/ into profiles/ (bench lines,
# reference arm, sweep, 2-rank line, launch list, ncu summaries, ceilings and traffic JSON).
set -e
O=gpurun_out; P=profiles
for f in r02_bench_S r02_bench_C r02_bench_B r02_bench_A r02_ref_S r02_mr_gloo_B; do cp $O/$f.json $P/$f.json; done
cp $O/r02_sweep.jsonl $P/
(echo "# ncu --metrics gpu__time_duration.sum --clock-control none, command:"
 echo "# python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e  (default workload S: 64 x 640x480 x 1M events, owner pipeline), final round-2 build"
 echo "# cold-cache serialised launches: compare SHARES, not absolutes; includes the untimed warm-up steps."
 python tools/ncu_launches.py $O/r02_launches_S.csv) > $P/r02_launches_S.txt
for w in C S; do
  (echo "# ncu --set full --clock-control none, one launch each (bench.py --workload $w --steps 1 --warmup 1), final round-2 build"
   echo "# columns: duration, DRAM read+write per launch, IPC, achieved occupancy, warp instructions, top stall reasons"
   python tools/ncu_summary.py $O/r02_full$w.ncu-rep
   echo; echo "# ceilings (% of peak; tools/ncu_ceilings.py)"
   python tools/ncu_ceilings.py $O/r02_full$w.ncu-rep) > $P/r02_ncu_full_${w}_summary.txt
  python tools/ncu_ceilings_json.py $O/r02_full$w.ncu-rep $w > /dev/null
done
python tools/ncu_traffic.py C=$O/r02_fullC.ncu-rep S=$O/r02_fullS.ncu-rep > /dev/null
