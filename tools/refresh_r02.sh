# Round-2 measurement refresh on one GPU (bash tools/refresh_r02.sh [part]):
#   bench lines (S default, C, B, A), the reference arm, the sweep, the 2-rank path
#   (gloo device sharing), the launch list of the default command, ncu --set full at C and S.
set -x
O=gpurun_out
mkdir -p $O
part=${1:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/r02_gpu.txt 2>&1
if [ "$part" = all ] || [ "$part" = bench ]; then
  timeout 900 python bench.py > $O/r02_bench_S.json 2> $O/r02_bench_S.err
  timeout 600 python bench.py --workload C > $O/r02_bench_C.json 2> $O/r02_bench_C.err
  timeout 600 python bench.py --workload B > $O/r02_bench_B.json 2> $O/r02_bench_B.err
  timeout 600 python bench.py --workload A > $O/r02_bench_A.json 2> $O/r02_bench_A.err
  timeout 900 python bench.py --impl reference > $O/r02_ref_S.json 2> $O/r02_ref_S.err
  timeout 600 python bench.py --sweep --steps 5 > $O/r02_sweep.jsonl 2> $O/r02_sweep.err
  timeout 900 python bench.py --gpus 2 --dist-backend gloo --workload B --no-cpu-baseline \
      > $O/r02_mr_gloo_B.json 2> $O/r02_mr_gloo_B.err
fi
if [ "$part" = all ] || [ "$part" = ncu ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_S.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/r02_launches_S.log 2>&1
  K='regex:k_(motion_field|traj_records|fwd_cells|bwd_event|bwd_cells)'
  timeout 1200 ncu --set full --clock-control none --import-source on -k "$K" -c 5 -f -o $O/r02_fullC \
      python bench.py --workload C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/r02_fullC.log 2>&1
  timeout 1800 ncu --set full --clock-control none --import-source on -k "$K" -c 5 -f -o $O/r02_fullS \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/r02_fullS.log 2>&1
fi
ls -la $O
