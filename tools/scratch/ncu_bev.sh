O=gpurun_out
for x in 0 1; do
EVCM_BWD_REGROUP=$x timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bwd_event -c 1 -f -o $O/bev_rg$x \
    python bench.py --workload C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/bev_rg$x.log 2>&1
done
