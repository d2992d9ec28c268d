# compute-sanitizer on the final build (one GPU): the smoke set (owner + atomic
# chains, products, L_geo, ingestion, predictor) under memcheck / synccheck /
# initcheck, and memcheck on a multi-round owner window (346x260, 100k events).
O=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  timeout 900 $CS --tool $tool python tools/sanitize_smoke.py > $O/r02_san_$tool.txt 2>&1
  echo "$tool rc=$?: $(grep -h 'ERROR SUMMARY' $O/r02_san_$tool.txt | tail -1)"
done
timeout 1200 $CS --tool memcheck python tools/scratch/hang_probe.py 346 260 100000 1 1 > $O/r02_san_memcheck_100k.txt 2>&1
echo "memcheck 100k rc=$?: $(grep -h 'ERROR SUMMARY' $O/r02_san_memcheck_100k.txt | tail -1)"
