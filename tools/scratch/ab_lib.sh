# same-box A/B: the current libevcm_cuda.so vs _lib/libevcm_cuda_old.so, alternating
L=paper_2412_06359_b200/_lib
cp $L/libevcm_cuda.so /tmp/new.so
for round in 1 2; do for v in old new; do
  if [ $v = old ]; then cp $L/libevcm_cuda_old.so $L/libevcm_cuda.so; else cp /tmp/new.so $L/libevcm_cuda.so; fi
  touch $L/libevcm_cuda.so
  bash tools/bench_quick.sh 2>&1 | sed "s/^/$v /"
done; done
cp /tmp/new.so $L/libevcm_cuda.so
