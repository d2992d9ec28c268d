# same-box A/B/C of library builds: _lib/libevcm_cuda_{old,a}.so and the current one
L=paper_2412_06359_b200/_lib
cp $L/libevcm_cuda.so /tmp/new.so
for round in 1 2; do for v in old a new; do
  case $v in old) cp $L/libevcm_cuda_old.so $L/libevcm_cuda.so;; a) cp $L/libevcm_cuda_a.so $L/libevcm_cuda.so;; new) cp /tmp/new.so $L/libevcm_cuda.so;; esac
  touch $L/libevcm_cuda.so
  bash tools/bench_quick.sh 2>&1 | sed "s/^/$v /"
done; done
cp /tmp/new.so $L/libevcm_cuda.so
