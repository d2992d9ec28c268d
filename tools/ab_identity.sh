# bitwise comparison of owner-pipeline outputs: _lib/libevcm_cuda_old.so vs the current build
L=paper_2412_06359_b200/_lib
cp $L/libevcm_cuda.so /tmp/new.so
cp $L/libevcm_cuda_old.so $L/libevcm_cuda.so; touch $L/libevcm_cuda.so
python tools/dump_outputs.py /tmp/old.npz
cp /tmp/new.so $L/libevcm_cuda.so; touch $L/libevcm_cuda.so
python tools/dump_outputs.py /tmp/new.npz
python -c "
import numpy as np
a, b = np.load('/tmp/old.npz'), np.load('/tmp/new.npz')
for k in a: print(k, 'identical' if np.array_equal(a[k], b[k]) else 'DIFFERENT max %g' % np.max(np.abs(a[k] - b[k])))"
