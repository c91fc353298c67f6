#!/bin/bash
O=gpurun_out/${1:-r2q}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -m gpu -x -q -k "fps or repetition" > $O/tests.log 2>&1
echo "tests rc $?" >> $O/tests.log
for C in C3 C2; do
  timeout 900 python tools/fsai_ab.py $C current alt_libs/libafn_wm2.so alt_libs/libafn_dkc16.so alt_libs/libafn_dkc32.so > $O/ab_$C.txt 2>&1
done
