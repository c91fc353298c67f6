#!/bin/bash
# A/B of whole builds (kernel timers per class) against alt_libs/*.so, plus the GPU tests
O=gpurun_out/${1:-ab}; mkdir -p $O
for C in C3 C2; do timeout 300 python tools/fsai_ab.py $C current alt_libs/*.so > $O/ab_$C.txt 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py tests/test_gpu_methods.py tests/test_gpu_cut.py -m gpu -x -q > $O/tests.log 2>&1
echo "tests rc $?" >> $O/tests.log
