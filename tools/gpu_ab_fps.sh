#!/bin/bash
# FPS A/B at C3 (whole builds) and the FPS parity tests
O=gpurun_out/${1:-abfps}; mkdir -p $O
timeout 300 python tools/fsai_ab.py C3 current alt_libs/*.so > $O/ab_C3.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -m gpu -x -q -k "fps or repetition or knn or permutation" > $O/tests_fps.log 2>&1; echo "rc $?" >> $O/tests_fps.log
timeout 1200 python -m pytest tests/test_gpu_large.py -m gpu -x -q -k C3 > $O/tests_large.log 2>&1; echo "rc $?" >> $O/tests_large.log
