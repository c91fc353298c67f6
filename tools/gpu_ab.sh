#!/bin/bash
O=gpurun_out/${1:-r3a}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py tests/test_gpu_methods.py -m gpu -x -q > $O/tests.log 2>&1
echo "tests rc $?" >> $O/tests.log
for C in C2 C3; do timeout 300 python tools/fsai_ab.py $C current > $O/ab_$C.txt 2>&1; done
timeout 600 python tools/profile_case.py C3 > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"group_union|pattern_positions|group_gemm|fsai_factor" --log-file $O/launches.csv python tools/profile_case.py C3 > $O/ncu.log 2>&1
python tools/launches_summary.py $O/launches.csv > $O/launches.txt 2>&1
