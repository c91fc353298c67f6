#!/bin/bash
O=gpurun_out/ga32; mkdir -p $O
AFN_FSAI_GA=32 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv -k regex:"group_gemm|fsai_factor|group_union" python tools/profile_case.py 1.0 > $O/n32.csv 2>&1
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv -k regex:"group_gemm|fsai_factor|group_union" python tools/profile_case.py 1.0 > $O/n16.csv 2>&1
AFN_FSAI_GA=32 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fsai or build or pcg" > $O/pt32.log 2>&1; echo rc=$? >> $O/pt32.log
AFN_FSAI_GA=32 timeout 300 python bench.py --no-cpu --no-e2e > $O/b32.json 2>/dev/null
