#!/bin/bash
O=gpurun_out/${1:-prof3}; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:group_gemm -c 1 -o $O/g16 python tools/profile_case.py 1.0 > $O/ncu_g16.log 2>&1
AFN_FSAI_GA=32 timeout 600 ncu --set full --clock-control none --import-source on -k regex:group_gemm -c 1 -o $O/g32 python tools/profile_case.py 1.0 > $O/ncu_g32.log 2>&1
