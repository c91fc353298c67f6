#!/bin/bash
# ncu full captures (C3) of the FSAI group product and factor; kmv A/B of alt_libs
O=gpurun_out/${1:-prof}; mkdir -p $O
timeout 600 python tools/kmv_ab.py alt_libs/*.so > $O/kmv_ab.txt 2>&1
timeout 600 python tools/profile_case.py C3 > $O/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"group_gemm|fsai_factor" -s 2 -c 2 \
  -o $O/c3_fsai python tools/profile_case.py C3 > $O/ncu.log 2>&1
