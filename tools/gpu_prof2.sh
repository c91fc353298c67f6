#!/bin/bash
# ncu full captures of the FSAI kernels (C2, l=1)
O=gpurun_out/${1:-prof2}; mkdir -p $O
for K in fsai_factor group_gemm; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o $O/$K \
  python tools/profile_case.py 1.0 > $O/ncu_$K.log 2>&1
ncu -i $O/$K.ncu-rep --page details --csv > $O/${K}_details.csv 2>/dev/null
ncu -i $O/$K.ncu-rep --page source --csv > $O/${K}_source.csv 2>/dev/null
done
