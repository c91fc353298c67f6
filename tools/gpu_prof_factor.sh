#!/bin/bash
# ncu --set full of fsai_factor_kernel on a C2 build (second build of tools/profile_case.py),
# with the per-source-line stall page
O=gpurun_out/${1:-pf}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:fsai_factor_kernel" -s 1 -c 1 \
  -o $O/factor python tools/profile_case.py C2 > $O/ncu.log 2>&1
ncu -i $O/factor.ncu-rep --page details --csv > $O/details.csv 2>&1
ncu -i $O/factor.ncu-rep --page raw --csv > $O/raw.csv 2>&1
ncu -i $O/factor.ncu-rep --page source --csv --print-source cuda > $O/source_cuda.csv 2>&1
ncu -i $O/factor.ncu-rep --page source --csv --print-source sass > $O/source_sass.csv 2>&1
