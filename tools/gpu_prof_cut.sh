#!/bin/bash
# ncu --set full of the cutoff-path kernels on one C3 build + solve (tools/profile_case.py)
O=gpurun_out/${1:-pz}; mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k "regex:group_zk_kernel|kmv_cut_kernel|wc_gemm_kernel|fsai_factor_kernel|group_union_kernel" -c 6 \
  -o $O/cut python tools/profile_case.py C3 > $O/ncu.log 2>&1
ncu -i $O/cut.ncu-rep --page details --csv > $O/details.csv 2>&1
ncu -i $O/cut.ncu-rep --page raw --csv > $O/raw.csv 2>&1
