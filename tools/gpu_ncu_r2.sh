#!/bin/bash
# ncu evidence (C3): full sets of the top kernels, DRAM of the apply kernels, the bench launch list
O=gpurun_out/${1:-ncu}; mkdir -p $O
timeout 600 python tools/profile_case.py C3 > $O/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"group_gemm_dmma|kmv_sym_kernel|fsai_factor" \
  -s 3 -c 3 -o $O/c3_top python tools/profile_case.py C3 > $O/ncu_top.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gemm_dmma_kernel<0>" -s 25 -c 1 \
  -o $O/c3_wgemm python tools/profile_case.py C3 > $O/ncu_w.log 2>&1
timeout 900 ncu --section MemoryWorkloadAnalysis --section SpeedOfLight --clock-control none \
  -k regex:"gemv_n2|gemv_t_partial|gemv_t_reduce|spmv|gemv_n_row" -s 40 -c 12 -o $O/c3_apply python tools/profile_case.py C3 > $O/ncu_apply.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sweep > $O/bench_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sweep > $O/ncu_launch.log 2>&1
python tools/launches_summary.py $O/launches.csv > $O/launches.txt 2>&1
