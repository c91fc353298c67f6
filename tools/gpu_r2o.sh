#!/bin/bash
O=gpurun_out/${1:-r2o}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_r2.py tests/test_gpu_large.py -q -x -k "repetition or nccl_path or C3 or matvec or cg_parity" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/apply_case.py C3 4 > $O/apply_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"gemv_n2|gemv_t_partial|spmv|gemv_n_row" -s 4 -c 6 \
  -o $O/c3_apply python tools/apply_case.py C3 4 > $O/ncu_apply.log 2>&1
timeout 600 python tools/profile_case.py C3 > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"group_gemm_dmma|fsai_factor|gemm_dmma_kernel<0>" -s 6 -c 3 -o $O/c3_build python tools/profile_case.py C3 > $O/ncu_build.log 2>&1
