#!/bin/bash
O=gpurun_out/${1:-r2p}; mkdir -p $O
timeout 600 python tools/profile_case.py C3 > $O/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"group_gemm_dmma|fsai_factor|gemm_dmma_kernel<\(int\)0>" -s 6 -c 6 -o $O/c3_build python tools/profile_case.py C3 > $O/ncu_build.log 2>&1
python -c "import sys; sys.path.insert(0,'.'); import paper_2304_05460_b200 as a; print('dfma TF', a.probe_dfma(), 'dmma TF', a.probe_dmma())" > $O/probe.txt 2>&1
