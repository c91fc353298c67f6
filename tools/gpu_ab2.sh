#!/bin/bash
O=gpurun_out/${1:-ab2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c2_build or pcg_parity or c2_sweep" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/kmv_ab.py alt_libs/libafn_r1.so alt_libs/libafn_stagemask.so > $O/kmv_ab.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:kmv_sym_kernel --log-file $O/kmv_ncu.csv \
  python tools/kmv_ab.py alt_libs/libafn_r1.so alt_libs/libafn_stagemask.so > $O/kmv_ncu.log 2>&1
timeout 600 python tools/fsai_ab.py C2 current alt_libs/libafn_nobulk.so > $O/fsai_c2.txt 2>&1
timeout 900 python tools/fsai_ab.py C3 current alt_libs/libafn_nobulk.so > $O/fsai_c3.txt 2>&1
timeout 1200 python tools/fsai_ab.py C5 current alt_libs/libafn_nobulk.so > $O/fsai_c5.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_large.py -x -q -k "C3" > $O/pytest_c3.log 2>&1; echo "rc=$?" >> $O/pytest_c3.log
