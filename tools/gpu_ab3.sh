#!/bin/bash
O=gpurun_out/${1:-ab3}; mkdir -p $O
L="alt_libs/libafn_r1.so alt_libs/libafn_upc0.so alt_libs/libafn_upc16.so alt_libs/libafn_upc64.so"
timeout 600 python tools/kmv_ab.py $L > $O/kmv_ab.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:kmv_sym_kernel --log-file $O/kmv_ncu.csv \
  python tools/kmv_ab.py $L > $O/kmv_ncu.log 2>&1
python tools/kmv_ab_parse.py $O/kmv_ncu.csv $L > $O/kmv_med.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -x -q -k "matvec or kmv or c2_build" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
