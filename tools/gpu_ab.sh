#!/bin/bash
# A/B runs: kmv (kernel durations under ncu) and whole C3 builds for alt_libs
O=gpurun_out/${1:-ab}; mkdir -p $O
timeout 600 python tools/kmv_ab.py alt_libs/libafn_r1.so alt_libs/libafn_repl.so > $O/kmv_ab.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:kmv_sym --log-file $O/kmv_ncu.csv \
  python tools/kmv_ab.py alt_libs/libafn_r1.so alt_libs/libafn_repl.so > $O/kmv_ncu.log 2>&1
timeout 900 python tools/fsai_ab.py C3 current alt_libs/libafn_ga32.so > $O/fsai_c3.txt 2>&1
timeout 900 python tools/fsai_ab.py C2 current alt_libs/libafn_ga32.so > $O/fsai_c2.txt 2>&1
timeout 1200 python tools/fsai_ab.py C5 current alt_libs/libafn_ga32.so > $O/fsai_c5.txt 2>&1
