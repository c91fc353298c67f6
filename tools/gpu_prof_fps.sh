#!/bin/bash
# ncu --set full of the C3 FPS (shared-memory cluster path with the spatial cull), second build
O=gpurun_out/${1:-pfps}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:fps_push_kernel" -s 1 -c 1 \
  -o $O/fps python tools/profile_case.py C3 > $O/ncu.log 2>&1
ncu -i $O/fps.ncu-rep --page details --csv > $O/details.csv 2>&1
ncu -i $O/fps.ncu-rep --page source --csv --print-source sass > $O/source_sass.csv 2>&1
