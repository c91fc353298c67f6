#!/bin/bash
for t in 1024 512; do
  AFN_TRIDIAG_T=$t ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv -k regex:tridiag python tools/profile_case.py 1.0 > gpurun_out/tri_$t.csv 2>&1
done
