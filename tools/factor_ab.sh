#!/bin/bash
# A/B of the FSAI factor kernel: current lib vs gpurun_out/alt/libafn_b16.so
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv -k regex:fsai_factor python tools/profile_case.py 1.0 > gpurun_out/fab_a.csv 2>&1
cp paper_2304_05460_b200/libafn.so /tmp/liba.so; cp gpurun_out/alt/libafn_b16.so paper_2304_05460_b200/libafn.so
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv -k regex:fsai_factor python tools/profile_case.py 1.0 > gpurun_out/fab_b.csv 2>&1
cp /tmp/liba.so paper_2304_05460_b200/libafn.so
