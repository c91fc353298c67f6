#!/bin/bash
# A/B of kernel times (ncu, warm) between the current build and alt_libs/*.so
# usage: tools/ab_ncu.sh REGEX [L]
RE=$1; L=${2:-1.0}
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv -k regex:$RE python tools/profile_case.py $L > gpurun_out/ab_cur.csv 2>&1
cp paper_2304_05460_b200/libafn.so /tmp/liba.so
for f in alt_libs/*.so; do
  b=$(basename $f .so); cp $f paper_2304_05460_b200/libafn.so
  ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv -k regex:$RE python tools/profile_case.py $L > gpurun_out/ab_$b.csv 2>&1
done
cp /tmp/liba.so paper_2304_05460_b200/libafn.so
