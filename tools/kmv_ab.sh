#!/bin/bash
# kmv timing for alternative builds in alt_libs/*.so (git-ignored, shipped by gpurun)
python tools/kmv_time.py > gpurun_out/kmvab.txt 2>&1
cp paper_2304_05460_b200/libafn.so /tmp/liba.so
for f in alt_libs/libafn_u*.so; do
  echo $f >> gpurun_out/kmvab.txt; cp $f paper_2304_05460_b200/libafn.so; python tools/kmv_time.py >> gpurun_out/kmvab.txt 2>&1
done
cp /tmp/liba.so paper_2304_05460_b200/libafn.so
