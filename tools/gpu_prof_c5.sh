#!/bin/bash
# C5 (n = 2^20) evidence: the bench line's launch list under ncu, and ncu sections (speed of light, memory, compute, warp states) of the
# build's two heaviest kernels at that size (tools/profile_case.py C5)
O=gpurun_out/${1:-c5prof}; mkdir -p $O
timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-sweep > $O/plain.json 2> $O/plain.err && \
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-sweep > $O/ncu_list.log 2>&1
python tools/launches_summary.py $O/launches.csv > $O/launches.txt 2>&1
timeout 600 python tools/profile_case.py C5 > $O/case.log 2>&1 && \
timeout 800 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis \
  --section WarpStateStats --section Occupancy --section LaunchStats --section SchedulerStats \
  --clock-control none -k "regex:group_zk_kernel|fsai_factor_kernel" -s 2 -c 2 \
  -o $O/c5 python tools/profile_case.py C5 > $O/ncu.log 2>&1
ncu -i $O/c5.ncu-rep --page details --csv > $O/details.csv 2>&1
ncu -i $O/c5.ncu-rep --page raw --csv > $O/raw.csv 2>&1
python tools/ncu_brief.py $O/c5.ncu-rep > $O/brief.txt 2>&1
rm -f $O/c5.ncu-rep.tmp
