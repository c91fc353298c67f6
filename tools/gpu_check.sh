#!/bin/bash
# full GPU suite + a C3 launch list (ncu, per-kernel durations) under gpurun_out/$1
O=gpurun_out/${1:-check}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-sweep > $O/ncu.log 2>&1
python tools/launches_summary.py $O/launches.csv > $O/launches.txt 2>&1
