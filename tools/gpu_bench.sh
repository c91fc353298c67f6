#!/bin/bash
# bench (C3 default), its launch list under ncu, and a C5 bench line
O=gpurun_out/${1:-bench}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sweep > $O/plain.json 2> $O/plain.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sweep > $O/ncu.log 2>&1
python tools/launches_summary.py $O/launches.csv > $O/launches.txt 2>&1
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-sweep > $O/bench_c5.json 2> $O/bench_c5.err
