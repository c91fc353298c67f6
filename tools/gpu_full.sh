#!/bin/bash
# One GPU session: tests, smoke, bench, launch list, ncu full of the top kernel.
# usage: tools/gpu_full.sh TAG [KERNEL_REGEX]
TAG=${1:-run}; KRE=${2:-kmv_partial}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1300 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1
python tools/launches_summary.py $O/launches.csv > $O/launches.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 2 -c 1 -o $O/full \
  python tools/profile_case.py 1.0 > $O/ncu_full.log 2>&1
ncu -i $O/full.ncu-rep --page details --csv > $O/full_details.csv 2>/dev/null
echo done
