#!/bin/bash
# GPU check: the whole -m gpu suite (or the given pytest -k expression) + a short bench
O=gpurun_out/${1:-check}; mkdir -p $O
K=${2:-}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
else
  timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
fi
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > $O/bench.json 2> $O/bench.err
timeout 600 python tools/large_times.py C3 C5 > $O/large.txt 2>&1
