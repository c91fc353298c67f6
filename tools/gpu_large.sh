#!/bin/bash
# Full-size component parity runs (C3, C4, C5), each under its own timeout.
O=gpurun_out/${1:-large}; mkdir -p $O
for c in C3-l1 C4-l1 C4-l3 C5-l1; do
  timeout ${2:-900} python -m pytest tests/test_gpu_large.py -x -q -s -k "$c" > $O/$c.log 2>&1
  echo "$c rc=$?" >> $O/summary.txt
  nvidia-smi --query-gpu=memory.used --format=csv >> $O/summary.txt
done
