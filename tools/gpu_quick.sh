#!/bin/bash
# quick GPU check: parity subset + dist + bench (no ncu)
O=gpurun_out/${1:-quick}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
