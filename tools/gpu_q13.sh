#!/bin/bash
O=gpurun_out/${1:-q13}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
AFN_FSAI_T48=0 timeout 300 python bench.py --no-cpu --no-e2e > $O/bench_old.json 2> $O/bench_old.err
