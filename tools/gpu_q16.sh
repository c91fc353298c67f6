#!/bin/bash
O=gpurun_out/${1:-q16}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
AFN_FSAI_GA=32 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fsai or build or pcg" > $O/pytest32.log 2>&1; echo "rc=$?" >> $O/pytest32.log
timeout 300 python bench.py --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
AFN_FSAI_GA=32 timeout 300 python bench.py --no-cpu --no-e2e > $O/bench32.json 2> $O/bench32.err
