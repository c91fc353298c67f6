#!/bin/bash
O=gpurun_out/${1:-q15}; mkdir -p $O
AFN_FSAI_MB=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fsai or build" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
AFN_FSAI_MB=1 timeout 300 python bench.py --no-cpu --no-e2e > $O/bench16.json 2> $O/bench16.err
AFN_FSAI_MB=1 AFN_FSAI_GA=32 timeout 300 python bench.py --no-cpu --no-e2e > $O/bench32.json 2> $O/bench32.err
