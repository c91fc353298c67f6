#!/bin/bash
O=gpurun_out/${1:-alg1}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "alg1 or c2_sweep or adaptive" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/phases.py C3 > $O/phases_c3.txt 2>&1
timeout 600 python tools/phases.py C3 >> $O/phases_c3.txt 2>&1
