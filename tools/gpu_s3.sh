#!/bin/bash
O=gpurun_out/s3; mkdir -p $O
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -k "not C4" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/c4_diag.py > $O/c4.log 2>&1; echo "rc=$?" >> $O/c4.log
timeout 300 python bench.py --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
