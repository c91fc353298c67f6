#!/bin/bash
# default (C3) bench line, the cutoff / large / parity tests, C5 bench line
O=gpurun_out/${1:-s6}; mkdir -p $O
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python -m pytest tests/test_gpu_cut.py tests/test_gpu_large.py tests/test_gpu_parity.py -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-sweep > $O/bench_c5.json 2> $O/bench_c5.err; echo "rc=$?" >> $O/bench_c5.err
