#!/bin/bash
# full GPU suite + quick bench
O=gpurun_out/${1:-t7}; mkdir -p $O
timeout 300 python bench.py --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
timeout 1300 python -m pytest tests -m gpu -q --durations=15 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
