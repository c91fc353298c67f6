#!/bin/bash
# Round-end evidence: GPU suite, smoke, bench (C3 + C2 sweep + e2e + CPU oracle), launch list, C5 line
O=gpurun_out/${1:-round}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tools/gpu_bench.sh $1
