#!/bin/bash
# full GPU suite + one compute-sanitizer tool over tools/sanitize_case.py
O=gpurun_out/${1:-san}; TOOL=${2:-racecheck}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/sanitize_case.py > $O/plain_case.log 2>&1 && \
timeout 2400 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_case.py > $O/sanitizer_$TOOL.log 2>&1
echo "sanitizer rc=$?" >> $O/sanitizer_$TOOL.log
