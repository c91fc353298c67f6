#!/bin/bash
# A/B of whole builds at C3 and C5 against alt_libs/*.so, then the full GPU suite
O=gpurun_out/${1:-ab2}; mkdir -p $O
for C in C3 C5; do timeout 600 python tools/fsai_ab.py $C current alt_libs/*.so > $O/ab_$C.txt 2>&1; done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1
echo "tests rc $?" >> $O/tests.log
