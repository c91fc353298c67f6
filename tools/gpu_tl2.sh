#!/bin/bash
O=gpurun_out/${1:-tl2}; mkdir -p $O
timeout 600 python tools/solve_timeline.py C3 16 > $O/tl.txt 2>&1
timeout 600 python tools/solve_timeline_lib.py alt_libs/libafn_noopp.so C3 16 > $O/tl_noopp.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-sweep > $O/bench.json 2> $O/bench.err
