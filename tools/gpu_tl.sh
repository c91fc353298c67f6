#!/bin/bash
O=gpurun_out/${1:-tl}; mkdir -p $O
timeout 600 python tools/solve_timeline.py C3 6 > $O/tl.txt 2>&1
timeout 600 python tools/solve_timeline.py C3 4 kt > $O/tl_kt.txt 2>&1
timeout 600 python tools/solve_timeline.py C2 6 > $O/tl_c2.txt 2>&1
