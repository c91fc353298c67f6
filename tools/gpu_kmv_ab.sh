#!/bin/bash
# matvec A/B of alt_libs/*.so: kernel_matvec timing (C2, C3) and the PCG matvec timer of whole solves
O=gpurun_out/${1:-kab}; mkdir -p $O
timeout 300 python tools/kmv_ab.py alt_libs/*.so > $O/kmv_ab.txt 2>&1
timeout 300 python tools/fsai_ab.py C3 current alt_libs/*.so > $O/ab_C3.txt 2>&1
