#!/bin/bash
# INT8-slicing W: whole-build A/B against alt_libs and one ncu capture of the GEMM kernel (C3)
O=gpurun_out/${1:-oz}; mkdir -p $O
for C in C3 C2; do timeout 300 python tools/fsai_ab.py $C current alt_libs/*.so > $O/ab_$C.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_r2.py -q -s -k w_product > $O/wp.log 2>&1


