#!/bin/bash
O=gpurun_out/${1:-ab4}; mkdir -p $O
timeout 900 python tools/fsai_ab.py C3 current alt_libs/libafn_ns3.so alt_libs/libafn_ns4.so > $O/fsai_c3.txt 2>&1
timeout 600 python tools/fsai_ab.py C2 current alt_libs/libafn_ns3.so alt_libs/libafn_ns4.so > $O/fsai_c2.txt 2>&1
