#!/bin/bash
# Build an alternative libafn.so for an A/B measurement: one source recompiled
# with extra nvcc flags, linked with the other objects of the current build.
#   tools/build_alt.sh NAME SRC.cu "-DFOO=1 ..."   ->  alt_libs/libafn_NAME.so
set -e
NAME=$1; SRC=$2; FLAGS=$3
B=paper_2304_05460_b200/_build
NCCLI=$(python -c "import nvidia.nccl,os;print(os.path.join(nvidia.nccl.__path__[0],'include'))")
mkdir -p alt_libs /tmp/alt_$NAME
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -diag-suppress 177 -I$NCCLI $FLAGS -c paper_2304_05460_b200/csrc/$SRC -o /tmp/alt_$NAME/${SRC%.cu}.o
OBJS=""
for o in $B/*.o; do
  if [ "$(basename $o)" == "${SRC%.cu}.o" ]; then OBJS="$OBJS /tmp/alt_$NAME/${SRC%.cu}.o"; else OBJS="$OBJS $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o alt_libs/libafn_$NAME.so $OBJS -ldl
echo alt_libs/libafn_$NAME.so
