#!/bin/bash
# Build a K4 variant library: sft_tc.cu recompiled with extra flags, linked with the
# in-tree objects of everything else.   tools/variant.sh <name> [-DFOO=1 ...]  -> .ab_libs/<name>.so
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
P=$R/paper_2110_11866_b200
mkdir -p $R/.ab_libs/obj_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I $R/include -I $P/csrc "$@" \
  -c $P/csrc/sft_tc.cu -o $R/.ab_libs/obj_$name/sft_tc.cu.o
objs=$(ls $P/build/*.o | grep -v '/sft_tc.cu.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $R/.ab_libs/$name.so $objs $R/.ab_libs/obj_$name/sft_tc.cu.o
echo $R/.ab_libs/$name.so
