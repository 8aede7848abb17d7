#!/bin/bash
# K1 variant library: the scan instantiation units recompiled with extra flags, linked with
# the in-tree objects of everything else.   tools/variant_k1.sh <name> [-DFOO=1 ...] -> .ab_libs/<name>.so
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
P=$R/paper_2110_11866_b200
mkdir -p $R/.ab_libs/obj_$name
for f in $P/csrc/scan_inst_*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I $R/include -I $P/csrc "$@" \
    -c $f -o $R/.ab_libs/obj_$name/$(basename $f).o &
done
wait
objs=$(ls $P/build/*.o | grep -v '/scan_inst_')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $R/.ab_libs/$name.so $objs $R/.ab_libs/obj_$name/*.o
echo $R/.ab_libs/$name.so
