#!/bin/bash
# Builds an experimental variant of libmmi.so: every .cu recompiled with extra -D flags.
# usage: build_variant.sh NAME "-DMMI_PROF ..."  -> paper_2504_16083_b200/libmmi_NAME.so (load with MMI_LIB=...)
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
NAME=$1; shift
NV=/usr/local/cuda/bin/nvcc
OUT=$ROOT/build/var/$NAME
mkdir -p $OUT
for f in $ROOT/paper_2504_16083_b200/csrc/*.cu; do
  $NV -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
    -I$ROOT/include $@ -c $f -o $OUT/$(basename $f .cu).o &
done
wait
$NV -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $OUT/*.o -o $ROOT/paper_2504_16083_b200/libmmi_$NAME.so
echo built libmmi_$NAME.so
