#!/bin/bash
# Builds an experimental variant of libmmi.so: attn.cu recompiled with extra -D flags, linked with
# the regular objects.  usage: build_variant.sh NAME "-DMMI_PROF -DMMI_EMU_MASK=0x11u"
# -> paper_2504_16083_b200/libmmi_NAME.so (load it with MMI_LIB=...)
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
NAME=$1; shift
python -c "import sys; sys.path.insert(0,'$ROOT'); from paper_2504_16083_b200.build import build; build()"
NV=/usr/local/cuda/bin/nvcc
OBJ=$ROOT/build/obj
mkdir -p $ROOT/build/var
$NV -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
  -I$ROOT/include $@ -c $ROOT/paper_2504_16083_b200/csrc/attn.cu -o $ROOT/build/var/attn_$NAME.o
OBJS=$(ls $OBJ/*.o | grep -v '/attn.o$')
$NV -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $OBJS $ROOT/build/var/attn_$NAME.o \
  -o $ROOT/paper_2504_16083_b200/libmmi_$NAME.so
echo built libmmi_$NAME.so
