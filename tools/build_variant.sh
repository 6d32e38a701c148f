#!/bin/bash
# Build a measurement variant of libcx.so: forward_tc.cu recompiled with extra
# -D flags, linked with the other objects of the default build.
#   tools/build_variant.sh NAME -DCX_TC_SMAX=12 ...   -> paper_2011_01383_b200/variants/libcx_NAME.so
# (load it with CX_LIB=paper_2011_01383_b200/variants/libcx_NAME.so)
set -e
name=$1; shift
P=paper_2011_01383_b200
mkdir -p $P/variants/$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 177 "$@" \
  -c $P/csrc/forward_tc.cu -o $P/variants/$name/forward_tc.o
objs=$(ls $P/build/*.o | grep -v forward_tc.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/variants/libcx_$name.so $objs $P/variants/$name/forward_tc.o
echo $P/variants/libcx_$name.so
