#!/bin/bash
# Build a measurement variant of libcx.so: one source (SRC, default
# forward_tc.cu) recompiled with extra -D flags, linked with the other objects
# of the default build.
#   tools/build_variant.sh NAME -DCX_TC_SMAX=12 ...   -> paper_2011_01383_b200/variants/libcx_NAME.so
# (load it with CX_LIB=paper_2011_01383_b200/variants/libcx_NAME.so)
set -e
name=$1; shift
P=paper_2011_01383_b200
SRC=${SRC:-forward_tc}
mkdir -p $P/variants/$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 177 "$@" \
  -c $P/csrc/$SRC.cu -o $P/variants/$name/$SRC.o
objs=$(ls $P/build/*.o | grep -v "/$SRC.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/variants/libcx_$name.so $objs $P/variants/$name/$SRC.o
echo $P/variants/libcx_$name.so
