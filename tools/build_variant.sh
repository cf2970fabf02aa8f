#!/bin/bash
# build an A/B variant of libf2gpu.so with extra nvcc defines:
#   tools/build_variant.sh NAME -DFOO=1 ...  -> paper_1209_5198_b200/ab/NAME.so (select with F2GPU_LIB)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_1209_5198_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -DF2GPU_EXPERIMENTAL=0 -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -diag-suppress 177 "$@" -shared -o ../ab/$name.so kernels.cu tc_leaf.cu tc_pair.cu api.cu -ldl
