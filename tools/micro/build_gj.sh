#!/bin/bash
# build the k_panel_gj phase profiler: tools/micro/build_gj.sh [extra nvcc flags]
set -e
D=$(cd "$(dirname "$0")" && pwd)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DGJ_PROFILE "$@" -o "$D/panel_gj_prof.bin" \
    "$D/panel_gj_prof.cu" "$D/../../paper_1209_5198_b200/csrc/kernels.cu" 2>&1 | grep -E "error" || true
