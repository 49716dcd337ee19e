#!/bin/bash
# Build a timing variant of the library: tools/build_variant.sh NAME "-DFLAG ..." [-v]
cd "$(dirname "$0")/.." || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $2 \
  -Xptxas -v -Wno-deprecated-declarations -o paper_2605_26659_b200/libfinom_dbg_$1.so \
  paper_2605_26659_b200/csrc/finom_1d.cu 2>&1 | grep -A2 "6k_stepILi" | grep -E "registers|spill" | head -4
