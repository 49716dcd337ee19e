#!/bin/bash
# Build the CUDA library + oracle from the repo root (prints ptxas usage of the tile kernels).
cd "$(dirname "$0")/.." || exit 1
python -c "import __graft_entry__ as g; g.build(force=True)" || exit 1
if [ "$1" = "-v" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -Xptxas -v \
    -Wno-deprecated-declarations -o /tmp/finom_v.so paper_2605_26659_b200/csrc/finom_1d.cu 2>&1 |
    grep -E "k_step|k_half|k_apply|k_pre|k_absorb" -A2 | grep -E "entry|registers|spill"
fi
