#!/bin/bash
# A/B of library variants on the config-5 group solve (interleaved runs).
# usage: tools/gpu_ab_group.sh LIB1 LIB2 ...
for r in 1 2; do
  for L in "$@"; do FINOM_LIB=$L timeout 300 python tools/prof_group.py 8192 200 3 2>&1 | tail -1; done
done
