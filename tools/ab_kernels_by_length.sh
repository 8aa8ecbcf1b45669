#!/bin/bash
# K1 (dp4a) vs K1t (mma) walk-kernel time per length: gpurun -- bash tools/ab_kernels_by_length.sh L...
for L in "$@"; do
  for K in dp4a mma; do
    LABS_KERNEL=$K python tools/profile_walk.py $L 1024 16 0 2>&1 | sed "s|^|$K |"
  done
done
