#!/bin/bash
# A/B of the walk kernels (K1 IDP4A vs K1t tensor-core G) on the bench workloads:
#   gpurun -- bash tools/ab_kernel.sh [L ...]
for L in ${@:-451}; do
  for k in dp4a mma; do
    for rep in 1 2; do
      LABS_KERNEL=$k python tools/profile_walk.py $L 1024 64 0 2>&1 | sed "s|^|$k |"
    done
  done
done
