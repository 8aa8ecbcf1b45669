#!/bin/bash
# A/B of lanes-per-walk on the bench-shaped workloads (65,536 walks): L = 451, 101, 527, 201.
mkdir -p gpurun_out
for lpw in ${LPWS:-32 16 8}; do
  for L in 451 101 527 201; do
    LABS_LPW=$lpw python tools/profile_walk.py $L 1024 64 0 2>&1 | sed "s|^|LPW=$lpw |"
  done
done
