#!/bin/bash
# A/B of lanes-per-walk on the bench workload (L=451, 65,536 walks), plus L=101 and 527.
mkdir -p gpurun_out
for lpw in 32 16; do
  for L in 451 101 527; do
    LABS_LPW=$lpw python tools/profile_walk.py $L 1024 64 0 2>&1 | sed "s|^|LPW=$lpw |"
  done
done
