#!/bin/bash
# A/B timing of walk-kernel builds on the bench workload (L=451, 1024 walkers x 64
# restarts): default _lib vs the variant lib directories given as arguments.
mkdir -p gpurun_out
for lib in paper_2409_07222_b200/_lib "$@"; do
  for rep in 1 2; do
    LABS_B200_LIB=$lib/libpaper_labs.so python tools/profile_walk.py 451 1024 64 0 2>&1 | sed "s|^|$lib |"
  done
done
