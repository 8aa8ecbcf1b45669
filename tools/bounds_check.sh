#!/bin/bash
# The K1t parity tests against the bounds-checked build (saw_walk_mma.cuh LABS_BC):
#   make -C paper_2409_07222_b200/csrc OUT=../_lib_check EXTRA=-DLABS_BOUNDS_CHECK \
#        ../_lib_check/libpaper_labs.so
#   gpurun -- bash tools/bounds_check.sh
mkdir -p gpurun_out
LABS_B200_LIB=$PWD/paper_2409_07222_b200/_lib_check/libpaper_labs.so LABS_KERNEL=mma \
  timeout 1500 python -m pytest tests -m gpu -x -q -k "(deltas or walks or pool or engine) and not budget and not overshoot" \
  > gpurun_out/bounds_check.log 2>&1
echo "bounds-checked K1t parity rc=$?"
tail -n 3 gpurun_out/bounds_check.log
