#!/bin/bash
# A/B of K4 builds at C2 (L=201 p=12 class 0, m=32): gpurun -- bash tools/ab_enum_libs.sh lib_dir...
for lib in paper_2409_07222_b200/_lib "$@"; do
  for rep in 1 2; do
    LABS_B200_LIB=$lib/libpaper_labs.so python tools/profile_enum.py 32 2>&1 | sed "s|^|$lib |"
  done
done
