#!/bin/bash
# A/B of walk-kernel builds: gpurun -- bash tools/ab_libs.sh "L [KERNEL]" lib_dir...
#   (default _lib first; LABS_KERNEL from the second word of the first argument)
set -- "$@"
SPEC=$1; shift
L=${SPEC%% *}; K=${SPEC#* }; [ "$K" = "$SPEC" ] && K=""
for lib in paper_2409_07222_b200/_lib "$@"; do
  for rep in 1 2; do
    LABS_KERNEL=$K LABS_B200_LIB=$lib/libpaper_labs.so python tools/profile_walk.py $L 1024 64 0 2>&1 | sed "s|^|$lib |"
  done
done
