#!/bin/bash
# compute-sanitizer passes over small walk / enumeration / scoring launches (one GPU).
#   gpurun -- bash tools/sanitize.sh
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for k in mma dp4a; do
    LABS_KERNEL=$k timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 \
      python tools/profile_walk.py 451 8 1 1 > gpurun_out/sanitize_${tool}_$k.log 2>&1
    echo "$tool $k rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_$k.log | tail -1)"
  done
done
