#!/bin/bash
# K4 A/B: C2-shaped enumeration (L=201, p=12, class 0, 2^34 Gray steps) for the in-tree
# build ("new") and _lib_<name> builds.  VARIANTS="base new" bash tools/ab_enum.sh
for v in ${VARIANTS:-base new base new}; do
  if [ $v = new ]; then unset LABS_B200_LIB; else export LABS_B200_LIB=$PWD/paper_2409_07222_b200/_lib_$v/libpaper_labs.so; fi
  python -c "
import paper_2409_07222_b200 as labs
labs.enumerate_class(201, 12, 0, 24, 4040, collect=False)
h, st = labs.enumerate_class(201, 12, 0, 34, 4040, collect=False)
print('$v', st['configurations'] / (st['kernel_ms'] / 1e3), st['best_energy'], st['emitted'])"
done
