#!/bin/bash
# A/B of K1 builds over the BASELINE pool configs: the in-tree build ("new") against
# _lib_<name> builds (e.g. `make -C paper_2409_07222_b200/csrc OUT=../_lib_base` from the
# previous commit).  VARIANTS="base new base new" gpurun -- bash tools/ab_minblocks.sh
set -u
mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('  %-9s %8.2f ms  %.4g evals/s' % (d['config'], d['ms_per_pool'], d['flip_delta_evals_per_s']))"; }
# VARIANTS: new (in-tree), lpw8/lpw16/lpw32 (in-tree, LABS_LPW forced), or any _lib_<name>
for v in ${VARIANTS:-base new}; do
  case $v in
    lpw8|lpw16|lpw32) unset LABS_B200_LIB; export LABS_LPW=${v#lpw};;
    new) unset LABS_B200_LIB LABS_LPW;;
    *) export LABS_B200_LIB=$PWD/paper_2409_07222_b200/_lib_$v/libpaper_labs.so; unset LABS_LPW;;
  esac
  echo "$v:"; timeout 600 python tools/bench_configs.py --pools-only 2> gpurun_out/ab_$v.err | summ
done
