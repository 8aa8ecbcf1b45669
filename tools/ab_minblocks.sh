#!/bin/bash
# A/B of the K1 register/occupancy policy: the in-tree build vs _lib_old (built with
# EXTRA=-DLABS_MINB_OLD), over the BASELINE pool configs.  gpurun -- bash tools/ab_minblocks.sh
set -u
mkdir -p gpurun_out
OLD=$PWD/paper_2409_07222_b200/_lib_old/libpaper_labs.so
summ() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('  %-9s %8.2f ms  %.4g evals/s' % (d['config'], d['ms_per_pool'], d['flip_delta_evals_per_s']))"; }
# VARIANTS: new (in-tree), old (_lib_old), lpw16 (in-tree, LABS_LPW=16), or any _lib_<name>
for v in ${VARIANTS:-new old lpw16}; do
  case $v in
    old) export LABS_B200_LIB=$OLD; unset LABS_LPW;;
    lpw16) unset LABS_B200_LIB; export LABS_LPW=16;;
    new) unset LABS_B200_LIB LABS_LPW;;
    *) export LABS_B200_LIB=$PWD/paper_2409_07222_b200/_lib_$v/libpaper_labs.so; unset LABS_LPW;;
  esac
  echo "$v:"; timeout 600 python tools/bench_configs.py --pools-only 2> gpurun_out/ab_$v.err | summ
done
