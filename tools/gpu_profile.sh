#!/bin/bash
# ncu evidence for the walk kernel (one GPU): launch list of a short bench run and a
# --set full capture of the walk kernel at L=451 at full residency.
# Usage: gpurun --timeout 1800 -- bash tools/gpu_profile.sh [tag]
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
CMD="python tools/profile_walk.py 451 1024 ${RESTARTS:-16} 0"  # 16,384 walks: every SM at full residency
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:saw_walk -c 1 \
    -o gpurun_out/walk_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
BCMD="python bench.py --steps 2 --warmup 1 --restarts 8 --no-cpu-baseline --no-c2"
$BCMD > gpurun_out/bench_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv $BCMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?"
