#!/bin/bash
# Iteration loop on one GPU: parity tests, then a short bench, then (optionally) an ncu
# capture of the walk kernel.  Usage: gpurun -- bash tools/gpu_iter.sh TAG [ncu]
set -u
TAG=${1:-dev}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
grep '^{' gpurun_out/bench_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g  ms/step %.1f  frac %.3f  e2e %.4g' % (d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value']))"
if [ "${2:-}" = "ncu" ]; then
  CMD="python tools/profile_walk.py 451 1024 4 0"
  $CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:saw_walk_kernel -c 1 \
      -o gpurun_out/walk_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu rc=$?"
fi
