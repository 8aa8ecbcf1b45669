#!/bin/bash
# GPU test pass only (optionally a -k filter): gpurun -- bash tools/gpu_tests.sh [pytest args]
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 30 gpurun_out/pytest_gpu.log
