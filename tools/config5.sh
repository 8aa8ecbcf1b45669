#!/bin/bash
# Config 5 (BASELINE.json configs[4]): full dual step at L=527 through the reference
# pipeline: GPU Step 1 + K5-scored Step 2 (labs_solve), GPU Step 1 + reference Step 2
# (labs_solve_s1), and the unmodified reference (labs_solve_ref) on a bounded sample.
mkdir -p gpurun_out
ARGS="-L 527 --rounds 1 --p 8 --walkers 1024 --restarts 8 --target-f 5.3 --refine-top 6 --tu 1054 --tr 5 --seed 1 --no-construct"
T=$(nproc)
echo "host threads: $T ($(lscpu | grep 'Model name' | sed 's/ *Model name: *//'))"
run() {  # label, command...
  local t0=$(date +%s.%N)
  "${@:2}" > gpurun_out/c5_out.txt 2> gpurun_out/c5_err.txt
  local rc=$?
  local t1=$(date +%s.%N)
  echo "$1 rc=$rc wall=$(python3 -c "print(round($t1-$t0,2))")s"
  cat gpurun_out/c5_out.txt; tail -n 1 gpurun_out/c5_err.txt
}
for exe in integration/_build/labs_solve integration/_build/labs_solve_s1; do
  run "$exe (1024x8 walks)" $exe solve $ARGS --threads $T
done
SMALL="-L 527 --rounds 1 --p 8 --walkers 256 --restarts 1 --target-f 5.3 --refine-top 6 --tu 1054 --tr 5 --seed 1 --no-construct --threads $T"
for exe in integration/_build/labs_solve integration/_build/labs_solve_s1 oracle/_ref/labs_solve_ref; do
  run "$exe (256 walks)" $exe solve $SMALL
done
