set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_mb.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_mb.log
for v in new old new old; do
  if [ $v = old ]; then export LABS_B200_LIB=$PWD/paper_2409_07222_b200/_lib_old/libpaper_labs.so; else unset LABS_B200_LIB; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mb_$v.log 2>&1
  echo -n "$v: "; grep '^{' gpurun_out/bench_mb_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g  ms/step %.1f  frac %.3f  e2e %.4g launches %s' % (d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d.get('gpu_launches')))"
done
