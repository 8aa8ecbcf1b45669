for v in base new base new; do
  if [ $v = base ]; then export LABS_B200_LIB=$PWD/paper_2409_07222_b200/_lib_base/libpaper_labs.so; else unset LABS_B200_LIB; fi
  python -c "
import paper_2409_07222_b200 as labs
labs.enumerate_class(201, 12, 0, 24, 4040, collect=False)
h, st = labs.enumerate_class(201, 12, 0, 34, 4040, collect=False)
print('$v', st['configurations'] / (st['kernel_ms'] / 1e3), st['best_energy'], st['emitted'])"
done
