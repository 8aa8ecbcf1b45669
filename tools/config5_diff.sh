#!/bin/bash
# One-off full-size config-5 diff: the unmodified reference `solve`
# (oracle/_ref/labs_solve_ref, CPU Step 1 + reference Step 2) vs the reference pipeline
# with the B200 Step 1 and K5 Step-2 scoring (integration/_build/labs_solve), both at
# L=527, 1024 walkers x 8 restarts, refine_top 6, T_u 1054, T_r 5, every host thread.
# With threads > 1 the reference's emission order is timing-dependent, so the candidate
# files are compared as sets (sorted); the refine agenda is the 6 lowest energies, the
# results file and the Step-1 statistics are compared exactly.
mkdir -p gpurun_out
T=$(nproc)
ARGS="-L 527 --rounds 1 --p 8 --walkers 1024 --restarts 8 --target-f 5.3 --refine-top 6 --tu 1054 --tr 5 --seed 1 --no-construct --deterministic --threads $T"
echo "host: $T threads ($(grep -m1 'model name' /proc/cpuinfo | cut -d: -f2 | xargs))"
for tag in b200 ref; do
  exe=integration/_build/labs_solve; [ $tag = ref ] && exe=oracle/_ref/labs_solve_ref
  t0=$(date +%s.%N)
  $exe solve $ARGS --out gpurun_out/c5_$tag.tsv --candidates gpurun_out/c5_${tag}_cands.tsv \
      > gpurun_out/c5_${tag}_stdout.txt 2> gpurun_out/c5_${tag}_stderr.txt
  rc=$?
  t1=$(date +%s.%N)
  echo "$tag: $exe rc=$rc wall=$(python3 -c "print(round($t1-$t0, 2))") s"
  cat gpurun_out/c5_${tag}_stdout.txt; cat gpurun_out/c5_${tag}_stderr.txt
done
python3 - <<'PY'
import hashlib
def rd(p): return open(p).read()
c = {t: sorted(rd(f"gpurun_out/c5_{t}_cands.tsv").splitlines()) for t in ("b200", "ref")}
r = {t: rd(f"gpurun_out/c5_{t}.tsv") for t in ("b200", "ref")}
o = {t: rd(f"gpurun_out/c5_{t}_stdout.txt") for t in ("b200", "ref")}
s = {t: rd(f"gpurun_out/c5_{t}_stderr.txt").split(" wall=")[0] for t in ("b200", "ref")}
h = lambda x: hashlib.sha256("\n".join(x).encode()).hexdigest()[:16]
print(f"candidates: b200 {len(c['b200'])}, ref {len(c['ref'])}; sorted sha256 {h(c['b200'])} vs {h(c['ref'])}; identical set: {c['b200'] == c['ref']}")
print(f"results file identical: {r['b200'] == r['ref']}")
print(f"best records (stdout) identical: {o['b200'] == o['ref']}")
print(f"Step-1 stats identical: {s['b200'] == s['ref']}  ({s['b200']})")
PY
