"""Walk throughput per lane width over a range of lengths (one B200): which LPW the
host policy should pick.  python tools/lpw_sweep.py [L ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r'''
import sys
import paper_2409_07222_b200 as labs
L = int(sys.argv[1])
base = dict(length=L, walkers=1024, prefix_len=8, target_merit=5.0, max_restarts=16, seed=1)
with labs.bench_plan(labs.SawConfig(**base)) as plan:
    plan.run(1)
    ms, st = plan.run(3)
print("%d %s R=%s %.2f ms %.4g deltas/s" % (L, sys.argv[2], labs.derive(labs.SawConfig(**base))["neighbours_per_lane"],
      ms, st.delta_evals_computed / (ms / 1e3)))
'''

for L in [int(a) for a in sys.argv[1:]] or [101, 151, 201, 251, 301, 401, 527, 601]:
    for lpw in ("8", "16", "32"):
        env = dict(os.environ, LABS_LPW=lpw)
        r = subprocess.run([sys.executable, "-c", CHILD, str(L), lpw], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr.strip().splitlines()[-1], flush=True)
