"""Small, profiler-friendly run of the Step-1 kernels (one seed + one walk launch).

    python tools/profile_walk.py [L] [walkers] [restarts] [count_visited]
Used under `ncu` (see profiles/README.md); prints device ms of the walk kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_07222_b200 as labs  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 451
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
R = int(sys.argv[3]) if len(sys.argv) > 3 else 4
CV = bool(int(sys.argv[4])) if len(sys.argv) > 4 else False
F = {101: 5.0, 201: 5.0, 301: 5.2, 451: 5.3, 527: 5.3}.get(L, 5.0)
cfg = labs.SawConfig(length=L, walkers=W, prefix_len=8, target_merit=F, max_restarts=R, seed=1,
                     count_visited=CV)
with labs.bench_plan(cfg) as plan:
    ms, st = plan.run(1)
print(f"L={L} walks={W * R} kernel_ms={st.kernel_ms:.3f} seed_ms={st.seed_ms:.3f} "
      f"iterations={st.iterations} wide={st.wide_iterations}")
