"""Throughput of the five BASELINE.json configs on one B200 (device time, CUDA events).

    python tools/bench_configs.py [--out profiles/rNN/configs.json]

C1-C4: the Step-1 pool (seed + walk kernels) as bench.py runs C4, reference-equivalent
flip-delta evals counted exactly on the same walks.  C2: K4 class enumeration (Gray
steps / s).  C5 is timed end to end by tools/config5.sh (reference pipeline)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_07222_b200 as labs  # noqa: E402

POOLS = [  # name, L, p, F, walkers, restarts
    ("C1", 101, 8, 5.0, 1024, 64),
    ("C3", 301, 8, 5.2, 1024, 16),
    ("C4", 451, 8, 5.3, 1024, 64),
    ("C5-step1", 527, 8, 5.3, 1024, 8),
]


def pool(name, L, p, F, walkers, restarts):
    base = dict(length=L, walkers=walkers, prefix_len=p, target_merit=F, max_restarts=restarts,
                seed=1)
    with labs.bench_plan(labs.SawConfig(count_visited=True, **base)) as cp:
        _, cst = cp.run(1)
    with labs.bench_plan(labs.SawConfig(**base)) as plan:
        plan.run(2)
        ms, st = plan.run(3)
    return {"config": name, "L": L, "p": p, "F": F, "walks": walkers * restarts,
            "ms_per_pool": ms, "delta_evals": cst.delta_evals,
            "flip_delta_evals_per_s": cst.delta_evals / (ms / 1e3),
            "iterations_per_s": cst.iterations / (ms / 1e3),
            "candidates": st.emitted, "candidates_per_s": st.emitted / (ms / 1e3),
            "neighbours_per_lane": labs.derive(labs.SawConfig(**base)).get("neighbours_per_lane"),
            "walk_kernel": {0: "K1", 1: "K1t"}.get(labs.derive(labs.SawConfig(**base)).get("kernel"))}


def enum_c2(m=36):
    L, p, cls = 201, 12, 0
    labs.enumerate_class(L, p, cls, 20, 4040, collect=False)  # warm-up
    t0 = time.perf_counter()
    hits, st = labs.enumerate_class(L, p, cls, m, 4040, collect=False)
    wall = time.perf_counter() - t0
    n = st["configurations"]
    return {"config": "C2", "L": L, "p": p, "class": cls, "free_bits_enumerated": m,
            "configurations": n, "kernel_ms": st["kernel_ms"],
            "gray_steps_per_s": n / (st["kernel_ms"] / 1e3), "wall_s": wall,
            "lag_updates_per_s": n * (L - 1) // 2 / (st["kernel_ms"] / 1e3),
            "best_energy": st["best_energy"], "emitted": st["emitted"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--m", type=int, default=36)
    ap.add_argument("--pools-only", action="store_true", help="skip C2 (kernel-variant A/B)")
    a = ap.parse_args()
    res = [pool(*c) for c in POOLS]
    for c in POOLS:  # the other walk kernel on the same pools (policy A/B)
        d = labs.derive(labs.SawConfig(length=c[1], walkers=c[4], prefix_len=c[2],
                                       target_merit=c[3], max_restarts=c[5]))
        os.environ["LABS_KERNEL"] = "dp4a" if d["kernel"] == 1 else "mma"
        r = pool(c[0] + "-alt", *c[1:])
        r["walk_kernel"] = os.environ["LABS_KERNEL"]
        del os.environ["LABS_KERNEL"]
        res.append(r)
    if not a.pools_only:
        res.insert(1, enum_c2(a.m))
    for r in res:
        print(json.dumps(r), flush=True)
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
