"""Generates tests/golden/*.json from the REFERENCE library compiled from its own
sources (oracle/_ref/liblabs_ref.so, see oracle/Makefile).  Run in the dev container
(where /root/reference exists):  python tests/golden/make_golden.py
The GPU tests compare the CUDA path against these committed vectors."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference, make_config  # noqa: E402

CASES = [
    # name, SawConfig fields (reference names)
    ("l31_w4_r3_f3", dict(length=31, walkers=4, max_restarts=3, target_merit=3.0, seed=31)),
    ("l51_w2_r4_el350", dict(length=51, walkers=2, max_restarts=4, energy_threshold=350, seed=123)),
    ("l71_w8_p4_r6_f4", dict(length=71, walkers=8, prefix_len=4, max_restarts=6, target_merit=4.0,
                             seed=9100)),
    ("l101_w32_p8_r2_f5", dict(length=101, walkers=32, prefix_len=8, max_restarts=2,
                               target_merit=5.0, seed=1)),
    ("l201_w8_p12_r1_f4_5", dict(length=201, walkers=8, prefix_len=12, max_restarts=1,
                                 target_merit=4.5, seed=1)),
    ("l51_quota5", dict(length=51, walkers=2, max_restarts=0, target_merit=3.0,
                        candidate_quota=5, seed=5)),
    ("l25_ti_mult4_fpr1e-3", dict(length=25, walkers=3, max_restarts=5, target_merit=3.0,
                                  ti_multiplier=4.0, bloom_fpr=1e-3, seed=99)),
]


def main():
    ref = Reference()
    out = []
    for name, kw in CASES:
        run = ref.run_saw_pool(make_config(**kw), threads=1)
        recs = [ref.format_record(c.seq, c.energy) for c in run.candidates]
        stats = {k: run.stats[k] for k in ("walks", "iterations", "emitted", "best_energy")}
        out.append(dict(name=name, config=kw, records=recs, stats=stats))
        print(name, len(recs), stats)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "saw_pool.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
