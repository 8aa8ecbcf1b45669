"""Bloom probe rounds per walk iteration in lazy mode (how often the argmin winner is
already visited).  python tools/probe_stats.py [L] [walks]"""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2409_07222_b200 as labs  # noqa: E402
L = int(sys.argv[1]) if len(sys.argv) > 1 else 451
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
p = 8
rng = np.random.default_rng(5)
h = rng.choice(np.array([-1, 1], np.int8), size=(n, (L + 1) // 2))
pre = labs.rank_prefixes(p)
h[:, :p] = pre[rng.integers(0, len(pre), size=n)]
res, _ = labs.saw_walks(L, p, 4 * (L + 1), int(L * L / 10.6), h)
it = sum(r.iterations for r in res)
pr = sum(r.probe_rounds for r in res)
print(f"L={L} walks={n} iterations={it} probe_rounds={pr} per_iteration={pr / it:.3f}")
