"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
    python tools/launch_summary.py gpurun_out/launches_TAG.csv TAG > profiles/rNN/launches_TAG.md"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
iK, iV, iU, iM = (h.index(n) for n in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[iM] != "gpu__time_duration.sum":
        continue
    v = float(r[iV].replace(",", "")) * scale[r[iU]]
    n, t = agg.get(r[iK], (0, 0.0))
    agg[r[iK]] = (n + 1, t + v)
tot = sum(t for _, t in agg.values())
tag = sys.argv[2] if len(sys.argv) > 2 else ""
print(f"# {tag} launch list: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400`\n")
print("Command: `python bench.py --steps 2 --warmup 1 --restarts 8 --no-cpu-baseline --no-c2` (L=451, 8192 walks per")
print("launch; the `k_*` launches are the in-run INT32/IDP4A/IMMA peak microbenchmarks).  Cold-cache")
print("serialised times: compare shares, not absolutes.\n")
print("| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k.split('(')[0]} | {n} | {t:.3f} | {100 * t / tot:.1f}% |")
def counting(k):  # the COUNT template argument (second of K1t's, last of K1's) is set
    args = [a.strip() for a in k.split("<", 1)[1].split(">", 1)[0].split(",")]
    return (args[1] if "mma" in k else args[-1]) in ("1", "true")


walk = sum(t for k, (n, t) in agg.items() if "saw_walk" in k and not counting(k))
seed = sum(t for k, (n, t) in agg.items() if "seed" in k)
print(f"\nPer timed step the walk kernel is {100 * walk / (walk + seed):.2f}% of the device time "
      "(seed kernel the rest; the `<..., 1>` launch is the untimed delta-counting pass).")
