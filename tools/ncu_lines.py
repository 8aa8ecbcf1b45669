"""Per-source-line instruction counts (per walk iteration) from an ncu report.
    python tools/ncu_lines.py gpurun_out/walk_TAG.ncu-rep [iterations] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
it = float(sys.argv[2]) if len(sys.argv) > 2 else 7405568
top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
f, res, tot, tots = "?", [], 0.0, 0.0
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0].isdigit() and len(r) > ie and r[2] == "-":
        try:
            v, s = float(r[ie]), float(r[ss])
        except ValueError:
            continue
        res.append((v, s, f, int(r[0]), r[1].strip()[:80]))
        tot += v
        tots += s
print(f"instructions per iteration: {tot / it:.1f}")
for v, s, f, l, src in sorted(res, reverse=True)[:top]:
    print(f"{f[:16]:16s}:{l:4d} {v / it:7.1f}/it  stall {s / tots * 100:5.1f}%  {src}")
