"""Key metrics + stall breakdown of an ncu report (first kernel).
    python tools/ncu_summary.py gpurun_out/walk_TAG.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2]
get = lambda n: v[h.index(n)] if n in h else "n/a"  # noqa: E731
for n in ["gpu__time_duration.sum", "sm__inst_issued.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "smsp__warps_eligible.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]:
    print(f"{n:60s} {get(n)}")
items = [(n, v[i]) for i, n in enumerate(h)
         if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")]
tot = sum(float(x) for _, x in items if x)
print("stalls:", ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {float(x) / tot * 100:.1f}%"
                           for n, x in sorted(items, key=lambda t: -float(t[1] or 0))[:9]))
