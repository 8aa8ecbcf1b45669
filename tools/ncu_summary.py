"""Key metrics + stall breakdown of an ncu report (first kernel).
    python tools/ncu_summary.py gpurun_out/walk_TAG.ncu-rep [--json profiles/ncu_summary.json
        --walks N --label TEXT --source TEXT]
--json writes the summary bench.py reads for roofline.traffic (DRAM bytes per walk)."""
import argparse
import csv
import io
import json
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--json", default=None)
ap.add_argument("--walks", type=int, default=0)
ap.add_argument("--label", default="")
ap.add_argument("--source", default="")
ap.add_argument("--round", default="r02")
ap.add_argument("--iterations", type=float, default=0, help="walk iterations in the launch")
a = ap.parse_args()

out = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, v = rows[0], rows[1], rows[2]
get = lambda n: v[h.index(n)] if n in h else "n/a"  # noqa: E731
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def nbytes(n):
    i = h.index(n)
    return float(v[i].replace(",", "")) * SCALE[units[i]]


KEYS = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__warps_eligible.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size"]
for n in KEYS:
    u = units[h.index(n)] if n in h else ""
    print(f"{n:60s} {get(n)} {u}")
items = [(n, v[i]) for i, n in enumerate(h)
         if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")]
tot = sum(float(x) for _, x in items if x)
stalls = {n.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x) / tot * 100
          for n, x in sorted(items, key=lambda t: -float(t[1] or 0))[:9]}
print("stalls:", ", ".join(f"{n} {p:.1f}%" for n, p in stalls.items()))

if a.json:
    dram = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
    f = lambda n: float(get(n))  # noqa: E731
    summary = {
        "round": a.round, "kernel": a.label, "source": a.source,
        "walk_kernel_dram_bytes_per_walk": round(dram / a.walks, 2) if a.walks else None,
        "walk_kernel_dram_bytes_per_launch_profiled": dram,
        "walks_per_launch_profiled": a.walks,
        "duration_ms": f("gpu__time_duration.sum"),
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "pipe_alu_pct": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "pipe_fma_pct": f("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "pipe_fma_cycles_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "pipe_fmaheavy_cycles_pct": f("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "pipe_alu_cycles_pct": f("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "pipe_tensor_imma_cycles_pct": f("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active"),
        "warp_instructions": f("smsp__inst_executed.sum"),
        "warp_instructions_per_walk_iteration":
            round(f("smsp__inst_executed.sum") / a.iterations, 1) if a.iterations else None,
        "pipe_lsu_pct": f("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        "achieved_occupancy_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers_per_thread": f("launch__registers_per_thread"),
        "stall_pct": {n: round(p, 1) for n, p in stalls.items()},
    }
    with open(a.json, "w") as fh:
        json.dump(summary, fh, indent=1)
    print("wrote", a.json)
