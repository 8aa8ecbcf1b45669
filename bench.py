#!/usr/bin/env python
"""bench.py -- Step-1 throughput on B200 (BASELINE.json metric, config C4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}]

Workload (BASELINE.json configs[3]): L=451, p=8 restriction classes,
F >= 5.3 (E_l = 19188), T_i = 1808, Bloom fpr 1e-4, seed 1, 1024 walkers x 64 restarts per
GPU (65,536 walks per GPU).  Weak scaling: at N GPUs the job is 1024*N walkers sharded by
restriction class (class c = w mod 128 goes to rank c mod N); ranks never communicate on the
data path; rank 0 reduces the device time (max over ranks) and counts with torch.distributed.

One step = the whole pool on every rank: K3 (seed streams -> initial halves) + K1 (walks,
sieve, compaction) over all 65,536 walks, inputs generated and resident in HBM.  `value` is
reference-equivalent flip-delta evaluations per second (the count skew_flip_delta_fast would
be called, saw.cpp:106-115, measured exactly with count_visited=1 on the same walks).
`e2e` is the same metric through the public API run_saw_pool() (host config in, candidates
out through the sink), timed by wall clock per call.
`--impl reference` times the reference library compiled from its own sources
(oracle/_ref, all host cores) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L, P, F, WALKERS_PER_GPU, RESTARTS, SEED = 451, 8, 5.3, 1024, 64, 1
OPS_PER_DELTA = 4 * (L - 1)  # (L-1)/2 lag-terms x 8 INT32 ops


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_bench_{os.getpid()}.csv")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                try:
                    sm.append(float(f[0]))
                    mx = max(mx, float(f[1]))
                except ValueError:
                    continue
                for n, v in zip(names, f[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
        except OSError:
            return None
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def ncu_traffic():
    """Per-launch DRAM bytes of the walk kernel from the committed ncu summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get("walk_kernel_dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def cpu_reference_run(threads, walkers):
    """Reference library (oracle/_ref, compiled from /root/reference sources) on host cores."""
    from oracle.oracle import Reference, Restated, make_config, reference_available
    cfg = make_config(L, walkers=walkers, prefix_len=P, target_merit=F, max_restarts=1, seed=SEED)
    if reference_available():
        lib, kind = Reference(), "reference"
        t0 = time.perf_counter()
        run = lib.run_saw_pool(cfg, threads=threads)
        dt = time.perf_counter() - t0
        return kind, dt, run, lib
    lib, kind = Restated(), "port"
    t0 = time.perf_counter()
    run = lib.run_saw_pool(cfg)
    dt = time.perf_counter() - t0
    return kind, dt, run, lib


_CPU_COUNTS = {}


def cpu_sample_counts(labs, walkers):
    """Reference-equivalent delta evals of the CPU sample (deterministic)."""
    if walkers not in _CPU_COUNTS:
        cfg = labs.SawConfig(length=L, walkers=walkers, prefix_len=P, target_merit=F,
                             max_restarts=1, seed=SEED, count_visited=True)
        st = labs.run_saw_pool(cfg, labs.CollectingSink())
        _CPU_COUNTS[walkers] = st.delta_evals
    return _CPU_COUNTS[walkers]


def cpu_sample_size():
    n = os.cpu_count() or 1
    return n, min(1024, max(16, 4 * n))


def run_reference_arm(args, ws, rank):
    if rank != 0:
        return
    threads, walkers = cpu_sample_size()
    from oracle.oracle import Reference, reference_available
    # count of skew_flip_delta_fast calls in the sample, from the reference's own run_walk
    # driven through its VisitedSet seam (oracle/ref_shim.cpp ref_walk_trace), untimed
    from oracle.oracle import make_config, Restated
    cfgc = make_config(L, walkers=walkers, prefix_len=P, target_merit=F, max_restarts=1, seed=SEED)
    counter = Reference() if reference_available() else None
    if counter is not None:
        evals = counter.walk_trace(cfgc).stats["delta_evals"]
    else:
        evals = Restated().run_saw_pool(cfgc).stats["delta_evals"]
    times = []
    kind, emitted = "reference", 0
    for i in range(args.warmup + args.steps):
        kind, dt, run, _ = cpu_reference_run(threads, walkers)
        emitted = run.stats["emitted"]
        if i >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    v = evals / t
    line = {
        "impl": "reference", "metric": "flip-delta evals/sec (L=451)", "value": v,
        "unit": "flip-deltas/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"C4 sample: L={L} p={P} F>={F} walkers [0,{walkers}) x 1 restart",
                   "threads": threads},
        "candidates_per_s": emitted / t,
        "cpu_baseline": {"value": v, "unit": "flip-deltas/s", "cores": threads, "kind": kind,
                         "sample": f"walkers [0,{walkers}) x 1 restart of C4 ({evals} delta evals)"},
        "e2e": {"value": v, "unit": "flip-deltas/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--walkers-per-gpu", type=int, default=WALKERS_PER_GPU)
    ap.add_argument("--restarts", type=int, default=RESTARTS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    ws, rank, local = dist_env()

    dist = None
    if ws > 1:
        import torch.distributed as dist
        backend = "nccl"
        dist.init_process_group(backend=backend)
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    import torch
    import paper_2409_07222_b200 as labs
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)

    walkers = args.walkers_per_gpu * ws
    base = dict(length=L, walkers=walkers, prefix_len=P, target_merit=F,
                max_restarts=args.restarts, seed=SEED, device=local,
                shard_index=rank, shard_count=ws)

    # ---- reference-equivalent counts for this rank's walks (identical walks, untimed)
    with labs.bench_plan(labs.SawConfig(count_visited=True, **base)) as cp:
        _, cst = cp.run(1)
    deltas_rank = cst.delta_evals
    iters_rank = cst.iterations

    peak = None
    if rank == 0:
        try:
            peak = labs.int32_peak()
        except labs.LabsError:
            peak = None

    plan = labs.bench_plan(labs.SawConfig(**base))
    for _ in range(args.warmup):
        plan.run(1)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local) if rank == 0 else None
    t_wall = time.perf_counter()
    ms_total, st = plan.run(args.steps)  # device time per step (CUDA events on the lib stream)
    ms_total *= args.steps
    wall = time.perf_counter() - t_wall
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    if dist is not None:
        dist.barrier()

    kernel_ms_step = st.kernel_ms  # last step's walk-kernel time
    vals = torch.tensor([ms_total, float(deltas_rank), float(st.emitted), float(iters_rank),
                         kernel_ms_step], dtype=torch.float64, device="cuda")
    if dist is not None:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, deltas_all, emitted_all, iters_all = mx[0].item(), sm[1].item(), sm[2].item(), sm[3].item()
        kms_max = mx[4].item()
    else:
        ms_max, deltas_all, emitted_all, iters_all, kms_max = [v.item() for v in vals]

    # ---- e2e through the public API (host in, candidates out), this rank's shard
    e2e_times, e2e_stats = [], None
    cfg_api = labs.SawConfig(**base)
    for i in range(1 + min(args.steps, 3)):
        sink = labs.CollectingSink()
        t0 = time.perf_counter()
        e2e_stats = labs.run_saw_pool(cfg_api, sink)
        dt = time.perf_counter() - t0
        if i > 0:
            e2e_times.append(dt)
    e2e_t = torch.tensor([statistics.mean(e2e_times)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_s = e2e_t.item()

    if rank == 0:
        step_s = ms_max / 1e3 / args.steps
        value = deltas_all / step_s
        # roofline: dominant kernel = K1 walk kernel; algorithmic INT32 ops per launch
        alg_ops = (deltas_rank + iters_rank) * OPS_PER_DELTA
        achieved = alg_ops / (kernel_ms_step / 1e3) / 1e12
        peak_v = None
        if peak:
            peak_v = max(peak["imad"], peak["ialu"], peak["mixed"]) / 1e12
        roof = {"bound": "int32", "achieved": achieved, "peak": peak_v, "unit": "Tops/s",
                "frac": (achieved / peak_v) if peak_v else None, "traffic": ncu_traffic(),
                "peak_source": "measured in this run by labs_int32_peak (max of IMAD, "
                               "IADD3/LOP3 and 1:1 mix issue rates)",
                "int32_peak_detail": peak,
                "alg_ops_per_launch": alg_ops,
                "note": "algorithmic ops = (reference-equivalent delta evals + applies) x 4(L-1) "
                        "(BASELINE.md §2); the kernel issues far fewer instructions per delta "
                        "(skew pairing, 4 lags per IDP4A), so frac can exceed 1"}
        cpu = None
        if not args.no_cpu_baseline:
            threads, cw = cpu_sample_size()
            try:
                evals = cpu_sample_counts(labs, cw)
                kind, dt, run, _ = cpu_reference_run(threads, cw)
                cpu = {"value": evals / dt, "unit": "flip-deltas/s", "cores": threads,
                       "kind": kind, "sample": f"C4 walkers [0,{cw}) x 1 restart "
                                               f"({evals} delta evals, {dt:.2f} s)"}
            except Exception as e:  # baseline is reported, never fatal
                cpu = {"value": None, "error": str(e)}
        free = (L + 1) // 2 - P
        line = {
            "metric": "flip-delta evals/sec (L=451)",
            "value": value,
            "unit": "flip-deltas/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": f"C4: L={L} p={P} F>={F} (E_l=19188) T_i=1808 fpr=1e-4 seed=1, "
                                   f"{args.walkers_per_gpu} walkers x {args.restarts} restarts "
                                   f"per GPU, class-sharded",
                       "walks_per_gpu": args.walkers_per_gpu * args.restarts,
                       "l2": "per-walk state is on-chip (shared memory); inputs are a 2 MB seed "
                             "table regenerated every step, no L2 flush needed",
                       "parallelism": f"class-shard x{ws}"},
            "candidates_per_s": emitted_all / step_s,
            "candidates_per_step": emitted_all,
            "walk_iterations_per_s": iters_all / step_s,
            "delta_evals_per_step": deltas_all,
            "delta_evals_computed_per_step": (iters_all + ws * args.walkers_per_gpu * args.restarts) * free,
            "kernel_ms_per_step": kms_max,
            "wall_s_timed_region": wall,
            "gpu_launches": 2 * args.steps * ws,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": deltas_all / e2e_s, "unit": "flip-deltas/s",
                    "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                    "s_per_step": e2e_s,
                    "path": "paper_2409_07222_b200.run_saw_pool (C ABI labs_saw_pool_run)"},
            "clocks": clk,
        }
        if e2e_stats is not None:
            line["e2e"]["h2d_bytes_per_step"] = getattr(e2e_stats, "h2d_bytes", None)
            line["e2e"]["d2h_bytes_per_step"] = getattr(e2e_stats, "d2h_bytes", None)
        print(json.dumps(line), flush=True)
    plan.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
