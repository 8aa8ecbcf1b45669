#!/usr/bin/env python
"""bench.py -- Step-1 throughput on B200 (BASELINE.json metric, config C4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}]

Workload (BASELINE.json configs[3]): L=451, p=8 restriction classes,
F >= 5.3 (E_l = 19188), T_i = 1808, Bloom fpr 1e-4, seed 1, 1024 walkers x 64 restarts per
GPU (65,536 walks per GPU).  Weak scaling: at N GPUs the job is 1024*N walkers sharded by
restriction class (class c = w mod 128 goes to rank c mod N); ranks never communicate on the
data path; rank 0 reduces the device time (max over ranks) and counts with torch.distributed.

One step = the whole pool on every rank: K3 (seed streams -> initial halves) + K1 (walks,
sieve, compaction) over all 65,536 walks, inputs resident in HBM, L2 flushed before every
step.  `value` is reference-equivalent flip-delta evaluations per second (the number of
skew_flip_delta_fast calls the reference makes, saw.cpp:106-115, counted exactly with
count_visited=1 on the same walks) over the device time (CUDA events, max over ranks).
`e2e` is the same metric through the public API run_saw_pool() (host config in, seed tables
H2D, sieve records + stats D2H, candidates out through the sink), wall clock per call.
`roofline` is the K1 walk kernel's algorithmic int8-MAC rate against the measured IDP4A
peak.  `cpu_baseline` / `--impl reference` time the reference library
compiled from its own sources (oracle/_ref) with all host cores on a bounded sample.
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
# Algorithmic work per delta-equivalent: with the skew pairing a flip delta
# is one inner product G(a) over the parity array, (L+1)/2 int8 MACs = L+1 int ops.
OPS_PER_DELTA = L + 1
# SURVEY.md §8(d)'s count of the reference formulation (4 sign products per lag-term).
REF_OPS_PER_DELTA = 4 * (L - 1)
CPU_WALKS_PER_CORE = 40  # ~10 s of reference work on the box's host cores


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms; summarised over [t0, t1]."""

    FIELDS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_bench_{os.getpid()}.csv")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index),
                 "--query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.5)  # first sample

    def stop(self, t0, t1):
        if self.proc is None:
            return None
        time.sleep(0.2)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        import datetime
        sm, mx, reasons, allsm = [], 0.0, set(), []
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                try:
                    ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    v, m = float(f[1]), float(f[2])
                except ValueError:
                    continue
                allsm.append(v)
                mx = max(mx, m)
                if t0 - 0.15 <= ts <= t1 + 0.15:
                    sm.append(v)
                    for n, r in zip(self.FIELDS, f[4:8]):
                        if r.lower() == "active":
                            reasons.add(n)
        except OSError:
            return None
        if not sm:  # timed region shorter than the sampling period: use all samples
            sm = allsm
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


ISSUE_PEAK_NOTE = ("warp-instructions per unit from the committed ncu capture (profiles/*.json, "
                   "smsp__inst_executed.sum / units) x units/s, over the issue peak: one "
                   "warp-instruction per cycle per SMSP = 4 x SMs x SM clock")


def issue_roofline(units_per_s, profile, key, peak_info):
    """The binding resource of K1t / K4: instruction issue.  Instructions per unit come
    from the committed ncu capture; the peak is 4 SMSPs x SMs x the SM clock."""
    try:
        with open(os.path.join(ROOT, "profiles", profile)) as f:
            per_unit = json.load(f).get(key)
    except (OSError, ValueError):
        per_unit = None
    if not per_unit or not peak_info:
        return None
    peak = 4 * peak_info["sm_count"] * peak_info["clock_khz"] * 1e3
    achieved = units_per_s * per_unit
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "warp-instr/s",
            "frac": achieved / peak, "per_unit": per_unit, "source": ISSUE_PEAK_NOTE}


def ncu_traffic(walks):
    """DRAM bytes per launch of the walk kernel: the committed ncu capture's bytes per walk
    (profiles/ncu_summary.json, dram__bytes_read.sum + dram__bytes_write.sum) x walks."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            per_walk = json.load(f).get("walk_kernel_dram_bytes_per_walk")
        return None if per_walk is None else per_walk * walks
    except (OSError, ValueError):
        return None


def cpu_sample(walkers_hint=None):
    """Size of the bounded CPU sample: walkers [0, n) x 1 restart of the C4 workload
    (BENCH_CPU_WALKERS overrides n; the CPU tests use a tiny sample)."""
    cores = os.cpu_count() or 1
    n = walkers_hint or int(os.environ.get("BENCH_CPU_WALKERS", "0")) or \
        min(WALKERS_PER_GPU, max(16, CPU_WALKS_PER_CORE * cores))
    return cores, n


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _sample_config(walkers):
    """Walkers [0, walkers) x 1 restart of C4: walker w keeps its class (w mod 128) and its
    Rng stream w, so these are exactly the first walks of the C4 pool."""
    from oracle.oracle import make_config
    return make_config(L, walkers=walkers, prefix_len=P, target_merit=F, max_restarts=1,
                       seed=SEED)


def reference_cpu(threads, walkers, reps=1, warmup=0, trace=True):
    """The reference's CPU path on the host: oracle/_ref (the reference library compiled from
    its own sources) when present, else the C restatement.  Timed: the stock run_saw_pool
    (saw.cpp:218-267) with `threads` std::threads on walkers [0, walkers) x 1 restart of C4.
    Untimed (trace=True): the same walks through the reference's run_walk with a counting
    VisitedSet, replayed in --threads 1 order through its DedupSink -- the delta-eval count
    and the ordered candidate list the GPU parity diff uses."""
    from oracle.oracle import Reference, Restated, reference_available
    cfg = _sample_config(walkers)
    tr = None
    if reference_available():
        lib, kind = Reference(), "reference"
        if trace:
            tr = lib.walk_trace_mt(cfg, threads)
        run = lambda: lib.run_saw_pool(cfg, threads=threads)  # noqa: E731
    else:
        lib, kind = Restated(), "port"
        threads = 1
        run = lambda: lib.run_saw_pool(cfg)  # noqa: E731
    times, res = [], None
    for i in range(warmup + reps):
        t0 = time.perf_counter()
        res = run()
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    if tr is None:
        tr = res if kind == "port" else None
    evals = tr.stats["delta_evals"] if tr is not None else None
    return dict(kind=kind, times=times, stats=res.stats, evals=evals, threads=threads, trace=tr)


def single_thread_leg(walkers=None):
    """threads = 1 rate of the reference: a smaller sample, timed."""
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        return None
    n = walkers or int(os.environ.get("BENCH_CPU_WALKERS_1T", "0")) or 16
    lib = Reference()
    cfg = _sample_config(n)
    evals = lib.count_deltas(cfg, os.cpu_count() or 1)["delta_evals"]
    t0 = time.perf_counter()
    lib.run_saw_pool(cfg, threads=1)
    dt = time.perf_counter() - t0
    return {"value": evals / dt, "unit": "flip-deltas/s", "cores": 1,
            "sample": f"C4 walkers [0,{n}) x 1 restart, {evals} delta evals in {dt:.2f} s "
                      f"(reference run_saw_pool, threads=1)"}


def tsv_lines(cands, fmt):
    """Candidate records with their (walker, restart) origin, in delivery order."""
    return [f"{c.walker}\t{c.restart}\t{fmt(c.seq, c.energy)}" for c in cands]


def gpu_parity(labs, ref, walkers):
    """Headline-scale parity: the C4 walks the CPU leg ran -- walkers
    [0, walkers) x 1 restart -- through the GPU's public run_saw_pool, diffed against the
    reference's --threads 1 candidate list (same order, same records) and pool stats."""
    import hashlib
    cfg = labs.SawConfig(length=L, walkers=walkers, prefix_len=P, target_merit=F,
                         max_restarts=1, seed=SEED, count_visited=True)
    sink = labs.CollectingSink()
    st = labs.run_saw_pool(cfg, sink)
    got = tsv_lines(sink.take(), labs.format_record)
    want = tsv_lines(ref.candidates, labs.format_record)
    sha = lambda lines: hashlib.sha256("\n".join(lines).encode()).hexdigest()  # noqa: E731
    stats = {k: (getattr(st, k), ref.stats[k])
             for k in ("walks", "iterations", "emitted", "best_energy", "delta_evals")}
    same_stats = all(a == b for a, b in stats.values())
    return {"workload": f"C4 walkers [0,{walkers}) x 1 restart (L={L} p={P} F>={F} seed={SEED})",
            "walks": st.walks, "candidates_gpu": len(got), "candidates_reference": len(want),
            "sha256_gpu": sha(got), "sha256_reference": sha(want),
            "stats_gpu_vs_reference": stats,
            "identical": got == want and same_stats,
            "compared": "ordered TSV records (walker, restart, L, E, F, hex, origin) and pool "
                        "stats (walks, iterations, emitted, best E, delta evals); reference = "
                        "its run_walk + DedupSink in --threads 1 order (oracle/_ref)"}


def enum_c2(labs, peak, m=36):
    """BASELINE config 2: K4 Gray enumeration of restriction class 0
    at L=201, p=12, over the lowest m = 36 free half positions (the rest +1; 2^36 Gray
    steps, ~2 s), sieve F >= 5.0.  Roofline: the FMA pipe (IDP4A + IMAD share it, 64
    lanes/clk/SM): per Gray step every even lag takes two IDP4A (its dc) and one IMAD (its
    C^2), i.e. 3 FMA-pipe lane-ops per lag, (L-1)/2 lags."""
    L2, p2, cls, e_l = 201, 12, 0, 4040
    labs.enumerate_class(L2, p2, cls, 20, e_l, collect=False)  # warm-up
    hits, st = labs.enumerate_class(L2, p2, cls, m, e_l, collect=False)
    steps_s = st["configurations"] / (st["kernel_ms"] / 1e3)
    fma_per_step = 3 * (L2 - 1) // 2
    achieved = steps_s * fma_per_step
    peak_fma = peak["dp4a"] if peak else None
    return {"workload": f"C2: L={L2} p={p2} class {cls}, Gray range over {m} free half positions "
                        f"(2^{m} configurations), E < {e_l} (F >= 5.0)",
            "gray_steps_per_s": steps_s, "lag_updates_per_s": steps_s * (L2 - 1) // 2,
            "kernel_ms": st["kernel_ms"], "best_energy": st["best_energy"],
            "emitted": st["emitted"],
            "roofline": {"bound": "fma_pipe", "achieved": achieved, "peak": peak_fma,
                         "unit": "lane-ops/s", "frac": achieved / peak_fma if peak_fma else None,
                         "per_step": f"{fma_per_step} FMA-pipe lane-ops (2 IDP4A + 1 IMAD per "
                                     f"even lag)",
                         "peak_source": "measured in this run: IDP4A lane-instr/s (the FMA "
                                        "pipe's issue rate, labs_int32_peak)",
                         "issue": issue_roofline(steps_s, "r02/enum_kernel_ncu.json",
                                                 "warp_instructions_per_gray_step", peak)}}


def run_reference_arm(args, ws, rank):
    if rank != 0:
        return
    threads, walkers = cpu_sample()
    r = reference_cpu(threads, walkers, args.steps, args.warmup)
    t = statistics.mean(r["times"])
    v = r["evals"] / t
    line = {
        "impl": "reference", "metric": "flip-delta evals/sec (L=451)", "value": v,
        "unit": "flip-deltas/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"C4 sample: L={L} p={P} F>={F} T_i=1808 fpr=1e-4 seed=1, "
                               f"walkers [0,{walkers}) x 1 restart",
                   "threads": r["threads"]},
        "candidates_per_s": r["stats"]["emitted"] / t,
        "cpu_baseline": {"value": v, "unit": "flip-deltas/s", "cores": r["threads"],
                         "kind": r["kind"], "cpu_model": cpu_model(),
                         "sample": f"C4 walkers [0,{walkers}) x 1 restart ({r['evals']} delta "
                                   f"evals per step, run_saw_pool threads={r['threads']})"},
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
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-c2", action="store_true", help="skip the C2 enumeration keys")
    args = ap.parse_args()
    ws, rank, local = dist_env()

    dist = None
    if ws > 1:
        import torch.distributed as dist
        # BENCH_DIST_BACKEND / BENCH_SAME_DEVICE: functional test of the N-rank flow on a
        # one-GPU box (all ranks on device 0, gloo); the driver's runs use neither
        backend = os.environ.get("BENCH_DIST_BACKEND") or ("nccl" if args.impl == "b200" else "gloo")
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
    if os.environ.get("BENCH_SAME_DEVICE"):
        local = 0
    # (the max / sum reductions of the per-rank timings: on the device under NCCL, on the
    # host under gloo)
    red_dev = "cpu" if dist is not None and dist.get_backend() == "gloo" else "cuda"
    torch.cuda.set_device(local)

    walkers = args.walkers_per_gpu * ws
    base = dict(length=L, walkers=walkers, prefix_len=P, target_merit=F,
                max_restarts=args.restarts, seed=SEED, device=local,
                shard_index=rank, shard_count=ws)

    # ---- reference-equivalent counts for this rank's walks (same walks, untimed)
    with labs.bench_plan(labs.SawConfig(count_visited=True, **base)) as cp:
        _, cst = cp.run(1)
    deltas_rank, iters_rank = cst.delta_evals, cst.iterations

    peak = labs.int32_peak() if rank == 0 else None

    plan = labs.bench_plan(labs.SawConfig(**base))
    clocks = Clocks(local) if rank == 0 else None
    for _ in range(args.warmup):
        plan.run(1)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    ms_step, st = plan.run(args.steps)  # device ms per step (CUDA events on the lib stream)
    torch.cuda.synchronize()
    t1 = time.time()
    if dist is not None:
        dist.barrier()
    clk = clocks.stop(t0, t1) if clocks else None

    vals = torch.tensor([ms_step, float(deltas_rank), float(st.emitted), float(iters_rank),
                         st.kernel_ms, float(st.walks)], dtype=torch.float64, device=red_dev)
    if dist is not None:
        mx, sm = vals.clone(), vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, kms_max = mx[0].item(), mx[4].item()
        deltas_all, emitted_all, iters_all, walks_all = (sm[1].item(), sm[2].item(),
                                                         sm[3].item(), sm[5].item())
    else:
        ms_max, deltas_all, emitted_all, iters_all, kms_max, walks_all = [v.item() for v in vals]

    # ---- e2e through the public API: host config in, candidates out through the sink.
    # Every call uploads its seed tables (pinned staging) and reads back the sieve records
    # and per-walk stats; wall clock per call (median of --e2e-steps calls), max over ranks.
    e2e_times, e2e_stats = [], None
    cfg_api = labs.SawConfig(**base)
    for i in range(1 + args.e2e_steps):
        sink = labs.CollectingSink()
        if dist is not None:
            dist.barrier()
        ta = time.perf_counter()
        e2e_stats = labs.run_saw_pool(cfg_api, sink)
        dt = time.perf_counter() - ta
        if i > 0:
            e2e_times.append(dt)
    e2e_t = torch.tensor([statistics.median(e2e_times)], dtype=torch.float64, device=red_dev)
    if dist is not None:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_s = e2e_t.item()

    if rank == 0:
        step_s = ms_max / 1e3
        value = deltas_all / step_s
        # roofline of the dominant kernel (the walk kernel: K1t at L=451): algorithmic int8 MACs
        # per launch / its CUDA-event duration.  The MAC work (the sliding dot products G) runs
        # on the int8 tensor cores (mma.sync) in K1t and on IDP4A in K1; both peaks are
        # measured in this run.  The step is bound by instruction issue of the per-step
        # bookkeeping, not by either MAC pipe: for K1t the headline `frac` is the
        # issue fraction (warp-instructions per walk iteration from the committed ncu capture x
        # iterations/s over 4 SMSPs x SMs x clock); `idp4a` keeps r01's basis (the CUDA-core
        # int8 MAC peak) and `tensor` is the same work against the mma.sync int8 peak.
        alg_ops = (deltas_rank + iters_rank) * OPS_PER_DELTA
        achieved = alg_ops / (st.kernel_ms / 1e3) / 1e12
        peak_v = peak["dp4a"] * 8 / 1e12 if peak else None
        imma = labs.imma_peak() if rank == 0 else None
        kern = labs.derive(labs.SawConfig(**base)).get("kernel", None)
        issue = issue_roofline(iters_rank / (st.kernel_ms / 1e3), "ncu_summary.json",
                               "warp_instructions_per_walk_iteration", peak)
        idp4a = {"bound": "int32", "achieved": achieved, "peak": peak_v, "unit": "Tops/s",
                 "frac": (achieved / peak_v) if peak_v else None,
                 "peak_source": "measured in this run (labs_int32_peak): IDP4A lane-instr/s x 8 "
                                "int ops (4 int8 MACs), the CUDA-core int8 MAC peak (r01 basis; "
                                "K1t runs G on the tensor pipe, so this can pass 1)"}
        tensor = {"peak": imma * 2 / 1e12 if imma else None, "unit": "Tops/s",
                  "frac": achieved / (imma * 2 / 1e12) if imma else None,
                  "peak_source": "measured in this run (labs_imma_peak): "
                                 "mma.sync.m16n8k32.s8 int8 MACs/s x 2 ops"}
        if kern == 1 and issue:  # K1t: instruction issue binds
            roof = dict(issue, idp4a=idp4a)
        else:  # K1: the IDP4A (FMA) pipe and issue
            roof = dict(idp4a, issue=issue)
        roof.update({"tensor": tensor, "traffic": ncu_traffic(st.walks),
                     "traffic_source": "profile constant: profiles/ncu_summary.json (ncu --set full "
                                       "capture of the walk kernel, DRAM bytes per walk x walks)",
                     "walk_kernel": {0: "K1 (IDP4A G)", 1: "K1t (mma.sync int8 G)"}.get(kern, kern),
                     "int32_peak_detail": peak,
                     "alg_ops_per_launch": alg_ops,
                     "alg_unit": f"(reference-equivalent delta evals + applies) x (L+1) ops: one "
                                 f"delta = inner product of (L+1)/2 = {(L + 1) // 2} int8 MACs",
                     "kernel_ms_per_launch": st.kernel_ms,
                     "ref_equiv_tops": deltas_all * REF_OPS_PER_DELTA / step_s / 1e12})
        cpu, parity = None, None
        if not args.no_cpu_baseline:
            try:
                threads, cw = cpu_sample()
                r = reference_cpu(threads, cw)
                dt = r["times"][0]
                cpu = {"value": r["evals"] / dt, "unit": "flip-deltas/s", "cores": r["threads"],
                       "kind": r["kind"], "cpu_model": cpu_model(),
                       "sample": f"C4 walkers [0,{cw}) x 1 restart, {r['evals']} delta evals "
                                 f"in {dt:.2f} s (reference run_saw_pool, {r['threads']} threads)",
                       "threads_1": single_thread_leg()}
                if r["trace"] is not None:
                    parity = gpu_parity(labs, r["trace"], cw)
            except Exception as e:  # baseline is reported, never fatal
                cpu = {"value": None, "error": f"{type(e).__name__}: {e}"}
        free = (L + 1) // 2 - P
        line = {
            "metric": "flip-delta evals/sec (L=451)",
            "value": value,
            "unit": "flip-deltas/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "int8x4->int32",
            "data": "synthetic",
            "config": {"workload": f"C4: L={L} p={P} F>={F} (E_l=19188) T_i=1808 fpr=1e-4 seed=1, "
                                   f"{args.walkers_per_gpu} walkers x {args.restarts} restarts "
                                   f"per GPU, class-sharded",
                       "walks_per_gpu": args.walkers_per_gpu * args.restarts,
                       "l2": "flushed: a 256 MiB buffer is written before every step (outside "
                             "the timed events); per-walk state lives in shared memory",
                       "parallelism": f"class-shard x{ws}"},
            "candidates_per_s": emitted_all / step_s,
            "candidates_per_step": emitted_all,
            "walks_per_step": walks_all,
            "walk_iterations_per_s": iters_all / step_s,
            "delta_evals_per_step": deltas_all,
            "delta_evals_computed_per_step": (iters_all + walks_all) * free,
            "kernel_ms_per_step": kms_max,
            "gpu_launches": 2 * args.steps * ws,
            "roofline": roof,
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": {"value": deltas_all / e2e_s, "unit": "flip-deltas/s",
                    "h2d_bytes_per_step": e2e_stats.h2d_bytes,
                    "d2h_bytes_per_step": e2e_stats.d2h_bytes,
                    "s_per_step": e2e_s, "candidates_per_step": e2e_stats.emitted,
                    "path": "paper_2409_07222_b200.run_saw_pool -> C ABI labs_saw_pool_run "
                            "(host seed tables in, deduplicated candidates out)"},
            "clocks": clk,
            "c2_enumeration": enum_c2(labs, peak) if not args.no_c2 else None,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
