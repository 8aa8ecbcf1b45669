"""Engine-level behaviour of the GPU pool (run_saw_pool, saw.cpp:218-267) on a B200:
pipelined multi-job pools, the sieve's record ring under pressure (no rerun, north_star (d)),
coupled stop conditions at full width (saw.cpp:153-170,204-208,242-257) and the in-process
multi-shard merge.  Results are compared with the oracle / the reference compiled from its
own sources (oracle/_ref) wherever the reference is deterministic."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.oracle import make_config

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(labs, **kw):
    sink = labs.CollectingSink()
    cfg = labs.SawConfig(**kw)
    if cfg.time_budget_s > 0:  # (device setup of a cold process stays out of the budget)
        labs.prepare_saw_pool(cfg)
    st = labs.run_saw_pool(cfg, sink)
    return st, sink.take()


def _key(c):
    return (c.walker, c.restart, c.iteration, c.energy, c.seq.tobytes())


def _same_as_reference(got, st, ref):
    assert [(c.walker, c.restart, c.energy, c.seq.tobytes()) for c in got] == \
        [(c.walker, c.restart, c.energy, c.seq.tobytes()) for c in ref.candidates]
    for k in ("walks", "iterations", "emitted", "best_energy"):
        assert getattr(st, k) == ref.stats[k], k


def test_pipelined_jobs_equal_one_job(labs, reference, monkeypatch):
    # total walks > 4 x resident: the independent pool runs as a pipeline of jobs on two
    # streams, generator streams continuing on the device between jobs; the result equals
    # the one-job run and the reference on a walker subset
    kw = dict(length=101, walkers=1024, prefix_len=8, target_merit=4.6, max_restarts=64, seed=5)
    st, got = _run(labs, **kw)
    monkeypatch.setenv("LABS_PIPELINE_BATCHES", "1")
    st1, got1 = _run(labs, **kw)
    monkeypatch.delenv("LABS_PIPELINE_BATCHES")
    monkeypatch.setenv("LABS_PRESEED", "0")  # one K3 per job instead of one for the pool
    st0, got0 = _run(labs, **kw)
    monkeypatch.delenv("LABS_PRESEED")
    assert st.walks == 65536 and [_key(c) for c in got] == [_key(c) for c in got1]
    assert [_key(c) for c in got] == [_key(c) for c in got0]
    for k in ("walks", "iterations", "emitted", "best_energy", "emitted_raw"):
        assert getattr(st, k) == getattr(st1, k) == getattr(st0, k), k
    # walkers 1000..1023 (their restarts sit in the pipeline's last jobs)
    sub = dict(kw, walker_begin=1000)
    st2, got2 = _run(labs, **sub)
    ref = reference.walk_trace_mt(make_config(**sub), os.cpu_count() or 1)
    _same_as_reference(got2, st2, ref)


def test_ring_wraps_without_rerun(labs, restated, monkeypatch):
    # a 64-slot record ring and a loose threshold: thousands of sieve hits per launch
    # stream through the ring while K1 runs (drained by async copies), none lost or reordered
    monkeypatch.setenv("LABS_RING_SLOTS", "64")
    kw = dict(length=101, walkers=64, prefix_len=8, target_merit=3.0, max_restarts=4, seed=17)
    st, got = _run(labs, **kw)
    ref = restated.run_saw_pool(make_config(**kw))
    assert st.emitted_raw > 64 * 50
    assert [_key(c) for c in got] == [(c.walker, c.restart, c.iteration, c.energy, c.seq.tobytes())
                                      for c in ref.candidates]
    for k in ("walks", "iterations", "emitted", "best_energy"):
        assert getattr(st, k) == ref.stats[k], k


def test_c4_loose_threshold_ring(labs, reference, monkeypatch):
    # C4 at --target-f 3.5 emits far more hits than the ring holds,
    # with identical output and no rerun
    monkeypatch.setenv("LABS_RING_SLOTS", "1024")
    kw = dict(length=451, walkers=1024, prefix_len=8, target_merit=3.5, max_restarts=1, seed=1,
              walker_end=16)
    st, got = _run(labs, **kw)
    assert st.emitted_raw > 1024 * 4
    ref = reference.walk_trace_mt(make_config(**kw), os.cpu_count() or 1)
    _same_as_reference(got, st, ref)


def test_unlimited_restarts_run_every_walker(labs):
    # max_restarts = 0 with a time budget and threads > 1: every walker runs concurrently
    # (saw.cpp:242-257 with threads >= walkers), so every restriction class is searched
    cfg = dict(length=101, walkers=256, prefix_len=8, target_merit=4.6, max_restarts=0,
               time_budget_s=1.0, seed=7, threads=16)
    st, got = _run(labs, **cfg)
    # (a loose threshold: ~1.7M candidates reach the Python sink inside the budget; the
    # overshoot is the replay of the batches in flight at the deadline)
    assert st.wall_seconds < 1.0 + 1.0, st.wall_seconds
    assert st.walks >= 256
    assert {c.walker for c in got} == set(range(256))
    assert {c.walker % 128 for c in got} == set(range(128))
    assert len({c.seq.tobytes() for c in got}) == len(got) == st.emitted
    # restarts of each walker are delivered in order
    last = {}
    for c in got:
        assert c.restart >= last.get(c.walker, 0)
        last[c.walker] = c.restart


def test_unlimited_restarts_single_thread_is_walker_zero(labs):
    # --threads 1 (the reference's serial pool): walker 0 restarts until the deadline
    st, got = _run(labs, length=101, walkers=64, prefix_len=8, target_merit=3.2, max_restarts=0,
                   time_budget_s=0.5, seed=7, threads=1)
    assert got and {c.walker for c in got} == {0}


def test_time_budget_overshoot_is_bounded(labs):
    # L=451 walks take ~10 ms per wave: batches sized from the measured rate and the
    # remaining budget keep the overshoot well under a second
    st, _ = _run(labs, length=451, walkers=1024, prefix_len=8, target_merit=5.3, max_restarts=0,
                 time_budget_s=1.5, seed=3, threads=8)
    assert st.walks > 1024 and st.wall_seconds < 1.5 + 0.5, (st.wall_seconds, st.walks)


def test_quota_full_width_and_multi_shard(labs):
    # quota with threads > 1 on two in-process shards: exactly `quota` distinct candidates
    for n_gpus in (1, 2):
        st, got = _run(labs, length=101, walkers=128, prefix_len=8, target_merit=4.0,
                       max_restarts=50, candidate_quota=500, seed=9, threads=8, n_gpus=n_gpus)
        assert st.emitted == len(got) == 500
        assert len({c.seq.tobytes() for c in got}) == 500


def test_stop_at_energy_full_width(labs):
    st, got = _run(labs, length=101, walkers=128, prefix_len=8, target_merit=4.0,
                   max_restarts=0, stop_at_energy=600, seed=4, threads=8)
    assert st.best_energy <= 600
    assert all(c.energy >= st.best_energy for c in got)


def test_coupled_exact_order_multi_shard(labs, restated):
    # --threads 1 semantics with a quota split over two in-process shards: the delivery
    # order (and so the quota cut) is the reference's --threads 1 order
    kw = dict(length=101, walkers=16, prefix_len=8, max_restarts=3, target_merit=4.0,
              candidate_quota=40, seed=3)
    st, got = _run(labs, n_gpus=2, **kw)
    ref = restated.run_saw_pool(make_config(**kw))
    assert [_key(c) for c in got] == [(c.walker, c.restart, c.iteration, c.energy, c.seq.tobytes())
                                      for c in ref.candidates]
    assert st.emitted == 40 and st.walks == ref.stats["walks"]


def test_in_process_two_shards_e2e(labs, restated):
    # n_gpus = 2 independent pool (shards share the one B200 on separate streams): the merged
    # list is the single-device --threads 1 list
    kw = dict(length=201, walkers=256, prefix_len=8, target_merit=5.0, max_restarts=8, seed=2)
    st2, got2 = _run(labs, n_gpus=2, **kw)
    st1, got1 = _run(labs, **kw)
    assert [_key(c) for c in got2] == [_key(c) for c in got1]
    for k in ("walks", "iterations", "emitted", "best_energy"):
        assert getattr(st2, k) == getattr(st1, k), k
    assert st2.n_gpus == 2


def test_torchrun_two_ranks_real_runner(labs, tmp_path):
    # one process per GPU (here both ranks on device 0): run_saw_pool_distributed with the
    # real GPU runner gives the single-process candidate list on rank 0
    out = tmp_path / "dist.tsv"
    script = tmp_path / "dist.py"
    script.write_text(f"""
import os, sys
sys.path.insert(0, {ROOT!r})
import torch.distributed as dist
import paper_2409_07222_b200 as labs
from paper_2409_07222_b200.distributed import run_saw_pool_distributed
dist.init_process_group("gloo")
cfg = labs.SawConfig(length=101, walkers=128, prefix_len=8, target_merit=5.0, max_restarts=4,
                     seed=13, device=0)
sink = labs.CollectingSink()
st = run_saw_pool_distributed(cfg, sink)
if dist.get_rank() == 0:
    with open({str(out)!r}, "w") as f:
        for c in sink.take():
            f.write(f"{{c.walker}}\\t{{c.restart}}\\t{{labs.format_record(c)}}\\n")
        f.write(f"#{{st.walks}} {{st.iterations}} {{st.emitted}} {{st.best_energy}}\\n")
dist.destroy_process_group()
""")
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), str(script)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    st, got = _run(labs, length=101, walkers=128, prefix_len=8, target_merit=5.0, max_restarts=4,
                   seed=13)
    want = [f"{c.walker}\t{c.restart}\t{labs.format_record(c)}" for c in got]
    want.append(f"#{st.walks} {st.iterations} {st.emitted} {st.best_energy}")
    assert out.read_text().splitlines() == want


def test_cli_saw_unlimited_restarts_searches_every_class(tmp_path, restated):
    # `labs saw --restarts 0 --seconds 2` (the CLI's default --threads is the
    # host's hardware concurrency, labs_main.cpp:21-28) searches every restriction class at
    # once -- all 128 p=8 prefixes appear among the records -- and stops within the budget
    exe = os.path.join(ROOT, "paper_2409_07222_b200", "_lib", "labs")
    out = tmp_path / "c.tsv"
    r = subprocess.run([exe, "saw", "-L", "101", "--walkers", "256", "--p", "8", "--restarts", "0",
                        "--seconds", "2", "--target-f", "4.8", "--out", str(out)],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    recs = out.read_text().splitlines()
    prefixes = set()
    for line in recs:
        hexs = line.split("\t")[3]
        bits = bin(int(hexs, 16))[2:].zfill(101)
        prefixes.add(bits[:8])  # s_0..s_7 = the class prefix (MSB-first, +1 -> 1)
    assert len(prefixes) == 128, len(prefixes)
    stats = dict(f.split("=") for f in r.stderr.split() if "=" in f)
    assert float(stats["wall"].rstrip("s")) < 2.0 + 1.0
    assert int(stats["walks"]) >= 256
