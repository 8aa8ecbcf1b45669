"""bench.py's launch contract: the reference arm under torchrun (N=2, gloo) on CPU, and the
b200 arm under torchrun (N=2 on one B200, -m gpu) print exactly one JSON line from rank 0
with the contract's keys, and every rank exits 0."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(args, env_extra):
    env = dict(os.environ, BENCH_CPU_WALKERS="2", **env_extra)
    return subprocess.run(args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)


def _check_line(out, n):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["n_gpus"] == n and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_single_process():
    r = _run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"], {})
    assert r.returncode == 0, r.stderr
    _check_line(r.stdout, 1)


def test_reference_arm_torchrun_two_ranks():
    r = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
              "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"], {})
    assert r.returncode == 0, r.stderr[-2000:]
    _check_line(r.stdout, 2)


@pytest.mark.gpu
def test_b200_arm_torchrun_two_ranks_one_device():
    # the N>1 b200 arm: torchrun world 2 (both ranks on the one B200, gloo for the
    # reductions), class shards per rank, max-over-ranks timing; one JSON line from rank 0
    r = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
              "--gpus", "2", "--steps", "1", "--warmup", "1", "--walkers-per-gpu", "128",
              "--restarts", "2", "--no-cpu-baseline", "--no-c2", "--e2e-steps", "1"],
             {"BENCH_SAME_DEVICE": "1", "BENCH_DIST_BACKEND": "gloo"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["walks_per_step"] == 2 * 128 * 2
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
