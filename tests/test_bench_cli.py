"""bench.py's launch contract on CPU: the reference arm under torchrun (N=2, gloo) prints
exactly one JSON line from rank 0 with the contract's keys, and every rank exits 0."""
import json
import os
import socket
import subprocess
import sys

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
