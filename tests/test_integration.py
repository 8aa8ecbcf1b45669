"""Config 5 path: the reference's own `solve` pipeline (run_pipeline, Step 2 = pq.cpp)
with the B200 Step 1 linked in (integration/_build/labs_solve), diffed end to end against
the unmodified reference solve (oracle/_ref/labs_solve_ref, CPU Step 1).  Because Step 1
delivers the same candidates in --threads 1 order, every downstream byte must match:
stdout records, the results file and the candidate file (acceptance.cpp:278-313 C10,
test_pipeline.cpp:144-171)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SOLVE_B200 = os.path.join(ROOT, "integration", "_build", "labs_solve")        # Step 1 + K5 Step 2
SOLVE_S1 = os.path.join(ROOT, "integration", "_build", "labs_solve_s1")       # Step 1 only
SOLVE_REF = os.path.join(ROOT, "oracle", "_ref", "labs_solve_ref")


def _run(exe, args, tmp, tag):
    out, cands = tmp / f"{tag}_out.tsv", tmp / f"{tag}_cands.tsv"
    r = subprocess.run([exe, "solve", *args, "--out", str(out), "--candidates", str(cands)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return r.stdout, r.stderr, out.read_text(), cands.read_text()


def test_integration_binaries_built():
    assert os.access(SOLVE_B200, os.X_OK) and os.access(SOLVE_S1, os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("exe", [SOLVE_S1, SOLVE_B200], ids=["gpu_step1", "gpu_step1_step2"])
@pytest.mark.parametrize("args", [
    # acceptance C10 (acceptance.cpp:295-297)
    "-L 25 --rounds 2 --walkers 4 --restarts 5 --target-f 3.5 --tu 80 --seed 99 --threads 1 "
    "--deterministic --no-construct",
    # even target -> odd walk lengths 31, 33 + length operators; two rounds
    "-L 32 --rounds 2 --walkers 8 --restarts 3 --target-f 3.5 --tu 60 --seed 7 --threads 1 "
    "--deterministic --no-construct",
    # config-5 shape at a CPU-checkable size: p=8 classes, refine_top 6, T_r 5
    "-L 101 --rounds 1 --p 8 --walkers 32 --restarts 2 --target-f 5.0 --refine-top 6 --tu 202 "
    "--tr 5 --seed 1 --threads 1 --deterministic --no-construct",
    # construction seeds (construct.cpp) refined alongside the walk candidates
    "-L 45 --rounds 1 --walkers 8 --restarts 2 --target-f 4.0 --refine-top 3 --tu 90 --tr 3 "
    "--seed 3 --threads 1 --deterministic",
])
def test_solve_matches_reference_pipeline(tmp_path, args, exe):
    if not os.access(SOLVE_REF, os.X_OK):
        pytest.skip("reference solve not built")
    a = args.split()
    got = _run(exe, a, tmp_path, "b200")
    want = _run(SOLVE_REF, a, tmp_path, "ref")
    assert got[0] == want[0]                      # best records on stdout
    assert got[1].split(" wall=")[0] == want[1].split(" wall=")[0]   # walks/candidates/calls
    assert got[1].split("fingerprint=")[1] == want[1].split("fingerprint=")[1]
    assert got[2] == want[2]                      # results file (deterministic: wall 0)
    assert got[3] == want[3]                      # candidate file, emission order
