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


@pytest.mark.gpu
@pytest.mark.parametrize("exe", [SOLVE_S1, SOLVE_B200], ids=["gpu_step1", "gpu_step1_step2"])
def test_experiment_matches_reference(tmp_path, exe):
    # experiment_compare (pipeline.cpp:390-438) runs two Step-1 pools
    # per run; with the B200 pool its per-run energies, medians and rank-sum test must be
    # the reference's
    if not os.access(SOLVE_REF, os.X_OK):
        pytest.skip("reference solve not built")
    args = ("experiment -L 61 --runs 5 --walkers 8 --restarts 3 --target-f 4.0 --tu 80 "
            "--tr 3 --refine-top 3 --seed 5").split()
    outs = []
    for tag, e in (("b200", exe), ("ref", SOLVE_REF)):
        csv = tmp_path / f"{tag}.csv"
        r = subprocess.run([e, *args, "--out", str(csv)], capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr
        outs.append((r.stdout, csv.read_text()))
    assert outs[0] == outs[1]
    assert outs[0][1].count("\n") == 6  # header + 5 runs


@pytest.mark.gpu
def test_verify_accepts_gpu_written_records(tmp_path):
    # verify_records (pipeline.cpp:335-388) over the GPU Step-1 TSVs:
    # the `labs saw` candidate file and the solve candidate/results files
    labs_cli = os.path.join(ROOT, "paper_2409_07222_b200", "_lib", "labs")
    saw = tmp_path / "saw.tsv"
    r = subprocess.run([labs_cli, "saw", "-L", "101", "--walkers", "64", "--p", "8",
                        "--restarts", "4", "--target-f", "4.5", "--out", str(saw)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    _, _, out, cands = _run(SOLVE_B200, "-L 45 --rounds 1 --walkers 8 --restarts 2 --target-f 4.0 "
                            "--refine-top 3 --tu 90 --tr 3 --seed 3 --threads 1 --deterministic "
                            "--no-construct".split(), tmp_path, "v")
    files = [str(saw), str(tmp_path / "v_out.tsv"), str(tmp_path / "v_cands.tsv")]
    r = subprocess.run([SOLVE_B200, "verify", *files], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout
    lines = r.stdout.strip().splitlines()
    assert len(lines) == 3 and all("0 mismatches, 0 malformed" in x for x in lines)
    assert int(lines[0].split(": ")[1].split()[0]) == len(saw.read_text().splitlines()) > 0


def test_verify_flags_corrupted_record(tmp_path):
    # (CPU) the verify path itself: a record whose stored energy disagrees is reported,
    # exit status 1 (labs_main.cpp:276-290)
    bad = tmp_path / "bad.tsv"
    # L=5 skew optimum +++-+ (hex 1D) has E=2; line 1 stores 3 instead
    bad.write_text("5\t3\t4.1667\t1D\tsaw\n5\t2\t6.2500\t1D\tsaw\nnot a record\n")
    r = subprocess.run([SOLVE_B200, "verify", str(bad)], capture_output=True, text=True,
                       timeout=60)
    assert r.returncode == 1
    assert "2 records, 1 mismatches, 1 malformed" in r.stdout
    assert "energy mismatch" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("exe", [SOLVE_S1, SOLVE_B200], ids=["gpu_step1", "gpu_step1_step2"])
def test_solve_multithreaded_matches_reference(tmp_path, exe):
    # --threads 4: the reference's Step-1 pool and refine_batch (pipeline.cpp:132-186) then
    # run concurrently, so emission order and equal-energy ties are timing-dependent even
    # for the reference; the candidate SET, the best energy per target length and the Step-1
    # statistics must match.  Exercises K5's per-thread context cache (refine threads
    # alternate lengths L-1, L, L+1 through refine_with_operators).
    if not os.access(SOLVE_REF, os.X_OK):
        pytest.skip("reference solve not built")
    a = ("-L 62 --rounds 2 --walkers 16 --restarts 3 --target-f 4.0 --refine-top 6 --tu 120 "
         "--tr 4 --seed 11 --threads 4 --deterministic --no-construct").split()
    got = _run(exe, a, tmp_path, "b200")
    want = _run(SOLVE_REF, a, tmp_path, "ref")
    assert sorted(got[3].splitlines()) == sorted(want[3].splitlines())   # candidate set
    best = lambda txt: sorted(tuple(l.split("\t")[:2]) for l in txt.splitlines() if l)  # noqa: E731
    assert best(got[2]) == best(want[2])                                 # (L, E) per target
    assert got[1].split(" wall=")[0].split("calls=")[0] == want[1].split(" wall=")[0].split("calls=")[0]


@pytest.mark.gpu
def test_acceptance_c5_search_quality():
    # The reference's acceptance criterion 5 (acceptance.cpp:147-176) through the pipeline
    # with the B200 Step 1 (and K5 Step 2): lengths 21 and 27, 60 s budget, stop at the
    # optimal merit, walkers 8, unlimited restarts, F >= 4 sieve, T_u 400, refine_top 4,
    # no construction, seeds 500..509 -- at least 9 of 10 runs reach the optimum energy
    # (oracle_exhaustive: E(21) = 26, E(27) = 37).  With threads >= walkers every walker
    # (restriction class) searches at once, as the reference's pool does with as many
    # threads (saw.cpp:242-257); with --threads 1 both the reference and this build search
    # walker 0's class only (2^7 starting halves at p = 4), which does not hold the optimum.
    for length, e_opt in ((21, 26), (27, 37)):
        f_opt = length * length / (2.0 * e_opt) * (1 - 1e-12)
        hits = 0
        for run in range(10):
            r = subprocess.run([SOLVE_B200, "solve", "-L", str(length), "--seconds", "60",
                                "--stop-at-merit", repr(f_opt), "--walkers", "8", "--restarts", "0",
                                "--target-f", "4.0", "--tu", "400", "--refine-top", "4",
                                "--seed", str(500 + run), "--threads", "8", "--no-construct"],
                               capture_output=True, text=True, timeout=120)
            assert r.returncode == 0, r.stderr
            rec = [dict(f.split("=", 1) for f in l.split()) for l in r.stdout.splitlines()
                   if l.startswith(f"L={length} ")]
            hits += bool(rec) and int(rec[0]["E"]) == e_opt
        assert hits >= 9, (length, hits)
