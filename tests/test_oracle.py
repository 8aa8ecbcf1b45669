"""Pins the CPU oracle (oracle/labs_oracle.c, test infrastructure) to the reference.

CPU only (no GPU marker).  Two anchors, as SURVEY.md §8(c) lists them:
  * the known-answer tests of the reference's own test suite (file:line cited per test);
  * the reference library compiled from its own sources (oracle/_ref/liblabs_ref.so) and
    the golden fixtures it generated (tests/golden/saw_pool.json, make_golden.py).
Once the restatement agrees with both, the GPU parity tests (test_gpu_parity.py) may use
it as the checker.
"""
import json
import os

import numpy as np
import pytest

from oracle.oracle import make_config

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand_signs(rng, n):
    return rng.choice(np.array([-1, 1], dtype=np.int8), size=n)


def _scratch_energy(s):
    s = s.astype(np.int64)
    n = len(s)
    return int(sum(int(np.dot(s[: n - k], s[k:])) ** 2 for k in range(1, n)))


# ------------------------------------------------------------------ KATs of the reference tests
def test_expand_skew_kat(restated):
    # test_skew.cpp:9-15
    assert list(restated.expand_skew(np.array([1, 1, 1], np.int8))) == [1, 1, 1, -1, 1]


def test_odd_lags_vanish(restated):
    # test_skew.cpp:21-29, acceptance.cpp:105-120 (1,000 expansions)
    rng = np.random.default_rng(7)
    for _ in range(200):
        L = int(rng.integers(2, 60)) * 2 + 1
        s = restated.expand_skew(_rand_signs(rng, (L + 1) // 2))
        c, _ = restated.correlations(s)
        assert not np.any(c[1::2])


def test_center_flip_kat(restated):
    # test_skew.cpp:31-42: [+,+,+,-,+] E=2; centre flip -> E=10, delta 8, C2=-3, C4=1
    s = restated.expand_skew(np.array([1, 1, 1], np.int8))
    c, e = restated.correlations(s)
    assert e == 2
    assert restated.skew_flip_delta_fast(s, 2) == 8
    s2, c2, e2 = restated.apply_skew_flip(s, 2)
    assert e2 == 10 and c2[2] == -3 and c2[4] == 1


def test_energy_threshold_kat(restated, ):
    # test_sequence.cpp:53 and the BASELINE thresholds
    assert restated.energy_threshold(455, 6.5) == 15925
    for L, f, el in [(101, 5.0, 1020), (201, 5.0, 4040), (301, 5.2, 8711), (451, 5.3, 19188),
                     (527, 5.3, 26200)]:
        assert restated.energy_threshold(L, f) == el


def test_walk_length_kat(restated):
    # test_saw.cpp:154-162 T_i(101) = 408; SURVEY.md A1
    assert restated.effective_iterations(101) == 408
    for L, t in [(201, 808), (301, 1208), (451, 1808), (527, 2112)]:
        assert restated.effective_iterations(L) == t


def test_bloom_sizing_kat(restated):
    # test_bloom.cpp:63-71 sizing formula; SURVEY.md A9 sizes
    for L, m in [(101, 7841), (201, 15509), (301, 23177), (451, 34679), (527, 40507)]:
        bits, k = restated.bloom_size(restated.effective_iterations(L) + 1, 1e-4)
        assert (bits, k) == (m, 13)


def test_skew_optima(restated):
    # test_pipeline.cpp:42-53: skew optima L=5 -> 2, L=21 -> 26, L=31 -> 79
    for L, e in [(5, 2), (21, 26), (31, 79)]:
        got, s = restated.oracle_skew_exhaustive(L)
        assert got == e and _scratch_energy(s) == e


def test_flip_delta_fast_equals_scratch(restated):
    # test_skew.cpp:71-101 (fast = slow = scratch), acceptance.cpp:62-102 (skew half)
    rng = np.random.default_rng(29)
    for L in (51, 101, 251, 527):
        for _ in range(6):
            half = _rand_signs(rng, (L + 1) // 2)
            s = restated.expand_skew(half)
            e0 = _scratch_energy(s)
            for hp in rng.integers(0, len(half), size=5):
                h2 = half.copy()
                h2[hp] = -h2[hp]
                want = _scratch_energy(restated.expand_skew(h2)) - e0
                assert restated.skew_flip_delta_fast(s, int(hp)) == want


def test_hex_and_record_format(restated):
    # test_hex.cpp:8-14 "1D" KAT: +1,+1,+1,-1,+1 -> 0b11101 = 0x1D
    s = np.array([1, 1, 1, -1, 1], np.int8)
    assert restated.format_record(s, 2) == "5\t2\t6.2500\t1D\tsaw"


# ------------------------------------------------------------------ restatement == reference
def test_primitives_match_reference(restated, reference):
    rng = np.random.default_rng(20250810)
    assert restated.rng_draws(1, 0, 64) == reference.rng_draws(1, 0, 64)
    assert restated.rng_draws(0xdeadbeef, 977, 16) == reference.rng_draws(0xdeadbeef, 977, 16)
    for p in (1, 3, 8, 12):
        assert np.array_equal(restated.rank_prefixes(p), reference.rank_prefixes(p))
    for L in (3, 51, 451, 527, 1023):  # kMaxLen = 1024 (rng.hpp:77)
        s = _rand_signs(rng, L)
        assert restated.canonical_hash(s, 0) == reference.canonical_hash(s, 0)
        assert restated.canonical_hash(s, 1) == reference.canonical_hash(s, 1)
    for pos in (0, 7, 225, 1023):
        for t in (0, 1):
            assert restated.flip_mask(pos, t) == reference.flip_mask(pos, t)
    for L in (101, 451, 527):
        for f in (4.0, 5.3, 6.5):
            assert restated.energy_threshold(L, f) == reference.energy_threshold(L, f)
        for mult in (8.0, 4.0, 2.5):
            assert restated.effective_iterations(L, 0, mult) == reference.effective_iterations(L, 0, mult)
    for cap, fpr in [(409, 1e-4), (1809, 1e-4), (100, 1e-3), (1, 0.5), (5, 0.3)]:
        assert restated.bloom_size(cap, fpr) == reference.bloom_size(cap, fpr)


def test_bloom_bit_array_matches_reference(restated, reference):
    # test_bloom.cpp:50-61: deterministic bit array (uint64 wrap-around indices)
    rng = np.random.default_rng(3)
    keys = [(int(a), int(b)) for a, b in rng.integers(0, 2**63, size=(300, 2), dtype=np.uint64)]
    keys += [(2**64 - 1, 2**64 - 3), (0, 0)]
    assert np.array_equal(restated.bloom_words(1809, 1e-4, keys),
                          reference.bloom_words(1809, 1e-4, keys))


def test_deltas_and_apply_match_reference(restated, reference):
    rng = np.random.default_rng(31)
    for _ in range(30):
        L = int(rng.integers(1, 60)) * 2 + 1
        s = restated.expand_skew(_rand_signs(rng, (L + 1) // 2))
        for hp in range((L + 1) // 2):
            assert restated.skew_flip_delta_fast(s, hp) == reference.skew_flip_delta_fast(s, hp)
        hp = int(rng.integers(0, (L + 1) // 2))
        a1, c1, e1 = restated.apply_skew_flip(s, hp)
        a2, c2, e2 = reference.apply_skew_flip(s, hp)
        assert np.array_equal(a1, a2) and e1 == e2 and np.array_equal(c1[1:], c2[1:])


@pytest.mark.parametrize("kw", [
    dict(length=31, walkers=4, max_restarts=3, target_merit=3.0, seed=31),
    dict(length=101, walkers=16, prefix_len=8, max_restarts=2, target_merit=5.0, seed=1),
    dict(length=201, walkers=4, prefix_len=12, max_restarts=1, target_merit=4.5, seed=1),
    dict(length=51, walkers=2, max_restarts=0, target_merit=3.0, candidate_quota=5, seed=5),
    dict(length=31, walkers=2, max_restarts=0, target_merit=3.0, stop_at_energy=200, seed=6),
    dict(length=25, walkers=3, max_restarts=5, target_merit=3.0, ti_multiplier=4.0,
         bloom_fpr=1e-3, seed=99),
])
def test_pool_matches_reference(restated, reference, kw):
    a = restated.run_saw_pool(make_config(**kw))
    b = reference.run_saw_pool(make_config(**kw), threads=1)
    assert len(a.candidates) == len(b.candidates)
    for x, y in zip(a.candidates, b.candidates):
        assert x.energy == y.energy and np.array_equal(x.seq, y.seq)
    for key in ("walks", "iterations", "emitted", "best_energy"):
        assert a.stats[key] == b.stats[key], key


def test_delta_eval_count_matches_reference_trace(restated, reference):
    # the reference's own run_walk through its VisitedSet seam counts skew_flip_delta_fast calls
    cfg = dict(length=101, walkers=8, prefix_len=8, max_restarts=2, target_merit=5.0, seed=1)
    a = restated.run_saw_pool(make_config(**cfg))
    t = reference.walk_trace(make_config(**cfg))
    assert a.stats["delta_evals"] == t.stats["delta_evals"]
    assert a.stats["iterations"] == t.stats["iterations"]


def test_thread_invariant_candidate_set(reference):
    # test_saw.cpp:260-282: 1-thread and 3-thread pools give the same candidate set
    cfg = make_config(length=51, walkers=6, max_restarts=2, target_merit=3.5, seed=17)
    one = reference.run_saw_pool(cfg, threads=1)
    three = reference.run_saw_pool(cfg, threads=3)
    assert {c.seq.tobytes() for c in one.candidates} == {c.seq.tobytes() for c in three.candidates}


def test_restated_reproduces_golden_fixtures(restated):
    with open(os.path.join(GOLDEN, "saw_pool.json")) as f:
        cases = json.load(f)
    assert len(cases) >= 5
    for case in cases:
        run = restated.run_saw_pool(make_config(**case["config"]))
        lines = [restated.format_record(c.seq, c.energy) for c in run.candidates]
        assert lines == case["records"], case["name"]
        for key, v in case["stats"].items():
            assert run.stats[key] == v, (case["name"], key)


def test_shard_union_is_whole_pool(restated):
    # class shards partition the pool; union in (w, r, it) order == whole
    base = dict(length=51, walkers=16, prefix_len=4, max_restarts=2, target_merit=3.5, seed=4,
                dedup=0)
    whole = restated.run_saw_pool(make_config(**base))
    parts = []
    for g in range(3):
        parts += restated.run_saw_pool(make_config(shard_index=g, shard_count=3, **base)).candidates
    parts.sort(key=lambda c: (c.walker, c.restart, c.iteration))
    assert [(c.walker, c.restart, c.iteration, c.energy) for c in parts] == \
        [(c.walker, c.restart, c.iteration, c.energy) for c in whole.candidates]


def test_enumeration_restatement(restated):
    # A14: Gray enumeration over all free bits of every class finds the global skew optimum
    # (cross-check against oracle_skew_exhaustive, oracle.cpp:37-67)
    for L, p in [(21, 3), (31, 4)]:
        kp1 = (L + 1) // 2
        best = min(restated.enumerate_class(L, p, c, kp1 - p, 1)[1]["best_energy"]
                   for c in range(1 << (p - 1)))
        assert best == restated.oracle_skew_exhaustive(L)[0]


def test_flip_delta_equals_scratch(restated):
    # test_sequence.cpp:83-98: flip_delta = scratch at L in {50, 101, 250}, seed 42
    rng = np.random.default_rng(42)
    for L in (50, 101, 250):
        s = _rand_signs(rng, L)
        e0 = _scratch_energy(s)
        for i in rng.integers(0, L, size=6):
            t = s.copy()
            t[i] = -t[i]
            assert restated.flip_delta(s, int(i)) == _scratch_energy(t) - e0
