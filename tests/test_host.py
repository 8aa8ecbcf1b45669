"""Host side of the C ABI without a GPU: the library loads, exports every entry point
include/labs_gpu.h declares, the host helpers equal the oracle (hashes, formats, prefix
ranking, config derivation, validation messages), and compute calls fail loudly instead
of falling back to the CPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "labs_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(labs_[a-z0-9_]+)\s*\(", src)
    return sorted(set(n for n in names if not n.endswith("_fn")))


def test_library_exports_every_declared_symbol(labs):
    lib = ctypes.CDLL(labs.library_path())
    syms = _declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_cli_binary_built():
    assert os.access(os.path.join(ROOT, "paper_2409_07222_b200", "_lib", "labs"), os.X_OK)


def test_no_cpu_fallback(labs):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(labs.api.NoDevice):
        labs.run_saw_pool(labs.SawConfig(length=31, target_merit=3.0, max_restarts=1))
    with pytest.raises(labs.api.NoDevice):
        labs.skew_flip_deltas(31, np.ones((1, 16), np.int8))
    with pytest.raises(labs.api.NoDevice):
        labs.prepare_saw_pool(labs.SawConfig(length=31, target_merit=3.0, max_restarts=1))


def test_host_helpers_match_oracle(labs, restated):
    rng = np.random.default_rng(5)
    for L in (5, 101, 451, 527, 1023):
        s = rng.choice(np.array([-1, 1], np.int8), size=L)
        assert labs.canonical_hash(s) == restated.canonical_hash(s, 0)
        assert labs.format_record(s, 1234) == restated.format_record(s, 1234)
        half = s[: (L + 1) // 2]
        assert np.array_equal(labs.expand_skew(half), restated.expand_skew(half))
    for p in (1, 2, 8, 12):
        assert np.array_equal(labs.rank_prefixes(p), restated.rank_prefixes(p))
    assert labs.hex_encode(np.array([1, 1, 1, -1, 1], np.int8)) == "1D"


@pytest.mark.parametrize("L,F,p", [(101, 5.0, 8), (201, 5.0, 12), (301, 5.2, 8), (451, 5.3, 8),
                                   (527, 5.3, 8)])
def test_derive_matches_oracle(labs, restated, L, F, p):
    d = labs.derive(labs.SawConfig(length=L, walkers=1024, prefix_len=p, target_merit=F,
                                   max_restarts=1))
    t_i = restated.effective_iterations(L)
    bits, k = restated.bloom_size(t_i + 1, 1e-4)
    assert d["iterations"] == t_i
    assert d["energy_threshold"] == restated.energy_threshold(L, F)
    assert (d["bloom_bits"], d["bloom_hashes"]) == (bits, k)
    assert d["free_bits"] == (L + 1) // 2 - p
    assert d["prefix_len"] == p


def test_default_prefix_len(labs):
    # saw.cpp:44-49: smallest p with 2^(p-1) >= walkers
    for w, p in [(1, 1), (2, 2), (3, 3), (128, 8), (129, 9)]:
        assert labs.derive(labs.SawConfig(length=101, walkers=w, target_merit=4.0))["prefix_len"] == p


def test_validation_messages(labs):
    # SawConfig::validate (saw.cpp:51-63) -> std::invalid_argument -> ValueError
    bad = [
        (dict(length=30, target_merit=3.0), "odd"),
        (dict(length=1, target_merit=3.0), "odd"),
        (dict(length=31), "E_l"),
        (dict(length=31, target_merit=3.0, max_restarts=0), "no stop condition"),
        (dict(length=31, target_merit=3.0, prefix_len=17), "prefix length"),
        (dict(length=31, target_merit=3.0, bloom_fpr=1.5), "fpr"),
        (dict(length=31, target_merit=3.0, walkers=0), "walkers"),
        (dict(length=1025, target_merit=3.0), "tabulation"),
    ]
    for kw, msg in bad:
        with pytest.raises(ValueError, match=msg):
            labs.derive(labs.SawConfig(**kw))
