"""ctypes access to the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  The product (paper_2409_07222_b200) never does.

Two libraries:
  * ``Restated`` -- oracle/build/liblabs_oracle.so, the plain-C restatement
    (oracle/labs_oracle.c) of the reference Step-1 path.
  * ``Reference`` -- oracle/_ref/liblabs_ref.so, the reference library compiled
    from its own sources under /root/reference/proj/src plus oracle/ref_shim.cpp.
    Built here (it travels to the GPU box as a prebuilt file); may be absent.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED_SO = os.path.join(HERE, "build", "liblabs_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "liblabs_ref.so")


class SawConfigC(C.Structure):
    _fields_ = [
        ("length", C.c_int32), ("prefix_len", C.c_int32), ("walkers", C.c_int32),
        ("_pad0", C.c_int32), ("max_iterations", C.c_int64), ("ti_multiplier", C.c_double),
        ("energy_threshold", C.c_int64), ("target_merit", C.c_double),
        ("bloom_fpr", C.c_double), ("seed", C.c_uint64), ("max_restarts", C.c_int64),
        ("time_budget_s", C.c_double), ("candidate_quota", C.c_int64),
        ("stop_at_energy", C.c_int64), ("walker_begin", C.c_int32),
        ("walker_end", C.c_int32), ("shard_index", C.c_int32), ("shard_count", C.c_int32),
        ("dedup", C.c_int32), ("_pad1", C.c_int32),
    ]


class PoolStatsC(C.Structure):
    _fields_ = [
        ("walks", C.c_int64), ("iterations", C.c_int64), ("emitted", C.c_int64),
        ("best_energy", C.c_int64), ("delta_evals", C.c_int64), ("bloom_hits", C.c_int64),
        ("exhausted_walks", C.c_int64), ("wall_seconds", C.c_double),
    ]


CAND_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_int8), C.c_int, C.c_int64, C.c_int64,
                      C.c_int64, C.c_int64)
WALK_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                      C.c_int64, C.c_int, C.c_int64)
ENUM_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_int64)


@dataclass
class OracleCandidate:
    seq: np.ndarray          # int8 signs, full length L
    energy: int
    walker: int
    restart: int
    iteration: int


@dataclass
class OracleWalk:
    walker: int
    restart: int
    iterations: int
    emitted: int
    best_energy: int
    delta_evals: int
    exhausted: bool


@dataclass
class OracleRun:
    candidates: list = field(default_factory=list)
    walks: list = field(default_factory=list)
    stats: dict = field(default_factory=dict)


def make_config(length, walkers=1, prefix_len=-1, max_iterations=0, ti_multiplier=8.0,
                energy_threshold=0, target_merit=0.0, bloom_fpr=1e-4, seed=1, max_restarts=1,
                time_budget_s=0.0, candidate_quota=0, stop_at_energy=0, walker_begin=0,
                walker_end=0, shard_index=0, shard_count=1, dedup=1) -> SawConfigC:
    return SawConfigC(length, prefix_len, walkers, 0, max_iterations, ti_multiplier,
                      energy_threshold, target_merit, bloom_fpr, seed, max_restarts,
                      time_budget_s, candidate_quota, stop_at_energy, walker_begin, walker_end,
                      shard_index, shard_count, dedup, 0)


def _stats(st: PoolStatsC) -> dict:
    return {k: getattr(st, k) for k, _ in PoolStatsC._fields_}


def _i8(a):
    a = np.ascontiguousarray(a, dtype=np.int8)
    return a, a.ctypes.data_as(C.POINTER(C.c_int8))


class _Base:
    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run __graft_entry__.build())")
        self.lib = C.CDLL(path)

    def _collect(self):
        run = OracleRun()

        def on_cand(user, seq, n, e, w, r, it):
            run.candidates.append(OracleCandidate(np.ctypeslib.as_array(seq, (n,)).copy(), e, w,
                                                  r, it))

        def on_walk(user, w, r, it, em, best, de, ex, e0):
            run.walks.append(OracleWalk(w, r, it, em, best, de, bool(ex)))

        return run, CAND_FN(on_cand), WALK_FN(on_walk)


class Restated(_Base):
    """The plain-C restatement (oracle/labs_oracle.c)."""

    def __init__(self, path: str = RESTATED_SO):
        super().__init__(path)
        L = self.lib
        L.lo_run_saw_pool.argtypes = [C.POINTER(SawConfigC), CAND_FN, WALK_FN, C.c_void_p,
                                      C.POINTER(PoolStatsC)]
        L.lo_last_error.restype = C.c_char_p
        for name in ("lo_skew_flip_delta_fast", "lo_flip_delta"):
            getattr(L, name).restype = C.c_int64
            getattr(L, name).argtypes = [C.POINTER(C.c_int8), C.c_int, C.POINTER(C.c_int64), C.c_int]
        L.lo_correlations.restype = C.c_int64
        L.lo_correlations.argtypes = [C.POINTER(C.c_int8), C.c_int, C.POINTER(C.c_int64)]
        L.lo_apply_skew_flip.restype = C.c_int64
        L.lo_apply_skew_flip.argtypes = [C.POINTER(C.c_int8), C.c_int, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int64), C.c_int]
        L.lo_expand_skew.argtypes = [C.POINTER(C.c_int8), C.c_int, C.POINTER(C.c_int8)]
        L.lo_energy_threshold.restype = C.c_int64
        L.lo_energy_threshold.argtypes = [C.c_int, C.c_double]
        L.lo_effective_iterations.restype = C.c_int64
        L.lo_effective_iterations.argtypes = [C.c_int, C.c_int64, C.c_double]
        L.lo_bloom_size.argtypes = [C.c_uint64, C.c_double, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
        L.lo_rank_prefixes.argtypes = [C.c_int, C.POINTER(C.c_int8)]
        L.lo_tab_hash.restype = C.c_uint64
        L.lo_tab_hash.argtypes = [C.POINTER(C.c_int8), C.c_int, C.c_int]
        L.lo_tab_flip_mask.restype = C.c_uint64
        L.lo_tab_flip_mask.argtypes = [C.c_int, C.c_int]
        L.lo_tab_salt.restype = C.c_uint64
        L.lo_tab_salt.argtypes = [C.c_int, C.c_int]
        L.lo_tab_entry.restype = C.c_uint64
        L.lo_tab_entry.argtypes = [C.c_int, C.c_int, C.c_int]
        L.lo_rng_init.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.lo_rng_next.restype = C.c_uint64
        L.lo_rng_next.argtypes = [C.c_void_p]
        L.lo_run_walk_from_half.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int8), C.c_int64,
                                            C.c_int64, C.c_uint64, C.c_int, CAND_FN, C.c_void_p,
                                            C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        L.lo_enumerate_class.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64,
                                         C.c_uint64, C.c_uint64, ENUM_FN, C.c_void_p,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64)]
        L.lo_oracle_skew_exhaustive.restype = C.c_int64
        L.lo_oracle_skew_exhaustive.argtypes = [C.c_int, C.POINTER(C.c_int8)]
        L.lo_format_record.argtypes = [C.POINTER(C.c_int8), C.c_int, C.c_int64, C.c_char_p, C.c_int]
        L.lo_bloom_insert.argtypes = [C.POINTER(C.c_uint64), C.c_uint64, C.c_int, C.c_uint64,
                                      C.c_uint64]
        L.lo_bloom_contains.argtypes = [C.POINTER(C.c_uint64), C.c_uint64, C.c_int, C.c_uint64,
                                        C.c_uint64]

    # -- pool
    def run_saw_pool(self, cfg: SawConfigC) -> OracleRun:
        run, cb, wb = self._collect()
        st = PoolStatsC()
        rc = self.lib.lo_run_saw_pool(C.byref(cfg), cb, wb, None, C.byref(st))
        if rc != 0:
            raise ValueError(self.lib.lo_last_error().decode())
        run.stats = _stats(st)
        return run

    def run_walk_from_half(self, length, prefix_len, half, t_i, e_l, bloom_bits, bloom_k):
        run, cb, _ = self._collect()
        h, hp = _i8(half)
        it, best, de = C.c_int64(), C.c_int64(), C.c_int64()
        ex = C.c_int()
        rc = self.lib.lo_run_walk_from_half(length, prefix_len, hp, t_i, e_l, bloom_bits, bloom_k,
                                            cb, None, C.byref(it), C.byref(best), C.byref(de),
                                            C.byref(ex))
        if rc != 0:
            raise ValueError(self.lib.lo_last_error().decode())
        return run.candidates, dict(iterations=it.value, best_energy=best.value,
                                    delta_evals=de.value, exhausted=bool(ex.value))

    def enumerate_class(self, length, p, class_index, m, e_l, g_begin=0, g_end=None):
        g_end = (1 << m) if g_end is None else g_end
        hits = []
        cb = ENUM_FN(lambda u, g, e: hits.append((g, e)))
        be, bg, ne = C.c_int64(), C.c_uint64(), C.c_uint64()
        rc = self.lib.lo_enumerate_class(length, p, class_index, m, e_l, g_begin, g_end, cb, None,
                                         C.byref(be), C.byref(bg), C.byref(ne))
        if rc != 0:
            raise ValueError(self.lib.lo_last_error().decode())
        return hits, dict(best_energy=be.value, best_g=bg.value, emitted=ne.value)

    # -- primitives
    def correlations(self, s):
        a, p = _i8(s)
        c = np.zeros(len(a), dtype=np.int64)
        e = self.lib.lo_correlations(p, len(a), c.ctypes.data_as(C.POINTER(C.c_int64)))
        return c, e

    def skew_flip_delta_fast(self, s, hp):
        a, p = _i8(s)
        c, _ = self.correlations(a)
        return self.lib.lo_skew_flip_delta_fast(p, len(a), c.ctypes.data_as(C.POINTER(C.c_int64)), hp)

    def flip_delta(self, s, i):
        a, p = _i8(s)
        c, _ = self.correlations(a)
        return self.lib.lo_flip_delta(p, len(a), c.ctypes.data_as(C.POINTER(C.c_int64)), i)

    def apply_skew_flip(self, s, hp):
        a, p = _i8(np.array(s, dtype=np.int8).copy())
        c, e = self.correlations(a)
        ee = C.c_int64(e)
        self.lib.lo_apply_skew_flip(p, len(a), c.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(ee), hp)
        return a, c, ee.value

    def expand_skew(self, half):
        h, hp = _i8(half)
        out = np.zeros(2 * len(h) - 1, dtype=np.int8)
        self.lib.lo_expand_skew(hp, len(h), out.ctypes.data_as(C.POINTER(C.c_int8)))
        return out

    def energy_threshold(self, length, f):
        return self.lib.lo_energy_threshold(length, f)

    def effective_iterations(self, length, max_it=0, mult=8.0):
        return self.lib.lo_effective_iterations(length, max_it, mult)

    def bloom_size(self, capacity, fpr):
        b, k = C.c_uint64(), C.c_int()
        self.lib.lo_bloom_size(capacity, fpr, C.byref(b), C.byref(k))
        return b.value, k.value

    def rank_prefixes(self, p):
        out = np.zeros((1 << (p - 1), p), dtype=np.int8)
        self.lib.lo_rank_prefixes(p, out.ctypes.data_as(C.POINTER(C.c_int8)))
        return out

    def canonical_hash(self, s, table=0):
        a, p = _i8(s)
        return self.lib.lo_tab_hash(p, len(a), table)

    def flip_mask(self, pos, table):
        return self.lib.lo_tab_flip_mask(table, pos)

    def tab_entry(self, table, pos, sign):
        return self.lib.lo_tab_entry(table, pos, sign)

    def salt(self, table, n):
        return self.lib.lo_tab_salt(table, n)

    def rng_draws(self, seed, stream, n):
        st = (C.c_uint64 * 4)()
        self.lib.lo_rng_init(st, seed, stream)
        return [self.lib.lo_rng_next(st) for _ in range(n)]

    def oracle_skew_exhaustive(self, length):
        out = np.zeros(length, dtype=np.int8)
        e = self.lib.lo_oracle_skew_exhaustive(length, out.ctypes.data_as(C.POINTER(C.c_int8)))
        return e, out

    def format_record(self, s, energy):
        a, p = _i8(s)
        buf = C.create_string_buffer(4096)
        self.lib.lo_format_record(p, len(a), energy, buf, 4096)
        return buf.value.decode()

    def bloom_words(self, capacity, fpr, keys):
        bits, k = self.bloom_size(capacity, fpr)
        w = np.zeros((bits + 63) // 64, dtype=np.uint64)
        wp = w.ctypes.data_as(C.POINTER(C.c_uint64))
        for h1, h2 in keys:
            self.lib.lo_bloom_insert(wp, bits, k, h1, h2)
        return w


class Reference(_Base):
    """The reference library compiled from its own sources (oracle/_ref)."""

    def __init__(self, path: str = REFERENCE_SO):
        super().__init__(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_run_saw_pool.argtypes = [C.POINTER(SawConfigC), C.c_int, CAND_FN, C.c_void_p,
                                       C.POINTER(PoolStatsC)]
        L.ref_count_deltas.argtypes = [C.POINTER(SawConfigC), C.c_int, C.POINTER(PoolStatsC)]
        L.ref_walk_trace_mt.argtypes = [C.POINTER(SawConfigC), C.c_int, CAND_FN, WALK_FN,
                                        C.c_void_p, C.POINTER(PoolStatsC)]
        L.ref_walk_trace.argtypes = [C.POINTER(SawConfigC), CAND_FN, WALK_FN, C.c_void_p,
                                     C.POINTER(PoolStatsC)]
        for name in ("ref_skew_flip_delta_fast", "ref_skew_flip_delta"):
            getattr(L, name).restype = C.c_int64
            getattr(L, name).argtypes = [C.POINTER(C.c_int8), C.c_int, C.c_int]
        L.ref_apply_skew_flip.restype = C.c_int64
        L.ref_apply_skew_flip.argtypes = [C.POINTER(C.c_int8), C.c_int, C.c_int, C.POINTER(C.c_int64)]
        L.ref_energy.restype = C.c_int64
        L.ref_energy.argtypes = [C.POINTER(C.c_int8), C.c_int]
        L.ref_expand_skew.argtypes = [C.POINTER(C.c_int8), C.c_int, C.POINTER(C.c_int8)]
        L.ref_energy_threshold.restype = C.c_int64
        L.ref_energy_threshold.argtypes = [C.c_int, C.c_double]
        L.ref_bloom_size.argtypes = [C.c_uint64, C.c_double, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
        L.ref_effective_iterations.restype = C.c_longlong
        L.ref_effective_iterations.argtypes = [C.c_int, C.c_longlong, C.c_double]
        L.ref_rank_prefixes.argtypes = [C.c_int, C.POINTER(C.c_int8)]
        L.ref_canonical_hash.restype = C.c_uint64
        L.ref_canonical_hash.argtypes = [C.POINTER(C.c_int8), C.c_int, C.c_int]
        L.ref_flip_mask.restype = C.c_uint64
        L.ref_flip_mask.argtypes = [C.c_int, C.c_int]
        L.ref_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]
        L.ref_oracle_skew_exhaustive.restype = C.c_int64
        L.ref_oracle_skew_exhaustive.argtypes = [C.c_int, C.POINTER(C.c_int8)]
        L.ref_format_record.argtypes = [C.POINTER(C.c_int8), C.c_int, C.c_int64, C.c_char_p, C.c_int]
        L.ref_bloom_words.argtypes = [C.c_uint64, C.c_double, C.POINTER(C.c_uint64), C.c_int,
                                      C.POINTER(C.c_uint64), C.c_int]

    def run_saw_pool(self, cfg: SawConfigC, threads: int = 1) -> OracleRun:
        run, cb, _ = self._collect()
        st = PoolStatsC()
        rc = self.lib.ref_run_saw_pool(C.byref(cfg), threads, cb, None, C.byref(st))
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        run.stats = _stats(st)
        return run

    def walk_trace(self, cfg: SawConfigC) -> OracleRun:
        run, cb, wb = self._collect()
        st = PoolStatsC()
        rc = self.lib.ref_walk_trace(C.byref(cfg), cb, wb, None, C.byref(st))
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        run.stats = _stats(st)
        return run

    def walk_trace_mt(self, cfg: SawConfigC, threads: int = 1) -> OracleRun:
        """The reference run_walk over every (walker, restart), walkers on `threads` threads,
        replayed in --threads 1 order through the reference DedupSink (ref_shim.cpp)."""
        run, cb, wb = self._collect()
        st = PoolStatsC()
        rc = self.lib.ref_walk_trace_mt(C.byref(cfg), threads, cb, wb, None, C.byref(st))
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        run.stats = _stats(st)
        return run

    def count_deltas(self, cfg: SawConfigC, threads: int = 1) -> dict:
        """skew_flip_delta_fast calls + iterations of the pool's walks (threaded, no sink)."""
        st = PoolStatsC()
        if self.lib.ref_count_deltas(C.byref(cfg), threads, C.byref(st)) != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return _stats(st)

    def skew_flip_delta_fast(self, s, hp):
        a, p = _i8(s)
        return self.lib.ref_skew_flip_delta_fast(p, len(a), hp)

    def skew_flip_delta(self, s, hp):
        a, p = _i8(s)
        return self.lib.ref_skew_flip_delta(p, len(a), hp)

    def apply_skew_flip(self, s, hp):
        a, p = _i8(np.array(s, dtype=np.int8).copy())
        c = np.zeros(len(a), dtype=np.int64)
        e = self.lib.ref_apply_skew_flip(p, len(a), hp, c.ctypes.data_as(C.POINTER(C.c_int64)))
        return a, c, e

    def energy(self, s):
        a, p = _i8(s)
        return self.lib.ref_energy(p, len(a))

    def expand_skew(self, half):
        h, hp = _i8(half)
        out = np.zeros(2 * len(h) - 1, dtype=np.int8)
        self.lib.ref_expand_skew(hp, len(h), out.ctypes.data_as(C.POINTER(C.c_int8)))
        return out

    def energy_threshold(self, length, f):
        return self.lib.ref_energy_threshold(length, f)

    def effective_iterations(self, length, max_it=0, mult=8.0):
        return self.lib.ref_effective_iterations(length, max_it, mult)

    def bloom_size(self, capacity, fpr):
        b, k = C.c_uint64(), C.c_int()
        self.lib.ref_bloom_size(capacity, fpr, C.byref(b), C.byref(k))
        return b.value, k.value

    def rank_prefixes(self, p):
        out = np.zeros((1 << (p - 1), p), dtype=np.int8)
        self.lib.ref_rank_prefixes(p, out.ctypes.data_as(C.POINTER(C.c_int8)))
        return out

    def canonical_hash(self, s, table=0):
        a, p = _i8(s)
        return self.lib.ref_canonical_hash(p, len(a), table)

    def flip_mask(self, pos, table):
        return self.lib.ref_flip_mask(pos, table)

    def rng_draws(self, seed, stream, n):
        out = (C.c_uint64 * n)()
        self.lib.ref_rng_draws(seed, stream, n, out)
        return list(out)

    def oracle_skew_exhaustive(self, length):
        out = np.zeros(length, dtype=np.int8)
        e = self.lib.ref_oracle_skew_exhaustive(length, out.ctypes.data_as(C.POINTER(C.c_int8)))
        return e, out

    def format_record(self, s, energy):
        a, p = _i8(s)
        buf = C.create_string_buffer(4096)
        self.lib.ref_format_record(p, len(a), energy, buf, 4096)
        return buf.value.decode()

    def bloom_words(self, capacity, fpr, keys):
        k = np.ascontiguousarray(np.array(keys, dtype=np.uint64).reshape(-1))
        nw = self.lib.ref_bloom_words(capacity, fpr, k.ctypes.data_as(C.POINTER(C.c_uint64)),
                                      len(keys), None, 0)
        w = np.zeros(nw, dtype=np.uint64)
        self.lib.ref_bloom_words(capacity, fpr, k.ctypes.data_as(C.POINTER(C.c_uint64)), len(keys),
                                 w.ctypes.data_as(C.POINTER(C.c_uint64)), nw)
        return w


def reference_available() -> bool:
    return os.path.exists(REFERENCE_SO)
