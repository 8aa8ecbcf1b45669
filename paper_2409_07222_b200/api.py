"""ctypes binding of libpaper_labs.so (include/labs_gpu.h) with a reference-shaped API.

Names, fields and error behaviour follow the reference's Step-1 interface:
  SawConfig        saw.hpp:34-61          (validate -> ValueError = std::invalid_argument)
  run_saw_pool     saw.hpp:172, saw.cpp:218-267
  PoolStats        saw.hpp:161-167
  Candidate        candidate.hpp:21-29
  CandidateSink / CollectingSink / DedupSink   candidate.hpp:56-99
  format_record    candidate.cpp:36-49;  hex_encode hex_codec.cpp:14-30
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LABS_B200_LIB: development override (kernel-variant A/B timing); default is the in-tree build
_LIB_PATH = os.environ.get("LABS_B200_LIB") or os.path.join(_HERE, "_lib", "libpaper_labs.so")

LABS_OK, LABS_EINVAL, LABS_ERANGE, LABS_ENODEV, LABS_ECUDA, LABS_ELOGIC, LABS_EABORT = (
    0, -1, -2, -3, -4, -5, -6)


class LabsError(RuntimeError):
    """A CUDA / device failure of the Step-1 engine."""


class InvalidArgument(ValueError, LabsError):
    """std::invalid_argument in the reference."""


class LogicError(LabsError):
    """std::logic_error in the reference (energy bookkeeping diverged)."""


class NoDevice(LabsError):
    """No CUDA device: the engine has no CPU fallback."""


# ----------------------------------------------------------------------------- structs
class _Config(C.Structure):
    _fields_ = [
        ("length", C.c_int32), ("prefix_len", C.c_int32), ("walkers", C.c_int32),
        ("threads", C.c_int32), ("max_iterations", C.c_int64), ("ti_multiplier", C.c_double),
        ("energy_threshold", C.c_int64), ("target_merit", C.c_double), ("bloom_fpr", C.c_double),
        ("seed", C.c_uint64), ("max_restarts", C.c_int64), ("time_budget_s", C.c_double),
        ("candidate_quota", C.c_int64), ("stop_at_energy", C.c_int64),
        ("debug_check_energy", C.c_int32), ("n_gpus", C.c_int32), ("device", C.c_int32),
        ("shard_index", C.c_int32), ("shard_count", C.c_int32), ("count_visited", C.c_int32),
        ("walker_begin", C.c_int32), ("walker_end", C.c_int32), ("reserved", C.c_int32 * 6),
    ]


class _Candidate(C.Structure):
    _fields_ = [
        ("length", C.c_int32), ("origin", C.c_int32), ("energy", C.c_int64),
        ("signs", C.POINTER(C.c_int8)), ("prefix", C.POINTER(C.c_int8)),
        ("prefix_len", C.c_int32), ("_pad", C.c_int32), ("walker", C.c_int64),
        ("restart", C.c_int64), ("iteration", C.c_int64),
    ]


class _PoolStats(C.Structure):
    _fields_ = [
        ("walks", C.c_int64), ("iterations", C.c_int64), ("emitted", C.c_int64),
        ("best_energy", C.c_int64), ("wall_seconds", C.c_double), ("emitted_raw", C.c_int64),
        ("delta_evals", C.c_int64), ("delta_evals_computed", C.c_int64),
        ("exhausted_walks", C.c_int64), ("wide_iterations", C.c_int64),
        ("kernel_ms", C.c_double), ("seed_ms", C.c_double), ("n_gpus", C.c_int32),
        ("_pad", C.c_int32), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
    ]


class _Derived(C.Structure):
    _fields_ = [
        ("prefix_len", C.c_int32), ("bloom_hashes", C.c_int32), ("iterations", C.c_int64),
        ("energy_threshold", C.c_int64), ("bloom_bits", C.c_uint64), ("free_bits", C.c_int32),
        ("neighbours_per_lane", C.c_int32),
        ("kernel", C.c_int32),
        ("lanes_per_walk", C.c_int32),
    ]


class _WalkResult(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "iterations", "emitted", "best_energy", "initial_energy", "exhausted", "delta_evals",
        "probe_rounds", "wide_iterations", "diverged")]


class _EnumStats(C.Structure):
    _fields_ = [
        ("best_energy", C.c_int64), ("best_g", C.c_uint64), ("configurations", C.c_uint64),
        ("emitted", C.c_uint64), ("kernel_ms", C.c_double),
    ]


class _CandidateBatch(C.Structure):
    _fields_ = [
        ("count", C.c_int32), ("length", C.c_int32), ("prefix_len", C.c_int32),
        ("origin", C.c_int32), ("signs", C.POINTER(C.c_int8)), ("energy", C.POINTER(C.c_int64)),
        ("walker", C.POINTER(C.c_int64)), ("restart", C.POINTER(C.c_int64)),
        ("iteration", C.POINTER(C.c_int64)), ("prefix_class", C.POINTER(C.c_int32)),
        ("prefixes", C.POINTER(C.c_int8)),
    ]


_CAND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(_Candidate))
_BATCH_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(_CandidateBatch))
_REC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_int8),
                      C.c_int32)
_ENUM_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_int64)

_lib = None
_lib_lock = threading.Lock()


def library_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libpaper_labs.so (fails loudly when it was not built)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise LabsError(f"CUDA extension not built: {_LIB_PATH} missing "
                            "(run __graft_entry__.build())")
        lib = C.CDLL(_LIB_PATH)
        lib.labs_last_error.restype = C.c_char_p
        lib.labs_version.restype = C.c_char_p
        lib.labs_saw_pool_run.argtypes = [C.POINTER(_Config), _CAND_FN, C.c_void_p,
                                          C.POINTER(_PoolStats)]
        lib.labs_saw_pool_run_batched.argtypes = [C.POINTER(_Config), _BATCH_FN, C.c_void_p,
                                                  C.POINTER(_PoolStats)]
        lib.labs_saw_derive.argtypes = [C.POINTER(_Config), C.POINTER(_Derived)]
        lib.labs_saw_prepare.argtypes = [C.POINTER(_Config)]
        lib.labs_saw_walks.argtypes = [C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_double,
                                       C.POINTER(C.c_int8), C.c_int64, C.c_int32, C.c_int32,
                                       C.POINTER(_WalkResult), _REC_FN, C.c_void_p]
        lib.labs_skew_flip_deltas.argtypes = [C.c_int32, C.POINTER(C.c_int8), C.c_int64,
                                              C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                              C.POINTER(C.c_int64)]
        lib.labs_enumerate_class.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                             C.c_int64, C.c_uint64, C.c_uint64, _ENUM_FN,
                                             C.c_void_p, C.POINTER(_EnumStats)]
        lib.labs_bench_create.argtypes = [C.POINTER(_Config), C.POINTER(C.c_void_p)]
        lib.labs_bench_run.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_double),
                                       C.POINTER(_PoolStats)]
        lib.labs_bench_destroy.argtypes = [C.c_void_p]
        lib.labs_pq_score.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int8),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_int64)]
        lib.labs_int32_peak.argtypes = [C.POINTER(C.c_double)] * 4 + [C.POINTER(C.c_int32)] * 2
        lib.labs_device_count.argtypes = [C.POINTER(C.c_int32)]
        lib.labs_imma_peak.argtypes = [C.POINTER(C.c_double)]
        lib.labs_canonical_hash.restype = C.c_uint64
        lib.labs_canonical_hash.argtypes = [C.POINTER(C.c_int8), C.c_int32, C.c_int32]
        lib.labs_format_record.argtypes = [C.POINTER(C.c_int8), C.c_int32, C.c_int64, C.c_char_p,
                                           C.c_int32]
        lib.labs_rank_prefixes.argtypes = [C.c_int32, C.POINTER(C.c_int8)]
        lib.labs_expand_skew.argtypes = [C.POINTER(C.c_int8), C.c_int32, C.POINTER(C.c_int8)]
        _lib = lib
        return lib


def _check(rc: int):
    if rc == LABS_OK:
        return
    msg = load_library().labs_last_error().decode()
    if rc in (LABS_EINVAL, LABS_ERANGE):
        raise InvalidArgument(msg)
    if rc == LABS_ENODEV:
        raise NoDevice(msg)
    if rc == LABS_ELOGIC:
        raise LogicError(msg)
    raise LabsError(f"{msg} (status {rc})")


def _i8(a):
    a = np.ascontiguousarray(a, dtype=np.int8)
    return a, a.ctypes.data_as(C.POINTER(C.c_int8))


# ----------------------------------------------------------------------------- types
@dataclass
class SawConfig:
    """saw.hpp:34-61 plus additive GPU controls."""
    length: int = 0
    prefix_len: int = -1
    walkers: int = 1
    max_iterations: int = 0
    ti_multiplier: float = 8.0
    energy_threshold: int = 0
    target_merit: float = 0.0
    bloom_fpr: float = 1e-4
    seed: int = 1
    threads: int = 1
    max_restarts: int = 1
    time_budget_s: float = 0.0
    candidate_quota: int = 0
    stop_at_energy: int = 0
    debug_check_energy: bool = False
    # GPU
    n_gpus: int = 1
    device: int = 0
    shard_index: int = 0
    shard_count: int = 1
    count_visited: bool = False
    walker_begin: int = 0
    walker_end: int = 0

    def _c(self) -> _Config:
        c = _Config()
        for name, _ in _Config._fields_:
            if name == "reserved":
                continue
            setattr(c, name, int(getattr(self, name)) if name not in (
                "ti_multiplier", "target_merit", "bloom_fpr", "time_budget_s")
                else float(getattr(self, name)))
        return c

    def derived(self) -> dict:
        return derive(self)

    def effective_iterations(self) -> int:
        return self.max_iterations if self.max_iterations > 0 else int(
            self.ti_multiplier * (self.length + 1) / 2)

    def effective_threshold(self) -> int:
        if self.target_merit > 0:
            return energy_threshold_for_merit(self.length, self.target_merit)
        return self.energy_threshold

    def effective_prefix_len(self) -> int:
        if self.prefix_len >= 0:
            return self.prefix_len
        p = 1
        while (1 << (p - 1)) < self.walkers:
            p += 1
        return p

    def validate(self):
        derive(self)


@dataclass
class Candidate:
    seq: np.ndarray             # int8 +1/-1, full length
    energy: int
    origin: str = "saw"
    prefix: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int8))
    walker: int = -1
    restart: int = -1
    iteration: int = -1

    def merit(self) -> float:
        return merit_factor(len(self.seq), self.energy)

    def hash(self) -> int:
        return canonical_hash(self.seq, 0)


class CandidateSink:
    def emit(self, c: Candidate) -> None:  # pragma: no cover - interface
        raise NotImplementedError


class CollectingSink(CandidateSink):
    """candidate.hpp:62-80.  Batches from the engine are kept as arrays and turned into
    Candidate objects only when taken."""

    def __init__(self):
        self.items: List[Candidate] = []
        self._batches: list = []
        self._mu = threading.Lock()

    def emit(self, c: Candidate) -> None:
        with self._mu:
            self._materialise()
            self.items.append(c)

    def emit_batch(self, signs, energy, walker, restart, iteration, prefixes) -> None:
        with self._mu:
            self._batches.append((signs, energy, walker, restart, iteration, prefixes))

    def _materialise(self):
        for signs, energy, walker, restart, iteration, prefixes in self._batches:
            e, w, r, it = energy.tolist(), walker.tolist(), restart.tolist(), iteration.tolist()
            self.items.extend(Candidate(signs[i], e[i], "saw", prefixes[i], w[i], r[i], it[i])
                              for i in range(len(e)))
        self._batches = []

    def arrays(self):
        """All collected candidates as (signs [n, L], energy [n]) without building objects."""
        with self._mu:
            self._materialise()
            if not self.items:
                return np.zeros((0, 0), dtype=np.int8), np.zeros(0, dtype=np.int64)
            return (np.stack([c.seq for c in self.items]),
                    np.array([c.energy for c in self.items], dtype=np.int64))

    def take(self) -> List[Candidate]:
        with self._mu:
            self._materialise()
            out, self.items = self.items, []
        return out

    def size(self) -> int:
        with self._mu:
            return len(self.items) + sum(len(b[1]) for b in self._batches)


class DedupSink(CandidateSink):
    """candidate.hpp:84-99: drops repeats by canonical_hash(0)."""

    def __init__(self, inner: CandidateSink):
        self.inner = inner
        self.seen = set()

    def emit(self, c: Candidate) -> None:
        h = c.hash()
        if h in self.seen:
            return
        self.seen.add(h)
        self.inner.emit(c)


@dataclass
class PoolStats:
    walks: int = 0
    iterations: int = 0
    emitted: int = 0
    best_energy: int = 0
    wall_seconds: float = 0.0
    emitted_raw: int = 0
    delta_evals: int = -1
    delta_evals_computed: int = 0
    exhausted_walks: int = 0
    wide_iterations: int = 0
    kernel_ms: float = 0.0
    seed_ms: float = 0.0
    n_gpus: int = 1
    h2d_bytes: int = 0
    d2h_bytes: int = 0

    @classmethod
    def _from(cls, s: _PoolStats) -> "PoolStats":
        return cls(**{n: getattr(s, n) for n, _ in _PoolStats._fields_ if n != "_pad"})


@dataclass
class WalkResult:
    iterations: int
    emitted: int
    best_energy: int
    initial_energy: int
    exhausted: bool
    delta_evals: int
    probe_rounds: int
    wide_iterations: int
    diverged: int


# ----------------------------------------------------------------------------- functions
def derive(cfg: SawConfig) -> dict:
    """Host-only derivation + validation (SawConfig::validate, saw.cpp:51-63)."""
    lib = load_library()
    d = _Derived()
    _check(lib.labs_saw_derive(C.byref(cfg._c()), C.byref(d)))
    return {n: getattr(d, n) for n, _ in _Derived._fields_}


def prepare_saw_pool(cfg: SawConfig) -> None:
    """Set up the device state run_saw_pool(cfg) would create on its first call (CUDA
    context, kernel modules, tables, rings) so that a later time budget is spent searching
    (labs_saw_prepare)."""
    _check(load_library().labs_saw_prepare(C.byref(cfg._c())))


def run_saw_pool(cfg: SawConfig, sink: Optional[CandidateSink] = None) -> PoolStats:
    """run_saw_pool (saw.cpp:218-267) on the GPU; candidates in --threads 1 order.

    Candidates cross the C ABI in batches (labs_saw_pool_run_batched); sinks with an
    `emit_batch(signs, energy, walker, restart, iteration, prefixes)` method receive the
    numpy arrays directly, others get one `emit(Candidate)` per candidate."""
    lib = load_library()
    err: list = []

    def on_batch(user, bp):
        try:
            b = bp.contents
            n, L, p = b.count, b.length, b.prefix_len
            signs = np.ctypeslib.as_array(b.signs, (n, L)).copy()
            energy = np.ctypeslib.as_array(b.energy, (n,)).copy()
            walker = np.ctypeslib.as_array(b.walker, (n,)).copy()
            restart = np.ctypeslib.as_array(b.restart, (n,)).copy()
            iteration = np.ctypeslib.as_array(b.iteration, (n,)).copy()
            cls = np.ctypeslib.as_array(b.prefix_class, (n,))
            if p > 0:
                table = np.ctypeslib.as_array(b.prefixes, (int(cls.max()) + 1, p))
                prefixes = table[cls].copy()
            else:
                prefixes = np.zeros((n, 0), dtype=np.int8)
            if sink is None:
                return 0
            if hasattr(sink, "emit_batch"):
                sink.emit_batch(signs, energy, walker, restart, iteration, prefixes)
            else:
                for i in range(n):
                    sink.emit(Candidate(signs[i], int(energy[i]), "saw", prefixes[i],
                                        int(walker[i]), int(restart[i]), int(iteration[i])))
            return 0
        except BaseException as e:  # propagate after the C call returns
            err.append(e)
            return 1

    st = _PoolStats()
    cb = _BATCH_FN(on_batch)
    rc = lib.labs_saw_pool_run_batched(C.byref(cfg._c()), cb, None, C.byref(st))
    if err:
        raise err[0]
    _check(rc)
    return PoolStats._from(st)


def saw_walks(length: int, prefix_len: int, iterations: int, energy_threshold: int,
              halves, bloom_fpr: float = 1e-4, count_visited: bool = False,
              debug_check: bool = False):
    """Walks from explicit initial halves (run_walk per half, saw.cpp:117-149).

    Returns (results: list[WalkResult], records: list[(walk, iteration, energy, half)])."""
    lib = load_library()
    h = np.ascontiguousarray(np.asarray(halves, dtype=np.int8))
    n = h.shape[0]
    res = (_WalkResult * max(n, 1))()
    recs = []

    def on_rec(user, w, it, e, half, kp1):
        recs.append((int(w), int(it), int(e), np.ctypeslib.as_array(half, (kp1,)).copy()))
        return 0

    cb = _REC_FN(on_rec)
    _check(lib.labs_saw_walks(length, prefix_len, iterations, energy_threshold, bloom_fpr,
                              h.ctypes.data_as(C.POINTER(C.c_int8)), n, int(count_visited),
                              int(debug_check), res, cb, None))
    out = [WalkResult(r.iterations, r.emitted, r.best_energy, r.initial_energy,
                      bool(r.exhausted), r.delta_evals, r.probe_rounds, r.wide_iterations,
                      r.diverged) for r in res[:n]]
    return out, recs


def skew_flip_deltas(length: int, halves):
    """skew_flip_delta_fast (skew.cpp:60-93) for every hp of each half, on the GPU.

    Returns (deltas [n, k+1], corr [n, k] = C_{2t}, energies [n])."""
    lib = load_library()
    h = np.ascontiguousarray(np.asarray(halves, dtype=np.int8))
    n, kp1 = h.shape
    deltas = np.zeros((n, kp1), dtype=np.int64)
    corr = np.zeros((n, max(kp1 - 1, 1)), dtype=np.int64)
    en = np.zeros(n, dtype=np.int64)
    P64 = C.POINTER(C.c_int64)
    _check(lib.labs_skew_flip_deltas(length, h.ctypes.data_as(C.POINTER(C.c_int8)), n,
                                     deltas.ctypes.data_as(P64), corr.ctypes.data_as(P64),
                                     en.ctypes.data_as(P64)))
    return deltas, corr[:, :kp1 - 1], en


def enumerate_class(length: int, prefix_len: int, class_index: int, m: int,
                    energy_threshold: int, g_begin: int = 0, g_end: Optional[int] = None,
                    collect: bool = True):
    """Gray enumeration of one restriction class (extension, oracle.cpp:37-67 pattern)."""
    lib = load_library()
    g_end = (1 << m) if g_end is None else g_end
    hits = []

    def on_hit(user, g, e):
        if collect:
            hits.append((int(g), int(e)))
        return 0

    cb = _ENUM_FN(on_hit)
    st = _EnumStats()
    _check(lib.labs_enumerate_class(length, prefix_len, class_index, m, energy_threshold,
                                    g_begin, g_end, cb, None, C.byref(st)))
    return hits, {n: getattr(st, n) for n, _ in _EnumStats._fields_}


def pq_score(pivot, t_r: int):
    """K5: Step-2 neighbourhood scores of one refine pivot (pq.cpp:114-176) on the GPU.

    Returns (pivot_energy, deltas [L], rot_energy [L, 2, t_r], rot_hash [L, 2, t_r]) where
    deltas[i] = flip_delta(pivot, i) and rot_*[i, dir, r-1] describe neighbour i rotated
    r steps left (dir 0) / right (dir 1)."""
    lib = load_library()
    a, p = _i8(pivot)
    n = len(a)
    d = np.zeros(n, dtype=np.int32)
    re = np.zeros((n, 2, max(t_r, 1)), dtype=np.int32)
    rh = np.zeros((n, 2, max(t_r, 1)), dtype=np.uint64)
    e = C.c_int64()
    _check(lib.labs_pq_score(n, t_r, p, d.ctypes.data_as(C.POINTER(C.c_int32)),
                             re.ctypes.data_as(C.POINTER(C.c_int32)),
                             rh.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(e)))
    return e.value, d, re[:, :, :t_r], rh[:, :, :t_r]


class bench_plan:
    """Device-resident plan for bench.py: the pool's walks with inputs in HBM."""

    def __init__(self, cfg: SawConfig):
        self.lib = load_library()
        self.h = C.c_void_p()
        _check(self.lib.labs_bench_create(C.byref(cfg._c()), C.byref(self.h)))

    def run(self, reps: int = 1):
        ms = C.c_double()
        st = _PoolStats()
        _check(self.lib.labs_bench_run(self.h, reps, C.byref(ms), C.byref(st)))
        return ms.value, PoolStats._from(st)

    def close(self):
        if self.h:
            self.lib.labs_bench_destroy(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def int32_peak() -> dict:
    lib = load_library()
    v = [C.c_double() for _ in range(4)]
    sm, clk = C.c_int32(), C.c_int32()
    _check(lib.labs_int32_peak(*[C.byref(x) for x in v], C.byref(sm), C.byref(clk)))
    return dict(imad=v[0].value, ialu=v[1].value, mixed=v[2].value, dp4a=v[3].value,
                sm_count=sm.value, clock_khz=clk.value)


def imma_peak() -> float:
    """int8 tensor-core MACs/s (mma.sync m16n8k32.s8 over every SM)."""
    lib = load_library()
    v = C.c_double()
    _check(lib.labs_imma_peak(C.byref(v)))
    return v.value


def device_count() -> int:
    lib = load_library()
    n = C.c_int32()
    lib.labs_device_count(C.byref(n))
    return n.value


def canonical_hash(seq, table: int = 0) -> int:
    a, p = _i8(seq)
    return load_library().labs_canonical_hash(p, len(a), table)


def format_record(c_or_seq, energy: Optional[int] = None) -> str:
    """candidate.cpp:36-49: 'L\\tE\\t%.4f\\tHEX\\tsaw'."""
    if isinstance(c_or_seq, Candidate):
        seq, energy = c_or_seq.seq, c_or_seq.energy
    else:
        seq = c_or_seq
    a, p = _i8(seq)
    buf = C.create_string_buffer(len(a) + 128)
    load_library().labs_format_record(p, len(a), int(energy), buf, len(buf))
    return buf.value.decode()


def hex_encode(seq) -> str:
    """hex_codec.cpp:14-30 (MSB first, +1 -> 1, left zero-padded to whole nibbles)."""
    return format_record(seq, 1).split("\t")[3]


def rank_prefixes(p: int) -> np.ndarray:
    out = np.zeros(((1 << (p - 1)) if 1 <= p <= 30 else 1, max(p, 1)), dtype=np.int8)
    rc = load_library().labs_rank_prefixes(p, out.ctypes.data_as(C.POINTER(C.c_int8)))
    _check(min(rc, 0))
    return out


def expand_skew(half) -> np.ndarray:
    a, p = _i8(half)
    out = np.zeros(2 * len(a) - 1, dtype=np.int8)
    _check(load_library().labs_expand_skew(p, len(a), out.ctypes.data_as(C.POINTER(C.c_int8))))
    return out


def energy_threshold_for_merit(length: int, target_merit: float) -> int:
    """sequence.cpp:36-40: floor(L^2 / (2F)) in double."""
    if target_merit <= 0:
        raise InvalidArgument("target merit must be positive")
    return int(np.floor(float(length) * length / (2.0 * target_merit)))


def merit_factor(length: int, energy: int) -> float:
    if energy < 0:
        raise InvalidArgument("merit_factor: negative energy")
    if energy == 0:
        raise ZeroDivisionError("merit factor is infinite (E = 0)")
    return float(length) * float(length) / (2.0 * float(energy))
