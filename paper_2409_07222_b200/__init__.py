"""paper_2409_07222_b200 -- B200-native Step 1 of the dual-step LABS search (arXiv 2409.07222).

Python view of the C ABI in ``include/labs_gpu.h`` (libpaper_labs.so, built in-tree into
``paper_2409_07222_b200/_lib``).  The API mirrors the reference's Step-1 surface
(/root/reference/proj/include/labs/saw.hpp, candidate.hpp):

    cfg = SawConfig(length=451, walkers=1024, prefix_len=8, target_merit=5.3, max_restarts=64)
    sink = CollectingSink()
    stats = run_saw_pool(cfg, sink)        # PoolStats, candidates in --threads 1 order

There is no CPU fallback: importing works anywhere, every compute call raises when the
CUDA library or device is missing.
"""
from .api import (  # noqa: F401
    Candidate,
    CandidateSink,
    CollectingSink,
    DedupSink,
    LabsError,
    PoolStats,
    SawConfig,
    WalkResult,
    bench_plan,
    canonical_hash,
    derive,
    device_count,
    energy_threshold_for_merit,
    enumerate_class,
    expand_skew,
    format_record,
    hex_encode,
    imma_peak,
    int32_peak,
    library_path,
    load_library,
    merit_factor,
    pq_score,
    rank_prefixes,
    prepare_saw_pool,
    run_saw_pool,
    saw_walks,
    skew_flip_deltas,
)

__all__ = [
    "Candidate", "CandidateSink", "CollectingSink", "DedupSink", "LabsError", "PoolStats",
    "SawConfig", "WalkResult", "bench_plan", "canonical_hash", "rank_prefixes", "derive", "device_count",
    "energy_threshold_for_merit", "enumerate_class", "expand_skew", "format_record",
    "hex_encode", "imma_peak", "int32_peak", "library_path", "load_library", "merit_factor", "pq_score",
    "prepare_saw_pool", "run_saw_pool", "saw_walks", "skew_flip_deltas",
]
