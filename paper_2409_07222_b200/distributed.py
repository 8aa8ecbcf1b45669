"""Multi-GPU Step 1: one process per GPU, restriction-class shards, host merge.

SURVEY.md §8(e): with no quota / time budget / stop_at_energy every (walker, restart) walk
depends only on (seed, walker, restart, prefixes[walker mod P]) (saw.cpp:196-214,65-75),
so the pool shards by restriction class with no data-path collective.  Rank g runs the
walkers whose class c = w mod P satisfies c mod world == g (`shard_index`/`shard_count`
of the C ABI).  The only communication is the gather of the (small) sieve output to rank
0, which restores the reference's --threads 1 order and DedupSink semantics
(candidate.hpp:84-99):

    concatenate -> sort by (walker, restart, iteration) -> keep the first occurrence of
    each canonical_hash(0)

Each shard was already deduplicated in its own (walker, restart, iteration) order, and a
hash's global first occurrence is also the first inside its shard, so this merge equals
the single-process pool exactly (tests/test_distributed.py checks it with gloo).
"""
from __future__ import annotations

from typing import Callable, Iterable, List, Optional, Sequence, Tuple

import numpy as np

from .api import Candidate, CandidateSink, PoolStats, SawConfig, canonical_hash, run_saw_pool

# stats merged by sum / by min (PoolStats fields, saw.hpp:161-167 + GPU counters)
_SUM_KEYS = ("walks", "iterations", "emitted_raw", "delta_evals_computed", "exhausted_walks",
             "wide_iterations")
_MAX_KEYS = ("kernel_ms", "seed_ms", "wall_seconds")


def shard_config(cfg: SawConfig, rank: int, world: int) -> SawConfig:
    """The SawConfig rank `rank` of `world` runs (class shard c mod world == rank)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad shard {rank}/{world}")
    if world > 1 and (cfg.candidate_quota > 0 or cfg.stop_at_energy > 0 or
                      cfg.time_budget_s > 0 or cfg.max_restarts == 0):
        # saw.cpp:162-188,204-208: these couple walkers; not shardable deterministically
        raise ValueError("quota / stop_at_energy / time budget / unlimited restarts couple the "
                         "walkers and cannot be sharded across processes")
    kw = dict(cfg.__dict__)
    kw.update(shard_index=rank, shard_count=world, n_gpus=1)
    return SawConfig(**kw)


def _key(seq: np.ndarray) -> bytes:
    return np.ascontiguousarray(seq, dtype=np.int8).tobytes()


def merge_shards(parts: Iterable[Sequence[Candidate]],
                 hash_fn: Optional[Callable[[np.ndarray], object]] = None) -> List[Candidate]:
    """Merge per-shard candidate lists into the single-pool --threads 1 order with dedup.

    The dedup key is the reference DedupSink's: the 64-bit canonical_hash(0) of the full
    sequence (candidate.hpp:84-99, rng.hpp:89-95), so even a tabulation-hash collision is
    resolved as the reference resolves it (the later sequence is dropped).  `hash_fn`
    replaces it (e.g. exact sequence bytes)."""
    h = hash_fn or (lambda seq: canonical_hash(seq, 0))
    allc = [c for part in parts for c in part]
    allc.sort(key=lambda c: (c.walker, c.restart, c.iteration))
    seen, out = set(), []
    for c in allc:
        k = h(c.seq)
        if k in seen:
            continue
        seen.add(k)
        out.append(c)
    return out


def merge_stats(parts: Sequence[PoolStats], emitted: int) -> PoolStats:
    st = PoolStats()
    for k in _SUM_KEYS:
        setattr(st, k, sum(getattr(p, k) for p in parts))
    for k in _MAX_KEYS:
        setattr(st, k, max((getattr(p, k) for p in parts), default=0.0))
    live = [p for p in parts if p.walks > 0]
    st.best_energy = min((p.best_energy for p in live), default=0)
    de = [p.delta_evals for p in parts]
    st.delta_evals = sum(de) if all(d >= 0 for d in de) else -1
    st.emitted = emitted
    st.n_gpus = sum(max(p.n_gpus, 1) for p in parts)
    return st


def run_saw_pool_distributed(cfg: SawConfig, sink: Optional[CandidateSink] = None,
                             group=None,
                             runner: Optional[Callable[[SawConfig], Tuple[List[Candidate],
                                                                          PoolStats]]] = None,
                             ) -> Optional[PoolStats]:
    """run_saw_pool over all ranks of a torch.distributed group (one GPU per rank).

    Every rank runs its class shard on its own device (cfg.device should be LOCAL_RANK);
    rank 0 receives the merged candidates (--threads 1 order, deduplicated) into `sink`
    and returns the merged PoolStats; other ranks return None.  `runner` replaces the
    per-rank GPU call (tests drive the host logic on CPU with it)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    scfg = shard_config(cfg, rank, world)
    if runner is None:
        from .api import CollectingSink

        local = CollectingSink()
        st = run_saw_pool(scfg, local)
        cands = local.take()
    else:
        cands, st = runner(scfg)
    if world == 1:
        gathered = [(cands, st)]
    else:
        gathered = [None] * world if rank == 0 else None
        dist.gather_object((cands, st), gathered, dst=0, group=group)
    if rank != 0:
        return None
    merged = merge_shards([g[0] for g in gathered])
    if sink is not None:
        for c in merged:
            sink.emit(c)
    return merge_stats([g[1] for g in gathered], len(merged))
