/*
 * labs_oracle.h -- CPU restatement of the reference Step-1 path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2409_07222_b200/,
 * include/, tools/) may include, link or call this.  It is the checker that
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg compare the
 * CUDA path against.  Every function cites the reference file:line it
 * restates (paths relative to /root/reference/proj).  The restatement itself
 * is pinned against the reference library compiled from its own sources
 * (oracle/_ref, see oracle/Makefile) and against the KATs of the reference
 * tests (tests/test_oracle.py).
 */
#ifndef LABS_ORACLE_H
#define LABS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG (include/labs/rng.hpp:10-52) ---- */
typedef struct { uint64_t s[4]; } lo_rng;
uint64_t lo_splitmix64(uint64_t* state);
void lo_rng_init(lo_rng* r, uint64_t seed, uint64_t stream);
uint64_t lo_rng_next(lo_rng* r);
int lo_rng_sign(lo_rng* r);
uint64_t lo_rng_below(lo_rng* r, uint64_t n);

/* ---- tabulation hash (rng.hpp:75-101, rng.cpp:13-21) ---- */
uint64_t lo_tab_entry(int table, int pos, int sign);
uint64_t lo_tab_flip_mask(int table, int pos);
uint64_t lo_tab_salt(int table, int len);
uint64_t lo_tab_hash(const int8_t* signs, int n, int table);

/* ---- config derivation ---- */
int64_t lo_energy_threshold(int length, double target_merit);           /* sequence.cpp:36-40 */
int64_t lo_effective_iterations(int length, int64_t max_it, double mult); /* saw.hpp:51-54 */
int lo_effective_prefix_len(int prefix_len, int walkers);               /* saw.cpp:44-49 */
void lo_bloom_size(uint64_t capacity, double fpr, uint64_t* bits, int* hashes); /* bloom.cpp:15-24 */

/* ---- sequence / skew (sequence.cpp:8-19, skew.cpp:14-105) ---- */
void lo_expand_skew(const int8_t* half, int kp1, int8_t* full);
int64_t lo_correlations(const int8_t* s, int n, int64_t* c); /* returns E; c[0]=n */
int64_t lo_skew_flip_delta_fast(const int8_t* s, int n, const int64_t* c, int hp);
int64_t lo_apply_skew_flip(int8_t* s, int n, int64_t* c, int64_t* energy, int hp);
int64_t lo_flip_delta(const int8_t* s, int n, const int64_t* c, int i);

/* ---- prefixes (saw.cpp:11-42) ---- */
int64_t lo_prefix_potential(const int8_t* signs, int p);
/* out: (2^(p-1)) x p signs, ranked (stable sort by potential) */
int lo_rank_prefixes(int p, int8_t* out);

/* ---- Bloom filter (bloom.cpp:26-40) ---- */
void lo_bloom_insert(uint64_t* words, uint64_t bits, int k, uint64_t h1, uint64_t h2);
int lo_bloom_contains(const uint64_t* words, uint64_t bits, int k, uint64_t h1, uint64_t h2);

/* ---- Step-1 pool, --threads 1 semantics (saw.cpp:117-267) ---- */
typedef struct {
    int32_t length;
    int32_t prefix_len;       /* -1 = default */
    int32_t walkers;
    int32_t _pad0;
    int64_t max_iterations;   /* 0 = default */
    double ti_multiplier;
    int64_t energy_threshold;
    double target_merit;
    double bloom_fpr;
    uint64_t seed;
    int64_t max_restarts;
    double time_budget_s;
    int64_t candidate_quota;
    int64_t stop_at_energy;
    /* subset controls (oracle extension for sharded / sampled runs):
       only walkers w in [walker_begin, walker_end) with
       ((w mod P) mod shard_count) == shard_index run. end<=0 = all. */
    int32_t walker_begin;
    int32_t walker_end;
    int32_t shard_index;
    int32_t shard_count;
    int32_t dedup;            /* 1 = DedupSink in the chain (reference), 0 = raw emissions */
    int32_t _pad1;
} lo_saw_config;

typedef struct {
    int64_t walks, iterations, emitted, best_energy;
    int64_t delta_evals;      /* skew_flip_delta_fast calls (unvisited free neighbours) */
    int64_t bloom_hits;       /* neighbours skipped as visited */
    int64_t exhausted_walks;
    double wall_seconds;
} lo_pool_stats;

/* candidate callback: full sequence (length L), energy, walker, restart, iteration (1-based step) */
typedef void (*lo_candidate_fn)(void* user, const int8_t* seq, int length, int64_t energy,
                                int64_t walker, int64_t restart, int64_t iteration);
/* per-walk stats callback */
typedef void (*lo_walk_fn)(void* user, int64_t walker, int64_t restart, int64_t iterations,
                           int64_t emitted, int64_t best_energy, int64_t delta_evals,
                           int exhausted, int64_t initial_energy);

/* returns 0 on success, <0 with message in lo_last_error() on invalid config */
int lo_run_saw_pool(const lo_saw_config* cfg, lo_candidate_fn cand, lo_walk_fn walk, void* user,
                    lo_pool_stats* out);
const char* lo_last_error(void);

/* ---- one walk from an explicit initial half (run_walk, saw.cpp:117-149) ---- */
int lo_run_walk_from_half(int length, int prefix_len, const int8_t* half, int64_t t_i,
                          int64_t e_l, uint64_t bloom_bits, int bloom_k, lo_candidate_fn cand,
                          void* user, int64_t* iterations, int64_t* best, int64_t* delta_evals,
                          int* exhausted);

/* ---- restriction-class Gray enumeration (extension, pattern of oracle.cpp:37-67) ----
 * Half = prefix (class `class_index` of rank_prefixes(p)) ++ all +1.  Visits the
 * 2^m configurations of free half positions [p, p+m) in Gray order: config g
 * differs from g-1 by the flip of position p + ctz(g).  Emits (g, E) for every
 * configuration g in [g_begin, g_end) with E < e_l.  Returns best E over the range
 * and its first g. */
typedef void (*lo_enum_fn)(void* user, uint64_t g, int64_t energy);
int lo_enumerate_class(int length, int p, int class_index, int m, int64_t e_l, uint64_t g_begin,
                       uint64_t g_end, lo_enum_fn cb, void* user, int64_t* best_e,
                       uint64_t* best_g, uint64_t* emitted);

/* global skew optimum by Gray enumeration (oracle.cpp:37-67) */
int64_t lo_oracle_skew_exhaustive(int length, int8_t* best_full);

/* ---- candidate file format (candidate.cpp:36-49, hex_codec.cpp:14-30) ---- */
int lo_hex_encode(const int8_t* s, int n, char* out); /* writes ceil(n/4) digits + NUL */
int lo_format_record(const int8_t* s, int n, int64_t energy, char* out, int cap);

#ifdef __cplusplus
}
#endif
#endif
