/*
 * labs_gpu.h -- C ABI of the B200-native Step-1 engine (libpaper_labs.so).
 *
 * Drop-in boundary for the reference's Step-1 entry point
 *     PoolStats run_saw_pool(const SawConfig&, CandidateSink&)
 *         /root/reference/proj/include/labs/saw.hpp:172, src/saw.cpp:218-267
 * Plain C types only (no torch, no CUDA types).  All entry points return
 * LABS_OK (0) or a negative status; labs_last_error() holds the message
 * (thread-local).  Validation happens on the host before any CUDA call and uses
 * the reference's messages (saw.cpp:51-63), so a C++ wrapper can rethrow them as
 * std::invalid_argument exactly like SawConfig::validate().
 *
 * There is no CPU fallback: when no sm_100 device is present every compute
 * entry point fails with LABS_ENODEV.
 */
#ifndef LABS_GPU_H
#define LABS_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    LABS_OK = 0,
    LABS_EINVAL = -1,      /* std::invalid_argument in the reference */
    LABS_ERANGE = -2,      /* std::out_of_range (skew.cpp:63) */
    LABS_ENODEV = -3,      /* no usable CUDA device */
    LABS_ECUDA = -4,       /* CUDA runtime failure */
    LABS_ELOGIC = -5,      /* std::logic_error: energy bookkeeping diverged (saw.cpp:141) */
    LABS_EABORT = -6       /* the candidate callback asked to stop */
};

/* Mirrors SawConfig (saw.hpp:34-61) field for field; GPU fields are additive. */
typedef struct labs_saw_config {
    int32_t length;            /* odd L >= 3 */
    int32_t prefix_len;        /* p; -1 = ceil(log2 walkers) + 1 */
    int32_t walkers;
    int32_t threads;           /* host threads (reference meaning); unused by the GPU path */
    int64_t max_iterations;    /* T_i; 0 = ti_multiplier * (L+1) / 2 */
    double ti_multiplier;
    int64_t energy_threshold;  /* E_l; > 0 unless target_merit set */
    double target_merit;       /* > 0: E_l = floor(L^2 / (2F)) */
    double bloom_fpr;
    uint64_t seed;
    int64_t max_restarts;      /* 0 = unlimited (needs another stop) */
    double time_budget_s;
    int64_t candidate_quota;
    int64_t stop_at_energy;
    int32_t debug_check_energy;
    /* --- additive GPU controls --- */
    int32_t n_gpus;            /* class shards run concurrently, shard g on device (device + g)
                                  mod the devices available; 0 or 1 = one */
    int32_t device;            /* first device ordinal */
    int32_t shard_index;       /* restriction-class shard of this process: walkers with */
    int32_t shard_count;       /*   (w mod 2^(p-1)) mod shard_count == shard_index      */
    int32_t count_visited;     /* 1: probe every free neighbour (exact delta-eval stats) */
    int32_t walker_begin;      /* optional walker sub-range [begin, end); end 0 = all */
    int32_t walker_end;
    int32_t reserved[6];
} labs_saw_config;

/* Candidate as delivered to the sink (candidate.hpp:21-29). Pointers valid only
 * during the callback. */
typedef struct labs_candidate {
    int32_t length;
    int32_t origin;            /* 0 = saw (Origin::saw) */
    int64_t energy;
    const int8_t* signs;       /* full expanded sequence, +1/-1, length L */
    const int8_t* prefix;      /* restriction-class prefix signs */
    int32_t prefix_len;
    int32_t _pad;
    int64_t walker, restart, iteration;
} labs_candidate;

/* CandidateSink::emit (candidate.hpp:56-60). Return 0 to continue, nonzero to abort. */
typedef int (*labs_candidate_fn)(void* user, const labs_candidate* c);

/* A batch of candidates (same order and semantics as labs_candidate_fn deliveries).
 * Arrays valid only during the callback; signs is count x length, row i the full
 * expanded sequence; prefix_class[i] indexes prefixes (P x prefix_len, rank order). */
typedef struct labs_candidate_batch {
    int32_t count;
    int32_t length;
    int32_t prefix_len;
    int32_t origin;            /* 0 = saw */
    const int8_t* signs;
    const int64_t* energy;
    const int64_t* walker;
    const int64_t* restart;
    const int64_t* iteration;
    const int32_t* prefix_class;
    const int8_t* prefixes;
} labs_candidate_batch;
typedef int (*labs_candidate_batch_fn)(void* user, const labs_candidate_batch* batch);

/* PoolStats (saw.hpp:161-167) + GPU counters */
typedef struct labs_pool_stats {
    int64_t walks;
    int64_t iterations;
    int64_t emitted;           /* post-dedup deliveries (what the reference counts) */
    int64_t best_energy;
    double wall_seconds;
    int64_t emitted_raw;       /* sieve hits before dedup */
    int64_t delta_evals;       /* unvisited free-neighbour evaluations (-1 unless counted) */
    int64_t delta_evals_computed; /* deltas the GPU actually computed */
    int64_t exhausted_walks;
    int64_t wide_iterations;   /* iterations on the int16-correlation path */
    double kernel_ms;          /* device time of the walk kernels (CUDA events, summed over
                                  batches; one device overlaps consecutive batches) */
    double seed_ms;            /* device time of the seed kernels */
    int32_t n_gpus;
    int32_t _pad;
    int64_t h2d_bytes;         /* host->device bytes copied by this call */
    int64_t d2h_bytes;         /* device->host bytes copied by this call */
} labs_pool_stats;

/* Replaces run_saw_pool (saw.cpp:218-267).  Candidates reach `emit` deduplicated
 * by canonical_hash(0) (DedupSink, candidate.hpp:84-99) and gated by the quota
 * (CountingSink, saw.cpp:173-194) in --threads 1 order: walker, restart,
 * iteration.  With no quota/time/stop_at_energy the candidate list is identical
 * to the reference's --threads 1 run. */
int labs_saw_pool_run(const labs_saw_config* cfg, labs_candidate_fn emit, void* user,
                      labs_pool_stats* stats);
/* Same, delivering candidates in batches (<= 8192 per call) -- cheaper across FFI
 * boundaries (the Python binding uses it). */
int labs_saw_pool_run_batched(const labs_saw_config* cfg, labs_candidate_batch_fn emit, void* user,
                              labs_pool_stats* stats);

/* Optional: set up now what a labs_saw_pool_run with this config's geometry (length,
 * prefix, T_i, Bloom size, devices) would set up on its first call -- CUDA context,
 * kernel modules, device tables, record rings -- so that a later pool's time budget
 * (time_budget_s) is spent searching.  The reference has no device to initialise
 * (saw.cpp:218 starts its clock on a warm process); the labs CLI calls this before
 * run_saw_pool. */
int labs_saw_prepare(const labs_saw_config* cfg);

/* Derived configuration (saw.cpp:44-63, sequence.cpp:36-40, bloom.cpp:15-24). */
typedef struct labs_saw_derived {
    int32_t prefix_len;
    int32_t bloom_hashes;
    int64_t iterations;        /* T_i */
    int64_t energy_threshold;  /* E_l */
    uint64_t bloom_bits;
    int32_t free_bits;         /* k + 1 - p */
    int32_t neighbours_per_lane;
    int32_t kernel;            /* walk kernel: 0 = K1 (IDP4A G), 1 = K1t (mma.sync int8 G) */
    int32_t lanes_per_walk;
} labs_saw_derived;
int labs_saw_derive(const labs_saw_config* cfg, labs_saw_derived* out);

/* Seed-table mode: walks from explicit initial halves (kp1 = (L+1)/2 signs each,
 * first `prefix_len` pinned).  Per-walk results and raw (undeduplicated) sieve
 * hits in (walk, iteration) order.  Replaces run_walk (saw.cpp:117-149) for a
 * batch of walks. */
typedef struct labs_walk_result {
    int64_t iterations, emitted, best_energy, initial_energy;
    int64_t exhausted, delta_evals, probe_rounds, wide_iterations, diverged;
} labs_walk_result;
typedef int (*labs_record_fn)(void* user, int64_t walk, int64_t iteration, int64_t energy,
                              const int8_t* half, int32_t kp1);
int labs_saw_walks(int32_t length, int32_t prefix_len, int64_t iterations,
                   int64_t energy_threshold, double bloom_fpr, const int8_t* halves,
                   int64_t nwalks, int32_t count_visited, int32_t debug_check,
                   labs_walk_result* results, labs_record_fn on_record, void* user);

/* skew_flip_delta_fast (skew.cpp:60-93) of every half index hp in [0, k] of each
 * expanded half, plus C_{2t} (t = 1..k) and E.  deltas: nseq x kp1;
 * corr: nseq x k (may be NULL); energies: nseq (may be NULL). */
int labs_skew_flip_deltas(int32_t length, const int8_t* halves, int64_t nseq, int64_t* deltas,
                          int64_t* corr, int64_t* energies);

/* Restriction-class Gray enumeration (extension; pattern of oracle.cpp:37-67):
 * half = rank_prefixes(p)[class_index] ++ (+1)^(k+1-p); configurations
 * g in [g_begin, g_end) of the 2^m Gray codes over half positions [p, p+m).
 * Emits (g, E) for E < energy_threshold in g order. */
typedef int (*labs_enum_fn)(void* user, uint64_t g, int64_t energy);
typedef struct labs_enum_stats {
    int64_t best_energy;
    uint64_t best_g;
    uint64_t configurations;
    uint64_t emitted;
    double kernel_ms;
} labs_enum_stats;
int labs_enumerate_class(int32_t length, int32_t prefix_len, int32_t class_index, int32_t m,
                         int64_t energy_threshold, uint64_t g_begin, uint64_t g_end,
                         labs_enum_fn emit, void* user, labs_enum_stats* stats);

/* K5, Step-2 neighbourhood scoring: everything refine
 * (pq.cpp:114-176) computes for one pivot, exactly, in one launch:
 *   deltas[i]                     flip_delta(pivot, i)                 (sequence.cpp:42-58)
 *   rot_energy[(i*2+dir)*t_r+r-1] energy of neighbour i after r one-step rotations,
 *                                 dir 0 = left, 1 = right              (pq.cpp:56-101)
 *   rot_hash[same index]          canonical_hash(0) of that sequence   (rng.hpp:89-95)
 *   *pivot_energy                 E(pivot)
 * The caller replays the frontier (seen / mark / push) in the reference order.
 * Thread-safe: each host thread uses its own stream and buffers. */
int labs_pq_score(int32_t length, int32_t t_r, const int8_t* pivot, int32_t* deltas,
                  int32_t* rot_energy, uint64_t* rot_hash, int64_t* pivot_energy);

/* Device-resident benchmark plan: the whole pool's walks with inputs in HBM.
 * labs_bench_run times `reps` launches (seed + walk kernels) with CUDA events on the
 * library's stream; before every rep (outside the timed events) a 256 MiB scratch
 * buffer is written so that no rep starts with a warm L2. */
typedef struct labs_bench_plan labs_bench_plan;
int labs_bench_create(const labs_saw_config* cfg, labs_bench_plan** out);
int labs_bench_run(labs_bench_plan* plan, int32_t reps, double* ms_per_rep,
                   labs_pool_stats* last);
void labs_bench_destroy(labs_bench_plan* plan);

/* INT32 issue-rate microbenchmark (all SMs, CUDA events): lane-ops/s of IMAD-only,
 * IADD3/LOP3/SHF-only and a 1:1 mix, and IDP4A lane-instructions/s (each = 4 int8 MACs). */
int labs_int32_peak(double* imad_ops, double* ialu_ops, double* mixed_ops, double* dp4a_ops,
                    int32_t* sm_count, int32_t* clock_khz);

/* int8 tensor-core MAC rate: mma.sync.m16n8k32.s8 chains on every SM (the path K1t's
 * sliding dot products use); MACs per second. */
int labs_imma_peak(double* int8_macs_per_s);

/* Host-side helpers (no GPU needed): the formats and hashes the sink chain uses. */
uint64_t labs_canonical_hash(const int8_t* signs, int32_t n, int32_t table); /* rng.hpp:89-95 */
int labs_format_record(const int8_t* signs, int32_t n, int64_t energy, char* out, int32_t cap);
int labs_rank_prefixes(int32_t p, int8_t* out);            /* saw.cpp:22-42, P x p signs */
int labs_expand_skew(const int8_t* half, int32_t kp1, int8_t* full);  /* skew.cpp:14-26 */

int labs_device_count(int32_t* n);
const char* labs_last_error(void);
const char* labs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LABS_GPU_H */
