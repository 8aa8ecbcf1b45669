/*
 * labs_oracle.c -- CPU restatement of the reference Step-1 path (plain C11).
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA path, never the product.
 * See labs_oracle.h.  Citations are /root/reference/proj/<file>:<line>.
 */
#define _POSIX_C_SOURCE 199309L
#include "labs_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static char g_err[256];
const char* lo_last_error(void) { return g_err; }
static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}

/* ------------------------------------------------------------------ RNG */
/* rng.hpp:10-15 */
uint64_t lo_splitmix64(uint64_t* state) {
    *state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:21-24: stream-mixed splitmix seeding of xoshiro256** */
void lo_rng_init(lo_rng* r, uint64_t seed, uint64_t stream) {
    uint64_t sm = seed ^ (0xa0761d6478bd642fULL * (stream + 1));
    for (int i = 0; i < 4; ++i) r->s[i] = lo_splitmix64(&sm);
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:26-36 (xoshiro256**) */
uint64_t lo_rng_next(lo_rng* r) {
    uint64_t* s = r->s;
    const uint64_t out = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
}

/* rng.hpp:45: +1 iff the top bit is set */
int lo_rng_sign(lo_rng* r) { return (lo_rng_next(r) >> 63) ? 1 : -1; }

/* rng.hpp:40-43: Lemire multiply-shift */
uint64_t lo_rng_below(lo_rng* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)lo_rng_next(r) * n) >> 64);
}

/* --------------------------------------------------------- tabulation */
/* rng.cpp:13-21: fixed-seed splitmix stream fills T[2][1024][2] then salts[2][1026] */
#define TAB_MAX 1024
static uint64_t g_tab[2][TAB_MAX][2];
static uint64_t g_salt[2][TAB_MAX + 2];
static int g_tab_ready = 0;

static void tab_init(void) {
    if (g_tab_ready) return;
    uint64_t sm = 0x5eed5eed5eed5eedULL;
    for (int t = 0; t < 2; ++t)
        for (int p = 0; p < TAB_MAX; ++p)
            for (int b = 0; b < 2; ++b) g_tab[t][p][b] = lo_splitmix64(&sm);
    for (int t = 0; t < 2; ++t)
        for (int l = 0; l < TAB_MAX + 2; ++l) g_salt[t][l] = lo_splitmix64(&sm);
    g_tab_ready = 1;
}

uint64_t lo_tab_entry(int table, int pos, int sign) {
    tab_init();
    return g_tab[table][pos][sign > 0 ? 1 : 0];
}
uint64_t lo_tab_flip_mask(int table, int pos) {
    tab_init();
    return g_tab[table][pos][0] ^ g_tab[table][pos][1];
}
uint64_t lo_tab_salt(int table, int len) {
    tab_init();
    return g_salt[table][len];
}
/* rng.hpp:89-95 */
uint64_t lo_tab_hash(const int8_t* signs, int n, int table) {
    tab_init();
    uint64_t h = g_salt[table][n];
    for (int i = 0; i < n; ++i) h ^= g_tab[table][i][signs[i] > 0 ? 1 : 0];
    return h;
}

/* --------------------------------------------------- config derivation */
int64_t lo_energy_threshold(int length, double target_merit) {
    const double l2 = (double)length * length;
    return (int64_t)floor(l2 / (2.0 * target_merit));
}

int64_t lo_effective_iterations(int length, int64_t max_it, double mult) {
    if (max_it > 0) return max_it;
    return (int64_t)(mult * (length + 1) / 2);
}

int lo_effective_prefix_len(int prefix_len, int walkers) {
    if (prefix_len >= 0) return prefix_len;
    int p = 1;
    while ((1 << (p - 1)) < walkers) ++p;
    return p;
}

void lo_bloom_size(uint64_t capacity, double fpr, uint64_t* bits, int* hashes) {
    if (capacity == 0) capacity = 1;
    const double ln2 = log(2.0);
    const double m = -(double)capacity * log(fpr) / (ln2 * ln2);
    uint64_t b = (uint64_t)ceil(m);
    int k = (int)lround(m / (double)capacity * ln2);
    if (k < 1) k = 1;
    *bits = b < 64 ? 64 : b;
    *hashes = k;
}

/* ------------------------------------------------------ sequence/skew */
/* skew.cpp:14-26 */
void lo_expand_skew(const int8_t* half, int kp1, int8_t* full) {
    const int k = kp1 - 1;
    for (int i = 0; i < kp1; ++i) full[i] = half[i];
    for (int i = 1; i <= k; ++i) full[k + i] = (i % 2 == 0) ? full[k - i] : (int8_t)-full[k - i];
}

/* sequence.cpp:8-19 */
int64_t lo_correlations(const int8_t* s, int n, int64_t* c) {
    int64_t e = 0;
    c[0] = n;
    for (int k = 1; k < n; ++k) {
        int64_t acc = 0;
        for (int i = 0; i + k < n; ++i) acc += (int64_t)s[i] * s[i + k];
        c[k] = acc;
        e += acc * acc;
    }
    return e;
}

/* sequence.cpp:42-58 */
int64_t lo_flip_delta(const int8_t* s, int n, const int64_t* c, int i) {
    const int64_t si = s[i];
    int64_t d = 0;
    const int kmax = i > n - 1 - i ? i : n - 1 - i;
    for (int k = 1; k <= kmax; ++k) {
        int t = 0;
        if (i - k >= 0) t += s[i - k];
        if (i + k < n) t += s[i + k];
        if (t == 0) continue;
        const int64_t dc = -2 * si * t;
        d += dc * (2 * c[k] + dc);
    }
    return d;
}

/* sequence.cpp:60-79 */
static int64_t apply_flip(int8_t* s, int n, int64_t* c, int64_t* energy, int i) {
    const int64_t si = s[i];
    int64_t d = 0;
    const int kmax = i > n - 1 - i ? i : n - 1 - i;
    for (int k = 1; k <= kmax; ++k) {
        int t = 0;
        if (i - k >= 0) t += s[i - k];
        if (i + k < n) t += s[i + k];
        if (t == 0) continue;
        const int64_t dc = -2 * si * t;
        d += dc * (2 * c[k] + dc);
        c[k] += dc;
    }
    *energy += d;
    s[i] = (int8_t)-s[i];
    return d;
}

/* skew.cpp:60-93: fused even-lag double-flip delta */
int64_t lo_skew_flip_delta_fast(const int8_t* x, int n, const int64_t* c, int hp) {
    const int a = hp, b = n - 1 - hp;
    int64_t d = 0;
    if (a == b) {
        for (int kk = 2; kk < n; kk += 2) {
            int t = 0;
            if (a - kk >= 0) t += x[a - kk];
            if (a + kk < n) t += x[a + kk];
            if (t == 0) continue;
            const int64_t dc = -2 * (int64_t)x[a] * t;
            d += dc * (2 * c[kk] + dc);
        }
        return d;
    }
    for (int kk = 2; kk < n; kk += 2) {
        int64_t dc = 0;
        if (a - kk >= 0) dc += (int64_t)x[a] * x[a - kk];
        if (a + kk < n && a + kk != b) dc += (int64_t)x[a] * x[a + kk];
        if (b - kk >= 0 && b - kk != a) dc += (int64_t)x[b] * x[b - kk];
        if (b + kk < n) dc += (int64_t)x[b] * x[b + kk];
        if (dc == 0) continue;
        dc *= -2;
        d += dc * (2 * c[kk] + dc);
    }
    return d;
}

/* skew.cpp:95-105: flip a, then its mirror (the centre alone when a == b) */
int64_t lo_apply_skew_flip(int8_t* s, int n, int64_t* c, int64_t* energy, int hp) {
    const int a = hp, b = n - 1 - hp;
    if (a == b) return apply_flip(s, n, c, energy, a);
    const int64_t d1 = apply_flip(s, n, c, energy, a);
    const int64_t d2 = apply_flip(s, n, c, energy, b);
    return d1 + d2;
}

/* ----------------------------------------------------------- prefixes */
/* saw.cpp:11-20 */
int64_t lo_prefix_potential(const int8_t* signs, int p) {
    int64_t e = 0;
    for (int k = 1; k < p; ++k) {
        int64_t c = 0;
        for (int i = 0; i + k < p; ++i) c += (int64_t)signs[i] * signs[i + k];
        e += c * c;
    }
    return e;
}

/* saw.cpp:22-42: enumerate s_0=+1 prefixes, bit j-1 of the counter -> s_j=-1,
   stable sort by potential (insertion into per-potential buckets keeps order) */
int lo_rank_prefixes(int p, int8_t* out) {
    if (p < 1 || p > 30) return fail("rank_prefixes: p out of range");
    const uint64_t count = 1ULL << (p - 1);
    int64_t* pot = (int64_t*)malloc(count * sizeof(int64_t));
    int8_t* tmp = (int8_t*)malloc(count * (size_t)p);
    int64_t maxpot = 0;
    for (uint64_t bits = 0; bits < count; ++bits) {
        int8_t* s = tmp + bits * (uint64_t)p;
        s[0] = 1;
        for (int j = 1; j < p; ++j) s[j] = ((bits >> (j - 1)) & 1) ? -1 : 1;
        pot[bits] = lo_prefix_potential(s, p);
        if (pot[bits] > maxpot) maxpot = pot[bits];
    }
    /* counting sort over potential values is a stable sort */
    uint64_t o = 0;
    for (int64_t v = 0; v <= maxpot; ++v)
        for (uint64_t bits = 0; bits < count; ++bits)
            if (pot[bits] == v) {
                memcpy(out + o * (uint64_t)p, tmp + bits * (uint64_t)p, (size_t)p);
                ++o;
            }
    free(pot);
    free(tmp);
    return 0;
}

/* --------------------------------------------------------------- Bloom */
/* bloom.cpp:26-40: idx = (h1 + i*h2) mod 2^64 mod bits */
void lo_bloom_insert(uint64_t* w, uint64_t bits, int k, uint64_t h1, uint64_t h2) {
    for (int i = 0; i < k; ++i) {
        const uint64_t idx = (h1 + (uint64_t)i * h2) % bits;
        w[idx >> 6] |= 1ULL << (idx & 63);
    }
}
int lo_bloom_contains(const uint64_t* w, uint64_t bits, int k, uint64_t h1, uint64_t h2) {
    for (int i = 0; i < k; ++i) {
        const uint64_t idx = (h1 + (uint64_t)i * h2) % bits;
        if (!(w[idx >> 6] & (1ULL << (idx & 63)))) return 0;
    }
    return 1;
}

/* ------------------------------------------------------ u64 hash set */
typedef struct {
    uint64_t* keys;
    uint8_t* used;
    size_t cap, n;
} hset;

static void hset_init(hset* h) {
    h->cap = 1024;
    h->n = 0;
    h->keys = (uint64_t*)calloc(h->cap, sizeof(uint64_t));
    h->used = (uint8_t*)calloc(h->cap, 1);
}
static void hset_free(hset* h) {
    free(h->keys);
    free(h->used);
}
static int hset_insert(hset* h, uint64_t key);
static void hset_grow(hset* h) {
    hset old = *h;
    h->cap *= 2;
    h->n = 0;
    h->keys = (uint64_t*)calloc(h->cap, sizeof(uint64_t));
    h->used = (uint8_t*)calloc(h->cap, 1);
    for (size_t i = 0; i < old.cap; ++i)
        if (old.used[i]) hset_insert(h, old.keys[i]);
    hset_free(&old);
}
/* returns 1 if newly inserted */
static int hset_insert(hset* h, uint64_t key) {
    if ((h->n + 1) * 2 > h->cap) hset_grow(h);
    uint64_t z = key * 0x9e3779b97f4a7c15ULL;
    size_t i = (size_t)(z >> 17) & (h->cap - 1);
    while (h->used[i]) {
        if (h->keys[i] == key) return 0;
        i = (i + 1) & (h->cap - 1);
    }
    h->used[i] = 1;
    h->keys[i] = key;
    ++h->n;
    return 1;
}

/* ---------------------------------------------------------------- walk */
typedef struct {
    int L, kp1, p;
    int8_t* seq;   /* full pivot */
    int64_t* c;    /* correlations */
    int64_t e;     /* state energy */
    uint64_t h1, h2;
} walk_state;

/* saw.cpp:77-89 */
static void walk_state_init(walk_state* ws, int L, int p, const int8_t* half) {
    ws->L = L;
    ws->kp1 = (L + 1) / 2;
    ws->p = p;
    lo_expand_skew(half, ws->kp1, ws->seq);
    ws->e = lo_correlations(ws->seq, L, ws->c);
    ws->h1 = lo_tab_salt(0, ws->kp1);
    ws->h2 = lo_tab_salt(1, ws->kp1);
    for (int i = 0; i < ws->kp1; ++i) {
        ws->h1 ^= lo_tab_entry(0, i, half[i]);
        ws->h2 ^= lo_tab_entry(1, i, half[i]);
    }
}

typedef struct {
    int64_t iterations, emitted, best, deltas, hits;
    int exhausted;
    int64_t e0;
} walk_result;

typedef void (*emit_fn)(void* ctx, const walk_state* ws, int64_t e, int64_t it);

/* saw.cpp:106-149: run_walk with best_neighbour inlined */
static void run_walk(walk_state* ws, int64_t t_i, int64_t e_l, uint64_t* bloom, uint64_t bbits,
                     int bk, emit_fn emit, void* ctx, walk_result* r) {
    const int k = ws->kp1 - 1;
    memset(bloom, 0, ((bbits + 63) / 64) * sizeof(uint64_t));
    lo_bloom_insert(bloom, bbits, bk, ws->h1, ws->h2);
    int64_t e = ws->e;
    memset(r, 0, sizeof *r);
    r->best = e;
    r->e0 = e;
    for (int64_t it = 0; it < t_i; ++it) {
        int best_hp = -1;
        int64_t best_d = 0;
        for (int hp = ws->p; hp <= k; ++hp) {
            const uint64_t n1 = ws->h1 ^ lo_tab_flip_mask(0, hp);
            const uint64_t n2 = ws->h2 ^ lo_tab_flip_mask(1, hp);
            if (lo_bloom_contains(bloom, bbits, bk, n1, n2)) {
                ++r->hits;
                continue;
            }
            const int64_t d = lo_skew_flip_delta_fast(ws->seq, ws->L, ws->c, hp);
            ++r->deltas;
            if (best_hp < 0 || d < best_d) {
                best_d = d;
                best_hp = hp;
            }
        }
        if (best_hp < 0) {
            r->exhausted = 1;
            break;
        }
        ++r->iterations;
        lo_apply_skew_flip(ws->seq, ws->L, ws->c, &ws->e, best_hp);
        ws->h1 ^= lo_tab_flip_mask(0, best_hp);
        ws->h2 ^= lo_tab_flip_mask(1, best_hp);
        lo_bloom_insert(bloom, bbits, bk, ws->h1, ws->h2);
        e += best_d;
        if (e < r->best) r->best = e;
        if (e < e_l) {
            emit(ctx, ws, e, it + 1);
            ++r->emitted;
        }
    }
}

/* ------------------------------------------------------------- pool */
typedef struct {
    const lo_saw_config* cfg;
    lo_candidate_fn cand;
    void* user;
    hset seen;
    int64_t emitted;
    int stop;
    int64_t walker, restart;
} pool_ctx;

/* DedupSink (candidate.hpp:84-99) -> CountingSink (saw.cpp:173-194) -> user sink */
static void pool_emit(void* vctx, const walk_state* ws, int64_t e, int64_t it) {
    pool_ctx* pc = (pool_ctx*)vctx;
    if (pc->cfg->dedup) {
        if (!hset_insert(&pc->seen, lo_tab_hash(ws->seq, ws->L, 0))) return;
    }
    const int64_t n = ++pc->emitted;
    if (pc->cfg->candidate_quota > 0) {
        if (n > pc->cfg->candidate_quota) {
            pc->stop = 1;
            --pc->emitted;
            return;
        }
        if (n >= pc->cfg->candidate_quota) pc->stop = 1;
    }
    if (pc->cand) pc->cand(pc->user, ws->seq, ws->L, e, pc->walker, pc->restart, it);
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int lo_run_saw_pool(const lo_saw_config* cfg, lo_candidate_fn cand, lo_walk_fn walkcb, void* user,
                    lo_pool_stats* out) {
    /* SawConfig::validate (saw.cpp:51-63) */
    const int L = cfg->length;
    if (L < 3 || L % 2 == 0) return fail("saw: length must be odd and >= 3");
    if (cfg->walkers < 1) return fail("saw: walkers must be >= 1");
    const int64_t e_l = cfg->target_merit > 0.0 ? lo_energy_threshold(L, cfg->target_merit)
                                                : cfg->energy_threshold;
    if (e_l <= 0) return fail("saw: energy threshold E_l must be positive");
    const int64_t t_i = lo_effective_iterations(L, cfg->max_iterations, cfg->ti_multiplier);
    if (t_i < 1) return fail("saw: T_i must be >= 1");
    const int kp1 = (L + 1) / 2;
    const int p = lo_effective_prefix_len(cfg->prefix_len, cfg->walkers);
    if (p > kp1) return fail("saw: prefix length exceeds half length k+1");
    if (cfg->max_restarts == 0 && cfg->time_budget_s <= 0 && cfg->candidate_quota == 0 &&
        cfg->stop_at_energy == 0)
        return fail("saw: no stop condition configured");
    if (kp1 > TAB_MAX) return fail("saw: length exceeds tabulation table");

    const double t0 = now_s();
    /* saw.cpp:228-231 */
    int64_t nprefix = 1;
    int8_t* prefixes = NULL;
    if (p > 0) {
        if (p > 30) return fail("rank_prefixes: p > 30 is not enumerable");
        nprefix = 1LL << (p - 1);
        prefixes = (int8_t*)malloc((size_t)nprefix * (size_t)p);
        lo_rank_prefixes(p, prefixes);
    }
    uint64_t bbits;
    int bk;
    lo_bloom_size((uint64_t)t_i + 1, cfg->bloom_fpr, &bbits, &bk);
    uint64_t* bloom = (uint64_t*)calloc((bbits + 63) / 64, sizeof(uint64_t));

    walk_state ws;
    ws.seq = (int8_t*)malloc((size_t)L);
    ws.c = (int64_t*)malloc(sizeof(int64_t) * (size_t)L);
    int8_t* half = (int8_t*)malloc((size_t)kp1);

    pool_ctx pc;
    memset(&pc, 0, sizeof pc);
    pc.cfg = cfg;
    pc.cand = cand;
    pc.user = user;
    hset_init(&pc.seen);

    lo_pool_stats st;
    memset(&st, 0, sizeof st);
    int best_set = 0;
    const int w0 = cfg->walker_begin > 0 ? cfg->walker_begin : 0;
    const int w1 = cfg->walker_end > 0 && cfg->walker_end < cfg->walkers ? cfg->walker_end
                                                                          : cfg->walkers;
    const int scount = cfg->shard_count > 0 ? cfg->shard_count : 1;
    const double deadline = t0 + cfg->time_budget_s;

    /* saw.cpp:238-241 (threads <= 1): walkers in order, walker_loop each */
    for (int w = w0; w < w1 && !pc.stop; ++w) {
        const int64_t cls = w % nprefix;
        if (scount > 1 && (int)(cls % scount) != cfg->shard_index) continue;
        const int8_t* pre = prefixes ? prefixes + cls * p : NULL;
        lo_rng rng;
        lo_rng_init(&rng, cfg->seed, (uint64_t)w);
        for (int64_t r = 0; cfg->max_restarts == 0 || r < cfg->max_restarts; ++r) {
            if (pc.stop) break;
            if (cfg->time_budget_s > 0 && now_s() >= deadline) {
                pc.stop = 1;
                break;
            }
            /* init_partitioned_sequence (saw.cpp:65-75) */
            for (int i = 0; i < p; ++i) half[i] = pre[i];
            for (int i = p; i < kp1; ++i) half[i] = (int8_t)lo_rng_sign(&rng);
            walk_state_init(&ws, L, p, half);
            pc.walker = w;
            pc.restart = r;
            walk_result wr;
            run_walk(&ws, t_i, e_l, bloom, bbits, bk, pool_emit, &pc, &wr);
            ++st.walks;
            st.iterations += wr.iterations;
            st.delta_evals += wr.deltas;
            st.bloom_hits += wr.hits;
            st.exhausted_walks += wr.exhausted;
            if (walkcb)
                walkcb(user, w, r, wr.iterations, wr.emitted, wr.best, wr.deltas, wr.exhausted,
                       wr.e0);
            /* PoolControl::offer_best (saw.cpp:160-169) */
            if (!best_set || wr.best < st.best_energy) {
                st.best_energy = wr.best;
                best_set = 1;
                if (cfg->stop_at_energy > 0 && wr.best <= cfg->stop_at_energy) pc.stop = 1;
            }
        }
    }
    st.emitted = pc.emitted;
    st.wall_seconds = now_s() - t0;
    if (out) *out = st;
    hset_free(&pc.seen);
    free(half);
    free(ws.seq);
    free(ws.c);
    free(bloom);
    free(prefixes);
    return 0;
}

typedef struct {
    lo_candidate_fn cand;
    void* user;
} raw_ctx;
static void raw_emit(void* vctx, const walk_state* ws, int64_t e, int64_t it) {
    raw_ctx* rc = (raw_ctx*)vctx;
    if (rc->cand) rc->cand(rc->user, ws->seq, ws->L, e, 0, 0, it);
}

int lo_run_walk_from_half(int length, int prefix_len, const int8_t* half, int64_t t_i,
                          int64_t e_l, uint64_t bloom_bits, int bloom_k, lo_candidate_fn cand,
                          void* user, int64_t* iterations, int64_t* best, int64_t* delta_evals,
                          int* exhausted) {
    if (length < 3 || length % 2 == 0) return fail("length must be odd and >= 3");
    walk_state ws;
    ws.seq = (int8_t*)malloc((size_t)length);
    ws.c = (int64_t*)malloc(sizeof(int64_t) * (size_t)length);
    walk_state_init(&ws, length, prefix_len, half);
    uint64_t* bloom = (uint64_t*)calloc((bloom_bits + 63) / 64, sizeof(uint64_t));
    raw_ctx rc = {cand, user};
    walk_result wr;
    run_walk(&ws, t_i, e_l, bloom, bloom_bits, bloom_k, raw_emit, &rc, &wr);
    if (iterations) *iterations = wr.iterations;
    if (best) *best = wr.best;
    if (delta_evals) *delta_evals = wr.deltas;
    if (exhausted) *exhausted = wr.exhausted;
    free(bloom);
    free(ws.seq);
    free(ws.c);
    return 0;
}

/* ------------------------------------------------------- enumeration */
static int ctz64(uint64_t v) { return __builtin_ctzll(v); }

int lo_enumerate_class(int L, int p, int class_index, int m, int64_t e_l, uint64_t g_begin,
                       uint64_t g_end, lo_enum_fn cb, void* user, int64_t* best_e,
                       uint64_t* best_g, uint64_t* emitted) {
    const int kp1 = (L + 1) / 2;
    if (L < 3 || L % 2 == 0) return fail("enumerate: length must be odd and >= 3");
    if (p < 1 || p > kp1) return fail("enumerate: bad prefix length");
    if (m < 0 || p + m > kp1 || m > 62) return fail("enumerate: bad free-bit count");
    const uint64_t total = 1ULL << m;
    if (g_end > total) g_end = total;
    if (class_index < 0 || class_index >= (1 << (p - 1))) return fail("enumerate: bad class");
    int8_t* pre = (int8_t*)malloc((size_t)(1 << (p - 1)) * (size_t)p);
    lo_rank_prefixes(p, pre);
    int8_t* half = (int8_t*)malloc((size_t)kp1);
    for (int i = 0; i < kp1; ++i) half[i] = 1;
    for (int i = 0; i < p; ++i) half[i] = pre[(size_t)class_index * (size_t)p + (size_t)i];
    /* configuration g = Gray(g) over positions p..p+m-1 (bit j -> position p+j is -1) */
    const uint64_t gray0 = g_begin ^ (g_begin >> 1);
    for (int j = 0; j < m; ++j)
        if ((gray0 >> j) & 1) half[p + j] = -1;
    int8_t* s = (int8_t*)malloc((size_t)L);
    int64_t* c = (int64_t*)malloc(sizeof(int64_t) * (size_t)L);
    lo_expand_skew(half, kp1, s);
    int64_t e = lo_correlations(s, L, c);
    int64_t be = e;
    uint64_t bg = g_begin, ne = 0;
    if (e < e_l) {
        ++ne;
        if (cb) cb(user, g_begin, e);
    }
    for (uint64_t g = g_begin + 1; g < g_end; ++g) {
        lo_apply_skew_flip(s, L, c, &e, p + ctz64(g));
        if (e < be) {
            be = e;
            bg = g;
        }
        if (e < e_l) {
            ++ne;
            if (cb) cb(user, g, e);
        }
    }
    if (best_e) *best_e = be;
    if (best_g) *best_g = bg;
    if (emitted) *emitted = ne;
    free(pre);
    free(half);
    free(s);
    free(c);
    return 0;
}

/* oracle.cpp:37-67 */
int64_t lo_oracle_skew_exhaustive(int L, int8_t* best_full) {
    const int k = (L - 1) / 2;
    int8_t* half = (int8_t*)malloc((size_t)k + 1);
    for (int i = 0; i <= k; ++i) half[i] = 1;
    int8_t* s = (int8_t*)malloc((size_t)L);
    int64_t* c = (int64_t*)malloc(sizeof(int64_t) * (size_t)L);
    lo_expand_skew(half, k + 1, s);
    int64_t e = lo_correlations(s, L, c);
    int64_t best = e;
    uint64_t code = 0;
    const uint64_t total = 1ULL << k;
    for (uint64_t g = 1; g < total; ++g) {
        lo_apply_skew_flip(s, L, c, &e, ctz64(g) + 1);
        if (e < best) {
            best = e;
            code = g ^ (g >> 1);
        }
    }
    for (int j = 1; j <= k; ++j) half[j] = ((code >> (j - 1)) & 1) ? -1 : 1;
    if (best_full) lo_expand_skew(half, k + 1, best_full);
    free(half);
    free(s);
    free(c);
    return best;
}

/* ---------------------------------------------------------- formats */
/* hex_codec.cpp:14-30: MSB-first, +1 -> 1, left zero pad to whole nibbles */
int lo_hex_encode(const int8_t* s, int n, char* out) {
    static const char* hx = "0123456789ABCDEF";
    const int digits = (n + 3) / 4;
    const int pad = digits * 4 - n;
    for (int d = 0; d < digits; ++d) {
        int v = 0;
        for (int b = 0; b < 4; ++b) {
            const int pos = d * 4 + b - pad;
            v = (v << 1) | (pos >= 0 && s[pos] > 0 ? 1 : 0);
        }
        out[d] = hx[v];
    }
    out[digits] = 0;
    return digits;
}

/* candidate.cpp:36-49 */
int lo_format_record(const int8_t* s, int n, int64_t energy, char* out, int cap) {
    char* hex = (char*)malloc((size_t)n / 4 + 2);
    lo_hex_encode(s, n, hex);
    const double f = (double)n * (double)n / (2.0 * (double)energy);
    const int w = snprintf(out, (size_t)cap, "%d\t%lld\t%.4f\t%s\tsaw", n, (long long)energy, f, hex);
    free(hex);
    return w;
}
