// ref_shim.cpp -- extern "C" seam over the REFERENCE library compiled from its
// own sources (/root/reference/proj/src/*.cpp, see oracle/Makefile).
//
// TEST INFRASTRUCTURE ONLY.  This file contains no reference code: it only
// calls the reference's public API (labs/*.hpp) so that Python tests can pin
// the C restatement (labs_oracle.c) and the CUDA path against the real thing,
// and so that bench.py --impl reference can time the unmodified reference.
#include <cstring>
#include <atomic>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "labs/candidate.hpp"
#include "labs/hex_codec.hpp"
#include "labs/oracle.hpp"
#include "labs/saw.hpp"
#include "labs_oracle.h"

using namespace labsearch;

namespace {
thread_local std::string g_err;

SawConfig to_saw(const lo_saw_config* c, int threads) {
    SawConfig s;
    s.length = c->length;
    s.prefix_len = c->prefix_len;
    s.walkers = c->walkers;
    s.max_iterations = c->max_iterations;
    s.ti_multiplier = c->ti_multiplier;
    s.energy_threshold = c->energy_threshold;
    s.target_merit = c->target_merit;
    s.bloom_fpr = c->bloom_fpr;
    s.seed = c->seed;
    s.threads = threads;
    s.max_restarts = c->max_restarts;
    s.time_budget_s = c->time_budget_s;
    s.candidate_quota = c->candidate_quota;
    s.stop_at_energy = c->stop_at_energy;
    return s;
}

class CallbackSink final : public CandidateSink {
public:
    CallbackSink(lo_candidate_fn fn, void* user) : fn_(fn), user_(user) {}
    void emit(const Candidate& c) override {
        std::lock_guard<std::mutex> lock(mu_);
        if (fn_) fn_(user_, c.seq.data(), c.seq.length(), c.energy, walker, restart, 0);
    }
    long long walker = -1, restart = -1;

private:
    std::mutex mu_;
    lo_candidate_fn fn_;
    void* user_;
};

// VisitedSet wrapper that counts probe misses (= skew_flip_delta_fast calls in
// best_neighbour, saw.cpp:109-113) around the reference BloomVisited.
class CountingVisited final : public VisitedSet {
public:
    CountingVisited(std::size_t cap, double fpr) : inner_(cap, fpr) {}
    void insert(std::uint64_t h1, std::uint64_t h2) override { inner_.insert(h1, h2); }
    bool maybe_contains(std::uint64_t h1, std::uint64_t h2) const override {
        const bool hit = inner_.maybe_contains(h1, h2);
        if (hit) ++hits; else ++misses;
        return hit;
    }
    void clear() override { inner_.clear(); }
    mutable long long hits = 0, misses = 0;

private:
    BloomVisited inner_;
};

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// The unmodified reference pool (saw.cpp:218-267) with `threads` std::threads.
int ref_run_saw_pool(const lo_saw_config* cfg, int threads, lo_candidate_fn cand, void* user,
                     lo_pool_stats* out) {
    try {
        CallbackSink sink(cand, user);
        const PoolStats ps = run_saw_pool(to_saw(cfg, threads), sink);
        if (out) {
            std::memset(out, 0, sizeof *out);
            out->walks = ps.walks;
            out->iterations = ps.iterations;
            out->emitted = ps.emitted;
            out->best_energy = ps.best_energy;
            out->wall_seconds = ps.wall_seconds;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// walker_loop replica (saw.cpp:196-214) driving the reference run_walk with a
// counting VisitedSet: per-walk stats and delta-eval counts for walkers
// [walker_begin, walker_end), threads=1 order, reference DedupSink in front.
int ref_walk_trace(const lo_saw_config* cfg, lo_candidate_fn cand, lo_walk_fn walkcb, void* user,
                   lo_pool_stats* out) {
    try {
        SawConfig sc = to_saw(cfg, 1);
        sc.validate();
        const int p = sc.effective_prefix_len();
        std::vector<PartitionPrefix> prefixes;
        if (p == 0) prefixes.push_back(PartitionPrefix{{}, 0});
        else prefixes = rank_prefixes(p);
        CallbackSink user_sink(cand, user);
        DedupSink dedup(user_sink);
        CandidateSink* sink = cfg->dedup ? static_cast<CandidateSink*>(&dedup)
                                         : static_cast<CandidateSink*>(&user_sink);
        lo_pool_stats st;
        std::memset(&st, 0, sizeof st);
        bool best_set = false;
        const int w0 = cfg->walker_begin > 0 ? cfg->walker_begin : 0;
        const int w1 = cfg->walker_end > 0 && cfg->walker_end < sc.walkers ? cfg->walker_end
                                                                            : sc.walkers;
        const int scount = cfg->shard_count > 0 ? cfg->shard_count : 1;
        for (int w = w0; w < w1; ++w) {
            const std::size_t cls = static_cast<std::size_t>(w) % prefixes.size();
            if (scount > 1 && static_cast<int>(cls % scount) != cfg->shard_index) continue;
            Rng rng(sc.seed, static_cast<std::uint64_t>(w));
            CountingVisited visited(static_cast<std::size_t>(sc.effective_iterations()) + 1,
                                    sc.bloom_fpr);
            for (long long r = 0; r < sc.max_restarts; ++r) {
                user_sink.walker = w;
                user_sink.restart = r;
                const long long m0 = visited.misses;
                const WalkStats ws = run_walk(sc, prefixes[cls], rng, visited, *sink);
                ++st.walks;
                st.iterations += ws.iterations;
                st.delta_evals += visited.misses - m0;
                st.exhausted_walks += ws.neighbourhood_exhausted ? 1 : 0;
                if (walkcb)
                    walkcb(user, w, r, ws.iterations, ws.emitted, ws.best_energy,
                           visited.misses - m0, ws.neighbourhood_exhausted ? 1 : 0, 0);
                if (!best_set || ws.best_energy < st.best_energy) {
                    st.best_energy = ws.best_energy;
                    best_set = true;
                }
            }
        }
        if (out) *out = st;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Threaded replica of ref_walk_trace: the reference's own run_walk for every (walker,
// restart) of [walker_begin, walker_end), walkers spread over `threads` std::threads (a
// walker's restarts stay on one thread, in order, on its own Rng stream and Bloom filter:
// walker_loop, saw.cpp:196-214).  Each walk's raw emissions are kept, then replayed in
// (walker, restart, emission) order through the reference DedupSink, so the candidate list
// is the --threads 1 list of run_saw_pool (walks are independent without quota / time /
// stop); per-walk stats carry the delta-eval counts.  Used by bench.py
// for the headline-scale parity diff.
int ref_walk_trace_mt(const lo_saw_config* cfg, int threads, lo_candidate_fn cand,
                      lo_walk_fn walkcb, void* user, lo_pool_stats* out) {
    try {
        SawConfig sc = to_saw(cfg, 1);
        sc.validate();
        if (sc.max_restarts <= 0 || sc.time_budget_s > 0 || sc.candidate_quota > 0 ||
            sc.stop_at_energy > 0)
            throw std::invalid_argument("walk_trace_mt: needs independent walks");
        const int p = sc.effective_prefix_len();
        std::vector<PartitionPrefix> prefixes;
        if (p == 0) prefixes.push_back(PartitionPrefix{{}, 0});
        else prefixes = rank_prefixes(p);
        const int w0 = cfg->walker_begin > 0 ? cfg->walker_begin : 0;
        const int w1 = cfg->walker_end > 0 && cfg->walker_end < sc.walkers ? cfg->walker_end
                                                                            : sc.walkers;
        struct Walk {
            std::vector<Candidate> cands;
            WalkStats ws;
            long long misses = 0;
        };
        const long long R = sc.max_restarts;
        const int nw = std::max(0, w1 - w0);
        std::vector<Walk> walks(static_cast<std::size_t>(nw) * static_cast<std::size_t>(R));
        std::atomic<int> next{0};
        auto job = [&]() {
            class Keep final : public CandidateSink {
            public:
                std::vector<Candidate>* out = nullptr;
                void emit(const Candidate& c) override { out->push_back(c); }
            } keep;
            for (int i = next++; i < nw; i = next++) {
                const int w = w0 + i;
                const std::size_t cls = static_cast<std::size_t>(w) % prefixes.size();
                Rng rng(sc.seed, static_cast<std::uint64_t>(w));
                CountingVisited visited(static_cast<std::size_t>(sc.effective_iterations()) + 1,
                                        sc.bloom_fpr);
                for (long long r = 0; r < R; ++r) {
                    Walk& wk = walks[static_cast<std::size_t>(i) * R + r];
                    keep.out = &wk.cands;
                    const long long m0 = visited.misses;
                    wk.ws = run_walk(sc, prefixes[cls], rng, visited, keep);
                    wk.misses = visited.misses - m0;
                }
            }
        };
        std::vector<std::thread> th;
        for (int t = 0; t < (threads > 0 ? threads : 1); ++t) th.emplace_back(job);
        for (auto& t : th) t.join();
        CallbackSink user_sink(cand, user);
        class Count final : public CandidateSink {
        public:
            explicit Count(CandidateSink& in) : inner(in) {}
            void emit(const Candidate& c) override {
                ++n;
                inner.emit(c);
            }
            CandidateSink& inner;
            long long n = 0;
        } counted(user_sink);
        DedupSink dedup(counted);
        lo_pool_stats st;
        std::memset(&st, 0, sizeof st);
        bool best_set = false;
        for (int i = 0; i < nw; ++i)
            for (long long r = 0; r < R; ++r) {
                const Walk& wk = walks[static_cast<std::size_t>(i) * R + r];
                user_sink.walker = w0 + i;
                user_sink.restart = r;
                for (const Candidate& c : wk.cands) dedup.emit(c);
                ++st.walks;
                st.iterations += wk.ws.iterations;
                st.delta_evals += wk.misses;
                st.exhausted_walks += wk.ws.neighbourhood_exhausted ? 1 : 0;
                if (walkcb)
                    walkcb(user, w0 + i, r, wk.ws.iterations, wk.ws.emitted, wk.ws.best_energy,
                           wk.misses, wk.ws.neighbourhood_exhausted ? 1 : 0, 0);
                if (!best_set || wk.ws.best_energy < st.best_energy) {
                    st.best_energy = wk.ws.best_energy;
                    best_set = true;
                }
            }
        st.emitted = counted.n;
        if (out) *out = st;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Counting-only, multi-threaded walker_loop replica: the number of
// skew_flip_delta_fast calls (unvisited free neighbours, saw.cpp:109-113) and
// iterations of the pool's walks, with `threads` std::threads striding walkers
// like run_saw_pool (saw.cpp:242-257).  Used to size the CPU baseline sample.
int ref_count_deltas(const lo_saw_config* cfg, int threads, lo_pool_stats* out) {
    try {
        SawConfig sc = to_saw(cfg, 1);
        sc.validate();
        const int p = sc.effective_prefix_len();
        std::vector<PartitionPrefix> prefixes;
        if (p == 0) prefixes.push_back(PartitionPrefix{{}, 0});
        else prefixes = rank_prefixes(p);
        const int w0 = cfg->walker_begin > 0 ? cfg->walker_begin : 0;
        const int w1 = cfg->walker_end > 0 && cfg->walker_end < sc.walkers ? cfg->walker_end
                                                                            : sc.walkers;
        std::atomic<long long> walks{0}, iters{0}, deltas{0};
        std::atomic<int> next{w0};
        auto job = [&]() {
            class NullSink final : public CandidateSink {
            public:
                void emit(const Candidate&) override {}
            } sink;
            for (int w = next++; w < w1; w = next++) {
                const std::size_t cls = static_cast<std::size_t>(w) % prefixes.size();
                Rng rng(sc.seed, static_cast<std::uint64_t>(w));
                CountingVisited visited(static_cast<std::size_t>(sc.effective_iterations()) + 1,
                                        sc.bloom_fpr);
                for (long long r = 0; r < sc.max_restarts; ++r) {
                    const WalkStats ws = run_walk(sc, prefixes[cls], rng, visited, sink);
                    ++walks;
                    iters += ws.iterations;
                }
                deltas += visited.misses;
            }
        };
        std::vector<std::thread> th;
        for (int t = 0; t < (threads > 0 ? threads : 1); ++t) th.emplace_back(job);
        for (auto& t : th) t.join();
        if (out) {
            std::memset(out, 0, sizeof *out);
            out->walks = walks;
            out->iterations = iters;
            out->delta_evals = deltas;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int64_t ref_skew_flip_delta_fast(const int8_t* signs, int n, int hp) {
    BinarySequence seq(std::vector<Sign>(signs, signs + n));
    CorrelationState st(seq);
    return skew_flip_delta_fast(seq, st, hp);
}

int64_t ref_skew_flip_delta(const int8_t* signs, int n, int hp) {
    BinarySequence seq(std::vector<Sign>(signs, signs + n));
    CorrelationState st(seq);
    return skew_flip_delta(seq, st, hp);
}

// applies the skew flip; writes the new signs, C_1..C_{n-1} and returns the new E
int64_t ref_apply_skew_flip(int8_t* signs, int n, int hp, int64_t* corr) {
    BinarySequence seq(std::vector<Sign>(signs, signs + n));
    CorrelationState st(seq);
    apply_skew_flip(seq, st, hp);
    for (int i = 0; i < n; ++i) signs[i] = seq[i];
    if (corr)
        for (int k = 0; k < n; ++k) corr[k] = st.correlation(k);
    return st.energy();
}

int64_t ref_energy(const int8_t* signs, int n) {
    return autocorrelation(BinarySequence(std::vector<Sign>(signs, signs + n))).energy();
}

void ref_expand_skew(const int8_t* half, int kp1, int8_t* full) {
    const auto s = expand_skew(SkewHalf(std::vector<Sign>(half, half + kp1)));
    for (int i = 0; i < s.length(); ++i) full[i] = s[i];
}

int64_t ref_energy_threshold(int length, double f) { return energy_threshold_for_merit(length, f); }

void ref_bloom_size(uint64_t capacity, double fpr, uint64_t* bits, int* k) {
    const auto bf = BloomFilter::with_capacity(capacity, fpr);
    *bits = bf.bit_count();
    *k = bf.hash_count();
}

long long ref_effective_iterations(int length, long long max_it, double mult) {
    SawConfig c;
    c.length = length;
    c.max_iterations = max_it;
    c.ti_multiplier = mult;
    return c.effective_iterations();
}

int ref_rank_prefixes(int p, int8_t* out) {
    const auto v = rank_prefixes(p);
    for (std::size_t i = 0; i < v.size(); ++i)
        for (int j = 0; j < p; ++j) out[i * static_cast<std::size_t>(p) + j] = v[i].signs[j];
    return static_cast<int>(v.size());
}

uint64_t ref_canonical_hash(const int8_t* signs, int n, int table) {
    return BinarySequence(std::vector<Sign>(signs, signs + n)).canonical_hash(table);
}

uint64_t ref_flip_mask(int pos, int table) { return TabulationHash::instance().flip_mask(pos, table); }

void ref_rng_draws(uint64_t seed, uint64_t stream, int n, uint64_t* out) {
    Rng r(seed, stream);
    for (int i = 0; i < n; ++i) out[i] = r.next_u64();
}

int64_t ref_oracle_skew_exhaustive(int length, int8_t* best) {
    const auto r = oracle_skew_exhaustive(length);
    if (best)
        for (int i = 0; i < length; ++i) best[i] = r.sequence[i];
    return r.energy;
}

int ref_format_record(const int8_t* signs, int n, int64_t energy, char* out, int cap) {
    Candidate c{BinarySequence(std::vector<Sign>(signs, signs + n)), energy, Origin::saw, {}};
    const std::string s = format_record(c);
    std::snprintf(out, static_cast<std::size_t>(cap), "%s", s.c_str());
    return static_cast<int>(s.size());
}

// Bloom determinism probe: insert n (h1,h2) pairs, return the word array
int ref_bloom_words(uint64_t capacity, double fpr, const uint64_t* keys, int n, uint64_t* words,
                    int max_words) {
    auto bf = BloomFilter::with_capacity(capacity, fpr);
    for (int i = 0; i < n; ++i) bf.insert(keys[2 * i], keys[2 * i + 1]);
    const auto& w = bf.words();
    const int cnt = static_cast<int>(w.size()) < max_words ? static_cast<int>(w.size()) : max_words;
    for (int i = 0; i < cnt; ++i) words[i] = w[static_cast<std::size_t>(i)];
    return static_cast<int>(w.size());
}

} // extern "C"
