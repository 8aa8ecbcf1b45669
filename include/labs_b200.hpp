// labs_b200.hpp -- header-only C++ adapter over the C ABI (labs_gpu.h) with the
// reference's Step-1 types and signature:
//     labs_b200::PoolStats labs_b200::run_saw_pool(const SawConfig&, CandidateSink&)
// mirroring /root/reference/proj/include/labs/saw.hpp:34-61,161-172 and
// candidate.hpp:21-99.  A maintainer drops the GPU path into the reference by
// making labsearch::run_saw_pool (saw.cpp:218) forward to labs_saw_pool_run; see
// INTEGRATION.md.  Errors are rethrown as the reference's exception types.
#pragma once

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "labs_gpu.h"

namespace labs_b200 {

using Sign = std::int8_t;
using Energy = std::int64_t;

struct SawConfig {                     // saw.hpp:34-61
    int length = 0;
    int prefix_len = -1;
    int walkers = 1;
    long long max_iterations = 0;
    double ti_multiplier = 8.0;
    Energy energy_threshold = 0;
    double target_merit = 0.0;
    double bloom_fpr = 1e-4;
    std::uint64_t seed = 1;
    int threads = 1;
    long long max_restarts = 1;
    double time_budget_s = 0.0;
    long long candidate_quota = 0;
    Energy stop_at_energy = 0;
    bool debug_check_energy = false;
    // additive GPU controls
    int gpus = 1;
    int device = 0;
    int shard_index = 0;
    int shard_count = 1;
    bool count_visited = false;

    labs_saw_config to_c() const {
        labs_saw_config c{};
        c.length = length;
        c.prefix_len = prefix_len;
        c.walkers = walkers;
        c.threads = threads;
        c.max_iterations = max_iterations;
        c.ti_multiplier = ti_multiplier;
        c.energy_threshold = energy_threshold;
        c.target_merit = target_merit;
        c.bloom_fpr = bloom_fpr;
        c.seed = seed;
        c.max_restarts = max_restarts;
        c.time_budget_s = time_budget_s;
        c.candidate_quota = candidate_quota;
        c.stop_at_energy = stop_at_energy;
        c.debug_check_energy = debug_check_energy ? 1 : 0;
        c.n_gpus = gpus;
        c.device = device;
        c.shard_index = shard_index;
        c.shard_count = shard_count;
        c.count_visited = count_visited ? 1 : 0;
        return c;
    }
};

struct Candidate {                     // candidate.hpp:21-29
    std::vector<Sign> seq;
    Energy energy = 0;
    std::vector<Sign> prefix;
    long long walker = -1, restart = -1, iteration = -1;
    double merit() const {
        const double n = static_cast<double>(seq.size());
        return n * n / (2.0 * static_cast<double>(energy));
    }
    std::uint64_t hash() const {
        return labs_canonical_hash(seq.data(), static_cast<int32_t>(seq.size()), 0);
    }
};

class CandidateSink {                  // candidate.hpp:56-60
public:
    virtual ~CandidateSink() = default;
    virtual void emit(const Candidate& c) = 0;
};

class CollectingSink final : public CandidateSink {  // candidate.hpp:62-80
public:
    void emit(const Candidate& c) override {
        std::lock_guard<std::mutex> lock(mu_);
        items_.push_back(c);
    }
    std::vector<Candidate> take() {
        std::lock_guard<std::mutex> lock(mu_);
        return std::move(items_);
    }
    std::size_t size() const {
        std::lock_guard<std::mutex> lock(mu_);
        return items_.size();
    }

private:
    mutable std::mutex mu_;
    std::vector<Candidate> items_;
};

struct PoolStats {                     // saw.hpp:161-167 + GPU counters
    long long walks = 0;
    long long iterations = 0;
    long long emitted = 0;
    Energy best_energy = 0;
    double wall_seconds = 0.0;
    labs_pool_stats gpu{};
};

inline std::string format_record(const Candidate& c) {  // candidate.cpp:36-49
    std::vector<char> buf(c.seq.size() + 128);
    labs_format_record(c.seq.data(), static_cast<int32_t>(c.seq.size()), c.energy, buf.data(),
                       static_cast<int32_t>(buf.size()));
    return std::string(buf.data());
}

inline void throw_status(int rc) {
    const std::string msg = labs_last_error();
    switch (rc) {
        case LABS_EINVAL: throw std::invalid_argument(msg);
        case LABS_ERANGE: throw std::out_of_range(msg);
        case LABS_ELOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

// Device setup ahead of run_saw_pool (labs_saw_prepare): keeps it out of a time budget.
inline void prepare_saw_pool(const SawConfig& config) {
    const labs_saw_config c = config.to_c();
    const int rc = labs_saw_prepare(&c);
    if (rc != LABS_OK) throw_status(rc);
}

inline PoolStats run_saw_pool(const SawConfig& config, CandidateSink& sink) {  // saw.cpp:218
    struct Ctx {
        CandidateSink* sink;
        std::string error;
    } ctx{&sink, {}};
    const labs_saw_config c = config.to_c();
    labs_pool_stats st{};
    const int rc = labs_saw_pool_run(
        &c,
        [](void* user, const labs_candidate* lc) -> int {
            auto* cx = static_cast<Ctx*>(user);
            try {
                Candidate cand;
                cand.seq.assign(lc->signs, lc->signs + lc->length);
                cand.energy = lc->energy;
                if (lc->prefix_len > 0) cand.prefix.assign(lc->prefix, lc->prefix + lc->prefix_len);
                cand.walker = lc->walker;
                cand.restart = lc->restart;
                cand.iteration = lc->iteration;
                cx->sink->emit(cand);
                return 0;
            } catch (const std::exception& e) {
                cx->error = e.what();
                return 1;
            }
        },
        &ctx, &st);
    if (!ctx.error.empty()) throw std::runtime_error(ctx.error);
    if (rc != LABS_OK) throw_status(rc);
    PoolStats out;
    out.walks = st.walks;
    out.iterations = st.iterations;
    out.emitted = st.emitted;
    out.best_energy = st.best_energy;
    out.wall_seconds = st.wall_seconds;
    out.gpu = st;
    return out;
}

}  // namespace labs_b200
