// run_saw_pool_b200.cpp -- the drop-in: labsearch::run_saw_pool (saw.hpp:172,
// saw.cpp:218-267) implemented over the B200 engine's C ABI (include/labs_gpu.h).
//
// The integration build (integration/Makefile) compiles the reference library from its
// own sources with the reference's CPU definition renamed (-Drun_saw_pool=...), so every
// reference caller -- run_pipeline Step 1 (pipeline.cpp:287), experiment_compare
// (pipeline.cpp:403,412) -- reaches this function instead.  This is the patch of
// INTEGRATION.md §1, applied at link time without touching the reference sources.
#include <cstdlib>
#include <exception>
#include <stdexcept>
#include <vector>

#include "labs/candidate.hpp"
#include "labs/saw.hpp"
#include "labs_gpu.h"

namespace labsearch {

PoolStats run_saw_pool(const SawConfig& config, CandidateSink& sink) {
    config.validate();  // the reference's exceptions, before any device work (saw.cpp:219)
    labs_saw_config c{};
    c.length = config.length;
    c.prefix_len = config.prefix_len;
    c.walkers = config.walkers;
    c.threads = config.threads;
    c.max_iterations = config.max_iterations;
    c.ti_multiplier = config.ti_multiplier;
    c.energy_threshold = config.energy_threshold;
    c.target_merit = config.target_merit;
    c.bloom_fpr = config.bloom_fpr;
    c.seed = config.seed;
    c.max_restarts = config.max_restarts;
    c.time_budget_s = config.time_budget_s;
    c.candidate_quota = config.candidate_quota;
    c.stop_at_energy = config.stop_at_energy;
    c.debug_check_energy = config.debug_check_energy ? 1 : 0;
    const char* g = std::getenv("LABS_GPUS");
    c.n_gpus = g ? std::atoi(g) : 1;
    struct Ctx {
        CandidateSink* sink;
        std::exception_ptr err;
    } ctx{&sink, nullptr};
    labs_pool_stats st{};
    const int rc = labs_saw_pool_run(
        &c,
        [](void* u, const labs_candidate* lc) -> int {
            auto* cx = static_cast<Ctx*>(u);
            try {
                Candidate cand{BinarySequence(std::vector<Sign>(lc->signs, lc->signs + lc->length)),
                               lc->energy, Origin::saw,
                               std::vector<Sign>(lc->prefix, lc->prefix + lc->prefix_len)};
                cx->sink->emit(cand);
                return 0;
            } catch (...) {
                cx->err = std::current_exception();
                return 1;
            }
        },
        &ctx, &st);
    if (ctx.err) std::rethrow_exception(ctx.err);
    switch (rc) {
        case LABS_OK: break;
        case LABS_EINVAL: throw std::invalid_argument(labs_last_error());
        case LABS_ERANGE: throw std::out_of_range(labs_last_error());
        case LABS_ELOGIC: throw std::logic_error(labs_last_error());
        default: throw std::runtime_error(labs_last_error());
    }
    PoolStats out;
    out.walks = st.walks;
    out.iterations = st.iterations;
    out.emitted = st.emitted;
    out.best_energy = st.best_energy;
    out.wall_seconds = st.wall_seconds;
    return out;
}

}  // namespace labsearch
