// labs_solve -- the reference's `labs solve` (tools/labs_main.cpp:71-92,174-181) built
// against the reference pipeline with the B200 Step 1 linked in (run_saw_pool_b200.cpp).
// Step 2 (priority-queue refinement, pq.cpp) and the pipeline stay the reference's C++.
// Flag surface and output are the reference's: best records on stdout
// ("L=.. E=.. F=.. hex=.. origin=.."), the summary line on stderr.
#include <cstdio>
#include <iostream>
#include <map>
#include <sstream>
#include <string>

#include "cli_args.hpp"
#include "labs/hex_codec.hpp"
#include "labs/pipeline.hpp"

namespace {

void print_record(const labsearch::Candidate& c) {  // labs_main.cpp:45-51
    std::cout << "L=" << c.seq.length() << "  E=" << c.energy;
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.4f", c.merit());
    std::cout << "  F=" << buf << "  hex=" << labsearch::hex_encode(c.seq)
              << "  origin=" << labsearch::origin_name(c.origin) << '\n';
}

}  // namespace

int main(int argc, char** argv) {
    using labs_cli::to_d;
    using labs_cli::to_ll;
    if (argc < 2 || std::string(argv[1]) != "solve") {
        std::cerr << "usage: labs_solve solve -L <len...> [reference solve flags]\n";
        return 109;
    }
    labsearch::RunConfig run;
    run.threads = labs_cli::default_threads();
    std::map<std::string, std::string> v;
    const char* names[] = {"--length", "--walkers", "--p", "--ti", "--ti-mult", "--el",
                           "--target-f", "--restarts", "--bloom-fpr", "--tu", "--tr",
                           "--capacity", "--seconds", "--rounds", "--refine-top",
                           "--construction-seeds", "--stop-at-merit", "--seed", "--threads",
                           "--out", "--candidates", "--log"};
    std::map<std::string, std::string*> opts;
    for (const char* n : names) opts[n] = &v[n];
    opts["-L"] = &v["--length"];
    bool no_construct = false, deterministic = false;
    std::map<std::string, bool*> flags{{"--no-construct", &no_construct},
                                       {"--deterministic", &deterministic}};
    labs_cli::Args a(argc, argv, 2);
    std::string err;
    if (!a.parse(opts, flags, err, {"--length", "-L"})) {
        std::cerr << err << "\nRun with --help for more information.\n";
        return 109;
    }
    try {
        if (v["--length"].empty()) {
            std::cerr << "--length is required\nRun with --help for more information.\n";
            return 106;
        }
        std::stringstream ls(v["--length"]);
        for (std::string tok; std::getline(ls, tok, ',');)
            run.lengths.push_back(static_cast<int>(to_ll(tok, "--length")));
        auto& saw = run.saw;  // add_saw_options (labs_main.cpp:53-62)
        if (!v["--walkers"].empty()) saw.walkers = static_cast<int>(to_ll(v["--walkers"], "--walkers"));
        if (!v["--p"].empty()) saw.prefix_len = static_cast<int>(to_ll(v["--p"], "--p"));
        if (!v["--ti"].empty()) saw.max_iterations = to_ll(v["--ti"], "--ti");
        if (!v["--ti-mult"].empty()) saw.ti_multiplier = to_d(v["--ti-mult"], "--ti-mult");
        if (!v["--el"].empty()) saw.energy_threshold = to_ll(v["--el"], "--el");
        if (!v["--target-f"].empty()) saw.target_merit = to_d(v["--target-f"], "--target-f");
        if (!v["--restarts"].empty()) saw.max_restarts = to_ll(v["--restarts"], "--restarts");
        if (!v["--bloom-fpr"].empty()) saw.bloom_fpr = to_d(v["--bloom-fpr"], "--bloom-fpr");
        if (!v["--tu"].empty()) run.pq.max_stale_pivots = to_ll(v["--tu"], "--tu");
        if (!v["--tr"].empty()) run.pq.max_rotation = static_cast<int>(to_ll(v["--tr"], "--tr"));
        if (!v["--capacity"].empty())
            run.pq.queue_capacity = static_cast<std::size_t>(to_ll(v["--capacity"], "--capacity"));
        if (!v["--seconds"].empty()) run.time_budget_s = to_d(v["--seconds"], "--seconds");
        if (!v["--rounds"].empty()) run.rounds = static_cast<int>(to_ll(v["--rounds"], "--rounds"));
        if (!v["--refine-top"].empty())
            run.refine_top = static_cast<int>(to_ll(v["--refine-top"], "--refine-top"));
        if (!v["--construction-seeds"].empty())
            run.construction_seeds =
                static_cast<int>(to_ll(v["--construction-seeds"], "--construction-seeds"));
        if (!v["--stop-at-merit"].empty())
            run.stop_at_merit = to_d(v["--stop-at-merit"], "--stop-at-merit");
        if (!v["--seed"].empty()) run.seed = static_cast<std::uint64_t>(to_ll(v["--seed"], "--seed"));
        if (!v["--threads"].empty()) run.threads = static_cast<int>(to_ll(v["--threads"], "--threads"));
        run.use_construction = !no_construct;
        run.deterministic = deterministic;
        run.results_path = v["--out"];
        run.candidates_path = v["--candidates"];
        run.log_path = v["--log"];

        const auto result = labsearch::run_pipeline(run);
        for (const auto& [l, rec] : result.best) print_record(rec.candidate);
        std::cerr << "walks=" << result.saw_stats.walks << " candidates=" << result.candidates
                  << " refine_calls=" << result.refine_calls << " wall=" << result.wall_seconds
                  << "s fingerprint=" << result.fingerprint << '\n';
        return 0;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
