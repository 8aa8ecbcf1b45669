// labs_solve -- the reference's Step-1 callers built against the reference pipeline with
// the B200 Step 1 linked in (run_saw_pool_b200.cpp):
//   solve      `labs solve` (tools/labs_main.cpp:71-92,174-181): best records on stdout
//              ("L=.. E=.. F=.. hex=.. origin=.."), the summary line on stderr;
//   experiment `labs experiment` (labs_main.cpp:158-169,292-302): walks-only vs dual-step
//              comparison, experiment_compare (pipeline.cpp:390-438), two pools per run;
//   verify     `labs verify` (labs_main.cpp:153-156,276-290): verify_records
//              (pipeline.cpp:335-388) over record files, e.g. GPU-written candidate TSVs.
// Step 2 (priority-queue refinement, pq.cpp) and the pipeline stay the reference's C++.
// Flag surfaces and outputs are the reference's.
#include <cstdio>
#include <fstream>
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

// add_saw_options (labs_main.cpp:53-62)
void apply_saw_options(std::map<std::string, std::string>& v, labsearch::SawConfig& saw) {
    using labs_cli::to_d;
    using labs_cli::to_ll;
    if (!v["--walkers"].empty()) saw.walkers = static_cast<int>(to_ll(v["--walkers"], "--walkers"));
    if (!v["--p"].empty()) saw.prefix_len = static_cast<int>(to_ll(v["--p"], "--p"));
    if (!v["--ti"].empty()) saw.max_iterations = to_ll(v["--ti"], "--ti");
    if (!v["--ti-mult"].empty()) saw.ti_multiplier = to_d(v["--ti-mult"], "--ti-mult");
    if (!v["--el"].empty()) saw.energy_threshold = to_ll(v["--el"], "--el");
    if (!v["--target-f"].empty()) saw.target_merit = to_d(v["--target-f"], "--target-f");
    if (!v["--restarts"].empty()) saw.max_restarts = to_ll(v["--restarts"], "--restarts");
    if (!v["--bloom-fpr"].empty()) saw.bloom_fpr = to_d(v["--bloom-fpr"], "--bloom-fpr");
}

int verify_main(int argc, char** argv) {  // labs_main.cpp:276-290
    if (argc < 3) {
        std::cerr << "files is required\nRun with --help for more information.\n";
        return 106;
    }
    try {
        bool all_clean = true;
        for (int i = 2; i < argc; ++i) {
            const std::string path = argv[i];
            const auto report = labsearch::verify_records(path);
            std::cout << path << ": " << report.records_checked << " records, "
                      << report.mismatches.size() << " mismatches, " << report.malformed.size()
                      << " malformed\n";
            for (const auto& m : report.malformed)
                std::cout << "  malformed line " << m.line << ": " << m.what << '\n';
            for (const auto& m : report.mismatches)
                std::cout << "  mismatch line " << m.line << ": " << m.what << '\n';
            all_clean = all_clean && report.clean();
        }
        return all_clean ? 0 : 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}

int experiment_main(int argc, char** argv) {  // labs_main.cpp:158-169, 292-302
    using labs_cli::to_ll;
    labsearch::ExperimentConfig exp;  // (saw.threads keeps its default, as in the reference)
    std::map<std::string, std::string> v;
    const char* names[] = {"--length", "--runs", "--walkers", "--p", "--ti", "--ti-mult", "--el",
                           "--target-f", "--restarts", "--bloom-fpr", "--tu", "--tr",
                           "--refine-top", "--seed", "--out"};
    std::map<std::string, std::string*> opts;
    for (const char* n : names) opts[n] = &v[n];
    opts["-L"] = &v["--length"];
    std::map<std::string, bool*> flags;
    labs_cli::Args a(argc, argv, 2);
    std::string err;
    if (!a.parse(opts, flags, err)) {
        std::cerr << err << "\nRun with --help for more information.\n";
        return 109;
    }
    try {
        if (v["--length"].empty()) {
            std::cerr << "--length is required\nRun with --help for more information.\n";
            return 106;
        }
        exp.length = static_cast<int>(to_ll(v["--length"], "--length"));
        if (!v["--runs"].empty()) exp.runs = static_cast<int>(to_ll(v["--runs"], "--runs"));
        apply_saw_options(v, exp.saw);
        if (!v["--tu"].empty()) exp.pq.max_stale_pivots = to_ll(v["--tu"], "--tu");
        if (!v["--tr"].empty()) exp.pq.max_rotation = static_cast<int>(to_ll(v["--tr"], "--tr"));
        if (!v["--refine-top"].empty())
            exp.refine_top = static_cast<int>(to_ll(v["--refine-top"], "--refine-top"));
        if (!v["--seed"].empty()) exp.seed = static_cast<std::uint64_t>(to_ll(v["--seed"], "--seed"));
        const auto result = labsearch::experiment_compare(exp);
        std::cout << "arm A (saw only)  median best E = " << result.median_saw << '\n'
                  << "arm B (dual step) median best E = " << result.median_dual << '\n'
                  << "rank-sum z = " << result.test.z << ", two-sided p = " << result.test.p_value
                  << '\n';
        if (!v["--out"].empty()) {
            std::ofstream out(v["--out"]);
            out << labsearch::experiment_csv(result);
        }
        return 0;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}

int main(int argc, char** argv) {
    using labs_cli::to_d;
    using labs_cli::to_ll;
    const std::string cmd = argc >= 2 ? argv[1] : "";
    if (cmd == "verify") return verify_main(argc, argv);
    if (cmd == "experiment") return experiment_main(argc, argv);
    if (cmd != "solve") {
        std::cerr << "usage: labs_solve solve|experiment|verify [reference flags]\n";
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
        apply_saw_options(v, run.saw);
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
