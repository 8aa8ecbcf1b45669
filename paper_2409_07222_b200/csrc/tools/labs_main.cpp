// labs -- command-line driver of the B200 Step-1 engine.
//
// Keeps the reference CLI's `saw` subcommand surface and output byte-for-byte
// (tools/labs_main.cpp:53-62, 95-106, 184-199): the same flags, the stderr
// summary "walks= iterations= emitted= bestE= wall=...s" and TSV records
// (format_record) on stdout or into --out.  GPU controls are additive:
// --gpus N, --device D, --count-visited, --stats-json.
//
// Extension subcommand `enumerate` runs the restriction-class Gray enumeration.
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "cli_args.hpp"
#include "labs_b200.hpp"

namespace {
using labs_cli::Args;
using labs_cli::default_threads;
using labs_cli::to_d;
using labs_cli::to_ll;

class FileSink final : public labs_b200::CandidateSink {  // labs_main.cpp:30-43
public:
    explicit FileSink(const std::string& path) : out_(path) {
        if (!out_) throw std::runtime_error("cannot open output file: " + path);
    }
    void emit(const labs_b200::Candidate& c) override { out_ << labs_b200::format_record(c) << '\n'; }

private:
    std::ofstream out_;
};

int cmd_saw(int argc, char** argv) {
    labs_b200::SawConfig saw;
    saw.threads = default_threads();
    std::map<std::string, std::string> v;
    const char* names[] = {"--length", "--walkers", "--p", "--ti", "--ti-mult", "--el",
                           "--target-f", "--restarts", "--bloom-fpr", "--seconds", "--quota",
                           "--stop-at-energy", "--seed", "--threads", "--out", "--gpus",
                           "--device", "--stats-json"};
    std::map<std::string, std::string*> opts;
    for (const char* n : names) opts[n] = &v[n];
    opts["-L"] = &v["--length"];
    bool count_visited = false, help = false;
    std::map<std::string, bool*> flags{{"--count-visited", &count_visited}, {"--help", &help},
                                       {"-h", &help}};
    Args a(argc, argv, 2);
    std::string err;
    if (!a.parse(opts, flags, err)) {
        std::cerr << err << "\nRun with --help for more information.\n";
        return 109;
    }
    if (help) {
        std::cout << "labs saw -L <odd L> [--walkers N] [--p P] [--ti T] [--ti-mult M] [--el E] "
                     "[--target-f F] [--restarts R] [--bloom-fpr X] [--seconds S] [--quota Q] "
                     "[--stop-at-energy E] [--seed S] [--threads N] [--out FILE] [--gpus N] "
                     "[--device D] [--count-visited] [--stats-json FILE]\n";
        return 0;
    }
    if (v["--length"].empty()) {
        std::cerr << "--length is required\nRun with --help for more information.\n";
        return 106;
    }
    saw.length = static_cast<int>(to_ll(v["--length"], "--length"));
    if (!v["--walkers"].empty()) saw.walkers = static_cast<int>(to_ll(v["--walkers"], "--walkers"));
    if (!v["--p"].empty()) saw.prefix_len = static_cast<int>(to_ll(v["--p"], "--p"));
    if (!v["--ti"].empty()) saw.max_iterations = to_ll(v["--ti"], "--ti");
    if (!v["--ti-mult"].empty()) saw.ti_multiplier = to_d(v["--ti-mult"], "--ti-mult");
    if (!v["--el"].empty()) saw.energy_threshold = to_ll(v["--el"], "--el");
    if (!v["--target-f"].empty()) saw.target_merit = to_d(v["--target-f"], "--target-f");
    if (!v["--restarts"].empty()) saw.max_restarts = to_ll(v["--restarts"], "--restarts");
    if (!v["--bloom-fpr"].empty()) saw.bloom_fpr = to_d(v["--bloom-fpr"], "--bloom-fpr");
    if (!v["--seconds"].empty()) saw.time_budget_s = to_d(v["--seconds"], "--seconds");
    if (!v["--quota"].empty()) saw.candidate_quota = to_ll(v["--quota"], "--quota");
    if (!v["--stop-at-energy"].empty())
        saw.stop_at_energy = to_ll(v["--stop-at-energy"], "--stop-at-energy");
    if (!v["--seed"].empty()) saw.seed = static_cast<std::uint64_t>(to_ll(v["--seed"], "--seed"));
    if (!v["--threads"].empty()) saw.threads = static_cast<int>(to_ll(v["--threads"], "--threads"));
    if (!v["--gpus"].empty()) saw.gpus = static_cast<int>(to_ll(v["--gpus"], "--gpus"));
    if (!v["--device"].empty()) saw.device = static_cast<int>(to_ll(v["--device"], "--device"));
    saw.count_visited = count_visited;

    labs_b200::CollectingSink collect;  // labs_main.cpp:184-199
    std::unique_ptr<FileSink> file;
    labs_b200::CandidateSink* sink = &collect;
    if (!v["--out"].empty()) {
        file = std::make_unique<FileSink>(v["--out"]);
        sink = file.get();
    }
    labs_b200::prepare_saw_pool(saw);  // (device setup outside the --seconds budget)
    const auto stats = labs_b200::run_saw_pool(saw, *sink);
    std::cerr << "walks=" << stats.walks << " iterations=" << stats.iterations
              << " emitted=" << stats.emitted << " bestE=" << stats.best_energy
              << " wall=" << stats.wall_seconds << "s\n";
    if (v["--out"].empty())
        for (const auto& c : collect.take()) std::cout << labs_b200::format_record(c) << '\n';
    if (!v["--stats-json"].empty()) {
        std::ofstream js(v["--stats-json"]);
        const auto& g = stats.gpu;
        js << "{\"walks\": " << g.walks << ", \"iterations\": " << g.iterations
           << ", \"emitted\": " << g.emitted << ", \"emitted_raw\": " << g.emitted_raw
           << ", \"best_energy\": " << g.best_energy << ", \"delta_evals\": " << g.delta_evals
           << ", \"delta_evals_computed\": " << g.delta_evals_computed
           << ", \"kernel_ms\": " << g.kernel_ms << ", \"seed_ms\": " << g.seed_ms
           << ", \"wall_seconds\": " << g.wall_seconds << ", \"n_gpus\": " << g.n_gpus << "}\n";
    }
    return 0;
}

int cmd_enumerate(int argc, char** argv) {
    std::map<std::string, std::string> v;
    std::map<std::string, std::string*> opts;
    for (const char* n : {"--length", "--p", "--class", "--free", "--el", "--target-f", "--out"})
        opts[n] = &v[n];
    opts["-L"] = &v["--length"];
    std::map<std::string, bool*> flags;
    Args a(argc, argv, 2);
    std::string err;
    if (!a.parse(opts, flags, err)) {
        std::cerr << err << '\n';
        return 109;
    }
    const int L = static_cast<int>(to_ll(v["--length"], "--length"));
    const int p = static_cast<int>(to_ll(v["--p"].empty() ? "12" : v["--p"], "--p"));
    const int cls = static_cast<int>(to_ll(v["--class"].empty() ? "0" : v["--class"], "--class"));
    const int m = static_cast<int>(to_ll(v["--free"], "--free"));
    long long el = v["--el"].empty() ? 0 : to_ll(v["--el"], "--el");
    if (!v["--target-f"].empty()) {
        const double f = to_d(v["--target-f"], "--target-f");
        el = static_cast<long long>(static_cast<double>(L) * L / (2.0 * f));
    }
    // Hits go out as candidate records (candidate.cpp:36-49), like `saw`: the half is the
    // class prefix, then Gray(g) over positions [p, p+m) (bit set <=> -1), +1 elsewhere.
    const int kp1 = (L + 1) / 2;
    if (p < 1 || p > 30 || cls < 0 || cls >= (1 << (p - 1)) || m < 0 || p + m > kp1) {
        std::cerr << "error: enumerate: bad --p / --class / --free for this length\n";
        return 1;
    }
    std::vector<int8_t> prefixes((static_cast<size_t>(1) << (p - 1)) * static_cast<size_t>(p));
    labs_rank_prefixes(p, prefixes.data());
    struct Ctx {
        std::ostream* out;
        int L, kp1, p, m;
        const int8_t* prefix;
        std::vector<int8_t> half, full;
        std::vector<char> line;
    };
    std::ofstream fo;
    std::ostream* out = &std::cout;
    if (!v["--out"].empty()) {
        fo.open(v["--out"]);
        out = &fo;
    }
    Ctx ctx{out, L, kp1, p, m, &prefixes[static_cast<size_t>(cls) * static_cast<size_t>(p)],
            std::vector<int8_t>(static_cast<size_t>(kp1)), std::vector<int8_t>(static_cast<size_t>(L)),
            std::vector<char>(static_cast<size_t>(L) + 128)};
    labs_enum_stats st{};
    const int rc = labs_enumerate_class(
        L, p, cls, m, el, 0, 1ull << m,
        [](void* u, uint64_t g, int64_t e) -> int {
            auto* c = static_cast<Ctx*>(u);
            const uint64_t gray = g ^ (g >> 1);
            for (int i = 0; i < c->kp1; ++i)
                c->half[static_cast<size_t>(i)] =
                    i < c->p ? c->prefix[i]
                             : ((i < c->p + c->m && ((gray >> (i - c->p)) & 1)) ? int8_t(-1) : int8_t(1));
            labs_expand_skew(c->half.data(), c->kp1, c->full.data());
            labs_format_record(c->full.data(), c->L, e, c->line.data(), static_cast<int32_t>(c->line.size()));
            *c->out << c->line.data() << '\n';
            return 0;
        },
        &ctx, &st);
    if (rc != LABS_OK) labs_b200::throw_status(rc);
    std::cerr << "configurations=" << st.configurations << " emitted=" << st.emitted
              << " bestE=" << st.best_energy << " best_g=" << st.best_g
              << " kernel_ms=" << st.kernel_ms << '\n';
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "A subcommand is required\nRun with --help for more information.\n";
        return 106;
    }
    const std::string sub = argv[1];
    try {
        if (sub == "saw") return cmd_saw(argc, argv);
        if (sub == "enumerate") return cmd_enumerate(argc, argv);
        if (sub == "--help" || sub == "-h") {
            std::cout << "labs {saw, enumerate} ... (B200 Step-1 engine)\n";
            return 0;
        }
        std::cerr << "The following argument was not expected: " << sub << '\n';
        return 109;
    } catch (const std::exception& ex) {  // labs_main.cpp:304-307
        std::cerr << "error: " << ex.what() << '\n';
        return 1;
    }
}
