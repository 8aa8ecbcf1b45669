// cli_args.hpp -- CLI11-compatible option parsing shared by the `labs` driver and the
// integration build's `labs_solve` (reference flag surface, labs_main.cpp:53-169).
#pragma once
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace labs_cli {

inline int default_threads() {  // labs_main.cpp:21-28
    if (const char* env = std::getenv("LABS_THREADS")) {
        const int n = std::atoi(env);
        if (n >= 1) return n;
    }
    const unsigned hc = std::thread::hardware_concurrency();
    return hc ? static_cast<int>(hc) : 1;
}

// Minimal CLI11-compatible option parsing: --opt v, --opt=v, -L v, -Lv, flags.
class Args {
public:
    Args(int argc, char** argv, int first) {
        for (int i = first; i < argc; ++i) toks_.emplace_back(argv[i]);
    }
    // returns false and sets error on malformed input
    // Options named in `multi` take every following non-option token (CLI11 vector
    // options, e.g. solve's `--length 25 27`); values are joined with ','.
    bool parse(const std::map<std::string, std::string*>& opts,
               const std::map<std::string, bool*>& flags, std::string& err,
               const std::vector<std::string>& multi = {}) {
        for (size_t i = 0; i < toks_.size(); ++i) {
            std::string t = toks_[i], val;
            bool has_val = false;
            if (t.rfind("--", 0) == 0) {
                const auto eq = t.find('=');
                if (eq != std::string::npos) {
                    val = t.substr(eq + 1);
                    t = t.substr(0, eq);
                    has_val = true;
                }
            } else if (t.size() > 2 && t[0] == '-' && t[1] != '-') {
                val = t.substr(2);
                if (!val.empty() && val[0] == '=') val = val.substr(1);
                t = t.substr(0, 2);
                has_val = true;
            }
            auto f = flags.find(t);
            if (f != flags.end()) {
                *f->second = true;
                continue;
            }
            auto o = opts.find(t);
            if (o == opts.end()) {
                err = "The following argument was not expected: " + toks_[i];
                return false;
            }
            if (!has_val) {
                if (i + 1 >= toks_.size()) {
                    err = t + " requires an argument";
                    return false;
                }
                val = toks_[++i];
            }
            bool is_multi = false;
            for (const auto& mname : multi) is_multi = is_multi || mname == o->first;
            if (is_multi) {
                while (i + 1 < toks_.size() && !toks_[i + 1].empty() && toks_[i + 1][0] != '-')
                    val += "," + toks_[++i];
                if (!o->second->empty()) val = *o->second + "," + val;
            }
            *o->second = val;
        }
        return true;
    }

private:
    std::vector<std::string> toks_;
};

inline long long to_ll(const std::string& s, const char* name) {
    char* end = nullptr;
    const long long v = std::strtoll(s.c_str(), &end, 10);
    if (s.empty() || *end) throw std::invalid_argument(std::string(name) + ": not an integer: " + s);
    return v;
}
inline double to_d(const std::string& s, const char* name) {
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (s.empty() || *end) throw std::invalid_argument(std::string(name) + ": not a number: " + s);
    return v;
}


}  // namespace labs_cli
