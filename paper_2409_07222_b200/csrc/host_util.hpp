// host_util.hpp -- host-side restatements needed around the GPU path: the
// tabulation tables, prefix ranking, config derivation, skew expansion,
// canonical hashing and the candidate record format.  Product code (C++),
// written from the reference's documented behaviour; each item cites the
// reference file:line whose semantics it keeps.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/labs_gpu.h"
#include "saw_device.h"

namespace labs_b200 {

// TabulationHash (rng.hpp:75-101, rng.cpp:10-18): fixed splitmix stream from
// 0x5eed5eed5eed5eed fills t[2][1024][2], then salt[2][1026].
struct TabTables {
    uint64_t t[2][kMaxHalf][2];
    uint64_t salt[2][kMaxHalf + 2];
    static const TabTables& get();
    uint64_t hash(const int8_t* s, int n, int table) const;  // rng.hpp:89-95
};

uint64_t splitmix64(uint64_t& s);                                   // rng.hpp:10-15
int64_t energy_threshold_for_merit(int length, double f);          // sequence.cpp:36-40
int64_t effective_iterations(int length, int64_t max_it, double m); // saw.hpp:51-54
int effective_prefix_len(int prefix_len, int walkers);              // saw.cpp:44-49
void bloom_size(uint64_t capacity, double fpr, uint64_t& bits, int& k);  // bloom.cpp:15-24
// rank_prefixes (saw.cpp:22-42): P x p signs, stable-sorted by prefix self-energy
std::vector<int8_t> rank_prefixes(int p);
void expand_skew(const int8_t* half, int kp1, int8_t* full);       // skew.cpp:14-26
std::string hex_encode(const int8_t* s, int n);                     // hex_codec.cpp:14-30
std::string format_record(const int8_t* s, int n, int64_t energy);  // candidate.cpp:36-49

// Everything the GPU launch needs, derived once per call.
struct Derived {
    int L = 0, k = 0, kp1 = 0, p = 0;
    int64_t t_i = 0, e_l = 0;
    uint64_t bloom_bits = 0;
    int bloom_k = 0;
    int nprefix = 1;                 // 2^(p-1), or 1 when p == 0
    std::vector<int8_t> prefixes;    // nprefix x p
    std::vector<uint32_t> prefix_bits;  // bit i set <=> +1
};

// SawConfig::validate (saw.cpp:51-63) + derivations.  Returns "" or the
// reference's error message.
std::string derive(const labs_saw_config& cfg, Derived& d);

// Geometry of the walk kernel for (L, p, T_i, Bloom).  Returns "" or an error.
std::string make_walk_params(int L, int p, int64_t t_i, int64_t e_l, uint64_t bloom_bits,
                             int bloom_k, WalkParams& wp);

void set_error(const std::string& msg);

}  // namespace labs_b200
