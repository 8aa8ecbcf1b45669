// host_util.cpp -- see host_util.hpp.
#include "host_util.hpp"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>

namespace labs_b200 {

uint64_t splitmix64(uint64_t& s) {
    s += 0x9e3779b97f4a7c15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

const TabTables& TabTables::get() {
    static const TabTables* inst = [] {
        auto* tt = new TabTables();
        uint64_t sm = 0x5eed5eed5eed5eedULL;
        for (auto& table : tt->t)
            for (auto& pos : table)
                for (auto& v : pos) v = splitmix64(sm);
        for (auto& table : tt->salt)
            for (auto& v : table) v = splitmix64(sm);
        return tt;
    }();
    return *inst;
}

uint64_t TabTables::hash(const int8_t* s, int n, int table) const {
    uint64_t h = salt[table][n];
    for (int i = 0; i < n; ++i) h ^= t[table][i][s[i] > 0 ? 1 : 0];
    return h;
}

int64_t energy_threshold_for_merit(int length, double f) {
    const double l2 = static_cast<double>(length) * length;
    return static_cast<int64_t>(std::floor(l2 / (2.0 * f)));
}

int64_t effective_iterations(int length, int64_t max_it, double mult) {
    if (max_it > 0) return max_it;
    return static_cast<int64_t>(mult * (length + 1) / 2);
}

int effective_prefix_len(int prefix_len, int walkers) {
    if (prefix_len >= 0) return prefix_len;
    int p = 1;
    while ((1 << (p - 1)) < walkers) ++p;
    return p;
}

void bloom_size(uint64_t capacity, double fpr, uint64_t& bits, int& k) {
    if (capacity == 0) capacity = 1;
    const double ln2 = std::log(2.0);
    const double m = -static_cast<double>(capacity) * std::log(fpr) / (ln2 * ln2);
    const auto b = static_cast<uint64_t>(std::ceil(m));
    k = static_cast<int>(std::lround(m / static_cast<double>(capacity) * ln2));
    if (k < 1) k = 1;
    bits = b < 64 ? 64 : b;
}

std::vector<int8_t> rank_prefixes(int p) {
    const uint32_t count = 1u << (p - 1);
    std::vector<std::pair<int64_t, uint32_t>> order(count);
    for (uint32_t code = 0; code < count; ++code) {
        int8_t s[32];
        s[0] = 1;
        for (int j = 1; j < p; ++j) s[j] = ((code >> (j - 1)) & 1) ? -1 : 1;
        int64_t pot = 0;  // prefix_potential (saw.cpp:11-20)
        for (int lag = 1; lag < p; ++lag) {
            int64_t c = 0;
            for (int i = 0; i + lag < p; ++i) c += s[i] * s[i + lag];
            pot += c * c;
        }
        order[code] = {pot, code};
    }
    std::stable_sort(order.begin(), order.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    std::vector<int8_t> out(static_cast<size_t>(count) * p);
    for (uint32_t r = 0; r < count; ++r) {
        const uint32_t code = order[r].second;
        int8_t* s = &out[static_cast<size_t>(r) * p];
        s[0] = 1;
        for (int j = 1; j < p; ++j) s[j] = ((code >> (j - 1)) & 1) ? -1 : 1;
    }
    return out;
}

void expand_skew(const int8_t* half, int kp1, int8_t* full) {
    const int k = kp1 - 1;
    std::copy(half, half + kp1, full);
    for (int i = 1; i <= k; ++i) full[k + i] = (i & 1) ? static_cast<int8_t>(-full[k - i]) : full[k - i];
}

std::string hex_encode(const int8_t* s, int n) {
    static const char* kHex = "0123456789ABCDEF";
    const int digits = (n + 3) / 4;
    const int pad = digits * 4 - n;
    std::string out(static_cast<size_t>(digits), '0');
    for (int d = 0; d < digits; ++d) {
        int v = 0;
        for (int b = 0; b < 4; ++b) {
            const int pos = 4 * d + b - pad;
            v = (v << 1) | ((pos >= 0 && s[pos] > 0) ? 1 : 0);
        }
        out[static_cast<size_t>(d)] = kHex[v];
    }
    return out;
}

std::string format_record(const int8_t* s, int n, int64_t energy) {
    char fbuf[40];
    std::snprintf(fbuf, sizeof fbuf, "%.4f",
                  static_cast<double>(n) * static_cast<double>(n) / (2.0 * static_cast<double>(energy)));
    std::string line = std::to_string(n);
    line += '\t';
    line += std::to_string(energy);
    line += '\t';
    line += fbuf;
    line += '\t';
    line += hex_encode(s, n);
    line += "\tsaw";
    return line;
}

std::string derive(const labs_saw_config& cfg, Derived& d) {
    const int L = cfg.length;
    if (L < 3 || L % 2 == 0) return "saw: length must be odd and >= 3";
    if (cfg.walkers < 1) return "saw: walkers must be >= 1";
    d.e_l = cfg.target_merit > 0.0 ? energy_threshold_for_merit(L, cfg.target_merit)
                                   : cfg.energy_threshold;
    if (d.e_l <= 0) return "saw: energy threshold E_l must be positive";
    d.t_i = effective_iterations(L, cfg.max_iterations, cfg.ti_multiplier);
    if (d.t_i < 1) return "saw: T_i must be >= 1";
    d.L = L;
    d.k = (L - 1) / 2;
    d.kp1 = d.k + 1;
    d.p = effective_prefix_len(cfg.prefix_len, cfg.walkers);
    if (d.p > d.kp1) return "saw: prefix length exceeds half length k+1";
    if (cfg.max_restarts == 0 && cfg.time_budget_s <= 0 && cfg.candidate_quota == 0 &&
        cfg.stop_at_energy == 0)
        return "saw: no stop condition configured";
    if (cfg.bloom_fpr <= 0 || cfg.bloom_fpr >= 1) return "BloomFilter: fpr must be in (0,1)";
    if (d.p > 30) return "rank_prefixes: p > 30 is not enumerable";
    if (L > kMaxHalf)  // canonical_hash(0) of the full sequence indexes t_[0][i < L] (rng.hpp:77,89-95)
        return "saw: length exceeds the tabulation hash range (L <= 1023)";
    bloom_size(static_cast<uint64_t>(d.t_i) + 1, cfg.bloom_fpr, d.bloom_bits, d.bloom_k);
    if (d.p == 0) {
        d.nprefix = 1;
        d.prefixes.clear();
        d.prefix_bits.assign(1, 0u);
    } else {
        d.nprefix = 1 << (d.p - 1);
        d.prefixes = rank_prefixes(d.p);
        d.prefix_bits.assign(static_cast<size_t>(d.nprefix), 0u);
        for (int c = 0; c < d.nprefix; ++c)
            for (int j = 0; j < d.p; ++j)
                if (d.prefixes[static_cast<size_t>(c) * d.p + j] > 0) d.prefix_bits[c] |= 1u << j;
    }
    return "";
}

static int round_up(int v, int m) { return (v + m - 1) / m * m; }

static std::string make_walk_params_impl(int L, int p, int64_t t_i, int64_t e_l,
                                         uint64_t bloom_bits, int bloom_k, WalkParams& wp,
                                         int lpw_force) {
    wp = WalkParams{};
    // (the (delta, hp) key fits 32 bits up to L = 1001; longer pools have >= 150 free half
    // positions and run K1t)
    if (L > 1001) return "saw: the IDP4A walk kernel covers L <= 1001 (K1t runs longer lengths)";
    wp.L = L;
    wp.k = (L - 1) / 2;
    wp.kp1 = wp.k + 1;
    wp.p = p;
    const int free_bits = wp.kp1 - p;
    // lanes per walk: the narrowest of 8 (four walks per warp), 16 (two walks) and 32 with
    // R <= 16 neighbours per lane.  Measured on B200 (tools/lpw_sweep.py, 16,384 walks,
    // flip-deltas/s at 8 / 16 / 32 lanes): L=101 1.23e11 / 0.96e11 / 0.58e11;
    // L=251 1.66e11 / 1.61e11 / 1.19e11; L=401 - / 1.57e11 / 1.21e11;
    // L=527 - / 1.39e11 / 1.30e11.
    // LABS_LPW=8|16|32 forces a width (A/B timing, tests).
    const char* lpw_env = std::getenv("LABS_LPW");
    const int lpw_want = lpw_force ? lpw_force : (lpw_env ? std::atoi(lpw_env) : 0);
    // (16-lane segments need bloom_k <= 16: one Bloom index per lane)
    const bool fit16 = (free_bits + 15) / 16 <= kMaxR && bloom_k <= 16;
    const bool fit8 = (free_bits + 7) / 8 <= kMaxR && bloom_k <= 16;
    if (lpw_want == 32 || !fit16) wp.lpw = 32;
    else if (fit8 && lpw_want != 16) wp.lpw = 8;  // (4 walks per warp, small lengths)
    else wp.lpw = 16;
    wp.R = std::max(1, (free_bits + wp.lpw - 1) / wp.lpw);
    if (wp.R > kMaxR) return "saw: more than 512 free half bits is not supported by the GPU path";
    wp.S = std::max(1, (wp.k + 3) / 4);
    if (wp.S > 128) return "saw: length too large for the GPU path";
    wp.nwx = (wp.kp1 + 3) / 4;
    // SW = lpw ceil(S/lpw): the lag words the lanes cover -- lanes past S update and store
    // zeros (their windows read the zero padding) instead of branching.
    // X arrays: backward reads down to index -(4SW+4) (C update), forward reads up to
    // k/2 + 4SW + 8 (C update), 4*nwx (main loop) and 4*(nwx+S+2) (correlation init).
    const int SW = wp.lpw * ((wp.S + wp.lpw - 1) / wp.lpw);
    wp.xoff = 4 * round_up(SW + 2, 2);  // >= 4SW+8, and the G loop's X words 8-byte aligned
    const int xhi = std::max({wp.k / 2 + 4 * SW + 12, 4 * wp.nwx + 8, 4 * (wp.nwx + wp.S + 3)});
    wp.xwords = round_up((wp.xoff + xhi + 3) / 4, 4);
    // kernel: main loop reads d in [-(p+lpw R)/2 - 4R - 8, 4 nwx + 8]; lanes write |d| <= 4SW+4
    const int amax_h = (p + wp.lpw * wp.R) / 2 + 1;  // a0 + 8m < p + lpw R
    int koff = std::max(amax_h + 4 * wp.R + 12, 4 * SW + 12);
    while (koff % 4 != 3) ++koff;
    wp.koff = koff;
    wp.kwords = round_up((koff + std::max(4 * wp.nwx, 4 * SW) + 16) / 4, 4);
    wp.hw = (wp.kp1 + 31) / 32;
    if (bloom_bits >= (1ull << 31)) return "saw: Bloom filter exceeds 2^31 bits";
    if (bloom_k > 32) return "saw: more than 32 Bloom hashes is not supported by the GPU path";
    wp.bloom_bits = static_cast<uint32_t>(bloom_bits);
    wp.bloom_k = bloom_k;
    wp.bloom_words = round_up(static_cast<int>((bloom_bits + 31) / 32), 4);
    wp.bloom_mu = static_cast<uint64_t>((static_cast<unsigned __int128>(1) << 64) / bloom_bits);
    wp.t_i = t_i;
    wp.e_l = e_l;
    // X0 and X1 start on different bank halves (lanes of both parities read each step)
    int x1 = wp.xwords;
    while (x1 % 32 != 16) x1 += 4;
    wp.off_x1 = x1;
    wp.off_kl = wp.off_x1 + wp.xwords;
    wp.off_kh = wp.off_kl + wp.kwords;
    wp.off_half = wp.off_kh + wp.kwords;
    wp.off_dc = wp.off_half;  // (no per-lag dc array: T's C term reads the sequence)
    wp.off_bloom = wp.off_half + round_up(wp.hw, 4);
    // C16 and KQ are read only while the walk initialises its T registers, before the
    // Bloom filter is cleared: they live inside the filter's words
    wp.off_c16 = wp.off_bloom;
    wp.off_kq = wp.off_c16 + 2 * round_up(wp.S, 4);
    const int init_words = 2 * round_up(wp.S, 4) + round_up(wp.kp1, 4);
    wp.warp_words = wp.off_bloom + std::max(wp.bloom_words, init_words);
    // walks of one warp (segments) sit warp_words apart: an odd multiple of 4 words puts
    // their X0 / X1 words (read together in the G loop) in distinct banks for 2 or 4 segments
    if (wp.warp_words % 8 == 0) wp.warp_words += 4;
    // the flip-mask table fm (3 kp1 u64, the same for every walk) is read through L1 or
    // copied per block; walk_blocks_per_sm decides, after the register budget is known
    const int fm_words = 0;
    wp.fm_words = fm_words;
    const int segs = 32 / wp.lpw;
    int wpb = 4;
    while (wpb > 1 && (fm_words + wpb * segs * wp.warp_words) * 4 > 227 * 1024) --wpb;
    if ((fm_words + wpb * segs * wp.warp_words) * 4 > 227 * 1024 && wp.lpw < 32) {
        wp.lpw = 32;  // two walks' state does not fit a block: one walk per warp
        return make_walk_params_impl(L, p, t_i, e_l, bloom_bits, bloom_k, wp, 32);
    }
    if ((fm_words + wpb * segs * wp.warp_words) * 4 > 227 * 1024)
        return "saw: per-walk state (Bloom filter) exceeds shared memory; lower T_i or raise "
               "--bloom-fpr";
    wp.warps_per_block = wpb;
    wp.walks_per_block = wpb * segs;
    wp.rec_words = kRecHeader + wp.hw;
    return "";
}

// K1t geometry (saw_walk_mma.cuh): one walk per warp, 16-row q-tiles covering half indices
// a in [2 b0, 2 b0 + 256 nq), b0 = p/2; parity arrays with three byte-shifted copies; the
// kernel's byte offset of d = 0 stays 3 mod 4 (K1's lag-word stores) and kdelta aligns the
// A fragments instead.
static std::string make_walk_params_mma(int L, int p, int64_t t_i, int64_t e_l,
                                        uint64_t bloom_bits, int bloom_k, WalkParams& wp) {
    wp = WalkParams{};
    wp.kernel = 1;
    wp.L = L;
    wp.k = (L - 1) / 2;
    wp.kp1 = wp.k + 1;
    wp.p = p;
    wp.lpw = 32;
    const int b0 = p >> 1;
    wp.nq = (wp.k - 2 * b0) / 256 + 1;  // k <= 2 b0 + 256 nq - 1
    if (wp.nq > 2) return "saw: K1t covers at most 512 half positions";
    wp.R = 8 * wp.nq;
    wp.S = std::max(1, (wp.k + 3) / 4);
    if ((wp.S + 31) / 32 > std::min(4, (256 * wp.nq + 64 + 127) / 128))
        return "saw: K1t lag words exceed the lane budget";
    wp.nwx = (wp.kp1 + 3) / 4;
    wp.kdelta = ((3 - b0 - 7) % 4 + 4) % 4;       // (koff - D) == 0 mod 4, koff == 3 mod 4
    const int D = b0 + 7 + wp.kdelta;
    wp.nks = round_up((wp.kp1 + 7 + wp.kdelta + 31) / 32, 2);  // (even: g_mma's unroll)
    if (wp.nq == 1 && wp.nks == 8 && (wp.S + 31) / 32 != 2)  // (the NKS = 8 kernels assume it)
        return "saw: K1t geometry (8 k-steps with other than two lag words per lane)";
    // SW = 32 ceil(S/32): the lag words the lanes cover -- lanes past S update and store
    // zeros (their windows read the zero padding) instead of branching.
    // X: front reads down to -(4 SW + 8) (C update) and -(k + 8) (T update), B reads from -10;
    // back reads up to k/2 + 4 SW + 12 (C update), 4 (nwx + S + 3) (correlation init),
    // 32 nks + 16 (B) and 1.5 k + 4 (T update)
    const int SW = 32 * ((wp.S + 31) / 32);
    wp.xoff = 4 * round_up(std::max(SW + 2, (wp.k + 12) / 4 + 1), 2);
    const int xhi = std::max({wp.k / 2 + 4 * SW + 12, 4 * wp.nwx + 8, 4 * (wp.nwx + wp.S + 3),
                              32 * wp.nks + 24, wp.k + wp.k / 2 + 8});
    wp.xwords = round_up((wp.xoff + xhi + 3) / 4, 4);
    // K: A reads d from -(128 nq + D + 4) to 32 nks - D + 4; lag-word stores |d| <= 4 SW + 4
    int koff = std::max(128 * wp.nq + D + 16, 4 * SW + 12);
    while (koff % 4 != 3) ++koff;
    wp.koff = koff;
    wp.kwords = round_up((koff + std::max(32 * wp.nks + 16, 4 * SW + 16)) / 4, 4);
    wp.hw = (wp.kp1 + 31) / 32;
    if (bloom_bits >= (1ull << 31)) return "saw: Bloom filter exceeds 2^31 bits";
    if (bloom_k > 32) return "saw: more than 32 Bloom hashes is not supported by the GPU path";
    wp.bloom_bits = static_cast<uint32_t>(bloom_bits);
    wp.bloom_k = bloom_k;
    wp.bloom_words = round_up(static_cast<int>((bloom_bits + 31) / 32), 4);
    wp.bloom_mu = static_cast<uint64_t>((static_cast<unsigned __int128>(1) << 64) / bloom_bits);
    wp.t_i = t_i;
    wp.e_l = e_l;
    int x1 = wp.xwords;
    while (x1 % 32 != 16) x1 += 4;
    wp.off_x1 = x1;
    // copies cover only the B reads: bytes [xoff - 16, xoff + 32 nks + 32)
    wp.xcl = wp.xoff - 16;
    wp.xcw = 8 * wp.nks + 12;
    wp.off_xc = wp.off_x1 + wp.xwords;
    wp.kpl = (wp.nq == 1 && wp.nks == 8) ? 1 : 0;
    wp.off_kl = wp.off_xc + 6 * wp.xcw;             // KL, or KP (pair layout: 2 kwords + 32)
    wp.off_kh = wp.off_kl + (wp.kpl ? 2 * wp.kwords + 32 : wp.kwords);
    wp.off_half = wp.off_kh + wp.kwords;
    wp.off_dc = wp.off_half;
    wp.off_bloom = wp.off_half + round_up(wp.hw, 4);
    wp.off_c16 = wp.off_bloom;
    wp.off_kq = wp.off_c16 + 2 * round_up(wp.S, 4);
    const int init_words = 2 * round_up(wp.S, 4) + round_up(wp.kp1, 4);
    wp.warp_words = wp.off_bloom + std::max(wp.bloom_words, init_words);
    if (wp.warp_words % 8 == 0) wp.warp_words += 4;
    wp.fm_words = 0;
    int wpb = 4;
    while (wpb > 1 && wpb * wp.warp_words * 4 > 227 * 1024) --wpb;
    if (wpb * wp.warp_words * 4 > 227 * 1024)
        return "saw: per-walk state (Bloom filter) exceeds shared memory; lower T_i or raise "
               "--bloom-fpr";
    wp.warps_per_block = wpb;
    wp.walks_per_block = wpb;
    wp.rec_words = kRecHeader + wp.hw;
    return "";
}

// Which walk kernel: K1t (tensor-core G) from kMmaMinFree free half positions on, K1
// below (LABS_KERNEL=dp4a|mma forces one: A/B timing, tests).
static constexpr int kMmaMinFree = 150;  // (same-box crossover: K1 wins at 143 free bits,
                                         //  K1t at 153 -- tools/ab_kernels_by_length.sh)

std::string make_walk_params(int L, int p, int64_t t_i, int64_t e_l, uint64_t bloom_bits,
                             int bloom_k, WalkParams& wp) {
    const char* kern = std::getenv("LABS_KERNEL");
    const int free_bits = (L + 1) / 2 - p;
    const int k = (L - 1) / 2;
    const bool fits_mma = k - 2 * (p >> 1) < 512 && std::getenv("LABS_LPW") == nullptr;
    bool mma = fits_mma && free_bits >= kMmaMinFree;
    if (kern && std::string(kern) == "mma") mma = fits_mma;
    if (kern && std::string(kern) == "dp4a") mma = false;
    if (mma) {
        std::string err = make_walk_params_mma(L, p, t_i, e_l, bloom_bits, bloom_k, wp);
        if (err.empty()) return err;
    }
    return make_walk_params_impl(L, p, t_i, e_l, bloom_bits, bloom_k, wp, 0);
}

}  // namespace labs_b200
