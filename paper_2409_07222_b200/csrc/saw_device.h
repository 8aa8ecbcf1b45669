// saw_device.h -- plain-old-data shared by the host orchestration (C++) and the
// sm_100a kernels.  No torch or CUDA types, so it is usable from both sides.
#pragma once
#include <stdint.h>

namespace labs_b200 {

constexpr int kMaxR = 16;          // neighbours per lane: free bits <= 32*16 = 512
constexpr int kMaxHalf = 1024;     // TabulationHash::kMaxLen (rng.hpp:77)
constexpr unsigned kRingWaitSpins = 5000000u;  // a full ring waits <= ~20 s for a drain
constexpr int kRecHeader = 6;      // record header: walk, iteration, energy, flags,
                                   // canonical_hash(0) of the full sequence (lo, hi)

// Derived, device-ready description of one Step-1 launch (one batch of walks).
// Per-walk shared-memory layout (32-bit word offsets inside a warp's slice):
//   X0, X1 : parity arrays, byte xoff+i = x_{2i+parity} in {-1,+1}, 0 = padding
//   KL, KH : symmetric correlation kernel, byte koff+d = low / high byte of C_{2|d|}
//            (KH only maintained while some |C| > 127)
//   C16    : int16 C_{2t}, t = 1..4S (pairs per word)
//   KQ     : int32 per half index a: 16 N(a) + 32 Q(a)  (a < k),  4 N + 8 Q (a = k)
//   HALF   : packed current half,  BLOOM : visited filter bits
struct WalkParams {
    int32_t L, k, kp1, p;          // L = 2k+1, half length k+1, prefix length p
    int32_t S;                     // 4-lag words covering even lags t=1..k (C update)
    int32_t R;                     // free neighbours per lane
    int32_t nwx;                   // 4-position words per parity array (main loop trip count)
    int32_t xoff, xwords;          // X array byte offset of index 0, words per array
    int32_t koff, kwords;          // kernel byte offset of d = 0 (== 3 mod 4), words per array
    int32_t hw;                    // 32-bit words per packed half
    int32_t bloom_k;               // hashes per key
    uint32_t bloom_bits;           // m
    int32_t bloom_words;           // ceil(m/32) rounded to 4
    uint64_t bloom_mu;             // floor(2^64 / m) (Barrett)
    int64_t t_i;                   // iteration cap
    int64_t e_l;                   // sieve: emit iff E < e_l
    int32_t warp_words;            // shared-memory words per walk (warp)
    int32_t off_x1, off_kl, off_kh, off_c16, off_kq, off_dc, off_half, off_bloom;  // X0 at 0
    int32_t warps_per_block;
    int32_t lpw;                   // lanes per walk (32: one walk per warp; 16: two)
    int32_t walks_per_block;       // warps_per_block * 32 / lpw
    int32_t debug_check;           // re-derive E from C every iteration, flag divergence
    int32_t count_visited;         // full Bloom probes of every free neighbour (exact stats)
    int32_t rec_words;             // kRecHeader + hw
    // K1t (tensor-core G, saw_walk_mma.cuh): kernel = 1
    int32_t kernel;                // 0 = K1 (IDP4A G), 1 = K1t (mma.sync s8 G)
    int32_t nq;                    // K1t: 16-row q-tiles per parity (neighbours 256 nq)
    int32_t nks;                   // K1t: 32-deep k-steps
    int32_t kdelta;                // K1t: D = p/2 + 7 + kdelta aligns the kernel words
    int32_t off_xc;                // K1t: three byte-shifted copies per parity array
    int32_t xcl, xcw;              // K1t: copy c word i = parity-array bytes xcl + 4i + c ..+3
    int32_t kpl;                   // K1t: low kernel bytes in the A-fragment pair layout (KP)
                                   //   -- one q-tile at 8 k-steps, where the extra words cost no
                                   //   resident block; else plain (KL)
    int64_t nwalks;                // walks in this launch
    int64_t rec_cap;               // record ring slots (a power of two)
    // inputs (device pointers)
    const uint64_t* fm;            // [3][kp1]: tabulation flip masks of half position j in
                                   //   tables 0/1 (Bloom keys), then the flip mask of the
                                   //   full-sequence hash t0[j]^t0[L-1-j] (dedup key)
    const uint64_t* tab;           // [2][kp1][2] tabulation entries (half hashes)
    const uint64_t* tabfull;       // [L][2] table-0 entries of full positions (dedup key)
    uint64_t salt0, salt1;         // length salts for kp1
    uint64_t salt_full;            // table-0 salt for L
    int32_t fm_words;              // u32 words of the block-level fm table in shared memory
    const uint32_t* halves;        // [nwalks][hw] initial half bits (bit i set <=> +1)
    // outputs: the sieve's record ring (K2, north_star (d)).  A warp reserves slots for all of
    // its segments' hits with one atomicAdd on rec_count (the ring head); a slot is written
    // once rec_count - rec_tail < rec_cap (the host advances rec_tail as it drains the ring
    // with async copies while the launch runs), and published by its tag (slot + 1, written
    // after a fence) -- the ring never overflows, so no batch is ever rerun.
    uint32_t* rec;                 // [rec_cap][rec_words]
    uint32_t* rec_tag;             // [rec_cap] (uint32)(rec_seq0 + slot + 1) once slot's record
                                   //   is complete (rec_seq0: records the ring carried in
                                   //   earlier launches, so stale tags never match)
    unsigned long long rec_seq0;
    unsigned long long* rec_count; // ring head: slots reserved in this launch
    const unsigned long long* rec_tail;  // ring tail: slots the host has drained (host-written)
    int* ctl;                      // [0] ring abort (no drain for ~20 s), [1] cancel
    unsigned long long* walk_next; // dynamic walk-group queue (zeroed per launch)
    int64_t* walk_stats;           // [nwalks][kWalkStatWords]
};

// per-walk stats record (int64 words)
enum WalkStat : int {
    kWsIterations = 0,
    kWsEmitted = 1,
    kWsBest = 2,
    kWsInitial = 3,
    kWsExhausted = 4,
    kWsDeltaEvals = 5,    // unvisited free neighbours evaluated (count_visited=1 only)
    kWsVisitedProbes = 6, // lazy-mode Bloom probe rounds
    kWsWideIters = 7,     // iterations that needed the int16 correlation path
    kWsDiverged = 8,      // debug_check failures
    kWalkStatWords = 9
};

// One seed segment = restarts [r0, r0+restarts) of one walker, drawn in order
// from the walker's xoshiro stream (state carried across segments).
struct SeedParams {
    int32_t kp1, p, hw, nseg;
    uint64_t seed;
    const uint32_t* walker_ids;    // [nseg] global walker index (RNG stream)
    const uint32_t* prefix_bits;   // [nseg] pinned prefix bits (bit i set <=> +1)
    const int64_t* seg_restarts;   // [nseg]
    const int64_t* seg_offset;     // [nseg] first walk index of the segment in `halves`
    const int32_t* seg_init;       // [nseg] 1 = fresh Rng(seed, walker)
    const uint32_t* seg_slot;      // [nseg] the walker's generator slot in rng_state
    uint64_t* rng_state;           // [walker slots][4] in/out: a walker's stream continues
                                   //   across segments (batches) from here
    uint32_t* halves;              // [nwalks][hw]
};

struct EnumParams {
    int32_t L, k, kp1, p, m;       // Gray range over half positions [p, p+m)
    int32_t chunk_log2;            // 2^chunk_log2 Gray steps per warp task
    int32_t hw;
    int64_t e_l;
    uint64_t g_begin, g_end;       // configuration index range
    const uint32_t* base_half;     // [hw] half bits of configuration 0
    uint32_t* rec;                 // [rec_cap][2] (g lo, g hi) + energy -> 4 words
    int64_t rec_cap;
    unsigned long long* rec_count;
    int64_t* best;                 // [nchunks][2] best energy, best g
};

}  // namespace labs_b200
