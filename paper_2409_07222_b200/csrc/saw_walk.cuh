// saw_walk.cuh -- K1, the sm_100a walk kernel of Step 1 of the dual-step LABS search
// (templates; instantiated per (R, LPW) in saw_walk_r*.cu, launched from saw_kernels.cu).
//
// K1 saw_walk_kernel : 8, 16 or 32 lanes = one self-avoiding walk (run_walk, saw.cpp:117-149);
//                      warps take groups of walks from an atomic queue.
//                      Fuses the Bloom probe, the skew flip-delta of every free
//                      neighbour (skew_flip_delta_fast, skew.cpp:60-93), the
//                      lexicographic argmin (best_neighbour, saw.cpp:106-115), the
//                      apply (apply_skew_flip, skew.cpp:95-105), the Bloom insert
//                      and the E < E_l sieve with compaction into a device
//                      record buffer (sink.emit, saw.cpp:143-146).
//
// Arithmetic.  For a skew-symmetric pivot the four sign products of
// the reference's fused delta pair up (x_b x_{b+-kk} = x_a x_{a-+kk}), so for half
// index a < k (b = L-1-a):
//     dE(a) = 16 N(a) + 32 Q(a) - 8 x_a G(a) + 8 (-1)^(k-a) C_{2(k-a)}
// and for the centre a = k:  dE = 4 N + 8 Q - 4 x_k G, where
//     G(a) = sum_{j = a mod 2, j != a} C_{|a-j|} x_j      (x = 0 outside [0, L))
//     N(a) = #valid single terms,  Q(a) = sum_t x_{a-2t} x_{a+2t} (b excluded).
// G is the only O(L) part.  On the parity array X_par it is a sliding dot product with
// the symmetric kernel K[d] = C_{2|d|}: G(a) = sum_i X_par[i] K[i - a/2].  A lane owns
// neighbours a0, a0+8, ..., so one X word is shared by its R neighbours and the kernel
// window slides by one word per neighbour: 4 positions per IDP4A (int8 C), plus a
// second IDP4A on the high bytes while some |C| > 127.  The rest of the delta,
// T(a) = 16N + 32Q + 8(-1)^(k-a) C_{2(k-a)}, is kept per neighbour in the owning lane's
// registers and updated in O(1) per flip.  Everything is exact integer math.
#include <cuda_runtime.h>
#include <stdint.h>
#ifdef LABS_PHASE_CLOCKS
#include <cstdio>
#endif

#include "saw_device.h"
#include "saw_walk.h"

namespace labs_b200 {

#define FULLMASK 0xffffffffu
#define INT_BIG 0x7fffffff

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    return __byte_perm(a, b, sel);
}

// (h1 + i*h2) mod 2^64 mod m  (bloom.cpp:28,36), Barrett with mu = floor(2^64/m), m < 2^32
__device__ __forceinline__ uint32_t bloom_index(uint64_t h1, uint64_t h2, uint32_t i, uint64_t mu,
                                                uint32_t m) {
    const uint64_t x = h1 + (uint64_t)i * h2;
    const uint64_t q = __umul64hi(x, mu);
    // x - q m lies in [0, 2m) and m < 2^31 (make_walk_params): its low 32 bits are exact
    const uint32_t r = (uint32_t)x - (uint32_t)q * m;
    return r >= m ? r - m : r;
}

__device__ __forceinline__ uint64_t shfl_xor64(uint64_t v, int lane_mask) {
    const uint32_t lo = __shfl_xor_sync(FULLMASK, (uint32_t)v, lane_mask);
    const uint32_t hi = __shfl_xor_sync(FULLMASK, (uint32_t)(v >> 32), lane_mask);
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    return v;
}

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += (long long)shfl_xor64((uint64_t)v, o);
    return v;
}

// PRMT selector of bytes o..o+3 of a word pair: o | (o+1)<<4 | (o+2)<<8 | (o+3)<<12
__device__ __forceinline__ uint32_t sel4(int o) { return 0x3210u + 0x1111u * (uint32_t)o; }
// bytes o+3..o (reversed): (o+3) | (o+2)<<4 | (o+1)<<8 | o<<12
__device__ __forceinline__ uint32_t sel4r(int o) { return 0x0123u + 0x1111u * (uint32_t)o; }
// sign-extended byte b of w
__device__ __forceinline__ int sbyte(uint32_t w, int b) {  // one PRMT, sign-replicate mode
    // (selector nibble 8|b copies the sign of byte b; __byte_perm drops that bit, so PTX)
    uint32_t r;
    const uint32_t sel = (uint32_t)(b | ((8 | b) << 4) | ((8 | b) << 8) | ((8 | b) << 12));
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "r"(sel));
    return (int)r;
}

// ---------------------------------------------------------------------------
// Main O(L) loop: G(a) for this lane's R neighbours a = a0 + 8m (a' = a0' + 4m).
// Step w: X word w (positions 4w..4w+3 of the lane's parity) is shared by all R
// neighbours; neighbour m needs kernel bytes koff + 4(w-m) - a0' .. +3, i.e. the
// PRMT-aligned word KW_{w-m}; KW slides one slot per step (one new raw word).
// acc[] accumulates onto its incoming value (the wide path runs the high-byte kernel
// first, scales by 256 and continues with the low bytes in the same registers).
template <int R>
__device__ __forceinline__ void g_step(uint32_t x, const uint32_t* __restrict__ Kw, int w, int j,
                                       int kb, uint32_t sel, uint32_t (&KW)[R], uint32_t& rw,
                                       int (&acc)[R]) {
    const uint32_t nw = Kw[kb + w + 2];
#pragma unroll
    for (int m = 0; m < R; ++m) acc[m] = __dp4a((int)x, (int)KW[(j - m + R) % R], acc[m]);
    KW[(j + 1) % R] = prmt(rw, nw, sel);
    rw = nw;
}

template <int R, int J>
struct GTail {
    static __device__ __forceinline__ void run(const uint32_t* __restrict__ Xw,
                                               const uint32_t* __restrict__ Kw, int w0, int rem,
                                               int kb, uint32_t sel, uint32_t (&KW)[R],
                                               uint32_t& rw, int (&acc)[R]) {
        if (J < rem) {
            g_step<R>(Xw[w0 + J], Kw, w0 + J, J, kb, sel, KW, rw, acc);
            GTail<R, J + 1>::run(Xw, Kw, w0, rem, kb, sel, KW, rw, acc);
        }
    }
};
template <int R>
struct GTail<R, R> {
    static __device__ __forceinline__ void run(const uint32_t* __restrict__, const uint32_t* __restrict__,
                                               int, int, int, uint32_t, uint32_t (&)[R],
                                               uint32_t&, int (&)[R]) {}
};

template <int R>
__device__ __forceinline__ void g_neighbours(const uint32_t* __restrict__ Xw,
                                             const uint32_t* __restrict__ Kw, int nwx, int kb,
                                             uint32_t sel, int (&acc)[R]) {
    uint32_t KW[R];
#pragma unroll
    for (int m = 0; m < R; ++m) KW[(R - m) % R] = prmt(Kw[kb - m], Kw[kb - m + 1], sel);
    uint32_t rw = Kw[kb + 1];
    const int nfull = (nwx / R) * R;
    for (int w0 = 0; w0 < nfull; w0 += R) {
        if constexpr (R % 2 == 0) {  // X words in pairs (Xw is 8-byte aligned, w0 even)
#pragma unroll
            for (int j = 0; j < R; j += 2) {
                const uint2 xx = *reinterpret_cast<const uint2*>(Xw + w0 + j);
                g_step<R>(xx.x, Kw, w0 + j, j, kb, sel, KW, rw, acc);
                g_step<R>(xx.y, Kw, w0 + j + 1, j + 1, kb, sel, KW, rw, acc);
            }
        } else {
#pragma unroll
            for (int j = 0; j < R; ++j) g_step<R>(Xw[w0 + j], Kw, w0 + j, j, kb, sel, KW, rw, acc);
        }
    }
    // remainder steps j = 0 .. nwx - nfull - 1: nested guards, so a remainder of r costs
    // r + 1 tests instead of R
    GTail<R, 0>::run(Xw, Kw, nfull, nwx - nfull, kb, sel, KW, rw, acc);
}

// Lane minimum of the (delta, hp) keys (dE + 2^22) * 512 + a over the neighbours not in
// `skip` (v[] holds the keys themselves: see the key-scaled T registers in run_walk_seg);
// pairwise (tree) minimum: log2(R) dependent steps, not R.
template <int R>
__device__ __forceinline__ uint32_t lane_min_key(const int (&v)[R], uint32_t skip) {
    uint32_t key[R];
#pragma unroll
    for (int m = 0; m < R; ++m) key[m] = (skip & (1u << m)) ? 0xffffffffu : (uint32_t)v[m];
#pragma unroll
    for (int h = 1; h < R; h <<= 1)
#pragma unroll
        for (int m = 0; m + h < R; m += 2 * h) key[m] = min(key[m], key[m + h]);
    return key[0];
}

// ---------------------------------------------------------------------------
struct WarpSmem {
    int8_t* X0;       // parity arrays (byte views, index xoff + i)
    int8_t* X1;
    uint32_t* X0w;
    uint32_t* X1w;
    uint32_t* KL;     // kernel low bytes (word view)
    uint32_t* KH;     // kernel high bytes
    uint32_t* C16;    // int16 C_{2t}, t = 4s+1..4s+4 in words 2s, 2s+1
    int* KQ;          // 16N+32Q per half index (walk initialisation only)
    uint32_t* half;   // half bits
    uint32_t* bloom;  // visited filter
};

// Sign of full-sequence position j of the skew expansion of `half` (skew.cpp:14-26).
__device__ __forceinline__ int x_of_half(const uint32_t* half, int k, int j) {
    int src = j, neg = 0;
    if (j > k) {
        const int i = j - k;
        src = k - i;
        neg = i & 1;
    }
    const int bit = (half[src >> 5] >> (src & 31)) & 1;
    return (bit ^ neg) ? 1 : -1;
}

// C_{2t} by direct summation over the parity arrays (sequence.cpp:8-19 restricted to
// even lags; odd lags of a skew sequence vanish): sum_par sum_i X[i] X[i+t].
__device__ __forceinline__ int corr_even_lag(const WarpSmem& w, const WalkParams& P, int t) {
    int acc = 0;
    const int dw = t >> 2;
    const uint32_t sel = sel4(t & 3);
    const int n0 = P.xoff >> 2;
#pragma unroll
    for (int par = 0; par < 2; ++par) {
        const uint32_t* Xw = par ? w.X1w : w.X0w;
        for (int n = n0; n < n0 + P.nwx; ++n)
            acc = __dp4a((int)Xw[n], (int)prmt(Xw[n + dw], Xw[n + dw + 1], sel), acc);
    }
    return acc;
}

__device__ __forceinline__ uint32_t pack4(int b0, int b1, int b2, int b3) {  // low bytes
    return prmt(prmt((uint32_t)b0, (uint32_t)b1, 0x0040), prmt((uint32_t)b2, (uint32_t)b3, 0x0040),
                0x5410);
}
__device__ __forceinline__ int hi_byte(int c) { return (c - (int)(int8_t)c) >> 8; }

// Store the 4 correlations c[0..3] of lag word s (t = 4s+1..4s+4) into C16 and the
// kernel arrays: forward word (d = 4s+1..4s+4) = (c0,c1,c2,c3); mirrored word
// (d = -4s-3..-4s) = (c2,c1,c0,cprev) with cprev = C_{2*4s} (0 for s = 0: K[0] = 0).
__device__ __forceinline__ void store_c_word(const WarpSmem& w, const WalkParams& P, int s,
                                             const int (&c)[4], int cprev, bool wide) {
    w.C16[2 * s] = prmt((uint32_t)c[0], (uint32_t)c[1], 0x5410);
    w.C16[2 * s + 1] = prmt((uint32_t)c[2], (uint32_t)c[3], 0x5410);
    const int fw = (P.koff + 1) / 4 + s;
    const int bw = (P.koff - 3) / 4 - s;
    const uint32_t lo = pack4(c[0], c[1], c[2], c[3]);
    w.KL[fw] = lo;
    w.KL[bw] = prmt(lo, (uint32_t)cprev, 0x4012);  // (c2, c1, c0, cprev)
    if (wide) {
        const uint32_t hi = pack4(hi_byte(c[0]), hi_byte(c[1]), hi_byte(c[2]), hi_byte(c[3]));
        w.KH[fw] = hi;
        w.KH[bw] = prmt(hi, (uint32_t)hi_byte(cprev), 0x4012);
    }
}

// Kernel words of lag word s without the int16 copy (main loop: C lives in registers).
__device__ __forceinline__ void store_k_word(const WarpSmem& w, const WalkParams& P, int s,
                                             const int (&c)[4], int cprev, bool wide) {
    const int fw = (P.koff + 1) / 4 + s;
    const int bw = (P.koff - 3) / 4 - s;
    const uint32_t lo = pack4(c[0], c[1], c[2], c[3]);
    w.KL[fw] = lo;
    w.KL[bw] = prmt(lo, (uint32_t)cprev, 0x4012);  // (c2, c1, c0, cprev)
    if (wide) {
        const uint32_t hi = pack4(hi_byte(c[0]), hi_byte(c[1]), hi_byte(c[2]), hi_byte(c[3]));
        w.KH[fw] = hi;
        w.KH[bw] = prmt(hi, (uint32_t)hi_byte(cprev), 0x4012);
    }
}

// ---------------------------------------------------------------------------
// Segments: a warp runs 32 / LPW walks side by side, LPW lanes each (LPW = 32: one walk
// per warp).  With LPW = 16 every warp-wide instruction of the per-step bookkeeping
// (argmin, Bloom probe, apply) serves two walks and each lane owns 2x the neighbours, so
// more walks share an SM's issue slots and latency.  All reductions stay inside a segment
// (width-LPW shuffles); control flow is per segment with warp-uniform loops.
template <int LPW>
struct Seg {
    static constexpr int kSegs = 32 / LPW;
    static constexpr uint32_t kLow = LPW == 32 ? 0xffffffffu : ((1u << LPW) - 1u);
    int lane, sl, base;
    __device__ __forceinline__ explicit Seg(int l) : lane(l), sl(l % LPW), base(l - l % LPW) {}
    __device__ __forceinline__ int sum(int v) const {
#pragma unroll
        for (int o = LPW / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o, LPW);
        return v;
    }
    __device__ __forceinline__ long long sum64(long long v) const {
#pragma unroll
        for (int o = LPW / 2; o > 0; o >>= 1) v += (long long)shfl_xor64((uint64_t)v, o);
        return v;
    }
    __device__ __forceinline__ uint64_t xor64(uint64_t v) const {
#pragma unroll
        for (int o = LPW / 2; o > 0; o >>= 1) v ^= shfl_xor64(v, o);
        return v;
    }
    __device__ __forceinline__ uint32_t umin(uint32_t v) const {
        if (LPW == 32) return __reduce_min_sync(FULLMASK, v);
        if (LPW == 16) {  // two independent warp REDUX (one per half) instead of 4 shuffle levels
            const bool hi = lane >= 16;
            const uint32_t lo_min = __reduce_min_sync(FULLMASK, hi ? 0xffffffffu : v);
            const uint32_t hi_min = __reduce_min_sync(FULLMASK, hi ? v : 0xffffffffu);
            return hi ? hi_min : lo_min;
        }
#pragma unroll
        for (int o = LPW / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(FULLMASK, v, o, LPW));
        return v;
    }
    __device__ __forceinline__ int imin(int v) const {
        if (LPW == 32) return __reduce_min_sync(FULLMASK, v);
        if (LPW == 16) {
            const bool hi = lane >= 16;
            const int lo_min = __reduce_min_sync(FULLMASK, hi ? INT_BIG : v);
            const int hi_min = __reduce_min_sync(FULLMASK, hi ? v : INT_BIG);
            return hi ? hi_min : lo_min;
        }
#pragma unroll
        for (int o = LPW / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(FULLMASK, v, o, LPW));
        return v;
    }
    __device__ __forceinline__ bool all(bool b) const {
        if (LPW == 32) return __all_sync(FULLMASK, b);
        return ((__ballot_sync(FULLMASK, b) >> base) & kLow) == kLow;
    }
    __device__ __forceinline__ bool any(bool b) const {
        if (LPW == 32) return __any_sync(FULLMASK, b);
        return ((__ballot_sync(FULLMASK, b) >> base) & kLow) != 0;
    }
    // "some segment of this warp has b" for a segment-uniform b (loop control); with one
    // segment per warp b is already warp-uniform and needs no vote
    __device__ __forceinline__ bool uni(bool b) const {
        if (LPW == 32) return b;
        return __any_sync(FULLMASK, b);
    }
    template <typename T>
    __device__ __forceinline__ T bcast(T v) const { return __shfl_sync(FULLMASK, v, 0, LPW); }
};

template <int R, int LPW>
struct LagWords {  // lag words a lane may own: s = sl + LPW jj, S = ceil(k/4) <= 128
    static constexpr int a = (LPW * R + 32 + 4 * LPW - 1) / (4 * LPW);
    static constexpr int b = 128 / LPW;
    static constexpr int value = a < b ? a : b;
};

// K1: LPW lanes = one walk.  The per-neighbour constant part of the delta
//     T(a) = 16 N(a) + 32 Q(a) + 8 (-1)^(k-a) C_{2(k-a)}   (a < k),   4 N + 8 Q  (a = k)
// and xs(a) = 8 x_a (4 x_k) live in the owning lane's registers, so a delta is one IMAD on
// the sliding dot product G(a): dE(a) = T(a) - xs(a) G(a) (for L <= 1001 both are kept
// key-scaled, so that IMAD yields the argmin key itself).  Per step T is updated in O(1) per
// neighbour (the C term and the Q pairs through the flipped positions, read from the zeroed
// pre-step sequence); the exact even-lag C live in the lag owners' registers.
template <int R, int LPW, bool COUNT>
__device__ void run_walk_seg(const WalkParams& P, const WarpSmem& w, const uint64_t* fm0,
                             const uint64_t* fm1, const uint64_t* fmf, int64_t walk, bool valid,
                             const Seg<LPW>& sg, int* score_out, int* corr_out) {
    constexpr int NJ = LagWords<R, LPW>::value;
    const int L = P.L, k = P.k, kp1 = P.kp1, S = P.S;
    const int sl = sg.sl;
    const int nj = (S + LPW - 1) / LPW;  // lag words owned per lane (<= NJ)

    // ---- load the initial half, build parity arrays, clear kernel + Bloom ----
    const uint32_t* src = P.halves + (valid ? walk : 0) * P.hw;
    for (int i = sl; i < P.hw; i += LPW) w.half[i] = valid ? src[i] : 0u;
    __syncwarp();
    for (int wi = sl; wi < 2 * P.xwords; wi += LPW) {
        const int par = wi >= P.xwords;
        const int word = wi - par * P.xwords;
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int li = word * 4 + b - P.xoff;
            const int j = 2 * li + par;
            const int x = (li >= 0 && j < L) ? x_of_half(w.half, k, j) : 0;
            v |= ((uint32_t)x & 0xffu) << (8 * b);
        }
        (par ? w.X1w : w.X0w)[word] = v;
    }
    for (int i = sl; i < 2 * P.kwords; i += LPW) w.KL[i] = 0;  // KL and KH are adjacent
    __syncwarp();

    // ---- exact C_{2t} of the owned lag words (registers), E, max|C| ----
    int e_part = 0, cmax = 0;
    int C[NJ][4];
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) {
        const int s = sl + LPW * jj;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int t = 4 * s + 1 + b;
            int v = 0;
            if (jj < nj && s < S && t <= k) v = corr_even_lag(w, P, t);
            C[jj][b] = v;
            e_part += v * v;
            cmax = max(cmax, abs(v));
        }
    }
    int energy = sg.sum(e_part);
    bool wide = sg.any(cmax > 127);
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) {
        const int up = __shfl_up_sync(FULLMASK, C[jj][3], 1, LPW);
        const int wrap = __shfl_sync(FULLMASK, jj > 0 ? C[jj > 0 ? jj - 1 : 0][3] : 0, LPW - 1, LPW);
        const int s = sl + LPW * jj;
        const int cprev = s == 0 ? 0 : (sl == 0 ? wrap : up);
        if (jj < nj && s < S) {
            store_c_word(w, P, s, C[jj], cprev, wide);
            if (corr_out && valid)
                for (int b = 0; b < 4; ++b)
                    if (4 * s + 1 + b <= k) corr_out[walk * k + 4 * s + b] = C[jj][b];
        }
    }

    // ---- 16N + 32Q per half index (lanes over a), once per walk ----
    for (int a = P.p + sl; a <= k; a += LPW) {
        const int8_t* Xb = ((a & 1) ? w.X1 : w.X0) + P.xoff + (a >> 1);
        const int tstar = (a < k) ? (k - a) : -1;
        int q = 0;
        for (int t = 1; 2 * t <= a; ++t)
            if (t != tstar) q += (int)Xb[-t] * (int)Xb[t];
        const int n = (a >> 1) + ((L - 1 - a) >> 1) - (a < k ? 1 : 0);
        w.KQ[a] = (a < k) ? 16 * n + 32 * q : 4 * n + 8 * q;
    }
    __syncwarp();

    // ---- lane geometry: this lane's neighbours a = a0 + 8m (all of parity `par`) ----
    const int cgrp = sl & 7, g = sl >> 3;
    const int a0 = P.p + cgrp + 8 * R * g;
    const int par = a0 & 1, a0h = a0 >> 1;
    const uint32_t* Xw = (par ? w.X1w : w.X0w) + (P.xoff >> 2);
    const int8_t* Xmine = (par ? w.X1 : w.X0) + P.xoff;
    const int kb = (P.koff - a0h) >> 2;
    const uint32_t ksel = sel4((P.koff - a0h) & 3);
    const int sgn8 = ((k - a0) & 1) ? -8 : 8;  // 8 (-1)^(k-a), the same for every m
    const uint32_t kbase = 0x80000000u + (uint32_t)a0;  // key = (dE + 2^22) * 512 + a
    // For L <= 1001, |dE| < 2^22 and the unsigned key (dE + 2^22) * 512 + a orders
    // (delta, hp) lexicographically.  T and xs are then kept key-scaled,
    //     T'(a) = 512 T(a) + 2^31 + a,   xs' = 512 xs,
    // so that one IMAD, T' - xs' G, yields the key itself (wrapping mod 2^32 exactly like
    // the unsigned key).  Longer lengths keep the plain delta (sc = 1).
    // K1 runs L <= 1001 only (make_walk_params_impl): (delta, hp) always fit one key.  The
    // diagnostic options (debug_check_energy, score_out) run in the COUNT kernels only, so the
    // plain kernel has no per-step test of them.
    constexpr bool one_key = true;
    const bool dbg = COUNT && P.debug_check != 0;
    const int sc = one_key ? 512 : 1;
    uint32_t T[R];  // (unsigned: the key form wraps mod 2^32; meaningless for a > k, masked)
    int xs[R];  // NEGATED, key-scaled: -512 * 8 x_a (-512 * 4 x_k), so a key is one IMAD
    {
        const int16_t* C16h = reinterpret_cast<const int16_t*>(w.C16);
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int a = a0 + 8 * m;
            int t = 0;
            xs[m] = 0;
            if (a < k) {
                t = w.KQ[a] + sgn8 * (int)C16h[k - a - 1];
                xs[m] = 8 * (int)Xmine[a >> 1];
            } else if (a == k) {
                t = w.KQ[a];
                xs[m] = 4 * (int)Xmine[a >> 1];
            }
            T[m] = (uint32_t)(t * sc) + (one_key ? kbase + 8u * m : 0u);
            xs[m] *= -sc;
        }
    }

    // ---- clear the Bloom filter (it held C16 and KQ until here) ----
    __syncwarp();
    {
        uint4* b4 = reinterpret_cast<uint4*>(w.bloom);
        for (int i = sl; i < (P.bloom_words >> 2); i += LPW) b4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();

    // ---- half hashes h1, h2 (saw.cpp:77-89) and the initial Bloom insert ----
    uint64_t h1 = 0, h2 = 0;
    for (int i = sl; i < kp1; i += LPW) {
        const int bit = (w.half[i >> 5] >> (i & 31)) & 1;
        h1 ^= P.tab[(0 * kp1 + i) * 2 + bit];
        h2 ^= P.tab[(1 * kp1 + i) * 2 + bit];
    }
    h1 = sg.xor64(h1) ^ P.salt0;
    h2 = sg.xor64(h2) ^ P.salt1;
    // canonical_hash(0) of the full expanded sequence (DedupSink key, candidate.hpp:84-99,
    // rng.hpp:89-95), kept incrementally: a skew flip at j toggles positions j and L-1-j
    uint64_t hf = 0;
    for (int j = sl; j < L; j += LPW) hf ^= P.tabfull[2 * j + (x_of_half(w.half, k, j) > 0)];
    hf = sg.xor64(hf) ^ P.salt_full;
    for (int i = sl; i < P.bloom_k; i += LPW) {
        const uint32_t idx = bloom_index(h1, h2, i, P.bloom_mu, P.bloom_bits);
        atomicOr(&w.bloom[idx >> 5], 1u << (idx & 31));
    }
    __syncwarp();

    const int e0 = energy;
    int best = energy;
    int iterations = 0, emitted = 0, wide_iters = 0, diverged = 0;  // each <= T_i < 2^28
    long long probes = 0;  // (up to kp1 per iteration)
    long long evals_part = 0;  // per-lane unvisited-neighbour count (COUNT mode)
    int exhausted = 0;
    // lane-local neighbours excluded from the argmin: a > k (not neighbours) and the undo
    // move of the last step (the previous pivot is always in the filter)
    uint32_t inval = 0;
#pragma unroll
    for (int m = 0; m < R; ++m)
        if (a0 + 8 * m > k) inval |= 1u << m;
    uint32_t skip = inval;
    const int64_t t_i = (COUNT && score_out) ? 1 : P.t_i;
    bool active = valid;  // this segment's walk is still running

    const int t_i32 = (int)t_i;  // T_i < 2^28 (make_walk_params: Bloom bits < 2^32)
#ifdef LABS_PHASE_CLOCKS
    long long ph_g = 0, ph_arg = 0, ph_apply = 0, ph_t = clock64();
#define LABS_PHASE(acc) { const long long _t = clock64(); acc += _t - ph_t; ph_t = _t; }
#else
#define LABS_PHASE(acc)
#endif
    for (int it = 0;; ++it) {
        const bool cont = active && it < t_i32;
        if (!sg.uni(cont)) break;
        // ---- G for all owned neighbours (the O(L) part: IDP4A sliding dot product) ----
        int acc[R];
#pragma unroll
        for (int m = 0; m < R; ++m) acc[m] = 0;
        if (sg.uni(wide && cont)) {  // G = 256 G_high + G_low (a narrow segment passes zeros)
            g_neighbours<R>(Xw, w.KH, P.nwx, kb, ksel, acc);
#pragma unroll
            for (int m = 0; m < R; ++m) acc[m] = wide ? acc[m] * 256 : 0;
        }
        g_neighbours<R>(Xw, w.KL, P.nwx, kb, ksel, acc);
        if (wide && cont) ++wide_iters;
        // ---- exact deltas: dE(a) = T(a) - xs(a) G(a) ----
        int delta[R];
#pragma unroll
        for (int m = 0; m < R; ++m)  // the key if one_key
            delta[m] = (int)(T[m] + (uint32_t)xs[m] * (uint32_t)acc[m]);
        if (COUNT && score_out) {
            if (valid)
#pragma unroll
                for (int m = 0; m < R; ++m)
                    if (a0 + 8 * m <= k)
                        score_out[walk * kp1 + a0 + 8 * m] =
                            one_key ? (int)((uint32_t)delta[m] - kbase - 8u * m) >> 9 : delta[m];
            break;
        }

        LABS_PHASE(ph_g)
        // ---- choose: lowest (delta, hp) among unvisited (best_neighbour, saw.cpp:106-115) ----
        if (COUNT && cont) {
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if (a0 + 8 * m > k) continue;  // in `inval`
                const int a = a0 + 8 * m;
                const uint64_t n1 = h1 ^ fm0[a], n2 = h2 ^ fm1[a];
                bool hit = true;
                for (int i = 0; i < P.bloom_k; ++i) {
                    const uint32_t idx = bloom_index(n1, n2, i, P.bloom_mu, P.bloom_bits);
                    if (!((w.bloom[idx >> 5] >> (idx & 31)) & 1)) {
                        hit = false;
                        break;
                    }
                }
                if (hit) skip |= 1u << m;
                else ++evals_part;
            }
        }
        // lane minimum, lowest m first; `skip` excludes the undo move (the previous pivot
        // is always in the filter) without a Bloom probe, and the non-neighbours a > k.
        // For L <= 1001, |dE| < 2^22 and one unsigned key (dE + 2^22) << 9 | a orders
        // (delta, hp) lexicographically, so one segment minimum finds the winner.
        int dstar = 0, astar = -1;
        uint32_t ins_idx = 0, ins_idx2 = 0;  // Bloom bits of the accepted neighbour (insert)
        uint32_t bkey = 0xffffffffu;
        int bd = INT_BIG, bm = 0;
        if (one_key) {
            bkey = lane_min_key<R>(delta, skip);
        } else {
#pragma unroll
            for (int m = 0; m < R; ++m)
                if (!(skip & (1u << m)) && delta[m] < bd) {
                    bd = delta[m];
                    bm = m;
                }
        }
        bool need = cont;  // this segment still has to pick its neighbour
        while (sg.uni(need)) {
            int md, ma;
            bool mine_won;
            if (one_key) {
                const uint32_t k_best = sg.umin(bkey);
                ma = (int)(k_best & 511u);
                md = (int)(k_best >> 9) - (1 << 22);
                mine_won = bkey == k_best;
                if (k_best == 0xffffffffu) need = false;  // every free neighbour visited
            } else {
                md = sg.imin(bd);
                const int mine = (bd == md) ? a0 + 8 * bm : INT_BIG;
                ma = sg.imin(mine);
                mine_won = mine == ma;
                if (md == INT_BIG) need = false;
            }
            if (LPW == 32 && !need) break;  // (warp-uniform with one segment per warp)
            const int mac = need ? ma : P.p;  // a safe index for segments not probing
            const uint64_t n1 = h1 ^ fm0[mac], n2 = h2 ^ fm1[mac];
            bool bit = true;
            if (LPW >= 32 || sl < P.bloom_k) {  // hash index sl (and sl + LPW for 8 lanes)
                const uint32_t idx = bloom_index(n1, n2, sl, P.bloom_mu, P.bloom_bits);
                if (sl < P.bloom_k) {
                    bit = (w.bloom[idx >> 5] >> (idx & 31)) & 1;
                    if (need) ins_idx = idx;  // kept for the insert if accepted
                }
                if (LPW < 16 && sl + LPW < P.bloom_k) {  // (bloom_k <= 2 LPW, host-checked)
                    const uint32_t idx2 = bloom_index(n1, n2, sl + LPW, P.bloom_mu, P.bloom_bits);
                    bit = bit && ((w.bloom[idx2 >> 5] >> (idx2 & 31)) & 1);
                    if (need) ins_idx2 = idx2;
                }
            }
            if (COUNT) {  // already filtered: the minimum is unvisited
                if (need) {
                    dstar = md;
                    astar = ma;
                }
                need = false;
                continue;
            }
            const bool visited = sg.all(bit);
            if (need) ++probes;
            if (need && visited) {
                if (mine_won) {  // drop the visited neighbour, recompute this lane's minimum
                    skip |= 1u << ((ma - a0) >> 3);
                    if (one_key) {
                        bkey = lane_min_key<R>(delta, skip);
                    } else {
                        bd = INT_BIG;
                        bm = 0;
#pragma unroll
                        for (int m = 0; m < R; ++m)
                            if (!(skip & (1u << m)) && delta[m] < bd) {
                                bd = delta[m];
                                bm = m;
                            }
                    }
                }
            } else if (need) {
                dstar = md;
                astar = ma;
                need = false;
            }
        }
        if (cont && astar < 0) {
            exhausted = 1;
            active = false;
        }
        const bool step = cont && astar >= 0;  // segment-uniform

        LABS_PHASE(ph_arg)
        // ---- apply the skew flip at astar (apply_skew_flip, skew.cpp:95-105) ----
        if (step) ++iterations;
        const int as = step ? astar : P.p;  // addresses stay in range for idle segments
        const bool cen = as == k;
        const int bstar = L - 1 - as;
        const int apar = as & 1, ah = as >> 1;
        int8_t* Xa = (apar ? w.X1 : w.X0) + P.xoff;
        const int xa = Xa[ah];
        const int xb = cen ? 0 : (((k - as) & 1) ? -xa : xa);
        const int dstar_l = as - a0;  // == 8m for the owner of astar
        // hashes of the new pivot and its Bloom insert depend on nothing below: issue them
        // first so they overlap the apply (the insert reuses the accepted probe's index)
        if (step) {
            h1 ^= fm0[as];
            h2 ^= fm1[as];
            hf ^= fmf[as];
            energy += dstar;
            best = min(best, energy);
        }
        // Bloom insert: lanes without a hash OR 0 into a valid word (no divergent branch)
        atomicOr(&w.bloom[ins_idx >> 5], (step && sl < P.bloom_k) ? 1u << (ins_idx & 31) : 0u);
        if (LPW < 16)
            atomicOr(&w.bloom[ins_idx2 >> 5], (step && sl + LPW < P.bloom_k) ? 1u << (ins_idx2 & 31) : 0u);
        // (1) zero x_a and x_b: the Q pairs below and the C windows then read 0 there,
        //     which is exactly the fused rule's treatment of the flipped pair
        __syncwarp();
        {  // (lane 0 x_a*, lane 1 x_b*; the other lanes write byte -1 of the zero padding)
            int zi = sl == 1 ? (bstar >> 1) : ah;
            zi = (step && sl < 2) ? zi : -1;
            Xa[zi] = 0;
        }
        __syncwarp();
        // (2) T updates, all from the (zeroed) pre-step sequence, so their loads issue together
        //     with the C update's:
        //   C term: T(a) += 8 (-1)^(k-a) dc_{k-a}, dc_t = mul (x_{a*+2t} + x_{a*-2t}); the zeroed
        //     x_a*, x_b* make t = 0 (the centre) and t = k-a* (the fused rule) come out right.
        //   Q pairs through the flipped positions, neighbours of astar's parity:
        //     dQ(a) = -x_a* x_{2a-a*} - x_b* x_{2a-b*}, except the pair excluded from Q(a)
        //     (its upper element is L-1-a, i.e. a* = 3a - (L-1)).  The centre's Q never
        //     changes (its only pair through a* is (a*, b*), both zeroed).
        const int mul = cen ? -2 * xa : -4 * xa;
        if (step) {
            // One convergent loop for both updates.  For a of a*'s parity the Q partner
            // x_{2a-b*} is the C-term's x_{a*-2t} (2a - b* = a* - 2(k-a)), so three byte
            // loads per neighbour serve both; lanes of the other parity take the Q part
            // with zero factors instead of diverging.
            const int8_t* Xf = Xa + ah + (k - a0);  // x_{a*+2t}, t = k - a = (k - a0) - 8m
            const int8_t* Xg = Xa + ah - (k - a0);  // x_{a*-2t}  (= x_{2a-b*})
            const int8_t* Xp = Xa + ((2 * a0 - as) >> 1);  // x_{2a-a*}
            const int cmul = sgn8 * mul * sc;
            const bool same = par == apar;  // (the owner of astar has astar's parity)
            const int qa = same ? -64 * sc * xa : 0, qb = same ? -64 * sc * xb : 0;
            const int ex3 = as + L - 1;  // == 3a for the pair excluded from Q(a)
            // the pivot's own entry (undo move): no Q change, xs flips, skipped next step
            const bool own_lane = same && dstar_l >= 0 && (dstar_l & 7) == 0 && dstar_l < 8 * R;
            skip = inval | (own_lane ? 1u << (dstar_l >> 3) : 0u);
#pragma unroll
            for (int m = 0; m < R; ++m) {
                const int f = Xf[-8 * m], g = Xg[8 * m];
                int xp = Xp[8 * m];
                if (3 * (a0 + 8 * m) == ex3) xp = 0;
                const bool own = dstar_l == 8 * m;  // (x_{2a*-a*} = x_{a*} reads the zeroed 0)
                T[m] += (uint32_t)(cmul * (f + g) + qa * xp + qb * (own ? 0 : g));
                const int om = own ? -1 : 0;  // (negation on the ALU: (x ^ -1) + 1)
                xs[m] = (xs[m] ^ om) - om;
            }
        }
        // (3) even-lag C update, lanes over lag words: dc_t = mul (x_{a+2t} + x_{a-2t})
        int cmx = 0, esp = 0;
        if (step) {
            const uint32_t* Xaw = apar ? w.X1w : w.X0w;
            const int awF = (P.xoff + ah + 1) >> 2;
            const uint32_t asF = sel4((P.xoff + ah + 1) & 3);
            const int awB = (P.xoff + ah - 4) >> 2;
            const uint32_t asB = sel4r((P.xoff + ah) & 3);
            // C_b += mul x_{a+2t} + mul x_{a-2t} as two IDP4A with the one-hot int8 selector
            // mul e_b (no byte unpacking)
            const uint32_t mb = (uint32_t)mul & 0xffu;
            int e1h[4];
#pragma unroll
            for (int b = 0; b < 4; ++b)  // mul in byte b, zeros elsewhere (PRMT, not a shift)
                e1h[b] = (int)prmt(mb, 0u, 0x4444u ^ (0x4u << (4 * b)));
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) {
                const int s = sl + LPW * jj;
                if (jj < nj) {  // (lanes past S: zero windows, C stays 0 -- no divergence)
                    const uint32_t fw = prmt(Xaw[awF + s], Xaw[awF + s + 1], asF);
                    const uint32_t bw = prmt(Xaw[awB - s], Xaw[awB - s + 1], asB);
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        C[jj][b] = __dp4a((int)fw, e1h[b], __dp4a((int)bw, e1h[b], C[jj][b]));
                    // bits above 7 of C + 128 set <=> |C| > 127 (wide kernel bytes needed)
                    cmx |= ((C[jj][0] + 128) | (C[jj][1] + 128)) | ((C[jj][2] + 128) | (C[jj][3] + 128));
                }
            }
        }
        const bool wide_next = sg.any((cmx & ~0xff) != 0);
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
            const int up = __shfl_up_sync(FULLMASK, C[jj][3], 1, LPW);
            const int wrap = __shfl_sync(FULLMASK, jj > 0 ? C[jj > 0 ? jj - 1 : 0][3] : 0, LPW - 1, LPW);
            const int s = sl + LPW * jj;
            const int cprev = s == 0 ? 0 : (sl == 0 ? wrap : up);
            if (step && jj < nj) store_k_word(w, P, s, C[jj], cprev, wide_next);  // (zeros past S)
        }
        if (step) wide = wide_next;
        __syncwarp();
        // (4) write the flipped pair, hashes, Bloom insert
        if (step) {
            if (sl == 0) Xa[ah] = (int8_t)(-xa);
            if (sl == 1 && !cen) Xa[bstar >> 1] = (int8_t)(-xb);
            if (sl == 2) w.half[as >> 5] ^= 1u << (as & 31);
        }
        if (dbg) {  // (debug_check_energy: E re-derived from the C registers every step)
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj)
                if (step && jj < nj && sl + LPW * jj < S)
#pragma unroll
                    for (int b = 0; b < 4; ++b) esp += C[jj][b] * C[jj][b];
            const int echk = sg.sum(esp);
            if (step && echk != energy) ++diverged;  // (energy already includes dstar)
        }
        __syncwarp();
        LABS_PHASE(ph_apply)
        const bool hit = step && energy < P.e_l;
        if (sg.uni(hit)) {  // K2: warp-aggregated compaction into the record ring
            // one atomicAdd per warp for the hits of all its segments: the segment leaders'
            // ballot gives the count and each segment's rank
            const uint32_t lead = __ballot_sync(FULLMASK, hit && sl == 0);
            const int first = __ffs(lead) - 1;
            unsigned long long base = 0;
            if (sg.lane == first) base = atomicAdd(P.rec_count, (unsigned long long)__popc(lead));
            base = __shfl_sync(FULLMASK, base, first);
            const unsigned long long slot =
                base + (unsigned long long)__popc(lead & ((1u << sg.base) - 1u));
            // a slot past the ring's first lap waits until the host has drained everything up
            // to slot - rec_cap (rec_tail).  The wait loop exits on a warp vote, so the walk
            // loop stays provably converged; after kRingWaitSpins sleeps of ~4 us (~20 s) it
            // gives up and raises ctl[0] (the host fails the call instead of hanging).
            bool wait = hit && slot >= (unsigned long long)P.rec_cap;
            bool wrote = hit;
            unsigned spins = 0;
            while (__any_sync(FULLMASK, wait)) {
                if (wait) {
                    const unsigned long long tail = *(volatile const unsigned long long*)P.rec_tail;
                    if (slot < tail + (unsigned long long)P.rec_cap) {
                        wait = false;
                    } else if (++spins >= kRingWaitSpins) {
                        atomicOr(&P.ctl[0], 1);
                        wait = wrote = false;
                    }
                }
                __nanosleep(4000);
            }
            if (hit) {
                ++emitted;
                if (wrote) {
                    uint32_t* r = P.rec + (slot & (unsigned long long)(P.rec_cap - 1)) *
                                              (unsigned long long)P.rec_words;
                    if (sl == 0) {
                        r[0] = (uint32_t)walk;
                        r[1] = (uint32_t)(it + 1);
                        r[2] = (uint32_t)energy;
                        r[3] = 0;
                        r[4] = (uint32_t)hf;
                        r[5] = (uint32_t)(hf >> 32);
                    }
                    for (int i = sl; i < P.hw; i += LPW) r[kRecHeader + i] = w.half[i];
                    __threadfence();  // each writer's record words before the tag
                }
            }
            __syncwarp();
            if (wrote && sl == 0)
                P.rec_tag[slot & (unsigned long long)(P.rec_cap - 1)] = (uint32_t)(P.rec_seq0 + slot + 1);
        }
    }
#ifdef LABS_PHASE_CLOCKS
    if (walk < 4 && sl == 0 && valid)
        printf("[phase] walk %lld iters %lld  G %.0f  argmin+probe %.0f  apply %.0f cycles/iter\n",
               (long long)walk, (long long)iterations, (double)ph_g / iterations, (double)ph_arg / iterations,
               (double)ph_apply / iterations);
#endif
#undef LABS_PHASE
    if (COUNT) evals_part = sg.sum64(evals_part);
    if (valid && sl == 0 && P.walk_stats) {
        int64_t* st = P.walk_stats + walk * kWalkStatWords;
        st[kWsIterations] = iterations;
        st[kWsEmitted] = emitted;
        st[kWsBest] = best;
        st[kWsInitial] = e0;
        st[kWsExhausted] = exhausted;
        st[kWsDeltaEvals] = (COUNT && P.count_visited) ? evals_part : -1;
        st[kWsVisitedProbes] = probes;
        st[kWsWideIters] = wide_iters;
        st[kWsDiverged] = diverged;
    }
    __syncwarp();
}

// Resident 128-thread blocks per SM the register allocation is sized for.  Per lane the
// state grows with R (neighbours) and the lag words; wider lanes get more registers
// instead of spilling.
template <int R, int LPW>
struct MinBlocks {
    // (4 blocks = 128 registers: R <= 14 fits without spills since the wide pass shares
    // the narrow pass's accumulators; 3 blocks = 168 registers for R = 15, 16)
    static constexpr int value =
        R <= 6 ? 5 : (R <= 8 ? 4 : (LPW == 16 ? (R <= 14 ? 4 : 3) : (R <= 16 ? 3 : 2)));
};

template <int R, int LPW, bool COUNT>
__global__ void __launch_bounds__(128, (MinBlocks<R, LPW>::value))
    saw_walk_kernel(WalkParams P, int* score_out, int* corr_out) {
    extern __shared__ uint4 smem_u4[];
    // flip-mask table: a block copy in shared memory, or (when that copy would cost a
    // resident block) read through L1 -- P.fm_words decides (walk_blocks_per_sm)
    const uint64_t* fm = P.fm;
    if (P.fm_words) {
        uint64_t* fs = reinterpret_cast<uint64_t*>(smem_u4);
        for (int i = threadIdx.x; i < 3 * P.kp1; i += blockDim.x) fs[i] = P.fm[i];
        __syncthreads();
        fm = fs;
    }
    constexpr int SEGS = Seg<LPW>::kSegs;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Seg<LPW> sg(lane);
    const int seg = lane / LPW;
    uint32_t* base = reinterpret_cast<uint32_t*>(smem_u4) + P.fm_words +
                     (warp * SEGS + seg) * P.warp_words;
    WarpSmem w;
    w.X0w = base;
    w.X1w = base + P.off_x1;
    w.X0 = reinterpret_cast<int8_t*>(w.X0w);
    w.X1 = reinterpret_cast<int8_t*>(w.X1w);
    w.KL = base + P.off_kl;
    w.KH = base + P.off_kh;
    w.C16 = base + P.off_c16;
    w.KQ = reinterpret_cast<int*>(base + P.off_kq);
    w.half = base + P.off_half;
    w.bloom = base + P.off_bloom;
    // walk groups (one per warp: SEGS walks) are handed out dynamically -- walks differ in
    // length (exhaustion, Bloom retries), so a static stride leaves SMs idle at the tail
    const int64_t nwarps = (int64_t)gridDim.x * P.warps_per_block;
    int64_t grp = (int64_t)blockIdx.x * P.warps_per_block + warp;
    while (grp * SEGS < P.nwalks) {
        if (*(volatile int*)&P.ctl[1]) break;  // cancelled by the host (pool stopped)
        const int64_t walk = grp * SEGS + seg;
        run_walk_seg<R, LPW, COUNT>(P, w, fm, fm + P.kp1, fm + 2 * P.kp1, walk, walk < P.nwalks,
                                    sg, score_out, corr_out);
        unsigned long long nx = 0;
        if (lane == 0) nx = atomicAdd(P.walk_next, 1ull);
        grp = nwarps + (int64_t)__shfl_sync(FULLMASK, nx, 0);
    }
}

// Per-(R, LPW) launch / occupancy helpers, explicitly instantiated in saw_walk_r*.cu so
// that the variants compile in parallel translation units.
template <int R, int LPW>
cudaError_t launch_walk_fixed(const WalkParams& P, int grid, size_t smem, cudaStream_t st,
                              int* score_out, int* corr_out, bool count) {
    // (the COUNT kernel also serves the diagnostic options: the plain one never tests them)
    const bool chk = count || P.debug_check || score_out || corr_out;
    auto kfn = chk ? saw_walk_kernel<R, LPW, true> : saw_walk_kernel<R, LPW, false>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, P.warps_per_block * 32, smem, st>>>(P, score_out, corr_out);
    return cudaGetLastError();
}

template <int R, int LPW>
int blocks_per_sm_fixed(const WalkParams& P, size_t smem) {
    int n = 0;
    cudaFuncSetAttribute(saw_walk_kernel<R, LPW, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, saw_walk_kernel<R, LPW, false>,
                                                      P.warps_per_block * 32, smem) != cudaSuccess)
        return 0;
    return n;
}

}  // namespace labs_b200
