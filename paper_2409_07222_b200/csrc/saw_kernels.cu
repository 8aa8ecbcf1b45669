// saw_kernels.cu -- sm_100a kernels for Step 1 of the dual-step LABS search.
//
// K1 saw_walk_kernel : one warp = one self-avoiding walk (run_walk, saw.cpp:117-149).
//                      Fuses the Bloom probe, the skew flip-delta of every free
//                      neighbour (skew_flip_delta_fast, skew.cpp:60-93), the
//                      lexicographic argmin (best_neighbour, saw.cpp:106-115), the
//                      apply (apply_skew_flip, skew.cpp:95-105), the Bloom insert
//                      and the E < E_l sieve with compaction into a device
//                      record buffer (sink.emit, saw.cpp:143-146).
// K3 saw_seed_kernel : xoshiro256** streams -> initial halves
//                      (Rng + init_partitioned_sequence, rng.hpp:21-45, saw.cpp:65-75).
//
// Arithmetic.  For a skew-symmetric pivot the four sign products of
// the reference's fused delta pair up (x_b x_{b+-kk} = x_a x_{a-+kk}), so for half
// index a < k:
//     dE(a) = 16 N(a) + 32 Q(a) - 8 x_a (DP(a) - 2 Csum) + 8 (-1)^(k-a) C_{k-a}
// and for the centre a = k:  dE = 4 N + 8 Q - 4 x_k (DP - 2 Csum), with
//     DP(a) = sum_t C_{2t} (y_{a-2t} + y_{a+2t}),  y = x + 1 in {0,1,2}, 1 = padding,
//     Csum = sum_t C_{2t},  N(a) = #valid single terms,  Q(a) = sum_t x_{a-2t} x_{a+2t}.
// DP is the only O(L) part: 4 lags per IDP4A on byte-packed y words (int8 C), or per
// two IDP2A (int16 C) while some |C| > 127.  Q is maintained incrementally (O(1) per
// neighbour per flip).  Everything is exact integer arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>

#include "saw_device.h"

namespace labs_b200 {

#define FULLMASK 0xffffffffu

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    return __byte_perm(a, b, sel);
}

// (h1 + i*h2) mod 2^64 mod m  (bloom.cpp:28,36), Barrett with mu = floor(2^64/m), m < 2^32
__device__ __forceinline__ uint32_t bloom_index(uint64_t h1, uint64_t h2, uint32_t i, uint64_t mu,
                                                uint32_t m) {
    const uint64_t x = h1 + (uint64_t)i * h2;
    const uint64_t q = __umul64hi(x, mu);
    const uint64_t r = x - q * (uint64_t)m;
    return (uint32_t)(r >= m ? r - m : r);
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

// y = x+1 byte -> x in {-1,0,1} per byte (no inter-byte carries: y+0x7F <= 0x81)
__device__ __forceinline__ uint32_t y_to_x(uint32_t y) { return (y + 0x7F7F7F7Fu) ^ 0x80808080u; }

// ---------------------------------------------------------------------------
// Main O(L) loop: DP(a) for this lane's R neighbours a = a0 + 8m.
// Fw: this lane's parity array (32-bit words).  Forward bytes for neighbour m at
// step s live in words wF+s+m (+1), backward bytes in words wB+m-s (+1); the
// PRMT'd forward/backward words slide by one word per step, so each new step
// loads one forward and one backward word and reuses the rest from registers.
template <int R, bool WIDE>
__device__ __forceinline__ void dp_step(const uint32_t* __restrict__ Fw,
                                        const uint32_t* __restrict__ Cw, int s, int j, int wF,
                                        int wB, uint32_t selF, uint32_t selB, uint32_t (&PF)[R],
                                        uint32_t (&PB)[R], uint32_t& rfl, uint32_t& rbf,
                                        int (&acc)[R]) {
    uint32_t c0, c1;
    if (WIDE) {
        const uint2 cc = *reinterpret_cast<const uint2*>(Cw + 2 * s);
        c0 = cc.x;
        c1 = cc.y;
    } else {
        c0 = Cw[s];
        c1 = 0;
    }
    const uint32_t nf = Fw[wF + s + R + 1];
    const uint32_t nb = Fw[wB - s - 1];
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const uint32_t y = PF[(j + m) % R] + PB[(m - j + R) % R];
        if (WIDE) {
            acc[m] = __dp2a_lo((int)c0, (int)y, acc[m]);
            acc[m] = __dp2a_hi((int)c1, (int)y, acc[m]);
        } else {
            acc[m] = __dp4a((int)y, (int)c0, acc[m]);
        }
    }
    PF[j] = prmt(rfl, nf, selF);
    rfl = nf;
    PB[(R - 1 - j) % R] = prmt(nb, rbf, selB);
    rbf = nb;
}

template <int R, bool WIDE>
__device__ __forceinline__ void dp_neighbours(const uint32_t* __restrict__ Fw,
                                              const uint32_t* __restrict__ Cw, int S, int wF,
                                              int wB, uint32_t selF, uint32_t selB,
                                              int (&acc)[R]) {
    uint32_t PF[R], PB[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
        PF[q] = prmt(Fw[wF + q], Fw[wF + q + 1], selF);
        PB[q] = prmt(Fw[wB + q], Fw[wB + q + 1], selB);
        acc[q] = 0;
    }
    uint32_t rfl = Fw[wF + R];
    uint32_t rbf = Fw[wB];
    const int nfull = (S / R) * R;
    for (int s0 = 0; s0 < nfull; s0 += R) {
#pragma unroll
        for (int j = 0; j < R; ++j)
            dp_step<R, WIDE>(Fw, Cw, s0 + j, j, wF, wB, selF, selB, PF, PB, rfl, rbf, acc);
    }
    if (nfull < S) {
#pragma unroll
        for (int j = 0; j < R; ++j)
            if (nfull + j < S)
                dp_step<R, WIDE>(Fw, Cw, nfull + j, j, wF, wB, selF, selB, PF, PB, rfl, rbf, acc);
    }
}

// ---------------------------------------------------------------------------
struct WarpSmem {
    uint32_t* F;      // [2][nwp] parity byte arrays (y = x+1, pad 1)
    uint8_t* Fb;
    uint32_t* C8;     // [S] int8 x4 packed C_{2t}, t = 4s+1..4s+4
    uint32_t* C16;    // [2S] int16 x2 packed
    uint32_t* half;   // [hw] half bits
    uint32_t* bloom;  // [bloom_words]
};

__device__ __forceinline__ int ybyte(const WarpSmem& w, const WalkParams& P, int j) {
    return w.Fb[(j & 1) * P.nwp * 4 + P.off + (j >> 1)];
}

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
// even lags; odd lags of a skew sequence vanish).
__device__ __forceinline__ int corr_even_lag(const WarpSmem& w, const WalkParams& P, int t) {
    int acc = 0;
    const int o = t & 3, dw = t >> 2;
    const uint32_t sel = (uint32_t)(o | ((o + 1) << 4) | ((o + 2) << 8) | ((o + 3) << 12));
#pragma unroll
    for (int par = 0; par < 2; ++par) {
        const uint32_t* Fw = w.F + par * P.nwp;
        const int imax = (P.L - 1 - par) >> 1;  // last logical index holding a real position
        const int n0 = P.off >> 2, n1 = (P.off + imax) >> 2;
        for (int n = n0; n <= n1; ++n) {
            const uint32_t xa = y_to_x(Fw[n]);
            const uint32_t xb = y_to_x(prmt(Fw[n + dw], Fw[n + dw + 1], sel));
            acc = __dp4a((int)xa, (int)xb, acc);
        }
    }
    return acc;
}

template <int R, bool COUNT>
__device__ void run_walk_warp(const WalkParams& P, const WarpSmem& w, const uint64_t* fm0,
                              const uint64_t* fm1, int64_t walk, int lane, int* score_out,
                              int* corr_out) {
    const int L = P.L, k = P.k, kp1 = P.kp1, S = P.S;
    const int nj = (S + 31) >> 5;  // steps owned per lane (<= 4)

    // ---- load the initial half, build parity arrays, clear Bloom ----
    const uint32_t* src = P.halves + walk * P.hw;
    for (int i = lane; i < P.hw; i += 32) w.half[i] = src[i];
    __syncwarp();
    for (int wi = lane; wi < 2 * P.nwp; wi += 32) {
        const int par = wi >= P.nwp;
        const int word = wi - par * P.nwp;
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int li = word * 4 + b - P.off;
            const int j = 2 * li + par;
            const int y = (li >= 0 && j < L) ? x_of_half(w.half, k, j) + 1 : 1;
            v |= (uint32_t)y << (8 * b);
        }
        w.F[wi] = v;
    }
    {
        uint4* b4 = reinterpret_cast<uint4*>(w.bloom);
        for (int i = lane; i < (P.bloom_words >> 2); i += 32) b4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();

    // ---- C_{2t} for owned steps (lanes over lags), E, Csum, max|C| ----
    int c[4][4];
    int e_part = 0, csum_part = 0, cmax = 0;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
        const int s = lane + 32 * jj;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int t = 4 * s + 1 + b;
            int v = 0;
            if (jj < nj && s < S && t <= k) v = corr_even_lag(w, P, t);
            c[jj][b] = v;
            e_part += v * v;
            csum_part += v;
            cmax = max(cmax, abs(v));
        }
    }
    int energy = warp_sum(e_part);
    int csum = warp_sum(csum_part);
    bool wide = __reduce_max_sync(FULLMASK, (unsigned)cmax) > 127u;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
        const int s = lane + 32 * jj;
        if (jj < nj && s < S) {
            const uint32_t p01 = prmt((uint32_t)c[jj][0], (uint32_t)c[jj][1], 0x0040);
            const uint32_t p23 = prmt((uint32_t)c[jj][2], (uint32_t)c[jj][3], 0x0040);
            w.C8[s] = prmt(p01, p23, 0x5410);
            w.C16[2 * s] = prmt((uint32_t)c[jj][0], (uint32_t)c[jj][1], 0x5410);
            w.C16[2 * s + 1] = prmt((uint32_t)c[jj][2], (uint32_t)c[jj][3], 0x5410);
            if (corr_out)
                for (int b = 0; b < 4; ++b)
                    if (4 * s + 1 + b <= k) corr_out[walk * k + 4 * s + b] = c[jj][b];
        }
    }

    // ---- lane geometry: neighbours a = a0 + 8m ----
    const int cgrp = lane & 7, g = lane >> 3;
    const int a0 = P.p + cgrp + 8 * R * g;
    const int par = a0 & 1, a0h = a0 >> 1;
    const uint32_t* Fw = w.F + par * P.nwp;
    const int wF = (P.off + a0h + 1) >> 2;
    const int oF = (P.off + a0h + 1) & 3;
    const uint32_t selF = (uint32_t)(oF | ((oF + 1) << 4) | ((oF + 2) << 8) | ((oF + 3) << 12));
    const int wB = (P.off + a0h - 4) >> 2;
    const int oB = (P.off + a0h) & 3;
    const uint32_t selB = (uint32_t)((oB + 3) | ((oB + 2) << 4) | ((oB + 1) << 8) | (oB << 12));

    // ---- Q(a) for owned neighbours ----
    int q[R];
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int a = a0 + 8 * m;
        int acc = 0;
        if (a <= k) {
            const uint8_t* Fb = w.Fb + par * P.nwp * 4 + P.off + (a >> 1);
            const int tstar = (a < k) ? (k - a) : -1;
            for (int t = 1; 2 * t <= a; ++t) {
                if (t == tstar) continue;
                acc += ((int)Fb[-t] - 1) * ((int)Fb[t] - 1);
            }
        }
        q[m] = acc;
    }

    // ---- half hashes h1, h2 (saw.cpp:77-89) and the initial Bloom insert ----
    uint64_t h1 = 0, h2 = 0;
    for (int i = lane; i < kp1; i += 32) {
        const int bit = (w.half[i >> 5] >> (i & 31)) & 1;
        h1 ^= P.tab[(0 * kp1 + i) * 2 + bit];
        h2 ^= P.tab[(1 * kp1 + i) * 2 + bit];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        h1 ^= shfl_xor64(h1, o);
        h2 ^= shfl_xor64(h2, o);
    }
    h1 ^= P.salt0;
    h2 ^= P.salt1;
    if (lane < P.bloom_k) {
        const uint32_t idx = bloom_index(h1, h2, lane, P.bloom_mu, P.bloom_bits);
        atomicOr(&w.bloom[idx >> 5], 1u << (idx & 31));
    }
    __syncwarp();

    const int e0 = energy;
    int best = energy;
    long long iterations = 0, emitted = 0, probes = 0, wide_iters = 0, diverged = 0;
    long long evals_part = 0;  // per-lane unvisited-neighbour count (COUNT mode)
    int exhausted = 0;
    int prev_hp = -1;
    const int64_t t_i = score_out ? 1 : P.t_i;

    for (long long it = 0; it < t_i; ++it) {
        // ---- DP for all owned neighbours ----
        int acc[R];
        if (wide) {
            dp_neighbours<R, true>(Fw, w.C16, S, wF, wB, selF, selB, acc);
            ++wide_iters;
        } else {
            dp_neighbours<R, false>(Fw, w.C8, S, wF, wB, selF, selB, acc);
        }
        // ---- epilogue: exact deltas ----
        int delta[R];
        uint32_t valid = 0;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int a = a0 + 8 * m;
            delta[m] = 0;
            if (a <= k) {
                valid |= 1u << m;
                const int xa = ybyte(w, P, a) - 1;
                const int n = (a >> 1) + ((L - 1 - a) >> 1) - (a < k ? 1 : 0);
                const int g2 = acc[m] - 2 * csum;
                int d;
                if (a < k) {
                    const int t = k - a;
                    const int ct = (int)reinterpret_cast<const int16_t*>(w.C16)[t - 1];
                    d = 16 * n + 32 * q[m] - 8 * xa * g2 + (((k - a) & 1) ? -8 : 8) * ct;
                } else {
                    d = 4 * n + 8 * q[m] - 4 * xa * g2;
                }
                delta[m] = d;
            }
        }
        if (score_out) {
#pragma unroll
            for (int m = 0; m < R; ++m)
                if (valid >> m & 1) score_out[walk * kp1 + a0 + 8 * m] = delta[m];
            break;
        }

        // ---- choose: lowest (delta, hp) among unvisited (best_neighbour) ----
        uint32_t excl = 0;
        if (COUNT) {
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if (!(valid >> m & 1)) continue;
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
                if (hit) excl |= 1u << m;
                else ++evals_part;
            }
        } else if (prev_hp >= 0) {
            // the undo move leads back to the previous pivot, which is in the filter
            const int r = prev_hp - P.p;
            if ((r & 7) == cgrp && ((r >> 3) / R) == g) excl |= 1u << ((r >> 3) % R);
        }
        int dstar = 0, astar = -1;
        while (true) {
            int bd = 0x7fffffff, ba = 0x7fffffff;
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if ((valid >> m & 1) && !(excl >> m & 1) && delta[m] < bd) {
                    bd = delta[m];
                    ba = a0 + 8 * m;
                }
            }
            const int md = __reduce_min_sync(FULLMASK, bd);
            if (md == 0x7fffffff) break;  // every free neighbour visited
            const int ma = __reduce_min_sync(FULLMASK, bd == md ? ba : 0x7fffffff);
            if (COUNT) {
                dstar = md;
                astar = ma;
                break;
            }
            ++probes;
            const uint64_t n1 = h1 ^ fm0[ma], n2 = h2 ^ fm1[ma];
            bool bit = true;
            if (lane < P.bloom_k) {
                const uint32_t idx = bloom_index(n1, n2, lane, P.bloom_mu, P.bloom_bits);
                bit = (w.bloom[idx >> 5] >> (idx & 31)) & 1;
            }
            if (__all_sync(FULLMASK, bit)) {
                if (ba == ma && bd == md) {
                    const int r = ma - P.p;
                    excl |= 1u << ((r >> 3) % R);
                }
                continue;
            }
            dstar = md;
            astar = ma;
            break;
        }
        if (astar < 0) {
            exhausted = 1;
            break;
        }

        // ---- apply the skew flip at astar (skew.cpp:95-105) ----
        ++iterations;
        const bool cen = astar == k;
        const int bstar = L - 1 - astar;
        const int xa = ybyte(w, P, astar) - 1;
        const int xb = ((k - astar) & 1) ? -xa : xa;
        {
            // even-lag correlation update: C_t += dc_t(astar), lanes over lags
            const int ah = astar >> 1, apar = astar & 1;
            const uint32_t* Fa = w.F + apar * P.nwp;
            const int awF = (P.off + ah + 1) >> 2, aoF = (P.off + ah + 1) & 3;
            const int awB = (P.off + ah - 4) >> 2, aoB = (P.off + ah) & 3;
            const uint32_t asF =
                (uint32_t)(aoF | ((aoF + 1) << 4) | ((aoF + 2) << 8) | ((aoF + 3) << 12));
            const uint32_t asB =
                (uint32_t)((aoB + 3) | ((aoB + 2) << 4) | ((aoB + 1) << 8) | (aoB << 12));
            const int tstar = cen ? -1 : (k - astar);
            const int mul = cen ? -2 * xa : -4 * xa;
            int csp = 0, cmx = 0, esp = 0;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int s = lane + 32 * jj;
                if (jj < nj && s < S) {
                    const uint32_t y = prmt(Fa[awF + s], Fa[awF + s + 1], asF) +
                                       prmt(Fa[awB - s], Fa[awB - s + 1], asB);
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int t = 4 * s + 1 + b;
                        int v = (int)((y >> (8 * b)) & 0xFF) - 2;
                        if (t == tstar) v -= xb;
                        if (t <= k) c[jj][b] += mul * v;
                        csp += c[jj][b];
                        cmx = max(cmx, abs(c[jj][b]));
                        esp += c[jj][b] * c[jj][b];
                    }
                }
            }
            // incremental Q: flip astar, then bstar (sequential single flips)
            if (par == apar) {
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    const int a = a0 + 8 * m;
                    if (a > k) continue;
                    const int lim = L - 1 - a;  // b(a)
                    // flip 1: j = astar, old value xa
                    if (a != astar) {
                        const int jp = 2 * a - astar;
                        if (jp >= 0 && jp <= L - 1 && !(a < k && max(astar, jp) == lim))
                            q[m] -= 2 * xa * (ybyte(w, P, jp) - 1);
                    }
                    // flip 2: j = bstar, old value xb, after astar flipped
                    if (!cen && a != bstar) {
                        const int jp = 2 * a - bstar;
                        if (jp >= 0 && jp <= L - 1 && !(a < k && max(bstar, jp) == lim)) {
                            const int xjp = (jp == astar) ? -xa : (ybyte(w, P, jp) - 1);
                            q[m] -= 2 * xb * xjp;
                        }
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int s = lane + 32 * jj;
                if (jj < nj && s < S) {
                    const uint32_t p01 = prmt((uint32_t)c[jj][0], (uint32_t)c[jj][1], 0x0040);
                    const uint32_t p23 = prmt((uint32_t)c[jj][2], (uint32_t)c[jj][3], 0x0040);
                    w.C8[s] = prmt(p01, p23, 0x5410);
                    w.C16[2 * s] = prmt((uint32_t)c[jj][0], (uint32_t)c[jj][1], 0x5410);
                    w.C16[2 * s + 1] = prmt((uint32_t)c[jj][2], (uint32_t)c[jj][3], 0x5410);
                }
            }
            if (lane == 0) w.Fb[apar * P.nwp * 4 + P.off + ah] = (uint8_t)(1 - xa);
            if (lane == 1 && !cen)
                w.Fb[(bstar & 1) * P.nwp * 4 + P.off + (bstar >> 1)] = (uint8_t)(1 - xb);
            if (lane == 2) w.half[astar >> 5] ^= 1u << (astar & 31);
            csum = warp_sum(csp);
            wide = __reduce_max_sync(FULLMASK, (unsigned)cmx) > 127u;
            if (P.debug_check) {
                const int echk = warp_sum(esp);
                if (echk != energy + dstar) ++diverged;
            }
        }
        h1 ^= fm0[astar];
        h2 ^= fm1[astar];
        if (lane < P.bloom_k) {
            const uint32_t idx = bloom_index(h1, h2, lane, P.bloom_mu, P.bloom_bits);
            atomicOr(&w.bloom[idx >> 5], 1u << (idx & 31));
        }
        energy += dstar;
        best = min(best, energy);
        prev_hp = astar;
        __syncwarp();
        if (energy < P.e_l) {
            ++emitted;
            unsigned long long slot = 0;
            if (lane == 0) slot = atomicAdd(P.rec_count, 1ull);
            slot = __shfl_sync(FULLMASK, slot, 0);
            if ((long long)slot < P.rec_cap) {
                uint32_t* r = P.rec + slot * (unsigned long long)P.rec_words;
                if (lane == 0) {
                    r[0] = (uint32_t)walk;
                    r[1] = (uint32_t)(it + 1);
                    r[2] = (uint32_t)energy;
                    r[3] = 0;
                }
                for (int i = lane; i < P.hw; i += 32) r[kRecHeader + i] = w.half[i];
            }
        }
    }
    if (COUNT) evals_part = warp_sum64(evals_part);
    if (lane == 0 && P.walk_stats) {
        int64_t* st = P.walk_stats + walk * kWalkStatWords;
        st[kWsIterations] = iterations;
        st[kWsEmitted] = emitted;
        st[kWsBest] = best;
        st[kWsInitial] = e0;
        st[kWsExhausted] = exhausted;
        st[kWsDeltaEvals] = COUNT ? evals_part : -1;
        st[kWsVisitedProbes] = probes;
        st[kWsWideIters] = wide_iters;
        st[kWsDiverged] = diverged;
    }
    __syncwarp();
}

template <int R, bool COUNT>
#ifndef LABS_MIN_BLOCKS
#define LABS_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(128, LABS_MIN_BLOCKS) saw_walk_kernel(WalkParams P, int* score_out,
                                                       int* corr_out) {
    extern __shared__ uint4 smem_u4[];
    uint64_t* fm = reinterpret_cast<uint64_t*>(smem_u4);
    for (int i = threadIdx.x; i < 2 * P.kp1; i += blockDim.x) fm[i] = P.fm[i];
    __syncthreads();
    const int fm_words = ((2 * P.kp1 * 2) + 3) & ~3;  // u32 words, 16-byte aligned
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* base = reinterpret_cast<uint32_t*>(smem_u4) + fm_words + warp * P.warp_words;
    WarpSmem w;
    w.F = base;
    w.Fb = reinterpret_cast<uint8_t*>(base);
    w.C8 = base + P.off_c8;
    w.C16 = base + P.off_c16;
    w.half = base + P.off_half;
    w.bloom = base + P.off_bloom;
    const int64_t stride = (int64_t)gridDim.x * P.warps_per_block;
    for (int64_t walk = (int64_t)blockIdx.x * P.warps_per_block + warp; walk < P.nwalks;
         walk += stride)
        run_walk_warp<R, COUNT>(P, w, fm, fm + P.kp1, walk, lane, score_out, corr_out);
}

// ---------------------------------------------------------------------------
// K3: one thread per walker; restarts drawn in order from the walker's stream.
__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t rotl_dev(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

__global__ void saw_seed_kernel(SeedParams P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.nseg) return;
    uint64_t s0, s1, s2, s3;
    if (P.seg_init[i]) {
        uint64_t sm = P.seed ^ (0xa0761d6478bd642fULL * ((uint64_t)P.walker_ids[i] + 1));
        s0 = splitmix64_dev(sm);
        s1 = splitmix64_dev(sm);
        s2 = splitmix64_dev(sm);
        s3 = splitmix64_dev(sm);
    } else {
        s0 = P.rng_state[4 * i + 0];
        s1 = P.rng_state[4 * i + 1];
        s2 = P.rng_state[4 * i + 2];
        s3 = P.rng_state[4 * i + 3];
    }
    const uint32_t pre = P.prefix_bits[i];
    for (int64_t r = 0; r < P.seg_restarts[i]; ++r) {
        uint32_t* out = P.halves + (P.seg_offset[i] + r) * P.hw;
        uint32_t word = 0;
        for (int pos = 0; pos < P.kp1; ++pos) {
            uint32_t bit;
            if (pos < P.p) {
                bit = (pre >> pos) & 1u;
            } else {
                const uint64_t result = rotl_dev(s1 * 5, 7) * 9;  // xoshiro256** (rng.hpp:26-36)
                const uint64_t t = s1 << 17;
                s2 ^= s0;
                s3 ^= s1;
                s1 ^= s2;
                s0 ^= s3;
                s2 ^= t;
                s3 = rotl_dev(s3, 45);
                bit = (uint32_t)(result >> 63);  // next_sign (rng.hpp:45)
            }
            word |= bit << (pos & 31);
            if ((pos & 31) == 31) {
                out[pos >> 5] = word;
                word = 0;
            }
        }
        if (P.kp1 & 31) out[P.kp1 >> 5] = word;
        for (int wd = (P.kp1 + 31) >> 5; wd < P.hw; ++wd) out[wd] = 0;
    }
    P.rng_state[4 * i + 0] = s0;
    P.rng_state[4 * i + 1] = s1;
    P.rng_state[4 * i + 2] = s2;
    P.rng_state[4 * i + 3] = s3;
}

// ---------------------------------------------------------------------------
// host-side launchers (called from the C++ orchestration)
template <int R, bool COUNT>
static cudaError_t launch_walk_r(const WalkParams& P, int grid, size_t smem, cudaStream_t st,
                                 int* score_out, int* corr_out) {
    auto kfn = saw_walk_kernel<R, COUNT>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, P.warps_per_block * 32, smem, st>>>(P, score_out, corr_out);
    return cudaGetLastError();
}

template <bool COUNT>
static cudaError_t launch_walk_c(const WalkParams& P, int grid, size_t smem, cudaStream_t st,
                                 int* score_out, int* corr_out) {
    switch (P.R) {
#define LABS_CASE(r) \
    case r: return launch_walk_r<r, COUNT>(P, grid, smem, st, score_out, corr_out);
        LABS_CASE(1) LABS_CASE(2) LABS_CASE(3) LABS_CASE(4) LABS_CASE(5) LABS_CASE(6)
        LABS_CASE(7) LABS_CASE(8) LABS_CASE(9) LABS_CASE(10) LABS_CASE(11) LABS_CASE(12)
        LABS_CASE(13) LABS_CASE(14) LABS_CASE(15) LABS_CASE(16)
#undef LABS_CASE
        default: return cudaErrorInvalidValue;
    }
}

size_t walk_smem_bytes(const WalkParams& P) {
    const int fm_words = ((2 * P.kp1 * 2) + 3) & ~3;
    return (size_t)(fm_words + P.warps_per_block * P.warp_words) * 4;
}

cudaError_t launch_saw_walk(const WalkParams& P, int grid, cudaStream_t st, int* score_out,
                            int* corr_out) {
    const size_t smem = walk_smem_bytes(P);
    return P.count_visited ? launch_walk_c<true>(P, grid, smem, st, score_out, corr_out)
                           : launch_walk_c<false>(P, grid, smem, st, score_out, corr_out);
}

int walk_blocks_per_sm(const WalkParams& P) {
    int n = 0;
    const size_t smem = walk_smem_bytes(P);
    cudaError_t e;
    switch (P.R) {
#define LABS_CASE(r)                                                                          \
    case r:                                                                                   \
        cudaFuncSetAttribute(saw_walk_kernel<r, false>,                                       \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, saw_walk_kernel<r, false>,       \
                                                          P.warps_per_block * 32, smem);      \
        break;
        LABS_CASE(1) LABS_CASE(2) LABS_CASE(3) LABS_CASE(4) LABS_CASE(5) LABS_CASE(6)
        LABS_CASE(7) LABS_CASE(8) LABS_CASE(9) LABS_CASE(10) LABS_CASE(11) LABS_CASE(12)
        LABS_CASE(13) LABS_CASE(14) LABS_CASE(15) LABS_CASE(16)
#undef LABS_CASE
        default: return 0;
    }
    return e == cudaSuccess ? n : 0;
}

cudaError_t launch_saw_seed(const SeedParams& P, cudaStream_t st) {
    const int bs = 128;
    const int grid = (P.nseg + bs - 1) / bs;
    if (grid == 0) return cudaSuccess;
    saw_seed_kernel<<<grid, bs, 0, st>>>(P);
    return cudaGetLastError();
}

}  // namespace labs_b200
