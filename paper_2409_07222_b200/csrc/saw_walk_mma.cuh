// saw_walk_mma.cuh -- K1t, the tensor-core variant of the Step-1 walk kernel (sm_100a).
//
// Same walk as K1 (saw_walk.cuh: run_walk, saw.cpp:117-149, with the fused Bloom probe,
// skew flip-delta argmin, apply and sieve), one walk per warp, but the O(L) part of every
// flip delta -- the sliding dot product G(a) of the parity array with the symmetric
// correlation kernel K[d] = C_{2|d|} -- runs on the int8 tensor cores as
// mma.sync.m16n8k32.s8 instead of IDP4A.
//
// G as a GEMM.  For neighbour a = 2a' + par, a' = b0 + 8q + r (b0 = p/2, q = 0..15 per
// q-tile, r = 0..7):
//     G(a) = sum_d K[d] X_par[a' + d] = sum_kk A[q][kk] B_par[kk][r]
//     A[q][kk]     = K[kk - 8q - D]         (16 x 32 per k-step: the correlation kernel,
//                                            row q shifted by 8q bytes -- aligned words)
//     B_par[kk][r] = X_par[b0 + r + kk - D]  (32 x 8: the parity array, column r shifted
//                                            by r bytes -- read from 4 byte-shifted copies
//                                            of X_par so every fragment word is aligned)
// with D = b0 + 7 + delta (delta aligns A to words).  A is shared by both parities, so a
// k-step is two MMAs (one per parity) per q-tile; nks = ceil((k+1+7+delta)/32) k-steps
// cover every nonzero product.  The accumulator fragment gives lane (g, t) the neighbours
// a = A0 + {0, 2, 128, 130} (par 0) and A0 + {1, 3, 129, 131} (par 1), A0 = 2 b0 + 16 g + 4 t
// (+256 per q-tile).  Products are int8 x {-1, 0, 1} accumulated in int32: exact.  While
// some |C| > 127 a second pass runs on the high bytes (G = 256 G_hi + G_lo), as in K1.
//
// The rest of the step (key-scaled T registers, lexicographic argmin by REDUX, lazy Bloom
// probe, even-lag C update by one-hot IDP4A, hashes, sieve + K2 ring compaction) is K1's
// bookkeeping at 32 lanes per walk; DESIGN.md §4 has the instruction budget.
#pragma once
#include "saw_walk.cuh"

#ifndef LABS_MMA_MINB
#define LABS_MMA_MINB 5  // resident 128-thread blocks per SM the register budget targets (NQ = 1):
                         // 96 registers (a few spilled) -- 20 walks per SM beat 16 at 128
                         // registers by 5 % (L=451) and 4 % (L=527)
#endif

namespace labs_b200 {

// Debug builds (-DLABS_BOUNDS_CHECK, `make OUT=../_lib_check EXTRA=-DLABS_BOUNDS_CHECK`) check
// every shared-memory window index of K1t against its array and raise ctl[0] bit 1; the host
// then fails the call ("shared-memory bounds check failed").  compute-sanitizer is not
// available on this GPU pool, so the parity suite runs against that build as well.
#ifdef LABS_BOUNDS_CHECK
#define LABS_BC(P, i, lo, hi)                                                   \
    do {                                                                        \
        if ((i) < (lo) || (i) >= (hi)) atomicOr(const_cast<int*>(&(P).ctl[0]), 2); \
    } while (0)
#else
#define LABS_BC(P, i, lo, hi) \
    do {                      \
    } while (0)
#endif

__device__ __forceinline__ void mma_s8(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Per-walk shared-memory views of K1t (offsets: make_walk_params, kernel 1).  Pointers are
// computed from (parity, copy) arithmetically: an indexed pointer table would live in local
// memory.
struct MmaSmem {
    uint32_t* base;
    int off_x1, off_xc, xcw;
    uint32_t* KP;        // low kernel bytes: plain (KL, byte koff + d = low byte of C_{2|d|}) or,
                         // with P.kpl, in A-fragment pairs KP[2i] = KL[i], KP[2i+1] = KL[i-16]
    uint32_t* KH;        // high bytes, plain (byte koff + d = high byte of C_{2|d|})
    uint32_t* C16;       // (initialisation only, inside the Bloom words)
    int* KQ;
    uint32_t* half;
    uint32_t* bloom;
    __device__ __forceinline__ uint32_t* Xw(int par) const { return base + par * off_x1; }
    __device__ __forceinline__ int8_t* X(int par) const { return reinterpret_cast<int8_t*>(Xw(par)); }
    // copy c (1..3) of parity par: word i = X(par) bytes xcl + 4i + c .. +3
    __device__ __forceinline__ uint32_t* Xc(int par, int c) const {
        return base + off_xc + (par * 3 + c - 1) * xcw;
    }
};

// neighbour slot m of a lane: a = A0 + kOff8[m % 8] + 256 (m / 8); accumulator element
// kOff8 order: par 0 d0..d3, par 1 d0..d3
__device__ __forceinline__ constexpr int mma_off(int m) {
    return (m / 8) * 256 + ((m & 4) ? 1 : 0) + ((m & 1) ? 2 : 0) + ((m & 2) ? 128 : 0);
}

// G of this lane's 8 NQ neighbours: acc[jq][par][i] (i = accumulator element).  nks is even
// (make_walk_params pads with zero k-steps).  The A fragment of k-step s is {a0(s), a0(s-2),
// a2(s), a2(s-2)} (rows g+8 sit 64 bytes = two k-steps lower), so each step loads two kernel
// words and reuses two; even and odd steps accumulate in separate chains.
template <int NQ>
__device__ __forceinline__ void g_mma(const uint32_t* __restrict__ Kw, int nks, int kidx0, int xb,
                                      const uint32_t* __restrict__ xc0,
                                      const uint32_t* __restrict__ xc1, int (&acc)[NQ][2][4]) {
    int ac2[NQ][2][4];
    uint32_t p0[NQ][2], p2[NQ][2];  // a0, a2 of steps s - 2 (h = 0) and s - 1 (h = 1)
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
        const int ki = kidx0 - 32 * j;
        p0[j][0] = Kw[ki - 16];
        p2[j][0] = Kw[ki - 12];
        p0[j][1] = Kw[ki - 8];
        p2[j][1] = Kw[ki - 4];
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int i = 0; i < 4; ++i) ac2[j][p][i] = 0;
    }
    const uint32_t* kp = Kw + kidx0;
    const uint32_t* x0 = xc0 + xb;
    const uint32_t* x1 = xc1 + xb;
    const uint32_t* const kend = kp + 8 * nks;
#pragma unroll 1
    for (; kp != kend; kp += 16, x0 += 16, x1 += 16) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t b00 = x0[8 * h], b01 = x0[8 * h + 4];
            const uint32_t b10 = x1[8 * h], b11 = x1[8 * h + 4];
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
                const uint32_t c0 = kp[8 * h - 32 * j], c2 = kp[8 * h - 32 * j + 4];
                const uint32_t a[4] = {c0, p0[j][h], c2, p2[j][h]};
                p0[j][h] = c0;
                p2[j][h] = c2;
                if (h == 0) {
                    mma_s8(acc[j][0], a, b00, b01);
                    mma_s8(acc[j][1], a, b10, b11);
                } else {
                    mma_s8(ac2[j][0], a, b00, b01);
                    mma_s8(ac2[j][1], a, b10, b11);
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < NQ; ++j)
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[j][p][i] += ac2[j][p][i];
}

// Fully unrolled k-step loop for a compile-time nks (the common lengths): no loop control
// and no register moves for the a0/a2 rotation.
template <int NQ, int NKS>
__device__ __forceinline__ void g_mma_fixed(const uint32_t* __restrict__ Kw, int kidx0, int xb,
                                            const uint32_t* __restrict__ xc0,
                                            const uint32_t* __restrict__ xc1, int (&acc)[NQ][2][4]) {
    // one accumulator chain per (q-tile, parity): with 20 walks per SM the MMA latency is
    // hidden by the other warps, and the second chain's registers and merge are saved
    uint32_t w0[NQ][NKS + 2], w2[NQ][NKS + 2];  // a0 / a2 words of steps -2 .. NKS-1
#pragma unroll
    for (int j = 0; j < NQ; ++j)
#pragma unroll
        for (int s = -2; s < NKS; ++s) {
            w0[j][s + 2] = Kw[kidx0 - 32 * j + 8 * s];
            w2[j][s + 2] = Kw[kidx0 - 32 * j + 8 * s + 4];
        }
#pragma unroll
    for (int s = 0; s < NKS; ++s) {
        const uint32_t b00 = xc0[xb + 8 * s], b01 = xc0[xb + 8 * s + 4];
        const uint32_t b10 = xc1[xb + 8 * s], b11 = xc1[xb + 8 * s + 4];
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
            const uint32_t a[4] = {w0[j][s + 2], w0[j][s], w2[j][s + 2], w2[j][s]};
            mma_s8(acc[j][0], a, b00, b01);
            mma_s8(acc[j][1], a, b10, b11);
        }
    }
}

// G from the pair layout KP: the A fragment of k-step s is two 8-byte loads, {a0, a1} =
// KP[2i], KP[2i + 1] and {a2, a3} at i + 4 (i = kidx0 - 32 j + 8 s), straight into the
// MMA's register quad (no register moves).  NKS = 0: runtime nks.
template <int NQ, int NKS>
__device__ __forceinline__ void g_mma_kp(const uint32_t* __restrict__ KP, int nks, int kidx0, int xb,
                                         const uint32_t* __restrict__ xc0,
                                         const uint32_t* __restrict__ xc1, int (&acc)[NQ][2][4]) {
    const uint2* kp2 = reinterpret_cast<const uint2*>(KP) + kidx0;
    const int n = NKS > 0 ? NKS : nks;
#pragma unroll(NKS > 0 ? NKS : 2)
    for (int s = 0; s < n; ++s) {
        const uint32_t b00 = xc0[xb + 8 * s], b01 = xc0[xb + 8 * s + 4];
        const uint32_t b10 = xc1[xb + 8 * s], b11 = xc1[xb + 8 * s + 4];
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
            const uint2 lo = kp2[8 * s - 32 * j], hi = kp2[8 * s - 32 * j + 4];
            const uint32_t a[4] = {lo.x, lo.y, hi.x, hi.y};
            mma_s8(acc[j][0], a, b00, b01);
            mma_s8(acc[j][1], a, b10, b11);
        }
    }
}

// Kernel words of lag word s (see store_c_word): the low bytes plain or into both places of
// the pair layout (KPL: compile-time 1 / 0, or -1 = P.kpl), the high bytes (wide walks) plain.
template <int KPL>
__device__ __forceinline__ void store_kp_word(const MmaSmem& w, const WalkParams& P, int s,
                                              const int (&c)[4], int cprev, bool wide) {
    const int fw = (P.koff + 1) / 4 + s;
    const int bw = (P.koff - 3) / 4 - s;
    const uint32_t lo = pack4(c[0], c[1], c[2], c[3]);
    const uint32_t lob = prmt(lo, (uint32_t)cprev, 0x4012);  // (c2, c1, c0, cprev)
    if (KPL == 1 || (KPL < 0 && P.kpl)) {
        w.KP[2 * fw] = lo;
        w.KP[2 * fw + 33] = lo;
        w.KP[2 * bw] = lob;
        w.KP[2 * bw + 33] = lob;
    } else {
        w.KP[fw] = lo;
        w.KP[bw] = lob;
    }
    if (wide) {
        const uint32_t hi = pack4(hi_byte(c[0]), hi_byte(c[1]), hi_byte(c[2]), hi_byte(c[3]));
        w.KH[fw] = hi;
        w.KH[bw] = prmt(hi, (uint32_t)hi_byte(cprev), 0x4012);
    }
}

template <int NQ, int NKS = 0>
__device__ __forceinline__ void g_mma_any(const uint32_t* __restrict__ Kw, int nks, int kidx0, int xb,
                                          const uint32_t* __restrict__ xc0,
                                          const uint32_t* __restrict__ xc1, int (&acc)[NQ][2][4]) {
    if (NKS > 0) {  // (a kernel specialised for this k-step count)
        g_mma_fixed<NQ, (NKS > 0 ? NKS : 2)>(Kw, kidx0, xb, xc0, xc1, acc);
        return;
    }
    switch (nks) {  // (warp-uniform)
        case 8: g_mma_fixed<NQ, 8>(Kw, kidx0, xb, xc0, xc1, acc); break;
        case 10: g_mma_fixed<NQ, 10>(Kw, kidx0, xb, xc0, xc1, acc); break;
        default: g_mma<NQ>(Kw, nks, kidx0, xb, xc0, xc1, acc); break;
    }
}

// The T updates of the lane's 8 NQ neighbours for one step (see run_walk_mma (2)): per
// group of four consecutive half indices A..A+3 three byte windows -- f, g and (for a*'s
// parity APAR) p -- and one-hot IDP4A selectors.
template <int APAR, int NQ>
__device__ __forceinline__ void t_update_groups(const WalkParams& P, const uint32_t* Xaw, int A0,
                                                int ah, const uint32_t (&sf)[4],
                                                const uint32_t (&sg)[4], const uint32_t (&sx)[4],
                                                int mo, int vo, int sc8, uint32_t (&T)[8 * NQ],
                                                int (&xs)[8 * NQ]) {
    const int k = P.k;
#pragma unroll
    for (int grp = 0; grp < 2 * NQ; ++grp) {
        const int Aa = min(A0 + 128 * grp, k);  // (addresses of invalid groups stay in range)
        const int bf = P.xoff + ah + k - Aa - 3, bg = P.xoff + ah - k + Aa,
                  bx = P.xoff + Aa - ah - APAR;
        const uint32_t wf = prmt(Xaw[bf >> 2], Xaw[(bf >> 2) + 1], sel4r(bf & 3));
        const uint32_t wg = prmt(Xaw[bg >> 2], Xaw[(bg >> 2) + 1], sel4(bg & 3));
        const uint32_t wx = prmt(Xaw[bx >> 2], Xaw[(bx >> 2) + 1], sel4(bx & 3));
        LABS_BC(P, bf >> 2, 0, P.xwords - 1);
        LABS_BC(P, bg >> 2, 0, P.xwords - 1);
        LABS_BC(P, bx >> 2, 0, P.xwords - 1);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int m = 8 * (grp >> 1) + 4 * (e & 1) + 2 * (grp & 1) + (e >> 1);
            const int vp = (e & 1) == APAR ? __dp4a((int)wx, (int)sx[e], 0) : 0;
            int v = __dp4a((int)wf, (int)sf[e], __dp4a((int)wg, (int)sg[e], vp));
            if ((e & 1) == APAR && m == mo) {  // (the pivot has a*'s parity)
                v += vo;
                xs[m] = -xs[m];
            }
            T[m] += (uint32_t)(v * sc8);
        }
    }
}

// MODE: 0 = the plain walk (the timed path), 1 = checked (debug_check_energy, score_out /
// corr_out allowed), 2 = counting (count_visited: every neighbour's Bloom lookup counted;
// also checked).  The plain kernel carries no per-step test of the diagnostic options.
// NKS > 0: the k-step count is compile-time (plain kernels of the common lengths).
template <int NQ, int MODE, int NKS>
__device__ void run_walk_mma(const WalkParams& P, const MmaSmem& w, const uint64_t* fm0,
                             const uint64_t* fm1, const uint64_t* fmf, int64_t walk, bool valid,
                             int* score_out, int* corr_out) {
    constexpr int LPW = 32;
    constexpr int R = 8 * NQ;
    // lag words a lane owns: S = ceil(k/4) <= (2 b0 + 256 NQ + 3) / 4 with b0 <= 15
    // (NKS = 8 implies 183 <= k+1 <= 249, 46 <= S <= 62: exactly two lag words per lane)
    constexpr int NJ = NKS == 8 ? 2 : ((256 * NQ + 64 + 127) / 128 < 4 ? (256 * NQ + 64 + 127) / 128 : 4);
    const Seg<LPW> sg(threadIdx.x & 31);
    const int L = P.L, k = P.k, kp1 = P.kp1, S = P.S;
    const int sl = sg.sl;
    const int nj = NKS == 8 ? 2 : (S + LPW - 1) / LPW;

    // ---- load the initial half, build parity arrays + their byte-shifted copies ----
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
        w.Xw(par)[word] = v;
    }
    for (int i = sl; i < P.off_kh - P.off_kl + P.kwords; i += LPW) w.KP[i] = 0;  // (KP, KH adjacent)
    __syncwarp();
    for (int wi = sl; wi < 6 * P.xcw; wi += LPW) {  // copies c = 1..3 of both parities
        const int par = wi / (3 * P.xcw);
        const int rem = wi - par * 3 * P.xcw;
        const int c = 1 + rem / P.xcw;
        const int word = rem - (c - 1) * P.xcw + (P.xcl >> 2);
        w.Xc(par, c)[word - (P.xcl >> 2)] = prmt(w.Xw(par)[word], w.Xw(par)[word + 1], sel4(c));
    }

    // ---- exact C_{2t} of the owned lag words (registers), E, max|C| ----
    WarpSmem ws{};  // (views the K1 helpers expect)
    ws.X0 = w.X(0);
    ws.X1 = w.X(1);
    ws.X0w = w.Xw(0);
    ws.X1w = w.Xw(1);
    ws.C16 = w.C16;
    ws.KQ = w.KQ;
    ws.half = w.half;
    ws.bloom = w.bloom;
    int e_part = 0, cmax = 0;
    int C[NJ][4];
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) {
        const int s = sl + LPW * jj;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int t = 4 * s + 1 + b;
            int v = 0;
            if (jj < nj && s < S && t <= k) v = corr_even_lag(ws, P, t);
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
            w.C16[2 * s] = prmt((uint32_t)C[jj][0], (uint32_t)C[jj][1], 0x5410);
            w.C16[2 * s + 1] = prmt((uint32_t)C[jj][2], (uint32_t)C[jj][3], 0x5410);
            store_kp_word<-1>(w, P, s, C[jj], cprev, wide);
            if (corr_out && valid)
                for (int b = 0; b < 4; ++b)
                    if (4 * s + 1 + b <= k) corr_out[walk * k + 4 * s + b] = C[jj][b];
        }
    }

    // ---- 16N + 32Q per half index (lanes over a), once per walk ----
    for (int a = P.p + sl; a <= k; a += LPW) {
        const int8_t* Xb = w.X(a & 1) + P.xoff + (a >> 1);
        const int tstar = (a < k) ? (k - a) : -1;
        int q = 0;
        for (int t = 1; 2 * t <= a; ++t)
            if (t != tstar) q += (int)Xb[-t] * (int)Xb[t];
        const int n = (a >> 1) + ((L - 1 - a) >> 1) - (a < k ? 1 : 0);
        w.KQ[a] = (a < k) ? 16 * n + 32 * q : 4 * n + 8 * q;
    }
    __syncwarp();

    // ---- lane geometry (the accumulator fragment layout) ----
    const int lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
    const int b0 = P.p >> 1;
    const int A0 = 2 * b0 + 16 * gq + 4 * tq;
    // A (kernel) word of k-step 0, q-tile 0, row gq, columns 4tq..4tq+3
    const int D = b0 + 7 + P.kdelta;
    const int kidx0 = (P.koff - D) / 4 + tq - 2 * gq;
    // B (parity) words: byte xoff + gq + 4tq - 7 - delta of X_par, from copy c
    const int jb = P.xoff + gq + 4 * tq - 7 - P.kdelta;
    const int cb = jb & 3;
    const int xb = cb == 0 ? jb >> 2 : (jb - cb - P.xcl) >> 2;
    const uint32_t* xc0 = cb == 0 ? w.Xw(0) : w.Xc(0, cb);
    const uint32_t* xc1 = cb == 0 ? w.Xw(1) : w.Xc(1, cb);
    // (G's reads: kernel words kidx0 - 32 (NQ-1) - 16 .. kidx0 + 8 nks - 4, parity words
    // xb .. xb + 8 nks - 4 of the primary array or a copy)
    LABS_BC(P, kidx0 - 32 * (NQ - 1) - 16, 0, P.kwords);
    LABS_BC(P, kidx0 + 8 * P.nks - 4, 0, P.kwords);
    LABS_BC(P, xb, 0, cb == 0 ? P.xwords : P.xcw);
    LABS_BC(P, xb + 8 * P.nks - 4, 0, cb == 0 ? P.xwords : P.xcw);
    // this lane's flip destination (lanes 0-7 at step (4)): copy c = sl & 3 of each parity,
    // indexed by the half index's parity-array position i (byte xoff + i of the primary)
    int8_t* flip0;
    int8_t* flip1;
    {
        const int c = sl & 3;
        flip0 = c == 0 ? w.X(0) + P.xoff : reinterpret_cast<int8_t*>(w.Xc(0, c)) + P.xoff - c - P.xcl;
        flip1 = c == 0 ? w.X(1) + P.xoff : reinterpret_cast<int8_t*>(w.Xc(1, c)) + P.xoff - c - P.xcl;
    }
    const bool one_key = NQ == 1 || L <= 1001;  // (NQ = 1: L < 573, compile-time true)
    constexpr bool COUNT = MODE == 2;
    constexpr bool CHK = MODE != 0;
    const bool dbg = CHK && P.debug_check != 0;
    const int sc = one_key ? 512 : 1;
    uint32_t T[R];
    int xs[R];
    uint32_t inval = 0;
    {
        const int16_t* C16h = reinterpret_cast<const int16_t*>(w.C16);
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int a = A0 + mma_off(m);
            int t = 0;
            xs[m] = 0;
            if (a < P.p || a > k) {
                inval |= 1u << m;
            } else if (a < k) {
                const int sgn8 = ((k - a) & 1) ? -8 : 8;
                t = w.KQ[a] + sgn8 * (int)C16h[k - a - 1];
                xs[m] = 8 * (int)w.X(a & 1)[P.xoff + (a >> 1)];
            } else {
                t = w.KQ[a];
                xs[m] = 4 * (int)w.X(a & 1)[P.xoff + (a >> 1)];
            }
            T[m] = (uint32_t)(t * sc) + (one_key ? 0x80000000u + (uint32_t)a : 0u);
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

    // ---- half hashes h1, h2 (saw.cpp:77-89), dedup hash, initial Bloom insert ----
    uint64_t h1 = 0, h2 = 0;
    for (int i = sl; i < kp1; i += LPW) {
        const int bit = (w.half[i >> 5] >> (i & 31)) & 1;
        h1 ^= P.tab[(0 * kp1 + i) * 2 + bit];
        h2 ^= P.tab[(1 * kp1 + i) * 2 + bit];
    }
    h1 = sg.xor64(h1) ^ P.salt0;
    h2 = sg.xor64(h2) ^ P.salt1;
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
    int iterations = 0, emitted = 0, wide_iters = 0, diverged = 0;
    long long probes = 0;
    long long evals_part = 0;
    int exhausted = 0;
    uint32_t skip = inval;
    const int t_i32 = (CHK && score_out) ? 1 : (int)P.t_i;
    bool active = valid;

    for (int it = 0;; ++it) {
        const bool cont = active && it < t_i32;
        if (!cont) break;  // (one walk per warp: warp-uniform)
        // ---- G for all neighbours on the tensor cores ----
        int acc[NQ][2][4];
#pragma unroll
        for (int j = 0; j < NQ; ++j)
#pragma unroll
            for (int p2 = 0; p2 < 2; ++p2)
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[j][p2][i] = 0;
        if (__builtin_expect(wide, 0)) {  // G = 256 G_high + G_low (rare)
            g_mma_any<NQ, NKS>(w.KH, P.nks, kidx0, xb, xc0, xc1, acc);
#pragma unroll
            for (int j = 0; j < NQ; ++j)
#pragma unroll
                for (int p2 = 0; p2 < 2; ++p2)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[j][p2][i] *= 256;
            ++wide_iters;
        }
        if (NKS == 8) g_mma_kp<NQ, 8>(w.KP, P.nks, kidx0, xb, xc0, xc1, acc);
        else if (NKS > 0 || !P.kpl) g_mma_any<NQ, NKS>(w.KP, P.nks, kidx0, xb, xc0, xc1, acc);
        else g_mma_kp<NQ, 0>(w.KP, P.nks, kidx0, xb, xc0, xc1, acc);
        // ---- exact deltas / keys: dE(a) = T(a) - xs(a) G(a) ----
        int delta[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int gv = acc[m / 8][(m >> 2) & 1][m & 3];
            delta[m] = (int)(T[m] + (uint32_t)xs[m] * (uint32_t)gv);
        }
        if (CHK && score_out) {
            if (valid)
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    const int a = A0 + mma_off(m);
                    if (!(inval & (1u << m)))
                        score_out[walk * kp1 + a] =
                            one_key ? (int)((uint32_t)delta[m] - 0x80000000u - (uint32_t)a) >> 9 : delta[m];
                }
            break;
        }

        // ---- choose: lowest (delta, hp) among unvisited (best_neighbour, saw.cpp:106-115) ----
        if (COUNT) {
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if (inval & (1u << m)) continue;
                const int a = A0 + mma_off(m);
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
        int dstar = 0, astar = -1;
        uint32_t ins_idx = 0;
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
        for (;;) {
            int md, ma;
            bool mine_won;
            if (one_key) {
                const uint32_t k_best = __reduce_min_sync(FULLMASK, bkey);
                if (__builtin_expect(k_best == 0xffffffffu, 0)) break;  // every free neighbour visited
                ma = (int)(k_best & 511u);
                md = (int)(k_best >> 9) - (1 << 22);
                mine_won = bkey == k_best;
            } else {
                md = __reduce_min_sync(FULLMASK, bd);
                if (md == INT_BIG) break;
                const int mine = (bd == md) ? A0 + mma_off(bm) : INT_BIG;
                ma = __reduce_min_sync(FULLMASK, mine);
                mine_won = mine == ma;
            }
            // (every lane computes its index -- no divergent branch; lanes past the k hashes
            // read word 0, a broadcast, and count as set)
            const bool hl = sl < P.bloom_k;
            const uint32_t idx = bloom_index(h1 ^ fm0[ma], h2 ^ fm1[ma], sl, P.bloom_mu, P.bloom_bits);
            const bool bit = !hl || ((w.bloom[hl ? idx >> 5 : 0] >> (idx & 31)) & 1);
            ins_idx = idx;
            if (COUNT) {
                dstar = md;
                astar = ma;
                break;
            }
            const bool visited = __all_sync(FULLMASK, bit);
            ++probes;
            if (!visited) {
                dstar = md;
                astar = ma;
                break;
            }
            if (one_key) {  // drop the visited neighbour from the winner's slots; every lane
                            // recomputes its minimum (unchanged but for the winner: no branch)
                const int d = ma - A0;
                const int mm = (d >> 8) * 8 + (d & 1) * 4 + (((d & 255) >> 7) << 1) + ((d >> 1) & 1);
                skip |= mine_won ? 1u << (mm & 31) : 0u;
                bkey = lane_min_key<R>(delta, skip);
            } else if (mine_won) {
                const int d = ma - A0;
                const int mm = (d >> 8) * 8 + (d & 1) * 4 + (((d & 255) >> 7) << 1) + ((d >> 1) & 1);
                skip |= 1u << mm;
                {
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
        }
        if (__builtin_expect(astar < 0, 0)) {
            exhausted = 1;
            active = false;
            break;
        }

        // ---- apply the skew flip at astar (apply_skew_flip, skew.cpp:95-105) ----
        ++iterations;
        const int as = astar;
        const bool cen = as == k;
        const int bstar = L - 1 - as;
        const int apar = as & 1, ah = as >> 1;
        int8_t* Xa = w.X(apar) + P.xoff;
        const int xa = Xa[ah];
        const int xb = cen ? 0 : (((k - as) & 1) ? -xa : xa);
        h1 ^= fm0[as];
        h2 ^= fm1[as];
        hf ^= fmf[as];
        // Bloom insert by lanes 0..k_hash-1; the other lanes OR 0 into their (valid) word --
        // no divergent branch around the atomic
        atomicOr(&w.bloom[ins_idx >> 5], sl < P.bloom_k ? 1u << (ins_idx & 31) : 0u);
        energy += dstar;
        best = min(best, energy);
        // (1) zero x_a and x_b in the primary array (the T and C updates read the fused
        //     rule's pre-step sequence from it; the MMA copies are rewritten in (4))
        __syncwarp();
        // (lane 0 x_a*, lane 1 x_b*, the others byte -1 of the zero front padding: one store
        //  instruction, no branch)
        {
            int zi = sl == 1 ? (bstar >> 1) : ah;
            zi = sl >= 2 ? -1 : zi;
            Xa[zi] = 0;
        }
        __syncwarp();
        // (2) T updates from the zeroed pre-step sequence (K1's rules), four neighbours a = A + e
        //     (e = 0..3) per group at once.  Byte e of three windows holds f_a = x_{a*+2(k-a)},
        //     g_a = x_{a*-2(k-a)} (= x_{2a-b*}) and p_a = x_{2a-a*}; one-hot int8 selectors carry
        //     the coefficients, so a neighbour costs three IDP4A and one IMAD:
        //       T(a) += 8 sc [ c_a (f_a + g_a) - 8 x_a* p_a - 8 x_b* g_a ],  c_a = (-1)^(k-a) mul
        //     (the Q terms only for a of a*'s parity; the pair excluded from Q(a) and the undo
        //     move's own Q term are taken back in the rare fix-up below).
        const int mul = cen ? -2 * xa : -4 * xa;
        {
            // the two exceptions, each in at most one lane: a = a* (the undo move: its Q term
            // through b* is excluded, xs flips, it is skipped next step) and a with
            // 3a = a* + L - 1 (its Q pair through a* is excluded)
            constexpr int kSlotMask = ~(0x83 | (NQ == 2 ? 0x100 : 0));  // slot offsets: bits 0,1,7(,8)
            const int down = as - A0;
            const int ex3 = as + L - 1;
            const int aex = ex3 / 3;
            // (warp-uniform: a* is; about one step in six has the excluded Q pair)
            const bool has_ex = ex3 - 3 * aex == 0 && (aex & 1) == apar && aex >= P.p;
            const int mo = (down >= 0 && (down & kSlotMask) == 0)
                               ? (down >> 8) * 8 + (down & 1) * 4 + ((down >> 6) & 2) + ((down >> 1) & 1) : -1;
            const int vo = 8 * xb * (int)Xa[ah - (k - as)];      // (unscaled correction)
            LABS_BC(P, P.xoff + ah - (k - as), 0, 4 * P.xwords);
            skip = inval | (mo >= 0 ? 1u << mo : 0u);
            const int c0 = (k & 1) ? -mul : mul;  // c_a for e = 0 (A is even); alternates with e
            uint32_t sf[4], sg[4], sx[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int ce = (e & 1) ? -c0 : c0;
                const bool same = (e & 1) == apar;
                sf[e] = ((uint32_t)ce & 0xffu) << (8 * e);
                sg[e] = ((uint32_t)(ce - (same ? 8 * xb : 0)) & 0xffu) << (8 * e);
                sx[e] = same ? ((uint32_t)(-8 * xa) & 0xffu) << (8 * e) : 0u;
            }
            const uint32_t* Xaw = w.Xw(apar);
            const int sc8 = 8 * sc;
            if (apar)  // (warp-uniform: the x_{2a-a*} term exists for a* 's parity only)
                t_update_groups<1, NQ>(P, Xaw, A0, ah, sf, sg, sx, mo, vo, sc8, T, xs);
            else
                t_update_groups<0, NQ>(P, Xaw, A0, ah, sf, sg, sx, mo, vo, sc8, T, xs);
            if (has_ex) {  // the pair excluded from Q(aex) passes through a*: take its term back
                const int dex = aex - A0;
                const int mx = (dex >= 0 && (dex & kSlotMask) == 0)
                                   ? (dex >> 8) * 8 + (dex & 1) * 4 + ((dex >> 6) & 2) + ((dex >> 1) & 1) : -1;
                const uint32_t vx = (uint32_t)(8 * sc8 * xa * (int)Xa[(2 * aex - as) >> 1]);
#pragma unroll
                for (int m = 0; m < R; ++m)
                    T[m] += m == mx ? vx : 0u;  // (a select, not a divergent branch)
            }
        }
        // (3) even-lag C update, lanes over lag words: dc_t = mul (x_{a+2t} + x_{a-2t})
        int cmx = 0, esp = 0;
        {
            const uint32_t* Xaw = w.Xw(apar);
            const int awF = (P.xoff + ah + 1) >> 2;
            const uint32_t asF = sel4((P.xoff + ah + 1) & 3);
            const int awB = (P.xoff + ah - 4) >> 2;
            const uint32_t asB = sel4r((P.xoff + ah) & 3);
            const uint32_t mb = (uint32_t)mul & 0xffu;
            int e1h[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) e1h[b] = (int)prmt(mb, 0u, 0x4444u ^ (0x4u << (4 * b)));
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) {
                const int s = sl + LPW * jj;
                if (jj < nj) {  // (lanes past S: zero windows, C stays 0 -- no divergence)
                    const uint32_t fw = prmt(Xaw[awF + s], Xaw[awF + s + 1], asF);
                    const uint32_t bw = prmt(Xaw[awB - s], Xaw[awB - s + 1], asB);
                    LABS_BC(P, awF + s, 0, P.xwords - 1);
                    LABS_BC(P, awB - s, 0, P.xwords - 1);
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        C[jj][b] = __dp4a((int)fw, e1h[b], __dp4a((int)bw, e1h[b], C[jj][b]));
                    cmx |= ((C[jj][0] + 128) | (C[jj][1] + 128)) | ((C[jj][2] + 128) | (C[jj][3] + 128));
                }
            }
        }
        const bool wide_next = __any_sync(FULLMASK, (cmx & ~0xff) != 0);
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
            const int up = __shfl_up_sync(FULLMASK, C[jj][3], 1, LPW);
            const int wrap = __shfl_sync(FULLMASK, jj > 0 ? C[jj > 0 ? jj - 1 : 0][3] : 0, LPW - 1, LPW);
            const int s = sl + LPW * jj;
            const int cprev = s == 0 ? 0 : (sl == 0 ? wrap : up);
            if (jj < nj) store_kp_word<NKS == 8 ? 1 : (NKS > 0 ? 0 : -1)>(w, P, s, C[jj], cprev, wide_next);  // (zeros past S)
        }
        wide = wide_next;
        __syncwarp();
        // (4) write the flipped pair into the primary array and its three shifted copies
        //     (lanes 0-3: x_a* in copy 0-3, lanes 4-7: x_b*).  (The packed half is not kept
        //     up to date: a sieve hit rebuilds it from the parity arrays.)
        if (sl < 8 && !(cen && sl >= 4))
            (apar ? flip1 : flip0)[(sl < 4) ? ah : (bstar >> 1)] = (int8_t)((sl < 4) ? -xa : -xb);
        if (dbg) {
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj)
                if (jj < nj && sl + LPW * jj < S)
#pragma unroll
                    for (int b = 0; b < 4; ++b) esp += C[jj][b] * C[jj][b];
            if (sg.sum(esp) != energy) ++diverged;
        }
        __syncwarp();
        if (__builtin_expect(energy < P.e_l, 0)) {  // K2: one ring slot (warp-uniform: one walk per warp)
            ++emitted;
            unsigned long long slot = 0;
            if (sl == 0) slot = atomicAdd(P.rec_count, 1ull);
            slot = __shfl_sync(FULLMASK, slot, 0);
            bool wrote = true;
            bool wait = slot >= (unsigned long long)P.rec_cap;
            unsigned spins = 0;
            while (wait) {  // (uniform: every lane evaluates the same slot and tail)
                const unsigned long long tail = *(volatile const unsigned long long*)P.rec_tail;
                if (slot < tail + (unsigned long long)P.rec_cap) {
                    wait = false;
                } else if (++spins >= kRingWaitSpins) {
                    if (sl == 0) atomicOr(&P.ctl[0], 1);
                    wait = wrote = false;
                } else {
                    __nanosleep(4000);
                }
                wait = __any_sync(FULLMASK, wait);
                wrote = __all_sync(FULLMASK, wrote);
            }
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
                // packed half: bit i <=> x_i = +1, x_i = X_{i&1}[i>>1] (one ballot per word)
                for (int wd = 0; wd < P.hw; ++wd) {
                    const int i = 32 * wd + sl;
                    const bool plus = i < kp1 && w.X(i & 1)[P.xoff + (i >> 1)] > 0;
                    const uint32_t word = __ballot_sync(FULLMASK, plus);
                    if (sl == 0) r[kRecHeader + wd] = word;
                }
                __threadfence();
            }
            __syncwarp();
            if (wrote && sl == 0)
                P.rec_tag[slot & (unsigned long long)(P.rec_cap - 1)] = (uint32_t)(P.rec_seq0 + slot + 1);
        }
    }
    if (COUNT) evals_part = sg.sum64(evals_part);
    if (valid && sl == 0 && P.walk_stats) {
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

// FMS: the flip-mask table fm has a shared copy per block (P.fm_words > 0, when that costs
// no resident block) -- a compile-time choice, so its reads are shared loads, not generic ones
template <int NQ, int MODE, bool FMS, int NKS = 0>
__global__ void __launch_bounds__(128, NQ == 1 ? LABS_MMA_MINB : 3) saw_walk_mma_kernel(WalkParams P, int* score_out, int* corr_out) {
    extern __shared__ uint4 smem_u4[];
    const uint64_t* fm = P.fm;
    if (FMS || P.fm_words) {  // (FMS = false keeps the generic-pointer form: fewer registers)
        uint64_t* fs = reinterpret_cast<uint64_t*>(smem_u4);
        for (int i = threadIdx.x; i < 3 * P.kp1; i += blockDim.x) fs[i] = P.fm[i];
        __syncthreads();
        fm = fs;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* base = reinterpret_cast<uint32_t*>(smem_u4) + P.fm_words + warp * P.warp_words;
    MmaSmem w;
    w.base = base;
    w.off_x1 = P.off_x1;
    w.off_xc = P.off_xc;
    w.xcw = P.xcw;
    w.KP = base + P.off_kl;
    w.KH = base + P.off_kh;
    w.C16 = base + P.off_c16;
    w.KQ = reinterpret_cast<int*>(base + P.off_kq);
    w.half = base + P.off_half;
    w.bloom = base + P.off_bloom;
    const int64_t nwarps = (int64_t)gridDim.x * P.warps_per_block;
    int64_t walk = (int64_t)blockIdx.x * P.warps_per_block + warp;
    while (walk < P.nwalks) {
        if (*(volatile int*)&P.ctl[1]) break;  // cancelled by the host (pool stopped)
        run_walk_mma<NQ, MODE, NKS>(P, w, fm, fm + P.kp1, fm + 2 * P.kp1, walk, true, score_out, corr_out);
        unsigned long long nx = 0;
        if (lane == 0) nx = atomicAdd(P.walk_next, 1ull);
        walk = nwarps + (int64_t)__shfl_sync(FULLMASK, nx, 0);
    }
}

template <int NQ>
cudaError_t launch_walk_mma(const WalkParams& P, int grid, size_t smem, cudaStream_t st,
                            int* score_out, int* corr_out, bool count) {
    const bool fms = P.fm_words > 0;
    const int mode = count ? 2 : ((P.debug_check || score_out || corr_out) ? 1 : 0);
    auto kfn = fms ? saw_walk_mma_kernel<NQ, 0, true> : saw_walk_mma_kernel<NQ, 0, false>;
    if constexpr (NQ == 1) {
        if (mode == 0 && P.nks == 8)
            kfn = fms ? saw_walk_mma_kernel<NQ, 0, true, 8> : saw_walk_mma_kernel<NQ, 0, false, 8>;
        if (mode == 0 && P.nks == 10)
            kfn = fms ? saw_walk_mma_kernel<NQ, 0, true, 10> : saw_walk_mma_kernel<NQ, 0, false, 10>;
    }
    if (mode == 1) kfn = fms ? saw_walk_mma_kernel<NQ, 1, true> : saw_walk_mma_kernel<NQ, 1, false>;
    if (mode == 2) kfn = fms ? saw_walk_mma_kernel<NQ, 2, true> : saw_walk_mma_kernel<NQ, 2, false>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, P.warps_per_block * 32, smem, st>>>(P, score_out, corr_out);
    return cudaGetLastError();
}

template <int NQ>
int blocks_per_sm_mma(const WalkParams& P, size_t smem) {
    int n = 0;
    auto kfn = P.fm_words > 0 ? saw_walk_mma_kernel<NQ, 0, true> : saw_walk_mma_kernel<NQ, 0, false>;
    if constexpr (NQ == 1) {
        if (P.nks == 8)
            kfn = P.fm_words > 0 ? saw_walk_mma_kernel<NQ, 0, true, 8> : saw_walk_mma_kernel<NQ, 0, false, 8>;
        if (P.nks == 10)
            kfn = P.fm_words > 0 ? saw_walk_mma_kernel<NQ, 0, true, 10> : saw_walk_mma_kernel<NQ, 0, false, 10>;
    }
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kfn, P.warps_per_block * 32, smem) != cudaSuccess)
        return 0;
    return n;
}

}  // namespace labs_b200
