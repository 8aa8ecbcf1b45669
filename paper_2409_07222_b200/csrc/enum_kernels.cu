// enum_kernels.cu -- K4: restriction-class Gray enumeration on sm_100a (extension;
// BASELINE config 2).
//
// The reference has no Step-1 enumeration mode; the pattern is oracle_skew_exhaustive
// (oracle.cpp:37-67): start from a half, visit configurations in Gray order, each step
// one apply_skew_flip (skew.cpp:95-105) at half position p + ctz(g), test E.  Here the
// half is rank_prefixes(p)[class] ++ (+1)^(k+1-p) and the Gray code runs over the m
// half positions [p, p+m); configuration g = Gray(g) (bit j set <=> position p+j is -1).
// Every g in [g_begin, g_end) with E < E_l is emitted; best E and its first g reported.
//
// Layout: 4 lanes (up to 32 lag words) -- eight chunks per warp -- or 16 / 32 lanes = one
// chunk of 2^chunk_log2 consecutive g each (chunks from an atomic queue).
// Lanes own the even lags t = 4(lane + LPW j) + 1 .. +4 (C_{2t} in registers); the
// sequence lives in shared memory as two parity byte arrays.  A step updates every owned
//     C_{2t} += dc_t,   dc_t = mul * (x_{a+2t} + x_{a-2t} - [t = k-a] x_b)
// (mul = -4 x_a, or -2 x_a for the centre; the same fused even-lag rule as the walk
// kernel's apply; dc by two one-hot IDP4A) and accumulates the new C^2, so one segment sum
// per step is the configuration's energy E = sum_t C_{2t}^2 (odd lags vanish); lane s of a
// batch keeps step s's E.  Exact integer arithmetic throughout.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <string>
#include <vector>

#include "host_util.hpp"

namespace labs_b200 {

#define FULLMASK 0xffffffffu
#ifndef LABS_ENUM_MINB
#define LABS_ENUM_MINB 7  // resident 128-thread blocks per SM the 4-lane variants target (72 registers;
                          // 6 blocks at 80: 2.95e10, 8 at 64: 2.97e10, 7: 3.11e10 Gray steps/s)
#endif

struct EnumLaunch {
    int32_t L, k, kp1, p, m;
    int32_t nj;            // lag groups per lane (t = 4(lane + 32j) + 1..4)
    int32_t S;             // 4-lag words covering t = 1..k
    int32_t xoff, xwords;  // parity arrays: byte xoff + i = x_{2i+par}, zero padded
    int32_t nwx;           // words per parity array holding data
    int32_t warp_words;
    int32_t chunk_log2;
    int64_t e_l;
    uint64_t g_begin, g_end;
    uint64_t nchunks;
    uint32_t base_half[kMaxHalf / 32];  // half of configuration 0 (bit set <=> +1)
    uint32_t* rec;                      // [rec_cap][4]: g lo, g hi, E, 0
    int64_t rec_cap;
    unsigned long long* rec_count;
    unsigned long long* chunk_next;     // dynamic chunk-group queue (zeroed per launch)
    int64_t* chunk_best;                // [nchunks][2]: best E, its first g
};

// PRMT selector of bytes o..o+3 of a word pair: o | (o+1)<<4 | (o+2)<<8 | (o+3)<<12
__device__ __forceinline__ uint32_t sel4(int o) { return 0x3210u + 0x1111u * (uint32_t)o; }
// bytes o+3..o (reversed): (o+3) | (o+2)<<4 | (o+1)<<8 | o<<12
__device__ __forceinline__ uint32_t sel4r(int o) { return 0x0123u + 0x1111u * (uint32_t)o; }

// One chunk of Gray codes per segment of LPW lanes (LPW = 16: two chunks per warp, the
// per-step bookkeeping -- ctz, addresses, the flip stores, loop control -- serves both).
template <int NJ, int LPW>
__device__ void enum_chunk(const EnumLaunch& P, int8_t* X0, int8_t* X1, uint64_t chunk,
                           bool valid, int sl) {
    const int L = P.L, k = P.k;
    const uint64_t g0 = P.g_begin + (chunk << P.chunk_log2);
    uint64_t g1 = g0 + (1ull << P.chunk_log2);
    if (!valid) g1 = g0 + 1;  // (an idle segment: no steps)
    if (g1 > P.g_end || g1 < g0) g1 = P.g_end > g0 ? P.g_end : g0 + 1;
    uint32_t* X0w = reinterpret_cast<uint32_t*>(X0);
    uint32_t* X1w = reinterpret_cast<uint32_t*>(X1);
    auto seg_sum = [](int v) {
        if (LPW == 32) return __reduce_add_sync(FULLMASK, v);
#pragma unroll
        for (int o = LPW / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o, LPW);
        return v;
    };

    // ---- configuration g0: half = base with Gray(g0) over [p, p+m) negated ----
    const uint64_t gray0 = g0 ^ (g0 >> 1);
    for (int wi = sl; wi < 2 * P.xwords; wi += LPW) {
        const int par = wi >= P.xwords;
        const int word = wi - par * P.xwords;
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int li = word * 4 + b - P.xoff;
            const int j = 2 * li + par;
            int x = 0;
            if (li >= 0 && j < L) {
                int src = j, neg = 0;
                if (j > k) {
                    src = 2 * k - j;
                    neg = (j - k) & 1;
                }
                int bit = (P.base_half[src >> 5] >> (src & 31)) & 1;
                if (src >= P.p && src < P.p + P.m && ((gray0 >> (src - P.p)) & 1)) bit ^= 1;
                x = (bit ^ neg) ? 1 : -1;
            }
            v |= ((uint32_t)x & 0xffu) << (8 * b);
        }
        (par ? X1w : X0w)[word] = v;
    }
    __syncwarp();

    // ---- C_{2t} of the owned lags (sequence.cpp:8-19 on the parity arrays) ----
    int C[NJ][4];
    int e_part = 0;
    const int n0 = P.xoff >> 2;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int t = 4 * (sl * NJ + j) + 1 + b;
            int acc = 0;
            if (t <= k) {
                const int dw = t >> 2;
                const uint32_t sel = sel4(t & 3);
                for (int n = n0; n < n0 + P.nwx; ++n) {
                    acc = __dp4a((int)X0w[n], (int)__byte_perm(X0w[n + dw], X0w[n + dw + 1], sel), acc);
                    acc = __dp4a((int)X1w[n], (int)__byte_perm(X1w[n + dw], X1w[n + dw + 1], sel), acc);
                }
            }
            C[j][b] = acc;
            e_part += acc * acc;
        }
    }
    int energy = seg_sum(e_part);

    int best_e = energy;
    uint64_t best_g = g0;
    if (valid && energy < P.e_l && sl == 0) {
        const unsigned long long slot = atomicAdd(P.rec_count, 1ull);
        if ((long long)slot < P.rec_cap) {
            uint32_t* r = P.rec + 4 * slot;
            r[0] = (uint32_t)g0;
            r[1] = (uint32_t)(g0 >> 32);
            r[2] = (uint32_t)energy;
            r[3] = 0;
        }
    }

    // ---- Gray steps g = g0+1 .. g1-1 in batches of LPW ----
    // ctz(g0 + i) = ctz(i) when the chunk start is a multiple of 2^chunk_log2 (every chunk
    // when g_begin is aligned); else the 64-bit path.
    const bool aligned = (g0 & ((1ull << P.chunk_log2) - 1)) == 0;
    const int nsteps = (int)(g1 - g0 - 1);  // (< 2^chunk_log2 <= 2^30)
    int nmax = nsteps;                      // warp-uniform bound
#pragma unroll
    for (int o = LPW; o < 32; o <<= 1) nmax = max(nmax, __shfl_xor_sync(FULLMASK, nmax, o));
    // The flip position of step i (1-based; idle steps: any valid position, no writes).
    const auto flip_pos = [&](int i) {
        const int tz = aligned ? __ffs(i) - 1 : __ffsll((long long)(g0 + (uint64_t)i)) - 1;
        return i <= nsteps ? P.p + tz : P.p;
    };
    // The fused rule's [t = k-a] x_b term: x_b is read once, by the forward window at
    // t* = k-a, so it is zero in the array during the step (written flipped after it).  The
    // zero of step i+1 is stored with step i's flips: one store and two warp barriers per step.
    int a = flip_pos(1);
    if (nsteps >= 1 && sl == 2 && a != k) ((a & 1) ? X1 : X0)[P.xoff + ((L - 1 - a) >> 1)] = 0;
    __syncwarp();
    // store lanes: 0 writes -x_a at a, 1 writes -x_b at b (not at the centre), 2 the next zero
    const int st_lane = sl < 3 ? sl : 3;
    for (int s0 = 0; s0 < nmax; s0 += LPW) {
        const int nb = min(max(nsteps - s0, 0), LPW);
        const int nbw = min(nmax - s0, LPW);
        int mine = 0;  // E after step s0 + sl
        for (int s = 0; s < nbw; ++s) {  // (rolled: small code, no instruction-cache misses)
            const bool live = s < nb;
            const int i = s0 + s + 1;
            const int ah = a >> 1;
            int8_t* Xa = ((a & 1) ? X1 : X0) + P.xoff;
            const uint32_t* Xaw = (a & 1) ? X1w : X0w;
            const int xa = Xa[ah];
            const bool cen = a == k;
            const int xb = ((k - a) & 1) ? -xa : xa;
            const int mul = live ? (cen ? -2 * xa : -4 * xa) : 0;
            const int awF = (P.xoff + ah + 1) >> 2;
            const uint32_t asF = sel4((P.xoff + ah + 1) & 3);
            const int awB = (P.xoff + ah - 4) >> 2;
            const uint32_t asB = sel4r((P.xoff + ah) & 3);
            int acc[4] = {0, 0, 0, 0};  // owned C_{2t}^2 after the step (four short chains)
            const uint32_t mb = (uint32_t)mul & 0xffu;  // int8 mul: one-hot IDP4A selectors
            const int e1[4] = {(int)mb, (int)(mb << 8), (int)(mb << 16), (int)(mb << 24)};
            // the lane's lag words s0 .. s0+NJ-1 are consecutive: NJ+1 words per window side
            // (lag words past the range read the zero padding: dc = 0, C stays 0)
            const int s0w = sl * NJ;
            uint32_t wf[NJ + 1], wb[NJ + 1];
#pragma unroll
            for (int q = 0; q <= NJ; ++q) {
                wf[q] = Xaw[awF + s0w + q];
                wb[q] = Xaw[awB - s0w + 1 - q];
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const uint32_t fw = __byte_perm(wf[j], wf[j + 1], asF);
                const uint32_t bw = __byte_perm(wb[j + 1], wb[j], asB);
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    // dc = mul (x_{a+2t} + x_{a-2t}): two IDP4A against mul e_b chained into
                    // C, no byte unpacking (0 beyond k)
                    C[j][b] = __dp4a((int)fw, e1[b], __dp4a((int)bw, e1[b], C[j][b]));
                    acc[b] += C[j][b] * C[j][b];
                }
            }
            const int tot = seg_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
            if (sl == s) mine = tot;
            const int an = flip_pos(i + 1);
            // (selects, not branches: every lane computes its store)
            const int pa = st_lane == 2 ? an : a;
            const int pos = st_lane == 0 ? ah : (L - 1 - pa) >> 1;
            const int val = st_lane == 0 ? -xa : (st_lane == 1 ? -xb : 0);
            const bool st = (st_lane == 0 && live) | (st_lane == 1 && live && !cen) |
                            (st_lane == 2 && i < nsteps && an != k);
            int8_t* dst = ((pa & 1) ? X1 : X0) + P.xoff + pos;
            __syncwarp();
            if (st) *dst = (int8_t)val;
            __syncwarp();
            a = an;
        }
        const bool vstep = sl < nb;
        const int e_mine = mine;
        const uint64_t g_mine = g0 + (uint64_t)(1 + s0 + sl);
        const int e_last = __shfl_sync(FULLMASK, e_mine, nb > 0 ? nb - 1 : 0, LPW);
        if (nb > 0) energy = e_last;
        if (vstep && e_mine < best_e) {
            best_e = e_mine;
            best_g = g_mine;
        }
        const bool hit = vstep && e_mine < P.e_l;
        const unsigned hm = __ballot_sync(FULLMASK, hit);
        if (hm) {
            const int base_lane = (threadIdx.x & 31) - sl;
            const unsigned seg_hm = (hm >> base_lane) & (LPW == 32 ? 0xffffffffu : ((1u << LPW) - 1u));
            unsigned long long base = 0;
            if (sl == 0 && seg_hm) base = atomicAdd(P.rec_count, (unsigned long long)__popc(seg_hm));
            base = __shfl_sync(FULLMASK, base, 0, LPW);
            if (hit) {
                const unsigned long long slot = base + __popc(seg_hm & ((1u << sl) - 1));
                if ((long long)slot < P.rec_cap) {
                    uint32_t* r = P.rec + 4 * slot;
                    r[0] = (uint32_t)g_mine;
                    r[1] = (uint32_t)(g_mine >> 32);
                    r[2] = (uint32_t)e_mine;
                    r[3] = 0;
                }
            }
        }
    }
    // chunk best: lowest E, then lowest g
#pragma unroll
    for (int o = LPW / 2; o > 0; o >>= 1) {
        const int oe = __shfl_xor_sync(FULLMASK, best_e, o, LPW);
        const unsigned long long og = __shfl_xor_sync(FULLMASK, (unsigned long long)best_g, o, LPW);
        if (oe < best_e || (oe == best_e && og < best_g)) {
            best_e = oe;
            best_g = og;
        }
    }
    if (valid && sl == 0) {
        P.chunk_best[2 * chunk] = best_e;
        P.chunk_best[2 * chunk + 1] = (int64_t)best_g;
    }
    __syncwarp();
}

template <int NJ, int LPW>
__global__ void __launch_bounds__(128, LPW == 4 ? LABS_ENUM_MINB : 1) enum_kernel(const __grid_constant__ EnumLaunch P);

// Launch with one wave of resident blocks (the occupancy limit per SM x SMs), capped by
// the work; the chunk queue balances the rest.
template <int NJ, int LPW>
void launch_enum(const EnumLaunch& P, size_t smem, cudaStream_t stream, int sms, uint64_t want) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, enum_kernel<NJ, LPW>, 128, smem) !=
            cudaSuccess || per_sm < 1)
        per_sm = 1;
    const int grid = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>(want, static_cast<uint64_t>(sms) * per_sm)));
    enum_kernel<NJ, LPW><<<grid, 128, smem, stream>>>(P);
}

template <int NJ, int LPW>
__global__ void __launch_bounds__(128, LPW == 4 ? LABS_ENUM_MINB : 1) enum_kernel(const __grid_constant__ EnumLaunch P) {
    extern __shared__ uint32_t esmem[];
    constexpr int SEGS = 32 / LPW;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int seg = lane / LPW, sl = lane % LPW;
    int8_t* X0 = reinterpret_cast<int8_t*>(esmem + (warp * SEGS + seg) * P.warp_words);
    int8_t* X1 = X0 + 4 * P.xwords;
    // chunk groups (SEGS chunks per warp) come from an atomic queue, so warps that finish
    // early take more and no SM idles at the end of the launch
    const uint64_t ngrp = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint64_t grp = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    while (grp * SEGS < P.nchunks) {
        const uint64_t c = grp * SEGS + seg;
        enum_chunk<NJ, LPW>(P, X0, X1, c < P.nchunks ? c : 0, c < P.nchunks, sl);
        unsigned long long nx = 0;
        if (lane == 0) nx = atomicAdd(P.chunk_next, 1ull);
        grp = ngrp + __shfl_sync(FULLMASK, nx, 0);
    }
}

namespace {
template <typename T>
struct DBuf {
    T* p = nullptr;
    ~DBuf() {
        if (p) cudaFree(p);
    }
};
#define ENUM_CUDA(call)                                                       \
    do {                                                                      \
        cudaError_t _e = (call);                                              \
        if (_e != cudaSuccess) {                                              \
            set_error(std::string(#call) + ": " + cudaGetErrorString(_e));    \
            return LABS_ECUDA;                                                \
        }                                                                     \
    } while (0)
}  // namespace

int enumerate_class_gpu(int32_t L, int32_t p, int32_t cls, int32_t m, int64_t e_l,
                        uint64_t g_begin, uint64_t g_end, labs_enum_fn emit, void* user,
                        labs_enum_stats* stats, int chunk_log2) {
    const int kp1 = (L + 1) / 2;
    if (L < 3 || L % 2 == 0) {
        set_error("enumerate: length must be odd and >= 3");
        return LABS_EINVAL;
    }
    if (L > kMaxHalf) {
        set_error("enumerate: length exceeds the tabulation hash range (L <= 1023)");
        return LABS_EINVAL;
    }
    if (p < 1 || p > kp1 || p > 30) {
        set_error("enumerate: bad prefix length");
        return LABS_EINVAL;
    }
    if (m < 0 || p + m > kp1 || m > 62) {
        set_error("enumerate: bad free-bit count");
        return LABS_EINVAL;
    }
    if (cls < 0 || cls >= (1 << (p - 1))) {
        set_error("enumerate: bad class");
        return LABS_EINVAL;
    }
    const uint64_t total = 1ull << m;
    if (g_end > total) g_end = total;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
        set_error("no CUDA device available (the enumeration has no CPU fallback)");
        return LABS_ENODEV;
    }
    labs_enum_stats st{};
    st.best_energy = 0;
    if (g_begin >= g_end) {
        if (stats) *stats = st;
        return LABS_OK;
    }
    EnumLaunch P{};
    P.L = L;
    P.k = (L - 1) / 2;
    P.kp1 = kp1;
    P.p = p;
    P.m = m;
    P.nj = (P.k + 127) / 128;
    P.nwx = (kp1 + 3) / 4;
    const int S = (P.k + 3) / 4;
    P.S = S;
    // 4 lanes per chunk (eight chunks per warp share the per-step bookkeeping -- ctz, window
    // addresses, the segment sum, the flip stores) up to 32 lag words, else 16 / 32;
    // LABS_ENUM_LPW=4|8|16|32 forces a width (A/B timing)
    const char* lenv = std::getenv("LABS_ENUM_LPW");
    const int lwant = lenv ? std::atoi(lenv) : 0;
    int lpw = S <= 32 ? 4 : (S <= 64 ? 16 : 32);
    if (lwant == 32 || (lwant == 16 && S <= 64) || ((lwant == 8 || lwant == 4) && S <= 32)) lpw = lwant;
    const int nj = (S + lpw - 1) / lpw;
    // window reads reach SW+1 words past any position on both sides, SW = lpw x nj >= S the
    // lanes' lag words (lanes past the lag range read zeros instead of branching); the
    // correlation prologue reads up to nwx + SW + 1 words
    const int SW = lpw * nj;
    P.xoff = 4 * (SW + 2) + 16;
    P.xwords = ((P.xoff + 4 * P.nwx + 4 * (SW + 2) + 32) / 4 + 3) & ~3;
    P.warp_words = 2 * P.xwords;
    const uint64_t range = g_end - g_begin;
    int cl = chunk_log2 > 0 ? std::min(chunk_log2, 30) : 12;  // (32-bit step counters)
    while (cl > 5 && (range >> cl) < 148ull * 32) --cl;  // enough chunks to fill the GPU
    P.chunk_log2 = cl;
    P.nchunks = (range + (1ull << cl) - 1) >> cl;
    P.e_l = e_l;
    P.g_begin = g_begin;
    P.g_end = g_end;
    const auto pre = rank_prefixes(p);
    for (int i = 0; i < kp1; ++i) {
        const bool plus = i < p ? pre[static_cast<size_t>(cls) * p + i] > 0 : true;
        if (plus) P.base_half[i >> 5] |= 1u << (i & 31);
    }
    cudaStream_t stream;
    ENUM_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    DBuf<uint32_t> rec;
    DBuf<unsigned long long> cnt;
    DBuf<int64_t> best;
    int64_t cap = 1 << 16;
    int rc = LABS_OK;
    std::vector<uint32_t> hrec;
    std::vector<int64_t> hbest(2 * P.nchunks);
    unsigned long long hcnt = 0;
    float ms_total = 0;
    do {
        cudaError_t ce = cudaSuccess;
        if (!cnt.p) ce = cudaMalloc(&cnt.p, 2 * sizeof(unsigned long long));  // count, queue
        if (ce == cudaSuccess && !best.p) ce = cudaMalloc(&best.p, 16 * P.nchunks);
        if (ce == cudaSuccess) {
            if (rec.p) cudaFree(rec.p);
            rec.p = nullptr;
            ce = cudaMalloc(&rec.p, 16 * static_cast<size_t>(cap));
        }
        if (ce != cudaSuccess) {
            set_error(std::string("enumerate: ") + cudaGetErrorString(ce));
            rc = LABS_ECUDA;
            break;
        }
        P.rec = rec.p;
        P.rec_cap = cap;
        P.rec_count = cnt.p;
        P.chunk_next = cnt.p + 1;
        P.chunk_best = best.p;
        cudaMemsetAsync(cnt.p, 0, 2 * sizeof(unsigned long long), stream);
        const int segs = 32 / lpw;
        const size_t smem = static_cast<size_t>(4) * segs * P.warp_words * 4;
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const uint64_t want = (P.nchunks + 4 * segs - 1) / (4 * segs);
        cudaEventRecord(e0, stream);
        if (lpw == 4) {
            switch (nj) {
                case 1: launch_enum<1, 4>(P, smem, stream, sms, want); break;
                case 2: launch_enum<2, 4>(P, smem, stream, sms, want); break;
                case 3: launch_enum<3, 4>(P, smem, stream, sms, want); break;
                case 4: launch_enum<4, 4>(P, smem, stream, sms, want); break;
                case 5: launch_enum<5, 4>(P, smem, stream, sms, want); break;
                case 6: launch_enum<6, 4>(P, smem, stream, sms, want); break;
                case 7: launch_enum<7, 4>(P, smem, stream, sms, want); break;
                default: launch_enum<8, 4>(P, smem, stream, sms, want); break;
            }
        } else if (lpw == 8) {
            switch (nj) {
                case 1: launch_enum<1, 8>(P, smem, stream, sms, want); break;
                case 2: launch_enum<2, 8>(P, smem, stream, sms, want); break;
                case 3: launch_enum<3, 8>(P, smem, stream, sms, want); break;
                default: launch_enum<4, 8>(P, smem, stream, sms, want); break;
            }
        } else if (lpw == 16) {
            switch (nj) {
                case 1: launch_enum<1, 16>(P, smem, stream, sms, want); break;
                case 2: launch_enum<2, 16>(P, smem, stream, sms, want); break;
                case 3: launch_enum<3, 16>(P, smem, stream, sms, want); break;
                default: launch_enum<4, 16>(P, smem, stream, sms, want); break;
            }
        } else {
            switch (nj) {
                case 1: launch_enum<1, 32>(P, smem, stream, sms, want); break;
                case 2: launch_enum<2, 32>(P, smem, stream, sms, want); break;
                case 3: launch_enum<3, 32>(P, smem, stream, sms, want); break;
                default: launch_enum<4, 32>(P, smem, stream, sms, want); break;
            }
        }
        cudaEventRecord(e1, stream);
        ce = cudaGetLastError();
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(&hcnt, cnt.p, sizeof hcnt, cudaMemcpyDeviceToHost, stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(stream);
        if (ce != cudaSuccess) {
            set_error(std::string("enumerate kernel: ") + cudaGetErrorString(ce));
            rc = LABS_ECUDA;
            break;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms_total += ms;
        if (static_cast<int64_t>(hcnt) > cap) {  // overflow: grow and rerun (deterministic)
            cap = static_cast<int64_t>(hcnt) + 1024;
            continue;
        }
        hrec.resize(4 * static_cast<size_t>(hcnt));
        if (hcnt) cudaMemcpy(hrec.data(), rec.p, hrec.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(hbest.data(), best.p, hbest.size() * 8, cudaMemcpyDeviceToHost);
        break;
    } while (true);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(stream);
    if (rc != LABS_OK) return rc;
    // emissions in g order
    std::vector<std::pair<uint64_t, int32_t>> hits(hcnt);
    for (size_t i = 0; i < hcnt; ++i)
        hits[i] = {static_cast<uint64_t>(hrec[4 * i]) | (static_cast<uint64_t>(hrec[4 * i + 1]) << 32),
                   static_cast<int32_t>(hrec[4 * i + 2])};
    std::sort(hits.begin(), hits.end());
    for (const auto& h : hits)
        if (emit && emit(user, h.first, h.second) != 0) {
            set_error("enumeration callback aborted");
            return LABS_EABORT;
        }
    int64_t be = hbest[0];
    uint64_t bg = static_cast<uint64_t>(hbest[1]);
    for (uint64_t c = 1; c < P.nchunks; ++c)
        if (hbest[2 * c] < be) {  // chunks in g order: strict < keeps the first g
            be = hbest[2 * c];
            bg = static_cast<uint64_t>(hbest[2 * c + 1]);
        }
    st.best_energy = be;
    st.best_g = bg;
    st.configurations = g_end - g_begin;
    st.emitted = hcnt;
    st.kernel_ms = ms_total;
    if (stats) *stats = st;
    return LABS_OK;
}

}  // namespace labs_b200

extern "C" int labs_enumerate_class(int32_t length, int32_t prefix_len, int32_t class_index,
                                    int32_t m, int64_t energy_threshold, uint64_t g_begin,
                                    uint64_t g_end, labs_enum_fn emit, void* user,
                                    labs_enum_stats* stats) {
    return labs_b200::enumerate_class_gpu(length, prefix_len, class_index, m, energy_threshold,
                                          g_begin, g_end, emit, user, stats, 0);
}
