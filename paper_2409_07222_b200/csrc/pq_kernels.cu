// pq_kernels.cu -- K5: Step-2 neighbourhood scoring on sm_100a.
//
// For one pivot of the priority-queue refinement (refine, pq.cpp:114-176) the host loop
// visits every single flip i of the pivot and, for each, the T_r one-step left and right
// cyclic rotations of that neighbour (make_rotations / rotation_chain, pq.cpp:56-112).
// Every quantity it needs is a function of the pivot alone, so this kernel computes them
// all at once, exactly:
//   delta[i]              flip_delta(pivot, i)                (sequence.cpp:42-58)
//   rot_e[i][dir][r-1]    energy after r one-step rotations   (rotate_*_once, pq.cpp:56-84)
//   rot_h[i][dir][r-1]    canonical_hash(0) of that sequence  (rng.hpp:89-95)
// The host then replays the frontier operations (seen / mark / push) in the reference
// order.  Layout: one warp per neighbour i; lanes own lags k (C_k in registers) for the
// incremental rotation updates and positions j for the hashes.  Exact int32 arithmetic
// (E <= L^3/3 < 2^31 for L <= 1023).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <string>
#include <vector>

#include "host_util.hpp"

namespace labs_b200 {

namespace {
constexpr int kPqWarps = 8;            // warps (neighbours) per block
constexpr int kPqMaxL = kMaxHalf;      // L <= 1024 (TabulationHash::kMaxLen, rng.hpp:77)
constexpr int kPqLagsPerLane = (kPqMaxL + 31) / 32;

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ uint64_t warp_xor64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, o);
        const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), o);
        v ^= ((uint64_t)hi << 32) | lo;
    }
    return v;
}

struct PqLaunch {
    int32_t L, t_r;
    const int8_t* pivot;        // [L]
    const uint64_t* tab0;       // [L][2] table-0 entries (canonical hash)
    uint64_t salt;              // table-0 salt for L
    int32_t* delta;             // [L]
    int32_t* rot_e;             // [L][2][t_r]
    uint64_t* rot_h;            // [L][2][t_r]
    int32_t* pivot_e;           // [1]
};

template <int NK>
__global__ void __launch_bounds__(32 * kPqWarps) pq_score_kernel(const __grid_constant__ PqLaunch P) {
    extern __shared__ int pq_smem[];
    const int L = P.L;
    int* Cs = pq_smem;                                        // pivot C_k, k < L
    int8_t* s = reinterpret_cast<int8_t*>(pq_smem + L);       // pivot signs
    int8_t* u_all = s + ((L + 15) & ~15);                     // per-warp neighbour signs
    for (int j = threadIdx.x; j < L; j += blockDim.x) s[j] = P.pivot[j];
    __syncthreads();
    // pivot correlations (sequence.cpp:8-19), threads over lags
    for (int k = threadIdx.x + 1; k < L; k += blockDim.x) {
        int c = 0;
        for (int i = 0; i + k < L; ++i) c += s[i] * s[i + k];
        Cs[k] = c;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * kPqWarps + warp;
    if (i >= L) return;
    int8_t* u = u_all + warp * ((L + 15) & ~15);
    for (int j = lane; j < L; j += 32) u[j] = (j == i) ? (int8_t)(-s[j]) : s[j];

    // ---- flip delta and the neighbour's correlations (apply_flip, sequence.cpp:60-79) ----
    int c[NK];
    int d_part = 0, e_part = 0;
    const int si = s[i];
#pragma unroll
    for (int q = 0; q < NK; ++q) {
        const int k = lane + 32 * q + 1;
        c[q] = 0;
        if (k < L) {
            int t = 0;
            if (i - k >= 0) t += s[i - k];
            if (i + k < L) t += s[i + k];
            const int ck = Cs[k];
            const int dc = -2 * si * t;
            d_part += dc * (2 * ck + dc);
            c[q] = ck + dc;
            e_part += ck * ck;
        }
    }
    const int d = warp_sum_i(d_part);
    const int e_pivot = warp_sum_i(e_part);
    if (lane == 0) {
        P.delta[i] = d;
        if (i == 0) P.pivot_e[0] = e_pivot;
    }
    __syncwarp();
    // ---- rotation chains of the neighbour (rotation_chain, pq.cpp:86-101) ----
    for (int dir = 0; dir < 2; ++dir) {
        int cc[NK];
#pragma unroll
        for (int q = 0; q < NK; ++q) cc[q] = c[q];
        int e = e_pivot + d;
        int off = 0;  // current sequence v_j = u_{(j + off) mod L}
        for (int r = 1; r <= P.t_r; ++r) {
            int de = 0;
            if (dir == 0) {  // left: C_k += v_0 (v_{L-k} - v_k); v_0 moves to the end
                const int v0 = u[off];
#pragma unroll
                for (int q = 0; q < NK; ++q) {
                    const int k = lane + 32 * q + 1;
                    if (k < L) {
                        int a = off + L - k, b = off + k;
                        if (a >= L) a -= L;
                        if (b >= L) b -= L;
                        const int dc = v0 * ((int)u[a] - (int)u[b]);
                        de += dc * (2 * cc[q] + dc);
                        cc[q] += dc;
                    }
                }
                off = off + 1 == L ? 0 : off + 1;
            } else {  // right: C_k += v_{L-1} (v_{k-1} - v_{L-1-k}); v_{L-1} moves to front
                int last = off + L - 1;
                if (last >= L) last -= L;
                const int vl = u[last];
#pragma unroll
                for (int q = 0; q < NK; ++q) {
                    const int k = lane + 32 * q + 1;
                    if (k < L) {
                        int a = off + k - 1, b = off + L - 1 - k;
                        if (a >= L) a -= L;
                        if (b >= L) b -= L;
                        const int dc = vl * ((int)u[a] - (int)u[b]);
                        de += dc * (2 * cc[q] + dc);
                        cc[q] += dc;
                    }
                }
                off = off == 0 ? L - 1 : off - 1;
            }
            e += warp_sum_i(de);
            uint64_t h = 0;
            for (int j = lane; j < L; j += 32) {
                int jj = j + off;
                if (jj >= L) jj -= L;
                h ^= P.tab0[2 * j + (u[jj] > 0)];
            }
            h = warp_xor64(h) ^ P.salt;
            if (lane == 0) {
                const size_t o = ((size_t)i * 2 + dir) * P.t_r + (r - 1);
                P.rot_e[o] = e;
                P.rot_h[o] = h;
            }
        }
    }
}

// Per-thread device contexts: refine_batch (pipeline.cpp:132-186) runs refines on several
// host threads at once, each gets its own streams and buffers.  refine_with_operators
// (pq.cpp:203-228) alternates lengths L-1, L, L+1, so a thread keeps a small cache of
// contexts keyed by (device, L, T_r) instead of freeing and reallocating -- cudaFree and
// cudaFreeHost synchronise the whole device, across every refine thread.
struct PqCtx {
    int dev = -1;
    cudaStream_t st = nullptr;
    int L = 0, t_r = -1;
    int8_t* d_pivot = nullptr;
    uint64_t* d_tab = nullptr;
    int32_t *d_delta = nullptr, *d_rot_e = nullptr, *d_pe = nullptr;
    uint64_t* d_rot_h = nullptr;
    int8_t* h_pivot = nullptr;  // pinned staging
    void* h_out = nullptr;
    size_t out_bytes = 0;
    ~PqCtx() { release(); }
    void release() {
        if (st) {
            cudaFree(d_pivot);
            cudaFree(d_tab);
            cudaFree(d_delta);
            cudaFree(d_rot_e);
            cudaFree(d_pe);
            cudaFree(d_rot_h);
            cudaFreeHost(h_pivot);
            cudaFreeHost(h_out);
            cudaStreamDestroy(st);
        }
        st = nullptr;
        L = 0;
        t_r = -1;
    }
};
constexpr int kPqCtxCache = 6;
struct PqCache {
    PqCtx ctx[kPqCtxCache];
    uint64_t used[kPqCtxCache] = {};
    uint64_t clock = 0;
};
thread_local PqCache g_pq;

#define PQ_CUDA(call)                                                          \
    do {                                                                       \
        cudaError_t _e = (call);                                               \
        if (_e != cudaSuccess) {                                               \
            set_error(std::string("pq_score: ") + cudaGetErrorString(_e));     \
            return LABS_ECUDA;                                                 \
        }                                                                      \
    } while (0)

int pq_init(PqCtx& c, int dev, int L, int t_r);

PqCtx* pq_prepare(int L, int t_r, int* rc) {
    int dev = 0;
    *rc = LABS_OK;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        set_error("pq_score: cudaGetDevice failed");
        *rc = LABS_ECUDA;
        return nullptr;
    }
    PqCache& cache = g_pq;
    int slot = 0;
    for (int i = 0; i < kPqCtxCache; ++i) {
        const PqCtx& c = cache.ctx[i];
        if (c.st && c.L == L && c.t_r == t_r && c.dev == dev) {
            cache.used[i] = ++cache.clock;
            return &cache.ctx[i];
        }
        if (cache.used[i] < cache.used[slot]) slot = i;  // least recently used (or empty)
    }
    *rc = pq_init(cache.ctx[slot], dev, L, t_r);
    cache.used[slot] = ++cache.clock;
    return *rc == LABS_OK ? &cache.ctx[slot] : nullptr;
}

int pq_init(PqCtx& c, int dev, int L, int t_r) {
    c.release();
    c.dev = dev;
    PQ_CUDA(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
    const size_t nrot = static_cast<size_t>(L) * 2 * (t_r > 0 ? t_r : 1);
    PQ_CUDA(cudaMalloc(&c.d_pivot, L));
    PQ_CUDA(cudaMalloc(&c.d_tab, 16 * static_cast<size_t>(L)));
    PQ_CUDA(cudaMalloc(&c.d_delta, 4 * static_cast<size_t>(L)));
    PQ_CUDA(cudaMalloc(&c.d_rot_e, 4 * nrot));
    PQ_CUDA(cudaMalloc(&c.d_rot_h, 8 * nrot));
    PQ_CUDA(cudaMalloc(&c.d_pe, 4));
    PQ_CUDA(cudaMallocHost(&c.h_pivot, L));
    c.out_bytes = 4 * static_cast<size_t>(L) + 4 * nrot + 8 * nrot + 8;
    PQ_CUDA(cudaMallocHost(&c.h_out, c.out_bytes));
    std::vector<uint64_t> tab(2 * static_cast<size_t>(L));
    const auto& tt = TabTables::get();
    for (int j = 0; j < L; ++j) {
        tab[2 * static_cast<size_t>(j)] = tt.t[0][j][0];
        tab[2 * static_cast<size_t>(j) + 1] = tt.t[0][j][1];
    }
    PQ_CUDA(cudaMemcpy(c.d_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
    c.L = L;
    c.t_r = t_r;
    return LABS_OK;
}
}  // namespace

int pq_score(int L, int t_r, const int8_t* pivot, int32_t* delta, int32_t* rot_e,
             uint64_t* rot_h, int64_t* pivot_energy) {
    if (L < 3 || L > kPqMaxL) {
        set_error("pq_score: length must be in [3, 1024]");
        return LABS_EINVAL;
    }
    if (t_r < 0 || t_r >= L) {
        set_error("make_rotations: T_r must be < L");
        return LABS_EINVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
        set_error("no CUDA device available (the Step-2 scorer has no CPU fallback)");
        return LABS_ENODEV;
    }
    int rc = LABS_OK;
    PqCtx* cp = pq_prepare(L, t_r, &rc);
    if (!cp) return rc;
    PqCtx& c = *cp;
    std::memcpy(c.h_pivot, pivot, static_cast<size_t>(L));
    PQ_CUDA(cudaMemcpyAsync(c.d_pivot, c.h_pivot, L, cudaMemcpyHostToDevice, c.st));
    PqLaunch P{};
    P.L = L;
    P.t_r = t_r;
    P.pivot = c.d_pivot;
    P.tab0 = c.d_tab;
    P.salt = TabTables::get().salt[0][L];
    P.delta = c.d_delta;
    P.rot_e = c.d_rot_e;
    P.rot_h = c.d_rot_h;
    P.pivot_e = c.d_pe;
    const int grid = (L + kPqWarps - 1) / kPqWarps;
    const size_t smem = 4 * static_cast<size_t>(L) + ((L + 15) & ~15) * (1 + kPqWarps);
    const int nk = (L - 1 + 31) / 32;
    if (nk <= 8) pq_score_kernel<8><<<grid, 32 * kPqWarps, smem, c.st>>>(P);
    else if (nk <= 16) pq_score_kernel<16><<<grid, 32 * kPqWarps, smem, c.st>>>(P);
    else pq_score_kernel<kPqLagsPerLane><<<grid, 32 * kPqWarps, smem, c.st>>>(P);
    PQ_CUDA(cudaGetLastError());
    const size_t nrot = static_cast<size_t>(L) * 2 * t_r;
    auto* out = static_cast<char*>(c.h_out);
    PQ_CUDA(cudaMemcpyAsync(out, c.d_delta, 4 * static_cast<size_t>(L), cudaMemcpyDeviceToHost, c.st));
    if (nrot) {
        PQ_CUDA(cudaMemcpyAsync(out + 4 * L, c.d_rot_e, 4 * nrot, cudaMemcpyDeviceToHost, c.st));
        PQ_CUDA(cudaMemcpyAsync(out + 4 * L + 4 * nrot, c.d_rot_h, 8 * nrot, cudaMemcpyDeviceToHost,
                                c.st));
    }
    PQ_CUDA(cudaMemcpyAsync(out + 4 * L + 12 * nrot, c.d_pe, 4, cudaMemcpyDeviceToHost, c.st));
    PQ_CUDA(cudaStreamSynchronize(c.st));
    std::memcpy(delta, out, 4 * static_cast<size_t>(L));
    if (nrot) {
        if (rot_e) std::memcpy(rot_e, out + 4 * L, 4 * nrot);
        if (rot_h) std::memcpy(rot_h, out + 4 * L + 4 * nrot, 8 * nrot);
    }
    int32_t pe = 0;
    std::memcpy(&pe, out + 4 * L + 12 * nrot, 4);
    if (pivot_energy) *pivot_energy = pe;
    return LABS_OK;
}

}  // namespace labs_b200

extern "C" int labs_pq_score(int32_t length, int32_t t_r, const int8_t* pivot, int32_t* deltas,
                             int32_t* rot_energy, uint64_t* rot_hash, int64_t* pivot_energy) {
    if (!pivot || !deltas || (t_r > 0 && (!rot_energy || !rot_hash))) {
        labs_b200::set_error("pq_score: null buffer");
        return LABS_EINVAL;
    }
    return labs_b200::pq_score(length, t_r, pivot, deltas, rot_energy, rot_hash, pivot_energy);
}
