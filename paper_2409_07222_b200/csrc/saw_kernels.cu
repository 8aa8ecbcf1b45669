// saw_kernels.cu -- K3 (seed streams) and the host-side dispatch of K1 over R
// (the walk kernel itself: saw_walk.cuh).
#include <cuda_runtime.h>
#include <stdint.h>

#include "saw_device.h"
#include "saw_walk.h"

namespace labs_b200 {
template <int NQ>
cudaError_t launch_walk_mma(const WalkParams& P, int grid, size_t smem, cudaStream_t st,
                            int* score_out, int* corr_out, bool count);
template <int NQ>
int blocks_per_sm_mma(const WalkParams& P, size_t smem);
}  // namespace labs_b200

namespace labs_b200 {

// ---------------------------------------------------------------------------
// K3: one thread per segment (restarts [r0, r1) of one walker), drawn in order from the
// walker's stream; the stream state lives in rng_state[seg_slot] between segments, so
// consecutive batches continue a walker on the device with no host round trip.
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
        const uint64_t* st = P.rng_state + 4 * (size_t)P.seg_slot[i];
        s0 = st[0];
        s1 = st[1];
        s2 = st[2];
        s3 = st[3];
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
    uint64_t* st = P.rng_state + 4 * (size_t)P.seg_slot[i];
    st[0] = s0;
    st[1] = s1;
    st[2] = s2;
    st[3] = s3;
}

// ---------------------------------------------------------------------------
// host-side launchers (called from the C++ orchestration)
size_t walk_smem_bytes(const WalkParams& P) {
    return (size_t)(P.fm_words + P.walks_per_block * P.warp_words) * 4;  // (warp_words: per walk)
}

cudaError_t launch_saw_walk(const WalkParams& P, int grid, cudaStream_t st, int* score_out,
                            int* corr_out) {
    const size_t smem = walk_smem_bytes(P);
    const bool count = P.count_visited != 0;
    if (P.kernel == 1)
        return P.nq == 1 ? launch_walk_mma<1>(P, grid, smem, st, score_out, corr_out, count)
                         : launch_walk_mma<2>(P, grid, smem, st, score_out, corr_out, count);
    switch (P.R * (P.lpw == 16 ? -1 : 1) + (P.lpw == 8 ? 1000 : 0)) {
#define LABS_CASE(r)                                                                   \
    case r: return launch_walk_fixed<r, 32>(P, grid, smem, st, score_out, corr_out, count); \
    case -r: return launch_walk_fixed<r, 16>(P, grid, smem, st, score_out, corr_out, count); \
    case 1000 + r: return launch_walk_fixed<r, 8>(P, grid, smem, st, score_out, corr_out, count);
        LABS_CASE(1) LABS_CASE(2) LABS_CASE(3) LABS_CASE(4) LABS_CASE(5) LABS_CASE(6)
        LABS_CASE(7) LABS_CASE(8) LABS_CASE(9) LABS_CASE(10) LABS_CASE(11) LABS_CASE(12)
        LABS_CASE(13) LABS_CASE(14) LABS_CASE(15) LABS_CASE(16)
#undef LABS_CASE
        default: return cudaErrorInvalidValue;
    }
}

static int walk_blocks_for(const WalkParams& P) {
    const size_t smem = walk_smem_bytes(P);
    if (P.kernel == 1) return P.nq == 1 ? blocks_per_sm_mma<1>(P, smem) : blocks_per_sm_mma<2>(P, smem);
    switch (P.R * (P.lpw == 16 ? -1 : 1) + (P.lpw == 8 ? 1000 : 0)) {
#define LABS_CASE(r)                                 \
    case r: return blocks_per_sm_fixed<r, 32>(P, smem); \
    case -r: return blocks_per_sm_fixed<r, 16>(P, smem); \
    case 1000 + r: return blocks_per_sm_fixed<r, 8>(P, smem);
        LABS_CASE(1) LABS_CASE(2) LABS_CASE(3) LABS_CASE(4) LABS_CASE(5) LABS_CASE(6)
        LABS_CASE(7) LABS_CASE(8) LABS_CASE(9) LABS_CASE(10) LABS_CASE(11) LABS_CASE(12)
        LABS_CASE(13) LABS_CASE(14) LABS_CASE(15) LABS_CASE(16)
#undef LABS_CASE
        default: return 0;
    }
}

// Resident blocks per SM, and where the flip-mask table fm lives: a per-block shared copy
// (shortest probe latency) unless that copy costs a resident block, else read through L1.
int walk_blocks_per_sm(WalkParams& P) {
    P.fm_words = 0;
    const int n_l1 = walk_blocks_for(P);
    WalkParams Q = P;
    Q.fm_words = (6 * P.kp1 + 3) / 4 * 4;
    if (walk_blocks_for(Q) >= n_l1 && walk_smem_bytes(Q) <= 227 * 1024) {
        P.fm_words = Q.fm_words;
        return walk_blocks_for(Q);
    }
    return n_l1;
}

// Load the seed kernel's module now (lazy loading would do it at the first job's launch).
cudaError_t preload_saw_seed() {
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, saw_seed_kernel);
}

cudaError_t launch_saw_seed(const SeedParams& P, cudaStream_t st) {
    const int bs = 128;
    const int grid = (P.nseg + bs - 1) / bs;
    if (grid == 0) return cudaSuccess;
    saw_seed_kernel<<<grid, bs, 0, st>>>(P);
    return cudaGetLastError();
}

}  // namespace labs_b200
