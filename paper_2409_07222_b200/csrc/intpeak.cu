// intpeak.cu -- INT32 issue-rate microbenchmark on the B200 (roofline denominator).
//
// Four kernels, each a set of independent dependency chains per thread (enough
// ILP to saturate the pipe), every SM fully occupied:
//   imad  : IMAD  (fma pipe)                 d = a*d + b
//   ialu  : LOP3/IADD3 (alu pipe)            d = (d ^ a) + b  -> IADD3/LOP3 mix
//   mixed : 1 IMAD + 1 LOP3 per step (both pipes)
//   dp4a  : IDP4A only                       d = dp4a(a, b, d)  (4 int8 MACs per lane)
// Each counts 1 "INT32 op" per lane per instruction (an IMAD is one op here, as
// in BASELINE.md §2's 8-ops-per-lag-term count).
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/labs_gpu.h"

namespace labs_b200 {
void set_error(const std::string& msg);
}

namespace {
constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void k_imad(int* out, int a, int b) {
    int d[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c] = threadIdx.x + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) d[c] = d[c] * a + b;
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= d[c];
    if (s == 0x7fffffff) out[0] = s;
}

__global__ void k_ialu(int* out, int a, int b) {
    unsigned d[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c] = threadIdx.x + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) d[c] = (d[c] ^ (unsigned)a) + (unsigned)b + (d[c] >> 1);
    }
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= d[c];
    if (s == 0x7fffffffu) out[0] = (int)s;
}

__global__ void k_mixed(int* out, int a, int b) {
    int d[kChains];
    unsigned e[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        d[c] = threadIdx.x + c;
        e[c] = threadIdx.x * 3u + c;
    }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            d[c] = d[c] * a + b;
            e[c] = (e[c] ^ (unsigned)a) + (unsigned)b + (e[c] >> 1);
        }
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= d[c] ^ (int)e[c];
    if (s == 0x7fffffff) out[0] = s;
}

__global__ void k_dp4a(int* out, int a, int b) {
    int d[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c] = threadIdx.x + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) d[c] = __dp4a(a, b, d[c]);
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= d[c];
    if (s == 0x7fffffff) out[0] = s;
}

// int8 tensor-core path the K1t walk kernel uses: mma.sync.m16n8k32.s8, kChains independent
// accumulator chains per warp (4096 int8 MACs per instruction per warp)
__global__ void k_imma(int* out, int a, int b) {
    uint32_t fa[4], fb[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) fa[i] = 0x01ff01ffu ^ ((unsigned)(a * (threadIdx.x + i)) & 0x02000200u);
    fb[0] = 0x0101ff01u ^ (unsigned)b;
    fb[1] = 0xff0101ffu;
    int d[kChains][4];  // (distinct chains: identical ones would be merged by the compiler)
#pragma unroll
    for (int c = 0; c < kChains; ++c)
#pragma unroll
        for (int i = 0; i < 4; ++i) d[c][i] = (int)threadIdx.x * 7 + c * 4 + i;
    for (int i = 0; i < kIters / 16; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                "{%8,%9}, {%0,%1,%2,%3};\n"
                : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
                : "r"(fa[0]), "r"(fa[1]), "r"(fa[2]), "r"(fa[3]), "r"(fb[0]), "r"(fb[1]));
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= d[c][0] ^ d[c][1] ^ d[c][2] ^ d[c][3];
    if (s == 0x7fffffff) out[0] = s;
}

template <typename K>
double time_kernel(K kern, int blocks, int threads, int* dout, double ops_per_thread) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(dout, 3, 5);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(dout, 3, 5);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ops_per_thread * blocks * (double)threads / (best * 1e-3);
}
}  // namespace

extern "C" int labs_int32_peak(double* imad_ops, double* ialu_ops, double* mixed_ops,
                               double* dp4a_ops, int32_t* sm_count, int32_t* clock_khz) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        labs_b200::set_error("no CUDA device available");
        return LABS_ENODEV;
    }
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    int* dout = nullptr;
    if (cudaMalloc(&dout, 64) != cudaSuccess) {
        labs_b200::set_error("cudaMalloc failed");
        return LABS_ECUDA;
    }
    const int threads = 256, blocks = sms * 8;
    const double per = (double)kIters * kChains;
    // ialu counts the 3 ALU instructions it issues per element (LOP3, SHF, IADD3)
    const double r_imad = time_kernel(k_imad, blocks, threads, dout, per);
    const double r_ialu = time_kernel(k_ialu, blocks, threads, dout, per * 3);
    const double r_mixed = time_kernel(k_mixed, blocks, threads, dout, per * 4);
    const double r_dp4a = time_kernel(k_dp4a, blocks, threads, dout, per);  // IDP4A lane-instr/s
    cudaFree(dout);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        labs_b200::set_error(cudaGetErrorString(e));
        return LABS_ECUDA;
    }
    if (imad_ops) *imad_ops = r_imad;
    if (ialu_ops) *ialu_ops = r_ialu;
    if (mixed_ops) *mixed_ops = r_mixed;
    if (dp4a_ops) *dp4a_ops = r_dp4a;
    if (sm_count) *sm_count = sms;
    if (clock_khz) *clock_khz = clk;
    return LABS_OK;
}

// int8 tensor-core MAC rate (mma.sync m16n8k32.s8 over all SMs): the peak of the path K1t's
// sliding dot products run on (roofline denominator of the tensor leg).
extern "C" int labs_imma_peak(double* int8_macs_per_s) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        labs_b200::set_error("no CUDA device available");
        return LABS_ENODEV;
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int* dout = nullptr;
    if (cudaMalloc(&dout, 64) != cudaSuccess) {
        labs_b200::set_error("cudaMalloc failed");
        return LABS_ECUDA;
    }
    const int threads = 256, blocks = sms * 8;
    // per thread: (kIters / 16) * kChains MMAs, each 4096 MACs per warp = 128 per lane
    const double per = (double)(kIters / 16) * kChains * 128.0;
    const double r = time_kernel(k_imma, blocks, threads, dout, per);
    cudaFree(dout);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        labs_b200::set_error(cudaGetErrorString(e));
        return LABS_ECUDA;
    }
    if (int8_macs_per_s) *int8_macs_per_s = r;
    return LABS_OK;
}
