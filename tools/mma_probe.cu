// mma_probe.cu -- throughput / latency of the warp-level tensor paths on sm_100a
// (mma.sync HMMA f16->f32 m16n8k16, IMMA s8->s32 m16n8k32) next to IDP4A, to decide
// how the walk kernel's sliding dot product G should be computed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 2048;

__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void imma(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int CH>
__global__ void k_hmma(float* out, uint32_t seed) {
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u ^ (seed * (threadIdx.x + i) & 0x00010001u);
    b[0] = 0x3c00bc00u; b[1] = 0xbc003c00u;
    float d[CH][4] = {};
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int c = 0; c < CH; ++c) hmma(d[c], a, b);
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 1234.5f) out[0] = s;
}

template <int CH>
__global__ void k_imma(float* out, uint32_t seed) {
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = 0x01ff01ffu ^ (seed * (threadIdx.x + i) & 0x02000200u);
    b[0] = 0x0101ff01u; b[1] = 0xff0101ffu;
    int d[CH][4] = {};
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int c = 0; c < CH; ++c) imma(d[c], a, b);
    int s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 12345) out[0] = (float)s;
}

template <int CH>
__global__ void k_dp4a(float* out, uint32_t seed) {
    int d[CH];
    const int a = 0x01ff01ff ^ (int)(seed * threadIdx.x);
#pragma unroll
    for (int c = 0; c < CH; ++c) d[c] = threadIdx.x + c;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int c = 0; c < CH; ++c) d[c] = __dp4a(a, 0x0101ff01, d[c]);
    int s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c];
    if (s == 12345) out[0] = (float)s;
}

template <typename K>
float run(K k, int blocks, int threads, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<blocks, threads>>>(out, 7);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(out, 7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    float* out;
    cudaMalloc(&out, 64);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ghz = clk / 1e6;
    struct Cfg { int blocks, threads; const char* name; };
    // throughput: all SMs, 8 warps/SMSP
    const int B = sms * 4, T = 256;
    auto report = [&](const char* what, float ms, double macs_per_warp_inst, int ch, int blocks,
                      int threads) {
        const double insts = (double)blocks * (threads / 32) * kIters * ch;
        const double s = ms * 1e-3;
        const double cyc = s * ghz * 1e9;
        printf("%-28s %8.3f ms  warp-inst/clk/SM %.3f  MAC/clk/SM %.1f  cyc/inst/SMSP(1 warp) %.2f\n",
               what, ms, insts / cyc / sms, insts * macs_per_warp_inst / cyc / sms,
               cyc / (insts / ((double)blocks * threads / 32 > sms * 4 ? 1 : 1)));
    };
    report("hmma m16n8k16 x4 chains", run(k_hmma<4>, B, T, out), 2048, 4, B, T);
    report("hmma m16n8k16 x8 chains", run(k_hmma<8>, B, T, out), 2048, 8, B, T);
    report("imma m16n8k32 x4 chains", run(k_imma<4>, B, T, out), 4096, 4, B, T);
    report("imma m16n8k32 x8 chains", run(k_imma<8>, B, T, out), 4096, 8, B, T);
    report("dp4a x8 chains", run(k_dp4a<8>, B, T, out), 128, 8, B, T);
    // latency: one warp on one SM, one dependent chain
    {
        float ms = run(k_hmma<1>, 1, 32, out);
        printf("hmma latency  %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / kIters);
        ms = run(k_imma<1>, 1, 32, out);
        printf("imma latency  %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / kIters);
        ms = run(k_dp4a<1>, 1, 32, out);
        printf("dp4a latency  %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / kIters);
        ms = run(k_hmma<4>, 1, 32, out);
        printf("hmma 1 warp x4 chains: %.1f cycles/inst\n", ms * 1e-3 * ghz * 1e9 / kIters / 4);
        ms = run(k_hmma<4>, 1, 128, out);
        printf("hmma 4 warps (1/SMSP) x4 chains: %.1f cycles/inst/SMSP\n", ms * 1e-3 * ghz * 1e9 / kIters / 4);
        ms = run(k_imma<4>, 1, 128, out);
        printf("imma 4 warps (1/SMSP) x4 chains: %.1f cycles/inst/SMSP\n", ms * 1e-3 * ghz * 1e9 / kIters / 4);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s, %d SMs, %.3f GHz\n", cudaGetErrorString(e), sms, ghz);
    return 0;
}
