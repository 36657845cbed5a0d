// alu_peak.cu -- integer-pipe throughput microbenchmark for the ALU roofline (SURVEY §8(d):
// "achieved int instructions / measured int-op peak").  One CTA of 1024 threads per SM,
// 8 independent dependency chains per thread, each chain a long run of one instruction
// kind; the CTA times itself with clock64, so the result is in thread-instructions per
// SM clock, independent of the clock frequency.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/alu_peak tools/alu_peak.cu
//   build/alu_peak > profiles/r01_alu_peak.json
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;
constexpr int kUnroll = 8;

enum Op { OP_VIMNMX = 0, OP_LOP3, OP_IADD3, OP_PRMT, OP_VIADDMNMX, OP_IMAD, OP_LOP3_IMAD, OP_HMNMX2, OP_LOP3_HMNMX2,
          OP_COUNT };
static const char *kNames[OP_COUNT] = {"VIMNMX.S16x2", "LOP3", "IADD3", "PRMT", "VIADDMNMX.S16x2.RELU", "IMAD",
                                       "LOP3+IMAD (dual issue)", "HMNMX2", "LOP3+HMNMX2 (dual issue)"};

// One instruction of kind OP.  Rounds alternate between two forms (min / max, two LUTs,
// add / sub, two selectors) and every chain reads its neighbour, so ptxas can neither fold
// consecutive rounds (e.g. two mins into one VIMNMX3) nor collapse them algebraically.
template <int OP>
__device__ __forceinline__ uint32_t step(int round, uint32_t x, uint32_t y, uint32_t z) {
    uint32_t r;
    const bool odd = round & 1;
    if constexpr (OP == OP_VIMNMX) {
        if (odd) asm volatile("max.s16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
        else asm volatile("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
    } else if constexpr (OP == OP_LOP3) {
        if (odd) asm volatile("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(r) : "r"(x), "r"(y), "r"(z));
        else asm volatile("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(r) : "r"(x), "r"(y), "r"(z));
    } else if constexpr (OP == OP_IADD3) {
        if (odd) asm volatile("{ .reg .u32 t; add.u32 t, %1, %2; sub.u32 %0, t, %3; }" : "=r"(r) : "r"(x), "r"(y), "r"(z));
        else asm volatile("{ .reg .u32 t; sub.u32 t, %1, %2; add.u32 %0, t, %3; }" : "=r"(r) : "r"(x), "r"(y), "r"(z));
    } else if constexpr (OP == OP_PRMT) {
        if (odd) asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(r) : "r"(x), "r"(y));
        else asm volatile("prmt.b32 %0, %1, %2, 0x6273;" : "=r"(r) : "r"(x), "r"(y));
    } else if constexpr (OP == OP_VIADDMNMX) {
        r = odd ? __viaddmax_s16x2_relu(x, y, z) : __viaddmin_s16x2_relu(x, y, z);
    } else if constexpr (OP == OP_HMNMX2) {
        if (odd) asm volatile("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
        else asm volatile("min.f16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
    } else if constexpr (OP == OP_IMAD) {
        asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(y), "r"(z));
    }
    return r;
}

template <int OP>
__global__ void __launch_bounds__(1024, 1) k_peak(uint32_t *sink, long long *cycles) {
    uint32_t v[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = ((threadIdx.x * 7u + 3u * c + 1u) & 0x3FFFu) * 0x10001u;   // finite fp16 pairs
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            uint32_t w[kChains];
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                const uint32_t x = v[c], y = v[(c + 1) % kChains], z = v[(c + 2) % kChains];
                if constexpr (OP == OP_LOP3_IMAD) w[c] = (c & 1) ? step<OP_IMAD>(u, x, y, z) : step<OP_LOP3>(u, x, y, z);
                else if constexpr (OP == OP_LOP3_HMNMX2) w[c] = (c & 1) ? step<OP_HMNMX2>(u, x, y, z) : step<OP_LOP3>(u, x, y, z);
                else w[c] = step<OP>(u, x, y, z);
            }
#pragma unroll
            for (int c = 0; c < kChains; ++c) v[c] = w[c];
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= v[c];
    if (s == 0x12345678u) sink[blockIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
static double run(int sms, uint32_t *sink, long long *cyc) {
    k_peak<OP><<<sms, 1024>>>(sink, cyc);   // warm-up
    k_peak<OP><<<sms, 1024>>>(sink, cyc);
    cudaDeviceSynchronize();
    long long *h = new long long[sms];
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)h[i];
    mean /= sms;
    delete[] h;
    const double ops = 1024.0 * kIters * kUnroll * kChains;
    return ops / mean;   // thread-instructions per SM clock
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    uint32_t *sink;
    long long *cyc;
    cudaMalloc(&sink, sizeof(uint32_t) * sms);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    double r[OP_COUNT];
    r[OP_VIMNMX] = run<OP_VIMNMX>(sms, sink, cyc);
    r[OP_LOP3] = run<OP_LOP3>(sms, sink, cyc);
    r[OP_IADD3] = run<OP_IADD3>(sms, sink, cyc);
    r[OP_PRMT] = run<OP_PRMT>(sms, sink, cyc);
    r[OP_VIADDMNMX] = run<OP_VIADDMNMX>(sms, sink, cyc);
    r[OP_IMAD] = run<OP_IMAD>(sms, sink, cyc);
    r[OP_LOP3_IMAD] = run<OP_LOP3_IMAD>(sms, sink, cyc);
    r[OP_HMNMX2] = run<OP_HMNMX2>(sms, sink, cyc);
    r[OP_LOP3_HMNMX2] = run<OP_LOP3_HMNMX2>(sms, sink, cyc);
    const cudaError_t e = cudaGetLastError();
    printf("{\"device\": \"%s\", \"sms\": %d, \"unit\": \"thread-instructions per SM clock\", \"error\": \"%s\",\n"
           " \"ops_per_sm_clk\": {",
           p.name, sms, cudaGetErrorString(e));
    for (int i = 0; i < OP_COUNT; ++i) printf("%s\"%s\": %.2f", i ? ", " : "", kNames[i], r[i]);
    printf("}}\n");
    return e == cudaSuccess ? 0 : 1;
}
