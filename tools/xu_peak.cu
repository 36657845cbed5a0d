// xu_peak.cu -- throughput of the conversions on the fp32 path's critical instructions
// (reading D28: F2I.S64 for every message placed on the 2^-34 grid, I2F.S64 for every
// gathered posterior), against FMUL and an integer-only alternative.  One CTA of 1024
// threads per SM, 8 independent chains per thread, timed with clock64 on the SM: thread
// instructions per SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/xu_peak tools/xu_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8, kIters = 2048, kUnroll = 8;
enum { OP_FMUL = 0, OP_F2I64, OP_I2F64, OP_F2I32, OP_I2F32, OP_I2F64_F64, OP_COUNT };
static const char *kNames[OP_COUNT] = {"FMUL", "F2I.S64 (float -> int64)", "I2F.S64 (int64 -> float)",
                                       "F2I.S32 (float -> int32)", "I2F.S32 (int32 -> float)",
                                       "I2F.F64.S64 (int64 -> double)"};

template <int OP>
__global__ void __launch_bounds__(1024, 1) k_peak(float *sink, long long *cycles) {
    float f[kChains];
    long long x[kChains];
    int y[kChains];
    double d[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        f[c] = 1.0f + threadIdx.x * 1e-3f + c;
        x[c] = 12345 + threadIdx.x + c;
        y[c] = 77 + threadIdx.x + c;
        d[c] = 0.0;
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                if constexpr (OP == OP_FMUL) f[c] = f[c] * 1.0000001f;
                else if constexpr (OP == OP_F2I64) { x[c] = __float2ll_rn(f[c]); f[c] = __int_as_float((int)x[c] | 0x3f800000); }
                else if constexpr (OP == OP_I2F64) { f[c] = __ll2float_rn(x[c]); x[c] = (long long)__float_as_int(f[c]) + c; }
                else if constexpr (OP == OP_F2I32) { y[c] = __float2int_rn(f[c]); f[c] = __int_as_float(y[c] | 0x3f800000); }
                else if constexpr (OP == OP_I2F32) { f[c] = __int2float_rn(y[c]); y[c] = __float_as_int(f[c]) + c; }
                else if constexpr (OP == OP_I2F64_F64) { d[c] = __ll2double_rn(x[c]); x[c] = __double_as_longlong(d[c]) + c; }
            }
        }
    }
    const long long t1 = clock64();
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc += f[c] + (float)x[c] + (float)y[c] + (float)d[c];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
double run(int sms, float *sink, long long *cyc) {
    k_peak<OP><<<sms, 1024>>>(sink, cyc);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < sms; ++i) m += h[i];
    m /= sms;
    // OP_F2I64 / I2F64 / 32-bit: each step is the conversion plus one ALU op (the bit trick
    // that keeps the chain dependent), so the conversion rate is an upper-bound estimate
    return 1024.0 * kIters * kUnroll * kChains / m;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *sink;
    long long *cyc;
    cudaMalloc(&sink, sizeof(float) * sms * 1024);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    double r[OP_COUNT];
    r[0] = run<0>(sms, sink, cyc); r[1] = run<1>(sms, sink, cyc); r[2] = run<2>(sms, sink, cyc);
    r[3] = run<3>(sms, sink, cyc); r[4] = run<4>(sms, sink, cyc); r[5] = run<5>(sms, sink, cyc);
    printf("{\"unit\": \"thread-instructions per SM clock (steps of conversion + 1 ALU op)\", \"sms\": %d", sms);
    for (int i = 0; i < OP_COUNT; ++i) printf(", \"%s\": %.2f", kNames[i], r[i]);
    printf("}\n");
    return 0;
}
