// rowcore_f32.cuh -- fp32 check-row core shared by the fp32 streaming kernels
// (k_stream.cuh, k_stream_pipe.cuh), the two-scan check pass and the fp32 layered kernel
// (k_resident_f32.cuh).
#pragma once
#include <cstdint>

namespace ldpc {

// fp32 check row (one frame per lane), branch-free.  Reading D11: one RN rounding
// per operation (__fsub_rn/__fmul_rn, no FMA).  Two minima with multiplicity:
// m2 = min(m2, max(m1, x)), m1 = min(m1, x), argmin on strict '<' (lowest position).
// State word W: bit j = sign of L_mn (1 = negative), bit 16 + ñ set (one-hot position).
// Selections work on the IEEE bit patterns: |L| = A or B is A + [j == ñ] (B - A) as a
// 32-bit integer (exact; IMAD on the FMA pipe), the sign is an XOR of bit 31.
// f32_row_q also returns q_mn = Z_n - L^(k-1)_mn (the layered update writes q + L^(k)_mn).
template <int DC>
__device__ __forceinline__ void f32_row_q(const float (&L)[DC], bool first_iter, float A0, float B0, uint32_t W0,
                                          float alpha, float beta, float &A, float &B, uint32_t &Wn, float (&r)[DC],
                                          float (&q)[DC]) {
    static_assert(DC <= 16, "one-hot position bits 16..31");
    if (first_iter) {
#pragma unroll
        for (int j = 0; j < DC; ++j) q[j] = L[j];                    // L^(0)_mn = 0
    } else {
        const uint32_t a0 = __float_as_uint(A0), db = __float_as_uint(B0) - a0;
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            const uint32_t isel = (W0 << (15 - j)) >> 31;            // [n == ñ]
            const uint32_t mag = isel * db + a0;                     // f(A,B,n,ñ)
            const uint32_t lold = mag ^ ((W0 << (31 - j)) & 0x80000000u);   // s_mn f(...)
            q[j] = __fsub_rn(L[j], __uint_as_float(lold));           // Z_n' - L_mn'  (D8)
        }
    }
    float m1 = fabsf(q[0]), m2 = __int_as_float(0x7f800000);
    int i1 = 0;
    uint32_t sq = q[0] < 0.0f ? 1u : 0u;
#pragma unroll
    for (int j = 1; j < DC; ++j) {
        const float x = fabsf(q[j]);
        i1 = x < m1 ? j : i1;
        m2 = fminf(m2, fmaxf(m1, x));
        m1 = fminf(m1, x);
        sq |= (q[j] < 0.0f ? 1u : 0u) << j;
    }
    const uint32_t par = __popc(sq) & 1u;
    // P:341-353; magnitudes saturate at 2^20 (reading D28: keeps the exact posterior sums bounded)
    A = fminf(fmaxf(__fsub_rn(__fmul_rn(alpha, m1), beta), 0.0f), 1048576.0f);
    B = fminf(fmaxf(__fsub_rn(__fmul_rn(alpha, m2), beta), 0.0f), 1048576.0f);
    const uint32_t sg = par ? (~sq & ((1u << DC) - 1u)) : sq;       // s = prod of the others' signs
    const uint32_t oh = 0x10000u << i1;
    Wn = sg | oh;
    const uint32_t a1 = __float_as_uint(A), db1 = __float_as_uint(B) - a1;
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        const uint32_t isel = (oh << (15 - j)) >> 31;
        const uint32_t mag = isel * db1 + a1;
        r[j] = __uint_as_float(mag ^ ((sg << (31 - j)) & 0x80000000u));
    }
}

template <int DC>
__device__ __forceinline__ void f32_row(const float (&L)[DC], bool first_iter, float A0, float B0, uint32_t W0,
                                        float alpha, float beta, float &A, float &B, uint32_t &Wn, float (&r)[DC]) {
    float q[DC];
    f32_row_q<DC>(L, first_iter, A0, B0, W0, alpha, beta, A, B, Wn, r, q);
}

}  // namespace ldpc
