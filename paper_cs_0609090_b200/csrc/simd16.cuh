// simd16.cuh -- 16x2 integer SIMD helpers for sm_100a (two frames per 32-bit lane).
//
// Each 32-bit register holds the same quantity for two frames: frame "lo" in bits
// 0-15, frame "hi" in bits 16-31, as signed 16-bit values.  The intrinsics below
// map to single SASS instructions on sm_100a (checked with cuobjdump -sass):
//   __vadd2 -> VIADD.16x2, __vmins2/__vmaxs2 -> VIMNMX.S16x2,
//   __viaddmin_s16x2_relu -> VIADDMNMX.S16x2.RELU, prmt -> PRMT, sel -> LOP3.
#pragma once
#include <cstdint>

namespace ldpc {

__device__ __forceinline__ uint32_t vadd(uint32_t a, uint32_t b) { return __vadd2(a, b); }
__device__ __forceinline__ uint32_t vmin(uint32_t a, uint32_t b) { return __vmins2(a, b); }
__device__ __forceinline__ uint32_t vmax(uint32_t a, uint32_t b) { return __vmaxs2(a, b); }
// Constants the kernels keep in REGISTERS (loaded from the kernel parameters, so ptxas
// cannot see their values): they let bitwise-NOT and some additions run as IMAD on
// the FMA pipe instead of LOP3 / IADD3 on the ALU pipe, which is the binding pipe of
// the integer row core (ncu: ALU 69% vs FMA 15% busy).
struct RegK {
    uint32_t zero;   // 0
    uint32_t m1;     // 0xFFFFFFFF
    uint32_t one;    // 1
    uint32_t m2;     // 0xFFFFFFFE (-2)
};
__host__ __device__ inline RegK make_regk() { return RegK{0u, 0xFFFFFFFFu, 1u, 0xFFFFFFFEu}; }
// ~a = a * (-1) + (-1): exact bitwise NOT as one IMAD (FMA pipe)
__device__ __forceinline__ uint32_t fnot(uint32_t a, const RegK &k) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %2;" : "=r"(d) : "r"(a), "r"(k.m1));
    return d;
}
// a + c (32-bit, wrapping) as one IMAD a * 1 + c (FMA pipe)
__device__ __forceinline__ uint32_t fadd32(uint32_t a, uint32_t c, const RegK &k) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(k.one), "r"(c));
    return d;
}
// packed 16x2 (P form) -> "V form" hi*65536 + lo as a 32-bit integer, so that one
// 32-bit integer add adds both lanes exactly: p - ((p & 0x8000) << 1)  (LOP3 + IMAD)
__device__ __forceinline__ uint32_t vform(uint32_t p, const RegK &k) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(p & 0x8000u), "r"(k.m2), "r"(p));
    return d;
}
// 0x10000 - a per half for halves in (0, 0x10000): one IMAD (the 0x8000-biased negation:
// (q + 0x8000) -> (-q + 0x8000))
__device__ __forceinline__ uint32_t negb(uint32_t a, const RegK &k) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(k.m1), "r"(0x00010000u));
    return d;
}
// -a per half (IMAD NOT + VIADD)
__device__ __forceinline__ uint32_t vneg(uint32_t a, const RegK &k) { return __vadd2(fnot(a, k), 0x00010001u); }
// min(a + b, c) per half, then max(., 0)   (VIADDMNMX.S16x2.RELU)
__device__ __forceinline__ uint32_t vaddmin_relu(uint32_t a, uint32_t b, uint32_t c) {
    return __viaddmin_s16x2_relu(a, b, c);
}
// min(a + b, c) per half  (VIADDMNMX.S16x2)
__device__ __forceinline__ uint32_t vaddmin(uint32_t a, uint32_t b, uint32_t c) {
    return __viaddmin_s16x2(a, b, c);
}
// bitwise select: m ? a : b   (one LOP3)
__device__ __forceinline__ uint32_t sel(uint32_t m, uint32_t a, uint32_t b) { return (a & m) | (b & ~m); }
// PTX prmt in its generic mode: bit 3 of each selector nibble replicates the sign
// (bit 7) of the selected byte.  __byte_perm() masks that bit off, hence inline PTX.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
    return d;
}
// per-half sign mask: 0xFFFF in each half whose value is negative
__device__ __forceinline__ uint32_t signmask(uint32_t a) { return prmt(a, 0u, 0xBB99u); }
// pack two int16 into a word (lo, hi)
__host__ __device__ __forceinline__ uint32_t pack2(int lo, int hi) {
    return (uint32_t)(lo & 0xFFFF) | ((uint32_t)hi << 16);
}
__device__ __forceinline__ int lo16(uint32_t v) { return (int)(int16_t)(v & 0xFFFFu); }
__device__ __forceinline__ int hi16(uint32_t v) { return (int)(int16_t)(v >> 16); }

}  // namespace ldpc
