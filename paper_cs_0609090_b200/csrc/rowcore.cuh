// rowcore.cuh -- one check row of the memory-efficient single-scan min-sum
// iteration (§5, with the offset modification P:347-353),
// for two frames at once in 16x2 SIMD lanes.
//
// Value domain: every LLR-like quantity is held DOUBLED (Lhat = 2 L, Ahat = 2 A,
// ...).  Doubling lets the magnitude be taken with one VIMNMX as
// m~ = max(q, ~q) = 2|q| - [q < 0]: m~ orders rows exactly like |q| and
// |q| = ceil(m~ / 2), so min1 / min2 / argmin come out exact.
//
// Compact state of a row (per frame pair), the paper's (A_m, B_m, ñ_m, s_mn):
//   A, B : doubled magnitudes 2A_m, 2B_m in each 16-bit half (B >= A)
//   W    : per-edge bits, one 16-bit half per frame (lo frame bits 0-15, hi frame 16-31):
//            half bit j     : s of edge j   (1 means L_mn < 0)
//            half bit 8 + j : idx of edge j (1 means n is an argmin, n = ñ_m)          dc <= 8.
//          One left shift by 7 - j puts edge j's two bits of both frames at bit 7 of every
//          byte (sign: bytes 0 / 2, idx: bytes 1 / 3), so one PRMT per mask expands them.
//          new_state builds W with IMADs on the FMA pipe only (pack_bits below).
//   1-bit message format (FMT_1BIT, "1-bit messages"): the persistent W keeps only
//          the sign bits (the only per-edge datum) and ñ_m as an INDEX per check and frame:
//          half bits 0-7 = signs, half bits 8-12 = ñ (the edge number; see pack_bits for ties),
//          so expand_idx() rebuilds the flags with two shifts when the state is loaded.
#pragma once
#include "args.cuh"
#include "rowcore_types.cuh"
#include "simd16.cuh"

namespace ldpc {

struct RowState {
    uint32_t A, B, W;
};

// index-coded ñ (FMT_1BIT) -> the per-edge flag layout the rebuild reads.  An index >= 8 (only
// after a tie in the minimum, see pack_bits) sets no flag: a tie means A == B, where the flag
// does not matter (reading D3).
__device__ __forceinline__ uint32_t expand_idx(uint32_t W) {
    const uint32_t tl = (W >> 8) & 15u, th = (W >> 24) & 15u;
    return (W & 0x00FF00FFu) | ((0x100u << tl) & 0x0000FF00u) | ((0x1000000u << th) & 0xFF000000u);
}

// Bit packing on the FMA pipe.  For a 16x2 mask m (0xFFFF in the halves where a condition
// holds: lo_m, hi_m in {0, 1}) and K = 2^p, p < 16, the 32-bit product is
//   m K = lo_m (2^16 - 1) K + hi_m (2^32 - 2^16) K == 2^16 (lo_m - hi_m) K - lo_m K  (mod 2^32),
// so a sum S of such products over distinct bit positions p is 2^16 (LO - HI) - LO with
// LO = sum lo_m 2^p, HI = sum hi_m 2^p (both < 2^16), and
//   -S (1 + 2^16) == LO + 2^16 HI  (mod 2^32):
// one IMAD per mask (S += m K) and one per row (W = S * -(0x10001)) give the packed word
// without an ALU-pipe instruction.  For an index code (FMT_1BIT) K = j 2^8 sums the edge
// numbers of the argmin flags: exact for the unique argmin; after a tie the sum (< 2^5) may
// be any value, which is harmless (expand_idx).
__device__ __forceinline__ uint32_t mad_bits(uint32_t m, uint32_t K, uint32_t S) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(m), "r"(K), "r"(S));
    return d;
}
__device__ __forceinline__ uint32_t unpack_bits(uint32_t S) {
    uint32_t d;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(S), "r"(0xFFFEFFFFu));
    return d;
}

// Rebuild L^(k-1)_mn = s f(A, B, n, ñ) and form
// q_mn = Z^(k-1)_n - L^(k-1)_mn (index reading D8) for all edges.
// BIASED: L holds Lhat + 0x4000 per lane (see k_resident_atom.cuh); the bias is folded
// into the four candidates so q comes out unbiased at no extra cost per edge.
template <int DC, bool BIASED = false>
__device__ __forceinline__ void rebuild_q(const uint32_t (&L)[DC], const RowState &st, uint32_t (&q)[DC],
                                          const RegK &k) {
    uint32_t nA, nB, A = st.A, B = st.B;
    if (BIASED) {
        nA = __vadd2(fnot(st.A, k), 0xC001C001u);              // -A - 0x4000 = ~A + 1 - 0x4000
        nB = __vadd2(fnot(st.B, k), 0xC001C001u);
        A = __vadd2(st.A, 0xC000C000u);                        // A - 0x4000
        B = __vadd2(st.B, 0xC000C000u);
    } else {
        nA = vneg(st.A, k);
        nB = vneg(st.B, k);
    }
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        const uint32_t ws = st.W << (7 - j);       // edge j's bits -> bit 7 of each byte
        const uint32_t sm = prmt(ws, 0u, 0xAA88u), ix = prmt(ws, 0u, 0xBB99u);
        const uint32_t mag = sel(ix, B, A), nmag = sel(ix, nB, nA);
        q[j] = vadd(L[j], sel(sm, mag, nmag));          // Z - L_old: L_old = s*mag
    }
}

// B8 rebuild for the barrier-free resident kernel: L holds 2Z + 0x4000 per lane; the four
// candidates 0x4000 -/+ A, B are formed by IMAD (lanes stay non-negative, no carries) and
// q + 0x8000 = L + candidate is one 32-bit IMAD per edge (FMA pipe).
// Q0 = (0x8000 - bias) per lane: 0x40004000 for words biased by 0x4000 (streaming kernels),
// 0x40014001 for words biased by 0x3FFF (barrier-free resident kernel, k_resident_atom.cuh).
template <int DC, uint32_t Q0 = 0x40004000u>
__device__ __forceinline__ void rebuild_q_b8(const uint32_t (&L)[DC], const RowState &st, uint32_t (&q)[DC],
                                             const RegK &k) {
    // -L_old + Q0 is Q0 + mag for a negative L_old and Q0 - mag for a positive one; per lane
    // the two sum to 2 Q0 (< 0x10000, no carries), so once the magnitude is selected by the
    // argmin mask the other sign is one IMAD: 2 Q0 - (Q0 + mag)
    const uint32_t nA = fadd32(st.A, Q0, k), nB = fadd32(st.B, Q0, k);
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        const uint32_t ws = st.W << (7 - j);       // edge j's bits -> bit 7 of each byte
        const uint32_t sm = prmt(ws, 0u, 0xAA88u), ix = prmt(ws, 0u, 0xBB99u);
        const uint32_t neg = sel(ix, nB, nA);                                   // Q0 + mag
        uint32_t pos;                                                           // Q0 - mag
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(pos) : "r"(neg), "r"(k.m1), "r"(Q0 + Q0));
        q[j] = fadd32(L[j], sel(sm, neg, pos), k);
    }
}

// Smallest and second smallest of DC packed values (with multiplicity), as a
// pairwise tree: leaves (min, max), merges m1 = min(a1, b1),
// m2 = min3(max(a1, b1), a2, b2).  Shorter dependency chains than a running scan.
// U: values are unsigned 16-bit lanes (the 0x8000-biased domain of new_state<B8>).
template <int DC, bool U = false>
__device__ __forceinline__ void two_min(const uint32_t (&v)[DC], uint32_t &m1, uint32_t &m2) {
    constexpr int NL = (DC + 1) / 2;
    uint32_t a1[NL], a2[NL];
#pragma unroll
    for (int i = 0; i < DC / 2; ++i) {
        a1[i] = U ? __vminu2(v[2 * i], v[2 * i + 1]) : vmin(v[2 * i], v[2 * i + 1]);
        a2[i] = U ? __vmaxu2(v[2 * i], v[2 * i + 1]) : vmax(v[2 * i], v[2 * i + 1]);
    }
    if (DC & 1) {
        a1[NL - 1] = v[DC - 1];
        a2[NL - 1] = U ? 0xFFFFFFFFu : 0x7FFF7FFFu;
    }
#pragma unroll
    for (int n = NL; n > 1; n = (n + 1) / 2) {
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            const uint32_t x1 = a1[2 * i], y1 = a1[2 * i + 1];
            if (U) {
                a1[i] = __vminu2(x1, y1);
                a2[i] = __vimin3_u16x2(__vmaxu2(x1, y1), a2[2 * i], a2[2 * i + 1]);
            } else {
                a1[i] = vmin(x1, y1);
                a2[i] = __vimin3_s16x2(vmax(x1, y1), a2[2 * i], a2[2 * i + 1]);
            }
        }
        if (n & 1) {
            a1[n / 2] = a1[n - 1];
            a2[n / 2] = a2[n - 1];
        }
    }
    m1 = a1[0];
    m2 = a2[0];
}

// doubled magnitude of the variant from m~ = 2|q| - [q < 0] (B8: m = 2|q| + 0x8000 per lane, exact)
// Normalized path out of line: a call cannot be if-converted, so the offset path (every
// BASELINE integer config) does not execute the normalized instructions speculatively.
static __device__ __noinline__ uint32_t variant_mag_norm(uint32_t m, uint32_t na, uint32_t ns, uint32_t nmask, uint32_t nb2,
                                                  uint32_t q2) {
    const uint32_t t = __vadd2(m, 0x00010001u) & 0xFFFEFFFEu;   // 2|q| per lane
    const uint32_t x = ((t * na) >> ns) & nmask;                  // 2 floor(na |q| / 2^ns) (no lane overflow: planner)
    return vaddmin_relu(x, nb2, q2);
}

// VM: -1 = decide offset / normalized at run time (v.norm); 0 / 1 = the caller already did
// (the barrier-free kernel dispatches once per iteration, keeping the branch out of its rows)
template <bool B8 = false, int VM = -1>
__device__ __forceinline__ uint32_t variant_mag(uint32_t m, const VarK &v, const RegK &k) {
    if (B8) {
        // m = 0x8000 + 2|q| exactly (new_state<B8>); as a signed half that is 2|q| - 0x8000, so
        // relu(min(2|q| - 2 beta, 2Q)) is one VIADDMNMX with the unbias folded into the added
        // constant 0x8000 - 2 beta (16-bit wrap-around add)
        if (VM == 1 || (VM < 0 && __builtin_expect(v.norm != 0, 0)))
            return variant_mag_norm(m ^ 0x80008000u, v.na, v.ns, v.nmask, v.nb2, v.q2);
        return vaddmin_relu(m, v.nb8, v.q2);
    }
    if (__builtin_expect(v.norm != 0, 0)) return variant_mag_norm(m, v.na, v.ns, v.nmask, v.nb2, v.q2);
    // relu(min(m~ + 1 - 2 beta, 2Q + 1)) with the low bit cleared is exact (m~ in {2|q|-1, 2|q|})
    return vaddmin_relu(m, v.nbeta2p1, v.q2p1) & 0xFFFEFFFEu;
}

// New compact state from the q's and the new messages L^(k)_mn (doubled) to be
// accumulated into Z^(k)_n:
//   A = min(max(min1 - beta, 0), Q), B = min(max(min2 - beta, 0), Q)  (readings D5, D6)
//   ñ = argmin |q| (ties: any minimiser -- unobservable, A = B then; reading D3)
//   s_mn = prod_{n' != n} sgn(q_mn')  (sgn(0) = +1, reading D1)
//
// B8 = true (barrier-free resident kernel): q arrives as q + 0x8000 per lane (unsigned),
// so 32-bit IMADs produced it without lane carries; magnitudes and minima are then
// unsigned, the per-lane sign mask is [q >= 0] (bit 15), and the returned messages are
// "V form + 0x8000": r ^ 0x8000 in the low lane == V(r) + 0x8000 as a 32-bit integer, so a
// 32-bit RED adds them exactly (the accumulator start value is lowered by dv_n 0x8000).
// IDX = true (FMT_1BIT): ñ is stored as an index code (header), one IMAD per edge.
template <int DC, bool B8 = false, int VM = -1, bool IDX = false>
__device__ __forceinline__ void new_state(const uint32_t (&q)[DC], const VarK &vk, RowState &st, uint32_t (&r)[DC],
                                          const RegK &k) {
    uint32_t mt[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j)                                 // 2|q| - [q<0]  (B8: 2|q| + 0x8000, exact)
        mt[j] = B8 ? __vmaxu2(q[j], negb(q[j], k)) : vmax(q[j], fnot(q[j], k));
    uint32_t m1, m2;
    two_min<DC, B8>(mt, m1, m2);
    uint32_t par = q[0];
#pragma unroll
    for (int j = 1; j < DC; ++j) par ^= q[j];
    // B8: bit 15 of q_b is [q >= 0], so the XOR counts non-negative q's; the product is
    // negative iff the count of negative ones, DC - that, is odd
    if (B8 && (DC & 1)) par ^= 0x80008000u;
    const uint32_t Pm = signmask(par);                          // product of all signs < 0
    const uint32_t A = variant_mag<B8, VM>(m1, vk, k);
    const uint32_t B = variant_mag<B8, VM>(m2, vk, k);
    uint32_t nA, nB, Ac = A, Bc = B;
    if (B8) {
        // message candidates V(+-A) + 0x8000 (the RED operand): V is linear and the lanes of
        // A are in [0, 2Q], so V(-A) + 0x8000 = 0x8000 - A is one IMAD (no lane borrow)
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(nA) : "r"(A), "r"(k.m1), "r"(0x00008000u));
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(nB) : "r"(B), "r"(k.m1), "r"(0x00008000u));
        Ac = fadd32(A, 0x00008000u, k);
        Bc = fadd32(B, 0x00008000u, k);
    } else {
        nA = vneg(A, k);
        nB = vneg(B, k);
    }
    // message for an edge whose own q is >= 0 carries the sign of the full product
    const uint32_t Apos = sel(Pm, nA, Ac), Bpos = sel(Pm, nB, Bc);
    uint32_t Aneg = 0, Bneg = 0;
    if (!B8) {
        Aneg = sel(Pm, Ac, nA);
        Bneg = sel(Pm, Bc, nB);
    }
    const uint32_t cm1 = fnot(m1, k);                           // -m1 - 1
    uint32_t S = 0;                                             // packed by IMADs (mad_bits)
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        const uint32_t ix = vaddmin(mt[j], cm1, k.zero);          // min(m~ - m1 - 1, 0): 0xFFFF iff argmin
        const uint32_t sq = signmask(q[j]);                     // 0xFFFF: q < 0  (B8: q >= 0)
        if (B8) {
            // per lane the two candidates of one magnitude sum to 0x10000 (0x8000 -+ A ...,
            // lanes never zero), so the opposite-sign message is one IMAD: 0x10000 - x
            const uint32_t x = sel(ix, Bpos, Apos);
            uint32_t y;
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(y) : "r"(x), "r"(k.m1), "r"(0x00010000u));
            r[j] = sel(sq, x, y);
        } else {
            r[j] = sel(sq, sel(ix, Bneg, Aneg), sel(ix, Bpos, Apos));
        }
        S = mad_bits(sq, 1u << j, S);                           // sign bit j
        S = mad_bits(ix, IDX ? (uint32_t)j << 8 : 0x100u << j, S);   // idx flag 8 + j / index code
    }
    uint32_t W = unpack_bits(S);
    if (B8) W ^= ~Pm & 0x00FF00FFu;                             // s = sgn(q) * product ([q>=0] bits stored)
    else W ^= Pm & 0x00FF00FFu;                                 // s = sgn(q) * product
    st.A = A;
    st.B = B;
    st.W = W;
}

// Hard-decision parity of the row for the syndrome (x̂ = 1 iff Z <= 0, P:168-172;
// H x̂ = 0 test): bit 15 / bit 31 set iff the row's parity is odd.
// Per half, sign(Lhat - 1) = [L <= 0].  The subtraction is one 32-bit IMAD of
// -0x00010001: the low half can borrow from the high half (when it is 0), which
// makes the high half Lhat_hi - 2 instead of Lhat_hi - 1 -- the same sign, because
// doubled values are even.
// cpar = -(0x00010001) for plain doubled values, -(0x40014001) for biased ones.
template <int DC>
__device__ __forceinline__ uint32_t row_parity(const uint32_t (&L)[DC], const RegK &k, uint32_t cpar = 0xFFFEFFFFu) {
    uint32_t p = 0;
#pragma unroll
    for (int j = 0; j < DC; ++j) p ^= fadd32(L[j], cpar, k);
    return p & 0x80008000u;
}

template <int FMT>
struct StateIO {
    static constexpr int kWords = FMT == FMT_C16 ? 3 : 2;
    __device__ __forceinline__ static RowState load(const uint32_t *base, size_t stride, size_t idx) {
        RowState s;
        if (FMT == FMT_C16) {
            s.A = __ldcg(base + idx);
            s.B = __ldcg(base + stride + idx);
            s.W = __ldcg(base + 2 * stride + idx);
        } else {
            const uint32_t X = __ldcg(base + idx);
            s.A = prmt(X, 0u, 0x4240u);
            s.B = prmt(X, 0u, 0x4341u);
            s.W = expand_idx(__ldcg(base + stride + idx));
        }
        return s;
    }
    __device__ __forceinline__ static void store(uint32_t *base, size_t stride, size_t idx, const RowState &s) {
        if (FMT == FMT_C16) {
            __stcg(base + idx, s.A);
            __stcg(base + stride + idx, s.B);
            __stcg(base + 2 * stride + idx, s.W);
        } else {
            __stcg(base + idx, prmt(s.A, s.B, 0x6240u));
            __stcg(base + stride + idx, s.W);
        }
    }
};

}  // namespace ldpc
