// k_resident_atom.cuh -- barrier-free decode-resident single-scan min-sum kernel
// (flooding schedule, integer LLRs).  Same residency as k_resident.cuh -- one CTA per
// frame pair, posterior double buffer in shared memory, compact state in TMEM, Z^(0)
// restarted by a TMA bulk copy -- but the accumulation Z^(k)_n += L^(k)_mn is
// a shared-memory atomic add (RED.ADD on 32-bit words), so rows need no conflict-free
// batching and there is no barrier inside an iteration: every thread runs through its
// own rows back to back.
//
// Exactness of a 32-bit add on two 16-bit lanes: every posterior word holds
// 2 Z_n + 0x3FFF in each lane (kAtomBias).  |2 Z_n| <= 2 Q (dv + 1) < 0x4000 (checked by the
// planner), and so does every partial sum in any order, so both lanes stay in
// [0, 0x8000): non-negative lanes never carry or borrow across the lane boundary.  The
// message is added in "V form" (hi * 65536 + lo as a signed 32-bit integer), which is
// exactly the lane-wise add.  Gathers read the biased words directly; the bias is
// folded into the rebuilt previous message (rowcore.cuh rebuild_q<BIASED>) and the
// syndrome constant, so q_mn comes out unbiased with no extra work per edge.
//
// Row ownership: QC codes -- thread r of group g owns circulant row r of the base rows
// listed for group g (QcTab slots b; the two groups get base-row lists of equal total
// degree); other codes -- thread t owns rows t, t + T, t + 2T, ...  The TMEM column of
// a row's state is its slot b.
#pragma once
#include <type_traits>

#include "k_resident.cuh"

namespace ldpc {

// Posterior words hold 2Z + 0x3FFF per lane.  With |2Z| <= 2Q(dv+1) < 0x4000 (planner) every
// lane stays in [1, 0x7FFF] and the hard decision [Z <= 0] is the complement of bit 14, so
// a row's syndrome bit is an XOR of its gathered words (no per-edge subtraction).  Being
// odd, the words never equal 0x4000, which keeps the subtract-based final-pass parity
// (cpar = -0x40004000, rowcore.cuh row_parity) exact despite the lane borrow.
constexpr int kAtomBias = 0x3FFF;
constexpr uint32_t kAtomQ0 = 0x40014001u;    // (0x8000 - bias) per lane: q + 0x8000 = word + Q0 - 2 L_old

// Fixed buffer bases (ResArgs::fixed_bases; early stop, 4 Np <= kAtomFixOff, QC codes or general
// codes with the column table in shared memory): buffer 1 starts kAtomFixOff bytes after
// buffer 0 and the shift / column table is copied to shared memory with the shared address of
// buffer 0 folded into its offsets, so a row scan specialised on the iteration parity FP
// addresses Z^(k-1) and Z^(k) as [d + imm] -- two IMADs fewer per edge than adding the buffer
// bases held in registers (the early-stop kernel cannot keep them in uniform registers, which
// is what the fixed-iteration kernels do: LDS / ATOMS [R + UR]).
// kAtomFixOff: args.cuh (the planner sizes shared memory with it).

// Hard-decision parity of a row from its biased words: bit 14 / 30 set iff odd (the other bits
// are garbage).  OR-ed into the early-stop syndrome word as it stands: bit 14 of an OR is the OR
// of the rows' bits 14, so the bits need no shift or mask per row (kAtomSyndLo / kAtomSyndHi).
constexpr uint32_t kAtomSyndLo = 0x00004000u, kAtomSyndHi = 0x40000000u;
template <int DC>
__device__ __forceinline__ uint32_t atom_row_parity(const uint32_t (&L)[DC]) {
    uint32_t x = L[0];
#pragma unroll
    for (int j = 1; j < DC; ++j) x ^= L[j];
    return (DC & 1) ? ~x : x;                           // [Z <= 0] = NOT bit 14 (30)
}

// CSM (general codes): the [dc][M] column table was staged in shared memory at byte
// address sct (ResArgs::csr_smem), so the per-edge offsets are shared-memory loads
// FP (QC, or CSM): -1 = buffer bases bp / ba in registers; 0 / 1 = fixed bases, iteration
// parity (0: Z^(k-1) in buffer 0, Z^(k) in buffer 1; 1: the reverse); sct = shared address of
// the shift table (QC: entries (4 s, 4 j Z + base of buffer 0)) or of the column table (CSM:
// byte offsets, + base of buffer 0 when FP >= 0)
template <int DC, bool QC, bool ES, int VM, int FMT, bool CSM = false, int FP = -1>
__device__ __forceinline__ void atom_row(const ResArgs &a, const QcTab &t, const VarK &vk, uint32_t bp, uint32_t ba, int e0,
                                         uint32_t r4, int p, bool first_iter, RowState &st, uint32_t &synd,
                                         uint32_t sct = 0) {
    constexpr uint32_t OFF_L = FP == 1 ? kAtomFixOff : 0u, OFF_A = FP == 0 ? kAtomFixOff : 0u;
    uint32_t d[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        if (QC && FP >= 0) {
            uint32_t ex, ey;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(ex), "=r"(ey) : "r"(sct + 8u * (uint32_t)(e0 + j)));
            const uint32_t u = r4 + ex;
            d[j] = min(u - t.Z4, u) + ey;                 // base0 + 4 * (jZ + (r + s) mod Z)
        } else if (QC) {
            const uint2 e = t.ent[e0 + j];
            const uint32_t u = r4 + e.x;
            d[j] = min(u - t.Z4, u) + e.y;                 // 4 * (jZ + (r + s) mod Z)
        } else if (CSM) {
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d[j]) : "r"(sct + 4u * (uint32_t)(j * a.M + p)));
        } else {
            d[j] = __ldg(a.colT + (size_t)j * a.M + p);
        }
    }
    uint32_t L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        if constexpr (FP >= 0) {
            static_assert(QC || CSM, "fixed buffer bases need the shift / column table in shared memory");
            LDPC_CHECK(d[j] - bp + OFF_L < 4u * (uint32_t)a.N && (d[j] & 3u) == 0);   // (bp: base of Z^(k-1))
            asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(L[j]) : "r"(d[j]), "n"(OFF_L));
        } else {
            LDPC_CHECK(d[j] < 4u * (uint32_t)a.N && (d[j] & 3u) == 0);      // a variable of this code
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(L[j]) : "r"(d[j] + bp));
        }
    }
    if (ES) synd |= atom_row_parity<DC>(L);
    uint32_t q[DC];                                                      // q_mn + 0x8000 per lane
    if (first_iter) {
#pragma unroll
        for (int j = 0; j < DC; ++j) q[j] = fadd32(L[j], kAtomQ0, a.rk);    // L^(0)_mn = 0
    } else {
        rebuild_q_b8<DC, kAtomQ0>(L, st, q, a.rk);                         // Z_n - L^(k-1)_mn
    }
    uint32_t rn[DC];                                                     // V(L^(k)_mn) + 0x8000
    new_state<DC, true, VM, FMT == FMT_1BIT>(q, vk, st, rn, a.rk);
#pragma unroll
    for (int j = 0; j < DC; ++j) {                                        // Z^(k)_n += L^(k)_mn
        if constexpr (FP >= 0)
            asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(d[j]), "r"(rn[j]), "n"(OFF_A) : "memory");
        else
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(d[j] + ba), "r"(rn[j]) : "memory");
    }
}

// ---------------------------------------------------------------- FMT_FULL (§4)
// The single-scan of PAPER.md §4 keeps every check message L_mn: here one
// TMEM word per edge per frame pair, stored as c = kAtomQ0 - V(L) (= kAtomQ0 + 0x8000 minus
// the RED value V(L) + 0x8000), so the next iteration's q_mn + 0x8000 per lane =
// (2Z_n + 0x3FFF) + c is one IMAD (no rebuild from a compact state).  Same messages, posteriors and stopping as the compact form.
template <int DC>
__device__ __forceinline__ void full_tmem_load(uint32_t taddr, uint32_t (&c)[8]) {
    if constexpr (DC == 8) {
        tmem_ld4(taddr, c[0], c[1], c[2], c[3]);
        tmem_ld4(taddr + 4, c[4], c[5], c[6], c[7]);
    } else {
        constexpr int o4 = DC >= 4 ? 4 : 0;
        if constexpr (DC >= 4) tmem_ld4(taddr, c[0], c[1], c[2], c[3]);
        constexpr int o2 = o4 + ((DC - o4) >= 2 ? 2 : 0);
        if constexpr ((DC - o4) >= 2) tmem_ld2(taddr + o4, c[o4], c[o4 + 1]);
        if constexpr ((DC - o2) == 1) tmem_ld1(taddr + o2, c[o2]);
    }
    tmem_wait_ld_dep8(c);
}
template <int DC>
__device__ __forceinline__ void full_tmem_store(uint32_t taddr, const uint32_t (&c)[8]) {
    if constexpr (DC == 8) {
        tmem_st4(taddr, c[0], c[1], c[2], c[3]);
        tmem_st4(taddr + 4, c[4], c[5], c[6], c[7]);
    } else {
        constexpr int o4 = DC >= 4 ? 4 : 0;
        if constexpr (DC >= 4) tmem_st4(taddr, c[0], c[1], c[2], c[3]);
        constexpr int o2 = o4 + ((DC - o4) >= 2 ? 2 : 0);
        if constexpr ((DC - o4) >= 2) tmem_st2(taddr + o4, c[o4], c[o4 + 1]);
        if constexpr ((DC - o2) == 1) tmem_st1(taddr + o2, c[o2]);
    }
}

template <int DC, bool QC, bool ES, int VM>
__device__ __forceinline__ void atom_row_full(const ResArgs &a, const QcTab &t, const VarK &vk, uint32_t bp,
                                              uint32_t ba, int e0, uint32_t r4, int p, bool first_iter,
                                              uint32_t (&c)[8], uint32_t &synd) {
    uint32_t d[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        if (QC) {
            const uint2 e = t.ent[e0 + j];
            const uint32_t u = r4 + e.x;
            d[j] = min(u - t.Z4, u) + e.y;
        } else {
            d[j] = __ldg(a.colT + (size_t)j * a.M + p);
        }
    }
    uint32_t L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(L[j]) : "r"(d[j] + bp));
    if (ES) synd |= atom_row_parity<DC>(L);
    uint32_t q[DC];                                                      // q_mn + 0x8000 per lane
#pragma unroll
    for (int j = 0; j < DC; ++j) q[j] = fadd32(L[j], first_iter ? kAtomQ0 : c[j], a.rk);   // Z - L_old
    uint32_t rn[DC];
    RowState st;                                                         // unused: no compact state
    new_state<DC, true, VM>(q, vk, st, rn, a.rk);                           // Eq.(3)
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(d[j] + ba), "r"(rn[j]) : "memory");   // Z += L
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(c[j]) : "r"(rn[j]), "r"(a.rk.m1), "r"(kAtomQ0 + 0x8000u));
    }
}

// Two rows of one group in flight (FMT_FULL, QC): both rows' gathers are issued before
// either row's arithmetic, so each thread overlaps the shared-memory latency of one row
// with the other's work.  The full-message kernel is held to 2 CTAs/SM by TMEM, so the
// 4 warps per scheduler alone cannot hide that latency.  Flooding reads Z^(k-1) and
// accumulates into Z^(k) (different buffers), so the order of the two rows is free.
template <int DC, bool ES, int VM>
__device__ __forceinline__ void atom_row_full_x2(const ResArgs &a, const QcTab &t, const VarK &vk, uint32_t bp,
                                                 uint32_t ba, int e0, int e1, uint32_t r4, bool first_iter,
                                                 uint32_t (&c0)[8], uint32_t (&c1)[8], uint32_t &synd) {
    uint32_t d0[DC], d1[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        const uint2 x = t.ent[e0 + j], y = t.ent[e1 + j];
        const uint32_t u = r4 + x.x, v = r4 + y.x;
        d0[j] = min(u - t.Z4, u) + x.y;
        d1[j] = min(v - t.Z4, v) + y.y;
    }
    uint32_t L0[DC], L1[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(L0[j]) : "r"(d0[j] + bp));
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(L1[j]) : "r"(d1[j] + bp));
    }
    if (ES) synd |= atom_row_parity<DC>(L0) | atom_row_parity<DC>(L1);
#pragma unroll
    for (int j = 0; j < DC; ++j) LDPC_CHECK(d0[j] < 4u * (uint32_t)a.N && d1[j] < 4u * (uint32_t)a.N);
    uint32_t q0[DC], q1[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        q0[j] = fadd32(L0[j], first_iter ? kAtomQ0 : c0[j], a.rk);
        q1[j] = fadd32(L1[j], first_iter ? kAtomQ0 : c1[j], a.rk);
    }
    uint32_t rn0[DC], rn1[DC];
    RowState st;
    new_state<DC, true, VM>(q0, vk, st, rn0, a.rk);
    new_state<DC, true, VM>(q1, vk, st, rn1, a.rk);
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(d0[j] + ba), "r"(rn0[j]) : "memory");
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(d1[j] + ba), "r"(rn1[j]) : "memory");
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(c0[j]) : "r"(rn0[j]), "r"(a.rk.m1), "r"(kAtomQ0 + 0x8000u));
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(c1[j]) : "r"(rn1[j]), "r"(a.rk.m1), "r"(kAtomQ0 + 0x8000u));
    }
}

template <int DC, bool ES, int FMT, int VM, int FP = -1>
__device__ __forceinline__ int atom_qc_run(int b, int bend, int g, const ResArgs &a, const QcTab &t, const VarK &vk, uint32_t tw,
                                           int nb, int rloc, uint32_t r4, uint32_t bp, uint32_t ba, bool first_iter,
                                           uint32_t &synd, uint32_t tabs = 0) {
    if constexpr (DC == 0) {
        return bend;
    } else if constexpr (FMT == FMT_FULL) {
        // slot b's DC message words start at column t.tcol[b][g] of this group's range
#if !defined(LDPC_FULL_X1)
#pragma unroll 1
        for (; b + 1 < bend; b += 2) {
            uint32_t c0[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u}, c1[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            const uint32_t col0 = tw + (uint32_t)t.tcol[b][g], col1 = tw + (uint32_t)t.tcol[b + 1][g];
            if (!first_iter) {
                full_tmem_load<DC>(col0, c0);
                full_tmem_load<DC>(col1, c1);
            }
            if (rloc < a.Z)
                atom_row_full_x2<DC, ES, VM>(a, t, vk, bp, ba, t.e0[b][g], t.e0[b + 1][g], r4, first_iter, c0, c1, synd);
            full_tmem_store<DC>(col0, c0);
            full_tmem_store<DC>(col1, c1);
        }
#endif
#pragma unroll 1
        for (; b < bend; ++b) {
            uint32_t c[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            const uint32_t col = tw + (uint32_t)t.tcol[b][g];
            if (!first_iter) full_tmem_load<DC>(col, c);
            if (rloc < a.Z) atom_row_full<DC, true, ES, VM>(a, t, vk, bp, ba, t.e0[b][g], r4, 0, first_iter, c, synd);
            full_tmem_store<DC>(col, c);
        }
        return b;
    } else {
#pragma unroll 1
        for (; b < bend; ++b) {
            RowState st = {0u, 0u, 0u};
            LDPC_CHECK(b < nb && (uint32_t)((FMT == FMT_C16 ? 3 : 2) * nb) <= (uint32_t)a.cols_per_group);
            if (!first_iter) state_tmem_load<FMT, true>(tw, b, nb, st);
            if (rloc < a.Z) atom_row<DC, true, ES, VM, FMT, false, FP>(a, t, vk, bp, ba, t.e0[b][g], r4, 0, first_iter, st, synd, tabs);
            state_tmem_store<FMT>(tw, b, nb, st);
        }
        return b;
    }
}

template <bool ES, int FMT, int VM, int FP = -1>
__device__ __forceinline__ int atom_qc_dispatch(int dc, int b, int bend, int g, const ResArgs &a, const QcTab &t,
                                                const VarK &vk, uint32_t tw, int nb, int rloc, uint32_t r4, uint32_t bp, uint32_t ba,
                                                bool first_iter, uint32_t &synd, uint32_t tabs = 0) {
    switch (dc) {
    case 2: return atom_qc_run<2, ES, FMT, VM, FP>(b, bend, g, a, t, vk, tw, nb, rloc, r4, bp, ba, first_iter, synd, tabs);
    case 3: return atom_qc_run<3, ES, FMT, VM, FP>(b, bend, g, a, t, vk, tw, nb, rloc, r4, bp, ba, first_iter, synd, tabs);
    case 4: return atom_qc_run<4, ES, FMT, VM, FP>(b, bend, g, a, t, vk, tw, nb, rloc, r4, bp, ba, first_iter, synd, tabs);
    case 5: return atom_qc_run<5, ES, FMT, VM, FP>(b, bend, g, a, t, vk, tw, nb, rloc, r4, bp, ba, first_iter, synd, tabs);
    case 6: return atom_qc_run<6, ES, FMT, VM, FP>(b, bend, g, a, t, vk, tw, nb, rloc, r4, bp, ba, first_iter, synd, tabs);
    case 7: return atom_qc_run<7, ES, FMT, VM, FP>(b, bend, g, a, t, vk, tw, nb, rloc, r4, bp, ba, first_iter, synd, tabs);
    case 8: return atom_qc_run<8, ES, FMT, VM, FP>(b, bend, g, a, t, vk, tw, nb, rloc, r4, bp, ba, first_iter, synd, tabs);
    default: return atom_qc_run<0, ES, FMT, VM, FP>(b, bend, g, a, t, vk, tw, nb, rloc, r4, bp, ba, first_iter, synd, tabs);
    }
}

template <bool ES, int VM, int FMT, bool CSM, int FP = -1>
__device__ __forceinline__ void atom_csr_dispatch(int dc, const ResArgs &a, const QcTab &t, const VarK &vk, uint32_t bp, uint32_t ba,
                                                  int p, bool first_iter, RowState &st, uint32_t &synd, uint32_t sct) {
    switch (dc) {
    case 2: atom_row<2, false, ES, VM, FMT, CSM, FP>(a, t, vk, bp, ba, 0, 0, p, first_iter, st, synd, sct); break;
    case 3: atom_row<3, false, ES, VM, FMT, CSM, FP>(a, t, vk, bp, ba, 0, 0, p, first_iter, st, synd, sct); break;
    case 4: atom_row<4, false, ES, VM, FMT, CSM, FP>(a, t, vk, bp, ba, 0, 0, p, first_iter, st, synd, sct); break;
    case 5: atom_row<5, false, ES, VM, FMT, CSM, FP>(a, t, vk, bp, ba, 0, 0, p, first_iter, st, synd, sct); break;
    case 6: atom_row<6, false, ES, VM, FMT, CSM, FP>(a, t, vk, bp, ba, 0, 0, p, first_iter, st, synd, sct); break;
    case 7: atom_row<7, false, ES, VM, FMT, CSM, FP>(a, t, vk, bp, ba, 0, 0, p, first_iter, st, synd, sct); break;
    case 8: atom_row<8, false, ES, VM, FMT, CSM, FP>(a, t, vk, bp, ba, 0, 0, p, first_iter, st, synd, sct); break;
    }
}

template <bool ES, int VM>
__device__ __forceinline__ void atom_csr_dispatch_full(int dc, const ResArgs &a, const QcTab &t, const VarK &vk,
                                                       uint32_t bp, uint32_t ba, int p, bool first_iter,
                                                       uint32_t (&c)[8], uint32_t &synd) {
    switch (dc) {
    case 2: atom_row_full<2, false, ES, VM>(a, t, vk, bp, ba, 0, 0, p, first_iter, c, synd); break;
    case 3: atom_row_full<3, false, ES, VM>(a, t, vk, bp, ba, 0, 0, p, first_iter, c, synd); break;
    case 4: atom_row_full<4, false, ES, VM>(a, t, vk, bp, ba, 0, 0, p, first_iter, c, synd); break;
    case 5: atom_row_full<5, false, ES, VM>(a, t, vk, bp, ba, 0, 0, p, first_iter, c, synd); break;
    case 6: atom_row_full<6, false, ES, VM>(a, t, vk, bp, ba, 0, 0, p, first_iter, c, synd); break;
    case 7: atom_row_full<7, false, ES, VM>(a, t, vk, bp, ba, 0, 0, p, first_iter, c, synd); break;
    case 8: atom_row_full<8, false, ES, VM>(a, t, vk, bp, ba, 0, 0, p, first_iter, c, synd); break;
    }
}

// Ingest one frame pair: saturate to +-Q, double, bias, pack; write the Z^(0) slot (the
// accumulator start, restored by the TMA restarts) and both shared buffers.  Four variables per thread per step with
// all eight loads issued first (the loads are latency-bound, not bandwidth-bound).
template <typename TIN>
__device__ __forceinline__ void atom_ingest(const ResArgs &a, const TIN *__restrict__ lo, const TIN *__restrict__ hi,
                                            uint32_t *z0w, uint32_t *buf0, uint32_t *buf1) {
    const int tid = threadIdx.x, nth = blockDim.x;
    constexpr int U = 4;
    for (int n0 = tid; n0 < a.Np; n0 += U * nth) {
        int zl[U], zh[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int n = n0 + u * nth;
            zl[u] = n < a.N ? (int)__ldg(lo + n) : 0;
            zh[u] = (n < a.N && hi) ? (int)__ldg(hi + n) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int n = n0 + u * nth;
            if (n < a.Np) {
                const int l = max(-a.Qsat, min(a.Qsat, zl[u])), h = max(-a.Qsat, min(a.Qsat, zh[u]));
                const uint32_t v = pack2(2 * l + kAtomBias, 2 * h + kAtomBias);
                // accumulator start: every one of the dv_n messages arrives as V(L) + 0x8000
                // (new_state<B8>), so start dv_n * 0x8000 lower (exact 32-bit arithmetic)
                const uint32_t dv = n < a.N ? (uint32_t)__ldg(a.coldeg + n) : 0u;
                const uint32_t acc = v - dv * 0x8000u;
                __stcg(z0w + n, acc);
                buf0[n] = v;
                buf1[n] = acc;
            }
        }
    }
}

// ---------------------------------------------------------------- message export
// Exit messages of one row for both frames of the pair, rebuilt from the persistent state
// exactly as the next iteration would rebuild them:
// L_mn = s_mn f(A_m, B_m, n, ñ_m), doubled values halved; written in CSR edge order.
__device__ __forceinline__ void export_row_compact(const ResArgs &a, int m, int dc, const RowState &st, int f0,
                                                   bool hi_valid) {
    const int64_t e0 = __ldg(a.row_ptr + m);
    for (int j = 0; j < dc; ++j) {
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) {
            if (fr == 1 && !hi_valid) break;
            const uint32_t wb = st.W >> (16 * fr);             // W layout: rowcore.cuh header
            const bool neg = (wb >> j) & 1u, isidx = (wb >> (8 + j)) & 1u;
            const int mag = (int)(((isidx ? st.B : st.A) >> (16 * fr)) & 0xFFFFu);   // doubled magnitude
            a.msg_out[(size_t)(f0 + fr) * a.E + e0 + j] = (int16_t)((neg ? -mag : mag) / 2);
        }
    }
}
// FMT_FULL: the stored word c = kAtomQ0 - V(2 L_mn) of each edge
__device__ __forceinline__ void export_row_full(const ResArgs &a, int m, int dc, const uint32_t (&c)[8], int f0,
                                                bool hi_valid) {
    const int64_t e0 = __ldg(a.row_ptr + m);
    for (int j = 0; j < dc; ++j) {
        const uint32_t v = kAtomQ0 - c[j];                    // V form hi * 65536 + lo
        const int lo = (int)(int16_t)(v & 0xFFFFu), hi = (int)((int32_t)(v - (uint32_t)lo) >> 16);
        a.msg_out[(size_t)f0 * a.E + e0 + j] = (int16_t)(lo / 2);
        if (hi_valid) a.msg_out[(size_t)(f0 + 1) * a.E + e0 + j] = (int16_t)(hi / 2);
    }
}
// all rows of this thread (TMEM loads are warp-collective: issued whenever the slot exists
// for the warp, results used only by threads that own a row)
template <bool QC, int FMT>
__device__ __forceinline__ void atom_export(const ResArgs &a, const QcTab &t, uint32_t tw, int nb, int grp, int rloc,
                                            int f0, bool hi_valid) {
    const int tid = threadIdx.x, nth = blockDim.x;
    tmem_wait_st();
    for (int b = 0; b < nb; ++b) {
        int m = -1, dc;
        if (QC) {
            dc = t.dc[b][grp];
            if (dc == 0) continue;                              // uniform over the group
            if (rloc < a.Z) m = t.brow[b][grp] * a.Z + rloc;
        } else {
            const int p = b * nth + tid;
            dc = p < a.M ? a.dcT[p] : 0;
            if (p < a.M) m = p;
        }
        if constexpr (FMT == FMT_FULL) {
            uint32_t c[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            const uint32_t col = QC ? tw + (uint32_t)t.tcol[b][grp] : tw + 8u * b;
            const int ncol = QC ? dc : 8;
#pragma unroll
            for (int j = 0; j < 8; ++j)                         // constant indices: c stays in registers
                if (j < ncol) tmem_ld1(col + j, c[j]);
            tmem_wait_ld_dep8(c);
            if (m >= 0) export_row_full(a, m, dc, c, f0, hi_valid);
        } else {
            RowState st;
            state_tmem_load<FMT>(tw, b, nb, st);
            if (m >= 0) export_row_compact(a, m, dc, st, f0, hi_valid);
        }
    }
}

template <bool QC, bool ES, int FMT, typename TIN>
__global__ void __launch_bounds__(256, FMT == FMT_FULL ? 2 : 3) k_resident_atom(const __grid_constant__ ResArgs a,
                                                          const __grid_constant__ QcTab t) {
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t zbar;
    constexpr bool FIXK = ES && FMT != FMT_FULL;   // kernels with the fixed-base row scans
    const bool fix = FIXK && a.fixed_bases;
    uint32_t *buf0 = smem, *buf1 = smem + (fix ? kAtomFixOff / 4 : (uint32_t)a.Np);
    const int tid = threadIdx.x, nth = blockDim.x;
    const int grp = QC ? (a.group_threads == 128 ? (tid >> 7) : 0) : 0;
    const int rloc = QC ? tid - grp * a.group_threads : tid;
    const uint32_t r4 = 4u * (uint32_t)rloc;
    const int nb = QC ? t.nsb : a.nbatch;                // row slots per thread
    if (tid == 0) mbar_init(&zbar, 1);
    if (FMT == FMT_1BIT) idx_tab_fill();                          // state_tmem_load<FMT, true>
    const uint32_t tbase = tmem_alloc_cta(&tslot, a.tmem_cols);   // includes a block barrier
    const uint32_t tw = tmem_warp_base(tbase) + (uint32_t)((tid >> 7) * a.cols_per_group);
    uint32_t *z0w = a.ws + (size_t)blockIdx.x * a.slot_words;
    const TIN *llr = (const TIN *)a.llr;
    const uint32_t zbytes = 4u * (uint32_t)a.Np;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(buf0), s1 = (uint32_t)__cvta_generic_to_shared(buf1);
    uint32_t zphase = 0;
    // general codes: stage the [dc][M] column table after the posterior buffers (planner:
    // ResArgs::csr_smem when it fits without costing occupancy); visible after the first
    // barrier of the pair loop
    // fixed bases: the shift / column table after buffer 1 (8-byte aligned), offsets + base of buffer 0
    const uint32_t tabw = (kAtomFixOff / 4 + (uint32_t)a.Np + 1u) & ~1u;
    const uint32_t tabs = s0 + 4u * tabw;
    const uint32_t sct = fix ? tabs : s0 + 8u * (uint32_t)a.Np;
    if (!QC && a.csr_smem) {
        const uint32_t w0 = fix ? tabw : 2u * (uint32_t)a.Np, add = fix ? s0 : 0u;
        for (int i = tid; i < a.csr_dc * a.M; i += nth) smem[w0 + i] = __ldg(a.colT + i) + add;
    }
    if (QC && fix)
        for (int i = tid; i < t.nent; i += nth) {
            smem[tabw + 2 * i] = t.ent[i].x;
            smem[tabw + 2 * i + 1] = t.ent[i].y + s0;
        }

    for (int pair = blockIdx.x; pair < a.npairs; pair += gridDim.x) {
        const int f0 = 2 * pair, f1 = f0 + 1;
        const bool hi_valid = f1 < a.nframes;
        __syncthreads();                             // previous pair's outputs read the buffers
        atom_ingest<TIN>(a, llr + (size_t)f0 * a.N, hi_valid ? llr + (size_t)f1 * a.N : nullptr, z0w, buf0, buf1);
        fence_proxy_async_all();                     // z0w (generic writes) is later read by TMA
        __syncthreads();
        int done = hi_valid ? 0 : 2;
        bool finished = false;
        for (int k = 1; k <= a.K; ++k) {
            const uint32_t bp = (k & 1) ? s0 : s1, ba = (k & 1) ? s1 : s0;   // Z^(k-1) | Z^(k)
            if (k > 1) { mbar_wait(&zbar, zphase); zphase ^= 1; }          // Z^(k) = Z^(0) landed
            uint32_t synd = 0;
            const bool first_iter = (k == 1);
            const VarK vk = a.nsched ? a.vk_sched[k - 1] : a.vk;   // lambda_k / beta_k
            // one scan over this thread's rows; the check-node variant (offset / normalized)
            // is fixed per iteration, so it is a template parameter of the row code
            auto scan = [&](auto vm_tag, auto fi_tag, auto cs_tag, auto fp_tag) __attribute__((always_inline)) {
                constexpr int VM = decltype(vm_tag)::value;
                constexpr bool FI = decltype(fi_tag)::value;   // first iteration: no rebuild, no state load
                constexpr bool CSM = decltype(cs_tag)::value;  // general codes: column table in shared memory
                constexpr int FP = decltype(fp_tag)::value;    // fixed bases: iteration parity (-1: off)
                if (QC) {
#pragma unroll 1
                    for (int b = 0; b < nb;) {
                        if (grp == 0) b = atom_qc_dispatch<ES, FMT, VM, FP>(t.dc[b][0], b, t.run_end[b][0], 0, a, t, vk, tw, nb, rloc, r4, bp, ba, FI, synd, tabs);
                        else b = atom_qc_dispatch<ES, FMT, VM, FP>(t.dc[b][1], b, t.run_end[b][1], 1, a, t, vk, tw, nb, rloc, r4, bp, ba, FI, synd, tabs);
                    }
                } else if (FMT != FMT_FULL && a.dc_uniform) {
                    // row-regular code (e.g. config 1's (3,6)-regular H): one dispatch on the
                    // degree per iteration instead of a switch in every row
                    auto rows = [&](auto dc_tag) {
                        constexpr int DC = decltype(dc_tag)::value;
#pragma unroll 1
                        for (int b = 0; b < nb; ++b) {
                            const int p = b * nth + tid;
                            RowState st = {0u, 0u, 0u};
                            if (!FI) state_tmem_load<FMT, true>(tw, b, nb, st);
                            if (p < a.M)
                                atom_row<DC, false, ES, VM, FMT, CSM, (CSM ? FP : -1)>(a, t, vk, bp, ba, 0, 0, p, FI, st, synd, sct);
                            state_tmem_store<FMT>(tw, b, nb, st);
                        }
                    };
                    switch (a.dc_uniform) {
                    case 2: rows(std::integral_constant<int, 2>{}); break;
                    case 3: rows(std::integral_constant<int, 3>{}); break;
                    case 4: rows(std::integral_constant<int, 4>{}); break;
                    case 5: rows(std::integral_constant<int, 5>{}); break;
                    case 6: rows(std::integral_constant<int, 6>{}); break;
                    case 7: rows(std::integral_constant<int, 7>{}); break;
                    case 8: rows(std::integral_constant<int, 8>{}); break;
                    }
                } else {
#pragma unroll 1
                    for (int b = 0; b < nb; ++b) {
                        const int p = b * nth + tid;
                        if constexpr (FMT == FMT_FULL) {
                            // rows of one slot differ in degree across the warp: 8 columns per slot
                            uint32_t c[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                            if (!FI) full_tmem_load<8>(tw + 8u * b, c);
                            if (p < a.M) atom_csr_dispatch_full<ES, VM>(a.dcT[p], a, t, vk, bp, ba, p, FI, c, synd);
                            full_tmem_store<8>(tw + 8u * b, c);
                        } else {
                            RowState st = {0u, 0u, 0u};
                            if (!FI) state_tmem_load<FMT, true>(tw, b, nb, st);
                            if (p < a.M) atom_csr_dispatch<ES, VM, FMT, CSM, (CSM ? FP : -1)>(a.dcT[p], a, t, vk, bp, ba, p, FI, st, synd, sct);
                            state_tmem_store<FMT>(tw, b, nb, st);
                        }
                    }
                }
            };
            using F1 = std::integral_constant<bool, true>;
            using F0 = std::integral_constant<bool, false>;
            using PN = std::integral_constant<int, -1>;
            // fixed bases: parity 0 = odd k reads buffer 0 and accumulates into buffer 1
            using P0 = std::integral_constant<int, FIXK ? 0 : -1>;
            using P1 = std::integral_constant<int, FIXK ? 1 : -1>;
            auto run = [&](auto vm) __attribute__((always_inline)) {
                if (!QC && FMT != FMT_FULL && a.csr_smem) {
                    if (FIXK && fix) {
                        if (first_iter) scan(vm, F1{}, F1{}, P0{});
                        else if (k & 1) scan(vm, F0{}, F1{}, P0{});
                        else scan(vm, F0{}, F1{}, P1{});
                    } else {
                        if (first_iter) scan(vm, F1{}, F1{}, PN{});
                        else scan(vm, F0{}, F1{}, PN{});
                    }
                } else if (QC && FIXK && fix) {
                    if (first_iter) scan(vm, F1{}, F0{}, P0{});
                    else if (k & 1) scan(vm, F0{}, F0{}, P0{});
                    else scan(vm, F0{}, F0{}, P1{});
                } else {
                    if (first_iter) scan(vm, F1{}, F0{}, PN{});
                    else scan(vm, F0{}, F0{}, PN{});
                }
            };
            if (vk.norm) run(std::integral_constant<int, 1>{});
            else run(std::integral_constant<int, 0>{});
            tmem_wait_st();
            const char *Lpb = (const char *)((k & 1) ? buf0 : buf1);
            if (ES) {
                // syndrome of Z^(k-1), gathered during this scan (1-iteration lag); the
                // __syncthreads_or is also the end-of-iteration barrier
                const int fail_lo = __syncthreads_or((synd & kAtomSyndLo) != 0);
                const int fail_hi = __syncthreads_or((synd & kAtomSyndHi) != 0);
                const int newly = ((fail_lo ? 0 : 1) | (fail_hi ? 0 : 2)) & ~done;
                if (newly) {
                    res_write_outputs(a, (const uint32_t *)Lpb, f0, newly, k - 1, 0, 0, kAtomBias);
                    done |= newly;
                }
                if (done == 3) { finished = true; break; }
            }
            if (k < a.K) {
                // restart the next accumulator (the buffer just read) from Z^(0) by TMA
                fence_proxy_async_smem();
                __syncthreads();
                if (tid == 0) tma_bulk_g2s((void *)Lpb, z0w, zbytes, &zbar);
            }
        }
        if (!finished) {
            __syncthreads();                         // all atomics of iteration K landed
            const char *Lpb = (const char *)(((a.K + 1) & 1) ? buf0 : buf1);
            uint32_t synd = 0;
            if (QC) {
                for (int b = 0; b < nb; ++b) {
                    const int dc = t.dc[b][grp];
                    if (rloc < a.Z && dc) synd |= res_parity_dispatch<true>(dc, a, t, Lpb, t.e0[b][grp], r4, 0);
                }
            } else {
                for (int b = 0; b < nb; ++b) {
                    const int p = b * nth + tid;
                    if (p < a.M) synd |= res_parity_dispatch<false>(a.dcT[p], a, t, Lpb, 0, 0, p);
                }
            }
            const int fail_lo = __syncthreads_or((synd & 0x00008000u) != 0);
            const int fail_hi = __syncthreads_or((synd & 0x80000000u) != 0);
            const int which = 3 & ~done;
            if (which) res_write_outputs(a, (const uint32_t *)Lpb, f0, which, a.K, fail_lo, fail_hi, kAtomBias);
        }
        if (a.msg_out) atom_export<QC, FMT>(a, t, tw, nb, grp, rloc, f0, hi_valid);
    }
    tmem_free_cta(tbase, a.tmem_cols);
}

}  // namespace ldpc
