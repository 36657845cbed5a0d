// k_resident.cuh -- decode-resident single-scan min-sum kernel (integer LLRs).
//
// One CTA decodes one PAIR of frames (two 16-bit SIMD lanes per register) for
// all iterations without leaving the SM: the posterior double buffer
// Z^(k-1)_n / Z^(k)_n (reading D7) lives in shared memory
// (2 * N words), so gathers and the scatter-accumulate of Z^(k)_n += L^(k)_mn
// never touch HBM.  The compact state (A_m, B_m, ñ_m, s_mn) of every
// row is kept in this CTA's L2-resident workspace slot, and Z^(0) is copied
// once per frame pair into the slot.  The grid is persistent (CTAs loop over
// frame pairs), sized to fill all SMs.
//
// Rows are processed in conflict-free BATCHES: no two rows of a batch share a
// variable, so the accumulation into the shared-memory posterior needs no
// atomics; a barrier separates batches.  For quasi-cyclic codes a batch is one
// base row (Z circulant rows, thread r = circulant row r, the address of edge
// (i,j) is jZ + (r + s_ij) mod Z computed on the fly -- no index loads); for
// other codes the host builds batches by greedy row colouring and the column
// indices come from a [DC][M] transposed table (coalesced).
//
// The first batch touching a variable (host-marked "first" edge) initialises
// Z^(k)_n = Z^(0)_n + L^(k)_mn instead of accumulating (P:318 + P:322), so no
// separate initialisation pass or barrier is needed.
#pragma once
#include "rowcore.cuh"

namespace ldpc {

constexpr int kMaxDC = 8;

struct ResArgs {
    int N, M, npairs, nframes, K, Qsat, wpf;   // wpf = ceil(N/32) hard-bit words per frame
    uint32_t nbeta2, q2;
    const void *llr;
    uint32_t *hard_bits;
    int16_t *post;
    uint8_t *ok;
    int32_t *iters;
    uint32_t *ws;
    size_t slot_words;
    int nbatch;
    const int32_t *bptr;     // CSR: batch b = schedule positions [bptr[b], bptr[b+1])
    const int32_t *colT;     // CSR: [kMaxDC][M], bit 31 = first touch of the variable
    const uint8_t *dcT;      // CSR: degree per schedule position
    int Z;                   // QC circulant size
    const uint32_t *qent;    // QC: entries (colbase | shift << 16 | first << 31), grouped by base row
    const int32_t *qbptr;    // QC: base row b = entries [qbptr[b], qbptr[b+1])
    int nqent;
};

template <typename TIN>
__device__ __forceinline__ int load_llr_sat(const TIN *p, int Q) {
    int v = (int)p[0];
    return max(-Q, min(Q, v));
}

template <int DC, bool QC, bool ES, int FMT>
__device__ __forceinline__ void res_row(const ResArgs &a, const uint32_t *__restrict__ Lp, uint32_t *__restrict__ La,
                                        const uint32_t *__restrict__ z0w, uint32_t *stbase, int p, int r,
                                        const uint32_t *qe, bool first_iter, uint32_t &synd) {
    uint32_t off[DC];
    bool ft[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        if (QC) {
            const uint32_t e = qe[j];
            uint32_t x = (uint32_t)r + ((e >> 16) & 0x7FFFu);
            x = min(x, x - (uint32_t)a.Z);                   // (r + s) mod Z, r + s < 2Z
            off[j] = (e & 0xFFFFu) + x;
            ft[j] = (e >> 31) != 0;
        } else {
            const uint32_t c = (uint32_t)__ldg(a.colT + (size_t)j * a.M + p);
            off[j] = c & 0x7FFFFFFFu;
            ft[j] = (c >> 31) != 0;
        }
    }
    uint32_t z0v[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) z0v[j] = ft[j] ? __ldcg(z0w + off[j]) : 0u;
    uint32_t L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) L[j] = Lp[off[j]];
    if (ES) synd |= row_parity<DC>(L);
    uint32_t q[DC];
    RowState st;
    if (first_iter) {
#pragma unroll
        for (int j = 0; j < DC; ++j) q[j] = L[j];           // L^(0)_mn = 0
    } else {
        st = StateIO<FMT>::load(stbase, (size_t)a.M, (size_t)p);
        rebuild_q<DC>(L, st, q);
    }
    uint32_t rn[DC];
    new_state<DC>(q, a.nbeta2, a.q2, st, rn);
    StateIO<FMT>::store(stbase, (size_t)a.M, (size_t)p, st);
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        const uint32_t base = ft[j] ? z0v[j] : La[off[j]];
        La[off[j]] = vadd(base, rn[j]);                      // Z^(k)_n += L^(k)_mn
    }
}

template <int DC>
__device__ __forceinline__ uint32_t res_row_parity_qc(const ResArgs &a, const uint32_t *Lp, int r, const uint32_t *qe) {
    uint32_t L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        const uint32_t e = qe[j];
        uint32_t x = (uint32_t)r + ((e >> 16) & 0x7FFFu);
        x = min(x, x - (uint32_t)a.Z);
        L[j] = Lp[(e & 0xFFFFu) + x];
    }
    return row_parity<DC>(L);
}

template <int DC>
__device__ __forceinline__ uint32_t res_row_parity_csr(const ResArgs &a, const uint32_t *Lp, int p) {
    uint32_t L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) L[j] = Lp[(uint32_t)__ldg(a.colT + (size_t)j * a.M + p) & 0x7FFFFFFFu];
    return row_parity<DC>(L);
}

// Write outputs of the frames selected by `which` (bit0 = lo frame, bit1 = hi frame)
// from the doubled posterior buffer Lsrc.
__device__ void res_write_outputs(const ResArgs &a, const uint32_t *Lsrc, int f0, int which, int iters,
                                  int fail_lo, int fail_hi) {
    const int f1 = f0 + 1;
    const int tid = threadIdx.x, nth = blockDim.x;
    if (a.post) {
        for (int n = tid; n < a.N; n += nth) {
            const uint32_t v = Lsrc[n];
            if (which & 1) a.post[(size_t)f0 * a.N + n] = (int16_t)(lo16(v) >> 1);
            if (which & 2) a.post[(size_t)f1 * a.N + n] = (int16_t)(hi16(v) >> 1);
        }
    }
    const int lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
    for (int w = warp; w < a.wpf; w += nw) {
        const int n = w * 32 + lane;
        const uint32_t v = n < a.N ? Lsrc[n] : 0x00020002u;
        const uint32_t blo = __ballot_sync(0xFFFFFFFFu, lo16(v) <= 0);
        const uint32_t bhi = __ballot_sync(0xFFFFFFFFu, hi16(v) <= 0);
        if (lane == 0) {
            if (which & 1) a.hard_bits[(size_t)f0 * a.wpf + w] = blo;
            if (which & 2) a.hard_bits[(size_t)f1 * a.wpf + w] = bhi;
        }
    }
    if (tid == 0) {
        if (which & 1) { a.ok[f0] = (uint8_t)!fail_lo; if (a.iters) a.iters[f0] = iters; }
        if (which & 2) { a.ok[f1] = (uint8_t)!fail_hi; if (a.iters) a.iters[f1] = iters; }
    }
}

template <bool QC, bool ES, int FMT, typename TIN>
__global__ void __launch_bounds__(256) k_resident(const ResArgs a) {
    extern __shared__ uint32_t smem[];
    uint32_t *buf0 = smem, *buf1 = smem + a.N;
    uint32_t *qtab = smem + 2 * a.N;                 // QC: entries, then base-row pointers
    int32_t *qbp = (int32_t *)(qtab + a.nqent);
    const int tid = threadIdx.x;
    if (QC) {
        for (int i = tid; i < a.nqent; i += blockDim.x) qtab[i] = a.qent[i];
        for (int i = tid; i <= a.nbatch; i += blockDim.x) qbp[i] = a.qbptr[i];
    }
    uint32_t *slot = a.ws + (size_t)blockIdx.x * a.slot_words;
    uint32_t *z0w = slot;
    uint32_t *stbase = slot + a.N;
    const TIN *llr = (const TIN *)a.llr;

    for (int pair = blockIdx.x; pair < a.npairs; pair += gridDim.x) {
        const int f0 = 2 * pair, f1 = f0 + 1;
        const bool hi_valid = f1 < a.nframes;
        __syncthreads();                             // previous pair's outputs read the buffers
        // ingest: saturate to +-Q, double, pack the pair; Z^(0) -> slot and Z^(k-1) buffer
        for (int n = tid; n < a.N; n += blockDim.x) {
            const int zl = load_llr_sat(llr + (size_t)f0 * a.N + n, a.Qsat);
            const int zh = hi_valid ? load_llr_sat(llr + (size_t)f1 * a.N + n, a.Qsat) : 0;
            const uint32_t v = pack2(2 * zl, 2 * zh);
            __stcg(z0w + n, v);
            buf0[n] = v;
        }
        __syncthreads();
        uint32_t *Lp = buf0, *La = buf1;
        int done = hi_valid ? 0 : 2;
        bool finished = false;
        for (int k = 1; k <= a.K; ++k) {
            uint32_t synd = 0;
            const bool first_iter = (k == 1);
            for (int b = 0; b < a.nbatch; ++b) {
                if (QC) {
                    const int e0 = qbp[b], dc = qbp[b + 1] - e0;
                    const int r = tid;
                    if (r < a.Z) {
                        const uint32_t *qe = qtab + e0;
                        const int p = b * a.Z + r;
                        switch (dc) {
                        case 2: res_row<2, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, r, qe, first_iter, synd); break;
                        case 3: res_row<3, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, r, qe, first_iter, synd); break;
                        case 4: res_row<4, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, r, qe, first_iter, synd); break;
                        case 5: res_row<5, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, r, qe, first_iter, synd); break;
                        case 6: res_row<6, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, r, qe, first_iter, synd); break;
                        case 7: res_row<7, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, r, qe, first_iter, synd); break;
                        case 8: res_row<8, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, r, qe, first_iter, synd); break;
                        }
                    }
                } else {
                    const int p = a.bptr[b] + tid;
                    if (p < a.bptr[b + 1]) {
                        const int dc = a.dcT[p];
                        switch (dc) {
                        case 2: res_row<2, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, 0, nullptr, first_iter, synd); break;
                        case 3: res_row<3, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, 0, nullptr, first_iter, synd); break;
                        case 4: res_row<4, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, 0, nullptr, first_iter, synd); break;
                        case 5: res_row<5, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, 0, nullptr, first_iter, synd); break;
                        case 6: res_row<6, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, 0, nullptr, first_iter, synd); break;
                        case 7: res_row<7, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, 0, nullptr, first_iter, synd); break;
                        case 8: res_row<8, QC, ES, FMT>(a, Lp, La, z0w, stbase, p, 0, nullptr, first_iter, synd); break;
                        }
                    }
                }
                __syncthreads();                     // batch b's accumulations complete
            }
            if (ES) {
                // syndrome of Z^(k-1) (computed during this scan's gathers; 1-iteration lag)
                const int fail_lo = __syncthreads_or((synd & 0x00008000u) != 0);
                const int fail_hi = __syncthreads_or((synd & 0x80000000u) != 0);
                const int conv = (fail_lo ? 0 : 1) | (fail_hi ? 0 : 2);
                const int newly = conv & ~done;
                if (newly) {
                    res_write_outputs(a, Lp, f0, newly, k - 1, 0, 0);
                    done |= newly;
                }
                if (done == 3) { finished = true; break; }
            }
            uint32_t *t = Lp; Lp = La; La = t;       // Z^(k) becomes the read buffer
        }
        if (!finished) {
            // final syndrome of Z^(K)
            uint32_t synd = 0;
            for (int b = 0; b < a.nbatch; ++b) {
                if (QC) {
                    const int e0 = qbp[b], dc = qbp[b + 1] - e0;
                    if (tid < a.Z) {
                        const uint32_t *qe = qtab + e0;
                        switch (dc) {
                        case 2: synd |= res_row_parity_qc<2>(a, Lp, tid, qe); break;
                        case 3: synd |= res_row_parity_qc<3>(a, Lp, tid, qe); break;
                        case 4: synd |= res_row_parity_qc<4>(a, Lp, tid, qe); break;
                        case 5: synd |= res_row_parity_qc<5>(a, Lp, tid, qe); break;
                        case 6: synd |= res_row_parity_qc<6>(a, Lp, tid, qe); break;
                        case 7: synd |= res_row_parity_qc<7>(a, Lp, tid, qe); break;
                        case 8: synd |= res_row_parity_qc<8>(a, Lp, tid, qe); break;
                        }
                    }
                } else {
                    const int p = a.bptr[b] + tid;
                    if (p < a.bptr[b + 1]) {
                        switch (a.dcT[p]) {
                        case 2: synd |= res_row_parity_csr<2>(a, Lp, p); break;
                        case 3: synd |= res_row_parity_csr<3>(a, Lp, p); break;
                        case 4: synd |= res_row_parity_csr<4>(a, Lp, p); break;
                        case 5: synd |= res_row_parity_csr<5>(a, Lp, p); break;
                        case 6: synd |= res_row_parity_csr<6>(a, Lp, p); break;
                        case 7: synd |= res_row_parity_csr<7>(a, Lp, p); break;
                        case 8: synd |= res_row_parity_csr<8>(a, Lp, p); break;
                        }
                    }
                }
            }
            const int fail_lo = __syncthreads_or((synd & 0x00008000u) != 0);
            const int fail_hi = __syncthreads_or((synd & 0x80000000u) != 0);
            const int which = 3 & ~done;
            if (which) res_write_outputs(a, Lp, f0, which, a.K, fail_lo, fail_hi);
        }
    }
}

}  // namespace ldpc
