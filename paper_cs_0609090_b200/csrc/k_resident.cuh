// k_resident.cuh -- decode-resident single-scan min-sum kernel (integer LLRs).
//
// One CTA decodes one PAIR of frames (two 16-bit SIMD lanes per register) for
// all iterations without leaving the SM:
//   * the posterior double buffer Z^(k-1)_n / Z^(k)_n (
//     reading D7) lives in shared memory (2 * N words), so the gathers and the
//     scatter-accumulate Z^(k)_n += L^(k)_mn never touch L2/HBM;
//   * the compact state (A_m, B_m, ñ_m, s_mn) of every check row -- the paper's
//     "persistent data" -- lives in Tensor Memory: the thread that owns
//     a row keeps its state in its own TMEM lane (tcgen05.ld / tcgen05.st);
//   * Z^(0)_n is packed once per frame pair into this CTA's L2-resident
//     workspace slot; each iteration restarts the accumulator from it with one
//     TMA bulk copy (cp.async.bulk + mbarrier; "Z^(k)_n = Z^(0)_n").
// The grid is persistent: CTAs loop over frame pairs, sized to fill all SMs.
//
// Rows are processed in conflict-free BATCHES: no two rows of a batch share a
// variable, so the shared-memory accumulation needs no atomics; a barrier
// separates batches.  Quasi-cyclic codes: a batch ("super-batch") is one or two
// base rows with disjoint column blocks, one 128-thread group per base row,
// thread r = circulant row r; edge (i,j) addresses variable jZ + (r + s_ij) mod Z
// from the shift table held in the constant bank (no index loads).  Other
// codes: the host builds batches by greedy row colouring and per-edge byte
// offsets come from a [DC][M] table.
#pragma once
#include <type_traits>
#include "args.cuh"
#include "rowcore.cuh"
#include "tmem.cuh"

namespace ldpc {

template <typename TIN>
__device__ __forceinline__ int load_llr_sat(const TIN *p, int Q) {
    int v = (int)p[0];
    return max(-Q, min(Q, v));
}

// ------------------------------------------------------------ mbarrier / TMA
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one thread: expect `bytes` and start a bulk global->shared copy completing on the barrier
__device__ __forceinline__ void tma_bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes, uint64_t *bar) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst_smem);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src_gmem), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(b), "r"(phase) : "memory");
    }
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }

// ------------------------------------------------------------ one check row
// LAY = false: flooding (Z^(k-1) read from Lpb, Z^(k) accumulated in Lab).
// LAY = true : layered / in-place (reading D25): one array, Z_n <- (Z_n - L_old) + L_new.
template <int DC, bool QC, bool ES, bool LAY, int FMT>
__device__ __forceinline__ void res_row(const ResArgs &a, const QcTab &t, const VarK &vk, const char *Lpb, char *Lab,
                                        int e0, uint32_t r4, int p, bool first_iter, RowState &st, uint32_t &synd) {
    // shared-memory byte addresses of the row's variables in both buffers:
    // 4 * (jZ + (r + s) mod Z) + base, one VIADDMNMX for the modulo and one IADD3 per buffer
    const uint32_t bp = (uint32_t)__cvta_generic_to_shared(Lpb), ba = (uint32_t)__cvta_generic_to_shared(Lab);
    uint32_t op[DC], oa[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        uint32_t d, cb;
        if (QC) {
            const uint2 e = t.ent[e0 + j];
            const uint32_t u = r4 + e.x;
            d = min(u - t.Z4, u);
            cb = e.y;
        } else {
            d = __ldg(a.colT + (size_t)j * a.M + p);
            cb = 0u;
        }
        op[j] = d + cb + bp;
        oa[j] = d + cb + ba;
    }
    uint32_t L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        LDPC_CHECK(op[j] - bp < 4u * (uint32_t)a.N && oa[j] - ba < 4u * (uint32_t)a.N);
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(L[j]) : "r"(op[j]));
    }
    if (ES) synd |= row_parity<DC>(L, a.rk);
    uint32_t q[DC];
    if (first_iter) {
#pragma unroll
        for (int j = 0; j < DC; ++j) q[j] = L[j];            // L^(0)_mn = 0
    } else {
        rebuild_q<DC>(L, st, q, a.rk);
    }
    uint32_t rn[DC];
    new_state<DC, false, -1, FMT == FMT_1BIT>(q, vk, st, rn, a.rk);
    if (LAY) {
#pragma unroll
        for (int j = 0; j < DC; ++j)                          // Z_n = (Z_n - L^(k-1)_mn) + L^(k)_mn
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(op[j]), "r"(vadd(q[j], rn[j])) : "memory");
    } else {
#pragma unroll
        for (int j = 0; j < DC; ++j) {                       // Z^(k)_n += L^(k)_mn
            uint32_t v;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(oa[j]) : "memory");
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(oa[j]), "r"(vadd(v, rn[j])) : "memory");
        }
    }
}

template <bool QC, bool ES, bool LAY, int FMT>
__device__ __forceinline__ void res_dispatch(int dc, const ResArgs &a, const QcTab &t, const VarK &vk, const char *Lpb, char *Lab,
                                             int e0, uint32_t r4, int p, bool first_iter, RowState &st,
                                             uint32_t &synd) {
    switch (dc) {
    case 2: res_row<2, QC, ES, LAY, FMT>(a, t, vk, Lpb, Lab, e0, r4, p, first_iter, st, synd); break;
    case 3: res_row<3, QC, ES, LAY, FMT>(a, t, vk, Lpb, Lab, e0, r4, p, first_iter, st, synd); break;
    case 4: res_row<4, QC, ES, LAY, FMT>(a, t, vk, Lpb, Lab, e0, r4, p, first_iter, st, synd); break;
    case 5: res_row<5, QC, ES, LAY, FMT>(a, t, vk, Lpb, Lab, e0, r4, p, first_iter, st, synd); break;
    case 6: res_row<6, QC, ES, LAY, FMT>(a, t, vk, Lpb, Lab, e0, r4, p, first_iter, st, synd); break;
    case 7: res_row<7, QC, ES, LAY, FMT>(a, t, vk, Lpb, Lab, e0, r4, p, first_iter, st, synd); break;
    case 8: res_row<8, QC, ES, LAY, FMT>(a, t, vk, Lpb, Lab, e0, r4, p, first_iter, st, synd); break;
    }
}

template <int DC, bool QC>
__device__ __forceinline__ uint32_t res_parity(const ResArgs &a, const QcTab &t, const char *Lpb, int e0, uint32_t r4,
                                               int p) {
    uint32_t L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        uint32_t off;
        if (QC) {
            const uint2 e = t.ent[e0 + j];
            const uint32_t u = r4 + e.x;
            off = min(u - t.Z4, u) + e.y;
        } else {
            off = __ldg(a.colT + (size_t)j * a.M + p);
        }
        L[j] = *(const uint32_t *)(Lpb + off);
    }
    return row_parity<DC>(L, a.rk, a.cpar);
}

template <bool QC>
__device__ __forceinline__ uint32_t res_parity_dispatch(int dc, const ResArgs &a, const QcTab &t, const char *Lpb,
                                                        int e0, uint32_t r4, int p) {
    switch (dc) {
    case 2: return res_parity<2, QC>(a, t, Lpb, e0, r4, p);
    case 3: return res_parity<3, QC>(a, t, Lpb, e0, r4, p);
    case 4: return res_parity<4, QC>(a, t, Lpb, e0, r4, p);
    case 5: return res_parity<5, QC>(a, t, Lpb, e0, r4, p);
    case 6: return res_parity<6, QC>(a, t, Lpb, e0, r4, p);
    case 7: return res_parity<7, QC>(a, t, Lpb, e0, r4, p);
    case 8: return res_parity<8, QC>(a, t, Lpb, e0, r4, p);
    }
    return 0;
}

// Write outputs of the frames selected by `which` (bit0 = lo frame, bit1 = hi frame)
// from the doubled posterior buffer Lsrc (each 16-bit lane holds 2 Z_n + bias).
static __device__ void res_write_outputs(const ResArgs &a, const uint32_t *Lsrc, int f0, int which, int iters,
                                  int fail_lo, int fail_hi, int bias = 0) {
    const int f1 = f0 + 1;
    LDPC_CHECK(f0 < a.nframes && (!(which & 2) || f1 < a.nframes));
    const int tid = threadIdx.x, nth = blockDim.x;
    if (a.post) {
        for (int n = tid; n < a.N; n += nth) {
            const uint32_t v = Lsrc[n];
            if (which & 1) a.post[(size_t)f0 * a.N + n] = (int16_t)((lo16(v) - bias) >> 1);
            if (which & 2) a.post[(size_t)f1 * a.N + n] = (int16_t)((hi16(v) - bias) >> 1);
        }
    }
    // hard bits: a warp forms 32 consecutive words (one ballot each) and lane j stores word j,
    // so each frame's words leave as one 128-byte store instead of 32 scattered 4-byte ones
    const int lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
    for (int w0 = warp * 32; w0 < a.wpf; w0 += nw * 32) {
        uint32_t mlo = 0, mhi = 0;
        const int nwd = min(32, a.wpf - w0);
        for (int j = 0; j < nwd; ++j) {
            const int n = (w0 + j) * 32 + lane;
            const uint32_t v = n < a.N ? Lsrc[n] : pack2(bias + 2, bias + 2);
            const uint32_t blo = __ballot_sync(0xFFFFFFFFu, lo16(v) - bias <= 0);
            const uint32_t bhi = __ballot_sync(0xFFFFFFFFu, hi16(v) - bias <= 0);
            if (lane == j) {
                mlo = blo;
                mhi = bhi;
            }
        }
        if (lane < nwd) {
            if (which & 1) a.hard_bits[(size_t)f0 * a.wpf + w0 + lane] = mlo;
            if (which & 2) a.hard_bits[(size_t)f1 * a.wpf + w0 + lane] = mhi;
        }
    }
    if (tid == 0) {
        if (which & 1) { a.ok[f0] = (uint8_t)!fail_lo; if (a.iters) a.iters[f0] = iters; }
        if (which & 2) { a.ok[f1] = (uint8_t)!fail_hi; if (a.iters) a.iters[f1] = iters; }
    }
}

// TMEM columns of batch b for this thread: FMT_C16 uses (A,B) at 2b and W at 2*nb + b;
// FMT_1BIT uses (X, W) at 2b.
// Index-coded ñ (FMT_1BIT) -> per-edge flags with a shared-memory table instead of shifts
// (expand_idx): the byte offset of the lo frame's entry is 16 x the index nibble (W bits
// 8-11, 16-byte stride), the hi frame's entry (W bits 24-27) sits 256 bytes on.  A kernel
// that loads state with TAB = true fills the table first (idx_tab_fill, before its first
// barrier).
static __shared__ __align__(16) uint32_t g_idx_tab[128];
__device__ __forceinline__ void idx_tab_fill() {
    const int t = threadIdx.x;
    if (t < 32) g_idx_tab[4 * t] = t < 16 ? (0x100u << t) & 0x0000FF00u : (0x1000000u << (t - 16)) & 0xFF000000u;
}
__device__ __forceinline__ uint32_t expand_idx_tab(uint32_t W) {
    const uint32_t ol = *(const uint32_t *)((const char *)g_idx_tab + ((W >> 4) & 0xF0u));
    const uint32_t oh = *(const uint32_t *)((const char *)g_idx_tab + 256 + ((W >> 20) & 0xF0u));
    return (W & 0x00FF00FFu) | ol | oh;
}

template <int FMT, bool TAB = false>
__device__ __forceinline__ void state_tmem_load(uint32_t tw, int b, int nb, RowState &st) {
    if (FMT == FMT_C16) {
        tmem_ld2(tw + 2 * b, st.A, st.B);
        tmem_ld1(tw + 2 * nb + b, st.W);
        tmem_wait_ld_dep(st.A, st.B, st.W);
    } else {
        uint32_t X;
        tmem_ld2(tw + 2 * b, X, st.W);
        tmem_wait_ld_dep(X, st.W, st.W);
        st.A = prmt(X, 0u, 0x4240u);
        st.B = prmt(X, 0u, 0x4341u);
        st.W = TAB ? expand_idx_tab(st.W) : expand_idx(st.W);   // index-coded ñ (rowcore.cuh)
    }
}
template <int FMT>
__device__ __forceinline__ void state_tmem_store(uint32_t tw, int b, int nb, const RowState &st) {
    if (FMT == FMT_C16) {
        tmem_st2(tw + 2 * b, st.A, st.B);
        tmem_st1(tw + 2 * nb + b, st.W);
    } else {
        tmem_st2(tw + 2 * b, prmt(st.A, st.B, 0x6240u), st.W);
    }
}

// Consecutive super-batches in which this group's rows have the same degree DC are
// processed by one loop (one dispatch per run instead of per batch).
template <int DC, bool ES, int FMT, bool LAY>
__device__ __forceinline__ int qc_run(int b, int bend, int g, const ResArgs &a, const QcTab &t, const VarK &vk, uint32_t tw, int nb,
                                      int rloc, uint32_t r4, const char *Lpb, char *Lab, bool first_iter,
                                      uint32_t &synd) {
#pragma unroll 1
    for (; b < bend; ++b) {
        RowState st = {0u, 0u, 0u};
        if constexpr (DC > 0) {
            if (!first_iter) state_tmem_load<FMT>(tw, b, nb, st);
            if (rloc < a.Z) res_row<DC, true, ES, LAY, FMT>(a, t, vk, Lpb, Lab, t.e0[b][g], r4, 0, first_iter, st, synd);
            state_tmem_store<FMT>(tw, b, nb, st);
        }
        __syncthreads();                         // batch b's accumulations complete
    }
    return b;
}

template <bool ES, int FMT, bool LAY>
__device__ __forceinline__ int qc_run_dispatch(int dc, int b, int bend, int g, const ResArgs &a, const QcTab &t,
                                               const VarK &vk, uint32_t tw, int nb, int rloc, uint32_t r4, const char *Lpb, char *Lab,
                                               bool first_iter, uint32_t &synd) {
    switch (dc) {
    case 2: return qc_run<2, ES, FMT, LAY>(b, bend, g, a, t, vk, tw, nb, rloc, r4, Lpb, Lab, first_iter, synd);
    case 3: return qc_run<3, ES, FMT, LAY>(b, bend, g, a, t, vk, tw, nb, rloc, r4, Lpb, Lab, first_iter, synd);
    case 4: return qc_run<4, ES, FMT, LAY>(b, bend, g, a, t, vk, tw, nb, rloc, r4, Lpb, Lab, first_iter, synd);
    case 5: return qc_run<5, ES, FMT, LAY>(b, bend, g, a, t, vk, tw, nb, rloc, r4, Lpb, Lab, first_iter, synd);
    case 6: return qc_run<6, ES, FMT, LAY>(b, bend, g, a, t, vk, tw, nb, rloc, r4, Lpb, Lab, first_iter, synd);
    case 7: return qc_run<7, ES, FMT, LAY>(b, bend, g, a, t, vk, tw, nb, rloc, r4, Lpb, Lab, first_iter, synd);
    case 8: return qc_run<8, ES, FMT, LAY>(b, bend, g, a, t, vk, tw, nb, rloc, r4, Lpb, Lab, first_iter, synd);
    default: return qc_run<0, ES, FMT, LAY>(b, bend, g, a, t, vk, tw, nb, rloc, r4, Lpb, Lab, first_iter, synd);
    }
}

// Parity of every row of this thread against the posterior array Lpb (bit 15 / 31 set
// iff some row of the lo / hi frame is unsatisfied): H x̂ = 0 test of P:174.
template <bool QC>
__device__ __forceinline__ uint32_t parity_pass(const ResArgs &a, const QcTab &t, const char *Lpb, int nb, int grp,
                                                int rloc, uint32_t r4, int tid) {
    uint32_t synd = 0;
    for (int b = 0; b < nb; ++b) {
        if (QC) {
            const int dc = t.dc[b][grp];
            if (rloc < a.Z && dc) synd |= res_parity_dispatch<QC>(dc, a, t, Lpb, t.e0[b][grp], r4, 0);
        } else {
            const int p = a.bptr[b] + tid;
            if (p < a.bptr[b + 1]) synd |= res_parity_dispatch<QC>(a.dcT[p], a, t, Lpb, 0, 0, p);
        }
    }
    return synd;
}

// LAY = false: flooding schedule (the paper's Eq.(3) with Z^(k-1) / Z^(k) double
// buffer, reading D7).  LAY = true: layered schedule (one in-place posterior array,
// rows in ascending m, reading D25): the batches then hold consecutive variable-
// disjoint rows (QC: consecutive base rows), so processing a batch in parallel is the
// same as processing its rows one after the other.
template <bool QC, bool ES, int FMT, typename TIN, bool LAY>
__global__ void __launch_bounds__(256, 3) k_resident(const __grid_constant__ ResArgs a, const __grid_constant__ QcTab t) {
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t zbar;
    uint32_t *buf0 = smem, *buf1 = LAY ? smem : smem + a.Np;
    uint32_t *sst = smem + a.Np;                 // layered, non-QC: compact state [3][M] (see below)
    const int tid = threadIdx.x, nth = blockDim.x;
    const int grp = QC ? (a.group_threads == 128 ? (tid >> 7) : 0) : tid >> 7;
    const int rloc = QC ? tid - grp * a.group_threads : tid;
    const uint32_t r4 = 4u * (uint32_t)rloc;
    const int nb = QC ? t.nsb : a.nbatch;
    if (!LAY && tid == 0) mbar_init(&zbar, 1);
    const uint32_t tbase = tmem_alloc_cta(&tslot, a.tmem_cols);   // includes a block barrier
    // TMEM lanes are per warp quadrant (warp % 4): threads 128..255 use a second column range
    const uint32_t tw = tmem_warp_base(tbase) + (uint32_t)((tid >> 7) * a.cols_per_group);
    uint32_t *z0w = a.ws + (size_t)blockIdx.x * a.slot_words;
    const TIN *llr = (const TIN *)a.llr;
    const uint32_t zbytes = 4u * (uint32_t)a.Np;
    uint32_t zphase = 0;

    for (int pair = blockIdx.x; pair < a.npairs; pair += gridDim.x) {
        const int f0 = 2 * pair, f1 = f0 + 1;
        const bool hi_valid = f1 < a.nframes;
        __syncthreads();                             // previous pair's outputs read the buffers
        // ingest: saturate to +-Q, double, pack the pair; Z^(0) -> slot, Z^(0) buffer and
        // the first accumulator (layered: the one posterior array)
        for (int n = tid; n < a.Np; n += nth) {
            uint32_t v = 0;
            if (n < a.N) {
                const int zl = load_llr_sat(llr + (size_t)f0 * a.N + n, a.Qsat);
                const int zh = hi_valid ? load_llr_sat(llr + (size_t)f1 * a.N + n, a.Qsat) : 0;
                v = pack2(2 * zl, 2 * zh);
            }
            if (!LAY) {
                __stcg(z0w + n, v);
                buf1[n] = v;
            }
            buf0[n] = v;
        }
        if (!LAY) fence_proxy_async_all();           // z0w (generic writes) is later read by TMA
        __syncthreads();
        int done = hi_valid ? 0 : 2;
        bool finished = false;
        int k = 1;
        for (; k <= a.K; ++k) {
            // buffers by iteration parity: Z^(k-1) in Lp, Z^(k) accumulates in La (layered: same array)
            const char *Lpb = (const char *)(((k & 1) ? buf0 : buf1));
            char *Lab = (char *)(((k & 1) ? buf1 : buf0));
            if (!LAY && k > 1) { mbar_wait(&zbar, zphase); zphase ^= 1; }   // La = Z^(0) has landed
            uint32_t synd = 0;
            const bool first_iter = (k == 1);
            const VarK vk = a.nsched ? a.vk_sched[k - 1] : a.vk;   // lambda_k / beta_k
            if (LAY && ES) {
                // syndrome of the posterior after iteration k-1, before this iteration
                // changes it in place
                synd = parity_pass<QC>(a, t, Lpb, nb, grp, rloc, r4, tid);
                const int fail_lo = __syncthreads_or((synd & 0x00008000u) != 0);
                const int fail_hi = __syncthreads_or((synd & 0x80000000u) != 0);
                const int newly = ((fail_lo ? 0 : 1) | (fail_hi ? 0 : 2)) & ~done;
                if (newly) {
                    res_write_outputs(a, (const uint32_t *)Lpb, f0, newly, k - 1, 0, 0);
                    done |= newly;
                    __syncthreads();                 // outputs read the array before it changes
                }
                if (done == 3) { finished = true; break; }
            }
            constexpr bool RES = ES && !LAY;         // flooding: syndrome fused into the gather
            // the first iteration (no rebuild, no state load) is a compile-time variant of the scan
            auto scan = [&](auto fi_tag) {
                constexpr bool FI = decltype(fi_tag)::value;
                if (QC) {
                    // warp-uniform group branch: uniform table indices
#pragma unroll 1
                    for (int b = 0; b < nb;) {
                        if (grp == 0) b = qc_run_dispatch<RES, FMT, LAY>(t.dc[b][0], b, t.run_end[b][0], 0, a, t, vk, tw, nb, rloc, r4, Lpb, Lab, FI, synd);
                        else b = qc_run_dispatch<RES, FMT, LAY>(t.dc[b][1], b, t.run_end[b][1], 1, a, t, vk, tw, nb, rloc, r4, Lpb, Lab, FI, synd);
                    }
                } else {
#pragma unroll 1
                    for (int b = 0; b < nb; ++b) {
                        RowState st = {0u, 0u, 0u};
                        const int p = a.bptr[b] + tid;
                        const bool valid = p < a.bptr[b + 1];
                        if (LAY) {
                            // layered general codes: batches can be single rows (e.g. a staircase),
                            // so the state lives in shared memory indexed by row, [3][M] words
                            if (!FI && valid) {
                                st.A = sst[p];
                                st.B = sst[a.M + p];
                                st.W = FMT == FMT_1BIT ? expand_idx(sst[2 * a.M + p]) : sst[2 * a.M + p];
                            }
                        } else if (!FI) {
                            state_tmem_load<FMT>(tw, b, nb, st);
                        }
                        if (valid) res_dispatch<QC, RES, LAY, FMT>(a.dcT[p], a, t, vk, Lpb, Lab, 0, 0, p, FI, st, synd);
                        if (LAY) {
                            if (valid) { sst[p] = st.A; sst[a.M + p] = st.B; sst[2 * a.M + p] = st.W; }
                        } else {
                            state_tmem_store<FMT>(tw, b, nb, st);
                        }
                        __syncthreads();                     // batch b's accumulations complete
                    }
                }
            };
            if (first_iter) scan(std::integral_constant<bool, true>{});
            else scan(std::integral_constant<bool, false>{});
            tmem_wait_st();
            if (RES) {
                // syndrome of Z^(k-1), gathered during this scan (1-iteration lag)
                const int fail_lo = __syncthreads_or((synd & 0x00008000u) != 0);
                const int fail_hi = __syncthreads_or((synd & 0x80000000u) != 0);
                const int conv = (fail_lo ? 0 : 1) | (fail_hi ? 0 : 2);
                const int newly = conv & ~done;
                if (newly) {
                    res_write_outputs(a, (const uint32_t *)Lpb, f0, newly, k - 1, 0, 0);
                    done |= newly;
                }
                if (done == 3) { finished = true; break; }
            }
            if (!LAY && k < a.K) {
                // restart the next accumulator (the buffer just read) from Z^(0) by TMA
                fence_proxy_async_smem();
                __syncthreads();
                if (tid == 0) tma_bulk_g2s((void *)Lpb, z0w, zbytes, &zbar);
            }
        }
        if (!finished) {
            // final syndrome of Z^(K)
            const char *Lpb = (const char *)(((a.K + 1) & 1) ? buf0 : buf1);
            const uint32_t synd = parity_pass<QC>(a, t, Lpb, nb, grp, rloc, r4, tid);
            const int fail_lo = __syncthreads_or((synd & 0x00008000u) != 0);
            const int fail_hi = __syncthreads_or((synd & 0x80000000u) != 0);
            const int which = 3 & ~done;
            if (which) res_write_outputs(a, (const uint32_t *)Lpb, f0, which, a.K, fail_lo, fail_hi);
        }
    }
    tmem_free_cta(tbase, a.tmem_cols);
}

}  // namespace ldpc
