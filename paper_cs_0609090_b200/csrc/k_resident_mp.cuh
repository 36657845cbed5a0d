// k_resident_mp.cuh -- multi-pair decode-resident kernel for quasi-cyclic codes.
//
// Same algorithm and data placement as k_resident (posterior double buffers in
// shared memory, compact state in TMEM, Z^(0) restart by TMA bulk copy; see
// k_resident.cuh), but one CTA holds NP frame pairs and each thread processes its
// circulant row for all NP pairs in the same batch step.  The row's variable
// addresses (jZ + (r + s) mod Z), the batch dispatch, the TMEM addressing and the
// batch barrier are shared by NP pairs, and the NP independent row computations
// give the scheduler instruction-level parallelism.  Used when NP pairs fit in
// shared memory (cfg2/cfg3: NP = 3, one CTA per SM).
#pragma once
#include "k_resident.cuh"

namespace ldpc {

// one circulant row r of one base row for NP frame pairs
template <int DC, int NP, bool ES>
__device__ __forceinline__ void mp_row(const ResArgs &a, const QcTab &t, uint32_t bp, uint32_t ba, uint32_t pstride,
                                       int e0, uint32_t r4, bool first_iter, RowState (&st)[NP],
                                       uint32_t (&synd)[NP]) {
    uint32_t d[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        const uint2 e = t.ent[e0 + j];
        const uint32_t u = r4 + e.x;
        d[j] = min(u - t.Z4, u) + e.y;                   // 4 * (jZ + (r + s) mod Z)
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const uint32_t bpp = bp + p * pstride, bap = ba + p * pstride;
        uint32_t L[DC];
#pragma unroll
        for (int j = 0; j < DC; ++j) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(L[j]) : "r"(bpp + d[j]));
        if (ES) synd[p] |= row_parity<DC>(L);
        uint32_t q[DC];
        if (first_iter) {
#pragma unroll
            for (int j = 0; j < DC; ++j) q[j] = L[j];    // L^(0)_mn = 0
        } else {
            rebuild_q<DC>(L, st[p], q);
        }
        uint32_t rn[DC];
        new_state<DC>(q, a.nbeta2p1, a.q2p1, st[p], rn, a.zero);
#pragma unroll
        for (int j = 0; j < DC; ++j) {                   // Z^(k)_n += L^(k)_mn
            uint32_t v;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(bap + d[j]) : "memory");
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(bap + d[j]), "r"(vadd(v, rn[j])) : "memory");
        }
    }
}

template <int NP, int FMT>
__device__ __forceinline__ void mp_state_load(uint32_t tw, int cpp, int b, int nb, RowState (&st)[NP]) {
    if (FMT == FMT_C16) {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            tmem_ld2(tw + p * cpp + 2 * b, st[p].A, st[p].B);
            tmem_ld1(tw + p * cpp + 2 * nb + b, st[p].W);
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) tmem_wait_ld_dep(st[p].A, st[p].B, st[p].W);
    } else {
        uint32_t X[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) tmem_ld2(tw + p * cpp + 2 * b, X[p], st[p].W);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            tmem_wait_ld_dep(X[p], st[p].W, st[p].W);
            st[p].A = prmt(X[p], 0u, 0x4240u);
            st[p].B = prmt(X[p], 0u, 0x4341u);
        }
    }
}

template <int NP, int FMT>
__device__ __forceinline__ void mp_state_store(uint32_t tw, int cpp, int b, int nb, const RowState (&st)[NP]) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        if (FMT == FMT_C16) {
            tmem_st2(tw + p * cpp + 2 * b, st[p].A, st[p].B);
            tmem_st1(tw + p * cpp + 2 * nb + b, st[p].W);
        } else {
            tmem_st2(tw + p * cpp + 2 * b, prmt(st[p].A, st[p].B, 0x6240u), st[p].W);
        }
    }
}

template <int DC, int NP, bool ES, int FMT>
__device__ __forceinline__ int mp_run(int b, int bend, int g, const ResArgs &a, const QcTab &t, uint32_t tw, int cpp,
                                      int nb, int rloc, uint32_t r4, uint32_t bp, uint32_t ba, uint32_t pstride,
                                      bool first_iter, uint32_t (&synd)[NP]) {
#pragma unroll 1
    for (; b < bend; ++b) {
        if constexpr (DC > 0) {
            RowState st[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) st[p] = RowState{0u, 0u, 0u};
            if (!first_iter) mp_state_load<NP, FMT>(tw, cpp, b, nb, st);
            if (rloc < a.Z) mp_row<DC, NP, ES>(a, t, bp, ba, pstride, t.e0[b][g], r4, first_iter, st, synd);
            mp_state_store<NP, FMT>(tw, cpp, b, nb, st);
        }
        __syncthreads();                                 // batch b's accumulations complete
    }
    return b;
}

template <int NP, bool ES, int FMT>
__device__ __forceinline__ int mp_run_dispatch(int dc, int b, int bend, int g, const ResArgs &a, const QcTab &t,
                                               uint32_t tw, int cpp, int nb, int rloc, uint32_t r4, uint32_t bp,
                                               uint32_t ba, uint32_t pstride, bool first_iter, uint32_t (&synd)[NP]) {
    switch (dc) {
    case 2: return mp_run<2, NP, ES, FMT>(b, bend, g, a, t, tw, cpp, nb, rloc, r4, bp, ba, pstride, first_iter, synd);
    case 3: return mp_run<3, NP, ES, FMT>(b, bend, g, a, t, tw, cpp, nb, rloc, r4, bp, ba, pstride, first_iter, synd);
    case 4: return mp_run<4, NP, ES, FMT>(b, bend, g, a, t, tw, cpp, nb, rloc, r4, bp, ba, pstride, first_iter, synd);
    case 5: return mp_run<5, NP, ES, FMT>(b, bend, g, a, t, tw, cpp, nb, rloc, r4, bp, ba, pstride, first_iter, synd);
    case 6: return mp_run<6, NP, ES, FMT>(b, bend, g, a, t, tw, cpp, nb, rloc, r4, bp, ba, pstride, first_iter, synd);
    case 7: return mp_run<7, NP, ES, FMT>(b, bend, g, a, t, tw, cpp, nb, rloc, r4, bp, ba, pstride, first_iter, synd);
    case 8: return mp_run<8, NP, ES, FMT>(b, bend, g, a, t, tw, cpp, nb, rloc, r4, bp, ba, pstride, first_iter, synd);
    default: return mp_run<0, NP, ES, FMT>(b, bend, g, a, t, tw, cpp, nb, rloc, r4, bp, ba, pstride, first_iter, synd);
    }
}

template <int NP>
__device__ __forceinline__ uint32_t mp_parity_row(const ResArgs &a, const QcTab &t, uint32_t bp, int dc, int e0,
                                                  uint32_t r4) {
    const char *base = (const char *)nullptr;
    (void)base;
    uint32_t par = 0;
    for (int j = 0; j < dc; ++j) {
        const uint2 e = t.ent[e0 + j];
        const uint32_t u = r4 + e.x;
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(bp + min(u - t.Z4, u) + e.y));
        par ^= vadd(v, 0xFFFFFFFFu);
    }
    return par & 0x80008000u;
}

// NP frame pairs per CTA ("pair group" pg = pairs NP*pg .. NP*pg + NP - 1).
template <int NP, bool ES, int FMT, typename TIN>
__global__ void __launch_bounds__(256, 1) k_resident_mp(const ResArgs a, const __grid_constant__ QcTab t) {
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t zbar;
    __shared__ uint32_t sflag[NP];
    const int tid = threadIdx.x, nth = blockDim.x;
    const int grp = a.group_threads == 128 ? (tid >> 7) : 0;
    const int rloc = tid - grp * a.group_threads;
    const uint32_t r4 = 4u * (uint32_t)rloc;
    const int nb = t.nsb;
    const int cpp = a.cols_per_group;                   // TMEM columns per (thread slice, pair)
    if (tid == 0) mbar_init(&zbar, 1);
    const uint32_t tbase = tmem_alloc_cta(&tslot, a.tmem_cols);
    const uint32_t tw = tmem_warp_base(tbase) + (uint32_t)((tid >> 7) * NP * cpp);
    const TIN *llr = (const TIN *)a.llr;
    const uint32_t zbytes = 4u * (uint32_t)a.Np;
    const uint32_t pstride = 8u * (uint32_t)a.Np;       // bytes between pairs' buffer sets
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    uint32_t zphase = 0;
    const int ngroups = (a.npairs + NP - 1) / NP;

    for (int pg = blockIdx.x; pg < ngroups; pg += gridDim.x) {
        __syncthreads();                                 // previous group's outputs read the buffers
        int done[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int pair = pg * NP + p;
            const int f0 = 2 * pair, f1 = f0 + 1;
            done[p] = pair >= a.npairs ? 3 : (f1 < a.nframes ? 0 : 2);
            uint32_t *z0w = a.ws + ((size_t)blockIdx.x * NP + p) * a.slot_words;
            uint32_t *b0 = smem + (size_t)p * 2 * a.Np, *b1 = b0 + a.Np;
            const bool lo_valid = pair < a.npairs, hi_valid = f1 < a.nframes;
            for (int n = tid; n < a.Np; n += nth) {
                uint32_t v = 0;
                if (n < a.N && lo_valid) {
                    const int zl = load_llr_sat(llr + (size_t)f0 * a.N + n, a.Qsat);
                    const int zh = hi_valid ? load_llr_sat(llr + (size_t)f1 * a.N + n, a.Qsat) : 0;
                    v = pack2(2 * zl, 2 * zh);
                }
                __stcg(z0w + n, v);
                b0[n] = v;
                b1[n] = v;
            }
        }
        fence_proxy_async_all();                         // z0 slots (generic writes) are later read by TMA
        __syncthreads();
        bool finished = false;
        for (int k = 1; k <= a.K; ++k) {
            const uint32_t bp = sbase + ((k & 1) ? 0u : 4u * (uint32_t)a.Np);   // Z^(k-1)
            const uint32_t ba = sbase + ((k & 1) ? 4u * (uint32_t)a.Np : 0u);   // Z^(k)
            if (k > 1) { mbar_wait(&zbar, zphase); zphase ^= 1; }               // accumulators = Z^(0)
            if (ES && tid < NP) sflag[tid] = 0;
            uint32_t synd[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) synd[p] = 0;
            const bool first_iter = (k == 1);
#pragma unroll 1
            for (int b = 0; b < nb;) {
                if (grp == 0) b = mp_run_dispatch<NP, ES, FMT>(t.dc[b][0], b, t.run_end[b][0], 0, a, t, tw, cpp, nb, rloc, r4, bp, ba, pstride, first_iter, synd);
                else b = mp_run_dispatch<NP, ES, FMT>(t.dc[b][1], b, t.run_end[b][1], 1, a, t, tw, cpp, nb, rloc, r4, bp, ba, pstride, first_iter, synd);
            }
            tmem_wait_st();
            if (ES) {
                // syndrome of Z^(k-1) per pair (gathered during this scan; 1-iteration lag)
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    const uint32_t w = __reduce_or_sync(0xFFFFFFFFu, synd[p]);
                    if ((tid & 31) == 0 && w) atomicOr(&sflag[p], w);
                }
                __syncthreads();
                bool all = true;
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    const uint32_t f = sflag[p];
                    const int conv = ((f & 0x00008000u) ? 0 : 1) | ((f & 0x80000000u) ? 0 : 2);
                    const int newly = conv & ~done[p];
                    if (newly) {
                        res_write_outputs(a, (const uint32_t *)smem + (size_t)p * 2 * a.Np + ((k & 1) ? 0 : a.Np),
                                          2 * (pg * NP + p), newly, k - 1, 0, 0);
                        done[p] |= newly;
                    }
                    all = all && done[p] == 3;
                }
                if (all) { finished = true; break; }
            }
            if (k < a.K) {
                // restart the next accumulators (the buffers just read) from Z^(0) by TMA
                fence_proxy_async_smem();
                __syncthreads();
                if (tid == 0) {
                    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&zbar);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(NP * zbytes) : "memory");
#pragma unroll
                    for (int p = 0; p < NP; ++p) {
                        const uint32_t dst = bp + p * pstride;
                        const uint32_t *src = a.ws + ((size_t)blockIdx.x * NP + p) * a.slot_words;
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                     ::"r"(dst), "l"(src), "r"(zbytes), "r"(b) : "memory");
                    }
                }
            }
        }
        if (!finished) {
            // final syndrome of Z^(K) and outputs of the frames still running
            const uint32_t bp = sbase + (((a.K + 1) & 1) ? 0u : 4u * (uint32_t)a.Np);
            uint32_t synd[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) synd[p] = 0;
            if (tid < NP) sflag[tid] = 0;
            __syncthreads();
            for (int b = 0; b < nb; ++b) {
                const int dc = t.dc[b][grp];
                if (rloc < a.Z && dc) {
#pragma unroll
                    for (int p = 0; p < NP; ++p) synd[p] |= mp_parity_row<NP>(a, t, bp + p * pstride, dc, t.e0[b][grp], r4);
                }
            }
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const uint32_t w = __reduce_or_sync(0xFFFFFFFFu, synd[p]);
                if ((tid & 31) == 0 && w) atomicOr(&sflag[p], w);
            }
            __syncthreads();
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const uint32_t f = sflag[p];
                const int which = 3 & ~done[p];
                if (which)
                    res_write_outputs(a, (const uint32_t *)smem + (size_t)p * 2 * a.Np + (((a.K + 1) & 1) ? 0 : a.Np),
                                      2 * (pg * NP + p), which, a.K, (f & 0x00008000u) != 0, (f & 0x80000000u) != 0);
            }
        }
    }
    tmem_free_cta(tbase, a.tmem_cols);
}

}  // namespace ldpc
