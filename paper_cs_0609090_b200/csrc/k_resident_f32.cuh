// k_resident_f32.cuh -- decode-resident single-scan min-sum for fp32 LLRs (flooding
// schedule).  The barrier-free structure of k_resident_atom.cuh with one frame per CTA:
// posterior double buffer Z^(k-1) | Z^(k) as fp32 in shared memory, the compact state
// (A_m, B_m, W_m = signs | one-hot position ñ_m) of every owned row in TMEM (three
// columns per row slot), the accumulation Z^(k)_n += L^(k)_mn as a shared-memory
// RED.ADD.F32 and the accumulator restart Z^(k) = Z^(0) as a TMA bulk copy.
//
// The per-row arithmetic is rowcore_f32.cuh f32_row, the same core as the fp32
// streaming kernel (reading D11: one RN rounding per operation, no contraction).  The
// order of the fp32 additions into Z_n is the order the atomics land, so posteriors
// agree with the oracle to rounding (the fp32 parity tolerance), not bit for bit.
//
// Row ownership and row tables are those of the integer barrier-free kernel (QcTab
// slots per 128-thread group for QC codes, rows t, t + T, ... otherwise).
#pragma once
#include "k_resident_atom.cuh"
#include "rowcore_f32.cuh"

namespace ldpc {

template <int DC, bool QC>
__device__ __forceinline__ void f32res_addr(const ResArgs &a, const QcTab &t, int e0, uint32_t r4, int p,
                                            uint32_t (&d)[DC]) {
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        if (QC) {
            const uint2 e = t.ent[e0 + j];
            const uint32_t u = r4 + e.x;
            d[j] = min(u - t.Z4, u) + e.y;                 // 4 * (jZ + (r + s) mod Z)
        } else {
            d[j] = __ldg(a.colT + (size_t)j * a.M + p);
        }
    }
}

template <int DC, bool QC, bool ES>
__device__ __forceinline__ void f32res_row(const ResArgs &a, const QcTab &t, float alpha, float beta, uint32_t bp,
                                           uint32_t ba, int e0, uint32_t r4, int p, bool first_iter, RowState &st,
                                           uint32_t &synd) {
    uint32_t d[DC];
    f32res_addr<DC, QC>(a, t, e0, r4, p, d);
    float L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(L[j]) : "r"(d[j] + bp));
    if (ES) {                                              // syndrome of Z^(k-1): hard bit = [Z_n <= 0]
        uint32_t par = 0;
#pragma unroll
        for (int j = 0; j < DC; ++j) par ^= L[j] <= 0.0f ? 1u : 0u;
        synd |= par;
    }
    float A, B, r[DC];
    uint32_t Wn;
    f32_row<DC>(L, first_iter, __uint_as_float(st.A), __uint_as_float(st.B), st.W, alpha, beta, A, B, Wn, r);
    st.A = __float_as_uint(A);
    st.B = __float_as_uint(B);
    st.W = Wn;
#pragma unroll
    for (int j = 0; j < DC; ++j)                                          // Z^(k)_n += L^(k)_mn
        asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(d[j] + ba), "f"(r[j]) : "memory");
}

template <int DC, bool QC>
__device__ __forceinline__ uint32_t f32res_parity(const ResArgs &a, const QcTab &t, uint32_t bz, int e0, uint32_t r4,
                                                  int p) {
    uint32_t d[DC];
    f32res_addr<DC, QC>(a, t, e0, r4, p, d);
    uint32_t par = 0;
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        float L;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(L) : "r"(d[j] + bz));
        par ^= L <= 0.0f ? 1u : 0u;
    }
    return par;
}

template <bool QC>
__device__ __forceinline__ uint32_t f32res_parity_dispatch(int dc, const ResArgs &a, const QcTab &t, uint32_t bz,
                                                           int e0, uint32_t r4, int p) {
    switch (dc) {
    case 2: return f32res_parity<2, QC>(a, t, bz, e0, r4, p);
    case 3: return f32res_parity<3, QC>(a, t, bz, e0, r4, p);
    case 4: return f32res_parity<4, QC>(a, t, bz, e0, r4, p);
    case 5: return f32res_parity<5, QC>(a, t, bz, e0, r4, p);
    case 6: return f32res_parity<6, QC>(a, t, bz, e0, r4, p);
    case 7: return f32res_parity<7, QC>(a, t, bz, e0, r4, p);
    case 8: return f32res_parity<8, QC>(a, t, bz, e0, r4, p);
    }
    return 0;
}

template <int DC, bool ES>
__device__ __forceinline__ int f32res_qc_run(int b, int bend, int g, const ResArgs &a, const QcTab &t, float alpha,
                                             float beta, uint32_t tw, int nb, int rloc, uint32_t r4, uint32_t bp,
                                             uint32_t ba, bool first_iter, uint32_t &synd) {
    if constexpr (DC == 0) {
        return bend;
    } else {
#pragma unroll 1
        for (; b < bend; ++b) {
            RowState st = {0u, 0u, 0u};
            if (!first_iter) state_tmem_load<FMT_C16>(tw, b, nb, st);
            if (rloc < a.Z) f32res_row<DC, true, ES>(a, t, alpha, beta, bp, ba, t.e0[b][g], r4, 0, first_iter, st, synd);
            state_tmem_store<FMT_C16>(tw, b, nb, st);
        }
        return b;
    }
}

template <bool ES>
__device__ __forceinline__ int f32res_qc_dispatch(int dc, int b, int bend, int g, const ResArgs &a, const QcTab &t,
                                                  float alpha, float beta, uint32_t tw, int nb, int rloc, uint32_t r4,
                                                  uint32_t bp, uint32_t ba, bool first_iter, uint32_t &synd) {
    switch (dc) {
    case 2: return f32res_qc_run<2, ES>(b, bend, g, a, t, alpha, beta, tw, nb, rloc, r4, bp, ba, first_iter, synd);
    case 3: return f32res_qc_run<3, ES>(b, bend, g, a, t, alpha, beta, tw, nb, rloc, r4, bp, ba, first_iter, synd);
    case 4: return f32res_qc_run<4, ES>(b, bend, g, a, t, alpha, beta, tw, nb, rloc, r4, bp, ba, first_iter, synd);
    case 5: return f32res_qc_run<5, ES>(b, bend, g, a, t, alpha, beta, tw, nb, rloc, r4, bp, ba, first_iter, synd);
    case 6: return f32res_qc_run<6, ES>(b, bend, g, a, t, alpha, beta, tw, nb, rloc, r4, bp, ba, first_iter, synd);
    case 7: return f32res_qc_run<7, ES>(b, bend, g, a, t, alpha, beta, tw, nb, rloc, r4, bp, ba, first_iter, synd);
    case 8: return f32res_qc_run<8, ES>(b, bend, g, a, t, alpha, beta, tw, nb, rloc, r4, bp, ba, first_iter, synd);
    default: return f32res_qc_run<0, ES>(b, bend, g, a, t, alpha, beta, tw, nb, rloc, r4, bp, ba, first_iter, synd);
    }
}

template <bool ES>
__device__ __forceinline__ void f32res_csr_dispatch(int dc, const ResArgs &a, const QcTab &t, float alpha, float beta,
                                                    uint32_t bp, uint32_t ba, int p, bool first_iter, RowState &st,
                                                    uint32_t &synd) {
    switch (dc) {
    case 2: f32res_row<2, false, ES>(a, t, alpha, beta, bp, ba, 0, 0, p, first_iter, st, synd); break;
    case 3: f32res_row<3, false, ES>(a, t, alpha, beta, bp, ba, 0, 0, p, first_iter, st, synd); break;
    case 4: f32res_row<4, false, ES>(a, t, alpha, beta, bp, ba, 0, 0, p, first_iter, st, synd); break;
    case 5: f32res_row<5, false, ES>(a, t, alpha, beta, bp, ba, 0, 0, p, first_iter, st, synd); break;
    case 6: f32res_row<6, false, ES>(a, t, alpha, beta, bp, ba, 0, 0, p, first_iter, st, synd); break;
    case 7: f32res_row<7, false, ES>(a, t, alpha, beta, bp, ba, 0, 0, p, first_iter, st, synd); break;
    case 8: f32res_row<8, false, ES>(a, t, alpha, beta, bp, ba, 0, 0, p, first_iter, st, synd); break;
    }
}

// outputs of frame f from the posterior buffer Ls: Z_n, hard bits [Z_n <= 0], ok, iterations
static __device__ void f32res_write_outputs(const ResArgs &a, const float *Ls, int f, int iters, int fail) {
    const int tid = threadIdx.x, nth = blockDim.x;
    if (a.post) {
        float *post = (float *)(void *)a.post + (size_t)f * a.N;
        for (int n = tid; n < a.N; n += nth) post[n] = Ls[n];
    }
    const int lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
    for (int w = warp; w < a.wpf; w += nw) {
        const int n = w * 32 + lane;
        const uint32_t word = __ballot_sync(0xFFFFFFFFu, n < a.N && Ls[n] <= 0.0f);
        if (lane == 0) a.hard_bits[(size_t)f * a.wpf + w] = word;
    }
    if (tid == 0) {
        a.ok[f] = (uint8_t)!fail;
        if (a.iters) a.iters[f] = iters;
    }
}

template <bool QC, bool ES>
__global__ void __launch_bounds__(256, 3) k_resident_f32(const __grid_constant__ ResArgs a,
                                                         const __grid_constant__ QcTab t) {
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t zbar;
    float *buf0 = (float *)smem, *buf1 = (float *)smem + a.Np;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int grp = QC ? (a.group_threads == 128 ? (tid >> 7) : 0) : 0;
    const int rloc = QC ? tid - grp * a.group_threads : tid;
    const uint32_t r4 = 4u * (uint32_t)rloc;
    const int nb = QC ? t.nsb : a.nbatch;
    if (tid == 0) mbar_init(&zbar, 1);
    const uint32_t tbase = tmem_alloc_cta(&tslot, a.tmem_cols);   // includes a block barrier
    const uint32_t tw = tmem_warp_base(tbase) + (uint32_t)((tid >> 7) * a.cols_per_group);
    uint32_t *z0w = a.ws + (size_t)blockIdx.x * a.slot_words;
    const uint32_t zbytes = 4u * (uint32_t)a.Np;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(buf0), s1 = (uint32_t)__cvta_generic_to_shared(buf1);
    uint32_t zphase = 0;

    for (int f = blockIdx.x; f < a.nframes; f += gridDim.x) {
        __syncthreads();                             // previous frame's outputs read the buffers
        const float *src = (const float *)a.llr + (size_t)f * a.N;
        for (int n = tid; n < a.Np; n += nth) {
            const float z = n < a.N ? __ldg(src + n) + 0.0f : 0.0f;   // canonicalise -0.0 (reading D13)
            __stcg(z0w + n, __float_as_uint(z));
            buf0[n] = z;
            buf1[n] = z;
        }
        fence_proxy_async_all();                     // z0w (generic writes) is later read by TMA
        __syncthreads();
        bool finished = false;
        for (int k = 1; k <= a.K; ++k) {
            const uint32_t bp = (k & 1) ? s0 : s1, ba = (k & 1) ? s1 : s0;   // Z^(k-1) | Z^(k)
            if (k > 1) { mbar_wait(&zbar, zphase); zphase ^= 1; }          // Z^(k) = Z^(0) landed
            uint32_t synd = 0;
            const bool first_iter = (k == 1);
            const float alpha = a.nsched ? a.alpha_sched[k - 1] : a.alpha;   // lambda_k / beta_k
            const float beta = a.nsched ? a.beta_sched[k - 1] : a.beta;
            // the first iteration (no rebuild, no state load) is a compile-time variant of the scan
            auto scan = [&](auto fi_tag) {
                constexpr bool FI = decltype(fi_tag)::value;
                if (QC) {
#pragma unroll 1
                    for (int b = 0; b < nb;) {
                        if (grp == 0) b = f32res_qc_dispatch<ES>(t.dc[b][0], b, t.run_end[b][0], 0, a, t, alpha, beta, tw, nb, rloc, r4, bp, ba, FI, synd);
                        else b = f32res_qc_dispatch<ES>(t.dc[b][1], b, t.run_end[b][1], 1, a, t, alpha, beta, tw, nb, rloc, r4, bp, ba, FI, synd);
                    }
                } else {
#pragma unroll 1
                    for (int b = 0; b < nb; ++b) {
                        const int p = b * nth + tid;
                        RowState st = {0u, 0u, 0u};
                        if (!FI) state_tmem_load<FMT_C16>(tw, b, nb, st);
                        if (p < a.M) f32res_csr_dispatch<ES>(a.dcT[p], a, t, alpha, beta, bp, ba, p, FI, st, synd);
                        state_tmem_store<FMT_C16>(tw, b, nb, st);
                    }
                }
            };
            if (first_iter) scan(std::integral_constant<bool, true>{});
            else scan(std::integral_constant<bool, false>{});
            tmem_wait_st();
            const float *Lp = (k & 1) ? buf0 : buf1;
            if (ES) {
                // syndrome of Z^(k-1), gathered during this scan (1-iteration lag)
                if (!__syncthreads_or(synd != 0)) {
                    f32res_write_outputs(a, Lp, f, k - 1, 0);
                    finished = true;
                    break;
                }
            }
            if (k < a.K) {
                fence_proxy_async_smem();
                __syncthreads();
                if (tid == 0) tma_bulk_g2s((void *)Lp, z0w, zbytes, &zbar);   // restart the next accumulator
            }
        }
        if (!finished) {
            __syncthreads();                         // all atomics of iteration K landed
            const float *Lz = ((a.K + 1) & 1) ? buf0 : buf1;
            const uint32_t bz = (uint32_t)__cvta_generic_to_shared(Lz);
            uint32_t synd = 0;
            if (QC) {
                for (int b = 0; b < nb; ++b) {
                    const int dc = t.dc[b][grp];
                    if (rloc < a.Z && dc) synd |= f32res_parity_dispatch<true>(dc, a, t, bz, t.e0[b][grp], r4, 0);
                }
            } else {
                for (int b = 0; b < nb; ++b) {
                    const int p = b * nth + tid;
                    if (p < a.M) synd |= f32res_parity_dispatch<false>(a.dcT[p], a, t, bz, 0, 0, p);
                }
            }
            const int fail = __syncthreads_or(synd != 0);
            f32res_write_outputs(a, Lz, f, a.K, fail);
        }
    }
    tmem_free_cta(tbase, a.tmem_cols);
}

// ------------------------------------------------------------------ layered (D25)
// LDPC_SCHED_LAYERED with fp32 LLRs: ONE posterior array, rows in ascending m, each row
// replacing its old message in place, Z_n <- (Z_n - L^(k-1)_mn) + L^(k)_mn.  Batches hold
// consecutive variable-disjoint rows (the integer layered kernel's tables), a barrier after
// each.  Every variable is then updated by one row at a time in the schedule's order, with
// the oracle's operations (D11), so unlike flooding the fp32 result is order-exact.
template <int DC, bool QC>
__device__ __forceinline__ void f32lay_row(const ResArgs &a, const QcTab &t, float alpha, float beta, uint32_t bz,
                                           int e0, uint32_t r4, int p, bool first_iter, RowState &st) {
    uint32_t d[DC];
    f32res_addr<DC, QC>(a, t, e0, r4, p, d);
    float L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(L[j]) : "r"(d[j] + bz));
    float A, B, r[DC], q[DC];
    uint32_t Wn;
    f32_row_q<DC>(L, first_iter, __uint_as_float(st.A), __uint_as_float(st.B), st.W, alpha, beta, A, B, Wn, r, q);
    st.A = __float_as_uint(A);
    st.B = __float_as_uint(B);
    st.W = Wn;
#pragma unroll
    for (int j = 0; j < DC; ++j)                                          // Z_n = (Z_n - L_old) + L_new
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(d[j] + bz), "f"(__fadd_rn(q[j], r[j])) : "memory");
}

template <bool QC>
__device__ __forceinline__ void f32lay_dispatch(int dc, const ResArgs &a, const QcTab &t, float alpha, float beta,
                                                uint32_t bz, int e0, uint32_t r4, int p, bool first_iter, RowState &st) {
    switch (dc) {
    case 2: f32lay_row<2, QC>(a, t, alpha, beta, bz, e0, r4, p, first_iter, st); break;
    case 3: f32lay_row<3, QC>(a, t, alpha, beta, bz, e0, r4, p, first_iter, st); break;
    case 4: f32lay_row<4, QC>(a, t, alpha, beta, bz, e0, r4, p, first_iter, st); break;
    case 5: f32lay_row<5, QC>(a, t, alpha, beta, bz, e0, r4, p, first_iter, st); break;
    case 6: f32lay_row<6, QC>(a, t, alpha, beta, bz, e0, r4, p, first_iter, st); break;
    case 7: f32lay_row<7, QC>(a, t, alpha, beta, bz, e0, r4, p, first_iter, st); break;
    case 8: f32lay_row<8, QC>(a, t, alpha, beta, bz, e0, r4, p, first_iter, st); break;
    }
}

// parity of all rows of this thread against the array at bz (nonzero iff some row fails)
template <bool QC>
__device__ __forceinline__ uint32_t f32lay_parity_pass(const ResArgs &a, const QcTab &t, uint32_t bz, int nb, int grp,
                                                       int rloc, uint32_t r4, int tid) {
    uint32_t synd = 0;
    for (int b = 0; b < nb; ++b) {
        if (QC) {
            const int dc = t.dc[b][grp];
            if (rloc < a.Z && dc) synd |= f32res_parity_dispatch<true>(dc, a, t, bz, t.e0[b][grp], r4, 0);
        } else {
            const int p = a.bptr[b] + tid;
            if (p < a.bptr[b + 1]) synd |= f32res_parity_dispatch<false>(a.dcT[p], a, t, bz, 0, 0, p);
        }
    }
    return synd;
}

template <bool QC, bool ES>
__global__ void __launch_bounds__(256, 3) k_resident_f32_lay(const __grid_constant__ ResArgs a,
                                                             const __grid_constant__ QcTab t) {
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint32_t tslot;
    float *zb = (float *)smem;                           // the one posterior array
    uint32_t *sst = smem + a.Np;                         // general codes: compact state [3][M], by row
    const int tid = threadIdx.x, nth = blockDim.x;
    const int grp = QC ? (a.group_threads == 128 ? (tid >> 7) : 0) : tid >> 7;
    const int rloc = QC ? tid - grp * a.group_threads : tid;
    const uint32_t r4 = 4u * (uint32_t)rloc;
    const int nb = QC ? t.nsb : a.nbatch;
    const uint32_t tbase = tmem_alloc_cta(&tslot, a.tmem_cols);   // includes a block barrier
    const uint32_t tw = tmem_warp_base(tbase) + (uint32_t)((tid >> 7) * a.cols_per_group);
    const uint32_t bz = (uint32_t)__cvta_generic_to_shared(zb);

    for (int f = blockIdx.x; f < a.nframes; f += gridDim.x) {
        __syncthreads();                             // previous frame's outputs read the array
        const float *src = (const float *)a.llr + (size_t)f * a.N;
        for (int n = tid; n < a.Np; n += nth) zb[n] = n < a.N ? __ldg(src + n) + 0.0f : 0.0f;   // -0.0 -> +0.0 (D13)
        __syncthreads();
        bool finished = false;
        for (int k = 1; k <= a.K; ++k) {
            if (ES) {
                // syndrome of the posterior after iteration k-1, before this iteration changes it
                const uint32_t synd = f32lay_parity_pass<QC>(a, t, bz, nb, grp, rloc, r4, tid);
                if (!__syncthreads_or(synd != 0)) {
                    f32res_write_outputs(a, zb, f, k - 1, 0);
                    finished = true;
                    break;
                }
            }
            const bool first_iter = (k == 1);
            const float alpha = a.nsched ? a.alpha_sched[k - 1] : a.alpha;   // lambda_k / beta_k
            const float beta = a.nsched ? a.beta_sched[k - 1] : a.beta;
#pragma unroll 1
            for (int b = 0; b < nb; ++b) {
                RowState st = {0u, 0u, 0u};
                if (QC) {
                    const int dc = t.dc[b][grp];
                    if (!first_iter) state_tmem_load<FMT_C16>(tw, b, nb, st);
                    if (rloc < a.Z && dc) f32lay_dispatch<true>(dc, a, t, alpha, beta, bz, t.e0[b][grp], r4, 0, first_iter, st);
                    state_tmem_store<FMT_C16>(tw, b, nb, st);
                } else {
                    const int p = a.bptr[b] + tid;
                    if (p < a.bptr[b + 1]) {
                        if (!first_iter) { st.A = sst[p]; st.B = sst[a.M + p]; st.W = sst[2 * a.M + p]; }
                        f32lay_dispatch<false>(a.dcT[p], a, t, alpha, beta, bz, 0, 0, p, first_iter, st);
                        sst[p] = st.A;
                        sst[a.M + p] = st.B;
                        sst[2 * a.M + p] = st.W;
                    }
                }
                __syncthreads();                         // batch b's in-place updates complete
            }
            if (QC) tmem_wait_st();
        }
        if (!finished) {
            const uint32_t synd = f32lay_parity_pass<QC>(a, t, bz, nb, grp, rloc, r4, tid);   // final syndrome
            const int fail = __syncthreads_or(synd != 0);
            f32res_write_outputs(a, zb, f, a.K, fail);
        }
    }
    tmem_free_cta(tbase, a.tmem_cols);
}

}  // namespace ldpc
