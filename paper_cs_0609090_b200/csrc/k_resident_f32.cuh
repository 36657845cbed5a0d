// k_resident_f32.cuh -- decode-resident LAYERED single-scan min-sum for fp32 LLRs
// (LDPC_SCHED_LAYERED, reading D25): one frame per CTA, its one posterior array in shared
// memory, the compact state (A_m, B_m, W_m = signs | one-hot position ñ_m) of every owned
// row in TMEM (QC codes: three columns per row slot) or shared memory (other codes).
// The per-row arithmetic is rowcore_f32.cuh f32_row_q, the core of the fp32 streaming
// kernels (reading D11: one RN rounding per operation, no contraction).
// (fp32 FLOODING decodes take the streaming kernels, whose exact int64 accumulation,
// reading D28, makes them order-free; a shared-memory fp32 or 64-bit atomic is a CAS loop
// on sm_100a, which is why round 1's resident fp32 flooding kernel was removed.)
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
        // -0.0 -> +0.0 (D13), saturation at +-2^20 (D28)
        for (int n = tid; n < a.Np; n += nth) zb[n] = n < a.N ? fminf(fmaxf(__ldg(src + n) + 0.0f, -1048576.0f), 1048576.0f) : 0.0f;
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
