// k_stream_layered.cuh -- the layered (in-place) single-scan schedule for codes too long for
// the resident kernel (LDPC_SCHED_LAYERED, reading D25).
//
// D25 processes the rows of H in ascending m, each row replacing its old message in the ONE
// posterior array, Z_n <- (Z_n - L^(k-1)_mn) + L^(k)_mn, so row m must see every update of
// the rows before it that share a variable.  On a DVB-S2-shaped code consecutive rows always
// share a staircase parity column, so within a frame the schedule is one chain of M dependent
// row updates per iteration: the only parallelism is across frames.  One warp
// owns one frame tile for the whole decode (lanes = frame pairs in 16x2 SIMD, or frames for
// fp32) and walks the rows in order; a lane's store of Z_n is seen by the same lane's later
// loads (program order), which is all the schedule needs.  Correct at any size, but with
// ceil(F / 64) warps in flight it is a latency-bound baseline, not a fast path.
//
// Layout: the streaming kernels' frame-interleaved planes ([tile][n][32] posterior words in
// Lb[0], biased 2Z + 0x4000 per lane for integer pairs as k_stream.cuh; fp32: plain floats
// with the per-operation rounding of D11 -- D28's exact sums are for flooding), compact state
// [tile][words][M][32] (StateIO for integer formats; A, B, W for fp32).
#pragma once
#include "k_stream.cuh"

namespace ldpc {

// per-iteration check-node variants of the single-launch layered kernel (lambda_k / beta_k,
// P:179), passed by value: n = 0 -> the constants in StreamArgs
struct LaySched {
    int n;
    VarK vk[kMaxSched];
    float alpha[kMaxSched], beta[kMaxSched];
};

// one row, integer pairs: q = Z - L_old (biased words in, unbiased q), new state, Z <- q + L_new
template <int DC, int FMT>
__device__ __forceinline__ void lay_row_i(const StreamArgs &a, const VarK &vk, uint32_t *Lt, uint32_t *stt, size_t ss,
                                          int m, const uint32_t (&col)[8], int lane, bool first, uint32_t keep) {
    uint32_t L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        LDPC_CHECK(col[j] < (uint32_t)a.N);
        L[j] = __ldcg(Lt + (size_t)col[j] * 32 + lane);
    }
    RowState st = {0u, 0u, 0u};
    uint32_t q[DC];
    if (first) {
#pragma unroll
        for (int j = 0; j < DC; ++j) q[j] = vadd(L[j], 0xC000C000u);      // L^(0)_mn = 0; unbias
    } else {
        st = StateIO<FMT>::load(stt + lane, ss, (size_t)m * 32);
        rebuild_q<DC, true>(L, st, q, a.rk);                               // Z_n - L^(k-1)_mn
    }
    uint32_t rn[DC];
    new_state<DC, false, -1, FMT == FMT_1BIT>(q, vk, st, rn, a.rk);
    StateIO<FMT>::store(stt + lane, ss, (size_t)m * 32, st);
#pragma unroll
    for (int j = 0; j < DC; ++j) {                                       // in place (D25); frozen lanes keep Z
        const uint32_t z = vadd(vadd(q[j], rn[j]), kPairBias);
        __stcg(Lt + (size_t)col[j] * 32 + lane, sel(keep, L[j], z));
    }
}

// one row, fp32 (D11: q = fl(Z - L_old), Z <- fl(q + L_new))
template <int DC>
__device__ __forceinline__ void lay_row_f(const StreamArgs &a, float alpha, float beta, float *Lt, uint32_t *stt,
                                          size_t ss, int m, const uint32_t (&col)[8], int lane, bool first,
                                          bool frozen) {
    float L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        LDPC_CHECK(col[j] < (uint32_t)a.N);
        L[j] = __ldcg(Lt + (size_t)col[j] * 32 + lane);
    }
    const size_t so = (size_t)m * 32 + lane;
    float A0 = 0.f, B0 = 0.f;
    uint32_t W0 = 0;
    if (!first) {
        A0 = __uint_as_float(__ldcg(stt + so));
        B0 = __uint_as_float(__ldcg(stt + ss + so));
        W0 = __ldcg(stt + 2 * ss + so);
    }
    float A, B, r[DC], q[DC];
    uint32_t Wn;
    f32_row_q<DC>(L, first, A0, B0, W0, alpha, beta, A, B, Wn, r, q);
    __stcg(stt + so, __float_as_uint(A));
    __stcg(stt + ss + so, __float_as_uint(B));
    __stcg(stt + 2 * ss + so, Wn);
    if (!frozen) {
#pragma unroll
        for (int j = 0; j < DC; ++j) __stcg(Lt + (size_t)col[j] * 32 + lane, __fadd_rn(q[j], r[j]));
    }
}

// parity of every row against the current posteriors: per-lane fail bits (pairs: bit 15 lo,
// bit 31 hi; fp32: bit 0), the stop test of P:174 on the posterior after a full iteration
template <bool PAIR>
__device__ __forceinline__ uint32_t lay_parity(const StreamArgs &a, const uint32_t *Lt, int lane) {
    uint32_t synd = 0;
    for (int m = 0; m < a.M; ++m) {
        const int e0 = __ldg(a.row_ptr + m), e1 = __ldg(a.row_ptr + m + 1);
        uint32_t p = 0;
        for (int e = e0; e < e1; ++e) {
            const uint32_t w = __ldcg(Lt + (size_t)__ldg(a.col_idx + e) * 32 + lane);
            if (PAIR) p ^= fadd32(w, kParBiased, a.rk);
            else p ^= __uint_as_float(w) <= 0.0f ? 1u : 0u;
        }
        synd |= PAIR ? (p & 0x80008000u) : (p & 1u);
    }
    return synd;
}

// frames of this lane that passed the test: frozen with iterations_used = k (ES), or the final
// flags (k = K)
template <bool PAIR>
__device__ __forceinline__ uint32_t lay_freeze(const StreamArgs &a, int tile, int lane, uint32_t synd, uint32_t done,
                                               int k, bool final_pass) {
    const int nh = PAIR ? 2 : 1;
    for (int h = 0; h < nh; ++h) {
        const int f = PAIR ? tile * 64 + 2 * lane + h : tile * 32 + lane;
        if (f >= a.nframes || (done & (1u << h))) continue;
        const bool fail = PAIR ? (h ? (synd & 0x80000000u) : (synd & 0x8000u)) : (synd & 1u);
        if (final_pass) {
            a.it_ws[f] = a.K;
            a.ok_ws[f] = fail ? 0 : 1;
        } else if (!fail) {
            a.it_ws[f] = k;
            a.ok_ws[f] = 1;
            done |= 1u << h;
        }
    }
    return done;
}

template <bool PAIR, int FMT, bool ES>
__global__ void __launch_bounds__(128) k_stream_layered(const StreamArgs a, const __grid_constant__ LaySched sch) {
    const int lane = threadIdx.x & 31;
    const int tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (tile >= a.ntiles) return;
    const size_t plane = (size_t)tile * a.N * 32;
    uint32_t *Lt = a.Lb[0] + plane;
    const int nst = PAIR ? StateIO<FMT>::kWords : 3;
    uint32_t *stt = a.st + (size_t)tile * nst * a.M * 32;
    const size_t ss = (size_t)a.M * 32;
    uint32_t done = 0;                                   // frames of this lane that stopped (bit per frame)
    if (ES) done = lay_freeze<PAIR>(a, tile, lane, lay_parity<PAIR>(a, Lt, lane), done, 0, false);   // k = 0 (D10)
    const uint32_t all = PAIR ? 3u : 1u;
    for (int k = 1; k <= a.K; ++k) {
        if (ES && __all_sync(0xFFFFFFFFu, done == all)) break;
        const uint32_t keep = PAIR ? (((done & 1) ? 0x0000FFFFu : 0u) | ((done & 2) ? 0xFFFF0000u : 0u)) : 0u;
        const bool frozen = !PAIR && (done & 1);
        const VarK vk = sch.n ? sch.vk[k - 1] : a.vk;            // iteration k's variant
        const float alpha = sch.n ? sch.alpha[k - 1] : a.alpha, beta = sch.n ? sch.beta[k - 1] : a.beta;
        for (int m = 0; m < a.M; ++m) {                  // rows in ascending m (D25)
            const RowT rt = load_rowt(a.rowtab, m, a.M);
            uint32_t col[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) col[j] = rt.c[j];
            switch (rt.dc) {
#define LDPC_LR(D)                                                                                      \
    case D:                                                                                             \
        if (PAIR) lay_row_i<D, FMT>(a, vk, Lt, stt, ss, m, col, lane, k == 1, keep);                    \
        else lay_row_f<D>(a, alpha, beta, (float *)Lt, stt, ss, m, col, lane, k == 1, frozen);          \
        break;
            LDPC_LR(2) LDPC_LR(3) LDPC_LR(4) LDPC_LR(5) LDPC_LR(6) LDPC_LR(7) LDPC_LR(8)
#undef LDPC_LR
            }
        }
        if (ES && k < a.K) done = lay_freeze<PAIR>(a, tile, lane, lay_parity<PAIR>(a, Lt, lane), done, k, false);
    }
    lay_freeze<PAIR>(a, tile, lane, lay_parity<PAIR>(a, Lt, lane), done, a.K, true);   // the rest: K iterations
}

}  // namespace ldpc
