// k_stream_pipe.cuh -- software-pipelined streaming kernels (long codes).
//
// Same data layout and per-row arithmetic as k_stream.cuh, but every warp keeps
// PD rows in flight: the 128-byte lines a row needs (its dc posterior lines and
// its compact-state lines for the warp's 32 lanes) are copied global -> shared
// with cp.async (LDGSTS, 16 B per lane) PD rows ahead of the row being computed,
// so memory-level parallelism is set by the shared-memory ring, not by
// registers.  A CTA owns a block of RB consecutive check rows of one frame tile;
// their column tables are staged in shared memory once.  Accumulation into
// Z^(k) stays a coalesced global RED (fire-and-forget).
#pragma once
#include <type_traits>

#include "k_stream.cuh"

namespace ldpc {

#ifndef LDPC_PIPE_D
#define LDPC_PIPE_D 4
#endif
#ifndef LDPC_PIPE_MINB
#define LDPC_PIPE_MINB 4
#endif
#ifndef LDPC_PIPE_RB
#define LDPC_PIPE_RB 64
#endif
#ifndef LDPC_PIPE_DF
#define LDPC_PIPE_DF 3
#endif
constexpr int kPipeRB = LDPC_PIPE_RB;   // rows per CTA
constexpr int kPipeWarps = 8;      // warps per CTA
// Ring slot of one row.  Integer pairs: 8 posterior lines (one 128-byte line of 32 lanes per
// variable) + up to 3 state lines, kPipeD rows in flight.  fp32 (reading D28): a posterior is
// an int64 grid value, two lines per variable: 16 lines, + 3 lines of the state of iteration
// k-1 + 3 of iteration k-2 (the delta accumulation below), kPipeDF rows in flight (the first
// iteration reads the fp32 Z^(0) plane, one line per variable).
template <bool PAIR> struct PipeCfg {
    static constexpr int LPV = PAIR ? 1 : 2;          // lines per variable (later iterations)
    static constexpr int SB = 8 * LPV;                // first state line
    static constexpr int LINES = PAIR ? SB + 3 : SB + 6;
    static constexpr int D = PAIR ? LDPC_PIPE_D : LDPC_PIPE_DF;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Issue the copies of one row's lines into a slot: posterior lines 0 .. dc*LPV-1 (variable
// col[l / LPV], 128-byte half l % LPV of its LPV*128-byte tile segment), state lines SB ..
// SB+nst-1 (the state words of row m).  Lane handles 16-byte chunk (lane & 7) of lines
// (lane >> 3) + 4 s; branch-free source selection, predicated copies.
template <int LPV, int SB>
__device__ __forceinline__ void pipe_issue_row(uint32_t slot, const char *Lpt, const uint32_t *stt, size_t sstride,
                                               const uint32_t *cols, int dc, int nst, int m, int lane,
                                               const uint32_t *stt2 = nullptr, int nst2 = 0) {
    const int chunk = lane & 7, l0 = lane >> 3;
#pragma unroll
    for (int step = 0; step < 2 * LPV; ++step) {         // posterior lines
        const int l = l0 + 4 * step;
        const char *src = Lpt + (size_t)cols[l / LPV] * (128 * LPV) + (l % LPV) * 128 + chunk * 16;
        if (l < dc * LPV) cp_async16(slot + (uint32_t)(l * 128 + chunk * 16), src);
    }
    if (l0 < nst) {                                        // state lines
        const char *src = (const char *)(stt + (size_t)m * 32) + chunk * 16 + (size_t)l0 * sstride * 4;
        cp_async16(slot + (uint32_t)((SB + l0) * 128 + chunk * 16), src);
    }
    if (l0 < nst2) {                                       // fp32 delta: the state two iterations back
        const char *src = (const char *)(stt2 + (size_t)m * 32) + chunk * 16 + (size_t)l0 * sstride * 4;
        cp_async16(slot + (uint32_t)((SB + 3 + l0) * 128 + chunk * 16), src);
    }
}

template <int DC, int FMT, bool ES, int VM>
__device__ __forceinline__ void pipe_row_i(const StreamArgs &a, const uint32_t *sl, const uint32_t *cols, int m,
                                           int lane, uint32_t *Lat, uint32_t *stt, size_t sstride, bool first_iter,
                                           uint32_t keep, uint32_t &synd) {
    uint32_t L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        LDPC_CHECK(cols[j] < (uint32_t)a.N && m < a.M);
        L[j] = sl[j * 32 + lane];
    }
    if (ES) synd |= row_parity<DC>(L, a.rk, kParBiased);
    RowState st;
    uint32_t q[DC];                                       // q + 0x8000 per lane
    if (first_iter) {
#pragma unroll
        for (int j = 0; j < DC; ++j) q[j] = fadd32(L[j], kPairBias, a.rk);
    } else {
        if (FMT == FMT_C16) {
            st.A = sl[8 * 32 + lane];
            st.B = sl[9 * 32 + lane];
            st.W = sl[10 * 32 + lane];
        } else {
            const uint32_t X = sl[8 * 32 + lane];
            st.A = prmt(X, 0u, 0x4240u);
            st.B = prmt(X, 0u, 0x4341u);
            st.W = expand_idx(sl[9 * 32 + lane]);       // index-coded ñ (rowcore.cuh)
        }
        rebuild_q_b8<DC>(L, st, q, a.rk);
    }
    uint32_t rn[DC];                                      // V(L^(k)_mn) + 0x8000
    new_state<DC, true, VM, FMT == FMT_1BIT>(q, a.vk, st, rn, a.rk);
    StateIO<FMT>::store(stt + lane, sstride, (size_t)m * 32, st);
#pragma unroll
    for (int j = 0; j < DC; ++j) atomicAdd(Lat + (size_t)cols[j] * 32 + lane, red_value(rn[j], keep));
}

// fp32 row (reading D11 arithmetic, D28 exact accumulation): posteriors from the ring
// (FI: fp32 Z^(0) lines; later: int64 grid values, rounded to fp32 here).
// Delta accumulation (a.f32delta): the plane of iteration k held the exact sum of iteration
// k-2, X_{k-2} = grid(Z^(0)) + sum_m grid(L^(k-2)_mn), so adding grid(L^(k)_mn) -
// grid(L^(k-2)_mn) for every edge leaves X_k = grid(Z^(0)) + sum_m grid(L^(k)_mn) -- the same
// exact integer as a fresh accumulation (integer addition is exact and associative), with no
// accumulator start to write: two posterior planes and two state planes instead of three
// posterior planes, and no DRAM round trip of start values written one iteration ahead.
// L^(k-2) is rebuilt from the state two iterations back (OLD2 = k >= 3; iterations 1 and 2
// start from grid(Z^(0)) written by the ingest into both planes).
template <int DC, bool ES, bool FI>
__device__ __forceinline__ void pipe_row_f(const StreamArgs &a, const uint32_t *sl, const uint32_t *cols, int m,
                                           int lane, long long *Xat, uint32_t *stt, size_t ss, bool frozen,
                                           uint32_t &synd, bool old2 = false) {
    constexpr int SB = PipeCfg<false>::SB;
    float L[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        LDPC_CHECK(cols[j] < (uint32_t)a.N && m < a.M);
        L[j] = FI ? __uint_as_float(sl[j * 32 + lane]) : val_of(((const long long *)sl)[j * 32 + lane]);
    }
    if (ES) {
        uint32_t p = 0;
#pragma unroll
        for (int j = 0; j < DC; ++j) p ^= L[j] <= 0.0f ? 1u : 0u;
        synd |= p;
    }
    float A0 = 0.f, B0 = 0.f;
    uint32_t W0 = 0;
    if (!FI) {
        A0 = __uint_as_float(sl[SB * 32 + lane]);
        B0 = __uint_as_float(sl[(SB + 1) * 32 + lane]);
        W0 = sl[(SB + 2) * 32 + lane];
    }
    float A, B, r[DC];
    uint32_t Wn;
    f32_row<DC>(L, FI, A0, B0, W0, a.alpha, a.beta, A, B, Wn, r);
    const size_t so = (size_t)m * 32 + lane;
    __stcg(stt + so, __float_as_uint(A));
    __stcg(stt + ss + so, __float_as_uint(B));
    __stcg(stt + 2 * ss + so, Wn);
    if (!frozen) {
        if (old2) {
            const uint32_t a2 = sl[(SB + 3) * 32 + lane], db2 = sl[(SB + 4) * 32 + lane] - a2;
            const uint32_t W2 = sl[(SB + 5) * 32 + lane];
#pragma unroll
            for (int j = 0; j < DC; ++j) {                                // + L^(k)_mn - L^(k-2)_mn, exact
                const uint32_t mag = ((W2 << (15 - j)) >> 31) * db2 + a2;    // f(A,B,n,ñ) of iteration k-2
                const float r2 = __uint_as_float(mag ^ ((W2 << (31 - j)) & 0x80000000u));
                atomicAdd((unsigned long long *)(Xat + (size_t)cols[j] * 32 + lane),
                          (unsigned long long)(grid_of(r[j]) - grid_of(r2)));
            }
        } else {
#pragma unroll
            for (int j = 0; j < DC; ++j)                                  // Z^(k)_n += L^(k)_mn, exact
                atomicAdd((unsigned long long *)(Xat + (size_t)cols[j] * 32 + lane), (unsigned long long)grid_of(r[j]));
        }
    }
}

template <bool PAIR, int FMT, bool ES, bool FI, int VM>
__device__ __forceinline__ void pipe_body(const StreamArgs &a, int k) {
    using C = PipeCfg<PAIR>;
    // first fp32 iteration: one line per variable (the fp32 Z^(0) plane), no state
    constexpr int LPV = (!PAIR && FI) ? 1 : C::LPV;
    extern __shared__ __align__(128) uint32_t psm[];
    uint32_t *coltab = psm;                                       // [RB][8]
    uint8_t *dctab = (uint8_t *)(psm + kPipeRB * 8);              // [RB]
    uint32_t *ring = psm + kPipeRB * 8 + kPipeRB / 4;             // [warps][D][lines][32]
    const int tile = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int mb0 = blockIdx.x * kPipeRB;
    const int nrows = min(kPipeRB, a.M - mb0);
    const size_t plane = (size_t)tile * a.N * 32;
    // integer pairs: biased 32-bit words; fp32: int64 grid values (Z^(0): fp32 plane)
    const uint32_t *Lpt = a.Lb[(k - 1) % 3] + plane;
    uint32_t *Lat = a.Lb[k % 3] + plane;
    uint32_t *Lnt = a.Lb[(k + 1) % 3] + plane;
    // fp32 (delta accumulation, pipe_row_f): posterior of iteration k in Lb[k & 1], compact
    // state of iteration k in plane k & 1 (st / st2); the rows read the state of k-1 and of
    // k-2 and overwrite the latter
    long long *Xat = (long long *)a.Lb[k & 1] + plane;
    const char *Lsrc = PAIR ? (const char *)Lpt
                            : (FI ? (const char *)(a.Z0 + plane) : (const char *)((const long long *)a.Lb[(k - 1) & 1] + plane));
    const int nst = PAIR ? StateIO<FMT>::kWords : 3;
    uint32_t *stt = (PAIR ? a.st : ((k & 1) ? a.st2 : a.st)) + (size_t)tile * nst * a.M * 32;   // written (and k-2)
    const uint32_t *stt_prev = (PAIR ? a.st : ((k & 1) ? a.st : a.st2)) + (size_t)tile * nst * a.M * 32;   // k-1
    const bool old2 = !PAIR && k >= 3;
    const size_t sstride = (size_t)a.M * 32;
    // compact row tables of this warp's rows -> its part of shared memory (one 32 B entry
    // per row); warp-local, so no CTA barrier before the row pipeline starts
    for (int i = lane; i < 2 * ((nrows - warp + kPipeWarps - 1) / kPipeWarps); i += 32) {
        const int r = warp + (i >> 1) * kPipeWarps;
        const uint4 v = __ldg(a.rowtab + 2 * (size_t)(mb0 + r) + (i & 1));
        uint4 w = v;
        if ((i & 1) == 0) {
            w.x = v.x & 0x0FFFFFFFu;
            int dc = (int)(v.x >> 28);
            if (dc == 15) dc = __ldg(a.row_ptr + mb0 + r + 1) - __ldg(a.row_ptr + mb0 + r);
            dctab[r] = (uint8_t)dc;
        }
        ((uint4 *)coltab)[2 * r + (i & 1)] = w;
    }
    uint32_t keep = 0;
    bool frozen = false;
    if (ES) {
        const uint32_t d = a.done[tile * 32 + lane];
        if (PAIR) keep = ((d & 1) ? 0x0000FFFFu : 0u) | ((d & 2) ? 0xFFFF0000u : 0u);
        else frozen = (d & 1u) != 0;
    }
    // integer pairs: the accumulator of the next iteration (it held Z^(k-2); not touched
    // otherwise by this launch: no barrier needed); fp32 needs none (delta accumulation)
    if (PAIR && k < a.K) {
        const int wg = blockIdx.x * kPipeWarps + warp, nwg = gridDim.x * kPipeWarps;
        const bool any_frozen = ES && __any_sync(0xFFFFFFFFu, keep != 0);
        if (!any_frozen) {
            stream_init_next(a.Z0 + plane, Lnt, a.N, wg, nwg, lane);
        } else {
            for (int n = wg; n < a.N; n += nwg) {
                const size_t idx = (size_t)n * 32 + lane;
                uint32_t v = __ldcg(a.Z0 + plane + idx);
                if (keep) v = keep_start(v, __ldcg(Lnt + idx), keep, (uint32_t)__ldg(a.coldeg + n));
                __stcg(Lnt + idx, v);
            }
        }
    }
    __syncwarp();
    constexpr bool first_iter = FI;                   // compile-time: no rebuild / state copy in iteration 1
    const int nst_copy = first_iter ? 0 : nst;
    constexpr int D = C::D, LINES = C::LINES;
    uint32_t *wring = ring + (size_t)warp * D * LINES * 32;
    const uint32_t wring_s = (uint32_t)__cvta_generic_to_shared(wring);
    // rows of this warp: warp, warp + W, ...
    int nmy = 0;
    for (int r = warp; r < nrows; r += kPipeWarps) ++nmy;
    // prologue
#pragma unroll
    for (int i = 0; i < D; ++i) {
        if (i < nmy) {
            const int r = warp + i * kPipeWarps;
            pipe_issue_row<LPV, C::SB>(wring_s + (uint32_t)(i * LINES * 128), Lsrc, stt_prev, sstride, coltab + r * 8,
                                       dctab[r], nst_copy, mb0 + r, lane, stt, old2 ? 3 : 0);
        }
        cp_async_commit();
    }
    uint32_t synd = 0;
    // the row loop, for one row degree DCF known to the compiler (every row of this warp has
    // it -- e.g. all but the first block of a DVB-S2-shaped code) or DCF = 0: a switch per row
    auto row_loop = [&](auto dcf_tag) {
        constexpr int DCF = decltype(dcf_tag)::value;
        for (int i = 0; i < nmy; ++i) {
            cp_async_wait<D - 1>();
            __syncwarp();
            const int r = warp + i * kPipeWarps;
            const int m = mb0 + r;
            const int slot = i % D;
            const uint32_t *sl = wring + slot * LINES * 32;
            const uint32_t *cols = coltab + r * 8;
            if constexpr (DCF > 0) {
                if (PAIR) pipe_row_i<DCF, FMT, ES, VM>(a, sl, cols, m, lane, Lat, stt, sstride, first_iter, keep, synd);
                else pipe_row_f<DCF, ES, FI>(a, sl, cols, m, lane, Xat, stt, sstride, frozen, synd, old2);
            } else {
                const int dc = dctab[r];
                if (PAIR) {
                    switch (dc) {
#define LDPC_PI(DD) \
                    case DD: pipe_row_i<DD, FMT, ES, VM>(a, sl, cols, m, lane, Lat, stt, sstride, first_iter, keep, synd); break;
                    LDPC_PI(2) LDPC_PI(3) LDPC_PI(4) LDPC_PI(5) LDPC_PI(6) LDPC_PI(7) LDPC_PI(8)
#undef LDPC_PI
                    }
                } else {
                    switch (dc) {
#define LDPC_PF(DD) \
                    case DD: pipe_row_f<DD, ES, FI>(a, sl, cols, m, lane, Xat, stt, sstride, frozen, synd, old2); break;
                    LDPC_PF(2) LDPC_PF(3) LDPC_PF(4) LDPC_PF(5) LDPC_PF(6) LDPC_PF(7) LDPC_PF(8)
#undef LDPC_PF
                    }
                }
            }
            __syncwarp();                                          // slot consumed before it is refilled
            const int inext = i + D;
            if (inext < nmy) {
                const int rn = warp + inext * kPipeWarps;
                pipe_issue_row<LPV, C::SB>(wring_s + (uint32_t)(slot * LINES * 128), Lsrc, stt_prev, sstride,
                                           coltab + rn * 8, dctab[rn], nst_copy, mb0 + rn, lane, stt, old2 ? 3 : 0);
            }
            cp_async_commit();
        }
    };
    const int dc0 = nmy > 0 ? dctab[warp] : 0;
    const bool uniform = __all_sync(0xFFFFFFFFu, lane >= nmy || dctab[warp + lane * kPipeWarps] == dc0);
    if (uniform && dc0 == 7) row_loop(std::integral_constant<int, 7>{});   // the DVB-S2-shaped codes (cfg4/5)
    else if (uniform && dc0 == 6) row_loop(std::integral_constant<int, 6>{});
    else row_loop(std::integral_constant<int, 0>{});
    cp_async_wait<0>();
    if (ES && synd) atomicOr(a.synd + tile * 32 + lane, synd);
}

// PAIR = true: int16 pairs (V-form accumulators); false: fp32.  The first iteration (no
// previous messages to rebuild, no state to read) is a separate instantiation of the body,
// so rows carry no per-row branch (or if-converted both paths) for it; likewise the
// check-node variant.
template <bool PAIR, int FMT, bool ES>
__global__ void __launch_bounds__(kPipeWarps * 32, LDPC_PIPE_MINB) k_stream_pipe(const StreamArgs a, int k) {
    // Iteration k + 1 is launched as a programmatic dependent of iteration k
    // (stream_launch.cu): its CTAs may be scheduled while k's last CTAs retire, so before
    // touching any plane each CTA waits for the previous grid to complete and its writes
    // to be visible; then it lets the next iteration's grid be scheduled.  Without the
    // launch attribute both instructions are no-ops.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // the integer check-node variant (offset / normalized) of this launch's iteration is a
    // template parameter of the rows as well (fp32 rows take alpha / beta directly)
    if constexpr (!PAIR) {
        if (k == 1) pipe_body<PAIR, FMT, ES, true, 0>(a, k);
        else pipe_body<PAIR, FMT, ES, false, 0>(a, k);
    } else if (a.vk.norm == 0) {
        if (k == 1) pipe_body<PAIR, FMT, ES, true, 0>(a, k);
        else pipe_body<PAIR, FMT, ES, false, 0>(a, k);
    } else {
        if (k == 1) pipe_body<PAIR, FMT, ES, true, 1>(a, k);
        else pipe_body<PAIR, FMT, ES, false, 1>(a, k);
    }
}

template <bool PAIR>
constexpr size_t pipe_smem_bytes() {
    return (size_t)kPipeRB * 8 * 4 + kPipeRB + (size_t)kPipeWarps * PipeCfg<PAIR>::D * PipeCfg<PAIR>::LINES * 128 + 64;
}

}  // namespace ldpc
