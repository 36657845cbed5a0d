// k_twoscan.cuh -- the two-scan min-sum decoder of PAPER.md §3, on the GPU.
//
// This is the baseline the paper's single-scan method is measured against (P:29-30,
// P:70-78).  It keeps BOTH per-edge message arrays the paper
// describes and uses BOTH addressings:
//   check pass  (horizontal scan, Eq.(1), P:150-153 + variant P:178-188): for every
//               row m, read Z_mn for n in N(m) (check->variable addressing) and
//               write L_mn;
//   variable pass (vertical scan, Eq.(2), and the posterior P:164-165):
//               for every column n, read L_mn for m in M(n) (variable->check
//               addressing), form Z_n = Z0_n + sum_m L_mn and the extrinsic
//               Z_mn = Z_n - L_mn, write both.
// Layout: frame-interleaved like the streaming single-scan kernels ([tile][edge][32]
// and [tile][n][32] words), so every access of a warp is one 128-byte line.
// Integer path: two frames per 32-bit word in packed 16x2 form (doubled values,
// exactly as the single-scan kernels); fp32: one frame per lane.  Posteriors go to
// the same rotating biased buffers Lb[k % 3] the streaming single-scan uses, so the
// syndrome / freeze / output kernels are shared.
//
// Reading (DESIGN.md §3 D24): the extrinsic Z_mn is computed as Z_n - L_mn.  In the
// integer modes this equals Eq.(2)'s Z0_n + sum_{m' != m} L_m'n exactly.  fp32 (reading
// D28): the column's sum is exact in int64 on the 2^-34 grid, so Z_n - L_mn is the exact
// sum over m' != m too, each rounded to fp32 once -- bit-exact with the oracle's Eq.(2);
// the posterior planes hold the int64 sums like the fp32 single-scan's.
#pragma once
#include "k_stream.cuh"

namespace ldpc {

constexpr int kTsMaxDV = 16;   // column degree limit of the variable pass (registers)


// Z^(0)_mn = Z^(0)_n for every m in M(n): one warp per (column, tile), one read
// of Z^(0)_n and independent stores to its edges
template <bool PAIR>
__global__ void __launch_bounds__(256) k_ts_init(const StreamArgs a, const TwoScanArgs t) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x >> 5);
    uint32_t *zvt = t.zv + (size_t)tile * t.E * 32;
    for (int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < a.N; n += nw) {
        uint32_t v = __ldcg(a.Z0 + ((size_t)tile * a.N + n) * 32 + lane);
        if (PAIR) v = vadd(v, 0xC000C000u);              // unbias (ingest with zpre = 0)
        const int b0 = __ldg(t.vptr + n), b1 = __ldg(t.vptr + n + 1);
        for (int b = b0; b < b1; ++b) __stcg(zvt + (size_t)__ldg(t.vedge + b) * 32 + lane, v);
    }
}

// hard-decision ballots of the posterior word just written for column n (lane 0 stores)
template <bool PAIR>
__device__ __forceinline__ void ts_store_hb(const StreamArgs &a, uint32_t *hbt, int n, uint32_t out, int lane) {
    if (PAIR) {
        const uint32_t p = fadd32(out, kParBiased, a.rk);   // sign bits 15 / 31 = [Z <= 0] per frame
        const uint32_t lo = __ballot_sync(0xFFFFFFFFu, (p & 0x8000u) != 0);
        const uint32_t hi = __ballot_sync(0xFFFFFFFFu, (p & 0x80000000u) != 0);
        if (lane == 0) ((uint2 *)hbt)[n] = make_uint2(lo, hi);
    } else {
        const uint32_t h = __ballot_sync(0xFFFFFFFFu, out != 0u);   // fp32: out = [Z <= 0]
        if (lane == 0) hbt[n] = h;
    }
}

// syndrome of the posterior of the last variable pass from the ballots: one thread per
// (row, tile), reading 8 (fp32: 4) bytes per edge instead of a 128-byte posterior line
template <bool PAIR>
__global__ void __launch_bounds__(256) k_ts_syndrome(const StreamArgs a, const TwoScanArgs t) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t xl = 0, xh = 0;
    if (m < a.M) {
        const int e0 = __ldg(a.row_ptr + m), e1 = __ldg(a.row_ptr + m + 1);
        if (PAIR) {
            const uint2 *hbt = (const uint2 *)t.hb + (size_t)tile * a.N;
            for (int e = e0; e < e1; ++e) {
                const uint2 v = __ldcg(hbt + __ldg(a.col_idx + e));
                xl ^= v.x;
                xh ^= v.y;
            }
        } else {
            const uint32_t *hbt = t.hb + (size_t)tile * a.N;
            for (int e = e0; e < e1; ++e) xl ^= __ldcg(hbt + __ldg(a.col_idx + e));
        }
    }
    xl = __reduce_or_sync(0xFFFFFFFFu, xl);              // frames (lanes) failing some row of this warp
    xh = __reduce_or_sync(0xFFFFFFFFu, xh);
    const uint32_t s = PAIR ? ((((xl >> lane) & 1u) << 15) | (((xh >> lane) & 1u) << 31)) : ((xl >> lane) & 1u);
    if (s) atomicOr(a.synd + tile * 32 + lane, s);
}

template <int DC, bool PAIR>
__device__ __forceinline__ void ts_check_row(const StreamArgs &a, const TwoScanArgs &t, const uint32_t *zvt,
                                             uint32_t *msgt, int64_t e0, int lane) {
    uint32_t z[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) z[j] = __ldcg(zvt + (e0 + j) * 32 + lane);
    uint32_t r[DC];
    if (PAIR) {
        RowState st;
        new_state<DC>(z, a.vk, st, r, a.rk);   // Eq.(1) + offset/clamp; state unused
    } else {
        float zf[DC], rf[DC], A, B;
        uint32_t W;
#pragma unroll
        for (int j = 0; j < DC; ++j) zf[j] = __uint_as_float(z[j]);
        f32_row<DC>(zf, true, 0.f, 0.f, 0u, a.alpha, a.beta, A, B, W, rf);
#pragma unroll
        for (int j = 0; j < DC; ++j) r[j] = __float_as_uint(rf[j]);
    }
#pragma unroll
    for (int j = 0; j < DC; ++j) __stcg(msgt + (e0 + j) * 32 + lane, r[j]);
}

// horizontal scan: one warp per (row, tile)
template <bool PAIR>
__global__ void __launch_bounds__(256) k_ts_check(const StreamArgs a, const TwoScanArgs t) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const uint32_t *zvt = t.zv + (size_t)tile * t.E * 32;
    uint32_t *msgt = t.msg + (size_t)tile * t.E * 32;
    const int nw = gridDim.x * (blockDim.x >> 5);
    for (int m = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); m < a.M; m += nw) {
        const int64_t e0 = __ldg(a.row_ptr + m);
        const int dc = __ldg(a.row_ptr + m + 1) - (int)e0;
        switch (dc) {
        case 2: ts_check_row<2, PAIR>(a, t, zvt, msgt, e0, lane); break;
        case 3: ts_check_row<3, PAIR>(a, t, zvt, msgt, e0, lane); break;
        case 4: ts_check_row<4, PAIR>(a, t, zvt, msgt, e0, lane); break;
        case 5: ts_check_row<5, PAIR>(a, t, zvt, msgt, e0, lane); break;
        case 6: ts_check_row<6, PAIR>(a, t, zvt, msgt, e0, lane); break;
        case 7: ts_check_row<7, PAIR>(a, t, zvt, msgt, e0, lane); break;
        case 8: ts_check_row<8, PAIR>(a, t, zvt, msgt, e0, lane); break;
        }
    }
}

// vertical scan + posterior of one column n with DV = |M(n)| edges (registers sized by
// the column degree: the degree-16 worst case would cap occupancy for every column)
template <int DV, bool PAIR, bool ES>
__device__ __forceinline__ void ts_var_col(const StreamArgs &a, const TwoScanArgs &t, const uint32_t *msgt,
                                           uint32_t *zvt, uint32_t *post, const uint32_t *z0t, uint32_t *hbt, int n,
                                           int b0, int lane, uint32_t keep) {
    int32_t eid[DV];
    uint32_t mv[DV];
#pragma unroll
    for (int b = 0; b < DV; ++b) {
        eid[b] = __ldg(t.vedge + b0 + b);
        LDPC_CHECK(eid[b] >= 0 && eid[b] < t.E);
    }
    const size_t ni = (size_t)n * 32 + lane;
    uint32_t Z = __ldcg(z0t + ni);
#pragma unroll
    for (int b = 0; b < DV; ++b) mv[b] = __ldcg(msgt + (size_t)eid[b] * 32 + lane);
    if (PAIR) {
        Z = vadd(Z, 0xC000C000u);                         // unbias
#pragma unroll
        for (int b = 0; b < DV; ++b) Z = vadd(Z, mv[b]);
#pragma unroll
        for (int b = 0; b < DV; ++b) __stcg(zvt + (size_t)eid[b] * 32 + lane, vadd(Z, vneg(mv[b], a.rk)));   // Eq.(2)
        uint32_t out = vadd(Z, kPairBias);                // biased posterior words (k_stream.cuh)
        if (ES && keep) out = sel(keep, __ldcg(post + ni), out);
        __stcg(post + ni, out);
        if (ES) ts_store_hb<true>(a, hbt, n, out, lane);
    } else {
        long long g[DV];
        long long X = grid_of(__uint_as_float(Z));                     // exact sums (reading D28)
#pragma unroll
        for (int b = 0; b < DV; ++b) {
            g[b] = grid_of(__uint_as_float(mv[b]));
            X += g[b];                                                 // Z_n
        }
#pragma unroll
        for (int b = 0; b < DV; ++b)                                   // Eq.(2): sum over m' != m
            __stcg(zvt + (size_t)eid[b] * 32 + lane, __float_as_uint(val_of(X - g[b])));
        if (!(ES && keep)) __stcg((long long *)post + ni, X);
        if (ES) ts_store_hb<false>(a, hbt, n, X <= 0 ? 1u : 0u, lane);
    }
}

// columns of degree > 8: two passes over the edges (sum, then extrinsics) instead of
// register arrays, so the rare high-degree columns do not set the kernel's register count
template <bool PAIR, bool ES>
__device__ __noinline__ void ts_var_col_wide(const StreamArgs &a, const TwoScanArgs &t, const uint32_t *msgt,
                                             uint32_t *zvt, uint32_t *post, const uint32_t *z0t, uint32_t *hbt, int n,
                                             int b0, int dv, int lane, uint32_t keep) {
    const size_t ni = (size_t)n * 32 + lane;
    uint32_t Z = __ldcg(z0t + ni);
    long long X = PAIR ? 0 : grid_of(__uint_as_float(Z));               // fp32: exact sums (D28)
    if (PAIR) Z = vadd(Z, 0xC000C000u);
    for (int b = 0; b < dv; ++b) {
        const uint32_t m = __ldcg(msgt + (size_t)__ldg(t.vedge + b0 + b) * 32 + lane);
        if (PAIR) Z = vadd(Z, m);
        else X += grid_of(__uint_as_float(m));
    }
    for (int b = 0; b < dv; ++b) {
        const size_t ei = (size_t)__ldg(t.vedge + b0 + b) * 32 + lane;
        const uint32_t m = __ldcg(msgt + ei);
        __stcg(zvt + ei, PAIR ? vadd(Z, vneg(m, a.rk)) : __float_as_uint(val_of(X - grid_of(__uint_as_float(m)))));
    }
    if (PAIR) {
        uint32_t out = vadd(Z, kPairBias);
        if (ES && keep) out = sel(keep, __ldcg(post + ni), out);
        __stcg(post + ni, out);
        if (ES) ts_store_hb<true>(a, hbt, n, out, lane);
    } else {
        if (!(ES && keep)) __stcg((long long *)post + ni, X);
        if (ES) ts_store_hb<false>(a, hbt, n, X <= 0 ? 1u : 0u, lane);
    }
}

// vertical scan + posterior of iteration k: one warp per (column, tile).  Frames
// frozen by early stop keep their posterior buffer (Lb[k % 3] is also the buffer of
// iteration k - 3).
// DVMAX (4 or 8): largest column degree handled with register arrays; the kernel's
// register count follows it, so codes with max_dv <= 4 get the smaller, higher-occupancy
// instantiation
template <bool PAIR, bool ES, int DVMAX>
__global__ void __launch_bounds__(256) k_ts_var(const StreamArgs a, const TwoScanArgs t, int k) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const uint32_t *msgt = t.msg + (size_t)tile * t.E * 32;
    uint32_t *zvt = t.zv + (size_t)tile * t.E * 32;
    // integer pairs: biased words; fp32: int64 grid sums (ts_var_col casts)
    uint32_t *post = PAIR ? a.Lb[k % 3] + (size_t)tile * a.N * 32
                          : (uint32_t *)((long long *)a.Lb[k % 3] + (size_t)tile * a.N * 32);
    const uint32_t *z0t = a.Z0 + (size_t)tile * a.N * 32;
    uint32_t *hbt = t.hb + (size_t)tile * a.N * (PAIR ? 2 : 1);
    uint32_t keep = 0;
    if (ES) {
        const uint32_t d = a.done[tile * 32 + lane];
        keep = PAIR ? (((d & 1) ? 0x0000FFFFu : 0u) | ((d & 2) ? 0xFFFF0000u : 0u)) : ((d & 1) ? 0xFFFFFFFFu : 0u);
    }
    const int nw = gridDim.x * (blockDim.x >> 5);
    for (int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < a.N; n += nw) {
        const int b0 = __ldg(t.vptr + n), dv = __ldg(t.vptr + n + 1) - b0;
#define LDPC_TS_COL(D) \
    case D: ts_var_col<D, PAIR, ES>(a, t, msgt, zvt, post, z0t, hbt, n, b0, lane, keep); break;
        if (DVMAX <= 4) {
            switch (dv) {
                LDPC_TS_COL(1) LDPC_TS_COL(2) LDPC_TS_COL(3) LDPC_TS_COL(4)
            default: ts_var_col_wide<PAIR, ES>(a, t, msgt, zvt, post, z0t, hbt, n, b0, dv, lane, keep);
            }
        } else {
            switch (dv) {
                LDPC_TS_COL(1) LDPC_TS_COL(2) LDPC_TS_COL(3) LDPC_TS_COL(4) LDPC_TS_COL(5) LDPC_TS_COL(6)
                LDPC_TS_COL(7) LDPC_TS_COL(8)
            default: ts_var_col_wide<PAIR, ES>(a, t, msgt, zvt, post, z0t, hbt, n, b0, dv, lane, keep);
            }
        }
#undef LDPC_TS_COL
    }
}

// Message export (ldpc_decode_batch_messages): the check messages L_mn of the last
// horizontal scan, [tile][E][32] -> [nframes][E] (integer: doubled 16x2 pairs, halved)
template <bool PAIR>
__global__ void __launch_bounds__(256) k_ts_export(const StreamArgs a, const TwoScanArgs t) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const uint32_t *msgt = t.msg + (size_t)tile * t.E * 32;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < t.E; e += nw) {
        const uint32_t v = __ldcg(msgt + e * 32 + lane);
        if (PAIR) {
            const int f = tile * 64 + 2 * lane;
            if (f < a.nframes) ((int16_t *)a.msg_out)[(size_t)f * t.E + e] = (int16_t)(lo16(v) / 2);
            if (f + 1 < a.nframes) ((int16_t *)a.msg_out)[(size_t)(f + 1) * t.E + e] = (int16_t)(hi16(v) / 2);
        } else {
            const int f = tile * 32 + lane;
            if (f < a.nframes) ((float *)a.msg_out)[(size_t)f * t.E + e] = __uint_as_float(v);
        }
    }
}

}  // namespace ldpc
