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
// integer modes this equals Eq.(2)'s Z0_n + sum_{m' != m} L_m'n exactly; in fp32 it is
// one rounding away from the ordered sum (checked against the oracle's Eq.(2) within
// the BASELINE fp32 tolerance).
#pragma once
#include "k_stream.cuh"

namespace ldpc {

constexpr int kTsMaxDV = 16;   // column degree limit of the variable pass (registers)


// Z^(0)_mn = Z^(0)_n for every m in M(n)
template <bool PAIR>
__global__ void __launch_bounds__(256) k_ts_init(const StreamArgs a, const TwoScanArgs t) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t e = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); e < t.E; e += nw) {
        const int n = __ldg(t.ecol + e);
        uint32_t v = __ldcg(a.Z0 + ((size_t)tile * a.N + n) * 32 + lane);
        if (PAIR) v = vadd(v, 0xC000C000u);              // unbias (ingest with zpre = 0)
        __stcg(t.zv + ((size_t)tile * t.E + e) * 32 + lane, v);
    }
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

// vertical scan + posterior of iteration k: one warp per (column, tile).  Frames
// frozen by early stop keep their posterior buffer (Lb[k % 3] is also the buffer of
// iteration k - 3).
template <bool PAIR, bool ES>
__global__ void __launch_bounds__(256) k_ts_var(const StreamArgs a, const TwoScanArgs t, int k) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const uint32_t *msgt = t.msg + (size_t)tile * t.E * 32;
    uint32_t *zvt = t.zv + (size_t)tile * t.E * 32;
    uint32_t *post = a.Lb[k % 3] + (size_t)tile * a.N * 32;
    uint32_t keep = 0;
    if (ES) {
        const uint32_t d = a.done[tile * 32 + lane];
        keep = PAIR ? (((d & 1) ? 0x0000FFFFu : 0u) | ((d & 2) ? 0xFFFF0000u : 0u)) : ((d & 1) ? 0xFFFFFFFFu : 0u);
    }
    const int nw = gridDim.x * (blockDim.x >> 5);
    for (int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < a.N; n += nw) {
        const int b0 = __ldg(t.vptr + n), dv = __ldg(t.vptr + n + 1) - b0;
        int32_t eid[kTsMaxDV];
        uint32_t mv[kTsMaxDV];
#pragma unroll
        for (int b = 0; b < kTsMaxDV; ++b) {
            if (b < dv) {
                eid[b] = __ldg(t.vedge + b0 + b);
                mv[b] = __ldcg(msgt + (size_t)eid[b] * 32 + lane);
            }
        }
        const size_t ni = (size_t)n * 32 + lane;
        uint32_t Z = __ldcg(a.Z0 + (size_t)tile * a.N * 32 + ni);
        if (PAIR) {
            Z = vadd(Z, 0xC000C000u);                     // unbias
#pragma unroll
            for (int b = 0; b < kTsMaxDV; ++b)
                if (b < dv) Z = vadd(Z, mv[b]);
#pragma unroll
            for (int b = 0; b < kTsMaxDV; ++b)
                if (b < dv) __stcg(zvt + (size_t)eid[b] * 32 + lane, vadd(Z, vneg(mv[b], a.rk)));   // Eq.(2)
            uint32_t out = vadd(Z, kPairBias);            // biased posterior words (k_stream.cuh)
            if (ES && keep) out = sel(keep, __ldcg(post + ni), out);
            __stcg(post + ni, out);
        } else {
            float Zf = __uint_as_float(Z);
#pragma unroll
            for (int b = 0; b < kTsMaxDV; ++b)
                if (b < dv) Zf = __fadd_rn(Zf, __uint_as_float(mv[b]));      // ascending m
#pragma unroll
            for (int b = 0; b < kTsMaxDV; ++b)
                if (b < dv) __stcg(zvt + (size_t)eid[b] * 32 + lane, __float_as_uint(__fsub_rn(Zf, __uint_as_float(mv[b]))));
            if (!(ES && keep)) __stcg(post + ni, __float_as_uint(Zf));
        }
    }
}

}  // namespace ldpc
