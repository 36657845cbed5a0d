// k_stream.cuh -- streaming single-scan min-sum kernels for long codes.
//
// Used when one frame pair's posterior double buffer does not fit in shared
// memory (e.g. N = 64800).  Frames are tiled TILE-wide and stored
// frame-interleaved ([tile][n][lane], 128 B per variable per warp) so every
// gather, state access and accumulation of a warp is one coalesced 128-byte
// line.  One launch per iteration; a warp processes whole check rows for the
// 32 lanes of its tile using only check->variable addressing (PAPER.md
// P:219-224); Z^(k)_n += L^(k)_mn is a coalesced global reduction
// (RED) into an accumulator that was initialised to Z^(0)_n by the previous
// iteration's launch (three rotating posterior buffers: read Z^(k-1),
// accumulate Z^(k), initialise the buffer for Z^(k+1)).
//
// Integer path: two frames per lane (16x2 SIMD).  Posterior words hold 2Z + 0x4000 per
// lane (non-negative lanes: the packed and the 32-bit "V form" hi*65536+lo coincide),
// messages are added by a 32-bit RED as V(L) + 0x8000 (rowcore new_state<B8>) and each
// accumulator starts d_v(n) * 0x8000 lower (the Z^(0) plane holds that start value), so
// the sums are exact and the gathers read the words directly -- the same representation
// as the barrier-free resident kernel (reading D26).  fp32 path: one frame per lane; the
// posterior planes hold the exact sums of reading D28 as int64 values on the 2^-34 grid
// (64-bit integer RED, order-free), read back as fl32(X 2^-34); the Z^(0) plane is fp32.
#pragma once
#include "args.cuh"
#include "rowcore.cuh"
#include "rowcore_f32.cuh"

namespace ldpc {

constexpr uint32_t kPairBias = 0x40004000u;      // 0x4000 per 16-bit lane
constexpr uint32_t kParBiased = 0xBFFEBFFFu;     // row_parity constant for biased words

// fp32 posteriors (reading D28): a sum of messages is exact on the grid 2^-34 (int64) and
// rounded to fp32 once when read.  Terms are saturated to +-2^20 (channel LLRs on ingest,
// message magnitudes in the row core), so the scaling by 2^34 is exact and sums of up to
// 255 terms stay far inside int64.
constexpr float kSatF = 1048576.0f;
__device__ __forceinline__ long long grid_of(float x) { return __float2ll_rn(x * 0x1p34f); }
__device__ __forceinline__ float val_of(long long X) { return __ll2float_rn(X) * 0x1p-34f; }

// Early stop: frozen lanes (mask `keep`) must come out of an accumulation unchanged.
// Every edge always adds 0x8000 to the low lane -- V(L) + 0x8000 for active lanes, a bare
// 0x8000 for a frozen low lane (red_value) -- so every accumulator start is lowered by
// d_v 0x8000 whatever the lanes' state, and a frame frozen between the start and the
// accumulation cannot upset the other lane.  Start word: frozen lanes keep `old`, active
// lanes restart from Z^(0) (P0 = start + d_v 0x8000).
__device__ __forceinline__ uint32_t keep_start(uint32_t start, uint32_t old, uint32_t keep, uint32_t dv) {
    return sel(keep, old, start + dv * 0x8000u) - dv * 0x8000u;
}
__device__ __forceinline__ uint32_t red_value(uint32_t rn, uint32_t keep) { return sel(keep, 0x00008000u, rn); }

// -------------------------------------------------------------- integer path
// ingest: user [F][N] -> doubled, saturated, biased words P0 = 2Z^(0) + 0x4000 per lane.
// Lb[0] = P0 (the posterior read by iteration 1); Z0 plane = Lb[1] = P0 - d_v 0x8000 (the
// accumulator start, see above).  zpre = 0 (two-scan): Z0 plane = P0.
template <typename TIN>
__global__ void k_stream_ingest_i(const StreamArgs a, int zpre) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const int f0 = tile * 64 + 2 * lane, f1 = f0 + 1;
    const TIN *llr = (const TIN *)a.llr;
    for (int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < a.N; n += gridDim.x * (blockDim.x >> 5)) {
        int zl = 0, zh = 0;
        if (f0 < a.nframes) zl = max(-a.Qsat, min(a.Qsat, (int)llr[(size_t)f0 * a.N + n]));
        if (f1 < a.nframes) zh = max(-a.Qsat, min(a.Qsat, (int)llr[(size_t)f1 * a.N + n]));
        const uint32_t v = pack2(2 * zl + 0x4000, 2 * zh + 0x4000);
        const uint32_t start = zpre ? v - (uint32_t)__ldg(a.coldeg + n) * 0x8000u : v;
        const size_t idx = ((size_t)tile * a.N + n) * 32 + lane;
        a.Z0[idx] = start;
        a.Lb[0][idx] = v;
        a.Lb[1][idx] = start;
    }
}

struct RowT {
    uint32_t c[8];
    int dc;
};
__device__ __forceinline__ RowT load_rowt(const uint4 *rt, int m, int M) {
    RowT r;
    if (m < M) {
        const uint4 x = __ldg(rt + 2 * m), y = __ldg(rt + 2 * m + 1);
        r.c[0] = x.x & 0x0FFFFFFFu; r.c[1] = x.y; r.c[2] = x.z; r.c[3] = x.w;
        r.c[4] = y.x; r.c[5] = y.y; r.c[6] = y.z; r.c[7] = y.w;
        r.dc = (int)(x.x >> 28);
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) r.c[j] = 0;
        r.dc = 0;
    }
    return r;
}

// Copy Z^(0) of this tile into the accumulator of the next iteration with 128-bit
// loads/stores, 4 in flight per thread (contiguous [n][32] plane segment of the tile).
__device__ __forceinline__ void stream_init_next(const uint32_t *Z0t, uint32_t *Lnt, int N, int wg, int nwg, int lane) {
    const uint4 *src = (const uint4 *)Z0t;
    uint4 *dst = (uint4 *)Lnt;
    const int total = N * 8;                     // uint4 per tile plane
    const int step = nwg * 32;
    int i = wg * 32 + lane;
    for (; i + 3 * step < total; i += 4 * step) {
        const uint4 v0 = __ldcg(src + i), v1 = __ldcg(src + i + step), v2 = __ldcg(src + i + 2 * step),
                    v3 = __ldcg(src + i + 3 * step);
        __stcg(dst + i, v0);
        __stcg(dst + i + step, v1);
        __stcg(dst + i + 2 * step, v2);
        __stcg(dst + i + 3 * step, v3);
    }
    for (; i < total; i += step) __stcg(dst + i, __ldcg(src + i));
}

// NR check rows of one tile (two frames per lane), all loads issued before any compute.
template <int DC, int NR, int FMT, bool ES>
__device__ __forceinline__ void stream_rows_i(const StreamArgs &a, int lane, const int (&m)[NR], const RowT *rt,
                                              const uint32_t *Lpt, uint32_t *Lat, uint32_t *stt, bool first_iter,
                                              uint32_t keep, uint32_t &synd) {
    uint32_t off[NR][DC];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            LDPC_CHECK(rt[r].c[j] < (uint32_t)a.N && m[r] < a.M);
            off[r][j] = rt[r].c[j] * 32u + (uint32_t)lane;
        }
    const size_t sstride = (size_t)a.M * 32;
    RowState st[NR];
    if (!first_iter) {
#pragma unroll
        for (int r = 0; r < NR; ++r) st[r] = StateIO<FMT>::load(stt + lane, sstride, (size_t)m[r] * 32);
    }
    uint32_t L[NR][DC];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int j = 0; j < DC; ++j) L[r][j] = __ldcg(Lpt + off[r][j]);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        if (ES) synd |= row_parity<DC>(L[r], a.rk, kParBiased);
        uint32_t q[DC];                                   // q + 0x8000 per lane
        if (first_iter) {
#pragma unroll
            for (int j = 0; j < DC; ++j) q[j] = fadd32(L[r][j], kPairBias, a.rk);
        } else {
            rebuild_q_b8<DC>(L[r], st[r], q, a.rk);
        }
        uint32_t rn[DC];                                  // V(L^(k)_mn) + 0x8000
        new_state<DC, true, -1, FMT == FMT_1BIT>(q, a.vk, st[r], rn, a.rk);
        StateIO<FMT>::store(stt + lane, sstride, (size_t)m[r] * 32, st[r]);
#pragma unroll
        for (int j = 0; j < DC; ++j) atomicAdd(Lat + off[r][j], red_value(rn[j], keep));
    }
}

template <int NR, int FMT, bool ES>
__device__ __forceinline__ void stream_dispatch_i(int dc, const StreamArgs &a, int lane, const int (&m)[NR],
                                                  const RowT *rt, const uint32_t *Lpt, uint32_t *Lat,
                                                  uint32_t *stt, bool first_iter, uint32_t keep, uint32_t &synd) {
    switch (dc) {
    case 2: stream_rows_i<2, NR, FMT, ES>(a, lane, m, rt, Lpt, Lat, stt, first_iter, keep, synd); break;
    case 3: stream_rows_i<3, NR, FMT, ES>(a, lane, m, rt, Lpt, Lat, stt, first_iter, keep, synd); break;
    case 4: stream_rows_i<4, NR, FMT, ES>(a, lane, m, rt, Lpt, Lat, stt, first_iter, keep, synd); break;
    case 5: stream_rows_i<5, NR, FMT, ES>(a, lane, m, rt, Lpt, Lat, stt, first_iter, keep, synd); break;
    case 6: stream_rows_i<6, NR, FMT, ES>(a, lane, m, rt, Lpt, Lat, stt, first_iter, keep, synd); break;
    case 7: stream_rows_i<7, NR, FMT, ES>(a, lane, m, rt, Lpt, Lat, stt, first_iter, keep, synd); break;
    case 8: stream_rows_i<8, NR, FMT, ES>(a, lane, m, rt, Lpt, Lat, stt, first_iter, keep, synd); break;
    }
}

// Register version of the integer iteration kernel (rows of degree > 8 are rejected for
// integer LLRs, so this serves LDPC_PIPE=0 runs -- the pipelined kernel's cross-check).
template <int FMT, bool ES>
__global__ void __launch_bounds__(256, 3) k_stream_iter_i(const StreamArgs a, int k) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nwg = gridDim.x * (blockDim.x >> 5);
    const size_t plane = (size_t)tile * a.N * 32;
    const uint32_t *Lpt = a.Lb[(k - 1) % 3] + plane;
    uint32_t *Lat = a.Lb[k % 3] + plane;
    uint32_t *Lnt = a.Lb[(k + 1) % 3] + plane;
    uint32_t *stt = a.st + (size_t)tile * StateIO<FMT>::kWords * a.M * 32;
    uint32_t keep = 0;                                   // 0xFFFF halves: frame frozen
    if (ES) {
        const uint32_t d = a.done[tile * 32 + lane];
        keep = ((d & 1) ? 0x0000FFFFu : 0u) | ((d & 2) ? 0xFFFF0000u : 0u);
        // no early exit for fully frozen warps: the accumulators started one iteration
        // ahead still need their d_v 0x8000 (keep_start / red_value)
    }
    // initialise the accumulator of the next iteration (it held Z^(k-2))
    if (k < a.K) {
        if (!ES || !__any_sync(0xFFFFFFFFu, keep != 0)) {
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
    uint32_t synd = 0;
    const bool first_iter = (k == 1);
    for (int m = wg; m < a.M; m += nwg) {
        const RowT rt = load_rowt(a.rowtab, m, a.M);
        const int mm[1] = {m};
        stream_dispatch_i<1, FMT, ES>(rt.dc, a, lane, mm, &rt, Lpt, Lat, stt, first_iter, keep, synd);
    }
    if (ES && synd) atomicOr(a.synd + tile * 32 + lane, synd);
}

// syndrome of the posterior after iteration k (Z^(0) for k = 0): the final check, and the
// two-scan's per-iteration check.  fp32: Z^(0) is the fp32 plane, later posteriors the
// int64 grid planes ([Z <= 0] = [X <= 0]).
template <bool PAIR>
__global__ void __launch_bounds__(256) k_stream_syndrome(const StreamArgs a, int k) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nwg = gridDim.x * (blockDim.x >> 5);
    const uint32_t *Lp = a.Lb[k % 3];
    const long long *Xp = (const long long *)a.Lb[a.f32delta ? (k & 1) : k % 3];
    uint32_t synd = 0;
    for (int m = wg; m < a.M; m += nwg) {
        const int e0 = __ldg(a.row_ptr + m), e1 = __ldg(a.row_ptr + m + 1);
        uint32_t p = 0;
        for (int e = e0; e < e1; ++e) {
            const size_t idx = ((size_t)tile * a.N + __ldg(a.col_idx + e)) * 32 + lane;
            if (PAIR) p ^= fadd32(__ldcg(Lp + idx), kParBiased, a.rk);
            else if (k == 0) p ^= (__uint_as_float(__ldcg(a.Z0 + idx)) <= 0.0f) ? 1u : 0u;
            else p ^= (__ldcg(Xp + idx) <= 0) ? 1u : 0u;
        }
        synd |= PAIR ? (p & 0x80008000u) : (p & 1u);
    }
    if (synd) atomicOr(a.synd + tile * 32 + lane, synd);
}

// early-stop bookkeeping after iteration k: frames whose Z^(k-1) passed the
// syndrome test are frozen with iterations_used = k-1.
template <bool PAIR>
__global__ void k_stream_freeze(const StreamArgs a, int k) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.ntiles * 32) return;
    const uint32_t s = a.synd[i];
    uint32_t d = a.done[i];
    const int tile = i >> 5, lane = i & 31;
    if (PAIR) {
        for (int h = 0; h < 2; ++h) {
            const int f = tile * 64 + 2 * lane + h;
            const bool fail = h ? (s & 0x80000000u) : (s & 0x8000u);
            if (!(d & (1u << h)) && !fail && f < a.nframes) {
                d |= 1u << h;
                a.it_ws[f] = k - 1;
                a.ok_ws[f] = 1;
            }
        }
    } else {
        const int f = tile * 32 + lane;
        if (!(d & 1) && !(s & 1) && f < a.nframes) { d |= 1; a.it_ws[f] = k - 1; a.ok_ws[f] = 1; }
    }
    a.done[i] = d;
    a.synd[i] = 0;
}

// outputs: frame-major posteriors and hard bits from the tiled buffers.  A block
// handles one tile x 32 variables, transposing through shared memory.
template <bool PAIR>
__global__ void __launch_bounds__(256) k_stream_output(const StreamArgs a) {
    __shared__ uint32_t sh[32][33];
    __shared__ uint32_t sh2[32][33];
    const int tile = blockIdx.y, n0 = blockIdx.x * 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;   // 8 warps
    const int tw = PAIR ? 64 : 32;
    // stage: sh[v][lane] = value of variable n0+v for the tile's lane (per-frame buffer choice)
    for (int v = warp; v < 32; v += 8) {
        const int n = n0 + v;
        uint32_t val = 0, val2 = 0;
        if (n < a.N) {
            const size_t idx = ((size_t)tile * a.N + n) * 32 + lane;
            if (PAIR) {
                const int f0 = tile * 64 + 2 * lane;
                const int k0 = f0 < a.nframes ? a.it_ws[f0] : a.K;
                const int k1 = f0 + 1 < a.nframes ? a.it_ws[f0 + 1] : a.K;
                val = vadd(__ldcg(a.Lb[a.layered ? 0 : k0 % 3] + idx), 0xC000C000u);    // unbias
                val2 = vadd(__ldcg(a.Lb[a.layered ? 0 : k1 % 3] + idx), 0xC000C000u);
                val = (val & 0xFFFFu) | (val2 & 0xFFFF0000u);
            } else {
                const int f = tile * 32 + lane;
                const int kk = f < a.nframes ? a.it_ws[f] : a.K;
                const int kb = a.f32delta ? (kk & 1) : kk % 3;
                if (a.layered) val = __ldcg(a.Lb[0] + idx);               // plain fp32 (D25 / D11)
                else val = kk == 0 ? __ldcg(a.Z0 + idx) : __float_as_uint(val_of(__ldcg((const long long *)a.Lb[kb] + idx)));
            }
        }
        sh[v][lane] = val;
        (void)sh2;
    }
    __syncthreads();
    // each warp handles frames; lane = variable offset
    for (int fl = warp; fl < tw; fl += 8) {
        const int f = tile * tw + fl;
        if (f >= a.nframes) continue;
        const int n = n0 + lane;
        bool hb = false;
        if (PAIR) {
            const uint32_t w = sh[lane][fl >> 1];
            const int v = (fl & 1) ? hi16(w) : lo16(w);
            hb = v <= 0;
            if (n < a.N && a.post) ((int16_t *)a.post)[(size_t)f * a.N + n] = (int16_t)(v >> 1);
        } else {
            const float v = __int_as_float(sh[lane][fl]);
            hb = v <= 0.0f;
            if (n < a.N && a.post) ((float *)a.post)[(size_t)f * a.N + n] = v;
        }
        const uint32_t word = __ballot_sync(0xFFFFFFFFu, hb && n < a.N);
        if (lane == 0) a.hard_bits[(size_t)f * a.wpf + blockIdx.x] = word;
        if (blockIdx.x == 0 && lane == 0) {
            a.ok[f] = a.ok_ws[f];
            if (a.iters) a.iters[f] = a.it_ws[f];
        }
    }
}

// Message export (ldpc_decode_batch_messages): the exit messages L_mn rebuilt from each
// row's persistent state, one warp per (row, tile), lane = frame pair
// (integer) or frame (fp32); messages [nframes][E] in CSR edge order (int16 raw units /
// float).  Integer state: doubled magnitudes A, B and the byte-interleaved W of rowcore.cuh;
// fp32 state: A, B and W = sign bits | one-hot ñ at bit 16 + position (rowcore_f32.cuh).
template <bool PAIR, int FMT>
__global__ void __launch_bounds__(256) k_stream_export(const StreamArgs a) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const int nst = PAIR ? StateIO<FMT>::kWords : 3;
    // fp32 delta accumulation: the state of iteration K is in plane K & 1
    const uint32_t *stt = (!PAIR && a.f32delta && (a.K & 1) ? a.st2 : a.st) + (size_t)tile * nst * a.M * 32;
    const size_t ss = (size_t)a.M * 32;
    const int nwg = gridDim.x * (blockDim.x >> 5);
    for (int m = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); m < a.M; m += nwg) {
        const int64_t e0 = __ldg(a.row_ptr + m);
        const int dc = __ldg(a.row_ptr + m + 1) - (int)e0;
        if (PAIR) {
            const RowState st = StateIO<FMT>::load(stt + lane, ss, (size_t)m * 32);
            for (int fr = 0; fr < 2; ++fr) {
                const int f = tile * 64 + 2 * lane + fr;
                if (f >= a.nframes) break;
                LDPC_CHECK(e0 + dc <= a.E);
                int16_t *out = (int16_t *)a.msg_out + (size_t)f * a.E + e0;
                for (int j = 0; j < dc; ++j) {
                    const uint32_t wb = st.W >> (16 * fr);     // W layout: rowcore.cuh header
                    const bool neg = (wb >> j) & 1u, isidx = (wb >> (8 + j)) & 1u;
                    const int mag = (int)(((isidx ? st.B : st.A) >> (16 * fr)) & 0xFFFFu);
                    out[j] = (int16_t)((neg ? -mag : mag) / 2);
                }
            }
        } else {
            const int f = tile * 32 + lane;
            if (f >= a.nframes) continue;
            const size_t so = (size_t)m * 32 + lane;
            const uint32_t A = __ldcg(stt + so), B = __ldcg(stt + ss + so), W = __ldcg(stt + 2 * ss + so);
            float *out = (float *)a.msg_out + (size_t)f * a.E + e0;
            for (int j = 0; j < dc; ++j) {
                const uint32_t mag = ((W >> (16 + j)) & 1u) ? B : A;
                out[j] = __uint_as_float(mag ^ (((W >> j) & 1u) << 31));
            }
        }
    }
}

// frames not frozen by early stop: iterations = K, ok from the final syndrome
template <bool PAIR>
__global__ void k_stream_finalize_flags(const StreamArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.ntiles * 32) return;
    const uint32_t s = a.synd[i], d = a.done[i];
    const int tile = i >> 5, lane = i & 31;
    const int nh = PAIR ? 2 : 1;
    for (int h = 0; h < nh; ++h) {
        const int f = PAIR ? tile * 64 + 2 * lane + h : tile * 32 + lane;
        if (f >= a.nframes || (d & (1u << h))) continue;
        const bool fail = PAIR ? (h ? (s & 0x80000000u) : (s & 0x8000u)) : (s & 1u);
        a.it_ws[f] = a.K;
        a.ok_ws[f] = fail ? 0 : 1;
    }
}

// -------------------------------------------------------------- fp32 path
// ingest: Z^(0) plane (fp32, saturated to +-2^20 and -0.0 -> +0.0, readings D13, D28) and the
// accumulator of iteration 1 (Lb[1] = grid(Z^(0))); iteration 1 reads the fp32 plane itself
__global__ void k_stream_ingest_f(const StreamArgs a) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const int f = tile * 32 + lane;
    const float *llr = (const float *)a.llr;
    for (int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < a.N; n += gridDim.x * (blockDim.x >> 5)) {
        float z = 0.0f;
        if (f < a.nframes) z = llr[(size_t)f * a.N + n];
        z = fminf(fmaxf(z + 0.0f, -kSatF), kSatF);
        const size_t idx = ((size_t)tile * a.N + n) * 32 + lane;
        a.Z0[idx] = __float_as_uint(z);
        ((long long *)a.Lb[1])[idx] = grid_of(z);
        if (a.f32delta) ((long long *)a.Lb[0])[idx] = grid_of(z);   // X_0: iteration 2's plane
        if (a.layered) a.Lb[0][idx] = __float_as_uint(z);             // the one in-place array (D25)
    }
}

// Accumulator start of the next iteration, X = grid(Z^(0)), for a tile with no frozen frame:
// 4 fp32 values in, 4 int64 out per thread (contiguous [n][32] plane segment of the tile).
__device__ __forceinline__ void stream_init_next_f(const uint32_t *Z0t, long long *Xnt, int N, int wg, int nwg,
                                                   int lane) {
    const uint4 *src = (const uint4 *)Z0t;
    longlong2 *dst = (longlong2 *)Xnt;
    const int total = N * 8;
    const int step = nwg * 32;
    auto put = [&](int i, const uint4 &v) {
        __stcg(dst + 2 * i, make_longlong2(grid_of(__uint_as_float(v.x)), grid_of(__uint_as_float(v.y))));
        __stcg(dst + 2 * i + 1, make_longlong2(grid_of(__uint_as_float(v.z)), grid_of(__uint_as_float(v.w))));
    };
    int i = wg * 32 + lane;
    for (; i + 3 * step < total; i += 4 * step) {     // 4 loads in flight (the loop is latency-bound)
        const uint4 v0 = __ldcg(src + i), v1 = __ldcg(src + i + step), v2 = __ldcg(src + i + 2 * step),
                    v3 = __ldcg(src + i + 3 * step);
        put(i, v0);
        put(i + step, v1);
        put(i + 2 * step, v2);
        put(i + 3 * step, v3);
    }
    for (; i < total; i += step) put(i, __ldcg(src + i));
}
// the same per lane, skipping frozen frames (early stop: their buffers keep the exit posterior)
__device__ __forceinline__ void stream_init_next_f_lanes(const uint32_t *Z0t, long long *Xnt, int N, int wg, int nwg,
                                                         int lane, bool frozen) {
    if (frozen) return;
    for (int n = wg; n < N; n += nwg) {
        const size_t idx = (size_t)n * 32 + lane;
        __stcg(Xnt + idx, grid_of(__uint_as_float(__ldcg(Z0t + idx))));
    }
}

// NR rows, one frame per lane, fp32 (reading D11: one RN rounding per operation,
// no FMA contraction: __fsub_rn / __fmul_rn; reading D28: exact int64 accumulation).
// All loads issued before any compute.  Iteration 1 reads the fp32 Z^(0) plane.
template <int DC, int NR, bool ES>
__device__ __forceinline__ void stream_rows_f(const StreamArgs &a, int lane, const int (&m)[NR], const RowT *rt,
                                              const uint32_t *Z0t, const long long *Xpt, long long *Xat,
                                              uint32_t *stt, bool first_iter, bool frozen, uint32_t &synd) {
    uint32_t off[NR][DC];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            // rows of degree <= 8 come with their column table; wider rows read the CSR
            const uint32_t c = DC <= 8 ? rt[r].c[j < 8 ? j : 0] : (uint32_t)__ldg(a.col_idx + __ldg(a.row_ptr + m[r]) + j);
            LDPC_CHECK(c < (uint32_t)a.N && m[r] < a.M);
            off[r][j] = c * 32u + (uint32_t)lane;
        }
    const size_t ss = (size_t)a.M * 32;
    float A0[NR], B0[NR];
    uint32_t W0[NR];
    if (!first_iter) {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const size_t so = (size_t)m[r] * 32 + lane;
            A0[r] = __uint_as_float(__ldcg(stt + so));
            B0[r] = __uint_as_float(__ldcg(stt + ss + so));
            W0[r] = __ldcg(stt + 2 * ss + so);
        }
    }
    float L[NR][DC];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int j = 0; j < DC; ++j)
            L[r][j] = first_iter ? __uint_as_float(__ldcg(Z0t + off[r][j])) : val_of(__ldcg(Xpt + off[r][j]));
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        if (ES) {
            uint32_t p = 0;
#pragma unroll
            for (int j = 0; j < DC; ++j) p ^= L[r][j] <= 0.0f ? 1u : 0u;
            synd |= p;
        }
        float A, B, rr[DC];
        uint32_t Wn;
        f32_row<DC>(L[r], first_iter, first_iter ? 0.f : A0[r], first_iter ? 0.f : B0[r], first_iter ? 0u : W0[r],
                    a.alpha, a.beta, A, B, Wn, rr);
        const size_t so = (size_t)m[r] * 32 + lane;
        __stcg(stt + so, __float_as_uint(A));
        __stcg(stt + ss + so, __float_as_uint(B));
        __stcg(stt + 2 * ss + so, Wn);
        if (!frozen) {
#pragma unroll
            for (int j = 0; j < DC; ++j)                                          // Z^(k)_n += L^(k)_mn (exact)
                atomicAdd((unsigned long long *)(Xat + off[r][j]), (unsigned long long)grid_of(rr[j]));
        }
    }
}

template <int NR, bool ES>
__device__ __forceinline__ void stream_dispatch_f(int dc, const StreamArgs &a, int lane, const int (&m)[NR],
                                                  const RowT *rt, const uint32_t *Z0t, const long long *Xpt,
                                                  long long *Xat, uint32_t *stt, bool first_iter, bool frozen,
                                                  uint32_t &synd) {
    switch (dc) {
#define LDPC_SF(D) \
    case D: stream_rows_f<D, NR, ES>(a, lane, m, rt, Z0t, Xpt, Xat, stt, first_iter, frozen, synd); break;
    LDPC_SF(2) LDPC_SF(3) LDPC_SF(4) LDPC_SF(5) LDPC_SF(6) LDPC_SF(7) LDPC_SF(8) LDPC_SF(9) LDPC_SF(10)
    LDPC_SF(11) LDPC_SF(12) LDPC_SF(13) LDPC_SF(14) LDPC_SF(15) LDPC_SF(16)
#undef LDPC_SF
    }
}

// Register version of the fp32 iteration kernel (rows of degree 9..16; the pipelined
// kernel takes rows of degree <= 8)
template <bool ES>
__global__ void __launch_bounds__(256, 4) k_stream_iter_f(const StreamArgs a, int k) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nwg = gridDim.x * (blockDim.x >> 5);
    const size_t plane = (size_t)tile * a.N * 32;
    const uint32_t *Z0t = a.Z0 + plane;
    const long long *Xpt = (const long long *)a.Lb[(k - 1) % 3] + plane;
    long long *Xat = (long long *)a.Lb[k % 3] + plane;
    long long *Xnt = (long long *)a.Lb[(k + 1) % 3] + plane;
    uint32_t *stt = a.st + (size_t)tile * 3 * a.M * 32;
    bool frozen = false;
    if (ES) {
        frozen = (a.done[tile * 32 + lane] & 1u) != 0;
        if (__all_sync(0xFFFFFFFFu, frozen)) return;
    }
    if (k < a.K) {
        if (!ES || !__any_sync(0xFFFFFFFFu, frozen)) stream_init_next_f(Z0t, Xnt, a.N, wg, nwg, lane);
        else stream_init_next_f_lanes(Z0t, Xnt, a.N, wg, nwg, lane, frozen);
    }
    uint32_t synd = 0;
    const bool first_iter = (k == 1);
    for (int m = wg; m < a.M; m += nwg) {
        const RowT rt = load_rowt(a.rowtab, m, a.M);
        int dc = rt.dc;
        if (dc == 15) dc = __ldg(a.row_ptr + m + 1) - __ldg(a.row_ptr + m);
        const int mm[1] = {m};
        stream_dispatch_f<1, ES>(dc, a, lane, mm, &rt, Z0t, Xpt, Xat, stt, first_iter, frozen, synd);
    }
    if (ES && synd) atomicOr(a.synd + tile * 32 + lane, synd);
}

}  // namespace ldpc
