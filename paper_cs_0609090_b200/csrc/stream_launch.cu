// stream_launch.cu -- launches of the streaming kernels (long codes) and the error counter.
#include <utility>
#include <algorithm>
#include <mutex>

#include "k_stream_layered.cuh"
#include "k_stream_pipe.cuh"
#include "k_twoscan.cuh"
#include "launch.h"

namespace ldpc {

// -------------------------------------------------------------- error counters
__global__ void k_count_errors(int64_t nframes, int wpf, const uint32_t *hb, const uint8_t *ok, const int32_t *it,
                               unsigned long long *cnt) {
    unsigned long long c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nframes; f += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long be = 0;
        for (int w = 0; w < wpf; ++w) be += __popc(hb[f * wpf + w]);
        c0 += be;
        c1 += be ? 1 : 0;
        c2 += (be && ok[f]) ? 1 : 0;
        c3 += ok[f] ? 0 : 1;
        c4 += it ? (unsigned long long)it[f] : 0ull;
    }
    for (int o = 16; o; o >>= 1) {
        c0 += __shfl_xor_sync(0xFFFFFFFFu, c0, o);
        c1 += __shfl_xor_sync(0xFFFFFFFFu, c1, o);
        c2 += __shfl_xor_sync(0xFFFFFFFFu, c2, o);
        c3 += __shfl_xor_sync(0xFFFFFFFFu, c3, o);
        c4 += __shfl_xor_sync(0xFFFFFFFFu, c4, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (c0) atomicAdd(cnt + 0, c0);
        if (c1) atomicAdd(cnt + 1, c1);
        if (c2) atomicAdd(cnt + 2, c2);
        if (c3) atomicAdd(cnt + 3, c3);
        if (c4) atomicAdd(cnt + 4, c4);
    }
}


namespace {
template <typename F>
cudaError_t launch(F f, int32_t *n) {
    f();
    ++*n;
    return cudaGetLastError();
}
// a launch that may overlap the retiring tail of the previous kernel in the stream
// (programmatic dependent launch): the kernel itself waits (griddepcontrol.wait) before
// reading anything the previous kernel wrote
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, int threads, size_t smem, cudaStream_t s, bool pdl,
                       int32_t *n, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    ++*n;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// the variant of iteration k (lambda_k, beta_k) for the launches of k
void set_iteration(StreamArgs &c, const StreamRun &r, int k) {
    if (r.vk_sched) c.vk = r.vk_sched[k - 1];
    if (r.alpha_sched) c.alpha = r.alpha_sched[k - 1];
    if (r.beta_sched) c.beta = r.beta_sched[k - 1];
}
// raise the dynamic shared memory cap of the pipelined kernels once (a cap only; each
// launch asks for its own size), so concurrent host threads never race on the attribute
cudaError_t pipe_prepare() {
    static std::once_flag flags[kMaxDevices];
    static cudaError_t errs[kMaxDevices];
    return once_per_device(flags, errs, [] {
        cudaError_t err = cudaSuccess;
        auto set = [&err](auto kern, size_t bytes) {
            if (err == cudaSuccess) err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        };
        set(k_stream_pipe<true, FMT_C16, true>, pipe_smem_bytes<true>());
        set(k_stream_pipe<true, FMT_C16, false>, pipe_smem_bytes<true>());
        set(k_stream_pipe<true, FMT_1BIT, true>, pipe_smem_bytes<true>());
        set(k_stream_pipe<true, FMT_1BIT, false>, pipe_smem_bytes<true>());
        set(k_stream_pipe<false, FMT_C16, true>, pipe_smem_bytes<false>());
        set(k_stream_pipe<false, FMT_C16, false>, pipe_smem_bytes<false>());
        return err;
    });
}
}  // namespace

cudaError_t count_errors_launch(int64_t nframes, int wpf, const uint32_t *hb, const uint8_t *ok, const int32_t *it,
                                unsigned long long *cnt, cudaStream_t s) {
    const unsigned blocks = (unsigned)std::min<int64_t>((nframes + 255) / 256, 4096);
    k_count_errors<<<blocks, 256, 0, s>>>(nframes, wpf, hb, ok, it, cnt);
    return cudaGetLastError();
}

cudaError_t stream_run(const StreamArgs &a, const StreamRun &r, cudaStream_t s, int32_t *nl) {
    cudaError_t e;
    // synd, done (contiguous) and per-frame flags
    if ((e = cudaMemsetAsync(a.synd, 0, r.flags_bytes, s)) != cudaSuccess) return e;
    const bool es = r.es;
    const bool pair = r.pair;
    const int nwarps_per_block = 8;
    dim3 gi((unsigned)std::min<int64_t>(((int64_t)a.N + 7) / 8, 1024), (unsigned)r.ntiles);
    // ~8 rows per warp per launch
    const int rows_per_block = nwarps_per_block * 8;
    dim3 gr((unsigned)std::max(1, (a.M + rows_per_block - 1) / rows_per_block), (unsigned)r.ntiles);
    if (pair) {
        if (r.i8) e = launch([&] { k_stream_ingest_i<int8_t><<<gi, 256, 0, s>>>(a, 1); }, nl);
        else e = launch([&] { k_stream_ingest_i<int16_t><<<gi, 256, 0, s>>>(a, 1); }, nl);
    } else {
        e = launch([&] { k_stream_ingest_f<<<gi, 256, 0, s>>>(a); }, nl);
    }
    if (e != cudaSuccess) return e;
    if (r.layered) {
        // one warp per frame tile walks the rows in order (k_stream_layered.cuh), then outputs
        const dim3 gl((unsigned)((r.ntiles + 3) / 4));
        LaySched sch{};
        if (r.vk_sched || r.alpha_sched || r.beta_sched) {
            if (r.max_iter > kMaxSched) return cudaErrorInvalidValue;   // the planner rejects these
            sch.n = r.max_iter;
            for (int k = 1; k <= r.max_iter; ++k) {
                sch.vk[k - 1] = r.vk_sched ? r.vk_sched[k - 1] : a.vk;
                sch.alpha[k - 1] = r.alpha_sched ? r.alpha_sched[k - 1] : a.alpha;
                sch.beta[k - 1] = r.beta_sched ? r.beta_sched[k - 1] : a.beta;
            }
        }
        if (pair) {
            if (r.fmt == FMT_C16) e = es ? launch([&] { k_stream_layered<true, FMT_C16, true><<<gl, 128, 0, s>>>(a, sch); }, nl)
                                         : launch([&] { k_stream_layered<true, FMT_C16, false><<<gl, 128, 0, s>>>(a, sch); }, nl);
            else e = es ? launch([&] { k_stream_layered<true, FMT_1BIT, true><<<gl, 128, 0, s>>>(a, sch); }, nl)
                        : launch([&] { k_stream_layered<true, FMT_1BIT, false><<<gl, 128, 0, s>>>(a, sch); }, nl);
        } else {
            e = es ? launch([&] { k_stream_layered<false, FMT_C16, true><<<gl, 128, 0, s>>>(a, sch); }, nl)
                   : launch([&] { k_stream_layered<false, FMT_C16, false><<<gl, 128, 0, s>>>(a, sch); }, nl);
        }
        if (e != cudaSuccess) return e;
        dim3 go((unsigned)a.wpf, (unsigned)r.ntiles);
        e = pair ? launch([&] { k_stream_output<true><<<go, 256, 0, s>>>(a); }, nl)
                 : launch([&] { k_stream_output<false><<<go, 256, 0, s>>>(a); }, nl);
        if (e != cudaSuccess || !a.msg_out) return e;
        if (!pair) return launch([&] { k_stream_export<false, FMT_C16><<<gr, 256, 0, s>>>(a); }, nl);
        if (r.fmt == FMT_C16) return launch([&] { k_stream_export<true, FMT_C16><<<gr, 256, 0, s>>>(a); }, nl);
        return launch([&] { k_stream_export<true, FMT_1BIT><<<gr, 256, 0, s>>>(a); }, nl);
    }
    // software-pipelined iteration kernel (cp.async row prefetch) for rows of degree <= 8,
    // unless the register kernels are requested (tuning cross-check)
    const unsigned fgrid = (unsigned)((r.ntiles * 32 + 255) / 256);
    const bool use_pipe = r.max_dc <= 8 && !r.register_kernels;
    // fp32 on the pipelined kernel uses the delta accumulation (k_stream_pipe.cuh); the
    // planner laid out the second state plane for exactly that case
    if (!pair && use_pipe != (a.f32delta != 0)) return cudaErrorInvalidValue;
    const size_t psmem = pair ? pipe_smem_bytes<true>() : pipe_smem_bytes<false>();
    if (use_pipe && (e = pipe_prepare()) != cudaSuccess) return e;
    // Frame tiles are decoded in CHUNKS whose per-iteration working set (Z^(0), the three
    // posterior planes and the compact state of the chunk's tiles) fits in L2: all
    // iterations of a chunk run before the next chunk starts, so after the first
    // iteration the streaming kernels hit L2 instead of HBM.  Every kernel of the
    // iteration loop indexes per tile, so a chunk is the same arguments with the
    // tile-major pointers advanced.
    const int chunk = r.chunk_tiles > 0 ? std::min(r.chunk_tiles, r.ntiles) : r.ntiles;
    const int tw = pair ? 64 : 32;
    const int nst = pair ? (r.fmt == FMT_C16 ? 3 : 2) : 3;
    for (int t0 = 0; t0 < r.ntiles; t0 += chunk) {
        const int nt = std::min(chunk, r.ntiles - t0);
        StreamArgs c = a;
        const size_t plane = (size_t)t0 * a.N * 32;
        c.Z0 = a.Z0 + plane;
        for (int i = 0; i < 3; ++i) c.Lb[i] = a.Lb[i] + (pair ? plane : 2 * plane);   // fp32: int64 planes
        c.st = a.st + (size_t)t0 * nst * a.M * 32;
        if (a.st2) c.st2 = a.st2 + (size_t)t0 * nst * a.M * 32;
        c.synd = a.synd + (size_t)t0 * 32;
        c.done = a.done + (size_t)t0 * 32;
        c.it_ws = a.it_ws + (size_t)t0 * tw;
        c.ok_ws = a.ok_ws + (size_t)t0 * tw;
        c.nframes = a.nframes - t0 * tw;
        c.ntiles = nt;
        const unsigned fgrid = (unsigned)((nt * 32 + 255) / 256);
        const dim3 gp((unsigned)((a.M + kPipeRB - 1) / kPipeRB), (unsigned)nt);
        const dim3 gr((unsigned)std::max(1, (a.M + rows_per_block - 1) / rows_per_block), (unsigned)nt);
        for (int k = 1; k <= r.max_iter && use_pipe; ++k) {
            set_iteration(c, r, k);
            // iterations 2.. follow the previous iteration's kernel directly (no freeze kernel
            // in between without early stop): programmatic dependent launches
            const bool pdl = k > 1 && !es;
            const int th = kPipeWarps * 32;
            if (pair) {
                if (r.fmt == FMT_C16) {
                    if (es) e = launch_pdl(k_stream_pipe<true, FMT_C16, true>, gp, th, psmem, s, pdl, nl, c, k);
                    else e = launch_pdl(k_stream_pipe<true, FMT_C16, false>, gp, th, psmem, s, pdl, nl, c, k);
                } else {
                    if (es) e = launch_pdl(k_stream_pipe<true, FMT_1BIT, true>, gp, th, psmem, s, pdl, nl, c, k);
                    else e = launch_pdl(k_stream_pipe<true, FMT_1BIT, false>, gp, th, psmem, s, pdl, nl, c, k);
                }
            } else {
                if (es) e = launch_pdl(k_stream_pipe<false, FMT_C16, true>, gp, th, psmem, s, pdl, nl, c, k);
                else e = launch_pdl(k_stream_pipe<false, FMT_C16, false>, gp, th, psmem, s, pdl, nl, c, k);
            }
            if (e != cudaSuccess) return e;
            if (es) {
                if (pair) e = launch([&] { k_stream_freeze<true><<<fgrid, 256, 0, s>>>(c, k); }, nl);
                else e = launch([&] { k_stream_freeze<false><<<fgrid, 256, 0, s>>>(c, k); }, nl);
                if (e != cudaSuccess) return e;
            }
        }
        for (int k = 1; k <= r.max_iter && !use_pipe; ++k) {
            set_iteration(c, r, k);
            if (pair) {
                if (r.fmt == FMT_C16) {
                    if (es) e = launch([&] { k_stream_iter_i<FMT_C16, true><<<gr, 256, 0, s>>>(c, k); }, nl);
                    else e = launch([&] { k_stream_iter_i<FMT_C16, false><<<gr, 256, 0, s>>>(c, k); }, nl);
                } else {
                    if (es) e = launch([&] { k_stream_iter_i<FMT_1BIT, true><<<gr, 256, 0, s>>>(c, k); }, nl);
                    else e = launch([&] { k_stream_iter_i<FMT_1BIT, false><<<gr, 256, 0, s>>>(c, k); }, nl);
                }
            } else {
                if (es) e = launch([&] { k_stream_iter_f<true><<<gr, 256, 0, s>>>(c, k); }, nl);
                else e = launch([&] { k_stream_iter_f<false><<<gr, 256, 0, s>>>(c, k); }, nl);
            }
            if (e != cudaSuccess) return e;
            if (es) {
                if (pair) e = launch([&] { k_stream_freeze<true><<<fgrid, 256, 0, s>>>(c, k); }, nl);
                else e = launch([&] { k_stream_freeze<false><<<fgrid, 256, 0, s>>>(c, k); }, nl);
                if (e != cudaSuccess) return e;
            }
        }
    }
    if (pair) e = launch([&] { k_stream_syndrome<true><<<gr, 256, 0, s>>>(a, r.max_iter); }, nl);
    else e = launch([&] { k_stream_syndrome<false><<<gr, 256, 0, s>>>(a, r.max_iter); }, nl);
    if (e != cudaSuccess) return e;
    if (pair) e = launch([&] { k_stream_finalize_flags<true><<<fgrid, 256, 0, s>>>(a); }, nl);
    else e = launch([&] { k_stream_finalize_flags<false><<<fgrid, 256, 0, s>>>(a); }, nl);
    if (e != cudaSuccess) return e;
    dim3 go((unsigned)a.wpf, (unsigned)r.ntiles);
    if (pair) e = launch([&] { k_stream_output<true><<<go, 256, 0, s>>>(a); }, nl);
    else e = launch([&] { k_stream_output<false><<<go, 256, 0, s>>>(a); }, nl);
    if (e != cudaSuccess || !a.msg_out) return e;
    if (!pair) return launch([&] { k_stream_export<false, FMT_C16><<<gr, 256, 0, s>>>(a); }, nl);
    if (r.fmt == FMT_C16) return launch([&] { k_stream_export<true, FMT_C16><<<gr, 256, 0, s>>>(a); }, nl);
    return launch([&] { k_stream_export<true, FMT_1BIT><<<gr, 256, 0, s>>>(a); }, nl);
}


// Two-scan min-sum (k_twoscan.cuh): ingest, Z_mn init, then per iteration the
// horizontal and vertical scans; early stop checks H x^ = 0 on Z^(k) after each
// iteration (and on Z^(0) first, reading D10) with the shared syndrome/freeze kernels.
cudaError_t twoscan_run(const StreamArgs &a0, const TwoScanArgs &t, const StreamRun &r, cudaStream_t s, int32_t *nl) {
    StreamArgs a = a0;
    cudaError_t e;
    if ((e = cudaMemsetAsync(a.synd, 0, r.flags_bytes, s)) != cudaSuccess) return e;
    const bool pair = r.pair, es = r.es;
    dim3 gi((unsigned)std::min<int64_t>(((int64_t)a.N + 7) / 8, 1024), (unsigned)r.ntiles);
    if (pair) {
        if (r.i8) e = launch([&] { k_stream_ingest_i<int8_t><<<gi, 256, 0, s>>>(a, 0); }, nl);
        else e = launch([&] { k_stream_ingest_i<int16_t><<<gi, 256, 0, s>>>(a, 0); }, nl);
    } else {
        e = launch([&] { k_stream_ingest_f<<<gi, 256, 0, s>>>(a); }, nl);
    }
    if (e != cudaSuccess) return e;
    const dim3 gm((unsigned)std::max(1, std::min((a.M + 7) / 8, 4096)), (unsigned)r.ntiles);
    const dim3 gn((unsigned)std::max(1, std::min((a.N + 7) / 8, 4096)), (unsigned)r.ntiles);
    const dim3 gr((unsigned)std::max(1, (a.M + 63) / 64), (unsigned)r.ntiles);
    const unsigned fgrid = (unsigned)((r.ntiles * 32 + 255) / 256);
    auto syndrome = [&](int k) {      // posterior after iteration k (k = 0: Z^(0))
        return pair ? launch([&] { k_stream_syndrome<true><<<gr, 256, 0, s>>>(a, k); }, nl)
                    : launch([&] { k_stream_syndrome<false><<<gr, 256, 0, s>>>(a, k); }, nl);
    };
    auto freeze = [&](int k) {
        return pair ? launch([&] { k_stream_freeze<true><<<fgrid, 256, 0, s>>>(a, k); }, nl)
                    : launch([&] { k_stream_freeze<false><<<fgrid, 256, 0, s>>>(a, k); }, nl);
    };
    e = pair ? launch([&] { k_ts_init<true><<<gn, 256, 0, s>>>(a, t); }, nl)
             : launch([&] { k_ts_init<false><<<gn, 256, 0, s>>>(a, t); }, nl);
    if (e != cudaSuccess) return e;
    if (es) {
        // k = 0: Z^(0) is in Lb[0]; frames passing freeze with iterations_used = 0
        if ((e = syndrome(0)) != cudaSuccess || (e = freeze(1)) != cudaSuccess) return e;
    }
    for (int k = 1; k <= r.max_iter; ++k) {
        set_iteration(a, r, k);
        e = pair ? launch([&] { k_ts_check<true><<<gm, 256, 0, s>>>(a, t); }, nl)
                 : launch([&] { k_ts_check<false><<<gm, 256, 0, s>>>(a, t); }, nl);
        if (e != cudaSuccess) return e;
        const bool d4 = t.max_dv <= 4;
#define LDPC_TS_VAR(P_, E_)                                                                      \
    (d4 ? launch([&] { k_ts_var<P_, E_, 4><<<gn, 256, 0, s>>>(a, t, k); }, nl)                   \
        : launch([&] { k_ts_var<P_, E_, 8><<<gn, 256, 0, s>>>(a, t, k); }, nl))
        if (pair) e = es ? LDPC_TS_VAR(true, true) : LDPC_TS_VAR(true, false);
        else e = es ? LDPC_TS_VAR(false, true) : LDPC_TS_VAR(false, false);
#undef LDPC_TS_VAR
        if (e != cudaSuccess) return e;
        if (es && k < r.max_iter) {
            // syndrome of Z^(k) from the variable pass's hard-decision ballots
            const dim3 gs((unsigned)((a.M + 255) / 256), (unsigned)r.ntiles);
            e = pair ? launch([&] { k_ts_syndrome<true><<<gs, 256, 0, s>>>(a, t); }, nl)
                     : launch([&] { k_ts_syndrome<false><<<gs, 256, 0, s>>>(a, t); }, nl);
            if (e != cudaSuccess || (e = freeze(k + 1)) != cudaSuccess) return e;
        }
    }
    // final syndrome of Z^(K); frames not frozen get iterations_used = K
    if ((e = syndrome(r.max_iter)) != cudaSuccess) return e;
    e = pair ? launch([&] { k_stream_finalize_flags<true><<<fgrid, 256, 0, s>>>(a); }, nl)
             : launch([&] { k_stream_finalize_flags<false><<<fgrid, 256, 0, s>>>(a); }, nl);
    if (e != cudaSuccess) return e;
    dim3 go((unsigned)a.wpf, (unsigned)r.ntiles);
    e = pair ? launch([&] { k_stream_output<true><<<go, 256, 0, s>>>(a); }, nl)
             : launch([&] { k_stream_output<false><<<go, 256, 0, s>>>(a); }, nl);
    if (e != cudaSuccess || !a.msg_out) return e;
    const dim3 ge((unsigned)std::max<int64_t>(1, std::min<int64_t>((t.E + 7) / 8, 8192)), (unsigned)r.ntiles);
    return pair ? launch([&] { k_ts_export<true><<<ge, 256, 0, s>>>(a, t); }, nl)
                : launch([&] { k_ts_export<false><<<ge, 256, 0, s>>>(a, t); }, nl);
}

}  // namespace ldpc
