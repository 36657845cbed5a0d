// launch.h -- host entry points of the kernel translation units (res_launch.cu,
// stream_launch.cu), called by the planner in ldpc_api.cu.  Split so the kernel
// instantiations compile in parallel.
#pragma once
#include <mutex>

#include "args.cuh"

namespace ldpc {

// Run f() once per CUDA device (function attributes are per device context): the first call
// made with device d current runs it, later calls on d return its result.
constexpr int kMaxDevices = 64;
template <typename F>
cudaError_t once_per_device(std::once_flag (&flags)[kMaxDevices], cudaError_t (&errs)[kMaxDevices], F f) {
    int dev = 0;
    const cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return f();
    std::call_once(flags[dev], [&] { errs[dev] = f(); });
    return errs[dev];
}

// Resident kernels.  i8 selects int8 channel LLRs (else int16).  kind: RES_BATCHED
// (k_resident.cuh, flooding in conflict-free batches), RES_LAYERED (k_resident.cuh,
// in-place schedule), RES_ATOM (k_resident_atom.cuh, flooding with shared atomics),
// RES_F32_LAY (k_resident_f32.cuh, fp32 LLRs, layered schedule, one frame per CTA).
enum { RES_BATCHED = 0, RES_LAYERED = 1, RES_ATOM = 2, RES_F32_LAY = 4 };
cudaError_t res_occupancy(bool qc, bool es, int fmt, bool i8, int kind, size_t dyn_smem, size_t smem_per_sm,
                          int threads, int *blocks);
cudaError_t res_launch(bool qc, bool es, int fmt, bool i8, int kind, int grid, int threads, size_t dyn_smem,
                       const ResArgs &a, const QcTab &t, cudaStream_t s);

// Streaming kernels (k_stream.cuh, k_stream_pipe.cuh): every launch of one decode.
struct StreamRun {
    bool pair;            // integer path (two frames per 16x2 lane) vs fp32
    bool i8;              // int8 channel LLRs (integer path)
    int fmt;              // FMT_C16 / FMT_1BIT
    bool es;              // per-frame early stop
    int max_iter, max_dc, ntiles;
    int chunk_tiles;      // tiles decoded together through all iterations (0 = all)
    bool register_kernels;  // integer / fp32 rows of degree <= 8: register kernels instead of the pipeline
    bool layered;           // LDPC_SCHED_LAYERED on the streaming layout (k_stream_layered.cuh)
    size_t flags_bytes;   // bytes from a.synd to the end of the per-tile flag words (zeroed first)
    // per-iteration variants (host arrays of max_iter entries, NULL = the constants in a)
    const VarK *vk_sched;
    const float *alpha_sched, *beta_sched;
};
cudaError_t stream_run(const StreamArgs &a, const StreamRun &r, cudaStream_t s, int32_t *launches);

// Two-scan min-sum baseline (k_twoscan.cuh), same workspace conventions plus the
// per-edge message planes in `t`.
cudaError_t twoscan_run(const StreamArgs &a, const TwoScanArgs &t, const StreamRun &r, cudaStream_t s,
                        int32_t *launches);

cudaError_t count_errors_launch(int64_t nframes, int wpf, const uint32_t *hb, const uint8_t *ok, const int32_t *it,
                                unsigned long long *cnt, cudaStream_t s);

}  // namespace ldpc
