// res_launch.cu -- instantiations and launches of the decode-resident kernel.
#include <algorithm>

#include "k_resident.cuh"
#include "k_resident_atom.cuh"
#include "k_resident_f32.cuh"
#include "launch.h"

namespace ldpc {
namespace {

template <bool QC, bool ES, int FMT, typename TIN, int KIND>
struct Kern {
    static auto get() {
        if constexpr (KIND == 4) return k_resident_f32_lay<QC, ES>;
        else if constexpr (KIND == 3) return k_resident_f32<QC, ES>;
        else if constexpr (KIND == 2) return k_resident_atom<QC, ES, FMT, TIN>;
        else return k_resident<QC, ES, FMT, TIN, KIND == 1>;
    }
};

template <bool QC, bool ES, int FMT, typename TIN, int KIND>
cudaError_t occ(size_t dyn_smem, size_t smem_per_sm, int threads, int *blocks) {
    // The occupancy API reports 1 block/SM for kernels that allocate TMEM; compute the
    // limit from the kernel's registers, shared memory and threads instead (TMEM is
    // accounted for by the caller).
    auto kern = Kern<QC, ES, FMT, TIN, KIND>::get();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, kern)) != cudaSuccess) return e;
    const size_t per_block_smem = dyn_smem + fa.sharedSizeBytes + 1024;   // + driver reserve
    const int by_smem = (int)(smem_per_sm / per_block_smem);
    const int regs = ((fa.numRegs + 7) / 8) * 8 * threads;
    const int by_regs = regs > 0 ? 65536 / regs : 32;
    const int by_threads = 2048 / threads;
    *blocks = std::max(0, std::min(std::min(by_smem, by_regs), std::min(by_threads, 32)));
    return cudaSuccess;
}

template <bool QC, bool ES, int FMT, typename TIN, int KIND>
cudaError_t launch(int grid, int threads, size_t dyn_smem, const ResArgs &a, const QcTab &t, cudaStream_t s) {
    auto kern = Kern<QC, ES, FMT, TIN, KIND>::get();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, dyn_smem, s>>>(a, t);
    return cudaGetLastError();
}

// dispatch over the template parameters; F is called with a pointer-to-instantiation tag
template <template <bool, bool, int, typename, int> class K, typename... Args>
cudaError_t dispatch(bool qc, bool es, int fmt, bool i8, int kind, Args... args) {
#define LDPC_RES_KIND(Q, E, F, KK) \
    if (kind == KK) return i8 ? K<Q, E, F, int8_t, KK>::run(args...) : K<Q, E, F, int16_t, KK>::run(args...);
#define LDPC_RES_CASE(Q, E, F)                                                    \
    if (qc == Q && es == E && fmt == F) {                                         \
        LDPC_RES_KIND(Q, E, F, 0) LDPC_RES_KIND(Q, E, F, 1) LDPC_RES_KIND(Q, E, F, 2) \
    }
    LDPC_RES_CASE(true, true, FMT_C16) LDPC_RES_CASE(true, true, FMT_1BIT)
    LDPC_RES_CASE(true, false, FMT_C16) LDPC_RES_CASE(true, false, FMT_1BIT)
    LDPC_RES_CASE(false, true, FMT_C16) LDPC_RES_CASE(false, true, FMT_1BIT)
    LDPC_RES_CASE(false, false, FMT_C16) LDPC_RES_CASE(false, false, FMT_1BIT)
    // FMT_FULL (§4 per-edge messages) exists for the barrier-free kernel only
#define LDPC_RES_FULL(Q, E)                                                               \
    if (qc == Q && es == E && fmt == FMT_FULL && kind == 2)                               \
        return i8 ? K<Q, E, FMT_FULL, int8_t, 2>::run(args...) : K<Q, E, FMT_FULL, int16_t, 2>::run(args...);
    LDPC_RES_FULL(true, true) LDPC_RES_FULL(true, false) LDPC_RES_FULL(false, true) LDPC_RES_FULL(false, false)
#undef LDPC_RES_FULL
    // fp32 LLRs: one frame per CTA (k_resident_f32.cuh; kind 4: layered schedule)
#define LDPC_RES_F32(Q, E) \
    if (qc == Q && es == E && kind == 3) return K<Q, E, FMT_C16, float, 3>::run(args...); \
    if (qc == Q && es == E && kind == 4) return K<Q, E, FMT_C16, float, 4>::run(args...);
    LDPC_RES_F32(true, true) LDPC_RES_F32(true, false) LDPC_RES_F32(false, true) LDPC_RES_F32(false, false)
#undef LDPC_RES_F32
#undef LDPC_RES_CASE
#undef LDPC_RES_KIND
    return cudaErrorInvalidValue;
}

template <bool QC, bool ES, int FMT, typename TIN, int KIND>
struct Occ {
    static cudaError_t run(size_t d, size_t sps, int th, int *b) { return occ<QC, ES, FMT, TIN, KIND>(d, sps, th, b); }
};
template <bool QC, bool ES, int FMT, typename TIN, int KIND>
struct Launch {
    static cudaError_t run(int g, int th, size_t d, const ResArgs *a, const QcTab *t, cudaStream_t s) {
        return launch<QC, ES, FMT, TIN, KIND>(g, th, d, *a, *t, s);
    }
};

}  // namespace

cudaError_t res_occupancy(bool qc, bool es, int fmt, bool i8, int kind, size_t dyn_smem, size_t smem_per_sm,
                          int threads, int *blocks) {
    return dispatch<Occ>(qc, es, fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks);
}

cudaError_t res_launch(bool qc, bool es, int fmt, bool i8, int kind, int grid, int threads, size_t dyn_smem,
                       const ResArgs &a, const QcTab &t, cudaStream_t s) {
    return dispatch<Launch>(qc, es, fmt, i8, kind, grid, threads, dyn_smem, &a, &t, s);
}

}  // namespace ldpc
