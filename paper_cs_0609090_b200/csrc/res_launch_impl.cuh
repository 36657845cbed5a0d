// res_launch_impl.cuh -- instantiation machinery of the decode-resident kernels, shared by
// the four translation units res_launch_q{0,1}e{0,1}.cu (one per QC x early-stop
// combination, so the heavily templated kernels compile in parallel) and dispatched by
// res_launch.cu.
#pragma once
#include <algorithm>
#include <mutex>

#include "k_resident.cuh"
#include "k_resident_atom.cuh"
#include "k_resident_f32.cuh"
#include "launch.h"

namespace ldpc {
namespace resimpl {

template <bool QC, bool ES, int FMT, typename TIN, int KIND>
struct Kern {
    static auto get() {
        if constexpr (KIND == 4) return k_resident_f32_lay<QC, ES>;
        else if constexpr (KIND == 2) return k_resident_atom<QC, ES, FMT, TIN>;
        else return k_resident<QC, ES, FMT, TIN, KIND == 1>;
    }
    // The dynamic shared memory cap is raised once per kernel to the device's opt-in limit
    // (it is only a cap: occupancy follows the size each launch asks for), so concurrent
    // host threads never race on the attribute.
    static cudaFuncAttributes *attrs() {
        static cudaFuncAttributes a[kMaxDevices];
        return a;
    }
    static cudaError_t prepare() {
        static std::once_flag flags[kMaxDevices];
        static cudaError_t errs[kMaxDevices];
        return once_per_device(flags, errs, [] {
            int dev = 0, optin = 0;
            cudaError_t err = cudaGetDevice(&dev);
            if (err == cudaSuccess) err = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            cudaFuncAttributes fa;
            if (err == cudaSuccess) err = cudaFuncGetAttributes(&fa, get());
            // the cap excludes the kernel's static shared memory
            if (err == cudaSuccess)
                err = cudaFuncSetAttribute(get(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           optin - (int)fa.sharedSizeBytes);
            if (err == cudaSuccess && dev >= 0 && dev < kMaxDevices) attrs()[dev] = fa;
            return err;
        });
    }
    // the kernel's attributes on the current device, queried once per device by prepare()
    static cudaError_t attributes(cudaFuncAttributes &fa) {
        cudaError_t e = prepare();
        if (e != cudaSuccess) return e;
        int dev = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
        if (dev >= 0 && dev < kMaxDevices) {
            fa = attrs()[dev];
            return cudaSuccess;
        }
        return cudaFuncGetAttributes(&fa, get());
    }
};

template <bool QC, bool ES, int FMT, typename TIN, int KIND>
cudaError_t occ(size_t dyn_smem, size_t smem_per_sm, int threads, int *blocks) {
    // The occupancy API reports 1 block/SM for kernels that allocate TMEM; compute the
    // limit from the kernel's registers, shared memory and threads instead (TMEM is
    // accounted for by the caller).
    cudaFuncAttributes fa;
    cudaError_t e = Kern<QC, ES, FMT, TIN, KIND>::attributes(fa);
    if (e != cudaSuccess) return e;
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
    cudaError_t e = Kern<QC, ES, FMT, TIN, KIND>::prepare();
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, dyn_smem, s>>>(a, t);
    return cudaGetLastError();
}

// dispatch over the remaining template parameters for one (QC, ES) combination.  PART splits
// the instantiations over translation units so they compile in parallel: -1 = all, 0 = the
// COMPACT format and the fp32 layered kernel, 1 = the 1-bit and full-message formats
// (res_part_of below picks the part of a call).
inline int res_part_of(int fmt, int kind) { return (fmt == FMT_C16 || kind == 4) ? 0 : 1; }
template <template <bool, bool, int, typename, int> class K, bool Q, bool E, int PART, typename... Args>
cudaError_t dispatch_qe(int fmt, bool i8, int kind, Args... args) {
#define LDPC_RES_KIND(F, KK) \
    if (kind == KK) return i8 ? K<Q, E, F, int8_t, KK>::run(args...) : K<Q, E, F, int16_t, KK>::run(args...);
#define LDPC_RES_CASE(F) \
    if (fmt == F) { LDPC_RES_KIND(F, 0) LDPC_RES_KIND(F, 1) LDPC_RES_KIND(F, 2) }
    if constexpr (PART != 1) {
        LDPC_RES_CASE(FMT_C16)
        // fp32 LLRs, layered schedule: one frame per CTA (k_resident_f32.cuh)
        if (kind == 4) return K<Q, E, FMT_C16, float, 4>::run(args...);
    }
    if constexpr (PART != 0) {
        LDPC_RES_CASE(FMT_1BIT)
        // FMT_FULL (§4 per-edge messages) exists for the barrier-free kernel only
        if (fmt == FMT_FULL && kind == 2)
            return i8 ? K<Q, E, FMT_FULL, int8_t, 2>::run(args...) : K<Q, E, FMT_FULL, int16_t, 2>::run(args...);
    }
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

}  // namespace resimpl

// per-(QC, ES, part) entry points, defined in res_launch_q*e*_p*.cu (each combination split in
// two translation units by format group; P = 2 would instantiate both parts in one unit)
#define LDPC_RES_QE_DECL(Q, E, P)                                                                                \
    cudaError_t res_occupancy_q##Q##e##E##p##P(int fmt, bool i8, int kind, size_t dyn_smem, size_t smem_per_sm,   \
                                               int threads, int *blocks);                                        \
    cudaError_t res_launch_q##Q##e##E##p##P(int fmt, bool i8, int kind, int grid, int threads, size_t dyn_smem,   \
                                            const ResArgs &a, const QcTab &t, cudaStream_t s);
LDPC_RES_QE_DECL(0, 0, 0) LDPC_RES_QE_DECL(0, 0, 1) LDPC_RES_QE_DECL(0, 1, 0) LDPC_RES_QE_DECL(0, 1, 1)
LDPC_RES_QE_DECL(1, 0, 0) LDPC_RES_QE_DECL(1, 0, 1) LDPC_RES_QE_DECL(1, 1, 0) LDPC_RES_QE_DECL(1, 1, 1)
#undef LDPC_RES_QE_DECL

#define LDPC_RES_QE_DEF(Q, E, P)                                                                                 \
    cudaError_t res_occupancy_q##Q##e##E##p##P(int fmt, bool i8, int kind, size_t dyn_smem, size_t smem_per_sm,   \
                                               int threads, int *blocks) {                                       \
        return resimpl::dispatch_qe<resimpl::Occ, (Q != 0), (E != 0), (P == 2 ? -1 : P)>(fmt, i8, kind, dyn_smem,  \
                                                                                          smem_per_sm, threads, blocks); \
    }                                                                                                            \
    cudaError_t res_launch_q##Q##e##E##p##P(int fmt, bool i8, int kind, int grid, int threads, size_t dyn_smem,   \
                                            const ResArgs &a, const QcTab &t, cudaStream_t s) {                  \
        return resimpl::dispatch_qe<resimpl::Launch, (Q != 0), (E != 0), (P == 2 ? -1 : P)>(fmt, i8, kind, grid,  \
                                                                                             threads, dyn_smem, &a, &t, s); \
    }

}  // namespace ldpc
