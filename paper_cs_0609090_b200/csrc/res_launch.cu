// res_launch.cu -- host entry points of the decode-resident kernels: dispatch on (QC, early
// stop, format group) to the translation unit that instantiates that combination
// (res_launch_q*e*_p*.cu).
#include "res_launch_impl.cuh"

namespace ldpc {

cudaError_t res_occupancy(bool qc, bool es, int fmt, bool i8, int kind, size_t dyn_smem, size_t smem_per_sm,
                          int threads, int *blocks) {
    if (qc) {
        const bool p1 = resimpl::res_part_of(fmt, kind) == 1;
        if (es) return p1 ? res_occupancy_q1e1p1(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks)
                          : res_occupancy_q1e1p0(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks);
        return p1 ? res_occupancy_q1e0p1(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks)
                  : res_occupancy_q1e0p0(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks);
    }
    const bool p1 = resimpl::res_part_of(fmt, kind) == 1;
    if (es) return p1 ? res_occupancy_q0e1p1(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks)
                      : res_occupancy_q0e1p0(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks);
    return p1 ? res_occupancy_q0e0p1(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks)
              : res_occupancy_q0e0p0(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks);
}

cudaError_t res_launch(bool qc, bool es, int fmt, bool i8, int kind, int grid, int threads, size_t dyn_smem,
                       const ResArgs &a, const QcTab &t, cudaStream_t s) {
    if (qc) {
        const bool p1 = resimpl::res_part_of(fmt, kind) == 1;
        if (es) return p1 ? res_launch_q1e1p1(fmt, i8, kind, grid, threads, dyn_smem, a, t, s)
                          : res_launch_q1e1p0(fmt, i8, kind, grid, threads, dyn_smem, a, t, s);
        return p1 ? res_launch_q1e0p1(fmt, i8, kind, grid, threads, dyn_smem, a, t, s)
                  : res_launch_q1e0p0(fmt, i8, kind, grid, threads, dyn_smem, a, t, s);
    }
    const bool p1 = resimpl::res_part_of(fmt, kind) == 1;
    if (es) return p1 ? res_launch_q0e1p1(fmt, i8, kind, grid, threads, dyn_smem, a, t, s)
                      : res_launch_q0e1p0(fmt, i8, kind, grid, threads, dyn_smem, a, t, s);
    return p1 ? res_launch_q0e0p1(fmt, i8, kind, grid, threads, dyn_smem, a, t, s)
              : res_launch_q0e0p0(fmt, i8, kind, grid, threads, dyn_smem, a, t, s);
}

}  // namespace ldpc
