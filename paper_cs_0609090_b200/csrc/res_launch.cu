// res_launch.cu -- host entry points of the decode-resident kernels: dispatch on (QC, early
// stop) to the translation unit that instantiates that combination (res_launch_q*e*.cu).
#include "res_launch_impl.cuh"

namespace ldpc {

cudaError_t res_occupancy(bool qc, bool es, int fmt, bool i8, int kind, size_t dyn_smem, size_t smem_per_sm,
                          int threads, int *blocks) {
    if (qc) return es ? res_occupancy_q1e1(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks)
                      : res_occupancy_q1e0(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks);
    return es ? res_occupancy_q0e1(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks)
              : res_occupancy_q0e0(fmt, i8, kind, dyn_smem, smem_per_sm, threads, blocks);
}

cudaError_t res_launch(bool qc, bool es, int fmt, bool i8, int kind, int grid, int threads, size_t dyn_smem,
                       const ResArgs &a, const QcTab &t, cudaStream_t s) {
    if (qc) return es ? res_launch_q1e1(fmt, i8, kind, grid, threads, dyn_smem, a, t, s)
                      : res_launch_q1e0(fmt, i8, kind, grid, threads, dyn_smem, a, t, s);
    return es ? res_launch_q0e1(fmt, i8, kind, grid, threads, dyn_smem, a, t, s)
              : res_launch_q0e0(fmt, i8, kind, grid, threads, dyn_smem, a, t, s);
}

}  // namespace ldpc
