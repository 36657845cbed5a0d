// res_launch_q1e0.cu -- resident-kernel instantiations for QC = True, early stop = False.
#include "res_launch_impl.cuh"

namespace ldpc {
LDPC_RES_QE_DEF(1, 0)
}  // namespace ldpc
