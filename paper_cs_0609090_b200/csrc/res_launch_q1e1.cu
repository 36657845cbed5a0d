// res_launch_q1e1.cu -- resident-kernel instantiations for QC = True, early stop = True.
#include "res_launch_impl.cuh"

namespace ldpc {
LDPC_RES_QE_DEF(1, 1)
}  // namespace ldpc
