// res_launch_q0e1.cu -- resident-kernel instantiations for QC = False, early stop = True.
#include "res_launch_impl.cuh"

namespace ldpc {
LDPC_RES_QE_DEF(0, 1, 2)
}  // namespace ldpc
