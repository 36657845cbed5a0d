// res_launch_q0e0.cu -- resident-kernel instantiations for QC = False, early stop = False.
#include "res_launch_impl.cuh"

namespace ldpc {
LDPC_RES_QE_DEF(0, 0, 2)
}  // namespace ldpc
