// res_launch_q0e0_p1.cu -- resident-kernel instantiations for QC = False, early stop = False:
// the 1-bit and full-message formats (res_launch_impl.cuh dispatch_qe PART 1).
#include "res_launch_impl.cuh"

namespace ldpc {
LDPC_RES_QE_DEF(0, 0, 1)
}  // namespace ldpc
