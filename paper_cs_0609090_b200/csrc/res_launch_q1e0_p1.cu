// res_launch_q1e0_p1.cu -- resident-kernel instantiations for QC = True, early stop = False:
// the 1-bit and full-message formats (res_launch_impl.cuh dispatch_qe PART 1).
#include "res_launch_impl.cuh"

namespace ldpc {
LDPC_RES_QE_DEF(1, 0, 1)
}  // namespace ldpc
