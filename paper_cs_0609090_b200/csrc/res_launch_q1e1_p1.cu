// res_launch_q1e1_p1.cu -- resident-kernel instantiations for QC = True, early stop = True:
// the 1-bit and full-message formats (res_launch_impl.cuh dispatch_qe PART 1).
#include "res_launch_impl.cuh"

namespace ldpc {
LDPC_RES_QE_DEF(1, 1, 1)
}  // namespace ldpc
