// res_launch_q0e1_p0.cu -- resident-kernel instantiations for QC = False, early stop = True:
// the COMPACT format and the fp32 layered kernel (res_launch_impl.cuh dispatch_qe PART 0).
#include "res_launch_impl.cuh"

namespace ldpc {
LDPC_RES_QE_DEF(0, 1, 0)
}  // namespace ldpc
