// res_launch_q1e0_p0.cu -- resident-kernel instantiations for QC = True, early stop = False:
// the COMPACT format and the fp32 layered kernel (res_launch_impl.cuh dispatch_qe PART 0).
#include "res_launch_impl.cuh"

namespace ldpc {
LDPC_RES_QE_DEF(1, 0, 0)
}  // namespace ldpc
