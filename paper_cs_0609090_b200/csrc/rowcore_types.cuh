// rowcore_types.cuh -- plain-data parameter blocks of the row core (rowcore.cuh),
// shared with the host planner through args.cuh.
#pragma once
#include <cstdint>

namespace ldpc {

// Check-node variant of one iteration on doubled values:
//   offset : |L| = min(max(min - beta, 0), Q)                       (readings D5, D6)
//   norm   : |L| = min(max(floor(lambda min) - beta, 0), Q), lambda = na / 2^ns  (D27)
struct VarK {
    uint32_t nbeta2p1, q2p1;   // offset path: packed (1 - 2 beta), (2Q + 1)
    uint32_t norm;             // 0: offset path; 1: normalized path
    uint32_t na, ns, nmask;    // normalized: lambda = na / 2^ns; lane mask (0xFFFF >> ns) & 0xFFFE, both lanes
    uint32_t nb2, q2;          // normalized: packed (-2 beta); both paths: (2Q)
    uint32_t nb8;              // offset path on 0x8000-biased magnitudes: packed (0x8000 - 2 beta)
};

}  // namespace ldpc
