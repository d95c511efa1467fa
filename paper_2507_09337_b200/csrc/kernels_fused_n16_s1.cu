// kernels_fused_n16_s1.cu -- fused stage kernels for 16^3 blocks, scheme 1
// (the grid's F4 flags: MC / HLLC); see fused_impl.cuh.
#include "fused_impl.cuh"

namespace orcha {
ORCHA_FUSED_TU(16, 1)
}  // namespace orcha
