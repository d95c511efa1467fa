// kernels_fused_n32_s1.cu -- fused stage kernels for 32^3 blocks, scheme 1
// (the grid's F4 flags: MC / HLLC); see fused_impl.cuh.
#include "fused_impl.cuh"

namespace orcha {
ORCHA_FUSED_TU(32, 1)
}  // namespace orcha
