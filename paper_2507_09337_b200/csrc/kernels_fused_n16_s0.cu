// kernels_fused_n16_s0.cu -- fused stage kernels for 16^3 blocks, scheme 0
// (minmod + HLL, the paper path); see fused_impl.cuh.
#include "fused_impl.cuh"

namespace orcha {
ORCHA_FUSED_TU(16, 0)
}  // namespace orcha
