// kernels_fused_n8_s0.cu -- fused stage kernels for 8^3 blocks, scheme 0
// (minmod + HLL, the paper path); see fused_impl.cuh.
#include "fused_impl.cuh"

namespace orcha {
ORCHA_FUSED_TU(8, 0)
}  // namespace orcha
