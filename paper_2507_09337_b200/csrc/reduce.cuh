// reduce.cuh -- deterministic (s, g) max-reduction helpers for the CFL dt (A4).
#pragma once
#include <cfloat>
#include <climits>

#include "orcha_internal.h"

namespace orcha {

// ------------------------------------------------------ dt reductions --
__device__ __forceinline__ void rec_combine(double& s, long long& g, double s2, long long g2) {
  if (dt_better(s2, g2, s, g)) { s = s2; g = g2; }
}

// Block-wide (s, g) reduction; result valid in thread 0.
template <int NT>
__device__ __forceinline__ void block_reduce_rec(double& s, long long& g) {
  __shared__ double ss[NT / 32];
  __shared__ long long sg[NT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double s2 = __shfl_down_sync(0xffffffffu, s, o);
    long long g2 = __shfl_down_sync(0xffffffffu, g, o);
    rec_combine(s, g, s2, g2);
  }
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { ss[w] = s; sg[w] = g; }
  __syncthreads();
  if (w == 0) {
    s = (lane < NT / 32) ? ss[lane] : -DBL_MAX;
    g = (lane < NT / 32) ? sg[lane] : LLONG_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double s2 = __shfl_down_sync(0xffffffffu, s, o);
      long long g2 = __shfl_down_sync(0xffffffffu, g, o);
      rec_combine(s, g, s2, g2);
    }
  }
}

}  // namespace orcha
