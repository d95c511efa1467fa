// probe.cu -- measured fp64-pipe peak of this GPU (the denominator of the
// bench's "alu" roofline beside the value derived from unit counts and the
// clock: 148 SMs x 64 fp64 lanes x f_SM, B200_PROFILING.md).  Not part of
// the method.
#include "orcha_internal.h"

namespace orcha {

// 8 independent DFMA chains per thread (enough ILP to cover the DFMA
// latency at 16 warps per SM sub-partition); the result is stored so the
// chains are live.
__global__ void __launch_bounds__(256) dfma_probe_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; c++) x[c] = (double)(threadIdx.x + c) * 1e-3;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int c = 0; c < 8; c++) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; c++) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace orcha

using namespace orcha;

extern "C" int32_t orcha_probe_fp64(int32_t iters, double* tinst_per_s, double* ms_out, void* stream) {
  if (!tinst_per_s || iters < 1) return fail(ORCHA_E_ARG, "orcha_probe_fp64: null output or iters < 1");
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_fail(e, "probe: device query");
  const int blocks = sms * 8, threads = 256;  // 64 warps per SM
  cudaStream_t s = (cudaStream_t)stream;
  double* out = nullptr;
  cudaEvent_t a, b;
  e = cudaMalloc(&out, sizeof(double) * blocks * threads);
  if (e == cudaSuccess) e = cudaEventCreate(&a);
  if (e == cudaSuccess) e = cudaEventCreate(&b);
  if (e != cudaSuccess) return cuda_fail(e, "probe: setup");
  dfma_probe_kernel<<<blocks, threads, 0, s>>>(out, iters / 10 + 1, 0.999999, 1e-9);  // warm-up
  cudaEventRecord(a, s);
  dfma_probe_kernel<<<blocks, threads, 0, s>>>(out, iters, 0.999999, 1e-9);
  cudaEventRecord(b, s);
  e = cudaEventSynchronize(b);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
  count_launch(2);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  if (e != cudaSuccess) return cuda_fail(e, "probe: run");
  *tinst_per_s = (double)blocks * threads * 8.0 * iters / (ms * 1e-3) / 1e12;
  if (ms_out) *ms_out = ms;
  return ORCHA_OK;
}
