// kernels_unit.cu -- unit entry points: the per-cell / per-face device
// functions the fused kernels call (hydro_math.cuh), applied to n independent
// inputs, so tests can fuzz them against the oracle's functions on SURVEY
// 8(d)'s seeded distribution (rho ~ logU[1e-2,1e2], p ~ logU[1e-6,1e3],
// v ~ U[-3,3] c: sub- and supersonic faces alike).  Test diagnostics only; the
// hot path never calls them.  Scheme selection is the fused kernels': the
// paper-path functions (minmod + HLL, production algebra in the production
// build) when the grid sets no F4 flag, the F4 variants otherwise.
#include "hydro_math.cuh"
#include "orcha_internal.h"

namespace orcha {

template <int SCH>
__global__ void unit_eos_kernel(DevGrid G, long long n, const double* __restrict__ U, double* __restrict__ Q,
                                double* __restrict__ c, double* __restrict__ s, int32_t* __restrict__ floored) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool f;
  const Prim q = (SCH == 0) ? eos(U[i], U[n + i], U[2 * n + i], U[3 * n + i], U[4 * n + i], G, &f)
                            : eos_var(U[i], U[n + i], U[2 * n + i], U[3 * n + i], U[4 * n + i], G, &f);
  Q[i] = q.r;
  Q[n + i] = q.u;
  Q[2 * n + i] = q.v;
  Q[3 * n + i] = q.w;
  Q[4 * n + i] = q.p;
  c[i] = (SCH == 0) ? sound_speed(q, G) : sound_speed_var(q, G);
  s[i] = (SCH == 0) ? signal_speed<3>(q, G) : signal_speed_var<3>(q, G);
  floored[i] = f ? 1 : 0;
}

__device__ __forceinline__ Prim load_prim(const double* q, long long n, long long i) {
  return Prim{q[i], q[n + i], q[2 * n + i], q[3 * n + i], q[4 * n + i]};
}

// PLM + Riemann flux of one face from its 4-cell stencil (face_flux<D, SCH>,
// exactly the call the fused kernels make per face task).
template <int D, int SCH>
__global__ void unit_face_flux_kernel(DevGrid G, long long n, const double* __restrict__ q, double* __restrict__ F) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Prim q0 = load_prim(q, n, i), q1 = load_prim(q + 5 * n, n, i), q2 = load_prim(q + 10 * n, n, i),
             q3 = load_prim(q + 15 * n, n, i);
  face_flux<D, SCH>(q0, q1, q2, q3, G, F + i, (int)n);
}

// Riemann flux alone from given face states (hll_store<D> / flux_store_var<D>).
template <int D, int SCH>
__global__ void unit_riemann_kernel(DevGrid G, long long n, const double* __restrict__ qL,
                                    const double* __restrict__ qR, double* __restrict__ F) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Prim L = load_prim(qL, n, i), R = load_prim(qR, n, i);
  if (SCH == 0) hll_store<D>(L, R, G, F + i, (int)n);
  else flux_store_var<D>(L, R, G, F + i, (int)n);
}

static bool variant_scheme(const DevGrid& G) { return G.riemann != 0 || G.limiter != 0 || G.eos != 0; }

static int32_t unit_check(const orcha_grid* g, long long n, int dir) {
  if (!g) return fail(ORCHA_E_ARG, "null grid");
  if (n < 0 || n > (1LL << 31) / 5) return fail(ORCHA_E_ARG, "unit: n out of range [0, 2^31/5]");
  if (dir < 0 || dir > 2) return fail(ORCHA_E_ARG, "unit: dir must be 0, 1 or 2");
  return ORCHA_OK;
}

}  // namespace orcha

using namespace orcha;

extern "C" int32_t orcha_unit_eos(const orcha_grid* g, int64_t n, const double* d_U, double* d_Q, double* d_c,
                                  double* d_s, int32_t* d_floored, void* stream) {
  int32_t rc = unit_check(g, n, 0);
  if (rc) return rc;
  if (n == 0) return ORCHA_OK;
  if (!d_U || !d_Q || !d_c || !d_s || !d_floored) return fail(ORCHA_E_ARG, "unit_eos: null buffer");
  const unsigned nb = (unsigned)((n + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  if (variant_scheme(g->dev)) unit_eos_kernel<1><<<nb, 256, 0, s>>>(g->dev, n, d_U, d_Q, d_c, d_s, d_floored);
  else unit_eos_kernel<0><<<nb, 256, 0, s>>>(g->dev, n, d_U, d_Q, d_c, d_s, d_floored);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ORCHA_OK : cuda_fail(e, "unit_eos");
}

extern "C" int32_t orcha_unit_face_flux(const orcha_grid* g, int32_t dir, int64_t n, const double* d_q,
                                        double* d_F, void* stream) {
  int32_t rc = unit_check(g, n, dir);
  if (rc) return rc;
  if (n == 0) return ORCHA_OK;
  if (!d_q || !d_F) return fail(ORCHA_E_ARG, "unit_face_flux: null buffer");
  const unsigned nb = (unsigned)((n + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  const bool v = variant_scheme(g->dev);
#define ORCHA_UF(D)                                                                              \
  (v ? unit_face_flux_kernel<D, 1><<<nb, 256, 0, s>>>(g->dev, n, d_q, d_F)                      \
     : unit_face_flux_kernel<D, 0><<<nb, 256, 0, s>>>(g->dev, n, d_q, d_F))
  if (dir == 0) ORCHA_UF(0);
  else if (dir == 1) ORCHA_UF(1);
  else ORCHA_UF(2);
#undef ORCHA_UF
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ORCHA_OK : cuda_fail(e, "unit_face_flux");
}

extern "C" int32_t orcha_unit_riemann(const orcha_grid* g, int32_t dir, int64_t n, const double* d_qL,
                                      const double* d_qR, double* d_F, void* stream) {
  int32_t rc = unit_check(g, n, dir);
  if (rc) return rc;
  if (n == 0) return ORCHA_OK;
  if (!d_qL || !d_qR || !d_F) return fail(ORCHA_E_ARG, "unit_riemann: null buffer");
  const unsigned nb = (unsigned)((n + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  const bool v = variant_scheme(g->dev);
#define ORCHA_UR(D)                                                                              \
  (v ? unit_riemann_kernel<D, 1><<<nb, 256, 0, s>>>(g->dev, n, d_qL, d_qR, d_F)                 \
     : unit_riemann_kernel<D, 0><<<nb, 256, 0, s>>>(g->dev, n, d_qL, d_qR, d_F))
  if (dir == 0) ORCHA_UR(0);
  else if (dir == 1) ORCHA_UR(1);
  else ORCHA_UR(2);
#undef ORCHA_UR
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ORCHA_OK : cuda_fail(e, "unit_riemann");
}
