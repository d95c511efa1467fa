// kernels_ref.cu -- reference ("one thread per output cell") stage kernels of
// the telescoped SSP-RK2 step.  Simple and slow: each thread evaluates the two
// face fluxes per axis of its own cell, recomputing primitives of the 5-cell
// stencil.  Kept as the structural reference the fused kernel is checked
// against bitwise (both under the parity build), and as variant 0.
#include <cfloat>

#include "hydro_math.cuh"
#include "orcha_internal.h"
#include "reduce.cuh"

namespace orcha {

__device__ __forceinline__ Prim load_prim(const double* __restrict__ p, long long cube, const DevGrid& G,
                                          bool* fl) {
  return eos_var(p[0], p[cube], p[2 * cube], p[3 * cube], p[4 * cube], G, fl);
}

// D(U) at cell c (offset `o` in the padded cube) along axis AX, accumulated
// into D exactly as ((dFx)*idx + (dFy)*idy) + (dFz)*idz (A8).
template <int AX>
__device__ __forceinline__ void accumulate_axis(const double* __restrict__ in, long long o, long long stride,
                                                const DevGrid& G, double D[5], bool* floored_center) {
  const long long cube = G.cube;
  Prim q[5];
#pragma unroll
  for (int s = 0; s < 5; s++) {
    bool fl;
    q[s] = load_prim(in + o + (s - 2) * stride, cube, G, &fl);
    if (s == 2) *floored_center = fl;
  }
  Prim L, R;
  double Fm[5], Fp[5];
  plm_face_var(q[0], q[1], q[2], q[3], G, &L, &R);  // face c-1/2
  if (G.riemann == 1) hllc_store<AX>(L, R, G, Fm, 1);
  else hll_store_lit<AX>(L, R, G, Fm, 1);
  plm_face_var(q[1], q[2], q[3], q[4], G, &L, &R);  // face c+1/2
  if (G.riemann == 1) hllc_store<AX>(L, R, G, Fp, 1);
  else hll_store_lit<AX>(L, R, G, Fp, 1);
#pragma unroll
  for (int v = 0; v < 5; v++) {
    double t = (Fp[v] - Fm[v]) * G.id[AX];
    D[v] = (AX == 0) ? t : (D[v] + t);
  }
}

// STAGE 1: region = box [-2, n+2) per active axis; U1 = U^n - dt*D(U^n) -> u1.
// STAGE 2: region = interior; U^{n+1} = 0.5*(U^n + (U1 - dt*D(U1))) -> state,
//          then the fused dt epilogue (s of U^{n+1}, one record per CTA).
// RING = width of the stage-1 ring beyond the interior: 2 for the telescoped
// step, 0 for the per-stage variant (F1, U1 guards refilled between stages).
template <int NDIM, int STAGE, int RING = 2>
__global__ void __launch_bounds__(256) stage_ref_kernel(DevGrid G, double* __restrict__ state,
                                                        double* __restrict__ u1, long long total,
                                                        const SlotInfo* __restrict__ slots,
                                                        const double* __restrict__ d_dt, double h_dt,
                                                        DtRecord* __restrict__ rec, DevStatus* st) {
  const int w = (STAGE == 1) ? RING : 0;
  int E[3];
#pragma unroll
  for (int d = 0; d < 3; d++) E[d] = (d < NDIM) ? G.nb[d] + 2 * w : 1;
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double s_rec = -DBL_MAX;
  long long g_rec = LLONG_MAX;
  if (t < total) {
    long long ncell = (long long)E[0] * E[1] * E[2];
    long long slot = t / ncell;
    long long c = t - slot * ncell;
    int i = (int)(c % E[0]) - ((NDIM > 0) ? w : 0);
    int j = (int)((c / E[0]) % E[1]) - ((NDIM > 1) ? w : 0);
    int k = (int)(c / ((long long)E[0] * E[1])) - ((NDIM > 2) ? w : 0);
    const double dt = d_dt ? *d_dt : h_dt;
    const long long cube = G.cube;
    const long long base = slot * kNVar * cube;
    const long long o = cell_off(G, i, j, k);
    const double* in = (STAGE == 1) ? state + base : u1 + base;
    double D[5];
    bool floored = false, fl;
    accumulate_axis<0>(in, o, 1, G, D, &floored);
    if (NDIM > 1) accumulate_axis<1>(in, o, G.P[0], G, D, &fl);
    if (NDIM > 2) accumulate_axis<2>(in, o, (long long)G.P[0] * G.P[1], G, D, &fl);
    bool inside = i >= 0 && i < G.nb[0] && j >= 0 && j < G.nb[1] && k >= 0 && k < G.nb[2];
    SlotInfo si = slots[slot];
    long long gcell = (((long long)si.bc[2] * G.nb[2] + k) * G.N[1] + ((long long)si.bc[1] * G.nb[1] + j)) * G.N[0] +
                      ((long long)si.bc[0] * G.nb[0] + i);
    if (inside && floored) atomicAdd(&st->floor_hits, 1ull);
    if (STAGE == 1) {
      double* out = u1 + base + o;
      const double* un = state + base + o;
#pragma unroll
      for (int v = 0; v < 5; v++) out[v * cube] = un[v * cube] - dt * D[v];
      if (inside && !(un[0] > 0.0)) atomicMin(&st->first_bad, (unsigned long long)gcell);
    } else {
      double* un = state + base + o;
      const double* v1 = u1 + base + o;
      double nw[5];
#pragma unroll
      for (int v = 0; v < 5; v++) nw[v] = 0.5 * (un[v * cube] + (v1[v * cube] - dt * D[v]));
#pragma unroll
      for (int v = 0; v < 5; v++) un[v * cube] = nw[v];
      bool f2;
      Prim q = eos_var(nw[0], nw[1], nw[2], nw[3], nw[4], G, &f2);
      s_rec = signal_speed_var<NDIM>(q, G);
      g_rec = gcell;
      bool finite = isfinite(nw[0]) && isfinite(nw[1]) && isfinite(nw[2]) && isfinite(nw[3]) && isfinite(nw[4]);
      if (!(nw[0] > 0.0) || !finite) atomicMin(&st->first_bad, (unsigned long long)gcell);
    }
  }
  if (STAGE == 2) {
    block_reduce_rec<256>(s_rec, g_rec);
    if (threadIdx.x == 0) { rec[blockIdx.x].s = s_rec; rec[blockIdx.x].g = g_rec; }
  }
}

template <int NDIM>
static cudaError_t launch_ref(const DevGrid& G, double* state, double* u1, int nslots, const SlotInfo* slots,
                              const double* d_dt, double h_dt, DtRecord* records, long long* nrecords,
                              DevStatus* st, cudaStream_t s) {
  long long c1 = 1, c2 = 1;
  for (int d = 0; d < NDIM; d++) { c1 *= G.nb[d] + 4; c2 *= G.nb[d]; }
  long long t1 = nslots * c1, t2 = nslots * c2;
  {
    PhaseScope ph(PH_STAGE1, s);
    stage_ref_kernel<NDIM, 1><<<(unsigned)((t1 + 255) / 256), 256, 0, s>>>(G, state, u1, t1, slots, d_dt, h_dt,
                                                                            records, st);
  }
  {
    PhaseScope ph(PH_STAGE2, s);
    stage_ref_kernel<NDIM, 2><<<(unsigned)((t2 + 255) / 256), 256, 0, s>>>(G, state, u1, t2, slots, d_dt, h_dt,
                                                                            records, st);
  }
  count_launch(2);
  *nrecords = (t2 + 255) / 256;
  return cudaGetLastError();
}

cudaError_t launch_advance_ref(const DevGrid& G, double* state, double* u1, int nslots, const SlotInfo* slots,
                               const double* d_dt, double h_dt, DtRecord* records, long long* nrecords,
                               DevStatus* st, cudaStream_t s) {
  if (G.ndim == 1) return launch_ref<1>(G, state, u1, nslots, slots, d_dt, h_dt, records, nrecords, st, s);
  if (G.ndim == 2) return launch_ref<2>(G, state, u1, nslots, slots, d_dt, h_dt, records, nrecords, st, s);
  return launch_ref<3>(G, state, u1, nslots, slots, d_dt, h_dt, records, nrecords, st, s);
}

// One stage of the per-stage variant (F1) with the reference kernels:
// stage 1 on the interior (RING 0) into the padded U1, stage 2 as above.
template <int NDIM>
static cudaError_t stage_ref(const DevGrid& G, int stage, double* state, double* u1, int nslots,
                             const SlotInfo* slots, const double* d_dt, double h_dt, DtRecord* records,
                             long long* nrecords, DevStatus* st, cudaStream_t s) {
  long long c = 1;
  for (int d = 0; d < NDIM; d++) c *= G.nb[d];
  long long t = nslots * c;
  unsigned blocks = (unsigned)((t + 255) / 256);
  PhaseScope ph(stage == 1 ? PH_STAGE1 : PH_STAGE2, s);
  if (stage == 1) {
    stage_ref_kernel<NDIM, 1, 0><<<blocks, 256, 0, s>>>(G, state, u1, t, slots, d_dt, h_dt, records, st);
  } else {
    stage_ref_kernel<NDIM, 2><<<blocks, 256, 0, s>>>(G, state, u1, t, slots, d_dt, h_dt, records, st);
    *nrecords = blocks;
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_stage_ref(const DevGrid& G, int stage, double* state, double* u1, int nslots,
                             const SlotInfo* slots, const double* d_dt, double h_dt, DtRecord* records,
                             long long* nrecords, DevStatus* st, cudaStream_t s) {
  if (G.ndim == 1) return stage_ref<1>(G, stage, state, u1, nslots, slots, d_dt, h_dt, records, nrecords, st, s);
  if (G.ndim == 2) return stage_ref<2>(G, stage, state, u1, nslots, slots, d_dt, h_dt, records, nrecords, st, s);
  return stage_ref<3>(G, stage, state, u1, nslots, slots, d_dt, h_dt, records, nrecords, st, s);
}

}  // namespace orcha
