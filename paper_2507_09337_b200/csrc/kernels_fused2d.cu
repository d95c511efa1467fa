// kernels_fused2d.cu -- the whole telescoped SSP-RK2 step of a 2D block in
// ONE kernel, U1 kept on chip (SURVEY 7 M4 "the fully fused single-kernel
// step"; A5-A9 in 2D: BASELINE configs[0] / [1] and large 2D Sedov grids).
//
// A 2D block with its guards (16^2 + 4 guards: 24^2 cells x 5 variables =
// 23 KB) fits in shared memory whole, so one CTA per block does:
//   1. EOS of the padded block (global -> primitives in smem);
//   2. stage 1 on the box [-2, n+2)^2: every x- and y-face flux once (PLM +
//      Riemann, face_flux<D, SCH>), then U1 = U^n - dt D(U^n), kept in smem
//      (conserved) and converted to primitives in place of U^n's;
//   3. stage 2 on the interior: faces from the U1 primitives, then
//      U^{n+1} = 0.5 (U^n + (U1 - dt D(U1))) written in place, and the CFL
//      signal speed of the new state reduced per CTA (the fused dt epilogue).
// No U1 round trip through HBM and one launch per step.  The guard cells must
// be materialised (the FULL fill: 2D grids do not use the gather fill mode).
// Expression order is hydro_math.cuh's: the parity build is bitwise equal to
// the reference kernels and the oracle; D = (dFx) idx + (dFy) idy (A8, 2D).
#include <cfloat>

#include "hydro_math.cuh"
#include "orcha_internal.h"
#include "reduce.cuh"

namespace orcha {

template <int NB>
struct Geo2 {
  static constexpr int P = NB + 8;            // padded extent (ng = 4)
  static constexpr int W1 = NB + 4;           // stage-1 box width
  static constexpr int FX1 = W1 * (W1 + 1);   // stage-1 x-faces (= y-faces)
  static constexpr int NT = NB >= 16 ? 256 : 128;
  static constexpr int MINB = NB >= 16 ? 3 : 6;  // CTAs per SM: 3 x 73 KB / 6 x 29 KB of smem, <= 85 registers
  static constexpr size_t SMEM = sizeof(double) * (size_t)(5 * P * P + 5 * W1 * W1 + 2 * 5 * FX1);
};

template <int NB, int SCH>
__global__ void __launch_bounds__(Geo2<NB>::NT, Geo2<NB>::MINB) step2d_kernel(DevGrid G, double* __restrict__ state,
                                                               const SlotInfo* __restrict__ slots,
                                                               const double* __restrict__ d_dt, double h_dt,
                                                               DtRecord* __restrict__ rec, DevStatus* st) {
  using C = Geo2<NB>;
  constexpr int P = C::P, W1 = C::W1, NT = C::NT, PP = P * P, WW = W1 * W1, FX1 = C::FX1;
  extern __shared__ __align__(16) double sm[];
  double* Q = sm;              // [5][P][P] primitives: of U^n, then (box cells) of U1
  double* U1 = Q + 5 * PP;     // [5][W1][W1] conserved U1 on the box
  double* Fx = U1 + 5 * WW;    // stage 1: [5][W1][W1+1]; stage 2: [5][NB][NB+1]
  double* Fy = Fx + 5 * FX1;   // stage 1: [5][W1+1][W1]; stage 2: [5][NB+1][NB]
  const int tid = threadIdx.x;
  const long long slot = blockIdx.x;
  const long long cube = G.cube;
  double* blk = state + slot * kNVar * cube;  // padded plane: cell (i, j) at (j + 4) P + i + 4
  const SlotInfo si = slots[slot];
  const double dt = d_dt ? *d_dt : h_dt;
  auto gcell = [&](int i, int j) -> long long {
    return ((long long)si.bc[1] * NB + j) * G.N[0] + ((long long)si.bc[0] * NB + i);
  };
  auto put = [&](double* a, int stride, int o, const Prim& q) {
    a[o] = q.r;
    a[stride + o] = q.u;
    a[2 * stride + o] = q.v;
    a[3 * stride + o] = q.w;
    a[4 * stride + o] = q.p;
  };
  auto get = [&](int o) -> Prim { return Prim{Q[o], Q[PP + o], Q[2 * PP + o], Q[3 * PP + o], Q[4 * PP + o]}; };
  unsigned long long hits = 0;

  // 1. primitives of the padded block (floor hits / non-physical: interior cells)
  for (int c = tid; c < PP; c += NT) {
    const int jp = c / P, ip = c - jp * P;
    bool fl;
    const Prim q = (SCH == 0) ? eos(blk[c], blk[cube + c], blk[2 * cube + c], blk[3 * cube + c], blk[4 * cube + c], G,
                                    &fl)
                              : eos_var(blk[c], blk[cube + c], blk[2 * cube + c], blk[3 * cube + c],
                                        blk[4 * cube + c], G, &fl);
    put(Q, PP, c, q);
    const int i = ip - 4, j = jp - 4;
    if (i >= 0 && i < NB && j >= 0 && j < NB) {
      hits += fl ? 1 : 0;
      if (!(blk[c] > 0.0)) atomicMin(&st->first_bad, (unsigned long long)gcell(i, j));
    }
  }
  __syncthreads();

  // 2a. stage-1 faces on the box: x-face (row j, between cells i-1 and i),
  //     i, j in [-2, n+2]; index (j+2)(W1+1) + (i+2) / y-face (j+2) W1 + (i+2)
  for (int t = tid; t < FX1; t += NT) {
    const int r = t / (W1 + 1), f = t - r * (W1 + 1);
    const int o = (r + 2) * P + f;  // padded offset of cell (i-2, j): i = f-2, j = r-2 -> (f-4+4), (r-2+4)
    face_flux<0, SCH>(get(o), get(o + 1), get(o + 2), get(o + 3), G, Fx + t, FX1);
  }
  for (int t = tid; t < FX1; t += NT) {
    const int f = t / W1, i = t - f * W1;
    const int o = f * P + (i + 2);  // cell (i-2, j-2) with j = f-2: padded row f, column i+2
    face_flux<1, SCH>(get(o), get(o + P), get(o + 2 * P), get(o + 3 * P), G, Fy + t, FX1);
  }
  __syncthreads();

  // 2b. U1 = U^n - dt D(U^n) on the box, kept conserved, and its primitives in
  //     place of U^n's (the box cells only; nothing reads Q until the barrier)
  for (int c = tid; c < WW; c += NT) {
    const int r = c / W1, i = c - r * W1;  // box cell (i-2, r-2)
    const int po = (r + 2) * P + (i + 2);
    double u1[5];
#pragma unroll
    for (int v = 0; v < 5; v++) {
      const double tx = (Fx[v * FX1 + r * (W1 + 1) + i + 1] - Fx[v * FX1 + r * (W1 + 1) + i]) * G.id[0];
      const double ty = (Fy[v * FX1 + (r + 1) * W1 + i] - Fy[v * FX1 + r * W1 + i]) * G.id[1];
      const double D = tx + ty;
      u1[v] = blk[v * cube + po] - dt * D;
      U1[v * WW + c] = u1[v];
    }
    bool fl;
    const Prim q = (SCH == 0) ? eos(u1[0], u1[1], u1[2], u1[3], u1[4], G, &fl)
                              : eos_var(u1[0], u1[1], u1[2], u1[3], u1[4], G, &fl);
    put(Q, PP, po, q);
    if (r >= 2 && r < NB + 2 && i >= 2 && i < NB + 2) hits += fl ? 1 : 0;
  }
  __syncthreads();

  // 3a. stage-2 faces on the interior (from U1's primitives)
  constexpr int FX2 = NB * (NB + 1);
  for (int t = tid; t < FX2; t += NT) {
    const int j = t / (NB + 1), f = t - j * (NB + 1);  // between cells f-1 and f of row j
    const int o = (j + 4) * P + (f + 2);
    face_flux<0, SCH>(get(o), get(o + 1), get(o + 2), get(o + 3), G, Fx + t, FX2);
  }
  for (int t = tid; t < FX2; t += NT) {
    const int f = t / NB, i = t - f * NB;  // between rows f-1 and f of column i
    const int o = (f + 2) * P + (i + 4);
    face_flux<1, SCH>(get(o), get(o + P), get(o + 2 * P), get(o + 3 * P), G, Fy + t, FX2);
  }
  __syncthreads();

  // 3b. U^{n+1} = 0.5 (U^n + (U1 - dt D(U1))) in place + the dt epilogue
  double s_rec = -DBL_MAX;
  long long g_rec = LLONG_MAX;
  for (int c = tid; c < NB * NB; c += NT) {
    const int j = c / NB, i = c - j * NB;
    const int po = (j + 4) * P + (i + 4), bo = (j + 2) * W1 + (i + 2);
    double nw[5];
#pragma unroll
    for (int v = 0; v < 5; v++) {
      const double tx = (Fx[v * FX2 + j * (NB + 1) + i + 1] - Fx[v * FX2 + j * (NB + 1) + i]) * G.id[0];
      const double ty = (Fy[v * FX2 + (j + 1) * NB + i] - Fy[v * FX2 + j * NB + i]) * G.id[1];
      const double D = tx + ty;
      nw[v] = 0.5 * (blk[v * cube + po] + (U1[v * WW + bo] - dt * D));
    }
#pragma unroll
    for (int v = 0; v < 5; v++) blk[v * cube + po] = nw[v];
    bool f2;
    const Prim q = (SCH == 0) ? eos(nw[0], nw[1], nw[2], nw[3], nw[4], G, &f2)
                              : eos_var(nw[0], nw[1], nw[2], nw[3], nw[4], G, &f2);
    const double s = (SCH == 0) ? signal_speed<2>(q, G) : signal_speed_var<2>(q, G);
    const long long g = gcell(i, j);
    if (dt_better(s, g, s_rec, g_rec)) { s_rec = s; g_rec = g; }
    const bool finite = isfinite(nw[0]) && isfinite(nw[1]) && isfinite(nw[2]) && isfinite(nw[3]) && isfinite(nw[4]);
    if (!(nw[0] > 0.0) || !finite) atomicMin(&st->first_bad, (unsigned long long)g);
  }
  if (hits) atomicAdd(&st->floor_hits, hits);
  block_reduce_rec<NT>(s_rec, g_rec);
  if (tid == 0) {
    rec[blockIdx.x].s = s_rec;
    rec[blockIdx.x].g = g_rec;
  }
}

template <int NB, int SCH>
static cudaError_t launch2d(const DevGrid& G, double* state, int nslots, const SlotInfo* slots, const double* d_dt,
                           double h_dt, DtRecord* records, long long* nrecords, DevStatus* st, cudaStream_t s) {
  using C = Geo2<NB>;
  static const cudaError_t attr = cudaFuncSetAttribute(step2d_kernel<NB, SCH>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (attr != cudaSuccess) return attr;
  {
    // one kernel does both stages: the phase is reported as stage 1
    PhaseScope ph(PH_STAGE1, s);
    step2d_kernel<NB, SCH><<<nslots, C::NT, C::SMEM, s>>>(G, state, slots, d_dt, h_dt, records, st);
  }
  count_launch();
  *nrecords = nslots;
  return cudaGetLastError();
}

// 2D blocks of 8^2 or 16^2 cells with ng = 4.
bool fused2d_supported(const DevGrid& G) {
  return G.ndim == 2 && G.ng == 4 && G.nb[0] == G.nb[1] && (G.nb[0] == 8 || G.nb[0] == 16);
}

cudaError_t launch_advance_fused2d(const DevGrid& G, double* state, int nslots, const SlotInfo* slots,
                                   const double* d_dt, double h_dt, DtRecord* records, long long* nrecords,
                                   DevStatus* st, cudaStream_t s) {
  const bool var = G.riemann != 0 || G.limiter != 0 || G.eos != 0;
  if (G.nb[0] == 16)
    return var ? launch2d<16, 1>(G, state, nslots, slots, d_dt, h_dt, records, nrecords, st, s)
               : launch2d<16, 0>(G, state, nslots, slots, d_dt, h_dt, records, nrecords, st, s);
  return var ? launch2d<8, 1>(G, state, nslots, slots, d_dt, h_dt, records, nrecords, st, s)
             : launch2d<8, 0>(G, state, nslots, slots, d_dt, h_dt, records, nrecords, st, s);
}

}  // namespace orcha
