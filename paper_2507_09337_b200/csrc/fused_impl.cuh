// fused_impl.cuh -- the performance advance: per-stage fused z-marching
// kernels (sm_100a, fp64).  Included by one translation unit per (block
// size, scheme) -- kernels_fused_n<NB>_s<SCH>.cu -- so the instantiations
// compile in parallel; kernels_fused.cu dispatches.
//
// A CTA owns a band of H output rows of one block's output x-y plane (16^3
// blocks: two bands per block, so 2-3 independent CTAs share an SM and one
// CTA's barrier is covered by another's work) and marches over the output
// z-planes of the stage.  Its input rows of each plane (5 variables x
// (H+4) rows x the padded row length -- a contiguous run per variable in the
// block-major SoA packet) are staged into a 5-deep shared-memory ring by bulk
// async copies (cp.async.bulk -> UBLKCP, completion on an mbarrier), and
// converted to primitives in place (EOS).  Per output plane k:
//   phase 1: every x-, y- and z-face flux of the band is one task (PLM/minmod
//            from the 4-cell stencil, then HLL), computed exactly once and
//            written to shared memory; tasks are dealt in warp-sized slots of
//            one direction (no divergence, no selects); z-faces k+1/2 are
//            double buffered so the k-1/2 ones survive the plane;
//   phase 2: the conservative update of the band's cells of plane k, and the
//            EOS of the next staged plane (measured: doing that EOS in phase
//            1 instead is slower, 3.44 vs 3.34 ms per cfg4 step).
// Stage 1 (box: interior + 2-cell ring) writes U1 to an (n+4)^3 scratch;
// stage 2 (interior) reads it, writes U^{n+1} in place and reduces the CFL
// signal speed of the new state (fused dt epilogue).  SURVEY 8(a) A5-A9;
// P:L665-674 sec 6.
//
// Expression order is that of hydro_math.cuh: the parity
// build of this kernel is bitwise equal to the reference kernel and the
// oracle.  The production build uses hydro_math.cuh's reciprocal / rsqrt
// refinements instead of IEEE divide and sqrt.
#pragma once

#include <cfloat>
#include <cstdlib>
#include <cstdint>

#include "hydro_math.cuh"
#include "orcha_internal.h"
#include "push.cuh"
#include "reduce.cuh"

// phase-2 converts by the warps without update cells only (ORCHA_CONV_SPLIT=0: by all threads)
#ifndef ORCHA_CONV_SPLIT
#define ORCHA_CONV_SPLIT 1
#endif
#ifndef ORCHA_CONV_BAL
#define ORCHA_CONV_BAL 0
#endif
// face-task rounds per warp (16^3 / 32^3): stage 1 (and both per-stage
// stages, and 32^3 blocks) / telescoped 16^3 stage 2 (3: 5-warp CTAs, 3 per
// SM; measured best -- 32^3 stage 2 is faster with 2: 5.57 vs 5.36 G)
#ifndef ORCHA_ROUNDS1
#define ORCHA_ROUNDS1 2
#endif
#ifndef ORCHA_ROUNDS2
#define ORCHA_ROUNDS2 3
#endif
// telescoped 16^3 stages: warps beyond the face-slot count (they convert in
// phase 2); stage 1: 12 warps instead of 11, 3.17 vs 3.22 ms per cfg4 step
#ifndef ORCHA_EXTRA_WARPS1
#define ORCHA_EXTRA_WARPS1 1
#endif
#ifndef ORCHA_EXTRA_WARPS2
#define ORCHA_EXTRA_WARPS2 0
#endif
// the same for the per-stage (F1) kernels and for 32^3 blocks
#ifndef ORCHA_EXTRA_WARPS_PS
#define ORCHA_EXTRA_WARPS_PS 0
#endif
#ifndef ORCHA_EXTRA_WARPS32
#define ORCHA_EXTRA_WARPS32 2
#endif
#ifndef ORCHA_EXTRA_WARPS8_1
#define ORCHA_EXTRA_WARPS8_1 0
#endif
#ifndef ORCHA_EXTRA_WARPS8_2
#define ORCHA_EXTRA_WARPS8_2 2
#endif
// 8^3 blocks: face rounds per warp (0: one warp per 32 cells of the plane)
#ifndef ORCHA_ROUNDS8
#define ORCHA_ROUNDS8 0
#endif
// One CTA barrier per plane instead of two.  The faces of plane it+1 wait
// only for the update warps to have read the face arrays of plane it (an
// mbarrier) instead of a CTA barrier at the end of the plane.  ORCHA_ONEBAR=1:
// the EOS of plane it+5 runs before the barrier that ends the faces phase;
// =2: it stays after it (by the warps without update cells) and the z-face
// tasks of plane it+1, the only readers of plane it+5 there, wait for it on a
// second mbarrier.  0: two CTA barriers per plane.
#ifndef ORCHA_ONEBAR
#define ORCHA_ONEBAR 0
#endif
// z-face carry (ORCHA_ZCARRY: bit 0 stage 1, bit 1 telescoped stage 2, bit 2
// per-stage stage 2; bits 0 and 1 measured faster, bit 1 only with the 4-deep
// ring -- profiles/r02_ab_zcarry*.txt, r02_ab_ring4_zc3.txt): the
// z-face task of a column computes the z-slope of cell k+1 once and keeps
// its upper face state q + s/2 (the left state of face k+3/2) in a
// per-column shared slot for the next plane, instead of recomputing that
// slope there (one slope per z-face instead of two; bitwise the same values)
#ifndef ORCHA_ZCARRY
#define ORCHA_ZCARRY 3
#endif
// x-face slope sharing (ORCHA_XSHFL): an x-face slot deals CELLS to lanes
// (31 new ones per warp, one overlap lane); each lane computes its cell's
// x-slope once, both face states q +- s/2, and takes the right state of its
// face from the next lane (__shfl_down) -- one slope per x-face instead of two
// (bitwise the same values)
#ifndef ORCHA_XSHFL
#define ORCHA_XSHFL 0
#endif
// z fluxes in registers (ORCHA_ZREG): the z-face task of column w runs in
// thread w -- the thread that updates cell w of the plane -- so the flux of
// face k-1/2 stays in its registers for the next plane (and, with the z-face
// carry, the carried face state too): no Fz double buffer, no Zc slots, no
// shared stores / loads of z fluxes; the z slots are the last round of the
// update warps.  Bit 0: stage-1 kernels, bit 1: stage-2 kernels (16^3
// blocks).  The fluxes and carried state hold 20 registers across the plane
// loop, so the stage-1 kernels (80 registers at their 3 / 2 CTAs per SM)
// would spill: stage 2 only by default
#ifndef ORCHA_ZREG
#define ORCHA_ZREG 2
#endif
// row bands per 16^3 block of the borrowed ring's 18 x 18 stage-1 kernel (3: 6-row
// bands, 3 CTAs per SM; 2.205 vs 2.217 ms per cfg4 step with 2, profiles/r02_ab_trim3.txt)
#ifndef ORCHA_TRIM_SPLIT
#define ORCHA_TRIM_SPLIT 3
#endif
// Stage 2 with one CTA barrier per plane (ORCHA_PIPE2): double-buffered x / y
// face arrays, so the faces of plane k+1 need not wait for the updates of
// plane k; the z-face tasks (the only readers of the plane converted in
// phase 2) wait for that EOS on an mbarrier instead of the end-of-plane barrier.
// Measured slower (stage 2 1.055 vs 1.009 ms per cfg4 step): off
#ifndef ORCHA_PIPE2
#define ORCHA_PIPE2 0
#endif
// stage 2: the dt epilogue (EOS + signal speed of the new state) of plane k
// in phase 1 of plane k+1, beside the face tasks (ORCHA_DEFER_DT).  Measured
// slower (2.29 ms, 2.25 with the static schedule, vs 2.19 per cfg4 step,
// profiles/r02_ab_deferdt.txt): off
#ifndef ORCHA_DEFER_DT
#define ORCHA_DEFER_DT 0
#endif
// borrowed-ring stage 1: the x / y ring-push targets of a thread's column
// computed once before the plane loop (ORCHA_PUSH_HOIST)
#ifndef ORCHA_PUSH_HOIST
#define ORCHA_PUSH_HOIST 1
#endif
#ifndef ORCHA_LDNA
#define ORCHA_LDNA 0
#endif
#ifndef ORCHA_STATIC3
#define ORCHA_STATIC3 0
#endif
// ORCHA_ISSUE_LAST=1 (experiment): the last warp issues the staging copies
// 4-deep staging ring for the kernels with the z-face carry (its z-faces
// never read the plane below the output plane after the prologue)
#ifndef ORCHA_RING4
#define ORCHA_RING4 1
#endif
#ifndef ORCHA_ISSUE_LAST
#define ORCHA_ISSUE_LAST 0
#endif

namespace orcha {

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "ORCHA_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra ORCHA_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// read-only global load that does not allocate in L1 (ORCHA_LDNA; the update
// operands are read once per step).  Measured within noise of __ldg (2.193
// vs 2.194 ms per cfg4 step): off
__device__ __forceinline__ double ld_once(const double* p) {
#if ORCHA_LDNA
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// ------------------------------------------------------------- geometry ----
// MODE 0 = telescoped step (stage 1 on the box interior+2, U1 in an (n+4)^3
// scratch, no refill); MODE 1 = per-stage step (both stages
// on the interior, U1 in a padded (n+8)^3 scratch whose guards are refilled
// between the stages).
// WXT / HT (borrowed-ring stage 1 of blocks with one x and/or one y self
// side): output columns and band rows other than the square default; the x /
// y output origin is then chosen per CTA (the self side's 2 ring columns /
// rows).
template <int NB, int STAGE, int SPLIT, int MODE = 0, int WXT = 0, int HT = 0>
struct Geo {
  static constexpr int W0 = (STAGE == 1 && MODE == 0) ? NB + 4 : NB;  // default output columns, rows, planes
  static constexpr int W = WXT ? WXT : W0;                   // output columns per plane
  static constexpr int OFF = (W0 - NB) / 2;                  // default output origin (interior-relative) = -OFF
  static constexpr int K0 = -OFF;                            // first output plane
  static constexpr int NK = W0;                              // output planes
  static constexpr int INO = (STAGE == 1 || MODE == 1) ? 4 : 2;  // input origin offset (guards / ring)
  static constexpr int ORG = INO - 2 - OFF;                  // first staged padded row / plane
  static constexpr int IPX = NB + 2 * INO;                   // padded input row length (= plane rows)
  static constexpr int PLANE = IPX * IPX;                    // doubles per input plane per variable
  static constexpr int NPLANES = NK + 4;                     // input planes streamed
  static constexpr int NSPLIT = SPLIT;                       // row bands per block
  static constexpr int H = HT ? HT : W0 / NSPLIT;           // output rows per CTA
  static constexpr int WY = H * NSPLIT;                      // output rows per plane
  // staged cells converted per band (kernel convert): output rows x output
  // columns +- 2, then the 4 y-halo rows x output columns
  static constexpr int NXR = H * (W + 4);
  static constexpr int NCONV = NXR + 4 * W;
  static constexpr int IR = H + 4;                           // staged input rows per plane
  static constexpr int BAND = IR * IPX;                      // doubles per staged band per variable
  // z-face carry (see ORCHA_ZCARRY): bit 0 stage 1 of both methods, bit 1 the
  // telescoped stage 2, bit 2 the per-stage variant's stage 2; not for 8^3
  // blocks, whose stage 1 fits 3 CTAs per SM without it and 2 with (measured:
  // 3.09 -> 2.59 G cu/s for one packet)
  static constexpr bool ZC = ((ORCHA_ZCARRY >> (STAGE == 1 ? 0 : MODE == 1 ? 2 : 1)) & 1) && NB >= 16;
  // ring depth: the faces of output plane k read staged planes k-1 .. k+2
  // (k .. k+2 with the z-face carry) while plane k+3 is converted and the
  // copy of the next one lands -- 5 slots, 4 with the carry (ORCHA_RING4)
  static constexpr int NS = (ZC && ORCHA_RING4) ? 4 : 5;
  static constexpr int FX = H * (W + 1);                     // x-faces per band
  static constexpr int FY = (H + 1) * W;                     // y-faces per band
  static constexpr int FZ = H * W;                           // z-faces per band (and cells)
  // face tasks are dealt out in warp-sized slots of one direction each; the
  // warp count is chosen so every warp gets two slots (two rounds)
  static constexpr int NCX = H * (W + 2);                    // x-slope cells per band plane (ORCHA_XSHFL)
  static constexpr int SX = ORCHA_XSHFL ? (NCX - 1 + 30) / 31 : (FX + 31) / 32;
  static constexpr int SY = (FY + 31) / 32, SZ = (FZ + 31) / 32;
  static constexpr int NSLOT = SX + SY + SZ;
  static constexpr int RQ = (STAGE == 1 || MODE == 1 || NB != 16) ? ORCHA_ROUNDS1 : ORCHA_ROUNDS2;  // face rounds per warp and plane
  static constexpr int NW8 = (NSLOT + ORCHA_ROUNDS8 - 1) / (ORCHA_ROUNDS8 > 0 ? ORCHA_ROUNDS8 : 1);
  static constexpr int NWU = (FZ + 31) / 32;                 // one update cell per thread
  static constexpr int XW = NB == 32 ? ORCHA_EXTRA_WARPS32
                            : NB != 16 ? 0
                            : MODE == 1 ? ORCHA_EXTRA_WARPS_PS
                                        : (STAGE == 1 ? ORCHA_EXTRA_WARPS1 : ORCHA_EXTRA_WARPS2);
  static constexpr int NW = (NB >= 16) ? (NSLOT + RQ - 1) / RQ + XW
                                       : (ORCHA_ROUNDS8 > 0 ? (NW8 > NWU ? NW8 : NWU) : (W * H + 31) / 32) +
                                             (STAGE == 2 ? ORCHA_EXTRA_WARPS8_2 : ORCHA_EXTRA_WARPS8_1);
  static constexpr int NT = NW * 32;
  static constexpr int ROUNDS = (NSLOT + NW - 1) / NW;
  // z slots in the last round of warps 0 .. SZ-1 (the update warps): the x / y
  // slots must fit the remaining rounds
  static constexpr bool ZREG = ((ORCHA_ZREG >> (STAGE - 1)) & 1) && NB == 16 && !ORCHA_ONEBAR && !ORCHA_XSHFL &&
                               SZ <= NW && SZ * (ROUNDS - 1) + (NW - SZ) * ROUNDS >= SX + SY;
  // ZREG with one x, one y and (warps < SZ) one z slot per warp: the phase-1
  // schedule is static (ORCHA_STATIC3; measured 1.011 vs 1.007 ms for stage 2:
  // off)
  static constexpr bool STATIC3 = ORCHA_STATIC3 && ZREG && SX == NW && SY == NW && ROUNDS == 3 && FZ % 32 == 0;
  static constexpr bool PIPE = ORCHA_PIPE2 && STAGE == 2 && ZREG && !ORCHA_ONEBAR;
  // + mbarriers (NS x 8 B) + per-staged-row sign-flip masks (NS x IR bytes, gather mode)
  // (+ the gather mode's per-row sources of the three z classes, 3 x IR x 16 B: SMEM_G)
  static constexpr size_t SMEM =
      sizeof(double) * (size_t)(NS * 5 * BAND + (PIPE ? 2 : 1) * 5 * (FX + FY) +
                                (ZREG ? 0 : 2 * 5 * FZ + (ZC ? 5 * FZ : 0))) + 64 +
      ((NS * IR + 15) / 16) * 16;
  // gather-mode instantiations also hold the per-row sources (kept out of
  // the plain kernels: 576 more bytes pushed the telescoped stage 2's 3 CTAs
  // past the 196 KB carveout, and its L1 from 60 to 28 KB -- 1.04 -> 1.13 ms)
  static constexpr size_t SMEM_G = SMEM + 3 * IR * 16;
  // CTAs per SM we aim for: shared memory bound (228 KB per SM, 1 KB of it
  // reserved per CTA), at most 8
#ifndef ORCHA_SMEM_PER_SM
#define ORCHA_SMEM_PER_SM 226000
#endif
  static constexpr int MINB_S = (int)(ORCHA_SMEM_PER_SM / (SMEM + 1024));
  static constexpr int MINB_R = 65536 / (NT * (ZREG ? 120 : 80));  // at ~80 registers per thread (~120 with ZREG)
  static constexpr int MINB_SR = MINB_S < MINB_R ? MINB_S : MINB_R;
#ifndef ORCHA_ST2_MINB  // experiments: CTAs per SM the stage-2 kernels are compiled for
#define ORCHA_ST2_MINB 0
#endif
  static constexpr int MINB = (STAGE == 2 && ORCHA_ST2_MINB) ? ORCHA_ST2_MINB
                              : MINB_SR < 1 ? 1 : (MINB_SR > 8 ? 8 : MINB_SR);
  static_assert(NT >= FZ, "one update cell per thread");
  static_assert((BAND * 8) % 16 == 0, "bulk copies need 16-byte multiples");
};

// Interior coordinate whose value the guard coordinate c (side o = -1/0/+1
// of an axis of NB cells) takes under neighbour-table mode m.
template <int NB>
__device__ __forceinline__ int guard_image(int c, int o, int m) {
  return o == 0 ? c : m == kShift ? c - o * NB : m == kClamp ? (o < 0 ? 0 : NB - 1) : (o < 0 ? -1 - c : 2 * NB - 1 - c);
}

// The fused kernels' padded block geometry is known at compile time (ng = 4,
// fused_supported): in-cube offsets in 32-bit arithmetic with constant
// strides instead of cell_off's 64-bit products of DevGrid fields (measured:
// ~50 integer instructions per cell-update of stage 2 went to those).
template <int NB>
__host__ __device__ constexpr int cube_c() {
  return (int)((((long long)(NB + 8) * (NB + 8) * (NB + 8) * 8 + (long long)kAlign - 1) / (long long)kAlign *
                (long long)kAlign) / 8);
}
template <int NB>
__device__ __forceinline__ int coff(int i, int j, int k) {
  return ((k + 4) * (NB + 8) + (j + 4)) * (NB + 8) + (i + 4);
}

// U1 scratch of the fused path: per (slot, var) an (n+4)^3 cube (origin -2),
// 256-byte aligned.
template <int NB>
__host__ __device__ constexpr long long u1_cube() {
  return ((long long)(NB + 4) * (NB + 4) * (NB + 4) * 8 + 255) / 256 * 256 / 8;
}

// The x-axis part of push_cell (push.cuh) for a padded target (the states, or
// the per-stage stage-1 buffers): interior cell (ci, cj, k) feeds the x-guards
// of the blocks the two cached x entries name (gather fill mode).
template <int NB>
__device__ __forceinline__ void push_x(const DevGrid& G, const PushEntry* sxp, int ci, int cj, int k,
                                       const double w[5]) {
  const int side = ci >= NB - 4 ? 1 : (ci < 4 ? 0 : -1);
  if (side < 0 || sxp[side].dst == nullptr) return;
  const PushEntry e = sxp[side];
  const int m = e.mode & 3;
  if (m == kShift) {  // the neighbour's guard: one plain copy (no sign flip)
    double* q = e.dst + coff<NB>(side ? ci - NB : ci + NB, cj, k);
#pragma unroll
    for (int v = 0; v < 5; v++) q[v * cube_c<NB>()] = w[v];
    return;
  }
  int t0, cnt = 1;
  if (m == kShift) t0 = side ? ci - NB : ci + NB;
  else if (m == kMirror) t0 = side ? 2 * NB - 1 - ci : -1 - ci;
  else { cnt = (side ? ci == NB - 1 : ci == 0) ? 4 : 0; t0 = side ? NB : -4; }
  for (int xx = 0; xx < cnt; xx++) {
    double* q = e.dst + coff<NB>(t0 + xx, cj, k);
#pragma unroll
    for (int v = 0; v < 5; v++) q[v * cube_c<NB>()] = ((e.flip >> v) & 1) ? -w[v] : w[v];
  }
}

// Borrowed-ring telescoped step (HYB = 1, stage 1): interior cell (ci, cj, k)
// of U1 also writes the ring (2 deep) of the compact U1 cubes of the face
// neighbours the hybrid push table names (nullptr: that neighbour computes
// its ring itself).  sxp[2a] = the -a neighbour (fed by cells with coordinate
// a < 2), sxp[2a+1] = the +a neighbour (coordinate >= n-2); a cell near an
// edge feeds each face neighbour separately (edge cells of the ring are read
// by no stage-2 stencil).
template <int NB>
__device__ __forceinline__ void push_u1(const PushEntry* sxp, int U1C, int ci, int cj, int k,
                                        const double w[5]) {
  if (ci < 0 || ci >= NB || cj < 0 || cj >= NB || k < 0 || k >= NB) return;
  const int c[3] = {ci, cj, k};
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const int side = c[a] < 2 ? 0 : (c[a] >= NB - 2 ? 1 : -1);
    if (side < 0) continue;
    double* d = sxp[2 * a + side].dst;
    if (d == nullptr) continue;
    int t[3] = {ci, cj, k};
    t[a] = side ? c[a] - NB : c[a] + NB;
    double* q = d + ((t[2] + 2) * (NB + 4) + (t[1] + 2)) * (NB + 4) + (t[0] + 2);
#pragma unroll
    for (int v = 0; v < 5; v++) q[v * U1C] = w[v];
  }
}

// PUSH: 0 none, 1 scatter the new state into every same-packet guard
// (push_cell), 2 into the x-guards only (push_x, gather mode).
// GATHER: the gather-mode staging (nbr is the per-slot neighbour table); a
// separate instantiation so the plain kernels carry none of its registers.
// SCH: 0 the paper-path scheme, 1 the grid's F4 flags (see face_flux).
// HYB: 1 = a stage-1 kernel of the borrowed-ring telescoped step (see
// launch_hybrid_nb): U1 always in the compact (n+4)^3 cubes, the CTA's slot
// and its self-ring sides from smap (slot | mask << 26), ring cells written
// only on self sides, the x-ring of the x-neighbours pushed (push_x_u1).
template <int NB, int STAGE, int SPLIT, int MODE, int PUSH, bool GATHER, int SCH, int HYB = 0, int WXT = 0,
          int HT = 0>
__global__ void __launch_bounds__(Geo<NB, STAGE, SPLIT, MODE, WXT, HT>::NT, Geo<NB, STAGE, SPLIT, MODE, WXT, HT>::MINB)
    stage_fused_kernel(DevGrid G, double* __restrict__ state, double* __restrict__ u1,
                       const SlotInfo* __restrict__ slots, const double* __restrict__ d_dt, double h_dt,
                       DtRecord* __restrict__ rec, DevStatus* st, const PushEntry* __restrict__ push,
                       const NbrEntry* __restrict__ nbr, const int* __restrict__ smap) {
  using Gm = Geo<NB, STAGE, SPLIT, MODE, WXT, HT>;
  constexpr int W = Gm::W, IPX = Gm::IPX, BAND = Gm::BAND, INO = Gm::INO, NS = Gm::NS;
  constexpr int NT = Gm::NT, H = Gm::H;
  // U1 cube stride: (n+4)^3 compact scratch (telescoped, and every hybrid
  // kernel) or the padded state layout (per-stage)
  constexpr bool CU1 = MODE == 0 || HYB;
  constexpr int U1C = CU1 ? (int)u1_cube<NB>() : cube_c<NB>();
  auto u1_off = [&](int ci, int cj, int k) -> int {
    return CU1 ? ((k + 2) * (NB + 4) + (cj + 2)) * (NB + 4) + (ci + 2) : coff<NB>(ci, cj, k);
  };
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;                                   // [NS][5][IR][IPX]
  double* const FxA = ring + NS * 5 * BAND;              // [5][H][W+1] (x2: Gm::PIPE)
  double* const FyA = FxA + 5 * Gm::FX;                  // [5][H+1][W]
  double* Fx = FxA;                                      // this plane's (Gm::PIPE: buffer it & 1)
  double* Fy = FyA;
  double* Fz = FyA + 5 * Gm::FY + (Gm::PIPE ? 5 * (Gm::FX + Gm::FY) : 0);  // [2][5][H][W] (not with Gm::ZREG)
  double* Zc = Fz + (Gm::ZREG ? 0 : 2 * 5 * Gm::FZ);     // [5][H][W] z-face carry (Gm::ZC, not Gm::ZREG)
  uint64_t* bar = reinterpret_cast<uint64_t*>(Zc + (Gm::ZC && !Gm::ZREG ? 5 * Gm::FZ : 0));
  // Gm::ZREG: this thread's z-face fluxes (k-1/2 and k+1/2) and carried face state
  double zf_prev[5], zf_cur[5];
  Prim zcar;
  unsigned char* flipm = reinterpret_cast<unsigned char*>(bar + 8);  // [NS][IR]
  // gather mode: where staged row r of a plane of z class c (z < 0, inside,
  // >= NB) comes from -- resolved once per CTA (RowSrc; the per-plane issue
  // only adds the plane offset)
  struct RowSrc {
    const double* base;  // source row (plane 0 of its cube)
    int zm;              // z image mode of the source entry; -1: the own padded plane
    short fl;            // sign-flip bits (rho*v: 4, rho*w: 8)
    short run;           // rows copied from here (0: not the first row of a run)
  };
  RowSrc* rsrc = reinterpret_cast<RowSrc*>(flipm + ((NS * Gm::IR + 15) / 16) * 16);  // [3][IR]

  const int tid = threadIdx.x;
  const int me = HYB ? smap[blockIdx.x / Gm::NSPLIT] : (int)(blockIdx.x / Gm::NSPLIT);
  const long long slot = HYB ? (me & 0x3ffffff) : me;
  const int selfm = HYB ? ((me >> 26) & 63) : 0;  // self-ring sides: bit 2a (-a), 2a+1 (+a)
  const int band = blockIdx.x % Gm::NSPLIT;
  // output planes [kz0, kz0 + nk): the geometry's, or (HYB stage 1) the
  // interior extended by the 2 ring planes on the self z sides only
  const int zlo = (HYB && STAGE == 1) ? ((selfm >> 4) & 1) * 2 : Gm::OFF;
  const int zhi = (HYB && STAGE == 1) ? ((selfm >> 5) & 1) * 2 : Gm::OFF;
  const int kz0 = -zlo, nk = NB + zlo + zhi, nplanes = nk + 4;
  const int porg = INO - 2 - zlo;  // padded plane of staged plane 0
  // output columns [-ox, W - ox), rows [-oy, WY - oy): centred, or (one ring
  // side wider than the interior) on the self side
  const int ox = (W - NB == 2) ? ((selfm & 1) ? 2 : (selfm & 2) ? 0 : 1) : (W - NB) / 2;
  const int oy = (Gm::WY - NB == 2) ? ((selfm & 4) ? 2 : (selfm & 8) ? 0 : 1) : (Gm::WY - NB) / 2;
  const int ORG = INO - 2 - oy;  // padded row of staged row 0 of band 0
  const int ccol0 = INO - ox;    // staged column of output column 0
  const int jj0 = band * H;                              // first output row of the band (0-based)
  constexpr int cube = cube_c<NB>();  // == G.cube (checked at launch)
  const double dt = d_dt ? *d_dt : h_dt;
  const double* in = (STAGE == 1) ? state + slot * 5 * cube : u1 + slot * 5 * U1C;
  constexpr int in_cube = (STAGE == 1) ? cube : U1C;
  const SlotInfo si = slots[slot];

  // PUSH == 2: the -x / +x push targets of this block; HYB stage 1: the six
  // face neighbours' (-x, +x, -y, +y, -z, +z)
  __shared__ PushEntry sxp[6];
  if (PUSH == 2 && tid < 2) sxp[tid] = push[slot * 27 + (tid ? 14 : 12)];
  if (HYB && STAGE == 1 && tid < 6) sxp[tid] = push[slot * 27 + (tid == 0 ? 12 : tid == 1 ? 14 : tid == 2 ? 10 : tid == 3 ? 16 : tid == 4 ? 4 : 22)];
  __shared__ NbrEntry snb[9];   // gather mode: the (0, oy, oz) neighbour entries of this block
  if (GATHER && tid < 9) snb[tid] = nbr[slot * 27 + (tid / 3) * 9 + (tid % 3) * 3 + 1];
  constexpr int UWARPS = (Gm::FZ + 31) / 32;  // warps with update cells
  uint64_t* fdone = &bar[NS];  // ORCHA_ONEBAR: the update warps have read the face arrays of the plane
  uint64_t* cdone = &bar[NS + 1];  // ORCHA_ONEBAR 2: the converting warps have converted plane it+5
  constexpr bool CSPLIT = ORCHA_CONV_SPLIT && Gm::NW - UWARPS >= 2;
  // ORCHA_CONV_BAL: the converting warps take 2 rounds of 32 cells each and
  // the update warps the rest after their update (one round each when the
  // band is small enough), instead of the converting warps taking all of it
  // (3 rounds in both stage-1 kernels against one update).  Measured slower
  // (2.46 vs 2.40 ms per cfg4 step, profiles/r02_ab_convbal.txt): off
  constexpr int NXR = Gm::NXR, NCONV = Gm::NCONV;
  constexpr int CONV_END = (CSPLIT && ORCHA_CONV_BAL && 2 * (Gm::NW - UWARPS) * 32 < NCONV)
                               ? 2 * (Gm::NW - UWARPS) * 32 : NCONV;
  if (tid == 0) {
    for (int s = 0; s < NS; s++) mbar_init(&bar[s], 1);
    mbar_init(fdone, UWARPS);
    mbar_init(cdone, CSPLIT ? Gm::NW - UWARPS : Gm::NW);
    fence_mbar_init();
  }
  __syncthreads();

  // input plane p (0-based, z = K0 - 2 + p): padded rows [jj0, jj0 + IR) -> ring slot p % NS.
  // Called by warp 0 (all lanes) after a CTA barrier that follows every
  // generic access to the slot; the proxy fence of each issuing lane orders
  // those before its async copies.
  auto issue = [&](int p) {
    if (p < nplanes) {
      const int s = p % NS, lane = tid & 31;
      if (GATHER) {  // the rows' sources of the plane's z class (rsrc, resolved in the prologue)
        const int pp = p + porg, z = pp - INO;
        const int oz = z < 0 ? -1 : (z >= NB ? 1 : 0);
        if (lane == 0) mbar_expect_tx(&bar[s], 5u * BAND * 8u);
        __syncwarp();
        if (lane < Gm::IR) {
          const RowSrc e = rsrc[(oz + 1) * Gm::IR + lane];
          flipm[s * Gm::IR + lane] = (unsigned char)e.fl;
          if (e.run) {
            const int zp = e.zm < 0 ? pp : guard_image<NB>(z, oz, e.zm) + INO;
            const double* rp = e.base + zp * Gm::PLANE;
            fence_proxy_async();
#pragma unroll
            for (int v = 0; v < 5; v++)
              bulk_load(ring + (s * 5 + v) * BAND + lane * IPX, rp + v * in_cube, (uint32_t)(e.run * IPX * 8),
                        &bar[s]);
          }
        }
      } else if (lane == 0) {
        fence_proxy_async();
        mbar_expect_tx(&bar[s], 5u * BAND * 8u);
#pragma unroll
        for (int v = 0; v < 5; v++)
          bulk_load(ring + (s * 5 + v) * BAND,
                    in + v * in_cube + (long long)(p + porg) * Gm::PLANE + (long long)(jj0 + ORG) * IPX, BAND * 8u,
                    &bar[s]);
      }
    }
  };
  auto wait_plane = [&](int p) { mbar_wait(&bar[p % NS], (p / NS) & 1); };
  // EOS in place over the staged band of plane p: cells c0, c0 + nthr, ...
  // Only the staged cells some stencil reads are converted (compact index
  // c < NCONV): the output rows x (the output columns +- 2: x-faces), then the
  // 2 + 2 y-halo rows x the output columns (y-faces); the corner cells of the
  // staged band and its columns beyond +- 2 are never read.
  auto convert = [&](int p, int c0 = -1, int nthr = Gm::NT, int cend = Gm::NCONV) {
    double* Q = ring + (p % NS) * 5 * BAND;
    const int z = kz0 - 2 + p;
    unsigned long long hits = 0;
    for (int ci = (c0 < 0 ? tid : c0); ci < cend; ci += nthr) {
      bool fl;
      int r, col;
      if (ci < NXR) {
        r = ci / (W + 4);
        col = ccol0 - 2 + (ci - r * (W + 4));
        r += 2;
      } else {
        const int c2 = ci - NXR, rr = c2 / W;
        r = rr < 2 ? rr : H + rr;
        col = ccol0 + (c2 - rr * W);
      }
      const int c = r * IPX + col;
      double my = Q[2 * BAND + c], mz = Q[3 * BAND + c];
      if (GATHER) {  // gather mode: mirrored guard rows negate rho*v / rho*w
        const unsigned fm = flipm[(p % NS) * Gm::IR + r];
        if (fm & 4) my = -my;
        if (fm & 8) mz = -mz;
      }
      Prim q = (SCH == 0) ? eos(Q[c], Q[BAND + c], my, mz, Q[4 * BAND + c], G, &fl)
                          : eos_var(Q[c], Q[BAND + c], my, mz, Q[4 * BAND + c], G, &fl);
      int x = col - INO, y = jj0 + ORG + r - INO;
      // own (non-overlapping) rows of the band only, so each cell counts once
      bool mine = r >= 2 && r < 2 + H;
      if (mine && x >= 0 && x < NB && y >= 0 && y < NB && z >= 0 && z < NB) {
        hits += fl ? 1 : 0;
        if (STAGE == 1 && !(q.r > 0.0)) {
          long long g = (((long long)si.bc[2] * NB + z) * G.N[1] + ((long long)si.bc[1] * NB + y)) * G.N[0] +
                        ((long long)si.bc[0] * NB + x);
          atomicMin(&st->first_bad, (unsigned long long)g);
        }
      }
      Q[c] = q.r;
      Q[BAND + c] = q.u;
      Q[2 * BAND + c] = q.v;
      Q[3 * BAND + c] = q.w;
      Q[4 * BAND + c] = q.p;
    }
    if (hits) atomicAdd(&st->floor_hits, hits);
  };
  auto ld = [&](const double* P, int o, Prim& q) {
    q.r = P[o];
    q.u = P[BAND + o];
    q.v = P[2 * BAND + o];
    q.w = P[3 * BAND + o];
    q.p = P[4 * BAND + o];
  };
  // band-local output row j (0..H) <-> staged row j + 2; output column i <-> staged column i - OFF + INO
  // x-face between columns f-1 and f of band row j
  // stencil base offset (in a staged band) of face task t of direction kind
  auto task_base = [&](int kind, int t) -> int {
    if (kind == 0) {
      int j = t / (W + 1), f = t - j * (W + 1);
      return (j + 2) * IPX + (f - ox - 2 + INO);
    }
    if (kind == 1) {
      int f = t / W, i = t - f * W;
      return f * IPX + (i - ox + INO);
    }
    int j = t / W, i = t - j * W;
    return (j + 2) * IPX + (i - ox + INO);
  };
  auto x_task = [&](int t, int base, int it) {
    const double* P = ring + ((it + 2) % NS) * 5 * BAND;
    if constexpr (ORCHA_XSHFL) {
      // t = the face index this lane stores (-1: none); base = its cell's
      // stencil (cells li-1 .. li+1); the whole warp runs this (shuffle)
      Prim qm, q, qp, up, dn, R;
      ld(P, base, qm);
      ld(P, base + 1, q);
      ld(P, base + 2, qp);
      plm_cell<SCH>(qm, q, qp, G, &up, &dn);
      R.r = __shfl_down_sync(0xffffffffu, dn.r, 1);
      R.u = __shfl_down_sync(0xffffffffu, dn.u, 1);
      R.v = __shfl_down_sync(0xffffffffu, dn.v, 1);
      R.w = __shfl_down_sync(0xffffffffu, dn.w, 1);
      R.p = __shfl_down_sync(0xffffffffu, dn.p, 1);
      if (t >= 0) riemann_store<0, SCH>(up, R, G, Fx + t, Gm::FX);
    } else {
      Prim q0, q1, q2, q3;
      ld(P, base, q0);
      ld(P, base + 1, q1);
      ld(P, base + 2, q2);
      ld(P, base + 3, q3);
      face_flux<0, SCH>(q0, q1, q2, q3, G, Fx + t, Gm::FX);
    }
  };
  // y-face between band rows f-1 and f of column i
  auto y_task = [&](int u, int base, int it) {
    const double* P = ring + ((it + 2) % NS) * 5 * BAND;
    Prim q0, q1, q2, q3;
    ld(P, base, q0);
    ld(P, base + IPX, q1);
    ld(P, base + 2 * IPX, q2);
    ld(P, base + 3 * IPX, q3);
    face_flux<1, SCH>(q0, q1, q2, q3, G, Fy + u, Gm::FY);
  };
  // z-face k+1/2 of column (i, j): stencil planes it+1 .. it+4 (z = k-1 .. k+2)
  auto z_task = [&](int w, int base, int it, double* fz_out) {
    if constexpr (Gm::ZC) {
      // left state of cell k: carried from the previous plane (the prologue
      // face seeds it); cells k, k+1, k+2 give cell k+1's two face states
      Prim L, R, Up, q0, q1, q2;
      if (it >= 0 && Gm::ZREG) {
        L = zcar;
      } else if (it >= 0) {
        L.r = Zc[w];
        L.u = Zc[Gm::FZ + w];
        L.v = Zc[2 * Gm::FZ + w];
        L.w = Zc[3 * Gm::FZ + w];
        L.p = Zc[4 * Gm::FZ + w];
      } else {
        Prim qm;
        ld(ring + ((it + 1) % NS) * 5 * BAND, base, qm);
        ld(ring + ((it + 2) % NS) * 5 * BAND, base, q0);
        ld(ring + ((it + 3) % NS) * 5 * BAND, base, q1);
        plm_cell<SCH>(qm, q0, q1, G, &L, &R);
      }
      ld(ring + ((it + 2) % NS) * 5 * BAND, base, q0);
      ld(ring + ((it + 3) % NS) * 5 * BAND, base, q1);
      ld(ring + ((it + 4) % NS) * 5 * BAND, base, q2);
      plm_cell<SCH>(q0, q1, q2, G, &Up, &R);
      if constexpr (Gm::ZREG) {
        zcar = Up;
        riemann_store<2, SCH>(L, R, G, fz_out, 1);
      } else {
        Zc[w] = Up.r;
        Zc[Gm::FZ + w] = Up.u;
        Zc[2 * Gm::FZ + w] = Up.v;
        Zc[3 * Gm::FZ + w] = Up.w;
        Zc[4 * Gm::FZ + w] = Up.p;
        riemann_store<2, SCH>(L, R, G, fz_out + w, Gm::FZ);
      }
    } else {
      Prim q0, q1, q2, q3;
      ld(ring + ((it + 1) % NS) * 5 * BAND, base, q0);
      ld(ring + ((it + 2) % NS) * 5 * BAND, base, q1);
      ld(ring + ((it + 3) % NS) * 5 * BAND, base, q2);
      ld(ring + ((it + 4) % NS) * 5 * BAND, base, q3);
      if constexpr (Gm::ZREG) face_flux<2, SCH>(q0, q1, q2, q3, G, fz_out, 1);
      else face_flux<2, SCH>(q0, q1, q2, q3, G, fz_out + w, Gm::FZ);
    }
  };
  const int warp = tid >> 5, lane = tid & 31;
  // this thread's face tasks (the same on every plane): warp-uniform direction
  // slots r*NW + warp, decoded once
  int tkind[Gm::ROUNDS], ttask[Gm::ROUNDS], tbase[Gm::ROUNDS];
#pragma unroll
  for (int r = 0; r < Gm::ROUNDS; r++) {
    // Gm::ZREG: z slot w in the last round of warp w (w < SZ); the x / y
    // slots, in order, over the remaining (round, warp) positions
    const bool zslot = Gm::ZREG && warp < Gm::SZ && r == Gm::ROUNDS - 1;
    const int m = !Gm::ZREG ? r * Gm::NW + warp
                  : zslot ? Gm::SX + Gm::SY + warp
                  : r < Gm::ROUNDS - 1 ? r * Gm::NW + warp
                  : (Gm::ROUNDS - 1) * Gm::NW + warp - Gm::SZ;
    const int mm = (Gm::ZREG && !zslot && m >= Gm::SX + Gm::SY) ? Gm::NSLOT : m;  // x / y positions left over
    int kind = 3, t = 0;
    int xbase = 0;
    if (mm < Gm::SX) {
      if constexpr (ORCHA_XSHFL) {
        // cell c of the band plane's rows of W+2 x-slope cells (output
        // columns -1 .. W); every lane of the slot runs the task (shuffle)
        const int c = m * 31 + lane, cc = c < Gm::NCX ? c : Gm::NCX - 1;
        const int j = cc / (W + 2), u = cc - j * (W + 2);
        kind = 0;
        t = (c < Gm::NCX && lane < 31 && u <= W) ? j * (W + 1) + u : -1;
        xbase = (j + 2) * IPX + (u - 2 - ox + INO);
      } else {
        t = m * 32 + lane;
        kind = t < Gm::FX ? 0 : 3;
      }
    }
    else if (mm < Gm::SX + Gm::SY) { t = (mm - Gm::SX) * 32 + lane; kind = t < Gm::FY ? 1 : 3; }
    else if (mm < Gm::NSLOT) { t = (mm - Gm::SX - Gm::SY) * 32 + lane; kind = t < Gm::FZ ? 2 : 3; }
    tkind[r] = kind;
    ttask[r] = t;
    tbase[r] = (ORCHA_XSHFL && kind == 0) ? xbase : kind < 3 ? task_base(kind, t) : 0;
  }

  // Gm::STATIC3: this thread's x and y faces (clamped to the last face)
  const int sx_t = min(warp * 32 + lane, Gm::FX - 1), sy_t = min(warp * 32 + lane, Gm::FY - 1);
  const int sx_b = Gm::STATIC3 ? task_base(0, sx_t) : 0, sy_b = Gm::STATIC3 ? task_base(1, sy_t) : 0;
  const int sz_b = Gm::STATIC3 && tid < Gm::FZ ? task_base(2, tid) : 0;
  bool writes_faces = false;
#pragma unroll
  for (int r = 0; r < Gm::ROUNDS; r++) writes_faces |= tkind[r] < 3;

  // ---- prologue: planes 0..4 (z in [K0-2, K0+3)), z-faces K0-1/2 -> Fz[1]
  const bool issuer = ORCHA_ISSUE_LAST ? warp == Gm::NW - 1 : warp == 0;  // the warp that stages planes
  if (GATHER && issuer) {
    // Gather mode: only the x-guards were filled.  Each staged row (padded
    // row pr of padded plane pp) is the (y, z) image of a row of the block
    // that owns it -- the neighbour table's (0, oy, oz) entry -- whose
    // x-guards are filled: the axis-ordered ghost fill composed on the fly (x,
    // then y over x-guards, then z over x,y-guards).  Lane r resolves row r
    // for each z class (its representative plane: the source entry, and so
    // which rows are consecutive in memory, is the same for every plane of
    // the class); rows whose sources are consecutive form one copy, issued by
    // the lane that starts the run.
#pragma unroll 1
    for (int c = 0; c < 3; c++) {
      const int oz = c - 1, z = oz < 0 ? -1 : oz > 0 ? NB : 0, pp = z + INO;
      const double* rp = nullptr;
      RowSrc r{nullptr, -1, 0, 0};
      if (lane < Gm::IR) {
        const int pr = jj0 + ORG + lane, y = pr - INO;
        const int oy = y < 0 ? -1 : (y >= NB ? 1 : 0);
        const NbrEntry e = snb[(oz + 1) * 3 + (oy + 1)];
        if (e.src == nullptr) {  // remote source: its rows were exchanged into our own guards
          r.base = in + (long long)pr * IPX;
          rp = r.base + (long long)pp * Gm::PLANE;
        } else {
          const int ys = guard_image<NB>(y, oy, (e.mode >> 2) & 3);
          r.zm = (e.mode >> 4) & 3;
          r.base = e.src + (long long)(ys + INO) * IPX;
          rp = r.base + (long long)(guard_image<NB>(z, oz, r.zm) + INO) * Gm::PLANE;
          r.fl = (short)(e.flip & 0xC);  // mirrored y -> negate rho*v (bit 2), z -> rho*w (bit 3)
        }
      }
      const double* prev = (const double*)__shfl_up_sync(0xffffffffu, (unsigned long long)rp, 1);
      const int pfl = __shfl_up_sync(0xffffffffu, (int)r.fl, 1);
      const bool start = lane < Gm::IR && (lane == 0 || rp != prev + IPX || r.fl != pfl);
      const unsigned starts = __ballot_sync(0xffffffffu, start);
      const unsigned later = starts & ~((2u << lane) - 1u);
      r.run = start ? (short)((later ? __ffs(later) - 1 : Gm::IR) - lane) : (short)0;
      if (lane < Gm::IR) rsrc[c * Gm::IR + lane] = r;
    }
    __syncwarp();
  }
  if (issuer)
    for (int p = 0; p < NS; p++) issue(p);
  if (GATHER) __syncthreads();  // the sign-flip masks thread 0 just wrote
  for (int p = 0; p < NS; p++) {
    wait_plane(p);
    convert(p);
  }
  __syncthreads();
  if constexpr (Gm::ZREG) {
    if (tid < Gm::FZ) z_task(tid, task_base(2, tid), -1, zf_prev);
  } else {
    for (int w = tid; w < Gm::FZ; w += NT) z_task(w, task_base(2, w), -1, Fz + 5 * Gm::FZ);
  }
  __syncthreads();
  if (issuer)  // into the slots of planes 0 (and 1: a 4-deep ring, dead once the prologue faces are done)
    for (int p = NS; p < 6; p++) issue(p);
  if (NS == 4) {  // plane 4 is read by the first output plane's z-faces
    if (GATHER) __syncthreads();  // its sign-flip masks
    wait_plane(4);
    convert(4);
    __syncthreads();
  }

  double s_rec = -DBL_MAX;
  long long g_rec = LLONG_MAX;
  // stage 2's dt epilogue for one new cell state: the CFL signal speed of the
  // new state into this thread's record, and the non-physical check
  auto dt_cell = [&](const double* nw, int k, int ci, int cj) {
    bool f2;
    Prim q = (SCH == 0) ? eos(nw[0], nw[1], nw[2], nw[3], nw[4], G, &f2)
                        : eos_var(nw[0], nw[1], nw[2], nw[3], nw[4], G, &f2);
    double s = (SCH == 0) ? signal_speed<3>(q, G) : signal_speed_var<3>(q, G);
    auto gidx = [&]() -> long long {
      return (((long long)si.bc[2] * NB + k) * G.N[1] + ((long long)si.bc[1] * NB + cj)) * G.N[0] +
             ((long long)si.bc[0] * NB + ci);
    };
    // this thread's cells come in increasing k at a fixed (i, j), so their
    // global indices increase: dt_better(s, g, s_rec, g_rec) reduces to a
    // larger s, or the first NaN -- g is formed only when the record moves
    const bool sn = s != s, rn = s_rec != s_rec;
    if (sn ? !rn : (!rn && s > s_rec)) { s_rec = s; g_rec = gidx(); }
    // finite: no exponent field of all ones (integer tests of the high words)
    bool finite = true;
#pragma unroll
    for (int v = 0; v < 5; v++) finite &= (__double2hiint(nw[v]) & 0x7ff00000) != 0x7ff00000;
    if (!(nw[0] > 0.0) || !finite) atomicMin(&st->first_bad, (unsigned long long)gidx());
  };
  double pnw[5];  // ORCHA_DEFER_DT: the last new state whose dt epilogue is pending (plane pk)
  int pk = -1;
  // ORCHA_PUSH_HOIST, stage 2 with the x-guard push: this thread's target
  // when it is a shift (gm 1: gx = its offset from `state` at plane 0 -- it
  // may be negative: another rank's packet in F2 peer mode), a clamp / mirror
  // target (gm 2: push_x per plane), or none (gm 0)
  long long gx = 0;
  int gm = 0;
  if (ORCHA_PUSH_HOIST && STAGE == 2 && PUSH == 2 && tid < Gm::FZ) {
    const int gci = (tid - (tid / W) * W) - ox, gcj = jj0 + tid / W - oy;
    const int side = gci >= NB - 4 ? 1 : (gci < 4 ? 0 : -1);
    if (side >= 0 && sxp[side].dst != nullptr) {
      if ((sxp[side].mode & 3) == kShift) {
        gx = (sxp[side].dst - state) + coff<NB>(side ? gci - NB : gci + NB, gcj, 0);
        gm = 1;
      } else {
        gm = 2;
      }
    }
  }
  // ORCHA_PUSH_HOIST (HYB stage 1): this thread's x / y ring-push targets
  long long hx = -1, hy = -1;
  if (ORCHA_PUSH_HOIST && HYB && STAGE == 1 && tid < Gm::FZ) {
    const int hci = (tid - (tid / W) * W) - ox, hcj = jj0 + tid / W - oy;
    if (hci >= 0 && hci < NB && hcj >= 0 && hcj < NB) {
      const int xs = hci < 2 ? 0 : (hci >= NB - 2 ? 1 : -1), ys = hcj < 2 ? 2 : (hcj >= NB - 2 ? 3 : -1);
      if (xs >= 0 && sxp[xs].dst)
        hx = (sxp[xs].dst - u1) + (2 * (NB + 4) + (hcj + 2)) * (NB + 4) + ((xs ? hci - NB : hci + NB) + 2);
      if (ys >= 0 && sxp[ys].dst)
        hy = (sxp[ys].dst - u1) + (2 * (NB + 4) + ((ys == 3 ? hcj - NB : hcj + NB) + 2)) * (NB + 4) + (hci + 2);
    }
  }
#pragma unroll 1
  for (int it = 0; it < nk; it++) {
    const int k = kz0 + it;
    // prefetch the update operands of this thread's cell of plane k
    const bool upd = tid < Gm::FZ;
    const int lj = upd ? tid / W : 0, li = upd ? tid - (tid / W) * W : 0;
    const int ci = li - ox, cj = jj0 + lj - oy;
    const int so = coff<NB>(ci, cj, k);
    double un[5], v1[5];
    if (upd) {
      const double* ub = state + slot * 5 * cube;
      int uo = so;
      int ufl = 0;
      if (STAGE == 1 && (MODE == 0 || HYB) && GATHER) {
        // gather mode: the box's y/z guard-ring cells were not filled; U^n of
        // such a cell is its image in the owning block (x-guards are filled)
        const int oy = cj < 0 ? -1 : (cj >= NB ? 1 : 0), oz = k < 0 ? -1 : (k >= NB ? 1 : 0);
        if (oy != 0 || oz != 0) {
          const NbrEntry e = snb[(oz + 1) * 3 + (oy + 1)];
          if (e.src != nullptr) {
            ub = e.src;
            uo = coff<NB>(ci, guard_image<NB>(cj, oy, (e.mode >> 2) & 3), guard_image<NB>(k, oz, (e.mode >> 4) & 3));
            ufl = e.flip & 0xC;
          }
        }
      }
#pragma unroll
      for (int v = 0; v < 5; v++) un[v] = ld_once(ub + v * cube + uo);
      if (ufl & 4) un[2] = -un[2];
      if (ufl & 8) un[3] = -un[3];
      if (STAGE == 2) {
        const int uo = u1_off(ci, cj, k);
#pragma unroll
        for (int v = 0; v < 5; v++) v1[v] = ld_once(u1 + slot * 5 * U1C + v * U1C + uo);
      }
    }
    // phase 1: all face fluxes of the band's plane k (inputs: planes it+1 .. it+4)
    double* fz_cur = Fz + (it & 1) * 5 * Gm::FZ;
    if constexpr (Gm::PIPE) {
      Fx = FxA + (it & 1) * 5 * (Gm::FX + Gm::FY);
      Fy = Fx + 5 * Gm::FX;
    }
    if (ORCHA_ONEBAR && it > 0 && writes_faces) mbar_wait(fdone, (it - 1) & 1);  // update(it-1) read the faces
    if (STAGE == 2 && ORCHA_DEFER_DT && pk >= 0) {  // the previous plane's dt epilogue
      const int pci = (tid - (tid / W) * W) - ox, pcj = jj0 + tid / W - oy;
      dt_cell(pnw, pk, pci, pcj);
      pk = -1;
    }
    if constexpr (Gm::STATIC3) {
      // every warp: x slot `warp`, y slot `warp`, z slot `warp` (w < SZ), in
      // straight-line code the compiler may interleave; the lanes past the
      // last face of a slot recompute (and store) that face
      x_task(sx_t, sx_b, it);
      y_task(sy_t, sy_b, it);
      if (warp < Gm::SZ) z_task(tid, sz_b, it, zf_cur);
    } else {
#pragma unroll
    for (int r = 0; r < Gm::ROUNDS; r++) {
      if (tkind[r] == 0) x_task(ttask[r], tbase[r], it);
      else if (tkind[r] == 1) y_task(ttask[r], tbase[r], it);
      else if (tkind[r] == 2) {
        if ((ORCHA_ONEBAR == 2 || Gm::PIPE) && it > 0) mbar_wait(cdone, (it - 1) & 1);  // plane it+4 converted
        if constexpr (Gm::ZREG) z_task(ttask[r], tbase[r], it, zf_cur);
        else z_task(ttask[r], tbase[r], it, fz_cur);
      }
    }
    }
    constexpr int UW = UWARPS;
    // the EOS of plane it+5 (read from iteration it+1 on; its copy was issued
    // one plane earlier): ORCHA_ONEBAR before the barrier, else after it
    auto convert_next = [&]() {
      if (it + 5 < nplanes) {
        if constexpr (CSPLIT) {
          if (warp >= UW) {
            wait_plane(it + 5);
            convert(it + 5, tid - UW * 32, NT - UW * 32, CONV_END);
          }
        } else {
          wait_plane(it + 5);
          convert(it + 5);
        }
      }
      if ((ORCHA_ONEBAR == 2 || Gm::PIPE) && (!CSPLIT || warp >= UW)) {  // plane it+5 is primitives
        __syncwarp();
        if (lane == 0) mbar_arrive(cdone);
      }
    };
    if (ORCHA_ONEBAR == 1) convert_next();
    __syncthreads();
    // phase 2: stage plane it+6 into the slot of plane it+1 (read for the
    // last time in phase 1), convert plane it+5, update the band's cells
    if (issuer) issue(it + 6);
    if (ORCHA_ONEBAR != 1) convert_next();
    if (upd || (ORCHA_ONEBAR && warp < UW)) {
      const double* fz_prev = Fz + ((it + 1) & 1) * 5 * Gm::FZ;
      double D[5];
      if (upd) {
#pragma unroll
        for (int v = 0; v < 5; v++) {
          double tx = (Fx[v * Gm::FX + lj * (W + 1) + li + 1] - Fx[v * Gm::FX + lj * (W + 1) + li]) * G.id[0];
          double ty = (Fy[v * Gm::FY + (lj + 1) * W + li] - Fy[v * Gm::FY + lj * W + li]) * G.id[1];
          double tz = Gm::ZREG ? (zf_cur[v] - zf_prev[v]) * G.id[2]
                               : (fz_cur[v * Gm::FZ + tid] - fz_prev[v * Gm::FZ + tid]) * G.id[2];
          D[v] = (tx + ty) + tz;
        }
        if constexpr (Gm::ZREG) {  // face k+1/2 is the next plane's k-1/2
#pragma unroll
          for (int v = 0; v < 5; v++) zf_prev[v] = zf_cur[v];
        }
      }
      if (ORCHA_ONEBAR) {  // the face arrays of plane it are consumed: the faces of it+1 may overwrite them
        __syncwarp();
        if (lane == 0) mbar_arrive(fdone);
      }
      if (upd) {
      if (STAGE == 1 && HYB) {
        // borrowed-ring step: a box ring cell is written only on a self side
        // (the other sides' rings are the neighbours' own cells: their x-ring
        // is pushed by them, their y/z rows are staged from them by stage 2);
        // edge and corner cells of the box are read by no stage-2 stencil
        const int ax = ci < 0 ? 0 : ci >= NB ? 1 : -1, ay = cj < 0 ? 2 : cj >= NB ? 3 : -1,
                  az = k < 0 ? 4 : k >= NB ? 5 : -1;
        const int nout = (ax >= 0) + (ay >= 0) + (az >= 0);
        const int sb = ax >= 0 ? ax : ay >= 0 ? ay : az;
        double w[5];
#pragma unroll
        for (int v = 0; v < 5; v++) w[v] = un[v] - dt * D[v];
        if (nout == 0 || (nout == 1 && ((selfm >> sb) & 1))) {
          double* out = u1 + slot * 5 * U1C + u1_off(ci, cj, k);
#pragma unroll
          for (int v = 0; v < 5; v++) out[v * U1C] = w[v];
        }
        if constexpr (ORCHA_PUSH_HOIST) {
          // x / y targets hoisted out of the plane loop (hx / hy: offsets from
          // u1 of this column's target at plane 0; -1: none); z per plane
          if (k >= 0 && k < NB) {
            constexpr int PL = (NB + 4) * (NB + 4);
            if (hx >= 0) {
#pragma unroll
              for (int v = 0; v < 5; v++) u1[hx + k * PL + v * U1C] = w[v];
            }
            if (hy >= 0) {
#pragma unroll
              for (int v = 0; v < 5; v++) u1[hy + k * PL + v * U1C] = w[v];
            }
            const int zs = k < 2 ? 4 : (k >= NB - 2 ? 5 : -1);
            if (zs >= 0 && ci >= 0 && ci < NB && cj >= 0 && cj < NB && sxp[zs].dst != nullptr) {
              double* q = sxp[zs].dst + ((zs == 5 ? k - NB : k + NB) + 2) * PL + (cj + 2) * (NB + 4) + (ci + 2);
#pragma unroll
              for (int v = 0; v < 5; v++) q[v * U1C] = w[v];
            }
          }
        } else {
          push_u1<NB>(sxp, U1C, ci, cj, k, w);
        }
      } else if (STAGE == 1) {
        double* out = u1 + slot * 5 * U1C + u1_off(ci, cj, k);
#pragma unroll
        for (int v = 0; v < 5; v++) out[v * U1C] = un[v] - dt * D[v];
        if (MODE == 1 && PUSH) {  // per-stage: scatter U1 into the U1 guards of the neighbours
          double w[5];
#pragma unroll
          for (int v = 0; v < 5; v++) w[v] = un[v] - dt * D[v];
          if (PUSH == 1) push_cell(G, push + slot * 27, ci, cj, k, w);
          else push_x<NB>(G, sxp, ci, cj, k, w);  // gather mode: the x-guards only
        }
      } else {
        double nw[5];
#pragma unroll
        for (int v = 0; v < 5; v++) nw[v] = 0.5 * (un[v] + (v1[v] - dt * D[v]));
        double* dst = state + slot * 5 * cube + so;
#pragma unroll
        for (int v = 0; v < 5; v++) dst[v * cube] = nw[v];
        if (PUSH == 1) push_cell(G, push + slot * 27, ci, cj, k, nw);  // next step's guards
        if (PUSH == 2) {  // next step's x-guards
          if (ORCHA_PUSH_HOIST && gm == 1) {  // a shift target, hoisted (gx: its offset at plane 0)
            constexpr int PP = (NB + 8) * (NB + 8);
#pragma unroll
            for (int v = 0; v < 5; v++) state[gx + (long long)k * PP + v * cube] = nw[v];
          } else if (!ORCHA_PUSH_HOIST || gm == 2) {
            push_x<NB>(G, sxp, ci, cj, k, nw);
          }
        }
        if constexpr (ORCHA_DEFER_DT) {  // the dt epilogue of this cell runs in the next plane's phase 1
#pragma unroll
          for (int v = 0; v < 5; v++) pnw[v] = nw[v];
          pk = k;
        } else {
          dt_cell(nw, k, ci, cj);
        }
      }
      }
    }
    if constexpr (CONV_END < NCONV) {  // the update warps' share of the next plane's EOS
      if (warp < UWARPS && it + 5 < nplanes) {
        wait_plane(it + 5);
        convert(it + 5, CONV_END + tid, UWARPS * 32, NCONV);
      }
    }
    if (!ORCHA_ONEBAR && !Gm::PIPE) __syncthreads();
  }
  if (STAGE == 2 && ORCHA_DEFER_DT && pk >= 0) {
    const int pci = (tid - (tid / W) * W) - ox, pcj = jj0 + tid / W - oy;
    dt_cell(pnw, pk, pci, pcj);
  }
  if (STAGE == 2) {
    block_reduce_rec<NT>(s_rec, g_rec);
    if (tid == 0) { rec[blockIdx.x].s = s_rec; rec[blockIdx.x].g = g_rec; }
  }
}
// The dynamic shared-memory attribute of every instantiation one launch_stage
// may pick (once per process; also loads them under CUDA lazy loading).
template <int NB, int STAGE, int SPLIT, int MODE, int SCH>
static cudaError_t stage_attrs() {
  using Gm = Geo<NB, STAGE, SPLIT, MODE>;
  constexpr bool P2 = (STAGE == 2) || (MODE == 1);
  constexpr bool GA = (STAGE == 1) || (MODE == 1);
  static cudaError_t once = [] {
    const int sm = (int)Gm::SMEM_G;  // the largest of the instantiations'
    cudaError_t e = cudaFuncSetAttribute(stage_fused_kernel<NB, STAGE, SPLIT, MODE, 0, false, SCH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(stage_fused_kernel<NB, STAGE, SPLIT, MODE, 1, false, SCH>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if constexpr (GA)
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(stage_fused_kernel<NB, STAGE, SPLIT, MODE, 0, true, SCH>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if constexpr (P2)
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(stage_fused_kernel<NB, STAGE, SPLIT, MODE, 2, false, SCH>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if constexpr (P2 && GA)
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(stage_fused_kernel<NB, STAGE, SPLIT, MODE, 2, true, SCH>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    return e;
  }();
  return once;
}

template <int NB, int STAGE, int SPLIT, int MODE, int SCH>
static void launch_stage(const DevGrid& G, double* state, double* u1, int nslots, const SlotInfo* slots,
                             const double* d_dt, double h_dt, DtRecord* records, DevStatus* st, cudaStream_t s,
                             const PushEntry* push = nullptr, const NbrEntry* nbr = nullptr,
                             int pushkind = 1) {
  using Gm = Geo<NB, STAGE, SPLIT, MODE>;
  // Instantiations: PUSH 0 / 1 / 2 x plain, PUSH 0 / 2 x gather (stage 1:
  // from the states; per-stage stage 2: from the stage-1 buffers).  PUSH 2
  // (x-guards only) exists for the kernels that feed a gather-mode step:
  // telescoped stage 2 and both per-stage stages.
  constexpr bool P2 = (STAGE == 2) || (MODE == 1);
  constexpr bool GA = (STAGE == 1) || (MODE == 1);
  stage_attrs<NB, STAGE, SPLIT, MODE, SCH>();
  // the guard-push epilogues and the gather staging are separate
  // instantiations so the default kernels carry none of their registers
  const dim3 grid(nslots * SPLIT);
#define ORCHA_K(P, GT)                                                                                  \
  stage_fused_kernel<NB, STAGE, SPLIT, MODE, P, GT, SCH><<<grid, Gm::NT, GT ? Gm::SMEM_G : Gm::SMEM, s>>>(G, state, u1, slots, \
                                                                                      d_dt, h_dt, records, st, \
                                                                                      push, nbr, nullptr)
  if (push && pushkind == 2) {
    if constexpr (P2) {
      if constexpr (GA) {
        if (nbr) ORCHA_K(2, true);
        else ORCHA_K(2, false);
      } else {
        ORCHA_K(2, false);
      }
    }
  } else if (push) {
    ORCHA_K(1, false);
  } else if (nbr) {
    if constexpr (GA) ORCHA_K(0, true);
  } else {
    ORCHA_K(0, false);
  }
#undef ORCHA_K
  count_launch();
}

// Row bands per block (CTAs per block) for 16^3: measured best by default;
// ORCHA_SPLIT1 / ORCHA_SPLIT2 (2 or 4) override for experiments.
static int split_env(const char* name, int dflt) {
  const char* e = getenv(name);
  if (!e) return dflt;
  int v = atoi(e);
  return (v == 2 || v == 4) ? v : dflt;
}

// parts: bit 0 = stage 1, bit 1 = stage 2 (F2 peer mode puts a cross-rank
// barrier between the two launches).
template <int NB, int SCH>
static cudaError_t launch_nb(const DevGrid& G, double* state, double* u1, int nslots, const SlotInfo* slots,
                             const double* d_dt, double h_dt, DtRecord* records, long long* nrecords, DevStatus* st,
                             cudaStream_t s, const PushEntry* push, const NbrEntry* nbr, int pk, int parts) {
  if (G.cube != cube_c<NB>() || G.gd[0] != 4 || G.P[0] != NB + 8) return cudaErrorInvalidValue;  // compile-time geometry
  int s2 = 1;
  if constexpr (NB == 16) {
    static const int s1 = split_env("ORCHA_SPLIT1", 2);
    static const int s2v = split_env("ORCHA_SPLIT2", 2);
    s2 = s2v;
    if (parts & 1) {
      PhaseScope ph(PH_STAGE1, s);
#ifdef ORCHA_SPLIT1_ONE  // experiment: one CTA per block for stage 1 (20 rows, 22 warps, 1 CTA per SM)
      (void)s1;
      launch_stage<NB, 1, 1, 0, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, nullptr, nbr);
#else
      if (s1 == 4) launch_stage<NB, 1, 4, 0, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, nullptr, nbr);
      else launch_stage<NB, 1, 2, 0, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, nullptr, nbr);
#endif
    }
    if (parts & 2) {
      PhaseScope ph(PH_STAGE2, s);
      if (s2 == 4) launch_stage<NB, 2, 4, 0, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, push, nullptr, pk);
      else launch_stage<NB, 2, 2, 0, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, push, nullptr, pk);
    }
  } else if constexpr (NB == 32) {
    if (parts & 1) {
      PhaseScope ph(PH_STAGE1, s);
      launch_stage<NB, 1, 4, 0, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, nullptr, nbr);
    }
    if (parts & 2) {
      PhaseScope ph(PH_STAGE2, s);
      launch_stage<NB, 2, 4, 0, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, push, nullptr, pk);
    }
    s2 = 4;
  } else {
    if (parts & 1) {
      PhaseScope ph(PH_STAGE1, s);
      launch_stage<NB, 1, 1, 0, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, nullptr, nbr);
    }
    if (parts & 2) {
      PhaseScope ph(PH_STAGE2, s);
      launch_stage<NB, 2, 1, 0, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, push, nullptr, pk);
    }
  }
  if (parts & 2) *nrecords = (long long)nslots * s2;
  return cudaGetLastError();
}


// One stage of the per-stage variant (F1) for one block size.
template <int NB, int SCH>
static cudaError_t launch_stage_nb(const DevGrid& G, int stage, double* state, double* u1, int nslots,
                                   const SlotInfo* slots, const double* d_dt, double h_dt, DtRecord* records,
                                   long long* nrecords, DevStatus* st, cudaStream_t s, const PushEntry* push,
                                   const NbrEntry* nbr, int pk) {
  constexpr int SP = (NB == 16) ? 2 : (NB == 32) ? 4 : 1;
  if (G.cube != cube_c<NB>() || G.gd[0] != 4 || G.P[0] != NB + 8) return cudaErrorInvalidValue;  // compile-time geometry
  PhaseScope ph(stage == 1 ? PH_STAGE1 : PH_STAGE2, s);
  if (stage == 1) {
    launch_stage<NB, 1, SP, 1, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, push, nbr, pk);
  } else {
    launch_stage<NB, 2, SP, 1, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, st, s, push, nbr, pk);
    *nrecords = (long long)nslots * SP;
  }
  return cudaGetLastError();
}

// ------------------------------------------- borrowed-ring telescoped step --
// The paper's telescoping computes stage 1 on the block plus a 2-cell ring so
// that stage 2 needs no second guard exchange (sec 6).  A ring
// cell whose owner block is resident in the same packet is that owner's own
// stage-1 value: the owner computes it from the same U^n cells (the guards
// are copies of them), so the telescoped result is unchanged when the ring is
// borrowed from the owner instead of recomputed.  Only "self" sides -- a
// physical boundary (the ring is U1 of the BC-imaged U^n, which no block
// owns) or an owner on another rank (no second exchange) -- need the ring
// computed.  So stage 1 runs in two launches over the slot map:
//   smap[0, nbnd):        blocks with an x or y self side: the box kernel
//                         (MODE 0 geometry: 20 x 20 output columns of 16^3),
//                         or for 16^3 blocks with at most one self side per
//                         axis the 18 x 18 kernel (the ring columns / rows of
//                         the self side; nb4 counts the groups);
//   smap[nbnd, +nint):    the rest: the interior kernel (MODE 1 geometry);
// in both the output planes are the interior plus the 2 ring planes on the
// self z sides only (runtime plane range), and ring cells are stored on
// self sides only.  Both write U1 into the compact (n+4)^3 cubes and push
// their 2-cell boundary layers into the ring of the face neighbours' cubes
// (hpush), so stage 2 is the plain telescoped stage-2 kernel over complete
// cubes.  Stage-1 cell-stages per cell-update on cfg4 (16^3 blocks, 16^3
// of them, outflow): 1.95 computed ring, 1.15 borrowed (1.0 away from self
// sides; 3.4 -> 1.0 at 8^3).
// The borrowed ring's (n+2)^2 stage-1 kernel: row bands per block (16^3: 3
// bands of 6 rows; 8^3: one band of 10); 32^3 blocks keep the box.
template <int NB>
struct TrimSplit {
  static constexpr bool on = NB == 16 || NB == 8;
  static constexpr int S = NB == 16 ? ORCHA_TRIM_SPLIT : 1;
};

template <int NB, int SCH, bool GT>
static cudaError_t hybrid_attrs_g() {
  constexpr int S = NB == 16 ? 2 : NB == 32 ? 4 : 1;
  cudaError_t e = cudaFuncSetAttribute(stage_fused_kernel<NB, 1, S, 0, 0, GT, SCH, 1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Geo<NB, 1, S, 0>::SMEM_G);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(stage_fused_kernel<NB, 1, S, 1, 0, GT, SCH, 1>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Geo<NB, 1, S, 1>::SMEM_G);
  if constexpr (TrimSplit<NB>::on) {
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(
          stage_fused_kernel<NB, 1, TrimSplit<NB>::S, 0, 0, GT, SCH, 1, NB + 2, (NB + 2) / TrimSplit<NB>::S>,
          cudaFuncAttributeMaxDynamicSharedMemorySize,
          (int)Geo<NB, 1, TrimSplit<NB>::S, 0, NB + 2, (NB + 2) / TrimSplit<NB>::S>::SMEM_G);
  }
  return e;
}

template <int NB, int SCH>
static cudaError_t hybrid_attrs() {
  constexpr int S = NB == 16 ? 2 : NB == 32 ? 4 : 1;
  static cudaError_t once = [] {
    cudaError_t e = hybrid_attrs_g<NB, SCH, true>();
    if (e == cudaSuccess) e = hybrid_attrs_g<NB, SCH, false>();
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(stage_fused_kernel<NB, 2, S, 0, 2, false, SCH, 0>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Geo<NB, 2, S, 0>::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(stage_fused_kernel<NB, 2, S, 0, 0, false, SCH, 0>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Geo<NB, 2, S, 0>::SMEM);
    return e;
  }();
  return once;
}

// The stage-1 launches of the borrowed ring over the slot map: the box, the
// 18 x 18 kernel (16^3) and the interior kernel; GT: the gather-mode staging
// (one packet, x-guards only filled) or the packet's own materialised guards
// (full fill: several packets per set, each with its own slot map).
template <int NB, int SCH, bool GT>
static void launch_hyb_stage1(const DevGrid& G, double* state, double* u1, const SlotInfo* slots, const int* smap,
                              const int* nb4, int nint, const PushEntry* hpush, const NbrEntry* nbr,
                              const double* d_dt, double h_dt, DtRecord* records, DevStatus* st, cudaStream_t sb,
                              cudaStream_t s) {
  constexpr int S = NB == 16 ? 2 : NB == 32 ? 4 : 1;
  const int* sm = smap;
  // the box (two x or two y self sides: a one-block-wide brick; every NB)
  if (nb4[0] > 0) {
    stage_fused_kernel<NB, 1, S, 0, 0, GT, SCH, 1>
        <<<nb4[0] * S, Geo<NB, 1, S, 0>::NT, Geo<NB, 1, S, 0>::SMEM_G, sb>>>(G, state, u1, slots, d_dt, h_dt, records,
                                                                            st, hpush, nbr, sm);
    count_launch();
  }
  sm += nb4[0];
  if constexpr (TrimSplit<NB>::on) {
    // at most one self side per axis: (n+2) x (n+2) output columns / rows,
    // the 2 ring columns (rows) on the self side, or one on each side of an
    // axis without one (computed, not stored)
    if (nb4[1] > 0) {
      constexpr int ST = TrimSplit<NB>::S;
      using GC = Geo<NB, 1, ST, 0, NB + 2, (NB + 2) / ST>;
      stage_fused_kernel<NB, 1, ST, 0, 0, GT, SCH, 1, NB + 2, (NB + 2) / ST>
          <<<nb4[1] * ST, GC::NT, GC::SMEM_G, sb>>>(G, state, u1, slots, d_dt, h_dt, records, st, hpush, nbr, sm);
      count_launch();
    }
    sm += nb4[1];
  }
  if (nint > 0) {
    stage_fused_kernel<NB, 1, S, 1, 0, GT, SCH, 1><<<nint * S, Geo<NB, 1, S, 1>::NT, Geo<NB, 1, S, 1>::SMEM_G, s>>>(
        G, state, u1, slots, d_dt, h_dt, records, st, hpush, nbr, sm);
    count_launch();
  }
}

template <int NB, int SCH>
static cudaError_t launch_hybrid_nb(const DevGrid& G, double* state, double* u1, int nslots, const SlotInfo* slots,
                                    const int* smap, const int* nb4, int nint, const PushEntry* hpush,
                                    const NbrEntry* nbr, const double* d_dt, double h_dt,
                                    DtRecord* records, long long* nrecords, DevStatus* st, cudaStream_t s,
                                    const PushEntry* push, int parts, cudaStream_t side, cudaEvent_t ev_fork,
                                    cudaEvent_t ev_join) {
  constexpr int S = NB == 16 ? 2 : NB == 32 ? 4 : 1;
  if (G.cube != cube_c<NB>() || G.gd[0] != 4 || G.P[0] != NB + 8) return cudaErrorInvalidValue;
  cudaError_t e = hybrid_attrs<NB, SCH>();
  if (e != cudaSuccess) return e;
  if (parts & 1) {
    PhaseScope ph(PH_STAGE1, s);
    // side stream (optional): the blocks with x / y self sides run beside the
    // interior kernel (they read only U^n and write disjoint cells), filling
    // each other's tail
    const int nbnd = nb4[0] + nb4[1] + nb4[2] + nb4[3];
    const bool fork = side != nullptr && nbnd > 0 && nint > 0;
    if (fork) {
      e = cudaEventRecord(ev_fork, s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ev_fork, 0);
      if (e != cudaSuccess) return e;
    }
    cudaStream_t sb = fork ? side : s;
    if (nbr) launch_hyb_stage1<NB, SCH, true>(G, state, u1, slots, smap, nb4, nint, hpush, nbr, d_dt, h_dt, records,
                                              st, sb, s);
    else launch_hyb_stage1<NB, SCH, false>(G, state, u1, slots, smap, nb4, nint, hpush, nbr, d_dt, h_dt, records, st,
                                           sb, s);
    if (fork) {
      e = cudaEventRecord(ev_join, side);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev_join, 0);
      if (e != cudaSuccess) return e;
    }
  }
  if (parts & 2) {
    PhaseScope ph(PH_STAGE2, s);
    if (push)  // gather mode: U^{n+1} into the x-guards too (the next fill launches nothing)
      stage_fused_kernel<NB, 2, S, 0, 2, false, SCH, 0><<<nslots * S, Geo<NB, 2, S, 0>::NT, Geo<NB, 2, S, 0>::SMEM, s>>>(
          G, state, u1, slots, d_dt, h_dt, records, st, push, nullptr, nullptr);
    else
      stage_fused_kernel<NB, 2, S, 0, 0, false, SCH, 0><<<nslots * S, Geo<NB, 2, S, 0>::NT, Geo<NB, 2, S, 0>::SMEM, s>>>(
          G, state, u1, slots, d_dt, h_dt, records, st, nullptr, nullptr, nullptr);
    count_launch();
    *nrecords = (long long)nslots * S;
  }
  return cudaGetLastError();
}

// Load (CUDA lazy loading) the telescoped gather-mode kernels of this block
// size and scheme ahead of time, with their shared-memory attribute: loading
// mid-step may wait for an idle device (F2 peer mode: a rank spinning in a
// barrier never lets it go idle).
template <int NB, int SCH>
static cudaError_t preload_nb() {
  constexpr int S1 = NB == 16 ? 2 : NB == 32 ? 4 : 1;
  cudaError_t e = stage_attrs<NB, 1, S1, 0, SCH>();
  if (e == cudaSuccess) e = stage_attrs<NB, 2, S1, 0, SCH>();
  return e;
}

// The exported entry points of one (block size, scheme) translation unit.
#define ORCHA_FUSED_TU(NB, SCH)                                                                                  \
  cudaError_t fused_advance_n##NB##_s##SCH(const DevGrid& G, double* state, double* u1, int nslots,             \
                                           const SlotInfo* slots, const double* d_dt, double h_dt,              \
                                           DtRecord* records, long long* nrecords, DevStatus* st,               \
                                           cudaStream_t s, const PushEntry* push, const NbrEntry* nbr, int pk,   \
                                           int parts) {                                                         \
    return launch_nb<NB, SCH>(G, state, u1, nslots, slots, d_dt, h_dt, records, nrecords, st, s, push, nbr, pk, \
                              parts);                                                                            \
  }                                                                                                              \
  cudaError_t fused_stage_n##NB##_s##SCH(const DevGrid& G, int stage, double* state, double* u1, int nslots,    \
                                         const SlotInfo* slots, const double* d_dt, double h_dt,                \
                                         DtRecord* records, long long* nrecords, DevStatus* st,                 \
                                         cudaStream_t s, const PushEntry* push, const NbrEntry* nbr, int pk) {  \
    return launch_stage_nb<NB, SCH>(G, stage, state, u1, nslots, slots, d_dt, h_dt, records, nrecords, st, s,   \
                                    push, nbr, pk);                                                              \
  }                                                                                                              \
  cudaError_t fused_preload_n##NB##_s##SCH() {                                                                   \
    cudaError_t e = preload_nb<NB, SCH>();                                                                       \
    return e == cudaSuccess ? hybrid_attrs<NB, SCH>() : e;                                                       \
  }                                                                                                              \
  cudaError_t fused_hybrid_n##NB##_s##SCH(const DevGrid& G, double* state, double* u1, int nslots,              \
                                          const SlotInfo* slots, const int* smap, const int* nb4, int nint,            \
                                          const PushEntry* hpush, const NbrEntry* nbr,                           \
                                          const double* d_dt, double h_dt, DtRecord* records,                    \
                                          long long* nrecords, DevStatus* st, cudaStream_t s,                    \
                                          const PushEntry* push, int parts, cudaStream_t side,                   \
                                          cudaEvent_t ev_fork, cudaEvent_t ev_join) {                            \
    return launch_hybrid_nb<NB, SCH>(G, state, u1, nslots, slots, smap, nb4, nint, hpush, nbr, d_dt, h_dt,       \
                                     records, nrecords, st, s, push, parts, side, ev_fork, ev_join);              \
  }

}  // namespace orcha
