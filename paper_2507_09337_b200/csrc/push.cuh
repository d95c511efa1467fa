// push.cuh -- scatter form of the guard fill, used in the
// epilogue of the kernels that produce a new state.
//
// The gather fill sets guard g of block T to the per-axis image of one
// interior cell of one block S (shift into the neighbour, clamp to the edge
// cell for outflow, mirror for reflect; the images compose axis by axis, which
// is the global axis-ordered ghost fill).  Inverting that map per axis: an
// interior cell l of S feeds, along axis a,
//   itself (o = 0, t = l), and
//   if l >= n - ng:  shift: the +a neighbour's guard t = l - n
//                    mirror: S's own +a guard t = 2n - 1 - l (negated momentum a)
//                    clamp:  S's own +a guards t = n .. n+ng-1 if l == n - 1
//   if l <  ng:      shift: the -a neighbour's guard t = l + n
//                    mirror: S's own -a guard t = -1 - l
//                    clamp:  S's own -a guards t = -ng .. -1 if l == 0
// and every combination of per-axis choices except "all stay" is one guard
// cell (of the block the push table names for that direction).  Pure copies:
// bitwise the values the gather fill would produce.
#pragma once

#include "hydro_math.cuh"
#include "orcha_internal.h"

namespace orcha {

// Per axis: offset o (0 = no push along this axis), first target coordinate
// t0 and the number of targets (1; ng for a clamped edge cell).
struct AxisPush {
  int o, t0, cnt;
};

__device__ __forceinline__ AxisPush axis_push(const PushEntry* __restrict__ tab, int a, int l, int n, int g) {
  AxisPush r{0, l, 1};
  if (g == 0) return r;
  if (l >= n - g) {
    const int m = (tab[(a == 0) ? 14 : (a == 1) ? 16 : 22].mode >> (2 * a)) & 3;  // direction +a
    if (m == kShift) r = AxisPush{1, l - n, 1};
    else if (m == kMirror) r = AxisPush{1, 2 * n - 1 - l, 1};
    else if (l == n - 1) r = AxisPush{1, n, g};
  } else if (l < g) {
    const int m = (tab[(a == 0) ? 12 : (a == 1) ? 10 : 4].mode >> (2 * a)) & 3;   // direction -a
    if (m == kShift) r = AxisPush{-1, l + n, 1};
    else if (m == kMirror) r = AxisPush{-1, -1 - l, 1};
    else if (l == 0) r = AxisPush{-1, -g, g};
  }
  return r;
}

__device__ __forceinline__ void push_cell(const DevGrid& G, const PushEntry* __restrict__ tab, int i, int j,
                                          int k, const double v[5]) {
  const AxisPush px = axis_push(tab, 0, i, G.nb[0], G.gd[0]);
  const AxisPush py = axis_push(tab, 1, j, G.nb[1], G.gd[1]);
  const AxisPush pz = axis_push(tab, 2, k, G.nb[2], G.gd[2]);
  if ((px.o | py.o | pz.o) == 0) return;
  const long long cube = G.cube;
#pragma unroll
  for (int c = 1; c < 8; c++) {  // combinations of (stay | push) per axis, "all stay" excluded
    const int ox = (c & 1) ? px.o : 0, oy = (c & 2) ? py.o : 0, oz = (c & 4) ? pz.o : 0;
    if (((c & 1) && !px.o) || ((c & 2) && !py.o) || ((c & 4) && !pz.o)) continue;
    const PushEntry e = tab[(oz + 1) * 9 + (oy + 1) * 3 + (ox + 1)];
    if (e.dst == nullptr) continue;  // target in another packet or rank: gathered / exchanged
    const int nx = (c & 1) ? px.cnt : 1, ny = (c & 2) ? py.cnt : 1, nz = (c & 4) ? pz.cnt : 1;
    const int tx = (c & 1) ? px.t0 : i, ty = (c & 2) ? py.t0 : j, tz = (c & 4) ? pz.t0 : k;
    double w[5];
#pragma unroll
    for (int q = 0; q < 5; q++) w[q] = ((e.flip >> q) & 1) ? -v[q] : v[q];
    if (nx == 1 && ny == 1 && nz == 1) {  // shift / mirror: one target
      double* p = e.dst + cell_off(G, tx, ty, tz);
#pragma unroll
      for (int q = 0; q < 5; q++) p[q * cube] = w[q];
    } else {                              // clamped edge cell: ng copies along the clamped axes
      for (int zz = 0; zz < nz; zz++)
        for (int yy = 0; yy < ny; yy++)
          for (int xx = 0; xx < nx; xx++) {
            double* p = e.dst + cell_off(G, tx + xx, ty + yy, tz + zz);
#pragma unroll
            for (int q = 0; q < 5; q++) p[q * cube] = w[q];
          }
    }
  }
}

}  // namespace orcha
