// kernels_common.cu -- guard fill, pack/unpack, dt reduction (sm_100a, fp64).
#include <cfloat>

#include "hydro_math.cuh"
#include "reduce.cuh"
#include "orcha_internal.h"

namespace orcha {

// ------------------------------------------------------------ guard fill --
// One thread per padded cell of every slot; interior cells return at once.
// Guard (i,j,k) reads the neighbour-table entry of its direction and maps
// each axis: shift (neighbour or periodic image), clamp (outflow: edge cell)
// or mirror (reflect, negating the normal momentum) -- the per-axis images
// compose to the global axis-ordered ghost fill.
// faces_only: fill only the face slabs (one axis outside the interior) to
// depth `depth` -- the stencil of ONE RK2 stage (per-stage variant, F1).
__global__ void __launch_bounds__(256) fill_kernel(DevGrid G, double* __restrict__ state,
                                                   long long total, const NbrEntry* __restrict__ table,
                                                   int faces_only, int depth) {
  // faces_only: 0 every guard, 1 face guards to `depth`, 2 the gather-mode
  // complement: x-guard cells of the y/z-guard rows whose row source is
  // remote (the exchange wrote the row's interior part into our guards; the
  // parts sourced from resident blocks are written here)
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  long long cells = (long long)G.P[0] * G.P[1] * G.P[2];
  long long slot = t / cells;
  long long c = t - slot * cells;
  int pi = (int)(c % G.P[0]);
  int pj = (int)((c / G.P[0]) % G.P[1]);
  int pk = (int)(c / ((long long)G.P[0] * G.P[1]));
  int l[3] = {pi - G.gd[0], pj - G.gd[1], pk - G.gd[2]};
  int o[3];
#pragma unroll
  for (int d = 0; d < 3; d++) o[d] = (l[d] < 0) ? -1 : (l[d] >= G.nb[d]) ? 1 : 0;
  if (o[0] == 0 && o[1] == 0 && o[2] == 0) return;
  if (faces_only == 2) {
    if (o[0] == 0 || (o[1] == 0 && o[2] == 0)) return;
    if (table[slot * 27 + (o[2] + 1) * 9 + (o[1] + 1) * 3 + 1].src != nullptr) return;  // row gathered by stage 1
  } else if (faces_only) {
    int outside = (o[0] != 0) + (o[1] != 0) + (o[2] != 0);
    bool deep = false;
#pragma unroll
    for (int d = 0; d < 3; d++) deep |= (l[d] < -depth) || (l[d] >= G.nb[d] + depth);
    if (outside > 1 || deep) return;
  }
  NbrEntry e = table[slot * 27 + (o[2] + 1) * 9 + (o[1] + 1) * 3 + (o[0] + 1)];
  if (e.src == nullptr) return;  // remote source: written by the halo exchange
  int s[3];
#pragma unroll
  for (int d = 0; d < 3; d++) {
    int m = (e.mode >> (2 * d)) & 3;
    int n = G.nb[d];
    if (o[d] == 0) s[d] = l[d];
    else if (m == kShift) s[d] = l[d] - o[d] * n;
    else if (m == kClamp) s[d] = (o[d] < 0) ? 0 : n - 1;
    else s[d] = (o[d] < 0) ? -1 - l[d] : 2 * n - 1 - l[d];
  }
  long long so = cell_off(G, s[0], s[1], s[2]);
  double* dst = state + slot * kNVar * G.cube + c;
#pragma unroll
  for (int v = 0; v < kNVar; v++) {
    double x = e.src[v * G.cube + so];
    if ((e.flip >> v) & 1) x = -x;
    dst[v * G.cube] = x;
  }
}

// x-guards only (gather mode: the fused stage 1 stages its y/z guard rows from
// the owning blocks, whose x-guards this fills).  One thread per x-guard cell.
__global__ void __launch_bounds__(256) fill_x_kernel(DevGrid G, double* __restrict__ state, long long total,
                                                     const NbrEntry* __restrict__ table) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int g = G.gd[0], n0 = G.nb[0];
  int q = (int)(t % (2 * g));
  long long r = t / (2 * g);
  int j = (int)(r % G.nb[1]);
  r /= G.nb[1];
  int k = (int)(r % G.nb[2]);
  long long slot = r / G.nb[2];
  const int side = q >= g;
  const int l = side ? n0 + (q - g) : q - g;
  const NbrEntry e = table[slot * 27 + (side ? 14 : 12)];
  if (e.src == nullptr) return;  // remote: exchanged
  const int m = e.mode & 3;
  const int sx = (m == kShift) ? l - (side ? n0 : -n0) : (m == kClamp) ? (side ? n0 - 1 : 0)
                                                                      : (side ? 2 * n0 - 1 - l : -1 - l);
  const long long so = cell_off(G, sx, j, k);
  double* dst = state + slot * kNVar * G.cube + cell_off(G, l, j, k);
#pragma unroll
  for (int v = 0; v < kNVar; v++) {
    double x = e.src[v * G.cube + so];
    if ((e.flip >> v) & 1) x = -x;
    dst[v * G.cube] = x;
  }
}

cudaError_t launch_fill_x(const DevGrid& G, double* state, int nslots, const NbrEntry* table, cudaStream_t s) {
  long long total = (long long)nslots * G.nb[2] * G.nb[1] * 2 * G.gd[0];
  fill_x_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(G, state, total, table);
  count_launch();
  return cudaGetLastError();
}

// Every slot of several packets in one launch: slot (slot0 + blockIdx.y)'s
// cube base and its 27 table entries come from sf (one slot per grid row, so
// the descriptor load is uniform across the CTA); same per-cell code as
// fill_kernel.
__global__ void __launch_bounds__(256) fill_multi_kernel(DevGrid G, const SlotFill* __restrict__ sf,
                                                         long long slot0, int faces_only) {
  const long long cells = (long long)G.P[0] * G.P[1] * G.P[2];
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const long long slot = slot0 + blockIdx.y;
  int pi = (int)(c % G.P[0]);
  int pj = (int)((c / G.P[0]) % G.P[1]);
  int pk = (int)(c / ((long long)G.P[0] * G.P[1]));
  int l[3] = {pi - G.gd[0], pj - G.gd[1], pk - G.gd[2]};
  int o[3];
#pragma unroll
  for (int d = 0; d < 3; d++) o[d] = (l[d] < 0) ? -1 : (l[d] >= G.nb[d]) ? 1 : 0;
  if (o[0] == 0 && o[1] == 0 && o[2] == 0) return;
  if (faces_only) {
    int outside = (o[0] != 0) + (o[1] != 0) + (o[2] != 0);
    bool deep = false;
#pragma unroll
    for (int d = 0; d < 3; d++) deep |= (l[d] < -2) || (l[d] >= G.nb[d] + 2);
    if (outside > 1 || deep) return;
  }
  // read-only-path loads of the descriptor and the table entry (16 bytes each)
  const longlong2 fd = __ldg(reinterpret_cast<const longlong2*>(sf) + slot);
  const longlong2 raw =
      __ldg(reinterpret_cast<const longlong2*>(fd.y) + ((o[2] + 1) * 9 + (o[1] + 1) * 3 + (o[0] + 1)));
  NbrEntry e;
  e.src = reinterpret_cast<const double*>(raw.x);
  e.mode = (int32_t)(raw.y & 0xffffffffll);
  e.flip = (int32_t)((unsigned long long)raw.y >> 32);
  SlotFill f;
  f.dst = reinterpret_cast<double*>(fd.x);
  if (e.src == nullptr) return;  // remote source: written by the halo exchange
  int s[3];
#pragma unroll
  for (int d = 0; d < 3; d++) {
    int m = (e.mode >> (2 * d)) & 3;
    int n = G.nb[d];
    if (o[d] == 0) s[d] = l[d];
    else if (m == kShift) s[d] = l[d] - o[d] * n;
    else if (m == kClamp) s[d] = (o[d] < 0) ? 0 : n - 1;
    else s[d] = (o[d] < 0) ? -1 - l[d] : 2 * n - 1 - l[d];
  }
  long long so = cell_off(G, s[0], s[1], s[2]);
  double* dst = f.dst + c;
#pragma unroll
  for (int v = 0; v < kNVar; v++) {
    double x = e.src[v * G.cube + so];
    if ((e.flip >> v) & 1) x = -x;
    dst[v * G.cube] = x;
  }
}

cudaError_t launch_fill_multi(const DevGrid& G, const SlotFill* sf, long long nslots, cudaStream_t s,
                              int faces_only) {
  const long long cells = (long long)G.P[0] * G.P[1] * G.P[2];
  for (long long s0 = 0; s0 < nslots; s0 += 65535) {
    const long long n = nslots - s0 < 65535 ? nslots - s0 : 65535;
    fill_multi_kernel<<<dim3((unsigned)((cells + 255) / 256), (unsigned)n), 256, 0, s>>>(G, sf, s0, faces_only);
    count_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_fill(const DevGrid& G, double* state, int nslots, const NbrEntry* table,
                        cudaStream_t s, int faces_only) {
  long long total = (long long)nslots * G.P[0] * G.P[1] * G.P[2];
  long long blocks = (total + 255) / 256;
  fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(G, state, total, table, faces_only, 2);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------- pack / unpack --
// staged: [slot][var][k][j][i] over nb extents (contiguous) <-> padded state.
__global__ void __launch_bounds__(256) pack_kernel(DevGrid G, double* __restrict__ state,
                                                   double* __restrict__ staged, long long total,
                                                   int to_state) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  long long ncell = (long long)G.nb[0] * G.nb[1] * G.nb[2];
  long long sv = t / ncell;  // slot*5 + var
  long long c = t - sv * ncell;
  int i = (int)(c % G.nb[0]);
  int j = (int)((c / G.nb[0]) % G.nb[1]);
  int k = (int)(c / ((long long)G.nb[0] * G.nb[1]));
  double* p = state + sv * G.cube + cell_off(G, i, j, k);
  if (to_state) *p = staged[t];
  else staged[t] = *p;
}

cudaError_t launch_pack(const DevGrid& G, double* state, const double* staged, int nslots,
                        bool to_state, cudaStream_t s) {
  long long total = (long long)nslots * kNVar * G.nb[0] * G.nb[1] * G.nb[2];
  long long blocks = (total + 255) / 256;
  pack_kernel<<<(unsigned)blocks, 256, 0, s>>>(G, state, const_cast<double*>(staged), total,
                                                to_state ? 1 : 0);
  count_launch();
  return cudaGetLastError();
}

__global__ void status_reset_kernel(DevStatus* st) {
  st->first_bad = ~0ull;
  st->floor_hits = 0ull;
}

cudaError_t launch_status_reset(DevStatus* st, cudaStream_t s) {
  status_reset_kernel<<<1, 1, 0, s>>>(st);
  count_launch();
  return cudaGetLastError();
}

// Standalone CFL kernel (K4): one thread per interior cell, one record per CTA.
template <int NDIM>
__global__ void __launch_bounds__(256) dt_kernel(DevGrid G, const double* __restrict__ state,
                                                 long long total, const SlotInfo* __restrict__ slots,
                                                 DtRecord* __restrict__ rec, DevStatus* st) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double s = -DBL_MAX;
  long long g = LLONG_MAX;
  if (t < total) {
    long long ncell = (long long)G.nb[0] * G.nb[1] * G.nb[2];
    long long slot = t / ncell;
    long long c = t - slot * ncell;
    int i = (int)(c % G.nb[0]);
    int j = (int)((c / G.nb[0]) % G.nb[1]);
    int k = (int)(c / ((long long)G.nb[0] * G.nb[1]));
    const double* p = state + slot * kNVar * G.cube + cell_off(G, i, j, k);
    bool fl;
    Prim q = eos_var(p[0], p[G.cube], p[2 * G.cube], p[3 * G.cube], p[4 * G.cube], G, &fl);
    s = signal_speed_var<NDIM>(q, G);
    SlotInfo si = slots[slot];
    long long gi = (long long)si.bc[0] * G.nb[0] + i;
    long long gj = (long long)si.bc[1] * G.nb[1] + j;
    long long gk = (long long)si.bc[2] * G.nb[2] + k;
    g = (gk * G.N[1] + gj) * G.N[0] + gi;
    if (!(q.r > 0.0)) atomicMin(&st->first_bad, (unsigned long long)g);
  }
  block_reduce_rec<256>(s, g);
  if (threadIdx.x == 0) { rec[blockIdx.x].s = s; rec[blockIdx.x].g = g; }
}

cudaError_t launch_dt(const DevGrid& G, const double* state, int nslots, const SlotInfo* slots,
                      DtRecord* records, long long* nrecords, DevStatus* st, cudaStream_t s) {
  long long total = (long long)nslots * G.nb[0] * G.nb[1] * G.nb[2];
  long long blocks = (total + 255) / 256;
  if (G.ndim == 1) dt_kernel<1><<<(unsigned)blocks, 256, 0, s>>>(G, state, total, slots, records, st);
  else if (G.ndim == 2) dt_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(G, state, total, slots, records, st);
  else dt_kernel<3><<<(unsigned)blocks, 256, 0, s>>>(G, state, total, slots, records, st);
  count_launch();
  *nrecords = blocks;
  return cudaGetLastError();
}

__global__ void __launch_bounds__(1024) dt_reduce_kernel(const DtRecord* __restrict__ rec, long long n,
                                                         DtRecord* out) {
  double s = -DBL_MAX;
  long long g = LLONG_MAX;
  for (long long t = threadIdx.x; t < n; t += blockDim.x) rec_combine(s, g, rec[t].s, rec[t].g);
  block_reduce_rec<1024>(s, g);
  if (threadIdx.x == 0) { out->s = s; out->g = g; }
}

cudaError_t launch_dt_reduce(const DtRecord* records, long long n, DtRecord* out, cudaStream_t s) {
  dt_reduce_kernel<<<1, 1024, 0, s>>>(records, n, out);
  count_launch();
  return cudaGetLastError();
}

__global__ void dt_gather_rec_kernel(const DtRecord* r, const DevStatus* st, GatherRec* out) {
  out->s = r->s;
  out->g = r->g;
  out->bad = st->first_bad != ~0ull ? 1 : 0;
  out->pad = 0;
}

cudaError_t launch_dt_gather_rec(const DtRecord* r, const DevStatus* st, GatherRec* out, cudaStream_t s) {
  dt_gather_rec_kernel<<<1, 1, 0, s>>>(r, st, out);
  count_launch();
  return cudaGetLastError();
}

// The host rule of orcha_compute_dt on the device (same IEEE operations, so
// bitwise the same dt): combine the ranks' records (max s, ties -> lowest g),
// dt = cfl / s_max, then the t_end clamp; clock->t advances by dt.
__device__ void dt_finish(const GatherRec* all, int nall, double cfl, DevClock* c);
__global__ void dt_finish_kernel(const GatherRec* all, int nall, double cfl, DevClock* c) { dt_finish(all, nall, cfl, c); }
__device__ void dt_finish(const GatherRec* all, int nall, double cfl, DevClock* c) {
  double sm = all[0].s;
  long long gm = all[0].g;
  long long bad = 0;
  for (int q = 0; q < nall; q++) {
    if (dt_better(all[q].s, all[q].g, sm, gm)) { sm = all[q].s; gm = all[q].g; }
    bad |= all[q].bad;
  }
  double dt = cfl / sm;
  int tag = 0;
  const double rem = c->t_end - c->t;
  if (rem < dt) { dt = rem; tag = 1; }
  c->dt = dt;
  c->smax = sm;
  c->argmax = gm;
  c->tag = tag;
  c->nonphysical = bad ? 1 : 0;
  c->t = c->t + dt;
  c->steps = c->steps + 1;
}

// One packet, one rank: dt_reduce + dt_gather_rec + dt_finish in one launch
// (the same combine rule, so the same dt, argmax and side outputs: the
// packet's reduced record `out` and its gather record `grec`).
__global__ void __launch_bounds__(1024) dt_reduce_finish_kernel(const DtRecord* __restrict__ rec, long long n,
                                                                DtRecord* out, const DevStatus* st,
                                                                GatherRec* grec, double cfl, DevClock* c) {
  double s = -DBL_MAX;
  long long g = LLONG_MAX;
  for (long long t = threadIdx.x; t < n; t += blockDim.x) rec_combine(s, g, rec[t].s, rec[t].g);
  block_reduce_rec<1024>(s, g);
  if (threadIdx.x == 0) {
    out->s = s;
    out->g = g;
    GatherRec r;
    r.s = s;
    r.g = g;
    r.bad = st->first_bad != ~0ull ? 1 : 0;
    r.pad = 0;
    *grec = r;
    dt_finish(&r, 1, cfl, c);
  }
}

cudaError_t launch_dt_reduce_finish(const DtRecord* records, long long n, DtRecord* out, const DevStatus* st,
                                    GatherRec* grec, double cfl, void* clock, cudaStream_t s) {
  dt_reduce_finish_kernel<<<1, 1024, 0, s>>>(records, n, out, st, grec, cfl, (DevClock*)clock);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_dt_finish(const GatherRec* all, int nall, double cfl, void* clock, cudaStream_t s) {
  dt_finish_kernel<<<1, 1, 0, s>>>(all, nall, cfl, (DevClock*)clock);
  count_launch();
  return cudaGetLastError();
}

// Several packets at once: the records of every packet (same rule, so the
// result equals the host-side combination of the per-packet reductions) and
// the packets' sticky status words (lowest first_bad, summed floor hits).
__global__ void __launch_bounds__(1024) dt_reduce_multi_kernel(const PacketDt* __restrict__ pd, int npk,
                                                               DtRecord* out, DevStatus* out_st) {
  double s = -DBL_MAX;
  long long g = LLONG_MAX;
  for (int q = 0; q < npk; q++) {
    const DtRecord* rec = pd[q].rec;
    const long long n = pd[q].n;
    for (long long t = threadIdx.x; t < n; t += blockDim.x) rec_combine(s, g, rec[t].s, rec[t].g);
  }
  block_reduce_rec<1024>(s, g);
  if (threadIdx.x == 0) {
    out->s = s;
    out->g = g;
    unsigned long long fb = ~0ull, fh = 0;
    for (int q = 0; q < npk; q++) {
      fb = pd[q].st->first_bad < fb ? pd[q].st->first_bad : fb;
      fh += pd[q].st->floor_hits;
    }
    out_st->first_bad = fb;
    out_st->floor_hits = fh;
  }
}

cudaError_t launch_dt_reduce_multi(const PacketDt* pd, int npk, DtRecord* out, DevStatus* out_st, cudaStream_t s) {
  dt_reduce_multi_kernel<<<1, 1024, 0, s>>>(pd, npk, out, out_st);
  count_launch();
  return cudaGetLastError();
}

// Load (CUDA lazy loading) every kernel of this unit the device-dt step and
// the fill use, ahead of time: loading a module mid-step can wait for the
// device to go idle, which a rank spinning in a peer barrier never does.
cudaError_t common_preload() {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, fill_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, fill_x_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, dt_kernel<3>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, dt_reduce_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, dt_gather_rec_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, dt_finish_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, dt_reduce_finish_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, status_reset_kernel);
  return e;
}

}  // namespace orcha
