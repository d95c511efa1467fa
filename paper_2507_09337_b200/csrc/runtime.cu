// runtime.cu -- host side of liborcha.so: grid/packet bookkeeping, neighbour
// tables, the guard-fill plan cache, dt selection and the C ABI entry points.
//
// Bookkeeping is bit-exact by construction (integers only): global block id
// b = (bk*NBy + bj)*NBx + bi, slot = position in the caller's block_ids,
// global cell g = (k*Ny + j)*Nx + i.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <functional>
#include <unordered_map>

#include "comm.h"
#include "orcha_internal.h"

using namespace orcha;

// ------------------------------------------------------------ errors ------
static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

namespace orcha {
int32_t fail(int32_t code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int32_t cuda_fail(cudaError_t e, const char* what) {
  return fail(ORCHA_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void count_launch(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

long long cube_doubles(const DevGrid& G) {
  long long cells = (long long)G.P[0] * G.P[1] * G.P[2];
  long long bytes = cells * 8;
  bytes = (bytes + (long long)kAlign - 1) / (long long)kAlign * (long long)kAlign;
  return bytes / 8;
}
size_t state_bytes(const DevGrid& G, long long nslots) { return (size_t)nslots * kNVar * G.cube * 8; }
long long records_capacity(const DevGrid& G, long long nslots) {
  long long ncell = (long long)G.nb[0] * G.nb[1] * G.nb[2];
  return nslots * ((ncell + 63) / 64) + 64;
}

static int g_variant = -1;
int kernel_variant() {
  if (g_variant < 0) {
    const char* e = getenv("ORCHA_KERNEL");
    g_variant = (e && e[0] == '0') ? 0 : 1;
  }
  return g_variant;
}

cudaError_t launch_advance_ref(const DevGrid& G, double* state, double* u1, int nslots, const SlotInfo* slots,
                               const double* d_dt, double h_dt, DtRecord* records, long long* nrecords,
                               DevStatus* st, cudaStream_t s);
cudaError_t launch_advance_fused(const DevGrid& G, double* state, double* u1, int nslots, const SlotInfo* slots,
                                 const double* d_dt, double h_dt, DtRecord* records, long long* nrecords,
                                 DevStatus* st, cudaStream_t s, const PushEntry* push, const NbrEntry* nbr,
                                 bool push_x_only, int parts = 3);
cudaError_t launch_stage_ref(const DevGrid& G, int stage, double* state, double* u1, int nslots,
                             const SlotInfo* slots, const double* d_dt, double h_dt, DtRecord* records,
                             long long* nrecords, DevStatus* st, cudaStream_t s);
cudaError_t launch_stage_fused(const DevGrid& G, int stage, double* state, double* u1, int nslots,
                               const SlotInfo* slots, const double* d_dt, double h_dt, DtRecord* records,
                               long long* nrecords, DevStatus* st, cudaStream_t s, const PushEntry* push,
                               const NbrEntry* nbr, bool push_x_only);
bool fused_supported(const DevGrid& G);
cudaError_t fused_preload(const DevGrid& G);
long long fused_u1_cube(int nb);
cudaError_t launch_advance_hybrid(const DevGrid& G, double* state, double* u1, int nslots, const SlotInfo* slots,
                                  const int* smap, const int* nb4, int nint, const PushEntry* hpush, const NbrEntry* nbr,
                                  const double* d_dt, double h_dt, DtRecord* records,
                                  long long* nrecords, DevStatus* st, cudaStream_t s, const PushEntry* push,
                                  int parts, cudaStream_t side, cudaEvent_t ev_fork, cudaEvent_t ev_join);
}  // namespace orcha

// Fill mode: 1 = gather (default): when every guard source of the packet set
// is resident and the fused kernels run, the state fill writes only the
// x-guards and stage 1 stages its y/z guard rows straight from the owning
// blocks (kernels_fused.cu); 0 = full: the fill materialises every guard.
static int g_fill_mode = -1;
static int fill_mode() {
  if (g_fill_mode < 0) {
    const char* e = getenv("ORCHA_FILL_MODE");
    g_fill_mode = (e && e[0] == '0') ? 0 : 1;
  }
  return g_fill_mode;
}
extern "C" int32_t orcha_set_fill_mode(int32_t mode) {
  if (mode != 0 && mode != 1) return fail(ORCHA_E_ARG, "fill mode must be 0 (full) or 1 (gather)");
  g_fill_mode = mode;
  return ORCHA_OK;
}

// Guard push on/off.  Default OFF: measured on cfg4 the per-cell scatter in
// the stage-2 epilogue costs more (+1.0 ms) than the gather fill it removes
// (0.73 ms); ORCHA_PUSH=1 (or orcha_set_guard_push(1)) turns it on.
static int g_push = -1;
static bool push_enabled() {
  if (g_push < 0) {
    const char* e = getenv("ORCHA_PUSH");
    g_push = (e && e[0] == '1') ? 1 : 0;
  }
  return g_push == 1;
}
extern "C" int32_t orcha_set_guard_push(int32_t on) {
  g_push = on ? 1 : 0;
  return ORCHA_OK;
}

// Ring mode of the telescoped step (orcha_set_ring_mode): 1 = borrowed ring
// (default; fused_impl.cuh launch_hybrid_nb), 0 = every block computes its
// whole stage-1 ring.  Env ORCHA_RING overrides the default.
static int g_ring = -1;
static int ring_mode() {
  if (g_ring < 0) {
    const char* e = getenv("ORCHA_RING");
    g_ring = (e && atoi(e) == 0) ? 0 : 1;
  }
  return g_ring;
}
extern "C" int32_t orcha_set_ring_mode(int32_t mode) {
  if (mode != 0 && mode != 1) return fail(ORCHA_E_ARG, "ring mode must be 0 (computed) or 1 (borrowed)");
  g_ring = mode;
  return ORCHA_OK;
}
extern "C" int32_t orcha_get_ring_mode(void) { return ring_mode(); }

extern "C" const char* orcha_last_error(void) { return g_last_error.c_str(); }
extern "C" int64_t orcha_launch_count(void) { return g_launches.load(); }
extern "C" int32_t orcha_build_is_parity(void) {
#ifdef ORCHA_PARITY
  return 1;
#else
  return 0;
#endif
}
extern "C" int32_t orcha_set_kernel_variant(int32_t v) {
  if (v < 0 || v > 1) return fail(ORCHA_E_ARG, "kernel variant must be 0 (reference) or 1 (fused)");
  g_variant = v;
  return ORCHA_OK;
}
extern "C" int32_t orcha_get_kernel_variant(void) { return kernel_variant(); }

// -------------------------------------------------------------- grid ------
extern "C" int32_t orcha_grid_create(const orcha_grid_desc* d, orcha_grid** out) {
  if (!d || !out) return fail(ORCHA_E_ARG, "null argument");
  *out = nullptr;
  if (d->ndim < 1 || d->ndim > 3) return fail(ORCHA_E_ARG, "ndim must be 1, 2 or 3");
  if (d->ng < 4) return fail(ORCHA_E_HALO, "ng < 4: the telescoped RK2 step needs a twice-thick halo (2 x PLM radius)");
  for (int a = 0; a < 3; a++) {
    if (a < d->ndim) {
      if (d->nb[a] < 1 || d->nblk[a] < 1) return fail(ORCHA_E_ARG, "nb and nblk must be >= 1 on active axes");
      if (d->nb[a] < d->ng) return fail(ORCHA_E_ARG, "nb < ng: guards would need second neighbours");
      if (!(d->xmax[a] > d->xmin[a])) return fail(ORCHA_E_ARG, "xmax must exceed xmin");
      for (int s = 0; s < 2; s++)
        if (d->bc[a][s] < 0 || d->bc[a][s] > 2) return fail(ORCHA_E_ARG, "bad boundary code");
      if ((d->bc[a][0] == ORCHA_BC_PERIODIC) != (d->bc[a][1] == ORCHA_BC_PERIODIC))
        return fail(ORCHA_E_ARG, "periodic must be set on both sides of an axis");
    } else if (d->nb[a] != 1 || d->nblk[a] != 1) {
      return fail(ORCHA_E_ARG, "inactive axes must have nb = nblk = 1");
    }
  }
  if (!(d->gamma > 1.0) || !(d->cfl > 0.0) || !(d->smallp >= 0.0)) return fail(ORCHA_E_ARG, "bad gamma/cfl/smallp");
  if (d->riemann < 0 || d->riemann > 1 || d->limiter < 0 || d->limiter > 1)
    return fail(ORCHA_E_ARG, "riemann must be ORCHA_RIEMANN_HLL/HLLC and limiter ORCHA_LIMITER_MINMOD/MC");
  if (d->eos < 0 || d->eos > 1 || (d->eos == 1 && (d->eos_work < 1 || !(d->arad >= 0.0))))
    return fail(ORCHA_E_ARG, "eos must be ORCHA_EOS_GAMMA_LAW or ORCHA_EOS_GAS_RADIATION with eos_work >= 1, arad >= 0");
  orcha_grid* g = new orcha_grid();
  g->desc = *d;
  DevGrid& G = g->dev;
  G.ndim = d->ndim;
  G.ng = d->ng;
  g->nblocks = 1;
  for (int a = 0; a < 3; a++) {
    bool act = a < d->ndim;
    G.nb[a] = d->nb[a];
    G.gd[a] = act ? d->ng : 0;
    G.P[a] = d->nb[a] + 2 * G.gd[a];
    G.nblk[a] = d->nblk[a];
    G.N[a] = d->nb[a] * d->nblk[a];
    double dx = act ? (d->xmax[a] - d->xmin[a]) / (double)G.N[a] : 1.0;
    G.id[a] = act ? 1.0 / dx : 0.0;
    g->nblocks *= d->nblk[a];
  }
  G.cube = cube_doubles(G);
  G.gamma = d->gamma;
  G.gm1 = d->gamma - 1.0;
  G.ig1 = 1.0 / (d->gamma - 1.0);
  G.riemann = d->riemann;
  G.limiter = d->limiter;
  G.eos = d->eos;
  G.eos_work = d->eos_work < 1 ? 1 : d->eos_work;
  G.arad = d->arad;
  G.cfl = d->cfl;
  G.smallp = d->smallp;
  *out = g;
  return ORCHA_OK;
}

extern "C" int32_t orcha_grid_destroy(orcha_grid* g) {
  delete g;
  return ORCHA_OK;
}
extern "C" int64_t orcha_grid_nblocks(const orcha_grid* g) { return g ? g->nblocks : -1; }

// ------------------------------------------------------------ packets -----
namespace {
struct Tail {
  size_t status_off, result_off, records_off, bytes;
};
Tail tail_layout(const DevGrid& G, long long nslots) {
  Tail t;
  t.status_off = state_bytes(G, nslots);  // the U1 cubes come first
  t.result_off = t.status_off + 256;
  t.records_off = t.result_off + 256;
  t.bytes = t.records_off + (size_t)records_capacity(G, nslots) * sizeof(DtRecord);
  t.bytes = (t.bytes + kAlign - 1) / kAlign * kAlign;
  return t;
}
}  // namespace

extern "C" int32_t orcha_packet_bytes(const orcha_grid* g, int32_t n, size_t* sb, size_t* xb) {
  if (!g || n < 1) return fail(ORCHA_E_ARG, "grid null or nblocks < 1");
  if (sb) *sb = state_bytes(g->dev, n);
  if (xb) *xb = tail_layout(g->dev, n).bytes;
  return ORCHA_OK;
}

// Borrowed-ring tables of one packet: the slot map (slots with an x / y self
// side first -- box, then 18 x 18 -- then the interior ones; each entry slot |
// self-side mask << 26) and the ring push table (face directions).
struct HybTables {
  int* d_smap = nullptr;
  int nb4[4] = {0, 0, 0, 0};  // box, 18 x 18 (16^3; other sizes: box only), unused, unused
  int nint = 0;
  PushEntry* d_push = nullptr;
};

struct FillPlan {
  std::vector<orcha_packet*> packets;
  std::vector<NbrEntry*> d_tables;   // one per packet (library-owned device memory)
  std::vector<NbrEntry*> d_tables_u1;  // same, sources in the stage-1 buffers (per-stage variant)
  std::vector<PushEntry*> d_push;      // push tables (targets in the states), one per packet
  std::vector<PushEntry*> d_push_u1;   // push tables (targets in the stage-1 buffers)
  std::vector<NbrEntry*> d_cross;      // gather tables of the cross-packet directions only (or null)
  std::vector<NbrEntry*> d_cross_u1;
  CommPlan* remote = nullptr;        // guard cells sourced from other ranks (comm.cu)
  bool has_remote = false;
  orcha_comm* peer = nullptr;        // F2 peer mode: other ranks' blocks addressed directly (no exchange)
  std::vector<orcha_packet*> sources;  // every packet the tables point into (own + peer mode's other ranks')
  // gather mode with remote sources: some y/z-guard row of the packet has a
  // remote source while one of its x-guard parts has a resident one
  std::vector<char> edge_fix;
  // multi-packet sets: every slot's (cube base, table) for one fill launch
  SlotFill* d_sf = nullptr;
  SlotFill* d_sf_u1 = nullptr;
  long long nslots_total = 0;
  // borrowed-ring telescoped step (not peer mode; fused_impl.cuh
  // launch_hybrid_nb), one set of tables per packet
  std::vector<HybTables> hyb;
};
// Frees a plan's device tables and the plan (not its packets' pointers).
static void free_plan_tables(FillPlan* f) {
  for (auto* t : f->d_tables) cudaFree(t);
  for (auto* t : f->d_tables_u1) cudaFree(t);
  for (auto* t : f->d_push) cudaFree(t);
  for (auto* t : f->d_push_u1) cudaFree(t);
  for (auto* t : f->d_cross) cudaFree(t);
  for (auto* t : f->d_cross_u1) cudaFree(t);
  cudaFree(f->d_sf);
  cudaFree(f->d_sf_u1);
  for (auto& h : f->hyb) {
    cudaFree(h.d_smap);
    cudaFree(h.d_push);
  }
  delete f;
}

// Multi-packet dt reduction: the packet set's record/status pointers and a
// device result (one kernel, one download per orcha_compute_dt call).
struct DtPlan {
  std::vector<orcha_packet*> packets;
  PacketDt* d_pd = nullptr;
  DtRecord* d_out = nullptr;   // followed by a DevStatus; + 64 B: a GatherRec (orcha_compute_dt_device)
  GatherRec* d_rec = nullptr;
  std::vector<PacketDt> uploaded;  // the table in d_pd (re-uploaded only when it changes)
};

// The packets' record table for the multi-packet reduction, uploaded only
// when it differs from the last upload (so steady-state calls enqueue
// kernels only: capturable in a CUDA graph).
static cudaError_t upload_dt_table(DtPlan* dp, orcha_packet* const* pk, int npk, cudaStream_t s) {
  std::vector<PacketDt> h(npk);
  for (int q = 0; q < npk; q++) h[q] = PacketDt{pk[q]->records, pk[q]->nrecords, pk[q]->status};
  bool same = dp->uploaded.size() == h.size();
  for (int q = 0; same && q < npk; q++)
    same = dp->uploaded[q].rec == h[q].rec && dp->uploaded[q].n == h[q].n && dp->uploaded[q].st == h[q].st;
  if (same) return cudaSuccess;
  cudaError_t e = cudaMemcpyAsync(dp->d_pd, h.data(), npk * sizeof(PacketDt), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // h is a temporary
  if (e == cudaSuccess) dp->uploaded = h;
  return e;
}
static std::vector<DtPlan*> g_dtplans;
static std::mutex g_plan_mu;
static std::vector<FillPlan*> g_plans;

namespace orcha {
// A peer-mode communicator is going away: forget the plans built on it (their
// tables point into its ranks' packets) and detach its packets.
void runtime_drop_comm(const orcha_comm* c) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  for (size_t i = 0; i < g_plans.size();) {
    FillPlan* f = g_plans[i];
    if (f->peer == c) {
      for (auto* q : f->packets) {
        if (q->push_plan == f) { q->push_plan = nullptr; q->d_push = q->d_push_u1 = nullptr; }
        if (q->peer_comm == c) { q->peer_comm = nullptr; q->guards_valid = false; }
      }
      free_plan_tables(f);
      g_plans.erase(g_plans.begin() + i);
    } else {
      i++;
    }
  }
}
}  // namespace orcha

static void drop_plans_with(orcha_packet* p) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  for (size_t i = 0; i < g_plans.size();) {
    FillPlan* f = g_plans[i];
    bool hit = false;
    for (auto* q : f->sources) hit |= (q == p);
    if (hit) {
      for (auto* q : f->packets)
        if (q->push_plan == f) { q->push_plan = nullptr; q->d_push = q->d_push_u1 = nullptr; }
      comm_free_plan(f->remote);
      free_plan_tables(f);
      g_plans.erase(g_plans.begin() + i);
    } else {
      i++;
    }
  }
  for (size_t i = 0; i < g_dtplans.size();) {
    DtPlan* d = g_dtplans[i];
    bool hit = false;
    for (auto* q : d->packets) hit |= (q == p);
    if (hit) {
      cudaFree(d->d_pd);
      cudaFree(d->d_out);
      delete d;
      g_dtplans.erase(g_dtplans.begin() + i);
    } else {
      i++;
    }
  }
}

static int32_t get_dtplan(orcha_packet* const* pk, int npk, DtPlan** out) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  for (auto* d : g_dtplans) {
    if ((int)d->packets.size() != npk) continue;
    bool same = true;
    for (int q = 0; q < npk; q++) same &= d->packets[q] == pk[q];
    if (same) { *out = d; return ORCHA_OK; }
  }
  DtPlan* d = new DtPlan();
  d->packets.assign(pk, pk + npk);
  cudaError_t e = cudaMalloc(&d->d_pd, npk * sizeof(PacketDt));
  if (e == cudaSuccess) e = cudaMalloc(&d->d_out, 64 + sizeof(GatherRec));
  if (e == cudaSuccess) d->d_rec = (GatherRec*)((char*)d->d_out + 64);
  if (e != cudaSuccess) {
    cudaFree(d->d_pd);
    delete d;
    return cuda_fail(e, "dt plan");
  }
  g_dtplans.push_back(d);
  *out = d;
  return ORCHA_OK;
}

extern "C" int32_t orcha_packet_create(const orcha_grid* g, int32_t n, const int64_t* ids, void* d_state,
                                       void* d_scratch, orcha_packet** out) {
  if (!g || !ids || !out || n < 1) return fail(ORCHA_E_ARG, "null argument or nblocks < 1");
  *out = nullptr;
  if (!d_state || !d_scratch) return fail(ORCHA_E_ARG, "null device buffer");
  if (((uintptr_t)d_state % kAlign) || ((uintptr_t)d_scratch % kAlign))
    return fail(ORCHA_E_LAYOUT, "device buffers must be 256-byte aligned");
  std::unordered_map<long long, int> seen;
  for (int s = 0; s < n; s++) {
    if (ids[s] < 0 || ids[s] >= g->nblocks) return fail(ORCHA_E_RANGE, "block id out of range (BlockOutOfRange)");
    if (!seen.emplace(ids[s], s).second) return fail(ORCHA_E_RANGE, "duplicate block id in packet");
  }
  orcha_packet* p = new orcha_packet();
  p->grid = g;
  p->nslots = n;
  p->ids.assign(ids, ids + n);
  p->state = (double*)d_state;
  p->scratch = (double*)d_scratch;
  Tail t = tail_layout(g->dev, n);
  char* base = (char*)d_scratch;
  p->status = (DevStatus*)(base + t.status_off);
  p->result = (DtRecord*)(base + t.result_off);
  p->d_grec = (GatherRec*)(base + t.result_off + 64);
  p->records = (DtRecord*)(base + t.records_off);
  p->records_cap = records_capacity(g->dev, n);
  p->nrecords = 0;
  p->guards_valid = false;
  p->records_valid = false;
  p->stage1_done = false;
  p->u1_guards_valid = false;
  p->d_push = p->d_push_u1 = nullptr;
  p->push_plan = nullptr;
  p->guards_pushed = p->u1_pushed = false;
  p->xguards_pushed = false;
  p->guards_xonly = false;
  p->d_nbr = nullptr;
  p->u1_xpushed = p->u1_guards_xonly = false;
  p->d_nbr_u1 = nullptr;
  std::vector<SlotInfo> si(n);
  const DevGrid& G = g->dev;
  for (int s = 0; s < n; s++) {
    long long b = ids[s];
    si[s].bc[0] = (int)(b % G.nblk[0]);
    si[s].bc[1] = (int)((b / G.nblk[0]) % G.nblk[1]);
    si[s].bc[2] = (int)(b / ((long long)G.nblk[0] * G.nblk[1]));
    si[s].pad = 0;
  }
  cudaError_t e = cudaMalloc(&p->d_slots, sizeof(SlotInfo) * n);
  if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaMalloc(slot table)"); }
  e = cudaMemcpy(p->d_slots, si.data(), sizeof(SlotInfo) * n, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(p->d_slots); delete p; return cuda_fail(e, "upload slot table"); }
  e = launch_status_reset(p->status, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { cudaFree(p->d_slots); delete p; return cuda_fail(e, "status reset"); }
  *out = p;
  return ORCHA_OK;
}

extern "C" int32_t orcha_packet_destroy(orcha_packet* p) {
  if (!p) return ORCHA_OK;
  drop_plans_with(p);
  comm_drop_packet(p);
  cudaFree(p->d_slots);
  if (p->side) cudaStreamDestroy(p->side);
  if (p->ev_ready) cudaEventDestroy(p->ev_ready);
  if (p->ev_halo) cudaEventDestroy(p->ev_halo);
  delete p;
  return ORCHA_OK;
}

extern "C" int32_t orcha_packet_nblocks(const orcha_packet* p) { return p ? p->nslots : -1; }

extern "C" int32_t orcha_packet_layout(const orcha_packet* p, void** d_state, size_t* cube_bytes,
                                       int32_t padded_extent[3]) {
  if (!p) return fail(ORCHA_E_ARG, "null packet");
  if (d_state) *d_state = p->state;
  if (cube_bytes) *cube_bytes = (size_t)p->grid->dev.cube * 8;
  if (padded_extent)
    for (int a = 0; a < 3; a++) padded_extent[a] = p->grid->dev.P[a];
  return ORCHA_OK;
}

static size_t interior_bytes(const orcha_packet* p) {
  const DevGrid& G = p->grid->dev;
  return (size_t)p->nslots * kNVar * G.nb[0] * G.nb[1] * G.nb[2] * 8;
}

static int32_t pack_impl(orcha_packet* p, const double* src, cudaMemcpyKind kind, void* stream) {
  if (!p || !src) return fail(ORCHA_E_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(p->scratch, src, interior_bytes(p), kind, s);
  if (e != cudaSuccess) return cuda_fail(e, "pack copy");
  e = launch_pack(p->grid->dev, p->state, p->scratch, p->nslots, true, s);
  if (e == cudaSuccess) e = launch_status_reset(p->status, s);
  if (e != cudaSuccess) return cuda_fail(e, "pack kernel");
  p->guards_valid = false;
  p->records_valid = false;
  p->stage1_done = false;       // the staging area overwrote the stage-1 buffer
  p->u1_guards_valid = false;
  p->guards_pushed = p->u1_pushed = false;  // new interior, not scattered into any guards
  p->xguards_pushed = false;
  p->u1_xpushed = p->u1_guards_xonly = false;
  return ORCHA_OK;
}

static int32_t check_status(const orcha_packet* p, cudaStream_t s, DevStatus* out) {
  DevStatus st;
  cudaError_t e = cudaMemcpyAsync(&st, p->status, sizeof(st), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "read status");
  if (out) *out = st;
  if (st.first_bad != ~0ull) {
    char buf[160];
    snprintf(buf, sizeof buf, "non-physical state (rho <= 0 or non-finite) first at global cell %llu (NonPositiveState)",
             st.first_bad);
    return fail(ORCHA_E_NONPHYSICAL, buf);
  }
  return ORCHA_OK;
}

static int32_t unpack_impl(const orcha_packet* p, double* dst, cudaMemcpyKind kind, void* stream) {
  if (!p || !dst) return fail(ORCHA_E_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_pack(p->grid->dev, p->state, p->scratch, p->nslots, false, s);
  if (e != cudaSuccess) return cuda_fail(e, "unpack kernel");
  e = cudaMemcpyAsync(dst, p->scratch, interior_bytes(p), kind, s);
  if (e != cudaSuccess) return cuda_fail(e, "unpack copy");
  return check_status(p, s, nullptr);
}

extern "C" int32_t orcha_packet_pack(orcha_packet* p, const double* h, void* stream) {
  return pack_impl(p, h, cudaMemcpyHostToDevice, stream);
}
extern "C" int32_t orcha_packet_pack_device(orcha_packet* p, const double* d, void* stream) {
  return pack_impl(p, d, cudaMemcpyDeviceToDevice, stream);
}
extern "C" int32_t orcha_packet_unpack(const orcha_packet* p, double* h, void* stream) {
  return unpack_impl(p, h, cudaMemcpyDeviceToHost, stream);
}
extern "C" int32_t orcha_packet_unpack_async(const orcha_packet* p, double* dst, void* stream) {
  if (!p || !dst) return fail(ORCHA_E_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_pack(p->grid->dev, p->state, p->scratch, p->nslots, false, s);
  if (e != cudaSuccess) return cuda_fail(e, "unpack kernel");
  e = cudaMemcpyAsync(dst, p->scratch, interior_bytes(p), cudaMemcpyDefault, s);
  if (e != cudaSuccess) return cuda_fail(e, "unpack copy");
  return ORCHA_OK;
}
extern "C" int32_t orcha_packet_unpack_device(const orcha_packet* p, double* d, void* stream) {
  return unpack_impl(p, d, cudaMemcpyDeviceToDevice, stream);
}

extern "C" int32_t orcha_packet_counters(const orcha_packet* p, int64_t* floor_hits, int64_t* first_bad,
                                         void* stream) {
  if (!p) return fail(ORCHA_E_ARG, "null packet");
  DevStatus st;
  int32_t rc = check_status(p, (cudaStream_t)stream, &st);
  if (rc == ORCHA_E_CUDA) return rc;
  if (floor_hits) *floor_hits = (int64_t)st.floor_hits;
  if (first_bad) *first_bad = st.first_bad == ~0ull ? -1 : (int64_t)st.first_bad;
  return ORCHA_OK;
}

// -------------------------------------------------------- guard fill -----
// Neighbour-table entry for (block coords bc, direction o): per axis either
// stay (o=0), step to the neighbour (inside, or periodic wrap), clamp
// (outflow) or mirror (reflect, flip the normal momentum).
struct HostEntry {
  long long src_block;
  int mode, flip;
};
static HostEntry make_entry(const orcha_grid* g, const int bc[3], const int o[3]) {
  const DevGrid& G = g->dev;
  HostEntry h{0, 0, 0};
  int nb3[3];
  for (int a = 0; a < 3; a++) {
    int m = kShift;
    int c = bc[a] + o[a];
    if (o[a] != 0 && (c < 0 || c >= G.nblk[a])) {
      int code = g->desc.bc[a][o[a] < 0 ? 0 : 1];
      if (code == ORCHA_BC_PERIODIC) {
        c = (c + G.nblk[a]) % G.nblk[a];
      } else if (code == ORCHA_BC_OUTFLOW) {
        c = bc[a];
        m = kClamp;
      } else {
        c = bc[a];
        m = kMirror;
        h.flip |= 1 << (1 + a);
      }
    }
    nb3[a] = c;
    h.mode |= m << (2 * a);
  }
  h.src_block = ((long long)nb3[2] * G.nblk[1] + nb3[1]) * G.nblk[0] + nb3[0];
  return h;
}

// Borrowed ring (orcha_set_ring_mode): the self-side mask of block b (bit
// 2a: side -a, 2a+1: +a) -- a side is self unless its face neighbour is
// reached by a shift (not across a clamp / mirror boundary) and local_of()
// gives its slot in the same packet -- and, per side, that slot and the
// entry's axis modes (-1 on a self side).
static int ring_sides(const orcha_grid* g, long long b, const std::function<int(long long)>& local_of, int slot6[6],
                      int mode6[6]) {
  const DevGrid& G = g->dev;
  int bc[3] = {(int)(b % G.nblk[0]), (int)((b / G.nblk[0]) % G.nblk[1]), (int)(b / ((long long)G.nblk[0] * G.nblk[1]))};
  int mask = 0;
  for (int a = 0; a < 3; a++)
    for (int sd = 0; sd < 2; sd++) {
      int o[3] = {0, 0, 0};
      o[a] = sd ? 1 : -1;
      const int i = 2 * a + sd;
      slot6[i] = -1;
      mode6[i] = 0;
      if (a >= g->desc.ndim) {
        mask |= 1 << i;
        continue;
      }
      HostEntry h = make_entry(g, bc, o);
      const bool shift = ((h.mode >> (2 * a)) & 3) == kShift;
      const int ns = shift ? local_of(h.src_block) : -1;
      if (ns < 0) {
        mask |= 1 << i;
      } else {
        slot6[i] = ns;
        mode6[i] = h.mode;
      }
    }
  return mask;
}

// The stage-1 kernel group of a block with self-side mask `mask`: 2 = the
// interior kernel (no x / y self side), 1 = the (n+2)^2 kernel (16^3 and 8^3
// blocks with at most one self side per x / y axis), 0 = the box.
static int ring_group(const DevGrid& G, int mask) {
  const int sx = (mask & 1) + ((mask >> 1) & 1), sy = ((mask >> 2) & 1) + ((mask >> 3) & 1);
  if (sx == 0 && sy == 0) return 2;
  if ((G.nb[0] != 16 && G.nb[0] != 8) || sx == 2 || sy == 2) return 0;
  return 1;
}

extern "C" int32_t orcha_ring_classify(const orcha_grid* g, int32_t n, const int64_t* ids, int32_t* masks,
                                       int32_t* groups) {
  if (!g || n < 0 || (n > 0 && (!ids || !masks || !groups))) return fail(ORCHA_E_ARG, "null argument");
  std::unordered_map<long long, int> slot;
  for (int s = 0; s < n; s++) {
    if (ids[s] < 0 || ids[s] >= g->nblocks) return fail(ORCHA_E_RANGE, "block id out of range");
    if (!slot.emplace(ids[s], s).second) return fail(ORCHA_E_RANGE, "block listed twice");
  }
  auto local_of = [&](long long blk) -> int {
    auto it = slot.find(blk);
    return it == slot.end() ? -1 : it->second;
  };
  for (int s = 0; s < n; s++) {
    int ns6[6], md6[6];
    masks[s] = ring_sides(g, ids[s], local_of, ns6, md6);
    groups[s] = ring_group(g->dev, masks[s]);
  }
  return ORCHA_OK;
}

static int32_t build_plan(orcha_packet* const* pk_in, int npk, orcha_comm* comm, FillPlan** out) {
  const orcha_grid* g = pk_in[0]->grid;
  const DevGrid& G = g->dev;
  // F2 peer mode: the other ranks' packets join the set as sources and push
  // targets (their pointers, reached directly; cross-rank barriers order the
  // accesses), so nothing is exchanged.  ext = this rank's packets, then theirs.
  const bool peer = comm_peer_mode(comm);
  std::vector<orcha_packet*> ext(pk_in, pk_in + npk);
  if (peer) {
    if (npk != 1) return fail(ORCHA_E_ARG, "peer mode: one packet per rank");
    std::vector<orcha_packet*> others;
    int32_t rc = comm_peer_packets(comm, &others);
    if (rc) return rc;
    ext.insert(ext.end(), others.begin(), others.end());
  }
  orcha_packet* const* pk = ext.data();
  const int next = (int)ext.size();
  std::unordered_map<long long, std::pair<int, int>> where;  // block -> (packet, slot)
  for (int q = 0; q < next; q++) {
    if (pk[q]->grid != g) return fail(ORCHA_E_ARG, "packets belong to different grids");
    for (int s = 0; s < pk[q]->nslots; s++)
      if (!where.emplace(pk[q]->ids[s], std::make_pair(q, s)).second)
        return fail(ORCHA_E_RANGE, "block resident in two packets");
  }
  FillPlan* f = new FillPlan();
  f->packets.assign(pk, pk + npk);
  f->peer = peer ? comm : nullptr;
  f->sources = ext;
  for (int q = 0; q < npk; q++) {
    orcha_packet* p = pk[q];
    std::vector<NbrEntry> tab((size_t)p->nslots * 27);
    for (int s = 0; s < p->nslots; s++) {
      long long b = p->ids[s];
      int bc[3] = {(int)(b % G.nblk[0]), (int)((b / G.nblk[0]) % G.nblk[1]),
                   (int)(b / ((long long)G.nblk[0] * G.nblk[1]))};
      for (int oz = -1; oz <= 1; oz++)
        for (int oy = -1; oy <= 1; oy++)
          for (int ox = -1; ox <= 1; ox++) {
            int o[3] = {ox, oy, oz};
            NbrEntry& e = tab[(size_t)s * 27 + (oz + 1) * 9 + (oy + 1) * 3 + (ox + 1)];
            bool valid = true;
            for (int a = g->desc.ndim; a < 3; a++) valid &= (o[a] == 0);
            if (!valid) { e.src = p->state; e.mode = 0; e.flip = 0; continue; }
            HostEntry h = make_entry(g, bc, o);
            e.mode = h.mode;
            e.flip = h.flip;
            auto it = where.find(h.src_block);
            if (it == where.end()) {
              if (!comm) {
                free_plan_tables(f);
                return fail(ORCHA_E_RANGE, "neighbour block " + std::to_string(h.src_block) +
                                               " is not resident on this device and no communicator was given");
              }
              e.src = nullptr;
              f->has_remote = true;
            } else {
              orcha_packet* sp = pk[it->second.first];
              e.src = sp->state + (long long)it->second.second * kNVar * G.cube;
            }
          }
    }
    // the same table for the stage-1 buffer (per-stage variant): sources in
    // each source packet's scratch, which has the state's padded layout
    std::vector<NbrEntry> tab1 = tab;
    for (auto& e : tab1)
      if (e.src) {
        for (int q2 = 0; q2 < next; q2++) {
          orcha_packet* sp = pk[q2];
          if (e.src >= sp->state && e.src < sp->state + (long long)sp->nslots * kNVar * G.cube) {
            e.src = sp->scratch ? sp->scratch + (e.src - sp->state) : nullptr;  // IPC shadows: no stage-1 buffer
            break;
          }
        }
      }
    NbrEntry* d = nullptr;
    NbrEntry* d1 = nullptr;
    cudaError_t err = cudaMalloc(&d, tab.size() * sizeof(NbrEntry));
    if (err == cudaSuccess) err = cudaMemcpy(d, tab.data(), tab.size() * sizeof(NbrEntry), cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMalloc(&d1, tab1.size() * sizeof(NbrEntry));
    if (err == cudaSuccess) err = cudaMemcpy(d1, tab1.data(), tab1.size() * sizeof(NbrEntry), cudaMemcpyHostToDevice);
    if (err != cudaSuccess) {
      cudaFree(d);
      cudaFree(d1);
      free_plan_tables(f);
      return cuda_fail(err, "upload neighbour table");
    }
    f->d_tables.push_back(d);
    f->d_tables_u1.push_back(d1);
    char fix = 0;
    for (int s = 0; s < p->nslots && !fix; s++)
      for (int dd = 0; dd < 27; dd++) {
        const int ox = dd % 3 - 1, row = dd - (ox + 1) + 1;  // (0, oy, oz) of the same row
        if (ox != 0 && row != 13 && !tab[(size_t)s * 27 + row].src && tab[(size_t)s * 27 + dd].src) fix = 1;
      }
    f->edge_fix.push_back(fix);
    // push tables: target of direction o = make_entry(b, o).src_block (the
    // neighbour at b+o, or b itself across a clamp/mirror boundary)
    std::vector<PushEntry> pt((size_t)p->nslots * 27), pt1;
    for (int s = 0; s < p->nslots; s++) {
      long long b = p->ids[s];
      int bc[3] = {(int)(b % G.nblk[0]), (int)((b / G.nblk[0]) % G.nblk[1]),
                   (int)(b / ((long long)G.nblk[0] * G.nblk[1]))};
      for (int dd = 0; dd < 27; dd++) {
        int o[3] = {dd % 3 - 1, (dd / 3) % 3 - 1, dd / 9 - 1};
        PushEntry& e = pt[(size_t)s * 27 + dd];
        bool valid = true;
        for (int a = g->desc.ndim; a < 3; a++) valid &= (o[a] == 0);
        if (!valid) { e.dst = nullptr; e.mode = 0; e.flip = 0; continue; }
        HostEntry h = make_entry(g, bc, o);
        e.mode = h.mode;
        e.flip = h.flip;
        // same packet only: a push into another packet's guards would land
        // before that packet's own advance has read them (stage 1) -- except
        // into other ranks' packets in peer mode, whose stage 1 ends before
        // any stage 2 starts (the cross-rank barrier between the stages)
        auto it = where.find(h.src_block);
        e.dst = (it == where.end() || (it->second.first != q && !(peer && it->second.first >= npk)))
                    ? nullptr
                    : pk[it->second.first]->state + (long long)it->second.second * kNVar * G.cube;
      }
    }
    pt1 = pt;
    for (auto& e : pt1)
      if (e.dst)
        for (int q2 = 0; q2 < next; q2++) {
          orcha_packet* sp = pk[q2];
          if (e.dst >= sp->state && e.dst < sp->state + (long long)sp->nslots * kNVar * G.cube) {
            e.dst = sp->scratch ? sp->scratch + (e.dst - sp->state) : nullptr;
            break;
          }
        }
    PushEntry* dp = nullptr;
    PushEntry* dp1 = nullptr;
    err = cudaMalloc(&dp, pt.size() * sizeof(PushEntry));
    if (err == cudaSuccess) err = cudaMemcpy(dp, pt.data(), pt.size() * sizeof(PushEntry), cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMalloc(&dp1, pt1.size() * sizeof(PushEntry));
    if (err == cudaSuccess) err = cudaMemcpy(dp1, pt1.data(), pt1.size() * sizeof(PushEntry), cudaMemcpyHostToDevice);
    if (err != cudaSuccess) {
      cudaFree(dp);
      cudaFree(dp1);
      free_plan_tables(f);
      return cuda_fail(err, "upload push table");
    }
    f->d_push.push_back(dp);
    f->d_push_u1.push_back(dp1);
    // cross-packet gather tables: only the directions whose source block lives
    // in another resident packet (the pushes cover the same-packet ones)
    std::vector<NbrEntry> xc = tab, xc1 = tab1;
    bool any_cross = false;
    for (int s = 0; s < p->nslots; s++) {
      long long b = p->ids[s];
      int bc[3] = {(int)(b % G.nblk[0]), (int)((b / G.nblk[0]) % G.nblk[1]),
                   (int)(b / ((long long)G.nblk[0] * G.nblk[1]))};
      for (int dd = 0; dd < 27; dd++) {
        size_t i = (size_t)s * 27 + dd;
        if (!xc[i].src) continue;
        int o[3] = {dd % 3 - 1, (dd / 3) % 3 - 1, dd / 9 - 1};
        bool valid = true;
        for (int a = g->desc.ndim; a < 3; a++) valid &= (o[a] == 0);
        auto it = valid ? where.find(make_entry(g, bc, o).src_block) : where.end();
        if (!valid || it == where.end() || it->second.first == q) {
          xc[i].src = nullptr;
          xc1[i].src = nullptr;
        } else {
          any_cross = true;
        }
      }
    }
    NbrEntry* dx = nullptr;
    NbrEntry* dx1 = nullptr;
    if (any_cross) {
      err = cudaMalloc(&dx, xc.size() * sizeof(NbrEntry));
      if (err == cudaSuccess) err = cudaMemcpy(dx, xc.data(), xc.size() * sizeof(NbrEntry), cudaMemcpyHostToDevice);
      if (err == cudaSuccess) err = cudaMalloc(&dx1, xc1.size() * sizeof(NbrEntry));
      if (err == cudaSuccess) err = cudaMemcpy(dx1, xc1.data(), xc1.size() * sizeof(NbrEntry), cudaMemcpyHostToDevice);
      if (err != cudaSuccess) {
        cudaFree(dx);
        cudaFree(dx1);
        free_plan_tables(f);
        return cuda_fail(err, "upload cross-packet table");
      }
    }
    f->d_cross.push_back(dx);
    f->d_cross_u1.push_back(dx1);
  }
  if (fused_supported(G)) {
    // borrowed-ring telescoped step, per packet: a side of a block is "self"
    // when its neighbour is not a resident block of the SAME packet reached by
    // a shift (physical boundary: clamp / mirror; another rank; another
    // packet -- its stage 1 runs in another launch) -- there the block
    // computes its stage-1 ring itself, elsewhere it borrows it
    const long long U1C = fused_u1_cube(G.nb[0]);
    f->hyb.resize(npk);
    for (int q = 0; q < npk; q++) {
      orcha_packet* p = pk[q];
      if (p->nslots >= (1 << 26)) continue;
      HybTables& ht = f->hyb[q];
      std::vector<int> grp[4], inr;
      std::vector<PushEntry> hp((size_t)p->nslots * 27, PushEntry{nullptr, 0, 0});
      auto local_of = [&](long long blk) -> int {
        auto it = where.find(blk);
        return (it == where.end() || it->second.first != q) ? -1 : it->second.second;
      };
      for (int s = 0; s < p->nslots; s++) {
        int ns6[6], md6[6];
        const int mask = ring_sides(g, p->ids[s], local_of, ns6, md6);
        for (int a = 0; a < 3; a++)
          for (int sd = 0; sd < 2; sd++) {
            if (ns6[2 * a + sd] < 0) continue;
            int o[3] = {0, 0, 0};
            o[a] = sd ? 1 : -1;
            hp[(size_t)s * 27 + (o[2] + 1) * 9 + (o[1] + 1) * 3 + (o[0] + 1)] =
                PushEntry{p->scratch + (long long)ns6[2 * a + sd] * kNVar * U1C, md6[2 * a + sd], 0};
          }
        const int e = s | (mask << 26);
        const int grpk = ring_group(G, mask);
        if (grpk == 2) inr.push_back(e);
        else grp[grpk].push_back(e);
      }
      std::vector<int> smap;
      for (int k = 0; k < 4; k++) {
        smap.insert(smap.end(), grp[k].begin(), grp[k].end());
        ht.nb4[k] = (int)grp[k].size();
      }
      smap.insert(smap.end(), inr.begin(), inr.end());
      ht.nint = (int)inr.size();
      cudaError_t err = cudaMalloc(&ht.d_smap, smap.size() * sizeof(int));
      if (err == cudaSuccess)
        err = cudaMemcpy(ht.d_smap, smap.data(), smap.size() * sizeof(int), cudaMemcpyHostToDevice);
      if (err == cudaSuccess) err = cudaMalloc(&ht.d_push, hp.size() * sizeof(PushEntry));
      if (err == cudaSuccess)
        err = cudaMemcpy(ht.d_push, hp.data(), hp.size() * sizeof(PushEntry), cudaMemcpyHostToDevice);
      if (err != cudaSuccess) {
        free_plan_tables(f);
        return cuda_fail(err, "upload borrowed-ring tables");
      }
    }
  }
  if (npk > 1) {
    std::vector<SlotFill> sf, sf1;
    for (int q = 0; q < npk; q++)
      for (int s = 0; s < pk[q]->nslots; s++) {
        const long long off = (long long)s * kNVar * G.cube;
        sf.push_back(SlotFill{pk[q]->state + off, f->d_tables[q] + (size_t)s * 27});
        sf1.push_back(SlotFill{pk[q]->scratch + off, f->d_tables_u1[q] + (size_t)s * 27});
      }
    f->nslots_total = (long long)sf.size();
    cudaError_t err = cudaMalloc(&f->d_sf, sf.size() * sizeof(SlotFill));
    if (err == cudaSuccess) err = cudaMemcpy(f->d_sf, sf.data(), sf.size() * sizeof(SlotFill), cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMalloc(&f->d_sf_u1, sf1.size() * sizeof(SlotFill));
    if (err == cudaSuccess)
      err = cudaMemcpy(f->d_sf_u1, sf1.data(), sf1.size() * sizeof(SlotFill), cudaMemcpyHostToDevice);
    if (err != cudaSuccess) {
      free_plan_tables(f);
      return cuda_fail(err, "upload slot fill table");
    }
  }
  *out = f;
  return ORCHA_OK;
}

static int32_t get_plan(orcha_packet* const* pk, int npk, orcha_comm* comm, FillPlan** out) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  for (auto* f : g_plans) {
    if ((int)f->packets.size() != npk) continue;
    bool same = true;
    for (int q = 0; q < npk; q++) same &= f->packets[q] == pk[q];
    const orcha_comm* want_peer = comm_peer_mode(comm) ? comm : nullptr;
    if (same && f->peer == want_peer && (!f->has_remote || comm)) { *out = f; return ORCHA_OK; }
  }
  FillPlan* f = nullptr;
  int32_t rc = build_plan(pk, npk, comm, &f);
  if (rc) return rc;
  g_plans.push_back(f);
  *out = f;
  return ORCHA_OK;
}

// only >= 0: fill the guards of pk[only] alone (streamed packets: the set's
// tables, every source resident, no exchange).
static int32_t fill_impl_body(orcha_packet* const* pk, int32_t npk, orcha_comm* comm, int buffer,
                              bool faces_only, void* stream, int only);

// The guard fill phase (incl. the exchange, which is also timed on its own).
static int32_t fill_impl(orcha_packet* const* pk, int32_t npk, orcha_comm* comm, int buffer, bool faces_only,
                         void* stream, int only = -1) {
  PhaseScope ph(PH_FILL, (cudaStream_t)stream);
  return fill_impl_body(pk, npk, comm, buffer, faces_only, stream, only);
}

static cudaError_t hyb_side(orcha_packet* p);
// Borrowed ring: the box / 18 x 18 and interior stage-1 kernels of a packet
// go on two streams when both are big enough for the overlap to pay for the
// fork / join (small packets: one stream, no side stream created).
static bool hyb_fork(const HybTables& h) {
  return h.d_smap && h.nint >= 128 && h.nb4[0] + h.nb4[1] + h.nb4[2] + h.nb4[3] >= 64;
}

static int32_t fill_impl_body(orcha_packet* const* pk, int32_t npk, orcha_comm* comm, int buffer,
                              bool faces_only, void* stream, int only) {
  if (!pk || npk < 1) return fail(ORCHA_E_ARG, "no packets");
  if (buffer != 0 && buffer != 1) return fail(ORCHA_E_ARG, "buffer must be 0 (state) or 1 (stage-1 state)");
  for (int q = 0; q < npk; q++) {
    if (!pk[q]) return fail(ORCHA_E_ARG, "null packet");
    if (buffer == 1 && !pk[q]->stage1_done)
      return fail(ORCHA_E_STATE, "stage-1 buffer refill requires orcha_hydro_stage(packet, 1, ...) first");
  }
  FillPlan* f = nullptr;
  int32_t rc = get_plan(pk, npk, comm, &f);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (only >= 0 && f->has_remote)
    return fail(ORCHA_E_ARG, "a per-packet fill needs every source block resident (no exchange)");
  if (f->has_remote) {
    CommPlan* cp = nullptr;  // cached by the communicator per packet set and buffer
    rc = comm_build_plan(comm, pk, npk, buffer, &cp);
    if (rc == ORCHA_OK) {
      PhaseScope phx(PH_EXCHANGE, s);
      rc = comm_exchange(comm, cp, s);
    }
    if (rc) return rc;
  }
  // If every packet's last update of this buffer scattered itself into the
  // guards with this plan's push tables (push.cuh), the local guards are
  // already current: only the exchange above was needed.
  bool all_pushed = push_enabled();
  for (int q = 0; q < npk; q++)
    if (only < 0 || q == only) all_pushed &= pk[q]->push_plan == f && (buffer ? pk[q]->u1_pushed : pk[q]->guards_pushed);
  // gather mode (state only, fused kernels, ONE packet per device; remote
  // sources were exchanged into its own guards above): x-guards only, plus
  // the resident-sourced parts of exchanged rows.  With several packets the advances run one after
  // another and a later packet's stage 1 would read a neighbour packet's
  // already-advanced interior, so multi-packet sets keep the full fill; so
  // does the guard-push mode (its kernels have no gather staging).
  const DevGrid& G0 = pk[0]->grid->dev;
  const bool xonly = buffer == 0 && npk == 1 && !push_enabled() && fill_mode() == 1 &&
                     kernel_variant() == 1 && fused_supported(G0);
  // per-stage stage-1 buffer in gather mode: stage 1 wrote the U1 x-guards
  // (same plan), stage 2 stages the y/z rows of U1 from their owners
  const bool xonly_u1 = buffer == 1 && npk == 1 && !push_enabled() && fill_mode() == 1 && kernel_variant() == 1 &&
                        fused_supported(G0) && pk[0]->u1_xpushed && pk[0]->push_plan == f;
  if (f->peer) {
    // F2 peer mode: the gather fills only (x-guards; the stage kernels stage
    // y/z rows from the owners, other ranks' included, and push x-guards into
    // them) -- the telescoped step, or the per-stage one (F1) whose U1
    // "refill" is then a barrier: every rank's stage 1 (its U1 and the U1
    // x-guards it wrote into other ranks' blocks) before any stage 2 reads them
    if (only >= 0 || !(xonly || xonly_u1))
      return fail(ORCHA_E_STATE, "peer mode needs the gather fills (fill mode 1, fused kernels, one packet, no "
                                 "guard push)");
    if (buffer == 1 || !(pk[0]->xguards_pushed && pk[0]->push_plan == f)) {
      // buffer 0 after a pack: the x-guard fill reads other ranks' interiors,
      // so every rank's pack must be done
      rc = comm_peer_barrier(f->peer, s);
      if (rc) return rc;
    }
  }
  if (xonly_u1) {
    if (f->edge_fix[0]) {  // exchanged rows' resident-sourced x-guard parts
      cudaError_t e = launch_fill(G0, pk[0]->scratch, pk[0]->nslots, f->d_tables_u1[0], s, 2);
      if (e != cudaSuccess) return cuda_fail(e, "fill kernel");
    }
    pk[0]->u1_guards_valid = true;
    pk[0]->u1_guards_xonly = true;
    pk[0]->d_nbr_u1 = f->d_tables_u1[0];
    return ORCHA_OK;
  }
  // several packets, full tables: every slot of the set in one launch
  // (from 128 packets on: the one-launch kernel pays a dependent descriptor
  // load per cell, ~0.5 ms on 16.8 M cells, which below that is more than the
  // per-packet launches cost)
  const bool multi = npk >= 128 && !all_pushed && f->d_sf != nullptr && only < 0;
  if (multi) {
    cudaError_t e = launch_fill_multi(G0, buffer ? f->d_sf_u1 : f->d_sf, f->nslots_total, s, faces_only ? 1 : 0);
    if (e != cudaSuccess) return cuda_fail(e, "fill kernel");
  }
  for (int q = 0; q < npk && !multi; q++) {
    if (only >= 0 && q != only) continue;
    double* dst = buffer ? pk[q]->scratch : pk[q]->state;
    cudaError_t e;
    if (xonly) {
      // rows with a remote source were exchanged into our guards: their
      // x-guard parts with resident sources are filled here
      if (f->edge_fix[q]) {
        e = launch_fill(G0, dst, pk[q]->nslots, f->d_tables[q], s, 2);
        if (e != cudaSuccess) return cuda_fail(e, "fill kernel");
      }
      // the last advance scattered U^{n+1} into the x-guards with this plan: nothing to do
      if (pk[q]->xguards_pushed && pk[q]->push_plan == f) continue;
      e = launch_fill_x(G0, dst, pk[q]->nslots, f->d_tables[q], s);
      if (e == cudaSuccess && f->peer) {  // every rank's x-guards before any rank's stage 1 reads them
        rc = comm_peer_barrier(f->peer, s);
        if (rc) return rc;
      }
    } else {
      const NbrEntry* tab = all_pushed ? (buffer ? f->d_cross_u1[q] : f->d_cross[q])   // cross-packet only
                                       : (buffer ? f->d_tables_u1[q] : f->d_tables[q]);
      if (!tab) continue;  // pushed, and no source in another packet
      e = launch_fill(pk[q]->grid->dev, dst, pk[q]->nslots, tab, s, faces_only ? 1 : 0);
    }
    if (e != cudaSuccess) return cuda_fail(e, "fill kernel");
  }
  for (int q = 0; q < npk; q++) {
    if (only >= 0 && q != only) continue;
    if ((size_t)q < f->hyb.size() && hyb_fork(f->hyb[q])) {  // the borrowed ring's side stream, ahead of the advance
      cudaError_t e = hyb_side(pk[q]);
      if (e != cudaSuccess) return cuda_fail(e, "side stream");
    }
    pk[q]->d_push = f->d_push[q];
    pk[q]->plan_q = q;
    pk[q]->d_push_u1 = f->d_push_u1[q];
    pk[q]->push_plan = f;
    pk[q]->peer_comm = buffer ? pk[q]->peer_comm : f->peer;
    if (buffer) {
      pk[q]->u1_guards_valid = true;
      pk[q]->u1_guards_xonly = false;
    } else {
      pk[q]->guards_valid = true;
      pk[q]->guards_xonly = xonly;
      pk[q]->d_nbr = f->d_tables[q];
      // a push writes every same-packet guard; cross-packet ones are full unless faces-only;
      // in gather mode stage 1 composes the y/z guards itself
      pk[q]->guards_full = xonly || !faces_only || (all_pushed && f->d_cross[q] == nullptr);
    }
  }
  return ORCHA_OK;
}

extern "C" int32_t orcha_fill_prepare(orcha_packet* const* pk, int32_t npk, orcha_comm* comm) {
  if (!pk || npk < 1) return fail(ORCHA_E_ARG, "no packets");
  for (int q = 0; q < npk; q++)
    if (!pk[q]) return fail(ORCHA_E_ARG, "null packet");
  FillPlan* f = nullptr;
  int32_t rc = get_plan(pk, npk, comm, &f);
  if (rc) return rc;
  if (f->has_remote) {
    CommPlan* cp = nullptr;
    rc = comm_build_plan(comm, pk, npk, 0, &cp);
    if (rc) return rc;
  }
  // and load the step's kernels now (CUDA lazy loading would otherwise load
  // them at their first launch, which may wait for an idle device)
  cudaError_t e = fused_preload(pk[0]->grid->dev);
  return e == cudaSuccess ? ORCHA_OK : cuda_fail(e, "preload kernels");
}

extern "C" int32_t orcha_fill_guardcells(orcha_packet* const* pk, int32_t npk, orcha_comm* comm, void* stream) {
  return fill_impl(pk, npk, comm, 0, false, stream);
}

extern "C" int32_t orcha_fill_guardcells_packet(orcha_packet* const* pk, int32_t npk, int32_t index,
                                                void* stream) {
  if (!pk || index < 0 || index >= npk) return fail(ORCHA_E_ARG, "packet index out of range");
  return fill_impl(pk, npk, nullptr, 0, false, stream, index);
}

extern "C" int32_t orcha_fill_guardcells_stage(orcha_packet* const* pk, int32_t npk, orcha_comm* comm,
                                               int32_t buffer, void* stream) {
  return fill_impl(pk, npk, comm, buffer, true, stream);
}

// --------------------------------------------------------------- dt ------
// The per-packet CFL records of every packet whose records are stale (after a
// pack); an advance leaves valid ones (the fused stage-2 epilogue).
static int32_t ensure_dt_records(orcha_packet* const* pk, int32_t npk, cudaStream_t s) {
  for (int q = 0; q < npk; q++) {
    orcha_packet* p = pk[q];
    if (!p) return fail(ORCHA_E_ARG, "null packet");
    if (!p->records_valid) {
      cudaError_t e = launch_dt(p->grid->dev, p->state, p->nslots, p->d_slots, p->records, &p->nrecords,
                                p->status, s);
      if (e != cudaSuccess) return cuda_fail(e, "dt kernel");
      p->records_valid = true;
    }
  }
  return ORCHA_OK;
}

extern "C" int32_t orcha_packet_dt_records(orcha_packet* p, void* stream) {
  if (!p) return fail(ORCHA_E_ARG, "null packet");
  cudaError_t e = launch_dt(p->grid->dev, p->state, p->nslots, p->d_slots, p->records, &p->nrecords, p->status,
                            (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "dt kernel");
  p->records_valid = true;
  return ORCHA_OK;
}

extern "C" int32_t orcha_compute_dt(orcha_packet* const* pk, int32_t npk, orcha_comm* comm, double t_remaining,
                                    orcha_dt_info* info, void* stream) {
  if (!pk || npk < 1 || !info) return fail(ORCHA_E_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<DtRecord> res(npk);
  std::vector<DevStatus> st(npk);
  PhaseScope ph(PH_DT, s);
  {
    int32_t rc = ensure_dt_records(pk, npk, s);
    if (rc) return rc;
  }
  if (npk > 1) {
    // one reduction over every packet's records and status word (the same
    // (max s, lowest g) rule, so the same result as combining per packet)
    DtPlan* dp = nullptr;
    int32_t rc = get_dtplan(pk, npk, &dp);
    if (rc) return rc;
    struct { DtRecord r; DevStatus st; } o;
    cudaError_t e = upload_dt_table(dp, pk, npk, s);
    if (e == cudaSuccess) e = launch_dt_reduce_multi(dp->d_pd, npk, dp->d_out, (DevStatus*)(dp->d_out + 1), s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&o, dp->d_out, sizeof(DtRecord) + sizeof(DevStatus),
                                              cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "dt reduce");
    res.assign(1, o.r);
    st.assign(1, o.st);
    npk = 1;
  } else {
    cudaError_t e = launch_dt_reduce(pk[0]->records, pk[0]->nrecords, pk[0]->result, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&res[0], pk[0]->result, sizeof(DtRecord), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&st[0], pk[0]->status, sizeof(DevStatus), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, "dt reduce");
  }
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "dt sync");
  double smax = res[0].s;
  long long g = res[0].g;
  bool bad = false;
  for (int q = 0; q < npk; q++) {
    if (dt_better(res[q].s, res[q].g, smax, g)) { smax = res[q].s; g = res[q].g; }
    bad |= st[q].first_bad != ~0ull;
  }
  if (comm) {
    PhaseScope phc(PH_DT_COMM, s);
    int32_t rc = comm_allreduce_dt(comm, &smax, &g, &bad, s);
    if (rc) return rc;
  }
  const double cfl = pk[0]->grid->dev.cfl;
  double dt = cfl / smax;
  int32_t tag = ORCHA_DT_CFL;
  if (t_remaining < dt) { dt = t_remaining; tag = ORCHA_DT_CLAMP; }
  info->dt = dt;
  info->smax = smax;
  info->argmax = g;
  info->tag = tag;
  info->nonphysical = bad ? 1 : 0;
  if (bad) return fail(ORCHA_E_NONPHYSICAL, "non-physical state (rho <= 0 or non-finite) in a packet (NonPositiveState)");
  return ORCHA_OK;
}

// This rank's dt record (device GatherRec: max s over its packets' records,
// lowest g, non-physical flag) -- what the allgather carries.
static int32_t rank_record(orcha_packet* const* pk, int32_t npk, cudaStream_t s, GatherRec** out) {
  {
    int32_t rc = ensure_dt_records(pk, npk, s);
    if (rc) return rc;
  }
  const DtRecord* r = nullptr;
  const DevStatus* st = nullptr;
  GatherRec* mine = nullptr;
  cudaError_t e;
  if (npk > 1) {
    DtPlan* dp = nullptr;
    int32_t rc = get_dtplan(pk, npk, &dp);
    if (rc) return rc;
    e = upload_dt_table(dp, pk, npk, s);
    if (e == cudaSuccess) e = launch_dt_reduce_multi(dp->d_pd, npk, dp->d_out, (DevStatus*)(dp->d_out + 1), s);
    if (e != cudaSuccess) return cuda_fail(e, "dt reduce");
    r = dp->d_out;
    st = (const DevStatus*)(dp->d_out + 1);
    mine = dp->d_rec;
  } else {
    e = launch_dt_reduce(pk[0]->records, pk[0]->nrecords, pk[0]->result, s);
    if (e != cudaSuccess) return cuda_fail(e, "dt reduce");
    r = pk[0]->result;
    st = pk[0]->status;
    mine = pk[0]->d_grec;
  }
  e = launch_dt_gather_rec(r, st, mine, s);
  if (e != cudaSuccess) return cuda_fail(e, "dt record");
  *out = mine;
  return ORCHA_OK;
}

extern "C" int32_t orcha_compute_dt_device(orcha_packet* const* pk, int32_t npk, orcha_comm* comm,
                                           orcha_dev_clock* d_clock, void* stream) {
  if (!pk || npk < 1 || !d_clock) return fail(ORCHA_E_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  GatherRec* mine = nullptr;
  PhaseScope ph(PH_DT, s);
  if (!comm && npk == 1) {  // one packet, one rank: reduce, record and finish in one launch
    int32_t rc = ensure_dt_records(pk, npk, s);
    if (rc) return rc;
    cudaError_t e = launch_dt_reduce_finish(pk[0]->records, pk[0]->nrecords, pk[0]->result, pk[0]->status,
                                            pk[0]->d_grec, pk[0]->grid->dev.cfl, d_clock, s);
    if (e != cudaSuccess) return cuda_fail(e, "dt reduce + finish");
    return ORCHA_OK;
  }
  int32_t rc = rank_record(pk, npk, s, &mine);
  if (rc) return rc;
  const GatherRec* all = mine;
  int nall = 1;
  if (comm) {
    PhaseScope phc(PH_DT_COMM, s);
    rc = comm_allgather_dt_device(comm, mine, &all, &nall, s);
    if (rc) return rc;
  }
  cudaError_t e = launch_dt_finish(all, nall, pk[0]->grid->dev.cfl, d_clock, s);
  if (e != cudaSuccess) return cuda_fail(e, "dt finish");
  return ORCHA_OK;
}

extern "C" int32_t orcha_comm_push_dt(orcha_comm* comm, orcha_packet* const* pk, int32_t npk, void* stream) {
  if (!comm || !pk || npk < 1) return fail(ORCHA_E_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  GatherRec* mine = nullptr;
  int32_t rc = rank_record(pk, npk, s, &mine);
  if (rc) return rc;
  return comm_push_dt_record(comm, mine, s);
}

// ----------------------------------------------------------- advance -----
// Borrowed ring: the box and interior stage-1 kernels on two streams
// (ORCHA_HYB_CONC=0: one after the other on the caller's stream).
static bool hyb_concurrent() {
  static const bool on = [] {
    const char* e = getenv("ORCHA_HYB_CONC");
    return !(e && atoi(e) == 0);
  }();
  return on;
}
static cudaError_t hyb_side(orcha_packet* p) {
  if (!hyb_concurrent() || p->side) return cudaSuccess;
  // the side stream (blocks with x / y self sides: the longer CTAs) at the
  // highest stream priority, so their CTAs are dispatched first and the
  // interior kernel's fill the tail (2.204 -> 2.195 ms per cfg4 step,
  // profiles/r02_ab_hybprio.txt; ORCHA_HYB_PRIO=0: default priority)
  static const bool prio = [] {
    const char* e = getenv("ORCHA_HYB_PRIO");
    return !(e && atoi(e) == 0);
  }();
  int lo = 0, hi = 0;
  cudaError_t e = prio ? cudaDeviceGetStreamPriorityRange(&lo, &hi) : cudaSuccess;
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, prio ? hi : 0);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_ready, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_halo, cudaEventDisableTiming);
  return e;
}

// The borrowed-ring tables of packet p's current plan, if its step can use
// them: the gather-mode fill of a one-packet set (x-guard push by stage 2),
// or the full fill (no guard push); not the guard-push mode.
static const HybTables* hyb_tables(const orcha_packet* p, bool xpush, const PushEntry* push) {
  if (ring_mode() != 1 || !p->push_plan || (push && !xpush)) return nullptr;
  const FillPlan* f = p->push_plan;
  const int q = p->plan_q;
  if (q < 0 || (size_t)q >= f->hyb.size() || f->packets[q] != p || !f->hyb[q].d_smap) return nullptr;
  if (xpush && p->d_nbr != f->d_tables[q]) return nullptr;
  return &f->hyb[q];
}

static int32_t advance_impl(orcha_packet* p, const double* d_dt, double h_dt, void* stream) {
  if (!p) return fail(ORCHA_E_ARG, "null packet");
  if (!p->guards_valid || !p->guards_full)
    return fail(ORCHA_E_STATE, "orcha_fill_guardcells must precede every orcha_hydro_advance (guards are stale, "
                               "or only the per-stage fill ran)");
  cudaStream_t s = (cudaStream_t)stream;
  const DevGrid& G = p->grid->dev;
  cudaError_t e;
  const bool fused = kernel_variant() == 1;
  const HybTables* hyb = nullptr;
  if (p->guards_xonly && !fused)
    return fail(ORCHA_E_STATE, "the gather-mode fill was done for the fused kernels; refill after changing the variant");
  const PushEntry* push = (fused && push_enabled() && fused_supported(G) && p->push_plan) ? p->d_push : nullptr;
  // gather mode: stage 2 scatters U^{n+1} into the x-guards (all the next
  // gather-mode fill would write), so that fill launches nothing
  const bool xpush = fused && !push && p->guards_xonly && p->push_plan != nullptr;
  if (xpush) push = p->d_push;
  if (!fused)
    e = launch_advance_ref(G, p->state, p->scratch, p->nslots, p->d_slots, d_dt, h_dt, p->records, &p->nrecords,
                           p->status, s);
  else if (!p->peer_comm && (hyb = hyb_tables(p, xpush, push)) != nullptr &&
           (!hyb_fork(*hyb) || (e = hyb_side(p)) == cudaSuccess))
    e = launch_advance_hybrid(G, p->state, p->scratch, p->nslots, p->d_slots, hyb->d_smap, hyb->nb4, hyb->nint,
                              hyb->d_push, xpush ? p->d_nbr : nullptr, d_dt, h_dt, p->records, &p->nrecords,
                              p->status, s, push, 3,
                              hyb_concurrent() && hyb_fork(*hyb) ? p->side : nullptr, p->ev_ready, p->ev_halo);
  else if (!p->peer_comm)
    e = launch_advance_fused(G, p->state, p->scratch, p->nslots, p->d_slots, d_dt, h_dt, p->records,
                             &p->nrecords, p->status, s, push, p->guards_xonly ? p->d_nbr : nullptr, xpush);
  else {
    // F2 peer mode: stage 2 overwrites U^n in place and pushes x-guards into
    // other ranks' blocks, whose stage 1 reads them: every rank's stage 1
    // ends before any stage 2 starts
    if (!p->guards_xonly || !xpush) return fail(ORCHA_E_STATE, "peer mode: gather-mode fill expected");
    // the borrowed ring too: the other ranks' sides are self sides (their
    // rows are read directly by stage 1), the own packet's borrowed
    hyb = hyb_tables(p, xpush, push);
    if (hyb && hyb_fork(*hyb)) {
      e = hyb_side(p);
      if (e != cudaSuccess) return cuda_fail(e, "side stream");
    }
    auto part = [&](int parts) {
      if (hyb)
        return launch_advance_hybrid(G, p->state, p->scratch, p->nslots, p->d_slots, hyb->d_smap, hyb->nb4,
                                     hyb->nint, hyb->d_push, p->d_nbr, d_dt, h_dt, p->records, &p->nrecords,
                                     p->status, s, push, parts,
                                     hyb_concurrent() && hyb_fork(*hyb) ? p->side : nullptr, p->ev_ready,
                                     p->ev_halo);
      return launch_advance_fused(G, p->state, p->scratch, p->nslots, p->d_slots, d_dt, h_dt, p->records,
                                  &p->nrecords, p->status, s, push, p->d_nbr, xpush, parts);
    };
    e = part(1);
    if (e == cudaSuccess) {
      int32_t rc = comm_peer_barrier(p->peer_comm, s);
      if (rc) return rc;
      e = part(2);
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "advance kernels");
  if (p->nrecords > p->records_cap) return fail(ORCHA_E_LAYOUT, "record capacity exceeded (internal)");
  p->guards_valid = false;
  p->guards_pushed = push != nullptr && !xpush;
  p->xguards_pushed = xpush;
  p->records_valid = true;
  p->stage1_done = false;
  p->u1_guards_valid = false;
  p->u1_pushed = false;
  p->u1_xpushed = p->u1_guards_xonly = false;  // the scratch now holds the telescoped U1
  return ORCHA_OK;
}

extern "C" int32_t orcha_hydro_advance(orcha_packet* p, double dt, void* stream) {
  return advance_impl(p, nullptr, dt, stream);
}
extern "C" int32_t orcha_hydro_advance_devdt(orcha_packet* p, const double* d_dt, void* stream) {
  if (!d_dt) return fail(ORCHA_E_ARG, "null d_dt");
  return advance_impl(p, d_dt, 0.0, stream);
}

// ------------------------------------ interior/boundary overlap (8(e)) ---
// One telescoped step of a rank's single packet with the halo exchange in
// flight while stage 1 runs on the packet's leading interior slots (blocks
// whose 26 neighbours are all resident: they read nothing the exchange
// writes); stage 1 of the remaining slots waits for the exchange, then stage 2
// runs on every slot.  dt is computed first (device clock), as in
// orcha_compute_dt_device.  Falls back to fill -> dt -> advance when there is
// nothing to overlap (no remote source, first step after a pack, a non-brick
// owner map needing the complement pass, no leading interior slot).
static int interior_prefix(const orcha_packet* p, const FillPlan* f) {
  // the table of slot s is f->d_tables[0] + 27 s on the device; recompute on
  // the host from the ids: a slot is interior when every neighbour block is
  // resident in this packet (or the slot itself across a physical boundary)
  const orcha_grid* g = p->grid;
  const DevGrid& G = g->dev;
  std::unordered_map<long long, int> mine;
  for (int s = 0; s < p->nslots; s++) mine[p->ids[s]] = s;
  (void)f;
  int n = 0;
  for (; n < p->nslots; n++) {
    long long b = p->ids[n];
    int bc[3] = {(int)(b % G.nblk[0]), (int)((b / G.nblk[0]) % G.nblk[1]),
                 (int)(b / ((long long)G.nblk[0] * G.nblk[1]))};
    bool ok = true;
    for (int dd = 0; dd < 27 && ok; dd++) {
      int o[3] = {dd % 3 - 1, (dd / 3) % 3 - 1, dd / 9 - 1};
      bool valid = true;
      for (int a = g->desc.ndim; a < 3; a++) valid &= (o[a] == 0);
      if (!valid) continue;
      ok = mine.count(make_entry(g, bc, o).src_block) > 0;
    }
    if (!ok) break;
  }
  return n;
}

extern "C" int32_t orcha_hydro_step_overlap(orcha_packet* p, orcha_comm* comm, orcha_dev_clock* d_clock,
                                            void* stream) {
  if (!p || !comm || !d_clock) return fail(ORCHA_E_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  orcha_packet* pk[1] = {p};
  FillPlan* f = nullptr;
  int32_t rc = get_plan(pk, 1, comm, &f);
  if (rc) return rc;
  const DevGrid& G = p->grid->dev;
  const bool gather = !push_enabled() && fill_mode() == 1 && kernel_variant() == 1 && fused_supported(G);
  const bool steady = p->xguards_pushed && p->push_plan == f;
  const int nint = (f->has_remote && gather && steady && !f->edge_fix[0] && !f->peer) ? interior_prefix(p, f) : 0;
  if (nint == 0) {  // nothing to overlap: the plain sequence
    rc = fill_impl(pk, 1, comm, 0, false, stream);
    if (rc == ORCHA_OK) rc = orcha_compute_dt_device(pk, 1, comm, d_clock, stream);
    if (rc == ORCHA_OK) rc = advance_impl(p, &d_clock->dt, 0.0, stream);
    return rc;
  }
  if (!p->side) {
    cudaError_t e = cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_halo, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "overlap stream");
  }
  CommPlan* cp = nullptr;
  rc = comm_build_plan(comm, pk, 1, 0, &cp);
  if (rc) return rc;
  // dt first (its allgather precedes the exchange on the communicator)
  rc = orcha_compute_dt_device(pk, 1, comm, d_clock, stream);
  if (rc) return rc;
  cudaError_t e = cudaEventRecord(p->ev_ready, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->side, p->ev_ready, 0);
  if (e != cudaSuccess) return cuda_fail(e, "overlap fork");
  {
    PhaseScope phf(PH_FILL, p->side);
    PhaseScope phx(PH_EXCHANGE, p->side);
    rc = comm_exchange(comm, cp, p->side);
  }
  if (rc) return rc;
  e = cudaEventRecord(p->ev_halo, p->side);
  if (e != cudaSuccess) return cuda_fail(e, "overlap join");
  // the fill's bookkeeping (what fill_impl records for a gather-mode fill)
  p->d_push = f->d_push[0];
  p->d_push_u1 = f->d_push_u1[0];
  p->push_plan = f;
  p->plan_q = 0;
  p->guards_valid = true;
  p->guards_xonly = true;
  p->d_nbr = f->d_tables[0];
  p->guards_full = true;
  const double* d_dt = &d_clock->dt;
  const long long c5 = (long long)kNVar * G.cube, u5 = (long long)kNVar * fused_u1_cube(G.nb[0]);
  // stage 1 on the interior slots [0, nint) while the halo is in flight
  e = launch_advance_fused(G, p->state, p->scratch, nint, p->d_slots, d_dt, 0.0, p->records, &p->nrecords,
                           p->status, s, p->d_push, p->d_nbr, true, 1);
  if (e == cudaSuccess && nint < p->nslots) {
    e = cudaStreamWaitEvent(s, p->ev_halo, 0);
    if (e == cudaSuccess)
      e = launch_advance_fused(G, p->state + nint * c5, p->scratch + nint * u5, p->nslots - nint, p->d_slots + nint,
                               d_dt, 0.0, p->records, &p->nrecords, p->status, s, p->d_push, p->d_nbr + 27LL * nint,
                               true, 1);
  } else if (e == cudaSuccess) {
    e = cudaStreamWaitEvent(s, p->ev_halo, 0);
  }
  if (e == cudaSuccess)
    e = launch_advance_fused(G, p->state, p->scratch, p->nslots, p->d_slots, d_dt, 0.0, p->records, &p->nrecords,
                             p->status, s, p->d_push, p->d_nbr, true, 2);
  if (e != cudaSuccess) return cuda_fail(e, "advance kernels (overlap)");
  if (p->nrecords > p->records_cap) return fail(ORCHA_E_LAYOUT, "record capacity exceeded (internal)");
  p->guards_valid = false;
  p->guards_pushed = false;
  p->xguards_pushed = true;
  p->records_valid = true;
  p->stage1_done = false;
  p->u1_guards_valid = false;
  p->u1_pushed = false;
  p->u1_xpushed = p->u1_guards_xonly = false;
  return ORCHA_OK;
}

// ------------------------------------------- per-stage variant (F1) ------
static int32_t stage_impl(orcha_packet* p, int32_t stage, const double* d_dt, double h_dt, void* stream) {
  if (!p) return fail(ORCHA_E_ARG, "null packet");
  if (stage != 1 && stage != 2) return fail(ORCHA_E_ARG, "stage must be 1 or 2");
  if (stage == 1 && !p->guards_valid)
    return fail(ORCHA_E_STATE, "stage 1 needs a guard fill of the state since the last pack/advance");
  if (stage == 2 && !(p->stage1_done && p->u1_guards_valid))
    return fail(ORCHA_E_STATE, "stage 2 needs stage 1 and a guard refill of the stage-1 buffer (buffer 1)");
  cudaStream_t s = (cudaStream_t)stream;
  const DevGrid& G = p->grid->dev;
  cudaError_t e;
  const bool fused = kernel_variant() == 1;
  if (stage == 1 && p->guards_xonly && !fused)
    return fail(ORCHA_E_STATE, "the gather-mode fill was done for the fused kernels; refill after changing the variant");
  if (stage == 2 && p->u1_guards_xonly && !fused)
    return fail(ORCHA_E_STATE, "the gather-mode refill was done for the fused kernels; refill after changing the variant");
  const PushEntry* push = nullptr;
  if (fused && push_enabled() && fused_supported(G) && p->push_plan) push = (stage == 1) ? p->d_push_u1 : p->d_push;
  // gather mode: each stage also writes the x-guards the next gather-mode
  // step reads (stage 1: U1's, stage 2: the state's), so no fill kernel runs
  const bool xpush = fused && !push && p->guards_xonly && p->push_plan != nullptr && fused_supported(G);
  if (xpush) push = (stage == 1) ? p->d_push_u1 : p->d_push;
  const NbrEntry* nbr = (stage == 1) ? (p->guards_xonly ? p->d_nbr : nullptr)
                                     : (p->u1_guards_xonly ? p->d_nbr_u1 : nullptr);
  if (!fused)
    e = launch_stage_ref(G, stage, p->state, p->scratch, p->nslots, p->d_slots, d_dt, h_dt, p->records,
                         &p->nrecords, p->status, s);
  else
    e = launch_stage_fused(G, stage, p->state, p->scratch, p->nslots, p->d_slots, d_dt, h_dt, p->records,
                           &p->nrecords, p->status, s, push, nbr, xpush);
  if (e != cudaSuccess) return cuda_fail(e, "stage kernels");
  if (p->nrecords > p->records_cap) return fail(ORCHA_E_LAYOUT, "record capacity exceeded (internal)");
  if (stage == 1) {
    p->stage1_done = true;
    p->u1_guards_valid = false;
    p->u1_guards_xonly = false;
    p->u1_pushed = push != nullptr && !xpush;
    p->u1_xpushed = xpush;
  } else {
    p->stage1_done = false;
    p->u1_guards_valid = false;
    p->u1_guards_xonly = false;
    p->u1_pushed = false;
    p->u1_xpushed = false;
    p->guards_valid = false;
    p->guards_pushed = push != nullptr && !xpush;
    p->xguards_pushed = xpush;
    p->records_valid = true;
  }
  return ORCHA_OK;
}

extern "C" int32_t orcha_hydro_stage(orcha_packet* p, int32_t stage, double dt, void* stream) {
  return stage_impl(p, stage, nullptr, dt, stream);
}
extern "C" int32_t orcha_hydro_stage_devdt(orcha_packet* p, int32_t stage, const double* d_dt, void* stream) {
  if (!d_dt) return fail(ORCHA_E_ARG, "null d_dt");
  return stage_impl(p, stage, d_dt, 0.0, stream);
}
