// comm.cu -- multi-GPU plumbing of liborcha.so: the cross-rank guard exchange
// and the global dt reduction.
//
// "The Hydro computation can have either 1 or 2 MPI operations interspersed
// with local node computations" (sec 6); "Milhoja only handles
// computations that do not involve any MPI operations".  Here each
// step has exactly two communication operations, both outside
// orcha_hydro_advance:
//   1. the guard exchange inside orcha_fill_guardcells: every rank gathers
//      the unique interior cells a peer's guards read (sorted by global cell
//      index g, a pure function of the grid and the block->rank map, so both
//      sides agree on the order without negotiating), one grouped
//      ncclSend/ncclRecv per neighbour rank, then a scatter of the received
//      values into the guards (with the reflect sign flips);
//   2. an ncclAllGather of each rank's (s_max, argmax, non-physical) record
//      inside orcha_compute_dt, reduced on the host with the same
//      deterministic (max s, lowest g) rule as the single-GPU path.
// NCCL is dlopen'ed (the libnccl.so.2 torch already loaded into the process),
// so liborcha.so has no link-time NCCL dependency.  A LOCAL transport (virtual
// ranks on one device, device-to-device copies) runs the same plan, pack and
// unpack kernels without NCCL for tests.
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "comm.h"
#include "orcha_internal.h"

namespace orcha {

// ------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { api.err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror(); return; }
    bool good = true;
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) good = false;
      return p;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.ok = good;
    if (!good) api.err = "libnccl.so.2 lacks an expected symbol";
  });
  return api;
}

static int32_t nccl_fail(ncclResult_t r, const char* what) {
  return fail(ORCHA_E_NCCL, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

// ------------------------------------------------------- host exchange plan
// One remote guard: destination (block id, padded cell offset), source global
// cell g, flip bits (bit 1+d = negate variable 1+d).
struct RemoteGuard {
  long long dst_block;
  long long dst_cell;  // padded cell offset in the block cube
  long long src_g;     // global cell index of the source
  long long src_block;
  long long src_cell;  // padded cell offset of the source in its block cube
  int flip;
};

// Enumerate the guards of blocks owned by `R` whose source block is owned by
// `S` (same per-axis shift / clamp / mirror images as the local fill).
static void enumerate_remote(const orcha_grid* g, const int32_t* owner, int R, int S,
                             std::vector<RemoteGuard>& out) {
  const DevGrid& G = g->dev;
  const int nd = g->desc.ndim;
  for (long long b = 0; b < g->nblocks; b++) {
    if (owner[b] != R) continue;
    int bc[3] = {(int)(b % G.nblk[0]), (int)((b / G.nblk[0]) % G.nblk[1]),
                 (int)(b / ((long long)G.nblk[0] * G.nblk[1]))};
    for (int oz = -1; oz <= 1; oz++)
      for (int oy = -1; oy <= 1; oy++)
        for (int ox = -1; ox <= 1; ox++) {
          int o[3] = {ox, oy, oz};
          if (ox == 0 && oy == 0 && oz == 0) continue;
          bool valid = true;
          for (int a = nd; a < 3; a++) valid &= (o[a] == 0);
          if (!valid) continue;
          // source block and per-axis modes (as make_entry in runtime.cu)
          int src[3], mode[3], flip = 0;
          for (int a = 0; a < 3; a++) {
            int c = bc[a] + o[a];
            mode[a] = kShift;
            if (o[a] != 0 && (c < 0 || c >= G.nblk[a])) {
              int code = g->desc.bc[a][o[a] < 0 ? 0 : 1];
              if (code == ORCHA_BC_PERIODIC) c = (c + G.nblk[a]) % G.nblk[a];
              else if (code == ORCHA_BC_OUTFLOW) { c = bc[a]; mode[a] = kClamp; }
              else { c = bc[a]; mode[a] = kMirror; flip |= 1 << (1 + a); }
            }
            src[a] = c;
          }
          long long sb = ((long long)src[2] * G.nblk[1] + src[1]) * G.nblk[0] + src[0];
          if (owner[sb] != S) continue;
          // guard cells of this direction
          int lo[3], hi[3];
          for (int a = 0; a < 3; a++) {
            if (o[a] < 0) { lo[a] = -G.gd[a]; hi[a] = 0; }
            else if (o[a] > 0) { lo[a] = G.nb[a]; hi[a] = G.nb[a] + G.gd[a]; }
            else { lo[a] = 0; hi[a] = G.nb[a]; }
          }
          for (int k = lo[2]; k < hi[2]; k++)
            for (int j = lo[1]; j < hi[1]; j++)
              for (int i = lo[0]; i < hi[0]; i++) {
                int l[3] = {i, j, k}, s[3];
                for (int a = 0; a < 3; a++) {
                  int n = G.nb[a];
                  if (o[a] == 0) s[a] = l[a];
                  else if (mode[a] == kShift) s[a] = l[a] - o[a] * n;
                  else if (mode[a] == kClamp) s[a] = (o[a] < 0) ? 0 : n - 1;
                  else s[a] = (o[a] < 0) ? -1 - l[a] : 2 * n - 1 - l[a];
                }
                RemoteGuard r;
                r.dst_block = b;
                r.dst_cell = ((long long)(k + G.gd[2]) * G.P[1] + (j + G.gd[1])) * G.P[0] + (i + G.gd[0]);
                long long gx = (long long)src[0] * G.nb[0] + s[0];
                long long gy = (long long)src[1] * G.nb[1] + s[1];
                long long gz = (long long)src[2] * G.nb[2] + s[2];
                r.src_g = (gz * G.N[1] + gy) * G.N[0] + gx;
                r.src_block = sb;
                r.src_cell = ((long long)(s[2] + G.gd[2]) * G.P[1] + (s[1] + G.gd[1])) * G.P[0] + (s[0] + G.gd[0]);
                r.flip = flip;
                out.push_back(r);
              }
        }
  }
}

// Exchange lists between `me` and `peer` (host only).
struct PeerLists {
  int peer;
  std::vector<long long> send_g, send_block, send_cell;  // sorted unique by g: what I send to peer
  std::vector<long long> recv_g;                         // sorted unique: what I receive from peer
  std::vector<RemoteGuard> guards;                       // my guards sourced by peer
  std::vector<long long> guard_idx;                      // index into recv_g per guard
};

static void unique_sorted(std::vector<RemoteGuard>& v, std::vector<long long>& g, std::vector<long long>* blk,
                          std::vector<long long>* cell) {
  std::vector<const RemoteGuard*> p;
  p.reserve(v.size());
  for (auto& r : v) p.push_back(&r);
  std::sort(p.begin(), p.end(), [](const RemoteGuard* a, const RemoteGuard* b) { return a->src_g < b->src_g; });
  for (auto* r : p) {
    if (!g.empty() && g.back() == r->src_g) continue;
    g.push_back(r->src_g);
    if (blk) blk->push_back(r->src_block);
    if (cell) cell->push_back(r->src_cell);
  }
}

static PeerLists make_lists(const orcha_grid* g, const int32_t* owner, int me, int peer) {
  PeerLists L;
  L.peer = peer;
  std::vector<RemoteGuard> out;
  enumerate_remote(g, owner, peer, me, out);  // peer's guards that read my cells
  unique_sorted(out, L.send_g, &L.send_block, &L.send_cell);
  enumerate_remote(g, owner, me, peer, L.guards);  // my guards that read peer's cells
  std::vector<RemoteGuard> tmp = L.guards;
  unique_sorted(tmp, L.recv_g, nullptr, nullptr);
  L.guard_idx.resize(L.guards.size());
  for (size_t i = 0; i < L.guards.size(); i++)
    L.guard_idx[i] = std::lower_bound(L.recv_g.begin(), L.recv_g.end(), L.guards[i].src_g) - L.recv_g.begin();
  return L;
}

// ----------------------------------------------------------- device side ---
struct UnpackEntry {
  double* dst;          // var-0 address of the guard cell
  const double* src;    // var-0 address in the receive buffer (var stride = n of that peer)
  long long vstride;    // receive-buffer variable stride (= n unique cells of that peer)
  int flip;
  int pad;
};

__global__ void halo_pack_kernel(const double* const* __restrict__ src, long long n, long long cube,
                                 double* __restrict__ buf) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* s = src[i];
#pragma unroll
  for (int v = 0; v < kNVar; v++) buf[v * n + i] = s[v * cube];
}

__global__ void halo_unpack_kernel(const UnpackEntry* __restrict__ e, long long n, long long cube) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  UnpackEntry u = e[i];
#pragma unroll
  for (int v = 0; v < kNVar; v++) {
    double x = u.src[v * u.vstride];
    if ((u.flip >> v) & 1) x = -x;
    u.dst[v * cube] = x;
  }
}

struct PeerBuf {
  int peer;
  long long n_send, n_recv;
  double* d_send = nullptr;  // [5][n_send]
  double* d_recv = nullptr;  // [5][n_recv]
};

struct CommPlan {
  std::vector<orcha_packet*> packets;
  int buffer = 0;
  std::vector<const double**> d_send_src;  // per peer (device array of n_send pointers)
  UnpackEntry* d_unpack = nullptr;
  long long n_unpack = 0;
};

// Virtual ranks sharing one device: members[r] is virtual rank r (nullptr
// once destroyed; the hub goes when every slot is empty).
struct Hub {
  std::vector<orcha_comm*> members;
  std::vector<orcha_packet*> peer_packet;       // F2 peer mode: each virtual rank's registered packet
  unsigned long long* d_ctr = nullptr;          // F2 peer mode: one barrier counter per virtual rank
  bool empty() const {
    for (auto* m : members)
      if (m) return false;
    return true;
  }
};

}  // namespace orcha

struct orcha_comm {
  const orcha_grid* grid;
  int nranks, rank;
  std::vector<int32_t> owner;
  bool local;
  ncclComm_t nc = nullptr;
  orcha::Hub* hub = nullptr;
  std::vector<orcha::PeerLists> lists;   // peers with any traffic
  std::vector<orcha::PeerBuf> bufs;      // same order as lists
  std::vector<orcha::CommPlan*> plans;
  void* d_gather = nullptr;              // allgather buffer: nranks * 32 B (+ 32 B send)
  // F2 peer mode: peers' packets addressed directly
  bool peer_mode = false;
  unsigned long long** d_ctr_ptrs = nullptr;  // device array: every rank's barrier counter
  unsigned long long bar_epoch = 0;           // barriers this rank has entered
  int* d_err = nullptr;                       // device flag: a peer barrier timed out
  std::vector<void*> peer_gather;             // every rank's dt gather buffer (index = rank)
  // F2 peer mode across processes (CUDA IPC; orcha_comm_create_ipc)
  bool ipc = false;
  unsigned long long* d_my_ctr = nullptr;     // this rank's barrier counter (exported)
  orcha_packet* own_packet = nullptr;         // the packet this rank exported
  std::vector<void*> ipc_mapped;              // opened peer allocations (closed on destroy)
  std::vector<orcha_packet*> shadow;          // other ranks' packets: their mapped state + ids (owned)
};

namespace orcha {

static std::mutex g_comm_mu;
static std::vector<orcha_comm*> g_comms;

static int32_t setup_lists(orcha_comm* c) {
  for (int q = 0; q < c->nranks; q++) {
    if (q == c->rank) continue;
    PeerLists L = make_lists(c->grid, c->owner.data(), c->rank, q);
    if (L.send_g.empty() && L.recv_g.empty()) continue;
    PeerBuf B;
    B.peer = q;
    B.n_send = (long long)L.send_g.size();
    B.n_recv = (long long)L.recv_g.size();
    cudaError_t e = cudaSuccess;
    if (B.n_send) e = cudaMalloc(&B.d_send, sizeof(double) * 5 * B.n_send);
    if (e == cudaSuccess && B.n_recv) e = cudaMalloc(&B.d_recv, sizeof(double) * 5 * B.n_recv);
    if (e != cudaSuccess) return cuda_fail(e, "allocate halo buffers");
    c->lists.push_back(std::move(L));
    c->bufs.push_back(B);
  }
  cudaError_t e = cudaMalloc(&c->d_gather, 32 * (size_t)(c->nranks + 1));
  if (e != cudaSuccess) return cuda_fail(e, "allocate dt gather buffer");
  return ORCHA_OK;
}

static int32_t validate_owner(const orcha_grid* g, int nranks, const int32_t* owner) {
  if (!g || !owner || nranks < 1) return fail(ORCHA_E_ARG, "null grid/owner or nranks < 1");
  for (long long b = 0; b < g->nblocks; b++)
    if (owner[b] < 0 || owner[b] >= nranks) return fail(ORCHA_E_RANGE, "block_owner entry out of [0, nranks)");
  return ORCHA_OK;
}

int32_t comm_build_plan(orcha_comm* c, orcha_packet* const* pk, int npk, int buffer, CommPlan** out) {
  for (auto* p : c->plans) {
    if ((int)p->packets.size() != npk || p->buffer != buffer) continue;
    bool same = true;
    for (int q = 0; q < npk; q++) same &= p->packets[q] == pk[q];
    if (same) { *out = p; return ORCHA_OK; }
  }
  const DevGrid& G = c->grid->dev;
  std::unordered_map<long long, std::pair<int, int>> where;
  for (int q = 0; q < npk; q++)
    for (int s = 0; s < pk[q]->nslots; s++) where[pk[q]->ids[s]] = {q, s};
  // buffer 0: the packet state; 1: the stage-1 buffer (scratch, same padded layout)
  auto addr = [&](long long block, long long cell, double** a) -> bool {
    auto it = where.find(block);
    if (it == where.end()) return false;
    orcha_packet* p = pk[it->second.first];
    *a = (buffer ? p->scratch : p->state) + (long long)it->second.second * kNVar * G.cube + cell;
    return true;
  };
  CommPlan* P = new CommPlan();
  P->packets.assign(pk, pk + npk);
  P->buffer = buffer;
  std::vector<UnpackEntry> un;
  for (size_t i = 0; i < c->lists.size(); i++) {
    const PeerLists& L = c->lists[i];
    std::vector<const double*> src(L.send_g.size());
    for (size_t k = 0; k < src.size(); k++) {
      double* a;
      if (!addr(L.send_block[k], L.send_cell[k], &a)) {
        delete P;
        return fail(ORCHA_E_RANGE, "a block this rank owns is not in the packets passed to the exchange");
      }
      src[k] = a;
    }
    const double** d = nullptr;
    if (!src.empty()) {
      cudaError_t e = cudaMalloc(&d, sizeof(double*) * src.size());
      if (e == cudaSuccess) e = cudaMemcpy(d, src.data(), sizeof(double*) * src.size(), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) { delete P; return cuda_fail(e, "upload halo send table"); }
    }
    P->d_send_src.push_back(d);
    for (size_t k = 0; k < L.guards.size(); k++) {
      UnpackEntry u;
      double* a;
      if (!addr(L.guards[k].dst_block, L.guards[k].dst_cell, &a)) {
        delete P;
        return fail(ORCHA_E_RANGE, "a block this rank owns is not in the packets passed to the exchange");
      }
      u.dst = a;
      u.src = c->bufs[i].d_recv + L.guard_idx[k];
      u.vstride = c->bufs[i].n_recv;
      u.flip = L.guards[k].flip;
      u.pad = 0;
      un.push_back(u);
    }
  }
  P->n_unpack = (long long)un.size();
  if (!un.empty()) {
    cudaError_t e = cudaMalloc(&P->d_unpack, sizeof(UnpackEntry) * un.size());
    if (e == cudaSuccess) e = cudaMemcpy(P->d_unpack, un.data(), sizeof(UnpackEntry) * un.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { delete P; return cuda_fail(e, "upload halo unpack table"); }
  }
  c->plans.push_back(P);
  *out = P;
  return ORCHA_OK;
}

void comm_free_plan(CommPlan*) {}  // plans are owned (and freed) by their communicator

static void free_plan(CommPlan* P) {
  for (auto* d : P->d_send_src) cudaFree((void*)d);
  cudaFree(P->d_unpack);
  delete P;
}

void comm_drop_packet(orcha_packet* p) {
  std::lock_guard<std::mutex> lk(g_comm_mu);
  for (auto* c : g_comms) {
    if (c->hub)
      for (auto*& q : c->hub->peer_packet)
        if (q == p) q = nullptr;  // peer mode: the rank must register a packet again
    if (c->own_packet == p) c->own_packet = nullptr;
  }
  for (auto* c : g_comms)
    for (size_t i = 0; i < c->plans.size();) {
      bool hit = false;
      for (auto* q : c->plans[i]->packets) hit |= q == p;
      if (hit) { free_plan(c->plans[i]); c->plans.erase(c->plans.begin() + i); }
      else i++;
    }
}

// Pack this rank's sources for every peer into `dst_of(i)` (own send buffer,
// or -- LOCAL transport -- the peer's receive buffer for this rank).
static int32_t pack_all(orcha_comm* c, CommPlan* P, bool into_peers, cudaStream_t s) {
  const long long cube = c->grid->dev.cube;
  for (size_t i = 0; i < c->bufs.size(); i++) {
    long long n = c->bufs[i].n_send;
    if (!n) continue;
    double* dst = c->bufs[i].d_send;
    if (into_peers) {
      orcha_comm* peer = c->hub->members[c->bufs[i].peer];
      if (!peer) return fail(ORCHA_E_STATE, "LOCAL peer rank was destroyed");
      dst = nullptr;
      for (auto& b : peer->bufs)
        if (b.peer == c->rank) dst = b.d_recv;
      if (!dst) return fail(ORCHA_E_ARG, "LOCAL peer has no receive buffer for this rank (plan mismatch)");
    }
    halo_pack_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P->d_send_src[i], n, cube, dst);
    count_launch();
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ORCHA_OK : cuda_fail(e, "halo pack");
}

static int32_t unpack_all(orcha_comm* c, CommPlan* P, cudaStream_t s) {
  if (!P->n_unpack) return ORCHA_OK;
  halo_unpack_kernel<<<(unsigned)((P->n_unpack + 255) / 256), 256, 0, s>>>(P->d_unpack, P->n_unpack,
                                                                           c->grid->dev.cube);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ORCHA_OK : cuda_fail(e, "halo unpack");
}

int32_t comm_exchange(orcha_comm* c, CommPlan* P, cudaStream_t s) {
  if (c->local) return unpack_all(c, P, s);  // peers pushed already (orcha_comm_push)
  int32_t rc = pack_all(c, P, false, s);
  if (rc) return rc;
  NcclApi& A = nccl();
  ncclResult_t r = A.GroupStart();
  for (auto& b : c->bufs) {
    if (r == ncclSuccess && b.n_send) r = A.Send(b.d_send, 5 * (size_t)b.n_send, ncclFloat64, b.peer, c->nc, s);
    if (r == ncclSuccess && b.n_recv) r = A.Recv(b.d_recv, 5 * (size_t)b.n_recv, ncclFloat64, b.peer, c->nc, s);
  }
  ncclResult_t r2 = A.GroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "halo send/recv");
  if (r2 != ncclSuccess) return nccl_fail(r2, "halo group end");
  return unpack_all(c, P, s);
}

// The allgather of the 32-byte per-rank records into d_gather + 32 (slot r
// = rank r), from this rank's record at `mine` (device).  NCCL: one
// ncclAllGather.  LOCAL: every virtual rank pushed its record into every
// member's slot beforehand (orcha_comm_push_dt); only the own slot is
// (re)written here -- the same array the NCCL path produces.
static int32_t gather_records(orcha_comm* c, const void* mine, cudaStream_t s) {
  char* base = (char*)c->d_gather;
  cudaError_t e = cudaSuccess;
  if (mine != base) e = cudaMemcpyAsync(base, mine, 32, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "dt record copy");
  if (c->peer_mode) {
    // F2: one-shot P2P -- this rank's record into slot `rank` of every rank's
    // gather buffer, then a device barrier: every slot is then filled
    for (int q = 0; q < c->nranks; q++) {
      void* g = (q < (int)c->peer_gather.size()) ? c->peer_gather[q] : nullptr;
      if (c->hub && (!c->hub->members[q])) g = nullptr;
      if (!g) return fail(ORCHA_E_STATE, "peer mode: rank " + std::to_string(q) + " is gone");
      e = cudaMemcpyAsync((char*)g + 32 + 32 * (size_t)c->rank, base, 32, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return cuda_fail(e, "dt record push (peer mode)");
    }
    return comm_peer_barrier(c, s);
  }
  if (c->local) {
    e = cudaMemcpyAsync(base + 32 + 32 * (size_t)c->rank, base, 32, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "dt record copy (LOCAL)");
    return ORCHA_OK;
  }
  ncclResult_t r = nccl().AllGather(base, base + 32, 32, ncclUint8, c->nc, s);
  if (r != ncclSuccess) return nccl_fail(r, "dt allgather");
  return ORCHA_OK;
}

// Host-result dt: this rank's (smax, g, bad) -> the global one by the
// single-GPU rule (max s, ties -> lowest g, NaN wins) over all ranks' records.
int32_t comm_allreduce_dt(orcha_comm* c, double* smax, long long* g, bool* bad, cudaStream_t s) {
  if (c->nranks == 1 && !c->local) return ORCHA_OK;
  GatherRec mine{*smax, *g, *bad ? 1 : 0, 0};
  char* base = (char*)c->d_gather;
  cudaError_t e = cudaMemcpyAsync(base, &mine, sizeof mine, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "dt gather upload");
  int32_t rc = gather_records(c, base, s);
  if (rc) return rc;
  std::vector<GatherRec> all(c->nranks);
  e = cudaMemcpyAsync(all.data(), base + 32, 32 * (size_t)c->nranks, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "dt gather download");
  double sm = all[0].s;
  long long gm = all[0].g;
  bool b = false;
  for (auto& x : all) {
    if (dt_better(x.s, x.g, sm, gm)) { sm = x.s; gm = x.g; }
    b |= x.bad != 0;
  }
  *smax = sm;
  *g = gm;
  *bad = b;
  return ORCHA_OK;
}

// Device-resident variant: this rank's record (device, 32 B) allgathered into
// the communicator's buffer, no host round trip; returns the gathered array.
int32_t comm_allgather_dt_device(orcha_comm* c, const GatherRec* mine, const GatherRec** all, int* nall,
                                 cudaStream_t s) {
  char* base = (char*)c->d_gather;
  if (c->nranks == 1 && !c->local) {
    cudaError_t e = cudaMemcpyAsync(base, mine, 32, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "dt record copy");
    *all = (const GatherRec*)base;
    *nall = 1;
    return ORCHA_OK;
  }
  int32_t rc = gather_records(c, mine, s);
  if (rc) return rc;
  *all = (const GatherRec*)(base + 32);
  *nall = c->nranks;
  return ORCHA_OK;
}

// LOCAL transport: this virtual rank's record (device) into slot `rank` of
// every live member's gather buffer (the allgather, emulated by pushes).
int32_t comm_push_dt_record(orcha_comm* c, const GatherRec* mine, cudaStream_t s) {
  if (!c->local) return fail(ORCHA_E_ARG, "orcha_comm_push_dt is for LOCAL communicators only");
  for (auto* m : c->hub->members) {
    if (!m) continue;
    cudaError_t e = cudaMemcpyAsync((char*)m->d_gather + 32 + 32 * (size_t)c->rank, mine, 32,
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "dt record push");
  }
  return ORCHA_OK;
}

// ------------------------------------------------------ F2 peer mode ------
// Device-side barrier over the ranks of a peer-mode communicator: every rank
// adds 1 to every rank's counter (system-scope atomics: the counters live in
// the ranks' own memory, reached by P2P), then waits until its own counter
// reaches epoch * nranks.  Counters only grow, so no reset is needed.  A wait
// longer than ~10 s (a rank that never arrives) sets the error flag and
// returns instead of hanging the device.
__global__ void peer_barrier_kernel(unsigned long long* const* ctr, int nranks, int me, unsigned long long target,
                                    int* err, long long timeout_cycles) {
  __threadfence_system();
  for (int q = 0; q < nranks; q++) atomicAdd_system(ctr[q], 1ull);
  const long long t0 = clock64();
  while (true) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr[me]) : "memory");
    if (v >= target) break;
    if (clock64() - t0 > timeout_cycles) {
      atomicExch(err, 1);
      break;
    }
    __nanosleep(200);
  }
  __threadfence_system();
}

int32_t comm_peer_barrier(orcha_comm* c, cudaStream_t s) {
  if (!c->peer_mode || !c->d_ctr_ptrs) return fail(ORCHA_E_STATE, "peer barrier outside peer mode");
  c->bar_epoch++;
  // timeout: ~10 s at ~2 GHz; ORCHA_PEER_TIMEOUT_MS overrides (tests)
  static const long long timeout = [] {
    const char* e = getenv("ORCHA_PEER_TIMEOUT_MS");
    return e ? (long long)atoll(e) * 2000000LL : 20000000000LL;
  }();
  peer_barrier_kernel<<<1, 1, 0, s>>>(c->d_ctr_ptrs, c->nranks, c->rank, c->bar_epoch * (unsigned long long)c->nranks,
                                      c->d_err, timeout);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ORCHA_OK : cuda_fail(e, "peer barrier");
}

bool comm_peer_mode(const orcha_comm* c) { return c && c->peer_mode; }
int comm_rank(const orcha_comm* c) { return c->rank; }

// Every other rank's registered packet (peer mode); ORCHA_E_STATE until all
// ranks have registered.
int32_t comm_peer_packets(const orcha_comm* c, std::vector<orcha_packet*>* out) {
  out->clear();
  if (!c->peer_mode) return fail(ORCHA_E_STATE, "not in peer mode");
  if (c->ipc) {
    *out = c->shadow;
    return ORCHA_OK;
  }
  for (int q = 0; q < c->nranks; q++) {
    orcha_packet* p = c->hub->peer_packet[q];
    if (!p) return fail(ORCHA_E_STATE, "peer mode: rank " + std::to_string(q) + " has not registered its packet");
    if (q != c->rank) out->push_back(p);
  }
  return ORCHA_OK;
}

static void destroy_comm(orcha_comm* c) {
  for (void* p : c->ipc_mapped) cudaIpcCloseMemHandle(p);
  for (auto* p : c->shadow) delete p;
  cudaFree(c->d_my_ctr);
  for (auto* p : c->plans) free_plan(p);
  for (auto& b : c->bufs) { cudaFree(b.d_send); cudaFree(b.d_recv); }
  cudaFree(c->d_gather);
  cudaFree(c->d_ctr_ptrs);
  cudaFree(c->d_err);
  if (c->nc && nccl().ok) nccl().CommDestroy(c->nc);
  delete c;
}

}  // namespace orcha

using namespace orcha;

extern "C" int32_t orcha_comm_unique_id(void* id) {
  if (!id) return fail(ORCHA_E_ARG, "null id buffer");
  NcclApi& A = nccl();
  if (!A.ok) return fail(ORCHA_E_NCCL, A.err);
  ncclUniqueId u;
  ncclResult_t r = A.GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id, &u, 128);
  return ORCHA_OK;
}

extern "C" int32_t orcha_comm_create(const orcha_grid* g, const void* id, int32_t nranks, int32_t rank,
                                     const int32_t* owner, orcha_comm** out) {
  if (!out || !id) return fail(ORCHA_E_ARG, "null argument");
  *out = nullptr;
  int32_t rc = validate_owner(g, nranks, owner);
  if (rc) return rc;
  if (rank < 0 || rank >= nranks) return fail(ORCHA_E_ARG, "rank out of range");
  NcclApi& A = nccl();
  if (!A.ok) return fail(ORCHA_E_NCCL, A.err);
  orcha_comm* c = new orcha_comm();
  c->grid = g;
  c->nranks = nranks;
  c->rank = rank;
  c->owner.assign(owner, owner + g->nblocks);
  c->local = false;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclResult_t r = A.CommInitRank(&c->nc, nranks, u, rank);
  if (r != ncclSuccess) { delete c; return nccl_fail(r, "ncclCommInitRank"); }
  rc = setup_lists(c);
  if (rc) { destroy_comm(c); return rc; }
  std::lock_guard<std::mutex> lk(g_comm_mu);
  g_comms.push_back(c);
  *out = c;
  return ORCHA_OK;
}

extern "C" int32_t orcha_comm_create_local(const orcha_grid* g, int32_t nranks, const int32_t* owner,
                                           orcha_comm** out) {
  if (!out) return fail(ORCHA_E_ARG, "null argument");
  int32_t rc = validate_owner(g, nranks, owner);
  if (rc) return rc;
  Hub* hub = new Hub();
  hub->members.assign(nranks, nullptr);
  for (int r = 0; r < nranks; r++) {
    orcha_comm* c = new orcha_comm();
    c->grid = g;
    c->nranks = nranks;
    c->rank = r;
    c->owner.assign(owner, owner + g->nblocks);
    c->local = true;
    c->hub = hub;
    rc = setup_lists(c);
    if (rc) {
      destroy_comm(c);
      for (auto* m : hub->members)
        if (m) destroy_comm(m);
      delete hub;
      return rc;
    }
    hub->members[r] = c;
  }
  std::lock_guard<std::mutex> lk(g_comm_mu);
  for (int r = 0; r < nranks; r++) {
    out[r] = hub->members[r];
    g_comms.push_back(out[r]);
  }
  return ORCHA_OK;
}

extern "C" int32_t orcha_comm_push(orcha_comm* c, orcha_packet* const* pk, int32_t npk, int32_t buffer,
                                   void* stream) {
  if (!c || !pk || npk < 1) return fail(ORCHA_E_ARG, "null argument");
  if (!c->local) return fail(ORCHA_E_ARG, "orcha_comm_push is for LOCAL communicators only");
  if (buffer != 0 && buffer != 1) return fail(ORCHA_E_ARG, "buffer must be 0 or 1");
  CommPlan* P = nullptr;
  int32_t rc = comm_build_plan(c, pk, npk, buffer, &P);
  if (rc) return rc;
  return pack_all(c, P, true, (cudaStream_t)stream);
}

extern "C" int32_t orcha_comm_destroy(orcha_comm* c) {
  if (!c) return ORCHA_OK;
  if (c->peer_mode) runtime_drop_comm(c);
  std::lock_guard<std::mutex> lk(g_comm_mu);
  g_comms.erase(std::remove(g_comms.begin(), g_comms.end(), c), g_comms.end());
  Hub* hub = c->hub;
  if (hub) {
    // the slot stays (members are indexed by rank); pushes to it now fail
    for (auto*& m : hub->members)
      if (m == c) m = nullptr;
    if (hub->empty()) {
      cudaFree(hub->d_ctr);
      delete hub;
    }
  }
  destroy_comm(c);
  return ORCHA_OK;
}

extern "C" int32_t orcha_comm_plan(const orcha_grid* g, int32_t nranks, int32_t rank, const int32_t* owner,
                                   int32_t peer, int32_t which, int64_t* out, int64_t cap, int64_t* count) {
  int32_t rc = validate_owner(g, nranks, owner);
  if (rc) return rc;
  if (rank < 0 || rank >= nranks || peer < 0 || peer >= nranks || peer == rank || which < 0 || which > 4 || !count)
    return fail(ORCHA_E_ARG, "bad rank/peer/which");
  PeerLists L = make_lists(g, owner, rank, peer);
  const DevGrid& G = g->dev;
  long long P3 = (long long)G.P[0] * G.P[1] * G.P[2];
  std::vector<long long> v;
  if (which == 0) v = L.send_g;
  else if (which == 1) v = L.recv_g;
  else
    for (size_t i = 0; i < L.guards.size(); i++)
      v.push_back(which == 2 ? L.guards[i].dst_block * P3 + L.guards[i].dst_cell
                  : which == 3 ? L.guard_idx[i] : (long long)L.guards[i].flip);
  *count = (int64_t)v.size();
  if (out)
    for (long long i = 0; i < (long long)v.size() && i < cap; i++) out[i] = v[i];
  return ORCHA_OK;
}

extern "C" int32_t orcha_comm_peer_register(orcha_comm* c, orcha_packet* p, void* stream) {
  (void)stream;
  if (!c || !p) return fail(ORCHA_E_ARG, "null argument");
  if (!c->local)
    return fail(ORCHA_E_ARG, "orcha_comm_peer_register: peer mode needs the ranks' packets addressable from this "
                             "process (LOCAL virtual ranks); NCCL communicators use the exchange");
  if (p->grid != c->grid) return fail(ORCHA_E_ARG, "packet of another grid");
  for (long long b : p->ids)
    if (c->owner[b] != c->rank) return fail(ORCHA_E_RANGE, "packet holds a block this rank does not own");
  long long owned = 0;
  for (long long b = 0; b < c->grid->nblocks; b++) owned += c->owner[b] == c->rank;
  if ((long long)p->ids.size() != owned)
    return fail(ORCHA_E_ARG, "peer mode needs ONE packet per rank holding every block the rank owns");
  Hub* hub = c->hub;
  std::lock_guard<std::mutex> lk(g_comm_mu);
  if (hub->peer_packet.empty()) hub->peer_packet.assign(hub->members.size(), nullptr);
  if (!hub->d_ctr) {
    cudaError_t e = cudaMalloc(&hub->d_ctr, sizeof(unsigned long long) * hub->members.size());
    if (e == cudaSuccess) e = cudaMemset(hub->d_ctr, 0, sizeof(unsigned long long) * hub->members.size());
    if (e != cudaSuccess) return cuda_fail(e, "allocate peer barrier counters");
  }
  if (!c->d_ctr_ptrs) {
    std::vector<unsigned long long*> ptrs(c->nranks);
    for (int q = 0; q < c->nranks; q++) ptrs[q] = hub->d_ctr + q;
    cudaError_t e = cudaMalloc(&c->d_ctr_ptrs, sizeof(void*) * c->nranks);
    if (e == cudaSuccess) e = cudaMemcpy(c->d_ctr_ptrs, ptrs.data(), sizeof(void*) * c->nranks, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->d_err, 0, sizeof(int));
    if (e != cudaSuccess) return cuda_fail(e, "peer barrier tables");
  }
  cudaFuncAttributes fa;  // load the barrier kernel now (lazy loading mid-step may wait for an idle device)
  cudaError_t e = cudaFuncGetAttributes(&fa, peer_barrier_kernel);
  if (e != cudaSuccess) return cuda_fail(e, "load peer barrier kernel");
  hub->peer_packet[c->rank] = p;
  c->peer_gather.assign(c->nranks, nullptr);
  for (int q = 0; q < c->nranks; q++)
    if (hub->members[q]) c->peer_gather[q] = hub->members[q]->d_gather;
  c->peer_mode = true;
  return ORCHA_OK;
}

extern "C" int32_t orcha_comm_check(orcha_comm* c) {
  if (!c) return fail(ORCHA_E_ARG, "null communicator");
  if (!c->d_err) return ORCHA_OK;
  int err = 0;
  cudaError_t e = cudaMemcpy(&err, c->d_err, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "read peer barrier flag");
  if (err) return fail(ORCHA_E_STATE, "a peer barrier timed out (a rank never arrived)");
  return ORCHA_OK;
}

// ----------------------------------------------- F2 peer mode over CUDA IPC ---
// The same peer mode between PROCESSES (one per GPU on a node, or several on
// one GPU): each rank exports its packet state, dt gather buffer and barrier
// counter as CUDA IPC handles in a blob, the caller exchanges the blobs
// (e.g. torch.distributed over gloo), and every rank maps the others' memory
// (cudaIpcOpenMemHandle, peer access over NVLink between GPUs).  The other
// ranks' packets become "shadow" packets (their mapped state and block ids)
// that the fill plan addresses like the LOCAL transport's.
namespace orcha {
namespace {
constexpr uint32_t kIpcMagic = 0x5049524fu;  // "ORIP"
struct IpcHeader {
  uint32_t magic;
  int32_t rank, nranks, nslots;
  uint64_t state_off, scratch_off;
  int32_t scratch_in_state_alloc;  // the stage-1 buffer lives in the state's allocation
  int32_t pad;
  cudaIpcMemHandle_t h_state, h_scratch, h_gather, h_ctr;
};
// base of the allocation holding p (the torch caching allocator sub-allocates)
cudaError_t alloc_base(void* p, void** base) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return (Fn)f;
  }();
  if (!fn) return cudaErrorNotSupported;
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (CUdeviceptr)p) != CUDA_SUCCESS) return cudaErrorInvalidValue;
  *base = (void*)b;
  return cudaSuccess;
}
}  // namespace
}  // namespace orcha

extern "C" int32_t orcha_comm_create_ipc(const orcha_grid* g, int32_t nranks, int32_t rank, const int32_t* owner,
                                         orcha_comm** out) {
  if (!out) return fail(ORCHA_E_ARG, "null argument");
  *out = nullptr;
  int32_t rc = validate_owner(g, nranks, owner);
  if (rc) return rc;
  if (rank < 0 || rank >= nranks) return fail(ORCHA_E_ARG, "rank out of range");
  orcha_comm* c = new orcha_comm();
  c->grid = g;
  c->nranks = nranks;
  c->rank = rank;
  c->owner.assign(owner, owner + g->nblocks);
  c->local = false;
  c->ipc = true;
  cudaError_t e = cudaMalloc(&c->d_gather, 32 * (size_t)(nranks + 1));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_my_ctr, 256);
  if (e == cudaSuccess) e = cudaMemset(c->d_my_ctr, 0, 256);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_err, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->d_err, 0, sizeof(int));
  if (e != cudaSuccess) {
    destroy_comm(c);
    return cuda_fail(e, "allocate IPC communicator buffers");
  }
  std::lock_guard<std::mutex> lk(g_comm_mu);
  g_comms.push_back(c);
  *out = c;
  return ORCHA_OK;
}

extern "C" int32_t orcha_comm_ipc_export(orcha_comm* c, orcha_packet* p, void* blob, size_t cap, size_t* size) {
  if (!c || !p || !size) return fail(ORCHA_E_ARG, "null argument");
  if (!c->ipc) return fail(ORCHA_E_ARG, "orcha_comm_ipc_export needs an orcha_comm_create_ipc communicator");
  if (p->grid != c->grid) return fail(ORCHA_E_ARG, "packet of another grid");
  long long owned = 0;
  for (long long b = 0; b < c->grid->nblocks; b++) owned += c->owner[b] == c->rank;
  for (long long b : p->ids)
    if (c->owner[b] != c->rank) return fail(ORCHA_E_RANGE, "packet holds a block this rank does not own");
  if ((long long)p->ids.size() != owned)
    return fail(ORCHA_E_ARG, "peer mode needs ONE packet per rank holding every block the rank owns");
  *size = sizeof(IpcHeader) + sizeof(int64_t) * p->ids.size();
  if (!blob) return ORCHA_OK;
  if (cap < *size) return fail(ORCHA_E_ARG, "blob buffer too small");
  IpcHeader h;
  memset(&h, 0, sizeof h);
  h.magic = kIpcMagic;
  h.rank = c->rank;
  h.nranks = c->nranks;
  h.nslots = p->nslots;
  void *base = nullptr, *sbase = nullptr;
  cudaError_t e = alloc_base(p->state, &base);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h.h_state, base);
  if (e == cudaSuccess) e = alloc_base(p->scratch, &sbase);  // the stage-1 buffer (per-stage variant)
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h.h_scratch, sbase);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h.h_gather, c->d_gather);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h.h_ctr, c->d_my_ctr);
  if (e != cudaSuccess) return cuda_fail(e, "IPC export");
  h.state_off = (uint64_t)((char*)p->state - (char*)base);
  h.scratch_off = (uint64_t)((char*)p->scratch - (char*)sbase);
  h.scratch_in_state_alloc = sbase == base ? 1 : 0;
  memcpy(blob, &h, sizeof h);
  memcpy((char*)blob + sizeof h, p->ids.data(), sizeof(int64_t) * p->ids.size());
  c->own_packet = p;
  return ORCHA_OK;
}

extern "C" int32_t orcha_comm_ipc_attach(orcha_comm* c, const void* blobs, size_t stride) {
  if (!c || !blobs) return fail(ORCHA_E_ARG, "null argument");
  if (!c->ipc || !c->own_packet) return fail(ORCHA_E_STATE, "orcha_comm_ipc_export first");
  if (c->peer_mode) return fail(ORCHA_E_STATE, "already attached");
  // a failed earlier attempt: release what it mapped before trying again
  for (void* p : c->ipc_mapped) cudaIpcCloseMemHandle(p);
  c->ipc_mapped.clear();
  for (auto* p : c->shadow) delete p;
  c->shadow.clear();
  std::vector<unsigned long long*> ctr(c->nranks, nullptr);
  c->peer_gather.assign(c->nranks, nullptr);
  for (int q = 0; q < c->nranks; q++) {
    const char* b = (const char*)blobs + stride * (size_t)q;
    IpcHeader h;
    memcpy(&h, b, sizeof h);
    if (h.magic != kIpcMagic || h.rank != q || h.nranks != c->nranks || h.nslots < 1 ||
        sizeof h + sizeof(int64_t) * (size_t)h.nslots > stride)
      return fail(ORCHA_E_ARG, "IPC blob " + std::to_string(q) + " is malformed or out of rank order");
    if (q == c->rank) {
      ctr[q] = c->d_my_ctr;
      c->peer_gather[q] = c->d_gather;
      continue;
    }
    std::vector<long long> ids((size_t)h.nslots);
    memcpy(ids.data(), b + sizeof h, sizeof(int64_t) * ids.size());
    for (long long id : ids)
      if (id < 0 || id >= c->grid->nblocks || c->owner[id] != q)
        return fail(ORCHA_E_RANGE, "IPC blob " + std::to_string(q) + " lists a block that rank does not own");
    void *st = nullptr, *sc = nullptr, *ga = nullptr, *ct = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&st, h.h_state, cudaIpcMemLazyEnablePeerAccess);
    if (e == cudaSuccess) c->ipc_mapped.push_back(st);
    // the state and the stage-1 buffer may be sub-allocations of one
    // allocation (the torch caching allocator): one handle, mapped once
    if (e == cudaSuccess) {
      if (h.scratch_in_state_alloc) {
        sc = st;
      } else {
        e = cudaIpcOpenMemHandle(&sc, h.h_scratch, cudaIpcMemLazyEnablePeerAccess);
        if (e == cudaSuccess) c->ipc_mapped.push_back(sc);
      }
    }
    if (e == cudaSuccess) e = cudaIpcOpenMemHandle(&ga, h.h_gather, cudaIpcMemLazyEnablePeerAccess);
    if (e == cudaSuccess) c->ipc_mapped.push_back(ga);
    if (e == cudaSuccess) e = cudaIpcOpenMemHandle(&ct, h.h_ctr, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "IPC open");
    c->ipc_mapped.push_back(ct);
    orcha_packet* sh = new orcha_packet();  // a source only: never filled, advanced or destroyed by the caller
    sh->grid = c->grid;
    sh->nslots = h.nslots;
    sh->ids = ids;
    sh->state = (double*)((char*)st + h.state_off);
    sh->scratch = (double*)((char*)sc + h.scratch_off);
    c->shadow.push_back(sh);
    ctr[q] = (unsigned long long*)ct;
    c->peer_gather[q] = ga;
  }
  cudaError_t e = cudaMalloc(&c->d_ctr_ptrs, sizeof(void*) * c->nranks);
  if (e == cudaSuccess) e = cudaMemcpy(c->d_ctr_ptrs, ctr.data(), sizeof(void*) * c->nranks, cudaMemcpyHostToDevice);
  cudaFuncAttributes fa;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, peer_barrier_kernel);
  if (e != cudaSuccess) return cuda_fail(e, "IPC barrier tables");
  c->peer_mode = true;
  return ORCHA_OK;
}
