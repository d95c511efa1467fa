// orcha_internal.h -- private declarations shared by the runtime (host) and the
// sm_100a kernels of liborcha.so.  Nothing here is part of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/orcha.h"

namespace orcha {

constexpr int kNVar = 5;          // rho, rho*u, rho*v, rho*w, E (SURVEY 8 "nvar = 5 in every dimension")
constexpr size_t kAlign = 256;    // every (slot, var) cube starts on a 256-byte boundary

// Per-axis guard-source mode of a neighbour-table entry.
enum : int { kShift = 0, kClamp = 1, kMirror = 2 };

// Device-side constant description of the grid (passed by value to kernels).
struct DevGrid {
  int ndim;
  int nb[3];        // cells per block per axis
  int ng;           // guard width
  int gd[3];        // guard width per axis (ng on active axes, 0 otherwise)
  int P[3];         // padded extents per axis
  int N[3];         // global cells per axis
  int nblk[3];      // blocks per axis
  long long cube;   // doubles between consecutive (slot, var) cubes
  double id[3];     // 1/dx per axis (1/dx computed once)
  double gamma, gm1, ig1, cfl, smallp;  // gm1 = gamma - 1, ig1 = 1/(gamma - 1)
  int riemann, limiter;                 // F4 scheme flags (0 = HLL / minmod)
  int eos, eos_work;                    // F4 EOS flag (0 = gamma law) and its work multiplier
  double arad;                          // F4 gas + radiation EOS: radiation constant
};

// One entry per (slot, neighbour direction); 27 per slot, dir = (oz+1)*9 + (oy+1)*3 + (ox+1).
struct NbrEntry {
  const double* src;   // base of the source block's var-0 cube (nullptr = remote, filled by exchange)
  int32_t mode;        // 2 bits per axis: kShift / kClamp / kMirror
  int32_t flip;        // bit (1+d) set -> negate variable 1+d (reflect on axis d)
};

// Push table: one entry per (slot, direction o): the block whose guards in
// direction -o (seen from it) are sourced by this block's cells -- the block
// at b+o (periodic wrap), or b itself along axes where b+o leaves the domain
// through a clamp / mirror boundary.  Per-axis modes as NbrEntry (shift,
// clamp, mirror); nullptr = target not resident (remote: exchange fills it).
struct PushEntry {
  double* dst;         // base of the target block's var-0 cube (state or stage-1 buffer)
  int32_t mode;        // 2 bits per axis
  int32_t flip;        // bit (1+d): negate variable 1+d
};

// Sticky per-packet status word (lives in the scratch tail).
struct DevStatus {
  unsigned long long first_bad;   // lowest global cell index with a non-physical state (ULLONG_MAX = none)
  unsigned long long floor_hits;  // pressure-floor hits (own-cell primitive recovery per cell-stage)
};

// (s, g) reduction record: max s, ties -> lowest g, NaN wins (lowest g among NaN).
struct DtRecord {
  double s;
  long long g;
};

using DevClock = orcha_dev_clock;

// Cross-rank dt record (32 bytes, allgathered by NCCL).
struct GatherRec {
  double s;
  long long g;
  long long bad;
  long long pad;
};

// Multi-packet dt reduction: one packet's records and status word.
struct PacketDt {
  const DtRecord* rec;
  long long n;
  const DevStatus* st;
};

// Multi-packet guard fill: one slot's padded cube base and its 27 table entries.
struct SlotFill {
  double* dst;
  const NbrEntry* tab;
};
static_assert(sizeof(SlotFill) == 16 && sizeof(NbrEntry) == 16, "16-byte descriptor loads (fill_multi_kernel)");

struct SlotInfo {     // per slot: block coordinates (bi, bj, bk)
  int bc[3];
  int pad;
};

__host__ __device__ inline bool dt_better(double sa, long long ga, double sb, long long gb) {
  bool na = sa != sa, nb = sb != sb;
  if (na || nb) return na && (!nb || ga < gb);
  return sa > sb || (sa == sb && ga < gb);
}

}  // namespace orcha

// --------------------------------------------------------------- host side --
struct orcha_grid {
  orcha_grid_desc desc;
  orcha::DevGrid dev;
  long long nblocks;
};

struct FillPlan;  // runtime.cu

struct orcha_packet {
  const orcha_grid* grid;
  int nslots;
  std::vector<long long> ids;
  double* state;               // caller-owned
  double* scratch;             // caller-owned: U1 cubes, then tail
  orcha::DevStatus* status;    // in scratch tail
  orcha::DtRecord* result;     // in scratch tail (1 record)
  orcha::GatherRec* d_grec;    // in scratch tail, 64 B after result (orcha_compute_dt_device)
  orcha::DtRecord* records;    // in scratch tail
  long long records_cap;
  long long nrecords;          // records written by the last advance/dt kernel
  orcha::SlotInfo* d_slots;    // library-owned device table
  bool guards_valid;
  bool records_valid;
  bool guards_full;            // false after the per-stage (faces, depth 2) fill
  bool stage1_done;            // per-stage variant: U1 computed, stage 2 pending
  bool u1_guards_valid;        // per-stage variant: U1 guards refilled
  // guard push (push.cuh): tables of the last fill plan this packet was filled with
  const orcha::PushEntry* d_push;     // targets in the states
  const orcha::PushEntry* d_push_u1;  // targets in the stage-1 buffers
  const FillPlan* push_plan;          // the plan those tables belong to
  int plan_q = -1;                    // this packet's index in push_plan's packet list
  bool guards_pushed;          // the last state update scattered itself into the guards (push_plan)
  bool u1_pushed;              // same for the stage-1 buffer
  bool xguards_pushed;         // the last advance scattered U^{n+1} into the x-guards only (gather mode)
  // gather mode: the last state fill wrote only the x-guards; stage 1 stages
  // the y/z guard rows from the owning blocks through d_nbr
  bool guards_xonly;
  const orcha::NbrEntry* d_nbr;
  // per-stage variant, gather mode: stage 1 scattered U1 into the U1
  // x-guards; the stage-1 buffer "fill" then only marks them valid and stage
  // 2 stages its y/z guard rows of U1 from the owning blocks (d_nbr_u1)
  bool u1_xpushed;
  bool u1_guards_xonly;
  const orcha::NbrEntry* d_nbr_u1;
  // F2 peer mode: the communicator whose ranks' packets this one's last fill
  // addressed directly (the advance then puts a cross-rank barrier between
  // its stage kernels); nullptr otherwise
  orcha_comm* peer_comm = nullptr;
  // interior/boundary overlap (orcha_hydro_step_overlap): a library-owned
  // side stream for the exchange and two events
  cudaStream_t side = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
};

namespace orcha {

// error plumbing (runtime.cu)
int32_t fail(int32_t code, const std::string& msg);
int32_t cuda_fail(cudaError_t e, const char* what);
void count_launch(long long n = 1);

// layout helpers
long long cube_doubles(const DevGrid& G);
size_t state_bytes(const DevGrid& G, long long nslots);
long long records_capacity(const DevGrid& G, long long nslots);

// kernel launchers (kernels_*.cu); all return cudaGetLastError()
// faces_only: 0 every guard, 1 face guards to depth 2, 2 the gather-mode
// complement (x-guards of y/z-guard rows whose row source is remote)
cudaError_t launch_fill(const DevGrid& G, double* state, int nslots, const NbrEntry* table,
                        cudaStream_t s, int faces_only = 0);
cudaError_t launch_fill_x(const DevGrid& G, double* state, int nslots, const NbrEntry* table, cudaStream_t s);
cudaError_t launch_pack(const DevGrid& G, double* state, const double* staged, int nslots,
                        bool to_state, cudaStream_t s);
cudaError_t launch_status_reset(DevStatus* st, cudaStream_t s);
cudaError_t launch_dt(const DevGrid& G, const double* state, int nslots, const SlotInfo* slots,
                      DtRecord* records, long long* nrecords, DevStatus* st, cudaStream_t s);
cudaError_t launch_dt_reduce(const DtRecord* records, long long n, DtRecord* out, cudaStream_t s);
// Device-resident dt (orcha_compute_dt_device): the reduced record and
// status -> this rank's GatherRec; then (after an optional allgather of
// nall records) dt, tag and the clock update in `clock` (orcha_dev_clock).
cudaError_t launch_dt_gather_rec(const DtRecord* r, const DevStatus* st, GatherRec* out, cudaStream_t s);
cudaError_t launch_dt_finish(const GatherRec* all, int nall, double cfl, void* clock, cudaStream_t s);
cudaError_t launch_dt_reduce_finish(const DtRecord* records, long long n, DtRecord* out, const DevStatus* st,
                                    GatherRec* grec, double cfl, void* clock, cudaStream_t s);
cudaError_t launch_dt_reduce_multi(const PacketDt* pd, int npk, DtRecord* out, DevStatus* out_st, cudaStream_t s);
cudaError_t launch_fill_multi(const DevGrid& G, const SlotFill* sf, long long nslots, cudaStream_t s,
                              int faces_only);
cudaError_t launch_advance(const DevGrid& G, double* state, double* u1, int nslots,
                           const SlotInfo* slots, const double* d_dt, double h_dt,
                           DtRecord* records, long long* nrecords, DevStatus* st, cudaStream_t s);

// kernel variant selection (0 = reference per-cell kernels, 1 = fused z-marching)
int kernel_variant();

// Phases of the hot path (phases.cu): an NVTX range always, a CUDA-event pair
// on the stream while orcha_set_phase_timing is on.  RAII: the scope's end
// records the closing event.  Indices are ORCHA_PHASE_* of orcha.h.
enum { PH_FILL = 0, PH_EXCHANGE = 1, PH_DT = 2, PH_DT_COMM = 3, PH_STAGE1 = 4, PH_STAGE2 = 5, PH_COUNT = 6 };
class PhaseScope {
 public:
  PhaseScope(int phase, cudaStream_t s);
  ~PhaseScope();
  PhaseScope(const PhaseScope&) = delete;
  PhaseScope& operator=(const PhaseScope&) = delete;

 private:
  int phase_;
  cudaStream_t stream_;
  int idx_;                 // 0: this scope holds an event pair (a_, b_)
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};

}  // namespace orcha
