/*
 * orcha.h -- C ABI of liborcha.so: the per-block explicit hydrodynamics update
 * that ORCHA orchestrates in its Flash-X Sedov case study (arXiv 2507.09337),
 * applied to a data packet of N equal blocks with guard cells, on one B200.
 *
 * Citations: P:Lnn = PAPER.md line nn (section in parentheses); SURVEY 8(x) =
 * the normative reading of the paper in SURVEY.md section 8 (the paper does
 * not name the reconstruction, Riemann solver, CFL rule or boundaries; see
 * DESIGN.md "Readings").
 *
 * Conventions for every call
 *   - Return value: ORCHA_OK (0) or a negative orcha_status.  On error,
 *     orcha_last_error() returns a thread-local, human-readable message.
 *     Argument errors are detected synchronously, before anything is queued.
 *   - Handles (orcha_grid, orcha_packet, orcha_comm) are opaque and owned by
 *     the library; destroy them with the matching *_destroy call.
 *   - Device buffers passed in (d_state, d_scratch) are OWNED BY THE CALLER
 *     (e.g. torch tensors), must stay alive while the packet exists, and are
 *     never freed by the library.  They must be 256-byte aligned.
 *   - Host arrays are owned by the caller and are only read/written during
 *     the call (or, for the async pack/unpack, until the stream reaches the
 *     copy; use pinned memory for overlap).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream), e.g.
 *     torch.cuda.current_stream().cuda_stream.  All device work of a call is
 *     enqueued on it.  A packet is used by one stream at a time.
 *   - Floating point is IEEE fp64 throughout; no fast-math.
 *
 * Data layout ("DataPacket", sec 4.3: "n AMR blocks" flattened into
 * one buffer; blocks per P:L567-569 sec 5.1: "each block has the same number
 * of cells"):
 *   state[slot][var][k][j][i], var = (rho, rho*u, rho*v, rho*w, E), always 5
 *   (inactive momenta are 0), padded extents nb_d + 2*ng on active axes and 1
 *   on inactive axes, i fastest; every (slot, var) cube starts on a 256-byte
 *   boundary (cube stride = cells*8 rounded up to 256 bytes).  Slot s holds
 *   global block block_ids[s]; global block id b = (bk*NBy + bj)*NBx + bi and
 *   global cell index g = (k*Ny + j)*Nx + i.
 */
#ifndef ORCHA_H
#define ORCHA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ORCHA_OK = 0,
  ORCHA_E_ARG = -1,         /* invalid argument / descriptor */
  ORCHA_E_RANGE = -2,       /* block id or slot out of range, duplicate block, neighbour not resident */
  ORCHA_E_HALO = -3,        /* ng < 4: the telescoped step needs a twice-thick halo */
  ORCHA_E_NONPHYSICAL = -4, /* rho <= 0 or non-finite state met on the device (sticky, see below) */
  ORCHA_E_LAYOUT = -5,      /* buffer misaligned or too small */
  ORCHA_E_CUDA = -6,        /* CUDA runtime error (message has the CUDA error string) */
  ORCHA_E_NCCL = -7,        /* NCCL error */
  ORCHA_E_STATE = -8        /* call order violated, e.g. advance without a guard fill */
} orcha_status;

enum { ORCHA_BC_OUTFLOW = 0, ORCHA_BC_PERIODIC = 1, ORCHA_BC_REFLECT = 2 };
enum { ORCHA_DT_CFL = 0, ORCHA_DT_CLAMP = 1 };

/* Global uniform grid of equal blocks.  Boundary conditions per axis and side
 * (SURVEY 8(c) c6): outflow = copy of the edge cell; periodic = wrap; reflect =
 * mirror with the normal momentum negated.  Physical extent [xmin, xmax] per
 * axis, cell size dx_d = (xmax_d - xmin_d) / (nblk_d * nb_d). */
typedef struct {
  int32_t ndim;       /* 1, 2 or 3 */
  int32_t nb[3];      /* cells per block per axis (nxb, nyb, nzb); 1 on inactive axes */
  int32_t ng;         /* guard cells per side on active axes; must be >= 4 */
  int32_t nblk[3];    /* blocks per axis of the GLOBAL grid; 1 on inactive axes */
  double xmin[3], xmax[3];
  int32_t bc[3][2];   /* [axis][0 = low side, 1 = high side] */
  double gamma;       /* ideal-gas gamma; e.g. 1.4 */
  double cfl;         /* CFL number (reading c7); e.g. 0.4 */
  double smallp;      /* pressure floor used in primitive recovery only (c10); e.g. 1e-30 */
  /* SURVEY 8(f) F4 scheme variants (zero = the paper-path defaults):
   * riemann: ORCHA_RIEMANN_HLL (A7) or ORCHA_RIEMANN_HLLC (Toro sec 10.4,
   * same wave speeds; reading c20); limiter: ORCHA_LIMITER_MINMOD
   * (A6) or ORCHA_LIMITER_MC (monotonized central, reading c21). */
  int32_t riemann;
  int32_t limiter;
  /* F4 expensive-EOS surrogate (reading c22): eos = ORCHA_EOS_GAMMA_LAW (A5)
   * or ORCHA_EOS_GAS_RADIATION: ideal gas + radiation with c_v = 1,
   * rho e = rho T + arad T^4, p = (gamma-1) rho T + arad T^4 / 3, the
   * temperature by Newton iteration (repeated eos_work >= 1 times: the
   * surrogate's cost knob), sound speed from Chandrasekhar's Gamma_1. */
  int32_t eos;
  int32_t eos_work;
  double arad;
} orcha_grid_desc;

enum { ORCHA_RIEMANN_HLL = 0, ORCHA_RIEMANN_HLLC = 1 };
enum { ORCHA_LIMITER_MINMOD = 0, ORCHA_LIMITER_MC = 1 };
enum { ORCHA_EOS_GAMMA_LAW = 0, ORCHA_EOS_GAS_RADIATION = 1 };

typedef struct orcha_grid orcha_grid;
typedef struct orcha_packet orcha_packet;
typedef struct orcha_comm orcha_comm;

/* Result of orcha_compute_dt. */
typedef struct {
  double dt;          /* selected time step */
  double smax;        /* max over interior cells of the signal speed sum s */
  int64_t argmax;     /* lowest global cell index g with s == smax */
  int32_t tag;        /* ORCHA_DT_CFL or ORCHA_DT_CLAMP (t_end won) */
  int32_t nonphysical;/* 1 if a non-positive/non-finite density was met */
} orcha_dt_info;

/* Device-resident clock of orcha_compute_dt_device (caller-owned DEVICE
 * memory, 8-byte aligned, 64 bytes).  The caller initialises t, t_end (and
 * steps) before the first step; every call writes dt, smax, argmax, tag and
 * nonphysical as orcha_compute_dt reports them and advances t by dt. */
typedef struct {
  double t;           /* simulation time (advanced by dt on every call) */
  double t_end;       /* end time: dt is clamped to t_end - t (tag CLAMP) */
  double dt;          /* selected time step (pass &clock->dt to *_devdt) */
  double smax;        /* max signal speed sum */
  int64_t argmax;     /* lowest global cell index g with s == smax */
  int32_t tag;        /* ORCHA_DT_CFL or ORCHA_DT_CLAMP */
  int32_t nonphysical;/* 1 if a non-positive/non-finite density was met */
  int64_t steps;      /* calls so far (incremented on every call) */
  int64_t reserved;
} orcha_dev_clock;

/* ------------------------------------------------------------- grid ---- */

/* Validate `desc` and create a grid handle (host only, no device work).
 * Errors: ORCHA_E_ARG (ndim, nb, nblk, extents, bc codes, gamma <= 1,
 * cfl <= 0, riemann / limiter / eos codes, eos_work < 1 or arad < 0 with the
 * gas + radiation EOS), ORCHA_E_HALO (ng < 4), ORCHA_E_ARG if a periodic axis has fewer
 * cells than ng. */
int32_t orcha_grid_create(const orcha_grid_desc* desc, orcha_grid** out);
int32_t orcha_grid_destroy(orcha_grid* grid);
/* Number of blocks of the global grid (NBx*NBy*NBz). */
int64_t orcha_grid_nblocks(const orcha_grid* grid);

/* ----------------------------------------------------------- packets ---- */

/* Bytes of caller-owned device memory a packet of `nblocks` blocks needs:
 * `state_bytes` for the padded conserved state (layout above) and
 * `scratch_bytes` for the stage-1 state U1 (same padded layout; also used as
 * the staging area of pack/unpack) plus reduction records and the status word.
 * Host only.  Errors: ORCHA_E_ARG if nblocks < 1. */
int32_t orcha_packet_bytes(const orcha_grid* grid, int32_t nblocks, size_t* state_bytes,
                           size_t* scratch_bytes);

/* Create a packet of `nblocks` blocks ("several blocks ... collected into a
 * single DataPacket", sec 3.2; "n is provided by the users at
 * runtime", sec 4.3).  `block_ids` (host, copied) gives the global
 * block id of each slot.  d_state / d_scratch: caller-owned device memory of
 * at least orcha_packet_bytes(), 256-byte aligned.  Allocates small
 * library-owned device tables (per-slot block coordinates) and uploads them
 * synchronously; no other device work.  Errors: ORCHA_E_RANGE (id outside the
 * grid or repeated), ORCHA_E_LAYOUT (alignment), ORCHA_E_CUDA. */
int32_t orcha_packet_create(const orcha_grid* grid, int32_t nblocks, const int64_t* block_ids,
                            void* d_state, void* d_scratch, orcha_packet** out);
int32_t orcha_packet_destroy(orcha_packet* packet);
int32_t orcha_packet_nblocks(const orcha_packet* packet);
/* Device pointer of the state and bytes of one (slot, var) cube stride. */
int32_t orcha_packet_layout(const orcha_packet* packet, void** d_state, size_t* cube_bytes,
                            int32_t padded_extent[3]);

/* Pack: copy the packet's INTERIOR cells from host memory into the device
 * state ("moving pointers into pinned memory and back", sec 4.3).
 * h_interior layout: [slot][var][k][j][i] over the packet's blocks, extents
 * nb_d (no guards), contiguous fp64.  Enqueued on `stream` (H2D into the
 * scratch staging area, then a scatter kernel into the padded cubes); guard
 * cells are left for orcha_fill_guardcells.  Marks the guards stale.
 * Errors: ORCHA_E_ARG, ORCHA_E_CUDA. */
int32_t orcha_packet_pack(orcha_packet* packet, const double* h_interior, void* stream);

/* Unpack: inverse of pack (gather kernel + D2H), then synchronizes `stream`.
 * Returns ORCHA_E_NONPHYSICAL if the packet's sticky status word recorded a
 * non-positive or non-finite density since the last pack (data is still
 * copied). */
int32_t orcha_packet_unpack(const orcha_packet* packet, double* h_interior, void* stream);

/* Device-to-device variants (d_interior: device pointer, same layout). */
int32_t orcha_packet_pack_device(orcha_packet* packet, const double* d_interior, void* stream);
int32_t orcha_packet_unpack_device(const orcha_packet* packet, double* d_interior, void* stream);

/* Unpack without the synchronizing status check, for streamed packets
 * (packets shipped in and out every cycle on copy streams
 * overlapping the other packets' compute): the gather kernel and
 * the copy into `interior` (pinned host or device memory; any address the
 * runtime can copy to asynchronously) are only enqueued on `stream`.  The
 * packet's sticky status is reported by the next orcha_compute_dt or
 * synchronizing unpack.  The packet's scratch holds the staged data until
 * the copy has run: order the next pack / advance of this packet after it.
 * Errors: ORCHA_E_ARG, ORCHA_E_CUDA. */
int32_t orcha_packet_unpack_async(const orcha_packet* packet, double* interior, void* stream);

/* -------------------------------------------------------- the hot path -- */

/* Guard-cell fill ("We assume that the first refresh occurs before we invoke
 * ORCHA", sec 6).  `packets` are ALL packets of
 * this device; together (plus `comm` for blocks on other ranks, NULL on one
 * GPU) they must hold every block the guards read.  Every guard cell of every
 * block (faces, edges and corners, depth ng) gets the value of the global
 * axis-ordered ghost fill (x, then y over x-guards, then z over x,y-guards):
 * a neighbour's interior cell or the physical boundary image.  Pure copies,
 * bitwise.  (In the default GATHER fill mode -- orcha_set_fill_mode -- a
 * single packet with all sources resident gets only its x-guards written here;
 * the advance composes the rest while staging.)  The first call with a given
 * packet set builds and caches the neighbour tables (host + one device
 * upload); later calls only launch.
 * Errors: ORCHA_E_RANGE (a needed block is not resident and comm is NULL),
 * ORCHA_E_ARG, ORCHA_E_CUDA, ORCHA_E_NCCL. */
int32_t orcha_fill_guardcells(orcha_packet* const* packets, int32_t npackets, orcha_comm* comm,
                              void* stream);

/* Streamed packets (the paper overlaps each DataPacket's
 * transfers with the other packets' work): the two local parts of
 * a step's preparation, per packet, so they run as soon as that packet's data
 * is on the device instead of after the whole set arrived.
 *
 * orcha_fill_guardcells_packet: the guard fill of orcha_fill_guardcells over
 * the set `packets` (same tables, same bitwise result), for packets[index]
 * only.  Every block its guards read must already hold this step's data (the
 * caller orders `stream` after those packets' packs).  Single device only:
 * returns ORCHA_E_ARG if a source block lives on another rank (use
 * orcha_fill_guardcells with a communicator).  Asynchronous.
 * Errors: ORCHA_E_ARG, ORCHA_E_RANGE, ORCHA_E_CUDA. */
int32_t orcha_fill_guardcells_packet(orcha_packet* const* packets, int32_t npackets, int32_t index,
                                     void* stream);

/* orcha_packet_dt_records: the per-packet part of orcha_compute_dt -- the CFL
 * signal-speed max and its lowest global index over the packet's interior
 * cells -- computed now on `stream` (asynchronous).  A later
 * orcha_compute_dt over a set containing the packet only reduces these
 * records (order its stream after this one); a pack or advance invalidates
 * them.  Non-positive densities set the sticky status word.
 * Errors: ORCHA_E_ARG, ORCHA_E_CUDA. */
int32_t orcha_packet_dt_records(orcha_packet* packet, void* stream);

/* CFL time step over the interior cells of `packets`:
 *   s = ((|u|+c)*idx + (|v|+c)*idy) + (|w|+c)*idz  (inactive axes omitted),
 *   c = sqrt((gamma*p)/rho), dt = cfl / max s; argmax = lowest global g with
 *   s == max (bitwise deterministic); then if t_remaining < dt, dt =
 *   t_remaining (tag CLAMP).  NaN in any s propagates to dt.  With `comm`,
 *   the max is reduced over all ranks (allreduce-max of 8 bytes).
 * Uses the s-max records the last orcha_hydro_advance wrote for the new state
 * when they are valid (bitwise identical to recomputing); otherwise launches
 * the dt kernels.  Synchronizes `stream`.  Returns ORCHA_E_NONPHYSICAL if a
 * non-positive/non-finite density was met (info still filled). */
int32_t orcha_compute_dt(orcha_packet* const* packets, int32_t npackets, orcha_comm* comm,
                         double t_remaining, orcha_dt_info* info, void* stream);

/* orcha_compute_dt with the result kept on the device (no host
 * synchronization, so a time loop of fill -> dt -> advance runs ahead of the
 * host and can be captured in a CUDA graph): the same records, the same
 * cross-rank rule (with `comm`: an NCCL allgather of one 32-byte record per
 * rank, reduced on the device) and the same IEEE operations as
 * orcha_compute_dt, so dt is bitwise identical; written to `d_clock`
 * (orcha_dev_clock), whose `dt` feeds orcha_hydro_advance_devdt.  With
 * several packets a small table of the packets' records is uploaded when it
 * changed since the last call (the first call; steady-state calls only
 * enqueue kernels and may be captured in a CUDA graph).  Non-physical states are reported in
 * d_clock->nonphysical and by the next synchronizing call.
 * Errors: ORCHA_E_ARG (null arguments; LOCAL virtual-rank communicators),
 * ORCHA_E_CUDA, ORCHA_E_NCCL. */
int32_t orcha_compute_dt_device(orcha_packet* const* packets, int32_t npackets, orcha_comm* comm,
                                orcha_dev_clock* d_clock, void* stream);

/* One full telescoped SSP-RK2 step of every block of the packet, in place
 * (sec 6: explicit finite volume with a guard-cell halo, "2nd-order
 * Runge-Kutta", the halo "twice as thick" so the second refresh is avoided):
 *   stage 1 on interior + 2-cell ring:  U1 = U^n - dt*D(U^n)
 *   stage 2 on the interior:            U^{n+1} = 0.5*(U^n + (U1 - dt*D(U1)))
 * with D from gamma-law EOS -> PLM/minmod -> HLL.  No
 * communication ("Milhoja only handles computations that do not involve any
 * MPI operations").  Requires a guard fill since the last pack or
 * advance (else ORCHA_E_STATE); marks the guards stale; writes the s-max
 * records of U^{n+1} for orcha_compute_dt (fused dt epilogue).  Asynchronous.
 * Non-positive densities set the sticky status word (reported by unpack /
 * compute_dt). */
int32_t orcha_hydro_advance(orcha_packet* packet, double dt, void* stream);

/* Same, reading dt from device memory (graph-capturable: no host value). */
int32_t orcha_hydro_advance_devdt(orcha_packet* packet, const double* d_dt, void* stream);

/* ---- per-stage variant (the two-refresh scheme P:L667-668
 * describes before the communication-avoidance trick) ----
 * One SSP-RK2 stage on the interior only:
 *   stage 1: U1 = U^n - dt*D(U^n) into the packet's stage-1 buffer (scratch,
 *            same padded layout as the state); requires a state guard fill;
 *   stage 2: U^{n+1} = 0.5*(U^n + (U1 - dt*D(U1))) in place, + dt records;
 *            requires orcha_fill_guardcells_stage(..., buffer = 1) after
 *            stage 1 (the second guard refresh, with the physical boundary
 *            conditions applied to U1 -- at outflow walls this differs from
 *            the telescoped step in round-off-level momentum tails, reading c5).
 * Errors: ORCHA_E_ARG (stage not 1/2), ORCHA_E_STATE (call order). */
int32_t orcha_hydro_stage(orcha_packet* packet, int32_t stage, double dt, void* stream);
int32_t orcha_hydro_stage_devdt(orcha_packet* packet, int32_t stage, const double* d_dt, void* stream);

/* Guard fill for the per-stage variant: buffer 0 (the state) or buffer 1
 * (the stage-1 buffer, after orcha_hydro_stage(..., 1, ...)).  Fills only
 * what ONE stage reads -- the face guards (one axis outside the block) to
 * depth 2 -- with the same values as orcha_fill_guardcells (exchange
 * included); a state filled this way is valid for orcha_hydro_stage, not for
 * the telescoped orcha_hydro_advance (ORCHA_E_STATE).  Errors as
 * orcha_fill_guardcells, plus ORCHA_E_STATE. */
int32_t orcha_fill_guardcells_stage(orcha_packet* const* packets, int32_t npackets, orcha_comm* comm,
                                    int32_t buffer, void* stream);

/* ----------------------------------------------------------- support ---- */

/* Counters since the last pack: pressure-floor hits in primitive recovery
 * (reading c10) and the sticky non-physical flag with the first (lowest)
 * offending global cell index (-1 if none).  Synchronizes `stream`. */
int32_t orcha_packet_counters(const orcha_packet* packet, int64_t* floor_hits,
                              int64_t* first_bad_cell, void* stream);

/* Which kernel variant this library was built as: 1 = parity build (no FMA
 * contraction, the exact expression order of SURVEY 8(c) c12; bitwise equal to
 * the CPU oracle), 0 = production build (FMA, <= 1e-12 relative). */
int32_t orcha_build_is_parity(void);

/* Number of kernel launches this library has enqueued since load (for the
 * bench's gpu_launches claim). */
int64_t orcha_launch_count(void);

/* Advance-kernel variant for orcha_hydro_advance: 0 = reference kernels (one
 * thread per output cell, stencil recomputed; the structural reference),
 * 1 = fused z-marching kernels (default; ORCHA_KERNEL=0 in the environment
 * selects 0 at load).  Both give bitwise-identical results in the parity
 * build.  Errors: ORCHA_E_ARG for another value. */
int32_t orcha_set_kernel_variant(int32_t variant);
int32_t orcha_get_kernel_variant(void);

/* Fill mode.  1 = GATHER (default): for a single packet whose guard sources
 * are all resident, with the fused kernels, orcha_fill_guardcells writes only
 * the x-guards, and stage 1 of the next advance / orcha_hydro_stage(.., 1, ..)
 * stages each y/z guard row straight from the block that owns it (that
 * block's padded row, x-guards included): the same axis-ordered ghost-fill
 * values, composed while loading (P:L668-669's refresh, done by the consumer).
 * Stage 2 of orcha_hydro_advance then writes U^{n+1} into the x-guards too, so
 * the next fill of the same packet launches nothing.  In this mode the y/z
 * guard cells of the state are NOT materialised (read them only after a FULL
 * fill).  0 = FULL: the fill materialises every guard cell (the packet's guard
 * cells then hold the documented values; multi-packet sets, remote sources and
 * the guard-push mode always use FULL).  ORCHA_FILL_MODE=0 selects FULL at
 * load.  Errors: ORCHA_E_ARG. */
int32_t orcha_set_fill_mode(int32_t mode);

/* Ring mode of the telescoped step (sec 6: stage 1 on the block
 * "plus the inner portion of the halo", so stage 2 needs no second guard
 * exchange).  1 = BORROWED (default): a block computes the stage-1 values of
 * its 2-cell ring only on its "self" sides -- a physical boundary (clamp /
 * mirror), or a neighbour that is not a block of the same packet (another
 * packet, another rank, F2 peer mode's other ranks) -- and takes the ring on
 * every other side from the neighbour that owns those cells, whose own stage 1
 * computes them from the same U^n values: the result is the telescoped step's
 * (bitwise in the parity build), with stage 1 on n^3 instead of (n+4)^3 cells
 * away from self sides.  0 = COMPUTED: every block computes its whole ring
 * (the paper's literal scheme).  Applies to the fused 3D kernels in the
 * gather and full fill modes; the guard-push mode always computes.
 * ORCHA_RING=0 selects COMPUTED at load.  Errors: ORCHA_E_ARG (mode not 0 /
 * 1). */
int32_t orcha_set_ring_mode(int32_t mode);
int32_t orcha_get_ring_mode(void);

/* The borrowed ring's classification, on the host (no device work): for a
 * packet of the n blocks `ids` of grid g taken alone -- a side is "self" when
 * its face neighbour is not one of these blocks reached by a shift (periodic
 * wrap included; a clamp / mirror boundary, or a block outside the list, is
 * self) -- masks[s] = the self sides of block ids[s] (bit 2a: side -a, bit
 * 2a+1: side +a; axes beyond ndim are self) and groups[s] = its stage-1
 * kernel: 2 the interior kernel (no x / y self side; planes extended on self
 * z sides), 1 the (n+2)^2 kernel (16^3 / 8^3 blocks with at most one self
 * side per x / y axis), 0 the (n+4)^2 box.  The same rule the packet plans
 * use (several packets: the sides towards the other packets are self).
 * masks / groups: caller-owned host arrays of n.  Errors: ORCHA_E_ARG (null
 * pointers, n < 0), ORCHA_E_RANGE (an id outside the grid, or repeated). */
int32_t orcha_ring_classify(const orcha_grid* g, int32_t n, const int64_t* ids, int32_t* masks, int32_t* groups);

/* Guard push (default OFF -- measured slower than the gather fill on B200,
 * DESIGN.md 6; ORCHA_PUSH=1 in the environment turns it on at load): the
 * fused kernels that produce a new state also scatter each new
 * interior cell into every guard cell of a resident block whose ghost-fill
 * source it is (the inverse of the gather fill's per-axis images, so the
 * guard values are bitwise the same).  The next orcha_fill_guardcells* call
 * with the same packet set then only runs the cross-rank exchange.  Turning it
 * off makes every fill gather.  Always returns ORCHA_OK. */
int32_t orcha_set_guard_push(int32_t on);

const char* orcha_last_error(void);

/* Per-phase instrumentation (SURVEY 8(d) timing protocol).  Every
 * phase the library enqueues -- ORCHA_PHASE_FILL (orcha_fill_guardcells*,
 * including the exchange), ORCHA_PHASE_EXCHANGE (the cross-rank exchange
 * alone), ORCHA_PHASE_DT (orcha_compute_dt*: record reduction, including the
 * allgather), ORCHA_PHASE_DT_COMM (the dt allgather alone), ORCHA_PHASE_STAGE1
 * and ORCHA_PHASE_STAGE2 (the two RK2 stage kernels of an advance, or of
 * orcha_hydro_stage) -- is an NVTX range named "orcha:<phase>" on the host.
 * With orcha_set_phase_timing(1) each phase also records a pair of CUDA
 * events on its stream (off by default: no events in timed loops).
 * orcha_phase_times synchronizes on every pair recorded since the previous
 * query and writes the summed device milliseconds per phase to ms[0..5] and
 * the number of occurrences to counts[0..5] (counts may be NULL); n >= 6.
 * Call it between library calls, not concurrently with them.  Errors:
 * ORCHA_E_ARG, ORCHA_E_CUDA. */
enum { ORCHA_PHASE_FILL = 0, ORCHA_PHASE_EXCHANGE = 1, ORCHA_PHASE_DT = 2, ORCHA_PHASE_DT_COMM = 3,
       ORCHA_PHASE_STAGE1 = 4, ORCHA_PHASE_STAGE2 = 5, ORCHA_NPHASES = 6 };
int32_t orcha_set_phase_timing(int32_t on);
int32_t orcha_phase_times(double* ms, int64_t* counts, int32_t n);

/* FNV-1a 64-bit hash of `nbytes` host bytes, continuing from *hash (start
 * from ORCHA_FNV1A64_OFFSET = 0xcbf29ce484222325; prime 0x100000001b3): the
 * mesh checksum of SPEC S:L433 ("per-variable FNV-1a over raw bytes").  The
 * binding's mesh_checksums / dump_mesh hash each variable over the blocks in
 * ascending global id, cells in (k, j, i) order, little-endian fp64 -- the
 * same value for any packet split or rank count.  Host only.
 * Errors: ORCHA_E_ARG. */
#define ORCHA_FNV1A64_OFFSET 0xcbf29ce484222325ULL
int32_t orcha_fnv1a64(const void* data, size_t nbytes, uint64_t* hash);

/* Measured fp64-pipe throughput of this GPU (the denominator of the bench's
 * fp64 roofline beside the value derived from unit counts): one launch of 8
 * SM-resident CTAs per SM, 8 independent DFMA chains of `iters` steps per
 * thread, timed with CUDA events on `stream` (synchronizes).  Writes thread
 * DFMA instructions per second / 1e12 and the kernel time.  Not part of the
 * method.  Errors: ORCHA_E_ARG, ORCHA_E_CUDA. */
int32_t orcha_probe_fp64(int32_t iters, double* tinst_per_s, double* ms, void* stream);

/* ------------------------------------------------ unit entry points ----- */
/* The per-cell / per-face device functions the fused kernels call, applied to
 * n independent inputs (test diagnostics for SURVEY 8(d)'s unit fuzz; the hot
 * path never calls these).  The scheme is the grid's: with no F4 flag set the
 * paper-path functions (A5 gamma-law EOS, A6 minmod PLM, A7 HLL -- in the
 * production build its expanded algebra), otherwise the F4 variants.  All
 * buffers are caller-owned DEVICE memory, variable-major with stride n
 * (element v of item i at [v*n + i]); n in [0, 2^31/5].  Asynchronous on
 * `stream`.  Errors: ORCHA_E_ARG (null grid/buffer, n or dir out of range),
 * ORCHA_E_CUDA.
 *
 * orcha_unit_eos: conserved d_U[5][n] -> primitives d_Q[5][n] (rho, u, v, w,
 *   p after the floor), sound speed d_c[n], 3D CFL signal-speed sum d_s[n]
 *   (A4's s with the grid's 1/dx), floor flag d_floored[n] (A5, c10).
 * orcha_unit_face_flux: primitives of the 4-cell stencil d_q[4][5][n]
 *   (cells i-1, i, i+1, i+2 along dir) -> flux through face i+1/2, d_F[5][n]
 *   (A6 + A7).
 * orcha_unit_riemann: face states d_qL[5][n], d_qR[5][n] (primitives) ->
 *   Riemann flux along dir, d_F[5][n] (A7; HLLC reading c20 with the flag). */
int32_t orcha_unit_eos(const orcha_grid* grid, int64_t n, const double* d_U, double* d_Q, double* d_c,
                       double* d_s, int32_t* d_floored, void* stream);
int32_t orcha_unit_face_flux(const orcha_grid* grid, int32_t dir, int64_t n, const double* d_q, double* d_F,
                             void* stream);
int32_t orcha_unit_riemann(const orcha_grid* grid, int32_t dir, int64_t n, const double* d_qL,
                           const double* d_qR, double* d_F, void* stream);

/* ------------------------------------------------------- multi-GPU ------ */

/* Communicator for blocks partitioned over ranks (one process per GPU,
 * "4 MPI ranks, each rank talking to one GPU", sec 6.1).
 * `block_owner[b]` (host, copied, length orcha_grid_nblocks) is the rank that
 * owns global block b.  `nccl_unique_id` is the 128-byte ncclUniqueId that
 * rank 0 created (orcha_comm_unique_id) and the caller broadcast (e.g. with
 * torch.distributed).  The guard exchange is one grouped ncclSend/ncclRecv per
 * neighbour rank of gathered guard sources; dt uses ncclAllReduce(max).
 * Errors: ORCHA_E_ARG, ORCHA_E_NCCL. */
int32_t orcha_comm_unique_id(void* nccl_unique_id_128);
int32_t orcha_comm_create(const orcha_grid* grid, const void* nccl_unique_id_128, int32_t nranks,
                          int32_t rank, const int32_t* block_owner, orcha_comm** out);
int32_t orcha_comm_destroy(orcha_comm* comm);

/* In-process transport for tests and single-GPU decomposition studies:
 * creates `nranks` communicators (out[r] for virtual rank r) that share one
 * device; their exchange is device-to-device copies instead of NCCL.  The
 * caller first calls orcha_comm_push for EVERY virtual rank (each packs its
 * guard sources straight into its peers' receive buffers) and then
 * orcha_fill_guardcells for each (which unpacks and fills).  No NCCL needed. */
int32_t orcha_comm_create_local(const orcha_grid* grid, int32_t nranks, const int32_t* block_owner,
                                orcha_comm** out);
int32_t orcha_comm_push(orcha_comm* comm, orcha_packet* const* packets, int32_t npackets, int32_t buffer,
                        void* stream);  /* buffer: 0 = state, 1 = stage-1 buffer */
/* LOCAL transport, dt: pushes this virtual rank's 32-byte dt record (max
 * signal speed s over its packets, lowest global cell index g, non-physical
 * flag -- what the NCCL path allgathers) into slot `rank` of every member's
 * gather buffer.  Call it for EVERY virtual rank (after the step's fill),
 * then orcha_compute_dt / orcha_compute_dt_device for each with its own
 * communicator: each reduces all ranks' records with the single-GPU rule
 * (max s, ties -> lowest g, NaN wins), exactly as after an ncclAllGather.
 * Errors: ORCHA_E_ARG (NCCL communicator, null argument), ORCHA_E_CUDA. */
int32_t orcha_comm_push_dt(orcha_comm* comm, orcha_packet* const* packets, int32_t npackets, void* stream);

/* Interior/boundary overlap (SURVEY 8(e) "Overlap"; the paper's streams
 * hiding transfers): one telescoped step of this rank's single
 * packet -- orcha_compute_dt_device into d_clock, then the guard exchange on
 * a library-owned stream while stage 1 runs on the packet's LEADING interior
 * slots (blocks whose 26 neighbours are all in this packet, so they read
 * nothing the exchange writes); stage 1 of the remaining slots waits for the
 * exchange, stage 2 runs on all.  Order the packet's block_ids interior-first
 * to get any overlap.  Results are bitwise those of orcha_fill_guardcells ->
 * orcha_compute_dt_device -> orcha_hydro_advance_devdt, which is also what
 * runs when there is nothing to overlap (first step after a pack, no remote
 * source, an owner map whose gather fill needs the complement pass, no
 * leading interior slot).  Gather fill mode and the fused kernels; a LOCAL
 * communicator needs every rank's orcha_comm_push (and orcha_comm_push_dt)
 * first, as for orcha_fill_guardcells.  Errors: as those calls. */
int32_t orcha_hydro_step_overlap(orcha_packet* packet, orcha_comm* comm, orcha_dev_clock* d_clock, void* stream);

/* F2 peer mode (the guard fill reads peer ranks' packets
 * directly instead of exchanging, and dt is reduced by a one-shot peer write).
 * Each rank registers its ONE packet (holding every block it owns).  Once all
 * ranks have, orcha_fill_guardcells with this communicator builds neighbour
 * and push tables that point into the other ranks' packets: the fill writes
 * only x-guards (gather fill mode, fused kernels), stage 1 stages y/z guard
 * rows straight from the owning block wherever it lives, stage 2 writes its
 * new cells into the x-guards of the blocks they feed, on every rank -- no
 * pack, send/recv or unpack.  Ordering across ranks is by a device-side
 * barrier (system-scope counters; a wait beyond ~10 s sets an error flag read
 * by orcha_comm_check instead of hanging): after a pack, before the first
 * x-guard fill; between the two stage kernels of every advance (stage 2
 * overwrites U^n in place while other ranks' stage 1 may read it); and in
 * orcha_compute_dt(_device), which writes this rank's dt record into every
 * rank's gather slot and then waits.  Each rank must therefore issue its
 * calls on its OWN stream, concurrently with the others (a single stream
 * serialising two ranks would wait forever at the first barrier -- and
 * time out), and must not allocate device memory between the ranks'
 * launches (CUDA's implicit synchronisation would serialise the streams):
 * call orcha_fill_prepare for every rank first.  orcha_comm_peer_register is
 * for LOCAL (virtual-rank) communicators, whose packets are directly
 * addressable in one process (same-device "peers"); across processes the CUDA
 * IPC communicator below enters the same mode (orcha_comm_ipc_attach).
 * Errors: ORCHA_E_ARG (NCCL communicator, packet of another grid, packet not
 * holding exactly the rank's blocks), ORCHA_E_RANGE, ORCHA_E_CUDA. */
int32_t orcha_comm_peer_register(orcha_comm* comm, orcha_packet* packet, void* stream);
/* Build (and cache) the guard-fill plan of a packet set -- neighbour, push and
 * exchange tables, uploaded with synchronous copies -- without filling.
 * orcha_fill_guardcells builds it on first use anyway; call this first where
 * a device allocation in the middle of a step would serialise streams (CUDA's
 * implicit synchronisation): peer mode with virtual ranks on one device must
 * prepare every rank after all have registered, before the first step.
 * Errors: as orcha_fill_guardcells. */
int32_t orcha_fill_prepare(orcha_packet* const* packets, int32_t npackets, orcha_comm* comm);
/* F2 peer mode between PROCESSES (one per GPU of a node, or several sharing
 * one GPU), no NCCL: orcha_comm_create_ipc makes rank `rank`'s communicator;
 * orcha_comm_ipc_export writes this rank's blob -- CUDA IPC handles of its
 * packet's state allocation (+ offset), its dt gather buffer and its barrier
 * counter, and the packet's block ids (packet = ONE packet holding every
 * block the rank owns; blob = NULL queries *size); the caller exchanges the
 * blobs (e.g. torch.distributed all_gather over gloo) and passes all of them,
 * in rank order, `stride` bytes apart, to orcha_comm_ipc_attach, which maps
 * the other ranks' memory (cudaIpcOpenMemHandle with lazy peer access) and
 * enters peer mode: from then on the calls behave exactly as for a LOCAL
 * communicator in peer mode (above) -- direct reads of other ranks' rows,
 * x-guard writes into them, device barriers over the mapped counters, the
 * one-shot peer dt.  Call orcha_fill_prepare after attaching.
 * Errors: ORCHA_E_ARG (bad blob, packet not holding exactly the rank's
 * blocks), ORCHA_E_RANGE, ORCHA_E_STATE (call order), ORCHA_E_CUDA (IPC). */
int32_t orcha_comm_create_ipc(const orcha_grid* grid, int32_t nranks, int32_t rank, const int32_t* block_owner,
                              orcha_comm** out);
int32_t orcha_comm_ipc_export(orcha_comm* comm, orcha_packet* packet, void* blob, size_t cap, size_t* size);
int32_t orcha_comm_ipc_attach(orcha_comm* comm, const void* blobs, size_t stride);
/* ORCHA_E_STATE if a peer barrier of this communicator timed out (device flag;
 * synchronizes), else ORCHA_OK. */
int32_t orcha_comm_check(orcha_comm* comm);

/* Host-only view of the guard exchange plan between `rank` and `peer` (no
 * device work; for tests and tooling).  The plan is a pure function of the
 * grid and block_owner: the cells rank SENDS to peer are the sorted unique
 * global cell indices g of its interior cells that peer's guards read; the
 * cells it RECEIVES from peer are the same list computed on the other side;
 * each remote guard of `rank` then takes value recv[idx] (negated in the
 * momentum components set in flip, reflect boundaries).
 * which: 0 = send cells (int64 g), 1 = receive cells (int64 g),
 *        2 = receiving guards (int64: dst block id * P^3 + padded cell index),
 *        3 = index into the receive cells (int64), 4 = flip bits (int64).
 * out may be NULL to query *count; otherwise up to cap entries are written.
 * Errors: ORCHA_E_ARG, ORCHA_E_RANGE (owner out of range). */
int32_t orcha_comm_plan(const orcha_grid* grid, int32_t nranks, int32_t rank, const int32_t* block_owner,
                        int32_t peer, int32_t which, int64_t* out, int64_t cap, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* ORCHA_H */
