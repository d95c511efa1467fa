"""Thin Python objects over the C ABI (include/orcha.h).

PyTorch supplies only device memory (caller-owned buffers handed to the
library as raw pointers) and streams; every step of the hot path runs in the
library's kernels.  Function names mirror the C entry points.
"""
from __future__ import annotations

import ctypes
import math
from typing import Optional, Sequence

import numpy as np
import torch

from . import abi


def _stream_ptr(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Grid:
    """A global grid of nblk blocks of nb cells with ng guard cells."""

    def __init__(self, ndim: int, nb: Sequence[int], nblk: Sequence[int], ng: int = 4,
                 xmin=(0.0, 0.0, 0.0), xmax=(1.0, 1.0, 1.0), bc=((0, 0), (0, 0), (0, 0)),
                 gamma: float = 1.4, cfl: float = 0.4, smallp: float = 1e-30, parity: bool = False,
                 riemann: int = abi.RIEMANN_HLL, limiter: int = abi.LIMITER_MINMOD,
                 eos: int = abi.EOS_GAMMA_LAW, eos_work: int = 1, arad: float = 0.0):
        self.lib = abi.load(parity)
        self.parity = parity
        nb = list(nb) + [1] * (3 - len(nb))
        nblk = list(nblk) + [1] * (3 - len(nblk))
        d = abi.orcha_grid_desc()
        d.ndim = ndim
        for a in range(3):
            d.nb[a] = int(nb[a])
            d.nblk[a] = int(nblk[a])
            d.xmin[a] = float(xmin[a]) if a < len(xmin) else 0.0
            d.xmax[a] = float(xmax[a]) if a < len(xmax) else 1.0
            d.bc[a][0] = int(bc[a][0])
            d.bc[a][1] = int(bc[a][1])
        d.ng = ng
        d.gamma, d.cfl, d.smallp = gamma, cfl, smallp
        d.riemann, d.limiter = int(riemann), int(limiter)
        d.eos, d.eos_work, d.arad = int(eos), int(eos_work), float(arad)
        self.riemann, self.limiter = int(riemann), int(limiter)
        self.eos, self.eos_work, self.arad = int(eos), int(eos_work), float(arad)
        self.desc = d
        self.ndim, self.nb, self.nblk, self.ng = ndim, tuple(nb), tuple(nblk), ng
        self.N = tuple(nb[a] * nblk[a] for a in range(3))
        h = ctypes.c_void_p()
        abi.call(self.lib, "orcha_grid_create", ctypes.byref(d), ctypes.byref(h))
        self.handle = h
        self.nblocks = int(self.lib.orcha_grid_nblocks(h))

    def __del__(self):
        if getattr(self, "handle", None):
            self.lib.orcha_grid_destroy(self.handle)
            self.handle = None

    def packet_bytes(self, nblocks: int):
        sb, xb = ctypes.c_size_t(), ctypes.c_size_t()
        abi.call(self.lib, "orcha_packet_bytes", self.handle, nblocks, ctypes.byref(sb), ctypes.byref(xb))
        return sb.value, xb.value


class Packet:
    """N blocks of the grid in caller-owned device memory (torch tensors)."""

    def __init__(self, grid: Grid, block_ids: Sequence[int], device="cuda"):
        self.grid = grid
        self.lib = grid.lib
        self.block_ids = np.ascontiguousarray(block_ids, dtype=np.int64)
        n = len(self.block_ids)
        sb, xb = grid.packet_bytes(n)
        self.state = torch.empty(sb, dtype=torch.uint8, device=device)
        self.scratch = torch.empty(xb, dtype=torch.uint8, device=device)
        h = ctypes.c_void_p()
        abi.call(self.lib, "orcha_packet_create", grid.handle, n,
                 self.block_ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                 ctypes.c_void_p(self.state.data_ptr()), ctypes.c_void_p(self.scratch.data_ptr()),
                 ctypes.byref(h))
        self.handle = h
        self.nblocks = n
        cb = ctypes.c_size_t()
        ext = (ctypes.c_int32 * 3)()
        abi.call(self.lib, "orcha_packet_layout", h, None, ctypes.byref(cb), ext)
        self.cube_doubles = cb.value // 8
        self.padded = tuple(ext)
        self.interior_shape = (n, 5, grid.nb[2], grid.nb[1], grid.nb[0])

    def __del__(self):
        if getattr(self, "handle", None):
            self.lib.orcha_packet_destroy(self.handle)
            self.handle = None

    # --- pack / unpack (packet moved as one flattened buffer) ---
    def pack(self, interior, stream=None):
        """interior: (nblocks, 5, nbz, nby, nbx) float64, numpy (host) or torch (host or device)."""
        if isinstance(interior, np.ndarray):
            a = np.ascontiguousarray(interior, dtype=np.float64)
            assert a.shape == self.interior_shape, (a.shape, self.interior_shape)
            abi.call(self.lib, "orcha_packet_pack", self.handle, ctypes.c_void_p(a.ctypes.data),
                     ctypes.c_void_p(_stream_ptr(stream)))
            torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
            return
        t = interior
        assert t.dtype == torch.float64 and t.is_contiguous() and tuple(t.shape) == self.interior_shape
        name = "orcha_packet_pack_device" if t.is_cuda else "orcha_packet_pack"
        abi.call(self.lib, name, self.handle, ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(_stream_ptr(stream)))

    def unpack(self, out=None, stream=None, sync: bool = True) -> np.ndarray:
        """Interior data of the packet's blocks.  sync=False (torch pinned-host
        or device `out` only): orcha_packet_unpack_async, enqueued on `stream`
        without the status check."""
        if not sync:
            assert isinstance(out, torch.Tensor) and (out.is_cuda or out.is_pinned())
            abi.call(self.lib, "orcha_packet_unpack_async", self.handle, ctypes.c_void_p(out.data_ptr()),
                     ctypes.c_void_p(_stream_ptr(stream)))
            return out
        if out is None:
            out = np.empty(self.interior_shape, dtype=np.float64)
        if isinstance(out, np.ndarray):
            abi.call(self.lib, "orcha_packet_unpack", self.handle, ctypes.c_void_p(out.ctypes.data),
                     ctypes.c_void_p(_stream_ptr(stream)))
            return out
        name = "orcha_packet_unpack_device" if out.is_cuda else "orcha_packet_unpack"
        abi.call(self.lib, name, self.handle, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream_ptr(stream)))
        return out

    def state_view(self) -> torch.Tensor:
        """(nblocks, 5, Pz, Py, Px) float64 view of the padded state incl. guards."""
        P = self.padded
        cells = P[0] * P[1] * P[2]
        v = self.state.view(torch.float64).view(self.nblocks, 5, self.cube_doubles)[:, :, :cells]
        return v.reshape(self.nblocks, 5, P[2], P[1], P[0])

    def counters(self, stream=None):
        fh, fb = ctypes.c_int64(), ctypes.c_int64()
        abi.call(self.lib, "orcha_packet_counters", self.handle, ctypes.byref(fh), ctypes.byref(fb),
                 ctypes.c_void_p(_stream_ptr(stream)))
        return fh.value, fb.value


def brick_owner(nblk: Sequence[int], brick: Sequence[int], gpu_grid: Sequence[int]) -> np.ndarray:
    """block -> rank for a grid of bricks (rank = (rz*py + ry)*px + rx), int32[nblocks]."""
    nblk = list(nblk) + [1] * (3 - len(nblk))
    brick = list(brick) + [1] * (3 - len(brick))
    px, py = gpu_grid[0], gpu_grid[1]
    b = np.arange(nblk[0] * nblk[1] * nblk[2], dtype=np.int64)
    bi, bj, bk = b % nblk[0], (b // nblk[0]) % nblk[1], b // (nblk[0] * nblk[1])
    return ((bk // brick[2]) * (px * py) + (bj // brick[1]) * px + bi // brick[0]).astype(np.int32)


class Comm:
    """Communicator for blocks partitioned over ranks (include/orcha.h)."""

    def __init__(self, grid: Grid, handle, nranks: int, rank: int, owner: np.ndarray):
        self.grid, self.lib, self.handle = grid, grid.lib, handle
        self.nranks, self.rank, self.owner = nranks, rank, owner

    @staticmethod
    def create(grid: Grid, nranks: int, rank: int, owner) -> "Comm":
        """NCCL communicator; the 128-byte unique id is broadcast with torch.distributed."""
        import torch.distributed as dist
        owner = np.ascontiguousarray(owner, dtype=np.int32)
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            abi.call(grid.lib, "orcha_comm_unique_id", uid)
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, 0)
        uid = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        h = ctypes.c_void_p()
        abi.call(grid.lib, "orcha_comm_create", grid.handle, uid, nranks, rank,
                 owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(h))
        return Comm(grid, h, nranks, rank, owner)

    @staticmethod
    def create_local(grid: Grid, nranks: int, owner) -> list:
        """Virtual ranks on one device (device-copy transport), for tests."""
        owner = np.ascontiguousarray(owner, dtype=np.int32)
        hs = (ctypes.c_void_p * nranks)()
        abi.call(grid.lib, "orcha_comm_create_local", grid.handle, nranks,
                 owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), hs)
        return [Comm(grid, ctypes.c_void_p(hs[r]), nranks, r, owner) for r in range(nranks)]

    @staticmethod
    def create_ipc(grid: Grid, nranks: int, rank: int, owner) -> "Comm":
        """F2 peer mode across processes (CUDA IPC; no NCCL): export, exchange, attach."""
        owner = np.ascontiguousarray(owner, dtype=np.int32)
        h = ctypes.c_void_p()
        abi.call(grid.lib, "orcha_comm_create_ipc", grid.handle, nranks, rank,
                 owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(h))
        return Comm(grid, h, nranks, rank, owner)

    def ipc_export(self, packet) -> bytes:
        n = ctypes.c_size_t()
        abi.call(self.lib, "orcha_comm_ipc_export", self.handle, packet.handle, None, 0, ctypes.byref(n))
        buf = ctypes.create_string_buffer(n.value)
        abi.call(self.lib, "orcha_comm_ipc_export", self.handle, packet.handle, buf, n.value, ctypes.byref(n))
        return buf.raw[:n.value]

    def ipc_attach(self, blobs) -> None:
        """blobs: every rank's export, in rank order."""
        stride = max(len(b) for b in blobs)
        raw = b"".join(b.ljust(stride, b"\0") for b in blobs)
        buf = ctypes.create_string_buffer(raw, len(raw))
        abi.call(self.lib, "orcha_comm_ipc_attach", self.handle, buf, stride)

    def push(self, packets, stream=None, buffer: int = 0):
        arr, n = _handles(packets)
        abi.call(self.lib, "orcha_comm_push", self.handle, arr, n, int(buffer), ctypes.c_void_p(_stream_ptr(stream)))

    def peer_register(self, packet, stream=None):
        """F2 peer mode: this rank's one packet becomes addressable by the other ranks."""
        abi.call(self.lib, "orcha_comm_peer_register", self.handle, packet.handle,
                 ctypes.c_void_p(_stream_ptr(stream)))

    def check(self):
        abi.call(self.lib, "orcha_comm_check", self.handle)

    def push_dt(self, packets, stream=None):
        """LOCAL transport: publish this virtual rank's dt record to every member."""
        arr, n = _handles(packets)
        abi.call(self.lib, "orcha_comm_push_dt", self.handle, arr, n, ctypes.c_void_p(_stream_ptr(stream)))

    def destroy(self):
        if self.handle:
            self.lib.orcha_comm_destroy(self.handle)
            self.handle = None


def comm_plan(grid: Grid, nranks: int, rank: int, owner, peer: int, which: int) -> np.ndarray:
    """Host-only exchange plan query (orcha_comm_plan); no device needed."""
    owner = np.ascontiguousarray(owner, dtype=np.int32)
    op = owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    n = ctypes.c_int64()
    abi.call(grid.lib, "orcha_comm_plan", grid.handle, nranks, rank, op, peer, which, None, 0, ctypes.byref(n))
    out = np.empty(n.value, dtype=np.int64)
    abi.call(grid.lib, "orcha_comm_plan", grid.handle, nranks, rank, op, peer, which,
             out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n.value, ctypes.byref(n))
    return out


def _handles(packets):
    arr = (ctypes.c_void_p * len(packets))(*[p.handle.value for p in packets])
    return arr, len(packets)


def orcha_fill_guardcells(packets, comm=None, stream=None):
    arr, n = _handles(packets)
    lib = packets[0].lib
    abi.call(lib, "orcha_fill_guardcells", arr, n, comm.handle if comm is not None else None,
             ctypes.c_void_p(_stream_ptr(stream)))


def orcha_hydro_step_overlap(packet: Packet, comm, clock: DevClock, stream=None):
    """One step with the halo exchange overlapping stage 1 of the interior slots."""
    abi.call(packet.lib, "orcha_hydro_step_overlap", packet.handle, comm.handle, ctypes.c_void_p(clock.ptr),
             ctypes.c_void_p(_stream_ptr(stream)))


def interior_first(nblk: Sequence[int], bc, owner, rank: int, ndim: int = 3) -> np.ndarray:
    """The block ids `rank` owns, ordered interior-first: blocks whose 26
    neighbours (periodic wrap; a clamp / mirror side counts as the block
    itself) are all owned by `rank` come first (ascending id), then the
    rest.  Host bookkeeping for orcha_hydro_step_overlap."""
    nblk = list(nblk) + [1] * (3 - len(nblk))
    owner = np.asarray(owner)
    ids = np.flatnonzero(owner == rank)
    inner, outer = [], []
    for b in ids:
        c0 = [b % nblk[0], (b // nblk[0]) % nblk[1], b // (nblk[0] * nblk[1])]
        ok = True
        for oz in (-1, 0, 1):
            for oy in (-1, 0, 1):
                for ox in (-1, 0, 1):
                    o = (ox, oy, oz)
                    if any(o[a] != 0 for a in range(ndim, 3)):
                        continue
                    c = []
                    for a in range(3):
                        x = c0[a] + o[a]
                        if x < 0 or x >= nblk[a]:
                            x = x % nblk[a] if bc[a][0 if x < 0 else 1] == abi.BC_PERIODIC else c0[a]
                        c.append(x)
                    nbk = (c[2] * nblk[1] + c[1]) * nblk[0] + c[0]
                    ok &= bool(owner[nbk] == rank)
        (inner if ok else outer).append(int(b))
    return np.array(inner + outer, dtype=np.int64)


def orcha_fill_prepare(packets, comm=None):
    arr, n = _handles(packets)
    abi.call(packets[0].lib, "orcha_fill_prepare", arr, n, comm.handle if comm is not None else None)


def orcha_fill_guardcells_packet(packets, index: int, stream=None):
    """Guards of packets[index] only, with the set's tables (streamed packets)."""
    arr, n = _handles(packets)
    abi.call(packets[0].lib, "orcha_fill_guardcells_packet", arr, n, int(index), ctypes.c_void_p(_stream_ptr(stream)))


def orcha_packet_dt_records(packet: Packet, stream=None):
    """The packet's CFL records now (the local part of orcha_compute_dt)."""
    abi.call(packet.lib, "orcha_packet_dt_records", packet.handle, ctypes.c_void_p(_stream_ptr(stream)))


def orcha_compute_dt(packets, t_remaining: float = math.inf, comm=None, stream=None, check: bool = True):
    arr, n = _handles(packets)
    lib = packets[0].lib
    info = abi.orcha_dt_info()
    rc = lib.orcha_compute_dt(arr, n, comm.handle if comm is not None else None, float(t_remaining),
                              ctypes.byref(info), ctypes.c_void_p(_stream_ptr(stream)))
    if check:
        abi.check(lib, rc, "orcha_compute_dt")
    return info


def orcha_hydro_advance(packet: Packet, dt: float, stream=None):
    abi.call(packet.lib, "orcha_hydro_advance", packet.handle, float(dt), ctypes.c_void_p(_stream_ptr(stream)))


class DevClock:
    """orcha_dev_clock in device memory (a 64-byte torch buffer): t, t_end
    set here; orcha_compute_dt_device writes dt and advances t on the device."""

    def __init__(self, t: float = 0.0, t_end: float = math.inf, device="cuda"):
        assert ctypes.sizeof(abi.orcha_dev_clock) == 64
        self.buf = torch.zeros(8, dtype=torch.float64, device=device)
        self.buf[0] = t
        self.buf[1] = t_end

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    @property
    def dt_tensor(self) -> torch.Tensor:
        return self.buf[2:3]  # &clock->dt, for orcha_hydro_advance_devdt

    def read(self) -> "abi.orcha_dev_clock":
        h = self.buf.cpu().numpy().tobytes()
        return abi.orcha_dev_clock.from_buffer_copy(h)


def orcha_compute_dt_device(packets, clock: DevClock, comm=None, stream=None):
    arr, n = _handles(packets)
    abi.call(packets[0].lib, "orcha_compute_dt_device", arr, n, comm.handle if comm is not None else None,
             ctypes.c_void_p(clock.ptr), ctypes.c_void_p(_stream_ptr(stream)))


def orcha_hydro_advance_devdt(packet: Packet, d_dt: torch.Tensor, stream=None):
    assert d_dt.dtype == torch.float64 and d_dt.is_cuda
    abi.call(packet.lib, "orcha_hydro_advance_devdt", packet.handle, ctypes.c_void_p(d_dt.data_ptr()),
             ctypes.c_void_p(_stream_ptr(stream)))


def set_kernel_variant(lib, v: int):
    abi.call(lib, "orcha_set_kernel_variant", int(v))


def orcha_hydro_stage(packet: Packet, stage: int, dt: float, stream=None):
    abi.call(packet.lib, "orcha_hydro_stage", packet.handle, int(stage), float(dt),
             ctypes.c_void_p(_stream_ptr(stream)))


def orcha_fill_guardcells_stage(packets, buffer: int, comm=None, stream=None):
    arr, n = _handles(packets)
    abi.call(packets[0].lib, "orcha_fill_guardcells_stage", arr, n, comm.handle if comm is not None else None,
             int(buffer), ctypes.c_void_p(_stream_ptr(stream)))


def step(packets, dt: float, comm=None, stream=None, method: str = "telescoped"):
    """One RK2 step after the state's guard fill: telescoped (the paper's
    communication-avoiding step) or per-stage (F1: refill U1's
    guards between the stages)."""
    if method == "telescoped":
        for p in packets:
            orcha_hydro_advance(p, dt, stream)
    elif method == "per-stage":
        # the caller's state fill may be the full one or the per-stage one
        for p in packets:
            orcha_hydro_stage(p, 1, dt, stream)
        orcha_fill_guardcells_stage(packets, 1, comm, stream)
        for p in packets:
            orcha_hydro_stage(p, 2, dt, stream)
    else:
        raise ValueError(method)


def orcha_hydro_stage_devdt(packet: Packet, stage: int, d_dt: torch.Tensor, stream=None):
    assert d_dt.dtype == torch.float64 and d_dt.is_cuda
    abi.call(packet.lib, "orcha_hydro_stage_devdt", packet.handle, int(stage), ctypes.c_void_p(d_dt.data_ptr()),
             ctypes.c_void_p(_stream_ptr(stream)))


def step_devdt(packets, d_dt: torch.Tensor, comm=None, stream=None, method: str = "telescoped"):
    """step() with dt read from device memory (e.g. DevClock.dt_tensor)."""
    if method == "telescoped":
        for p in packets:
            orcha_hydro_advance_devdt(p, d_dt, stream)
    elif method == "per-stage":
        for p in packets:
            orcha_hydro_stage_devdt(p, 1, d_dt, stream)
        orcha_fill_guardcells_stage(packets, 1, comm, stream)
        for p in packets:
            orcha_hydro_stage_devdt(p, 2, d_dt, stream)
    else:
        raise ValueError(method)


def run(packets, nsteps: Optional[int] = None, t_end: float = math.inf, comm=None, stream=None,
        method: str = "telescoped"):
    """The driver loop of SURVEY 8(c): fill -> dt (then t_end clamp) -> step,
    every call through the C ABI.  Returns (t, steps, [dt_info...])."""
    t = 0.0
    log = []
    n = 0
    while (nsteps is None or n < nsteps) and t < t_end:
        if method == "per-stage":
            orcha_fill_guardcells_stage(packets, 0, comm, stream)
        else:
            orcha_fill_guardcells(packets, comm, stream)
        info = orcha_compute_dt(packets, t_end - t, comm, stream)
        step(packets, info.dt, comm, stream, method)
        t = t + info.dt
        n += 1
        log.append((info.dt, info.smax, info.argmax, info.tag))
    return t, n, log


def run_device(packets, nsteps: int, t_end: float = math.inf, comm=None, stream=None, record: bool = True,
               method: str = "telescoped"):
    """The same loop with dt kept on the device (orcha_compute_dt_device ->
    the *_devdt step calls): no host synchronization per step.  Returns (clock, log) -- log = [(dt, smax, argmax, tag)] per step,
    read after the loop (record=False: none)."""
    clock = DevClock(0.0, t_end)
    s = stream if stream is not None else torch.cuda.current_stream()
    hist = torch.empty((nsteps, 8), dtype=torch.float64, device=clock.buf.device) if record else None
    for n in range(nsteps):
        if method == "per-stage":
            orcha_fill_guardcells_stage(packets, 0, comm, s)
        else:
            orcha_fill_guardcells(packets, comm, s)
        orcha_compute_dt_device(packets, clock, comm, s)
        step_devdt(packets, clock.dt_tensor, comm, s, method)
        if record:
            with torch.cuda.stream(s):
                hist[n].copy_(clock.buf)
    s.synchronize()
    log = []
    if record:
        for row in hist.cpu().numpy():
            c = abi.orcha_dev_clock.from_buffer_copy(row.tobytes())
            log.append((c.dt, c.smax, c.argmax, c.tag))
    return clock, log


def capture_steps(packets, clock: DevClock, nsteps: int, comm=None, method: str = "telescoped"):
    """A CUDA graph of `nsteps` device-dt time steps (fill -> orcha_compute_dt_device
    -> *_devdt step): the host state machine must be in steady state (call
    this after at least one plain device-dt step, so the fill launches
    nothing new and every kernel's attributes are set); each replay advances
    the packets and the device clock by `nsteps` steps (run two plain steps
    after a pack first: the first one's dt records come from the dt kernel,
    later ones from the fused epilogue).  Single rank only (NCCL
    calls inside a capture need a graph-aware communicator)."""
    assert comm is None, "capture_steps: single rank"
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=side):
        for _ in range(nsteps):
            if method == "per-stage":
                orcha_fill_guardcells_stage(packets, 0, None, side)
            else:
                orcha_fill_guardcells(packets, None, side)
            orcha_compute_dt_device(packets, clock, None, side)
            step_devdt(packets, clock.dt_tensor, None, side, method)
    torch.cuda.current_stream().wait_stream(side)
    return g


# ---- unit entry points (test diagnostics; include/orcha.h "unit entry points")
def _dev_f64(a) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def orcha_unit_eos(grid: Grid, U: np.ndarray):
    """U: (5, n) conserved -> (Q (5, n) primitives, c (n,), s (n,), floored (n,))."""
    n = U.shape[1]
    dU = _dev_f64(U)
    dQ = torch.empty((5, n), dtype=torch.float64, device="cuda")
    dc = torch.empty(n, dtype=torch.float64, device="cuda")
    ds = torch.empty(n, dtype=torch.float64, device="cuda")
    df = torch.empty(n, dtype=torch.int32, device="cuda")
    abi.call(grid.lib, "orcha_unit_eos", grid.handle, n, ctypes.c_void_p(dU.data_ptr()),
             ctypes.c_void_p(dQ.data_ptr()), ctypes.c_void_p(dc.data_ptr()), ctypes.c_void_p(ds.data_ptr()),
             ctypes.c_void_p(df.data_ptr()), ctypes.c_void_p(_stream_ptr(None)))
    torch.cuda.synchronize()
    return dQ.cpu().numpy(), dc.cpu().numpy(), ds.cpu().numpy(), df.cpu().numpy()


def orcha_unit_face_flux(grid: Grid, d: int, q: np.ndarray) -> np.ndarray:
    """q: (4, 5, n) primitives of cells i-1 .. i+2 along d -> F (5, n) at i+1/2."""
    n = q.shape[2]
    dq = _dev_f64(q)
    dF = torch.empty((5, n), dtype=torch.float64, device="cuda")
    abi.call(grid.lib, "orcha_unit_face_flux", grid.handle, int(d), n, ctypes.c_void_p(dq.data_ptr()),
             ctypes.c_void_p(dF.data_ptr()), ctypes.c_void_p(_stream_ptr(None)))
    torch.cuda.synchronize()
    return dF.cpu().numpy()


def orcha_unit_riemann(grid: Grid, d: int, qL: np.ndarray, qR: np.ndarray) -> np.ndarray:
    """qL, qR: (5, n) face-state primitives -> F (5, n)."""
    n = qL.shape[1]
    a, b = _dev_f64(qL), _dev_f64(qR)
    dF = torch.empty((5, n), dtype=torch.float64, device="cuda")
    abi.call(grid.lib, "orcha_unit_riemann", grid.handle, int(d), n, ctypes.c_void_p(a.data_ptr()),
             ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(dF.data_ptr()), ctypes.c_void_p(_stream_ptr(None)))
    torch.cuda.synchronize()
    return dF.cpu().numpy()


# ---- instrumentation (include/orcha.h "per-phase instrumentation")
def orcha_set_phase_timing(lib, on: bool):
    abi.call(lib, "orcha_set_phase_timing", 1 if on else 0)


def orcha_phase_times(lib) -> dict:
    """{phase: (ms summed since the last query, occurrences)} (synchronizes)."""
    ms = (ctypes.c_double * 6)()
    cnt = (ctypes.c_int64 * 6)()
    abi.call(lib, "orcha_phase_times", ms, cnt, 6)
    return {name: (ms[i], cnt[i]) for i, name in enumerate(abi.PHASES)}


def orcha_probe_fp64(lib, iters: int = 20000, stream=None):
    """Measured fp64 DFMA thread-instructions/s / 1e12 and the probe kernel's ms."""
    t, ms = ctypes.c_double(), ctypes.c_double()
    abi.call(lib, "orcha_probe_fp64", int(iters), ctypes.byref(t), ctypes.byref(ms), ctypes.c_void_p(_stream_ptr(stream)))
    return t.value, ms.value


# ---- mesh checksums and dump
VAR_NAMES = ("rho", "rho_u", "rho_v", "rho_w", "E")


def fnv1a64(lib, data: bytes, h: int = abi.FNV1A64_OFFSET) -> int:
    hv = ctypes.c_uint64(h)
    buf = ctypes.create_string_buffer(data, len(data))
    abi.call(lib, "orcha_fnv1a64", ctypes.cast(buf, ctypes.c_void_p), len(data), ctypes.byref(hv))
    return hv.value


def _blocks_by_id(packets):
    """{global block id: (5, nbz, nby, nbx) interior} over the packets (unpack, synchronizes)."""
    out = {}
    for p in packets:
        arr = p.unpack()
        for s, b in enumerate(p.block_ids):
            out[int(b)] = arr[s]
    return out


def mesh_checksums(packets, blocks=None) -> dict:
    """Per-variable FNV-1a 64 (hex) over the blocks in ascending global id,
    cells in (k, j, i) order, little-endian fp64: independent of the packet split."""
    lib = packets[0].lib
    blocks = blocks if blocks is not None else _blocks_by_id(packets)
    out = {}
    for v, name in enumerate(VAR_NAMES):
        h = abi.FNV1A64_OFFSET
        for b in sorted(blocks):
            h = fnv1a64(lib, np.ascontiguousarray(blocks[b][v], dtype="<f8").tobytes(), h)
        out[name] = f"{h:016x}"
    return out


def dump_mesh(path: str, packets, t: Optional[float] = None, step: Optional[int] = None) -> dict:
    """Raw mesh dump: `path`.bin = for each variable, for each block in
    ascending global id, its interior cells (k, j, i order) as little-endian
    fp64; `path`.json = the sidecar (dims, order, block ids, per-variable
    checksums).  Returns the sidecar."""
    import json
    g = packets[0].grid
    blocks = _blocks_by_id(packets)
    ids = sorted(blocks)
    with open(path + ".bin", "wb") as f:
        for v in range(5):
            for b in ids:
                f.write(np.ascontiguousarray(blocks[b][v], dtype="<f8").tobytes())
    side = {"format": "orcha-mesh-v1", "dtype": "<f8", "vars": list(VAR_NAMES),
            "order": "var, block (ascending global id b = (bk*NBy + bj)*NBx + bi), k, j, i",
            "ndim": g.ndim, "nb": list(g.nb), "nblk": list(g.nblk), "ng": g.ng, "N": list(g.N),
            "xmin": list(g.desc.xmin), "xmax": list(g.desc.xmax), "block_ids": ids,
            "checksums_fnv1a64": mesh_checksums(packets, blocks), "t": t, "step": step}
    with open(path + ".json", "w") as f:
        json.dump(side, f, indent=1)
    return side


def load_mesh(path: str):
    """Inverse of dump_mesh: (sidecar, {block id: (5, nbz, nby, nbx)})."""
    import json
    side = json.load(open(path + ".json"))
    nbz, nby, nbx = side["nb"][2], side["nb"][1], side["nb"][0]
    ids = side["block_ids"]
    raw = np.fromfile(path + ".bin", dtype="<f8").reshape(5, len(ids), nbz, nby, nbx)
    return side, {b: np.ascontiguousarray(raw[:, s]) for s, b in enumerate(ids)}
