"""CPU oracle for the ORCHA Sedov hydro hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2507_09337_b200``) never imports it and shares no code with it.

The arithmetic lives in ``orcha_oracle.c`` (plain C, fp64, compiled with
``-O2 -ffp-contract=off``; see its header for the passages of PAPER.md it
follows).  This module only compiles it, marshals numpy arrays in and out and
drives the time loop of SURVEY.md 8(c):

    per step: ghost fill -> dt (CFL, lowest-index argmax, then t_end clamp)
              -> telescoped SSP-RK2 step          (section 6)

Array convention: a global array of shape (5, Pz, Py, Px), variables
(rho, rho*u, rho*v, rho*w, E), P_d = N_d + 2*ng on active axes and 1 on
inactive ones, i fastest.

Parity status: every function here is pinned by
tests/test_oracle_*.py; the one unpinned aspect is agreement with Flash-X's
Spark solver itself ("parity unpinned": the paper prints no solution values
and does not name Spark's reconstruction or Riemann solver).
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "orcha_oracle.c")
_LIB = os.path.join(_HERE, "liborcha_oracle.so")
_LIB_OMP = os.path.join(_HERE, "liborcha_oracle_omp.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]

OUTFLOW, PERIODIC, REFLECT = 0, 1, 2
HLL, HLLC = 0, 1          # Riemann solver flag
MINMOD, MC = 0, 1         # limiter flag
GAMMA_LAW, GAS_RADIATION = 0, 1   # EOS flag (SURVEY 8(f) F4 expensive-EOS surrogate)
TAG_CFL, TAG_CLAMP = 0, 1


def build(force: bool = False, omp: bool = False) -> str:
    """Compile the oracle shared library (gcc) if it is missing or stale;
    omp=True: the same source with -fopenmp ("oracle-omp", bitwise the same
    results)."""
    lib = _LIB_OMP if omp else _LIB
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(_SRC):
        tmp = lib + f".{os.getpid()}.tmp"
        subprocess.run(["gcc", *CFLAGS, *(["-fopenmp"] if omp else []), "-o", tmp, _SRC, "-lm"], check=True)
        os.replace(tmp, lib)
    return lib


def use_threads(n: int) -> int:
    """Switch this process's oracle to the -fopenmp build with n threads
    (n <= 1: back to the plain build).  Returns the thread count in use."""
    global _lib
    _lib = None
    _load(omp=n > 1)
    return _lib.oracle_set_threads(int(n)) if n > 1 else 1


class _CGrid(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("N", ctypes.c_int32 * 3),
        ("ng", ctypes.c_int32),
        ("xmin", ctypes.c_double * 3),
        ("xmax", ctypes.c_double * 3),
        ("bc", (ctypes.c_int32 * 2) * 3),
        ("gamma", ctypes.c_double),
        ("cfl", ctypes.c_double),
        ("smallp", ctypes.c_double),
        ("riemann", ctypes.c_int32),
        ("limiter", ctypes.c_int32),
        ("eos", ctypes.c_int32),
        ("eos_work", ctypes.c_int32),
        ("arad", ctypes.c_double),
    ]


_lib = None


def _load(omp: bool = False):
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build(omp=omp))
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        lib.oracle_set_threads.restype = ctypes.c_int
        P = ctypes.POINTER
        d = ctypes.c_double
        dp = P(d)
        g = P(_CGrid)
        lib.oracle_array_len.argtypes = [g]
        lib.oracle_array_len.restype = ctypes.c_int64
        lib.oracle_fill_ghosts.argtypes = [g, dp]
        lib.oracle_fill_ghosts.restype = ctypes.c_int
        lib.oracle_prim.argtypes = [g, dp, dp]
        lib.oracle_prim.restype = ctypes.c_int
        lib.oracle_sound_speed.argtypes = [g, dp]
        lib.oracle_sound_speed.restype = d
        lib.oracle_minmod_slope.argtypes = [d, d, d]
        lib.oracle_minmod_slope.restype = d
        lib.oracle_hll.argtypes = [g, ctypes.c_int, dp, dp, dp]
        lib.oracle_hll.restype = None
        lib.oracle_hllc.argtypes = [g, ctypes.c_int, dp, dp, dp]
        lib.oracle_hllc.restype = None
        lib.oracle_mc_slope.argtypes = [d, d, d]
        lib.oracle_mc_slope.restype = d
        lib.oracle_eint_from_p.argtypes = [g, d, d]
        lib.oracle_eint_from_p.restype = d
        lib.oracle_face_flux.argtypes = [g, ctypes.c_int, dp, dp, dp, dp, dp]
        lib.oracle_face_flux.restype = None
        lib.oracle_dt.argtypes = [g, dp, d, dp, P(ctypes.c_int64), P(ctypes.c_int32), dp]
        lib.oracle_dt.restype = ctypes.c_int
        lib.oracle_step.argtypes = [g, dp, d, ctypes.c_int32, dp, P(ctypes.c_int64)]
        lib.oracle_step.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclasses.dataclass
class Grid:
    """Global uniform grid (SURVEY 8(b) orcha_grid_desc without the blocking)."""

    N: Tuple[int, ...]                      # interior cells per active axis
    ng: int = 4
    xmin: Tuple[float, ...] = (0.0, 0.0, 0.0)
    xmax: Tuple[float, ...] = (1.0, 1.0, 1.0)
    bc: Tuple[Tuple[int, int], ...] = ((OUTFLOW, OUTFLOW),) * 3
    gamma: float = 1.4
    cfl: float = 0.4
    smallp: float = 1e-30
    riemann: int = HLL                      # F4: HLL (default) or HLLC
    limiter: int = MINMOD                   # F4: minmod (default) or MC
    eos: int = GAMMA_LAW                    # F4: gamma law (default) or gas + radiation (Newton)
    eos_work: int = 1                       # F4: temperature solves per EOS evaluation
    arad: float = 0.0                       # F4: radiation constant a

    @property
    def ndim(self) -> int:
        return len(self.N)

    @property
    def N3(self) -> Tuple[int, int, int]:
        return tuple(list(self.N) + [1] * (3 - self.ndim))  # type: ignore

    @property
    def shape(self) -> Tuple[int, int, int, int]:
        """Padded array shape (5, Pz, Py, Px)."""
        P = [n + 2 * self.ng if d < self.ndim else 1 for d, n in enumerate(self.N3)]
        return (5, P[2], P[1], P[0])

    @property
    def interior(self) -> Tuple[slice, ...]:
        g = self.ng
        sl = [slice(g, g + n) if d < self.ndim else slice(0, 1) for d, n in enumerate(self.N3)]
        return (slice(None), sl[2], sl[1], sl[0])

    def c(self) -> _CGrid:
        cg = _CGrid()
        cg.ndim = self.ndim
        for d in range(3):
            cg.N[d] = self.N3[d]
            cg.xmin[d] = float(self.xmin[d]) if d < len(self.xmin) else 0.0
            cg.xmax[d] = float(self.xmax[d]) if d < len(self.xmax) else 1.0
            cg.bc[d][0] = int(self.bc[d][0])
            cg.bc[d][1] = int(self.bc[d][1])
        cg.ng = self.ng
        cg.gamma = self.gamma
        cg.cfl = self.cfl
        cg.smallp = self.smallp
        cg.riemann = int(self.riemann)
        cg.limiter = int(self.limiter)
        cg.eos = int(self.eos)
        cg.eos_work = int(self.eos_work)
        cg.arad = float(self.arad)
        return cg


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def padded(grid: Grid, interior: np.ndarray) -> np.ndarray:
    """Global interior array (5, Nz, Ny, Nx) -> padded array, ghosts zero."""
    U = np.zeros(grid.shape, dtype=np.float64)
    U[grid.interior] = interior
    return U


def fill_ghosts(grid: Grid, U: np.ndarray) -> np.ndarray:
    rc = _load().oracle_fill_ghosts(ctypes.byref(grid.c()), _dp(U))
    if rc:
        raise ValueError(f"oracle_fill_ghosts: {rc}")
    return U


def prim(grid: Grid, u5: Sequence[float]) -> Tuple[np.ndarray, int]:
    u = np.ascontiguousarray(u5, dtype=np.float64)
    q = np.zeros(5)
    r = _load().oracle_prim(ctypes.byref(grid.c()), _dp(u), _dp(q))
    return q, r


def sound_speed(grid: Grid, q5: Sequence[float]) -> float:
    q = np.ascontiguousarray(q5, dtype=np.float64)
    return _load().oracle_sound_speed(ctypes.byref(grid.c()), _dp(q))


def minmod_slope(qm: float, q0: float, qp: float) -> float:
    return _load().oracle_minmod_slope(qm, q0, qp)


def eint_from_p(grid: Grid, rho: float, p: float) -> float:
    return _load().oracle_eint_from_p(ctypes.byref(grid.c()), rho, p)


def mc_slope(qm: float, q0: float, qp: float) -> float:
    return _load().oracle_mc_slope(qm, q0, qp)


def hllc(grid: Grid, d: int, qL: Sequence[float], qR: Sequence[float]) -> np.ndarray:
    a = np.ascontiguousarray(qL, dtype=np.float64)
    b = np.ascontiguousarray(qR, dtype=np.float64)
    F = np.zeros(5)
    _load().oracle_hllc(ctypes.byref(grid.c()), d, _dp(a), _dp(b), _dp(F))
    return F


def hll(grid: Grid, d: int, qL: Sequence[float], qR: Sequence[float]) -> np.ndarray:
    a = np.ascontiguousarray(qL, dtype=np.float64)
    b = np.ascontiguousarray(qR, dtype=np.float64)
    F = np.zeros(5)
    _load().oracle_hll(ctypes.byref(grid.c()), d, _dp(a), _dp(b), _dp(F))
    return F


def face_flux(grid: Grid, d: int, qm, q0, q1, q2) -> np.ndarray:
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (qm, q0, q1, q2)]
    F = np.zeros(5)
    _load().oracle_face_flux(ctypes.byref(grid.c()), d, *[_dp(a) for a in arrs], _dp(F))
    return F


@dataclasses.dataclass
class DtResult:
    dt: float
    argmax: int
    tag: int
    smax: float
    status: int


def compute_dt(grid: Grid, U: np.ndarray, t_remaining: float = math.inf) -> DtResult:
    dt = ctypes.c_double()
    am = ctypes.c_int64()
    tag = ctypes.c_int32()
    smax = ctypes.c_double()
    rc = _load().oracle_dt(ctypes.byref(grid.c()), _dp(U), t_remaining, ctypes.byref(dt),
                           ctypes.byref(am), ctypes.byref(tag), ctypes.byref(smax))
    return DtResult(dt.value, am.value, tag.value, smax.value, rc)


def step(grid: Grid, U: np.ndarray, dt: float, mode: str = "telescoped",
         U1_out: Optional[np.ndarray] = None) -> Tuple[int, int]:
    """One SSP-RK2 step in place.  Returns (status, floor_hits)."""
    m = {"telescoped": 0, "refill": 1}[mode]
    hits = ctypes.c_int64(0)
    u1 = _dp(U1_out) if U1_out is not None else None
    rc = _load().oracle_step(ctypes.byref(grid.c()), _dp(U), dt, m, u1, ctypes.byref(hits))
    return rc, hits.value


@dataclasses.dataclass
class RunLog:
    t: float
    steps: int
    dts: list
    argmax: list
    tags: list
    floor_hits: int


def run(grid: Grid, U: np.ndarray, nsteps: Optional[int] = None, t_end: float = math.inf,
        mode: str = "telescoped") -> RunLog:
    """Advance the padded array U in place: nsteps steps, or until t_end.

    Per step: fill ghosts, dt from U^n (then clamp to t_end - t),
    one RK2 step."""
    t = 0.0
    log = RunLog(0.0, 0, [], [], [], 0)
    n = 0
    while True:
        if nsteps is not None and n >= nsteps:
            break
        if t >= t_end:
            break
        fill_ghosts(grid, U)
        r = compute_dt(grid, U, t_end - t)
        if r.status:
            raise FloatingPointError(f"non-physical state before step {n}")
        rc, hits = step(grid, U, r.dt, mode)
        if rc:
            raise FloatingPointError(f"non-physical state in step {n}")
        t = t + r.dt
        n += 1
        log.dts.append(r.dt)
        log.argmax.append(r.argmax)
        log.tags.append(r.tag)
        log.floor_hits += hits
    log.t = t
    log.steps = n
    return log
