"""Seeded / closed-form synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no EOS, reconstruction, flux,
update or dt): only the initial conditions of the paper's workloads and
seeded random states.  It imports neither ``oracle`` nor the product package,
and both may import it.

Workloads (SURVEY.md 8(c) "Initial conditions", 8(d) configs):

* Sedov blast (sec 5.2: "a pressure spike at the center"):
  rho = 1, v = 0, E_blast = 1, p_amb = 1e-5, gamma = 1.4 on [0,1]^d (or the
  given box); the blast is deposited as uniform energy density
  E_blast / (n_D * dV) on the cells whose centres lie within 3.5 dx of the
  centre vertex, tested exactly on integers:
      sum_d (2*i_d + 1 - N_d)^2 < 49          (N_d even; reading c11)
  every other cell has E = p_amb * (1/(gamma-1)).
* Sod shock tube (Toro test 1): (rho, p) = (1, 1) for x_c < 0.5 and
  (0.125, 0.1) otherwise, v = 0, along a chosen axis.
* Random primitive states for unit fuzz: seed 20250709,
  rho ~ logU[1e-2, 1e2], p ~ logU[1e-6, 1e3], v ~ U[-3, 3] * sqrt(1.4 p / rho).

Arrays are global interiors of shape (5, Nz, Ny, Nx) (inactive axes size 1),
variables (rho, rho*u, rho*v, rho*w, E), float64, i fastest; block-major
packet order is produced by ``to_blocks`` (a pure reshape).
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np

SEED = 20250709


def _dims(N: Sequence[int]) -> Tuple[int, int, int]:
    N = list(N) + [1] * (3 - len(N))
    return int(N[0]), int(N[1]), int(N[2])


def sedov_deposit_mask(N: Sequence[int]) -> np.ndarray:
    """Boolean (Nz, Ny, Nx) mask of deposit cells: sum_d (2 i_d + 1 - N_d)^2 < 49."""
    nd = len(N)
    Nx, Ny, Nz = _dims(N)
    for n in N:
        if n % 2:
            raise ValueError("Sedov deposit needs even N on every active axis")
    r2 = np.zeros((Nz, Ny, Nx), dtype=np.int64)
    axes = [(Nx, 2), (Ny, 1), (Nz, 0)]
    for d in range(nd):
        n, ax = axes[d]
        a = (2 * np.arange(n, dtype=np.int64) + 1 - n) ** 2
        shape = [1, 1, 1]
        shape[ax] = n
        r2 = r2 + a.reshape(shape)
    return r2 < 49


def sedov(N: Sequence[int], xmin=(0.0, 0.0, 0.0), xmax=(1.0, 1.0, 1.0), gamma: float = 1.4,
          E_blast: float = 1.0, p_amb: float = 1e-5, rho0: float = 1.0) -> np.ndarray:
    nd = len(N)
    Nx, Ny, Nz = _dims(N)
    dx = [(xmax[d] - xmin[d]) / N[d] for d in range(nd)]
    dV = dx[0]
    for d in range(1, nd):
        dV = dV * dx[d]
    mask = sedov_deposit_mask(N)
    nD = int(mask.sum())
    U = np.zeros((5, Nz, Ny, Nx), dtype=np.float64)
    U[0] = rho0
    U[4] = p_amb * (1.0 / (gamma - 1.0))
    U[4][mask] = E_blast / (nD * dV)
    return U


def sedov_packet(N: Sequence[int], nb: Sequence[int], block_ids: Sequence[int], xmin=(0.0, 0.0, 0.0),
                 xmax=(1.0, 1.0, 1.0), gamma: float = 1.4, E_blast: float = 1.0, p_amb: float = 1e-5,
                 rho0: float = 1.0) -> np.ndarray:
    """The Sedov initial state restricted to the given blocks, directly in packet
    interior order (nblocks, 5, nbz, nby, nbx): bitwise equal to
    to_blocks(sedov(N, ...), nb, block_ids) without building the global array
    (a rank of the weak-scaling run only materialises its own brick)."""
    nd = len(N)
    Nx, Ny, Nz = _dims(N)
    bx, by, bz = _dims(nb)
    NBx, NBy = Nx // bx, Ny // by
    dx = [(xmax[d] - xmin[d]) / N[d] for d in range(nd)]
    dV = dx[0]
    for d in range(1, nd):
        dV = dV * dx[d]
    # deposit cells lie within 4 cells of the centre vertex on every axis
    lo = [n // 2 - 4 for n in (Nx, Ny, Nz)[:nd]]
    sub = [min(8, n) for n in (Nx, Ny, Nz)[:nd]]
    r2 = np.zeros([1, 1, 1][: 3 - nd] + list(reversed(sub)), dtype=np.int64)
    axes_len = list(reversed(sub))
    for d in range(nd):
        n = (Nx, Ny, Nz)[d]
        a = (2 * (np.arange(sub[d], dtype=np.int64) + lo[d]) + 1 - n) ** 2
        shape = [1, 1, 1]
        shape[2 - d] = sub[d]
        r2 = r2 + a.reshape(shape)
    for n in N:
        if n % 2:
            raise ValueError("Sedov deposit needs even N on every active axis")
    full = np.argwhere(r2.reshape([1] * (3 - len(axes_len)) + axes_len) < 49)
    nD = len(full)
    ids = np.asarray(block_ids, dtype=np.int64)
    out = np.empty((len(ids), 5, bz, by, bx), dtype=np.float64)
    out[:, 0] = rho0
    out[:, 1:4] = 0.0
    out[:, 4] = p_amb * (1.0 / (gamma - 1.0))
    slot_of = {int(b): s for s, b in enumerate(ids)}
    Edep = E_blast / (nD * dV)
    for kz, jy, ix in full:
        gi = ix + lo[0]
        gj = (jy + lo[1]) if nd > 1 else 0
        gk = (kz + lo[2]) if nd > 2 else 0
        b = ((gk // bz) * NBy + gj // by) * NBx + gi // bx
        s = slot_of.get(int(b))
        if s is not None:
            out[s, 4, gk % bz, gj % by, gi % bx] = Edep
    return out


def sedov_deposit_count(ndim: int) -> int:
    """n_D for any even N >= 8: 32 in 2D, 160 in 3D (12 in 1D)."""
    return int(sedov_deposit_mask([8] * ndim).sum())


def sod(N: Sequence[int], axis: int = 0, xmin=(0.0, 0.0, 0.0), xmax=(1.0, 1.0, 1.0),
        gamma: float = 1.4, left=(1.0, 1.0), right=(0.125, 0.1), x0: float = 0.5) -> np.ndarray:
    """Riemann problem along `axis`: (rho, p) = left for x_c < x0, right otherwise."""
    Nx, Ny, Nz = _dims(N)
    n = N[axis]
    dx = (xmax[axis] - xmin[axis]) / n
    xc = xmin[axis] + (np.arange(n) + 0.5) * dx
    is_left = xc < x0
    shape = [1, 1, 1]
    shape[2 - axis] = n
    is_left = is_left.reshape(shape)
    U = np.zeros((5, Nz, Ny, Nx), dtype=np.float64)
    U[0] = np.where(is_left, left[0], right[0])
    U[4] = np.where(is_left, left[1], right[1]) * (1.0 / (gamma - 1.0))
    return U


def uniform(N: Sequence[int], rho: float, vel: Sequence[float], p: float,
            gamma: float = 1.4) -> np.ndarray:
    Nx, Ny, Nz = _dims(N)
    U = np.zeros((5, Nz, Ny, Nx), dtype=np.float64)
    U[0] = rho
    for d in range(3):
        U[1 + d] = rho * vel[d]
    U[4] = p * (1.0 / (gamma - 1.0)) + 0.5 * rho * (vel[0] ** 2 + vel[1] ** 2 + vel[2] ** 2)
    return U


def random_prims(n: int, seed: int = SEED, ndim: int = 3) -> np.ndarray:
    """(n, 5) primitive states (rho, u, v, w, p) for unit fuzz."""
    rng = np.random.default_rng(seed)
    rho = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), n))
    p = np.exp(rng.uniform(np.log(1e-6), np.log(1e3), n))
    cs = np.sqrt(1.4 * p / rho)
    vel = rng.uniform(-3.0, 3.0, (n, 3)) * cs[:, None]
    vel[:, ndim:] = 0.0
    return np.stack([rho, vel[:, 0], vel[:, 1], vel[:, 2], p], axis=1)


def random_field(N: Sequence[int], seed: int = SEED, amp: float = 0.3,
                 gamma: float = 1.4) -> np.ndarray:
    """Rough but positive conserved field: rho in [0.5,1.5]*(1+amp noise), p likewise,
    velocities ~ amp * U[-1,1]; exercises every limiter / HLL branch."""
    Nx, Ny, Nz = _dims(N)
    nd = len(N)
    rng = np.random.default_rng(seed)
    shp = (Nz, Ny, Nx)
    rho = 1.0 + amp * rng.uniform(-1.0, 1.0, shp)
    p = 1.0 + amp * rng.uniform(-1.0, 1.0, shp)
    vel = [amp * 3.0 * rng.uniform(-1.0, 1.0, shp) if d < nd else np.zeros(shp) for d in range(3)]
    U = np.zeros((5,) + shp, dtype=np.float64)
    U[0] = rho
    for d in range(3):
        U[1 + d] = rho * vel[d]
    U[4] = p * (1.0 / (gamma - 1.0)) + 0.5 * rho * ((vel[0] * vel[0] + vel[1] * vel[1]) + vel[2] * vel[2])
    return U


def supersonic_field(N: Sequence[int], seed: int = SEED, mach: float = 2.5, amp: float = 0.2,
                     gamma: float = 1.4) -> np.ndarray:
    """Rough field with supersonic shear flow along every active axis, for the
    HLL / HLLC one-sided branches (S_L >= 0, S_R <= 0): velocity component d
    is +mach*c0 on one half of the domain along the next axis and -mach*c0 on
    the other half (c0 = sqrt(gamma) at rho = p = 1), plus amp-sized noise in
    rho, p and every velocity.  Along its own axis each component is smooth,
    so the flow stays supersonic there without shocks."""
    Nx, Ny, Nz = _dims(N)
    nd = len(N)
    rng = np.random.default_rng(seed)
    shp = (Nz, Ny, Nx)
    c0 = np.sqrt(gamma)
    rho = 1.0 + amp * rng.uniform(-1.0, 1.0, shp)
    p = 1.0 + amp * rng.uniform(-1.0, 1.0, shp)
    idx = np.indices(shp)                     # (k, j, i)
    ext = (Nx, Ny, Nz)
    vel = []
    for d in range(3):
        if d >= nd:
            vel.append(np.zeros(shp))
            continue
        e = (d + 1) % nd                      # the axis the sign flips along
        half = idx[2 - e] < ext[e] // 2
        sign = np.where(half, 1.0, -1.0) if nd > 1 else np.ones(shp)
        vel.append(mach * c0 * sign + amp * rng.uniform(-1.0, 1.0, shp))
    U = np.zeros((5,) + shp, dtype=np.float64)
    U[0] = rho
    for d in range(3):
        U[1 + d] = rho * vel[d]
    U[4] = p * (1.0 / (gamma - 1.0)) + 0.5 * rho * ((vel[0] * vel[0] + vel[1] * vel[1]) + vel[2] * vel[2])
    return U


def to_blocks(U: np.ndarray, nb: Sequence[int], block_ids: Sequence[int]) -> np.ndarray:
    """Global interior (5, Nz, Ny, Nx) -> packet interior (nblocks, 5, nbz, nby, nbx)
    for the given global block ids b = (bk*NBy + bj)*NBx + bi."""
    _, Nz, Ny, Nx = U.shape
    bx, by, bz = _dims(nb)
    NBx, NBy, NBz = Nx // bx, Ny // by, Nz // bz
    V = U.reshape(5, NBz, bz, NBy, by, NBx, bx).transpose(1, 3, 5, 0, 2, 4, 6)
    V = V.reshape(NBz * NBy * NBx, 5, bz, by, bx)
    return np.ascontiguousarray(V[np.asarray(block_ids, dtype=np.int64)])


def from_blocks(B: np.ndarray, N: Sequence[int], nb: Sequence[int],
                block_ids: Sequence[int], out: np.ndarray = None) -> np.ndarray:
    """Inverse of to_blocks (writes the given blocks into a global interior)."""
    Nx, Ny, Nz = _dims(N)
    bx, by, bz = _dims(nb)
    NBx, NBy, NBz = Nx // bx, Ny // by, Nz // bz
    if out is None:
        out = np.zeros((5, Nz, Ny, Nx), dtype=np.float64)
    V = out.reshape(5, NBz, bz, NBy, by, NBx, bx)
    for s, b in enumerate(block_ids):
        bi = b % NBx
        bj = (b // NBx) % NBy
        bk = b // (NBx * NBy)
        V[:, bk, :, bj, :, bi, :] = B[s]
    return out
