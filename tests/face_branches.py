"""Count the Riemann-solver branches a state takes (test diagnostic only).

Given a ghost-filled global array (oracle layout (5, Pz, Py, Px)), recompute
the PLM/minmod face states of every face between two cells of the interior
plus a 2-cell ring (the telescoped stage-1 box) and the Davis
speeds S_L = min(n_L - c_L, n_R - c_R), S_R = max(n_L + c_L, n_R + c_R)
(A6, A7), and count the faces with S_L >= 0 (flux = F_L) and S_R <= 0
(flux = F_R).  This only proves that a test case reaches the one-sided
branches; it is not a pin of anything and is not compared with any result."""
from __future__ import annotations

import numpy as np


def _minmod(qm, q0, qp):
    dm = q0 - qm
    dp = qp - q0
    return np.where(dm * dp > 0.0, np.where(np.abs(dm) < np.abs(dp), dm, dp), 0.0)


def count(U: np.ndarray, ndim: int, ng: int = 4, gamma: float = 1.4, smallp: float = 1e-30):
    """Returns {axis: (n_left, n_right, n_faces)}."""
    rho = U[0]
    ir = 1.0 / rho
    q = [rho, U[1] * ir, U[2] * ir, U[3] * ir]
    ke = (0.5 * rho) * ((q[1] * q[1] + q[2] * q[2]) + q[3] * q[3])
    p = (gamma - 1.0) * (U[4] - ke)
    q.append(np.where(p < smallp, smallp, p))
    Q = np.stack(q)                       # (5, Pz, Py, Px)
    out = {}
    for d in range(ndim):
        ax = 3 - d                        # array axis of direction d
        n = Q.shape[ax]

        def sl(a, b):
            s = [slice(None)] * 4
            s[ax] = slice(a, n - b)
            return tuple(s)
        # faces between cells c and c+1 for c in [1, n-3): stencil c-1 .. c+2
        qm, q0, q1, q2 = Q[sl(0, 3)], Q[sl(1, 2)], Q[sl(2, 1)], Q[sl(3, 0)]
        L = q0 + 0.5 * _minmod(qm, q0, q1)
        R = q1 - 0.5 * _minmod(q0, q1, q2)
        cL = np.sqrt(gamma * L[4] / L[0])
        cR = np.sqrt(gamma * R[4] / R[0])
        nL, nR = L[1 + d], R[1 + d]
        SL = np.minimum(nL - cL, nR - cR)
        SR = np.maximum(nL + cL, nR + cR)
        # restrict to faces of the stage-1 box: cells [ng-2, ng+N+2) along d
        # (face index f between array cells f+1 and f+2) and the box across
        keep = [slice(None)] * 3
        for e in range(ndim):
            a = 2 - e
            m = SL.shape[a]
            if e == d:
                keep[a] = slice(ng - 3, m - (ng - 3))
            else:
                keep[a] = slice(ng - 2, m - (ng - 2))
        kk = tuple(keep)
        sL, sR = SL[kk], SR[kk]
        left = sL >= 0.0
        right = ~left & (sR <= 0.0)
        out[d] = (int(left.sum()), int(right.sum()), int(sL.size))
    return out
