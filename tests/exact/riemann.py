"""Exact Riemann solver for the 1D Euler equations, ideal gas (Toro, "Riemann
Solvers and Numerical Methods for Fluid Dynamics", ch. 4).

Independent of the oracle (test utility only): used to pin the whole scheme
on the Sod shock tube (BASELINE.json config 2; SURVEY 8(c) "Whole scheme:
Sod").  Newton iteration on the star pressure p*, then self-similar sampling
at x/t.
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np


def _f_and_df(p: float, rho: float, pk: float, ck: float, g: float) -> Tuple[float, float]:
    """Toro (4.6)-(4.7): pressure function f_K and its derivative."""
    if p > pk:  # shock
        A = 2.0 / ((g + 1.0) * rho)
        B = (g - 1.0) / (g + 1.0) * pk
        sq = math.sqrt(A / (p + B))
        return (p - pk) * sq, sq * (1.0 - 0.5 * (p - pk) / (B + p))
    # rarefaction
    e = (g - 1.0) / (2.0 * g)
    return (2.0 * ck / (g - 1.0)) * ((p / pk) ** e - 1.0), (1.0 / (rho * ck)) * (p / pk) ** (-(g + 1.0) / (2.0 * g))


def star_state(rhoL, uL, pL, rhoR, uR, pR, g=1.4, tol=1e-14):
    """Return (p*, u*)."""
    cL = math.sqrt(g * pL / rhoL)
    cR = math.sqrt(g * pR / rhoR)
    du = uR - uL
    # two-rarefaction initial guess (Toro 4.46), positive
    e = (g - 1.0) / (2.0 * g)
    p = ((cL + cR - 0.5 * (g - 1.0) * du) / (cL / pL ** e + cR / pR ** e)) ** (1.0 / e)
    p = max(p, 1e-12)
    for _ in range(200):
        fL, dL = _f_and_df(p, rhoL, pL, cL, g)
        fR, dR = _f_and_df(p, rhoR, pR, cR, g)
        pn = p - (fL + fR + du) / (dL + dR)
        pn = max(pn, 1e-14)
        if abs(pn - p) / (0.5 * (pn + p)) < tol:
            p = pn
            break
        p = pn
    fL, _ = _f_and_df(p, rhoL, pL, cL, g)
    fR, _ = _f_and_df(p, rhoR, pR, cR, g)
    u = 0.5 * (uL + uR) + 0.5 * (fR - fL)
    return p, u


def star_densities(rhoL, pL, rhoR, pR, pstar, g=1.4):
    def side(rho, pk):
        if pstar > pk:
            r = pstar / pk
            gg = (g - 1.0) / (g + 1.0)
            return rho * (r + gg) / (gg * r + 1.0)
        return rho * (pstar / pk) ** (1.0 / g)
    return side(rhoL, pL), side(rhoR, pR)


def sample(x: np.ndarray, t: float, x0: float, left, right, g=1.4):
    """Exact (rho, u, p) at positions x and time t for the Riemann problem
    left = (rho, u, p) for x < x0, right otherwise."""
    rhoL, uL, pL = left
    rhoR, uR, pR = right
    ps, us = star_state(rhoL, uL, pL, rhoR, uR, pR, g)
    rsL, rsR = star_densities(rhoL, pL, rhoR, pR, ps, g)
    cL = math.sqrt(g * pL / rhoL)
    cR = math.sqrt(g * pR / rhoR)
    out = np.zeros((3, x.size))
    S = (x - x0) / t
    for n, s in enumerate(S):
        if s <= us:  # left of contact
            if ps > pL:  # left shock
                SL = uL - cL * math.sqrt((g + 1) / (2 * g) * ps / pL + (g - 1) / (2 * g))
                st = (rhoL, uL, pL) if s <= SL else (rsL, us, ps)
            else:  # left rarefaction
                SHL = uL - cL
                STL = us - cL * (ps / pL) ** ((g - 1) / (2 * g))
                if s <= SHL:
                    st = (rhoL, uL, pL)
                elif s >= STL:
                    st = (rsL, us, ps)
                else:
                    c = 2 / (g + 1) * (cL + (g - 1) / 2 * (uL - s))
                    u = 2 / (g + 1) * (cL + (g - 1) / 2 * uL + s)
                    rho = rhoL * (c / cL) ** (2 / (g - 1))
                    st = (rho, u, pL * (c / cL) ** (2 * g / (g - 1)))
        else:  # right of contact
            if ps > pR:  # right shock
                SR = uR + cR * math.sqrt((g + 1) / (2 * g) * ps / pR + (g - 1) / (2 * g))
                st = (rhoR, uR, pR) if s >= SR else (rsR, us, ps)
            else:
                SHR = uR + cR
                STR = us + cR * (ps / pR) ** ((g - 1) / (2 * g))
                if s >= SHR:
                    st = (rhoR, uR, pR)
                elif s <= STR:
                    st = (rsR, us, ps)
                else:
                    c = 2 / (g + 1) * (cR - (g - 1) / 2 * (uR - s))
                    u = 2 / (g + 1) * (-cR + (g - 1) / 2 * uR + s)
                    rho = rhoR * (c / cR) ** (2 / (g - 1))
                    st = (rho, u, pR * (c / cR) ** (2 * g / (g - 1)))
        out[:, n] = st
    return out


def wave_positions(t: float, x0: float, left, right, g=1.4):
    """(rarefaction head, tail, contact, shock) positions for a Sod-like problem
    (left rarefaction, right shock)."""
    rhoL, uL, pL = left
    rhoR, uR, pR = right
    ps, us = star_state(rhoL, uL, pL, rhoR, uR, pR, g)
    cL = math.sqrt(g * pL / rhoL)
    cR = math.sqrt(g * pR / rhoR)
    head = x0 + (uL - cL) * t
    tail = x0 + (us - cL * (ps / pL) ** ((g - 1) / (2 * g))) * t
    contact = x0 + us * t
    SR = uR + cR * math.sqrt((g + 1) / (2 * g) * ps / pR + (g - 1) / (2 * g))
    return head, tail, contact, x0 + SR * t, SR


def cell_averages(N: int, t: float, x0: float, left, right, g=1.4, sub: int = 16):
    """Exact cell averages of rho on [0,1] with N cells (sub-sampled midpoint rule)."""
    dx = 1.0 / N
    xs = (np.arange(N * sub) + 0.5) * (dx / sub)
    s = sample(xs, t, x0, left, right, g)
    return s.reshape(3, N, sub).mean(axis=2)
