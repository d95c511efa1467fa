"""Sedov-Taylor self-similar blast wave: the similarity constant xi_0.

Independent of the oracle (test utility only).  PAPER.md P:L591-593 (sec 5.2):
"an analytical expression exists for how far the shock has traveled in a given
time"; north_star: r ~ (E t^2 / rho)^(1/5) in 3D.  In n dimensions (n = 3
spherical, 2 cylindrical -- the 2D Cartesian blast with energy per unit
length, reading c16 -- and 1 planar):

    R(t) = xi_0 * (E t^2 / rho_0)^(1/(n+2)).

Derivation used here.  With m = 2/(n+2), D = dR/dt = m R/t, eta = r/R and
u = D f(eta), rho = rho_0 g(eta), p = rho_0 D^2 h(eta), the Euler equations
with geometric source become three ODEs linear in (f', g', h'):

    (f - eta) g' + g f'                 = -(n-1) g f / eta           (mass)
    (f - eta) f' + h'/g                 = -((m-1)/m) f               (momentum)
    (f - eta) (h'/h - gamma g'/g)       = -2 (m-1)/m                 (entropy)

integrated from the strong-shock jump at eta = 1 (g = (gamma+1)/(gamma-1),
f = h = 2/(gamma+1)) inward.  Energy conservation E = sigma_n m^2 xi_0^(n+2)
E I with I = int_0^1 (g f^2/2 + h/(gamma-1)) eta^(n-1) d eta and
sigma_n = 4 pi, 2 pi, 2 gives xi_0 = (sigma_n m^2 I)^(-1/(n+2)).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.integrate import solve_ivp


def _rhs(eta, y, n, gam, m):
    f, g, h = y
    a = f - eta
    # unknowns x = (f', g', h')
    A = np.array([
        [g, a, 0.0],
        [a, 0.0, 1.0 / g],
        [0.0, -gam * a / g, a / h],
    ])
    b = np.array([-(n - 1) * g * f / eta, -((m - 1.0) / m) * f, -2.0 * (m - 1.0) / m])
    return np.linalg.solve(A, b)


def xi0(n: int, gamma: float = 1.4, eta_min: float = 1e-7) -> float:
    m = 2.0 / (n + 2.0)
    y0 = [2.0 / (gamma + 1.0), (gamma + 1.0) / (gamma - 1.0), 2.0 / (gamma + 1.0)]

    def rhs(eta, y):
        return _rhs(eta, y, n, gamma, m)

    # integrand of I carried as a 4th component
    def full(eta, z):
        d = rhs(eta, z[:3])
        f, g, h = z[:3]
        return [d[0], d[1], d[2], (g * f * f / 2.0 + h / (gamma - 1.0)) * eta ** (n - 1)]

    sol = solve_ivp(full, (1.0, eta_min), y0 + [0.0], method="LSODA", rtol=1e-12, atol=1e-14)
    I = -sol.y[3, -1]  # integrated from 1 down to eta_min
    sigma = {1: 2.0, 2: 2.0 * math.pi, 3: 4.0 * math.pi}[n]
    return (sigma * m * m * I) ** (-1.0 / (n + 2.0))


def shock_radius(t: float, n: int, E: float = 1.0, rho0: float = 1.0, gamma: float = 1.4) -> float:
    return xi0(n, gamma) * (E * t * t / rho0) ** (1.0 / (n + 2.0))
