"""Pins of the oracle's expensive-EOS surrogate (DESIGN.md
reading c22): ideal gas + radiation (c_v = 1), rho e = rho T + a T^4,
p = (gamma-1) rho T + a T^4/3, temperature by Newton, sound speed from
Chandrasekhar's Gamma_1.  Pinned by the gamma-law limit (a = 0), the
radiation-dominated limit, the e -> p -> e round trip through two different
Newton solves, and Gamma_1 against the adiabatic derivative of the EOS
itself (first law, finite differences) -- not by retyping the formulas."""
import math

import numpy as np
import pytest

import oracle
import orcha_inputs as inp


def G(a=0.0, w=1, **kw):
    return oracle.Grid(N=(8,), eos=oracle.GAS_RADIATION, arad=a, eos_work=w, **kw)


def _states(n, seed):
    rng = np.random.default_rng(seed)
    rho = 10 ** rng.uniform(-2, 2, n)
    e = 10 ** rng.uniform(-2, 2, n)          # specific internal energy
    vel = rng.uniform(-2, 2, (n, 3))
    return rho, e, vel


def _U(rho, e, vel):
    return [rho, rho * vel[0], rho * vel[1], rho * vel[2], rho * e + 0.5 * rho * vel @ vel]


def test_a_zero_is_the_gamma_law():
    g, g0 = G(0.0), oracle.Grid(N=(8,))
    rho, e, vel = _states(300, 1)
    for r, ei, v in zip(rho, e, vel):
        U = _U(r, ei, v)
        q, _ = oracle.prim(g, U)
        q0, _ = oracle.prim(g0, U)
        assert abs(q[4] - q0[4]) <= 4e-16 * 8 * q0[4]
        assert abs(oracle.sound_speed(g, q) - math.sqrt(1.4 * q[4] / q[0])) <= 1e-15 * 8 * oracle.sound_speed(g, q)
        assert abs(oracle.eint_from_p(g, q[0], q[4]) - q[4] / (0.4 * q[0])) <= 1e-14 * q[4] / q[0]


@pytest.mark.parametrize("a", [1e-3, 0.3, 50.0])
def test_round_trip_through_both_newton_solves(a):
    # e -> (prim) p -> (eint_from_p) e: two independent temperature solves
    g = G(a)
    rho, e, vel = _states(300, 2)
    for r, ei, v in zip(rho, e, vel):
        q, hit = oracle.prim(g, _U(r, ei, v))
        assert hit == 0
        e2 = oracle.eint_from_p(g, q[0], q[4])
        assert abs(e2 - ei) <= 1e-12 * ei


def test_radiation_dominated_limit():
    # a T^4 >> rho T: p -> rho e / 3 and Gamma_1 -> 4/3, with deviations bounded
    # by the gas share: T <= (rho e / a)^(1/4), p_gas = (gamma-1) rho T
    a = 1e8
    g = G(a)
    for r, ei in ((1e-3, 5.0), (1e-2, 50.0)):
        q, _ = oracle.prim(g, _U(r, ei, np.zeros(3)))
        pgas = 0.4 * r * (r * ei / a) ** 0.25
        assert abs(q[4] - r * ei / 3) <= pgas
        beta = pgas / q[4]
        c = oracle.sound_speed(g, q)
        assert abs(c * c * q[0] / q[4] - 4.0 / 3.0) <= 4 * beta


@pytest.mark.parametrize("a", [0.05, 1.0, 20.0])
def test_gamma1_is_the_adiabatic_exponent_of_the_eos(a):
    # Gamma_1 = (d ln p / d ln rho)_s; on an adiabat de = (p / rho^2) d rho (first
    # law).  Central differences of the EOS's own p(rho, e) give it independently.
    g = G(a)
    for r, ei in ((1.0, 1.0), (0.3, 4.0), (5.0, 0.2)):
        q, _ = oracle.prim(g, _U(r, ei, np.zeros(3)))
        p = q[4]
        h = 1e-5 * r
        ps = []
        for s in (-1, 1):
            r2 = r + s * h
            # integrate de = p/rho^2 drho along the adiabat (two half steps, midpoint)
            qm, _ = oracle.prim(g, _U(r + s * h / 2, ei + s * (h / 2) * p / r ** 2, np.zeros(3)))
            e2 = ei + s * h * qm[4] / (r + s * h / 2) ** 2
            ps.append(oracle.prim(g, _U(r2, e2, np.zeros(3)))[0][4])
        g1_fd = (ps[1] - ps[0]) / (2 * h) * r / p
        c = oracle.sound_speed(g, q)
        assert abs(c * c * r / p - g1_fd) <= 1e-6 * g1_fd


def test_work_multiplier_repeats_the_same_solve():
    rho, e, vel = _states(100, 3)
    g1, g4 = G(0.7, 1), G(0.7, 4)
    for r, ei, v in zip(rho, e, vel):
        U = _U(r, ei, v)
        q1, q4 = oracle.prim(g1, U)[0], oracle.prim(g4, U)[0]
        assert np.array_equal(q1, q4)
        assert oracle.sound_speed(g1, q1) == oracle.sound_speed(g4, q4)


def test_scheme_with_gas_only_surrogate_matches_gamma_law_sod():
    # a = 0 through the Newton path: the Sod run equals the gamma-law run to round-off
    out = []
    for kw in ({}, dict(eos=oracle.GAS_RADIATION, arad=0.0)):
        gg = oracle.Grid(N=(256,), **kw)
        U = oracle.padded(gg, inp.sod(gg.N))
        oracle.run(gg, U, t_end=0.1)
        out.append(U[gg.interior].copy())
    for v in (0, 1, 4):
        assert np.abs(out[0][v] - out[1][v]).max() <= 1e-12 * np.abs(out[0][v]).max()


def test_scheme_with_radiation_conserves_and_keeps_uniform_flow():
    per = ((oracle.PERIODIC,) * 2,) * 3
    g = oracle.Grid(N=(16, 16), bc=per, eos=oracle.GAS_RADIATION, arad=0.5, eos_work=2)
    U0 = inp.random_field(g.N, seed=17)
    U = oracle.padded(g, U0)
    log = oracle.run(g, U, nsteps=6)
    I = U[g.interior]
    for v in (0, 1, 2, 4):
        assert abs(I[v].sum() - U0[v].sum()) <= 1e-12 * np.abs(U0[v]).sum()
    uni = np.zeros((5, 1, 16, 16))
    uni[0], uni[1], uni[2], uni[4] = 1.3, 1.3 * 0.7, -1.3 * 0.2, 2.0
    V = oracle.padded(g, uni)
    oracle.run(g, V, nsteps=4)
    assert np.array_equal(V[g.interior], uni)
    assert log.floor_hits == 0
