"""Pins of the oracle's SURVEY 8(f) F4 scheme variants (CPU): the MC limiter
(reading c21) and the HLLC Riemann solver (reading c20, Toro sec
10.4).  Each pin is a property the textbook fixes -- an independent
formulation, a closed form, an invariant or the exact Riemann solution --
not the oracle's expression retyped."""
import math

import numpy as np
import pytest

import oracle
import orcha_inputs as inp
from tests.exact import riemann
from tests.test_oracle_pins import ULP, euler_flux


def G3(**kw):
    return oracle.Grid(N=(8, 8, 8), **kw)


# ------------------------------------------------------------------ MC ----

def test_mc_is_the_sweby_limiter_function():
    # Sweby's flux-limiter form of MC: slope = phi(r) * dp with r = dm / dp and
    # phi(r) = max(0, min(2 r, (1 + r) / 2, 2)) -- a different evaluation path
    rng = np.random.default_rng(20250709)
    for _ in range(4000):
        qm, q0, qp = rng.normal(size=3) * 10.0 ** rng.uniform(-3, 3)
        dm, dp = q0 - qm, qp - q0
        s = oracle.mc_slope(qm, q0, qp)
        if dp == 0.0:
            assert s == 0.0
            continue
        r = dm / dp
        ref = max(0.0, min(2 * r, (1 + r) / 2, 2.0)) * dp
        assert abs(s - ref) <= 8 * ULP * (abs(dm) + abs(dp))


def test_mc_linear_exact_extrema_zero_and_odd():
    for a, b in ((0.0, 1.0), (-3.5, 2.25), (1e-300, 7.0)):
        assert oracle.mc_slope(a - b, a, a + b) == b          # linear data: the exact slope
    assert oracle.mc_slope(0.0, 1.0, 0.0) == 0.0              # extremum
    assert oracle.mc_slope(1.0, 0.0, 1.0) == 0.0
    rng = np.random.default_rng(5)
    for qm, q0, qp in rng.normal(size=(500, 3)):
        assert oracle.mc_slope(qp, q0, qm) == -oracle.mc_slope(qm, q0, qp)   # mirror


def test_mc_face_values_bounded_and_steeper_than_minmod():
    # monotonicity: the PLM face values q0 +- s/2 lie between the neighbours;
    # MC is the least diffusive of the two limiters (|s_MC| >= |s_minmod|)
    rng = np.random.default_rng(9)
    for qm, q0, qp in rng.normal(size=(2000, 3)):
        s = oracle.mc_slope(qm, q0, qp)
        lo, hi = min(qm, q0, qp), max(qm, q0, qp)
        for f in (q0 + 0.5 * s, q0 - 0.5 * s):
            assert lo - 1e-15 <= f <= hi + 1e-15
        assert abs(s) >= abs(oracle.minmod_slope(qm, q0, qp))


# ---------------------------------------------------------------- HLLC ----

@pytest.mark.parametrize("d", [0, 1, 2])
def test_hllc_consistency(d):
    # F_HLLC(U, U) = F(U): the star states of a uniform state are the state itself
    g = G3(riemann=oracle.HLLC)
    for q in inp.random_prims(300, seed=inp.SEED + 7 + d):
        F = oracle.hllc(g, d, q, q)
        Fe = euler_flux(q, d)
        scale = np.abs(Fe).max() + q[4] + q[0] * (q[1] ** 2 + q[2] ** 2 + q[3] ** 2)
        assert np.all(np.abs(F - Fe) <= 64 * ULP * scale)


def test_hllc_supersonic_is_hll():
    # outside the fan both solvers return the upwind physical flux, bitwise
    g = G3()
    qL = [1.0, 10.0, 0.3, -0.1, 1.0]
    for qR in inp.random_prims(50):
        qR = qR.copy()
        qR[1] = abs(qR[1]) + 10.0 + math.sqrt(1.4 * qR[4] / qR[0])
        assert np.array_equal(oracle.hllc(g, 0, qL, qR), oracle.hll(g, 0, qL, qR))


def test_hllc_resolves_a_stationary_contact():
    # u = 0, equal pressure, density jump: the exact flux is (0, p, 0, 0, 0).
    # HLLC restores the contact wave (S* = 0), HLL diffuses it (mass flux > 0).
    g = G3()
    for rl, rr, p in ((1.0, 0.125, 1.0), (3.0, 0.2, 0.01), (1e-3, 10.0, 5.0)):
        qL, qR = [rl, 0.0, 0.3, -0.2, p], [rr, 0.0, -0.1, 0.4, p]
        F = oracle.hllc(g, 0, qL, qR)
        assert abs(F[0]) <= 8 * ULP * rl * math.sqrt(1.4 * p / min(rl, rr))
        assert abs(F[1] - p) <= 8 * ULP * p
        assert abs(F[4]) <= 64 * ULP * p * math.sqrt(1.4 * p / min(rl, rr))
        assert abs(oracle.hll(g, 0, qL, qR)[0]) > 1e-3 * abs(rl - rr)


@pytest.mark.parametrize("d", [0, 1, 2])
def test_hllc_mirror_symmetry(d):
    g = G3()
    P = inp.random_prims(400, seed=31 + d)
    for a, b in zip(P[::2], P[1::2]):
        F = oracle.hllc(g, d, a, b)
        ma, mb = a.copy(), b.copy()
        ma[1 + d] = -ma[1 + d]
        mb[1 + d] = -mb[1 + d]
        sign = -np.ones(5)
        sign[1 + d] = 1.0
        Fm = oracle.hllc(g, d, mb, ma)
        # S* >= 0 picks the left star state: at S* == 0 the mirrored problem
        # picks the other side, equal only up to rounding
        assert np.allclose(Fm, sign * F, rtol=1e-13, atol=1e-13 * np.abs(F).max())


def _hllc_batten(q_l, q_r, d, gam=1.4):
    """HLLC in the flux form of Toro eq. 10.44 / Batten et al. (1997):
    F*_K = (S* (S_K U_K - F_K) + S_K p* D*) / (S_K - S*), D* = (0, e_d, S*),
    p* = p_L + rho_L (S_L - u_L)(S* - u_L) -- a different algebraic route to
    the star fluxes than the oracle's star states (eq. 10.38-10.39)."""
    def U_of(q):
        rho, vel, p = q[0], np.array(q[1:4], dtype=float), q[4]
        return np.array([rho, *(rho * vel), p / (gam - 1) + 0.5 * rho * vel @ vel])
    UL, UR = U_of(q_l), U_of(q_r)
    FL, FR = euler_flux(q_l, d, gam), euler_flux(q_r, d, gam)
    cl, cr = math.sqrt(gam * q_l[4] / q_l[0]), math.sqrt(gam * q_r[4] / q_r[0])
    ul, ur = q_l[1 + d], q_r[1 + d]
    SL, SR = min(ul - cl, ur - cr), max(ul + cl, ur + cr)
    if SL >= 0:
        return FL
    if SR <= 0:
        return FR
    Ss = (q_r[4] - q_l[4] + q_l[0] * ul * (SL - ul) - q_r[0] * ur * (SR - ur)) / (q_l[0] * (SL - ul) - q_r[0] * (SR - ur))
    ps = q_l[4] + q_l[0] * (SL - ul) * (Ss - ul)
    D = np.zeros(5)
    D[1 + d], D[4] = 1.0, Ss
    if Ss >= 0:
        return (Ss * (SL * UL - FL) + SL * ps * D) / (SL - Ss)
    return (Ss * (SR * UR - FR) + SR * ps * D) / (SR - Ss)


@pytest.mark.parametrize("d", [0, 1, 2])
def test_hllc_equals_the_batten_flux_form(d):
    g = G3()
    P = inp.random_prims(600, seed=77 + d)
    for a, b in zip(P[::2], P[1::2]):
        F = oracle.hllc(g, d, a, b)
        Fb = _hllc_batten(a, b, d)
        scale = np.abs(euler_flux(a, d)).max() + np.abs(euler_flux(b, d)).max() + a[4] + b[4]
        assert np.all(np.abs(F - Fb) <= 1e-12 * scale), (a, b, F, Fb)


def test_hllc_contact_speed_of_the_exact_riemann_problem():
    # for two states joined by a pure contact (same u and p) S* equals u and the
    # flux is the exact upwind flux of the moving contact: rho flux rho_L u or
    # rho_R u depending on the side the contact sits
    g = G3()
    for u in (0.4, -0.7):
        qL, qR = [1.0, u, 0.0, 0.0, 1.0], [0.25, u, 0.0, 0.0, 1.0]
        F = oracle.hllc(g, 0, qL, qR)
        up = qL if u > 0 else qR
        assert abs(F[0] - up[0] * u) <= 64 * ULP
        assert abs(F[1] - (up[0] * u * u + 1.0)) <= 64 * ULP


# ------------------------------------------------- whole scheme variants ----

def _sod(N, **kw):
    g = oracle.Grid(N=(N,), **kw)
    U = oracle.padded(g, inp.sod(g.N))
    log = oracle.run(g, U, t_end=0.2)
    return U[g.interior][:, 0, 0], log


@pytest.mark.parametrize("riemann_,limiter", [(oracle.HLLC, oracle.MINMOD), (oracle.HLL, oracle.MC),
                                              (oracle.HLLC, oracle.MC)])
def test_variants_converge_to_exact_sod_and_beat_hll_minmod(riemann_, limiter):
    ex = riemann.cell_averages(512, 0.2, 0.5, (1, 0, 1), (0.125, 0, 0.1))
    base, _ = _sod(512)
    I, log = _sod(512, riemann=riemann_, limiter=limiter)
    assert log.t == 0.2 and log.floor_hits == 0
    e0 = np.abs(base[0] - ex[0]).mean()
    e1 = np.abs(I[0] - ex[0]).mean()
    assert e1 < e0 and e1 <= 2.5e-3
    # star-region pressure plateau (between the rarefaction tail and the
    # contact) within 2e-3 of the exact p* (Toro test 1)
    x = (np.arange(512) + 0.5) / 512
    q = (x > 0.52) & (x < 0.66)
    p = (I[4] - 0.5 * I[1] ** 2 / I[0]) * 0.4
    assert np.abs(p[q] - 0.3031301780506468).max() < 2e-3
    # conserved totals (closed by outflow walls that see no flow before t = 0.2)
    assert abs(I[0].sum() - base[0].sum()) <= 1e-12 * base[0].sum()
    assert abs(I[4].sum() - base[4].sum()) <= 1e-12 * base[4].sum()


def test_variants_keep_uniform_flow_and_conservation_periodic():
    for riemann_, limiter in ((oracle.HLLC, oracle.MC), (oracle.HLLC, oracle.MINMOD)):
        g = oracle.Grid(N=(16, 16), bc=((oracle.PERIODIC,) * 2,) * 3, riemann=riemann_, limiter=limiter)
        U0 = inp.random_field(g.N, seed=12)
        U = oracle.padded(g, U0)
        oracle.run(g, U, nsteps=8)
        I = U[g.interior]
        for v in (0, 1, 2, 4):
            assert abs(I[v].sum() - U0[v].sum()) <= 1e-12 * np.abs(U0[v]).sum()
        g2 = oracle.Grid(N=(16, 16), bc=((oracle.PERIODIC,) * 2,) * 3, riemann=riemann_, limiter=limiter)
        uni = np.zeros((5, 1, 16, 16))
        uni[0], uni[1], uni[2], uni[4] = 1.3, 1.3 * 0.7, -1.3 * 0.2, 2.0
        V = oracle.padded(g2, uni)
        oracle.run(g2, V, nsteps=5)
        assert np.array_equal(V[g2.interior], uni)
