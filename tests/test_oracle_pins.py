"""Unit pins of the oracle's building blocks against things other than itself:
worked examples, closed forms, library routines and invariants (SURVEY.md 8(c)
"What pins each part").  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import orcha_inputs as inp
from tests.exact import riemann, sedov

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ULP = np.finfo(np.float64).eps


def G3(**kw):
    return oracle.Grid(N=(8, 8, 8), **kw)


# ------------------------------------------------------------------- EOS (A5)

def test_eos_worked_example():
    # dens=1, eint=1, gamma=1.4 -> pres=0.4 ("simple algebraic expression")
    q, r = oracle.prim(G3(), [1.0, 0.0, 0.0, 0.0, 1.0])
    assert r == 0
    assert abs(q[4] - 0.4) <= 2 * ULP * 0.4
    assert q[0] == 1.0 and q[1] == 0.0


def test_eos_kinetic_energy_and_velocity():
    # rho=2, v=(3,-4,12) (|v|=13), eint=5 -> E = rho*eint + rho*|v|^2/2 = 10 + 169
    q, r = oracle.prim(G3(), [2.0, 6.0, -8.0, 24.0, 179.0])
    assert (q[1], q[2], q[3]) == (3.0, -4.0, 12.0)
    assert abs(q[4] - 0.4 * 10.0) <= 4 * ULP * 4.0


def test_eos_floor_and_nonpositive_density():
    g = G3()
    q, r = oracle.prim(g, [1.0, 2.0, 0.0, 0.0, 1.0])  # E < ke -> p < 0 -> floor
    assert r == 1 and q[4] == g.smallp
    q, r = oracle.prim(g, [1.0, 0.0, 0.0, 0.0, float("nan")])  # NaN is kept, not floored
    assert r == 0 and math.isnan(q[4])
    _, r = oracle.prim(g, [0.0, 0.0, 0.0, 0.0, 1.0])
    assert r == -1


def test_sod_sound_speeds():
    # c_L = 1.183216, c_R = 1.058301 (sqrt(1.4), sqrt(1.12))
    g = G3()
    assert abs(oracle.sound_speed(g, [1.0, 0, 0, 0, 1.0]) - 1.183216) < 5e-7
    assert abs(oracle.sound_speed(g, [0.125, 0, 0, 0, 0.1]) - 1.058301) < 5e-7


def test_eos_idempotent():
    # EOS applied twice is idempotent on pressure (prim -> cons -> prim)
    g = G3()
    for rho, u, v, w, p in inp.random_prims(200):
        E = p / 0.4 + 0.5 * rho * (u * u + v * v + w * w)
        q, _ = oracle.prim(g, [rho, rho * u, rho * v, rho * w, E])
        E2 = q[4] / 0.4 + 0.5 * q[0] * (q[1] ** 2 + q[2] ** 2 + q[3] ** 2)
        q2, _ = oracle.prim(g, [q[0], q[0] * q[1], q[0] * q[2], q[0] * q[3], E2])
        assert abs(q2[4] - q[4]) <= 1e-9 * (abs(q[4]) + 1e-12 * E)


# -------------------------------------------------------- reconstruction (A6)

def test_minmod_linear_exact_and_extremum_zero():
    assert oracle.minmod_slope(1.0, 3.0, 5.0) == 2.0          # linear -> exact slope
    assert oracle.minmod_slope(5.0, 3.0, 1.0) == -2.0
    assert oracle.minmod_slope(1.0, 3.0, 4.0) == 1.0          # smaller one-sided difference
    assert oracle.minmod_slope(1.0, 3.0, 2.0) == 0.0          # local maximum
    assert oracle.minmod_slope(3.0, 1.0, 2.0) == 0.0          # local minimum
    assert oracle.minmod_slope(2.0, 2.0, 7.0) == 0.0          # flat side
    assert oracle.minmod_slope(2.0, 2.0, 2.0) == 0.0          # uniform


def test_minmod_tvd_face_values_bounded():
    rng = np.random.default_rng(inp.SEED)
    for qm, q0, qp in rng.normal(size=(2000, 3)):
        s = oracle.minmod_slope(qm, q0, qp)
        lo, hi = min(qm, q0, qp), max(qm, q0, qp)
        for face in (q0 + 0.5 * s, q0 - 0.5 * s):
            assert lo - 1e-15 <= face <= hi + 1e-15
        # minmod is the limiter with |s| = min(|dm|, |dp|) when they agree in sign
        dm, dp = q0 - qm, qp - q0
        assert abs(s) == (min(abs(dm), abs(dp)) if dm * dp > 0 else 0.0)


def test_face_flux_uniform_state_is_physical_flux():
    # uniform data -> slopes 0 -> HLL(U, U) must be the Euler flux of U
    g = G3()
    q = [1.3, 0.7, -0.2, 0.4, 2.1]
    F = oracle.face_flux(g, 0, q, q, q, q)
    assert np.array_equal(F, oracle.hll(g, 0, q, q))


# ----------------------------------------------------------------- HLL (A7)

def euler_flux(q, d, gam=1.4):
    """Textbook Euler flux in direction d (not the oracle's expression order)."""
    rho, vel, p = q[0], np.array(q[1:4]), q[4]
    E = p / (gam - 1) + 0.5 * rho * vel @ vel
    un = vel[d]
    F = np.array([rho * un, rho * vel[0] * un, rho * vel[1] * un, rho * vel[2] * un, (E + p) * un])
    F[1 + d] += p
    return F


@pytest.mark.parametrize("d", [0, 1, 2])
def test_hll_consistency(d):
    # F_HLL(U, U) = F(U) (consistency) within a few ulp of the largest term
    g = G3()
    for q in inp.random_prims(300, seed=inp.SEED + d):
        F = oracle.hll(g, d, q, q)
        Fe = euler_flux(q, d)
        scale = np.abs(Fe).max() + q[4] + q[0] * (q[1] ** 2 + q[2] ** 2 + q[3] ** 2)
        assert np.all(np.abs(F - Fe) <= 16 * ULP * scale)


def test_hll_supersonic_upwinding():
    # S_L >= 0 -> F = F_L independent of the right state; S_R <= 0 -> F = F_R
    g = G3()
    qL = [1.0, 10.0, 0.3, -0.1, 1.0]   # u - c > 0 for any right state below
    for qR in inp.random_prims(50):
        qR = qR.copy()
        qR[1] = abs(qR[1]) + 10.0 + math.sqrt(1.4 * qR[4] / qR[0])
        assert np.array_equal(oracle.hll(g, 0, qL, qR), oracle.hll(g, 0, qL, qL))
    qR = [0.5, -12.0, 0.0, 0.2, 0.7]
    for qL2 in inp.random_prims(50, seed=3):
        qL2 = qL2.copy()
        qL2[1] = -abs(qL2[1]) - 12.0 - math.sqrt(1.4 * qL2[4] / qL2[0])
        assert np.array_equal(oracle.hll(g, 0, qL2, qR), oracle.hll(g, 0, qR, qR))


@pytest.mark.parametrize("d", [0, 1, 2])
def test_hll_mirror_symmetry_bitwise(d):
    # mirror: negate the normal velocity and swap L<->R -> mass, energy and
    # tangential momentum flux change sign exactly; normal momentum flux is unchanged
    g = G3()
    P = inp.random_prims(400, seed=11 + d)
    for a, b in zip(P[::2], P[1::2]):
        F = oracle.hll(g, d, a, b)
        ma, mb = a.copy(), b.copy()
        ma[1 + d] = -ma[1 + d]
        mb[1 + d] = -mb[1 + d]
        Fm = oracle.hll(g, d, mb, ma)
        sign = -np.ones(5)
        sign[1 + d] = 1.0
        assert np.array_equal(Fm, sign * F)


def test_hll_between_one_sided_fluxes_for_contact():
    # stationary contact (u=0, equal p): exact solution has zero mass flux; HLL
    # diffuses it with flux = -S_L S_R/(S_R-S_L) (rho_R - rho_L), same sign as -(drho)
    g = G3()
    F = oracle.hll(g, 0, [1.0, 0, 0, 0, 1.0], [0.125, 0, 0, 0, 1.0])
    assert F[0] > 0 and abs(F[1] - 1.0) < 1e-12


# -------------------------------------------------------------- ghost fill

@pytest.mark.parametrize("bc,mode", [(oracle.OUTFLOW, "edge"), (oracle.PERIODIC, "wrap"),
                                     (oracle.REFLECT, "symmetric")])
@pytest.mark.parametrize("N", [(8,), (8, 12), (8, 6, 10)])
def test_ghost_fill_is_numpy_pad(bc, mode, N):
    # the axis-ordered ghost fill is np.pad(mode) per axis; reflect also
    # negates the normal momentum component in the ghosts of that axis
    g = oracle.Grid(N=N, bc=((bc, bc),) * 3)
    rng = np.random.default_rng(1)
    interior = rng.normal(size=g.shape[:1] + tuple(reversed(g.N3)))
    U = oracle.padded(g, interior)
    oracle.fill_ghosts(g, U)
    ref = interior.copy()
    for d in range(g.ndim):
        ax = 3 - d
        if bc == oracle.REFLECT:
            padw = [(0, 0)] * 4
            padw[ax] = (4, 4)
            sgn = np.ones_like(ref)
            sgn[1 + d] = -1.0
            pad_plain = np.pad(ref, padw, mode="symmetric")
            pad_flip = np.pad(ref * sgn, padw, mode="symmetric")
            n = ref.shape[ax]
            idx = np.arange(n + 8)
            ghost = (idx < 4) | (idx >= n + 4)
            sel = [None] * 4
            sel[ax] = slice(None)
            gm = ghost.reshape([-1 if a == ax else 1 for a in range(4)])
            ref = np.where(gm, pad_flip, pad_plain)
        else:
            padw = [(0, 0)] * 4
            padw[ax] = (4, 4)
            ref = np.pad(ref, padw, mode=mode)
    assert np.array_equal(U, ref)


# ------------------------------------------------------------------ dt (A4)

def test_dt_uniform_state_closed_form():
    g = oracle.Grid(N=(8, 16, 32), xmax=(1.0, 2.0, 0.5))
    U = oracle.padded(g, inp.uniform(g.N, 1.7, (0.3, -0.5, 0.9), 2.2))
    r = oracle.compute_dt(g, U)
    c = math.sqrt(1.4 * 2.2 / 1.7)
    s = (0.3 + c) * 8 + (0.5 + c) * 8 + (0.9 + c) * 64
    assert abs(r.dt - 0.4 / s) <= 8 * ULP * r.dt
    assert r.argmax == 0 and r.tag == oracle.TAG_CFL


@pytest.mark.parametrize("nd,N", [(2, 32), (3, 16), (2, 64)])
def test_dt_sedov_t0_closed_form_and_tiebreak(nd, N):
    # dt0 = cfl*dx/(d*c_dep), c_dep = sqrt(gamma(gamma-1) E/(n_D dV)); the n_D
    # deposit cells tie -> argmax is the lowest global index among them
    g = oracle.Grid(N=(N,) * nd)
    U = oracle.padded(g, inp.sedov(g.N))
    r = oracle.compute_dt(g, U)
    nD = {2: 32, 3: 160}[nd]
    dV = (1.0 / N) ** nd
    c = math.sqrt(1.4 * 0.4 * 1.0 / (nD * dV))
    assert abs(r.dt - 0.4 * (1.0 / N) / (nd * c)) <= 1e-14 * r.dt
    mask = inp.sedov_deposit_mask(g.N).reshape(-1)
    assert r.argmax == int(np.flatnonzero(mask)[0])


def test_dt_cfg1_golden_and_clamp():
    gold = json.load(open(os.path.join(GOLD, "sedov2d_cfg1.json")))
    g = oracle.Grid(N=tuple(gold["N"]))
    U = oracle.padded(g, inp.sedov(g.N))
    r = oracle.compute_dt(g, U)
    assert r.dt == gold["dt0"]
    r2 = oracle.compute_dt(g, U, t_remaining=1e-4)
    assert r2.dt == 1e-4 and r2.tag == oracle.TAG_CLAMP
    r3 = oracle.compute_dt(g, U, t_remaining=r.dt)  # equal -> CFL wins (selection order c8)
    assert r3.tag == oracle.TAG_CFL


def test_dt_nan_propagates():
    g = oracle.Grid(N=(8, 8))
    U = oracle.padded(g, inp.uniform(g.N, 1.0, (0, 0, 0), 1.0))
    U[4, 0, 4 + 3, 4 + 5] = float("nan")
    r = oracle.compute_dt(g, U)
    assert math.isnan(r.dt) and r.argmax == 3 * 8 + 5


# ------------------------------------------------- exact-solution utilities

def test_exact_riemann_matches_toro():
    gold = json.load(open(os.path.join(GOLD, "toro_riemann.json")))
    t1 = gold["test1_sod"]
    ps, us = riemann.star_state(*t1["left"], *t1["right"])
    assert abs(ps - t1["p_star"]) < 1e-5 and abs(us - t1["u_star"]) < 1e-5
    rl, rr = riemann.star_densities(t1["left"][0], t1["left"][2], t1["right"][0], t1["right"][2], ps)
    assert abs(rl - t1["rho_star_L"]) < 1e-5 and abs(rr - t1["rho_star_R"]) < 1e-5
    t3 = gold["test3"]
    ps3, us3 = riemann.star_state(*t3["left"], *t3["right"])
    assert abs(ps3 - t3["p_star"]) < 1e-3 and abs(us3 - t3["u_star"]) < 1e-4
    w = gold["sod_waves_t0.2"]
    head, tail, contact, shock, S = riemann.wave_positions(0.2, 0.5, t1["left"], t1["right"])
    for a, b in ((head, w["head"]), (tail, w["tail"]), (contact, w["contact"]), (shock, w["shock"])):
        assert abs(a - b) < 1e-6


def test_sedov_similarity_constant():
    gold = json.load(open(os.path.join(GOLD, "toro_riemann.json")))["sedov_xi0"]
    assert abs(sedov.xi0(3, 5.0 / 3.0) - gold["gamma_5_3_spherical"]) < 2e-5   # literature value
    assert abs(sedov.xi0(3, 1.4) - gold["gamma_1_4_spherical"]) < 2e-6
    assert abs(sedov.xi0(2, 1.4) - gold["gamma_1_4_cylindrical"]) < 2e-6
