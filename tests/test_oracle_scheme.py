"""Whole-scheme pins of the oracle (SURVEY.md 8(c) "What pins each part"):
exact solutions, closed forms, conservation, symmetries, dimensional
reduction, the telescoping equivalence and the independent survey-time
prototype's values.  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle
import orcha_inputs as inp
from tests.exact import riemann, sedov

GOLD = os.path.join(os.path.dirname(__file__), "golden")
O, P, R = oracle.OUTFLOW, oracle.PERIODIC, oracle.REFLECT


def run_fresh(g, U0, **kw):
    U = oracle.padded(g, U0)
    log = oracle.run(g, U, **kw)
    return U[g.interior].copy(), log


def test_cfg1_matches_independent_prototype():
    # BASELINE configs[0]; values of the survey's numpy prototype
    gold = json.load(open(os.path.join(GOLD, "sedov2d_cfg1.json")))
    g = oracle.Grid(N=tuple(gold["N"]))
    I, log = run_fresh(g, inp.sedov(g.N), nsteps=gold["steps"])
    dV = 1.0 / (g.N[0] * g.N[1])
    assert log.dts[0] == gold["dt0"]
    assert log.t == gold["t10"]
    rho = I[0, 0]
    assert rho.max() == gold["max_rho"]
    assert list(np.unravel_index(rho.argmax(), rho.shape)) == gold["max_rho_at_ji"]
    assert rho.sum() * dV == gold["sum_rho_dV"]
    assert I[4].sum() * dV == gold["sum_E_dV"]
    assert log.floor_hits == gold["floor_hits"]


def sedov_energy_closed_form(N):
    """E_blast + (N_cells - n_D) dV p_amb/(gamma-1) (SURVEY 8(c) "Initial conditions")."""
    nd = len(N)
    dV = 1.0
    ncell = 1
    for n in N:
        dV = dV / n
        ncell *= n
    return 1.0 + (ncell - inp.sedov_deposit_count(nd)) * dV * 1e-5 / 0.4


@pytest.mark.slow
def test_cfg3_matches_independent_prototype():
    # BASELINE configs[2] (128^3, 10 steps) against the survey-time numpy
    # prototype.  Its sums ran in numpy's pairwise order, the oracle's here in
    # np.sum's order over a different array view, so sum E (a 2M-term sum of
    # values ~1e-5 and ~1e3) agrees to a few ulp, not bitwise: the closed-form
    # initial energy (the blast has not reached the outflow walls, so E is
    # conserved) is the exact pin, the prototype value a 1e-14 cross-check.
    gold = json.load(open(os.path.join(GOLD, "sedov3d_cfg3.json")))
    g = oracle.Grid(N=tuple(gold["N"]))
    I, log = run_fresh(g, inp.sedov(g.N), nsteps=gold["steps"])
    assert abs(log.dts[0] - gold["dt0"]) <= 1e-15 * gold["dt0"]
    assert log.t == gold["t10"]
    assert abs(I[0].max() - gold["max_rho"]) <= 1e-15 * gold["max_rho"]
    sumE = I[4].sum() / 128 ** 3
    assert abs(sumE - sedov_energy_closed_form(g.N)) <= 1e-15
    assert abs(sumE - gold["sum_E_dV"]) <= 1e-14
    assert abs(I[0].sum() / 128 ** 3 - 1.0) <= 1e-15


def _shell_radius(rho, dx):
    """Radius of the peak of the shell-averaged density (cells binned by
    floor(r/dx) about the centre vertex)."""
    n = rho.shape[-1]
    xc = (np.arange(n) + 0.5) * dx - 0.5
    r2 = xc[None, None, :] ** 2 + xc[None, :, None] ** 2 + xc[:, None, None] ** 2
    b = (np.sqrt(r2) / dx).astype(int).ravel()
    mean = np.bincount(b, rho.ravel()) / np.bincount(b)
    return (np.argmax(mean) + 0.5) * dx


@pytest.mark.parametrize("N", [32, pytest.param(64, marks=pytest.mark.slow)])
def test_sedov_3d_shock_radius(N):
    # P:L591-593 (sec 5.2): "an analytical expression exists for how far the
    # shock has traveled"; north_star: r = xi0 (E t^2/rho)^(1/5) in 3D with
    # xi0 = 1.032777 (gamma = 1.4, tests/exact/sedov.py).  Gate |R - R_th| <=
    # 2 dx at t = 0.05 (R_th = 0.3116).  Mass and energy are conserved to
    # round-off while the shock is inside the box.
    g = oracle.Grid(N=(N, N, N))
    I, log = run_fresh(g, inp.sedov(g.N), t_end=0.05)
    dx = 1.0 / N
    Rth = sedov.shock_radius(0.05, 3)
    assert abs(sedov.xi0(3) - 1.032777) < 2e-6
    assert abs(Rth - 0.31160) < 1e-5
    R = _shell_radius(I[0], dx)
    assert abs(R - Rth) <= 2 * dx, (R, Rth, dx)
    assert log.t == 0.05 and log.tags[-1] == oracle.TAG_CLAMP
    assert abs(I[0].sum() * dx ** 3 - 1.0) <= 1e-14
    assert abs(I[4].sum() * dx ** 3 - sedov_energy_closed_form(g.N)) <= 1e-14
    assert log.floor_hits == 0


def _advance_prescribed(g, U0, dts):
    """Advance with a given dt sequence (ghost fill + one RK2 step each)."""
    U = oracle.padded(g, U0)
    for dt in dts:
        oracle.fill_ghosts(g, U)
        rc, _ = oracle.step(g, U, dt)
        assert rc == 0
    return U[g.interior].copy()


def test_noncubic_cells_tube_along_y_equals_1d_run():
    # The flux divergence's per-axis 1/dx: a Sod tube along y
    # on cells with dx != dy (x periodic, so every x-face flux difference is
    # exactly 0) must advance exactly like the 1D tube with spacing dy, given
    # the same dt sequence.  Multiplying dF_y by 1/dx (or the wrong axis'
    # spacing anywhere) changes every cell.
    N = 64
    d1 = oracle.Grid(N=(N,))
    X, log = run_fresh(d1, inp.sod(d1.N), nsteps=25)
    nx = 6
    g2 = oracle.Grid(N=(nx, N), xmax=(0.37, 1.0), bc=((P, P), (O, O), (O, O)))
    Y = _advance_prescribed(g2, inp.sod(g2.N, axis=1), log.dts)
    for i in range(nx):
        col = Y[:, 0, :, i]
        assert np.array_equal(col[0], X[0, 0, 0])
        assert np.array_equal(col[2], X[1, 0, 0])      # normal momentum
        assert np.array_equal(col[4], X[4, 0, 0])
        assert np.all(col[1] == 0.0) and np.all(col[3] == 0.0)


def test_noncubic_cells_tube_along_z_equals_1d_run():
    # the same along z with three different spacings (dz = 1/48)
    N = 48
    d1 = oracle.Grid(N=(N,))
    X, log = run_fresh(d1, inp.sod(d1.N), nsteps=20)
    g3 = oracle.Grid(N=(4, 6, N), xmax=(0.29, 0.53, 1.0), bc=((P, P), (P, P), (O, O)))
    Z = _advance_prescribed(g3, inp.sod(g3.N, axis=2), log.dts)
    for j in range(6):
        for i in range(4):
            assert np.array_equal(Z[0, :, j, i], X[0, 0, 0])
            assert np.array_equal(Z[3, :, j, i], X[1, 0, 0])
            assert np.array_equal(Z[4, :, j, i], X[4, 0, 0])
    assert np.all(Z[1] == 0.0) and np.all(Z[2] == 0.0)


def test_noncubic_cells_cfl_closed_form():
    # A4 on a uniform moving state with three different spacings and three
    # different speeds: dt = cfl / sum_d (|v_d| + c)/dx_d, c = sqrt(gamma p/rho).
    # Pairing a speed with the wrong spacing moves dt by > 10 %.
    g = oracle.Grid(N=(8, 10, 12), xmax=(0.5, 2.0, 0.3), bc=((P, P),) * 3)
    rho, vel, p = 1.7, (0.9, -2.3, 0.4), 0.6
    U = oracle.padded(g, inp.uniform(g.N, rho, vel, p))
    oracle.fill_ghosts(g, U)
    r = oracle.compute_dt(g, U)
    c = np.sqrt(1.4 * p / rho)
    dxs = (0.5 / 8, 2.0 / 10, 0.3 / 12)
    expect = 0.4 / sum((abs(v) + c) / h for v, h in zip(vel, dxs))
    assert abs(r.dt - expect) <= 4e-16 * expect
    perm = 0.4 / sum((abs(v) + c) / h for v, h in zip(vel, dxs[::-1]))
    assert abs(perm - expect) > 0.1 * expect
    assert r.argmax == 0 and r.tag == oracle.TAG_CFL


@pytest.mark.parametrize("nd", [2, 3])
def test_sedov_initial_energy_closed_form(nd):
    # E_total = E_blast + (N_cells - n_D) dV p_amb/(gamma-1)
    N = (16,) * nd
    U = inp.sedov(N)
    dV = (1.0 / 16) ** nd
    nD = inp.sedov_deposit_count(nd)
    assert nD == {2: 32, 3: 160}[nd]
    expect = 1.0 + (16 ** nd - nD) * dV * 1e-5 / 0.4
    assert abs(U[4].sum() * dV - expect) <= 1e-14


@pytest.mark.parametrize("N", [(16, 16, 16), (24, 20)])
def test_conservation_closed_domain(N):
    # periodic box: sum rho, sum m, sum E change <= 1e-13 relative over 10 steps
    g = oracle.Grid(N=N, bc=((P, P),) * 3)
    U0 = inp.random_field(N)
    I, log = run_fresh(g, U0, nsteps=10)
    for v in range(5):
        scale = np.abs(U0[v]).sum()
        assert abs(I[v].sum() - U0[v].sum()) <= 1e-13 * scale, v
    assert log.floor_hits == 0


def test_uniform_moving_state_stays_bitwise_uniform():
    g = oracle.Grid(N=(12, 8, 10), bc=((P, P),) * 3)
    U0 = inp.uniform(g.N, 1.3, (0.7, -0.4, 0.2), 0.9)
    I, _ = run_fresh(g, U0, nsteps=5)
    for v in range(5):
        assert np.all(I[v] == I[v].flat[0])


@pytest.mark.parametrize("N", [(32, 32), (12, 12, 12)])
def test_telescoped_equals_refill_periodic(N):
    # the twice-thick halo with redundant stage-1 ring computation
    # replaces the second refresh; bitwise identical under periodic BCs
    g = oracle.Grid(N=N, bc=((P, P),) * 3)
    U0 = inp.random_field(N, seed=7)
    A, _ = run_fresh(g, U0, nsteps=5, mode="telescoped")
    B, _ = run_fresh(g, U0, nsteps=5, mode="refill")
    assert np.array_equal(A, B)


def test_telescoped_differs_from_refill_only_in_tails_at_outflow():
    # reading c5: at physical outflow boundaries the telescoped step is NOT the
    # refill step; on Sedov they differ only in round-off-level momentum tails
    g = oracle.Grid(N=(32, 32))
    A, _ = run_fresh(g, inp.sedov(g.N), nsteps=10, mode="telescoped")
    B, _ = run_fresh(g, inp.sedov(g.N), nsteps=10, mode="refill")
    assert np.array_equal(A[0], B[0]) and np.array_equal(A[4], B[4])
    assert np.abs(A - B).max() < 1e-40


def _mirror(I, d, nd):
    ax = 3 - d
    M = np.flip(I, axis=ax).copy()
    M[1 + d] = -M[1 + d]
    return M


@pytest.mark.parametrize("N", [(32, 32), (16, 16, 16)])
def test_sedov_octant_mirror_symmetry_bitwise(N):
    g = oracle.Grid(N=N)
    I, _ = run_fresh(g, inp.sedov(N), nsteps=10)
    for d in range(len(N)):
        assert np.array_equal(I, _mirror(I, d, len(N))), d


@pytest.mark.parametrize("N", [(32, 32), (16, 16, 16)])
def test_sedov_xy_transpose_bitwise(N):
    g = oracle.Grid(N=N)
    I, _ = run_fresh(g, inp.sedov(N), nsteps=10)
    T = np.swapaxes(I, 2, 3).copy()
    T[[1, 2]] = T[[2, 1]]
    assert np.array_equal(I, T)


def test_tube_dimensional_reduction_and_transpose():
    # 2D x-tube with periodic y: all rows bitwise identical, rho*v == 0 and
    # rho*w == 0 bitwise; the y-tube is its exact transpose
    N = 64
    gx = oracle.Grid(N=(N, 8), xmax=(1.0, 8.0 / N), bc=((O, O), (P, P), (O, O)))
    X, _ = run_fresh(gx, inp.sod(gx.N, axis=0), nsteps=20)
    assert np.all(X == X[:, :, :1, :])
    assert np.all(X[2] == 0.0) and np.all(X[3] == 0.0)
    gy = oracle.Grid(N=(8, N), xmax=(8.0 / N, 1.0), bc=((P, P), (O, O), (O, O)))
    Y, _ = run_fresh(gy, inp.sod(gy.N, axis=1), nsteps=20)
    T = np.swapaxes(Y, 2, 3).copy()
    T[[1, 2]] = T[[2, 1]]
    assert np.array_equal(X, T)


def test_sod_exact_solution_and_convergence():
    # BASELINE configs[1]: Sod vs the exact Riemann solution (Toro test 1) at
    # t = 0.2; L1(rho) <= 1.5e-3 at 1024 cells and observed order >= 0.7
    L1 = {}
    for N in (256, 1024):
        g = oracle.Grid(N=(N,))
        I, log = run_fresh(g, inp.sod(g.N), t_end=0.2)
        assert log.t == 0.2 and log.tags[-1] == oracle.TAG_CLAMP
        assert log.floor_hits == 0
        ex = riemann.cell_averages(N, 0.2, 0.5, (1, 0, 1), (0.125, 0, 0.1))
        L1[N] = np.abs(I[0, 0, 0] - ex[0]).mean()
        # star-region plateau between tail and contact within 1e-3 of p*
        x = (np.arange(N) + 0.5) / N
        q = (x > 0.52) & (x < 0.66)
        p = (I[4, 0, 0] - 0.5 * I[1, 0, 0] ** 2 / I[0, 0, 0]) * 0.4
        assert np.abs(p[q] - 0.3031301780506468).max() < 2e-3
    assert L1[1024] <= 1.5e-3
    assert np.log2(L1[256] / L1[1024]) / 2 >= 0.7


def test_sedov_2d_shock_radius():
    # analytic shock position; 2D Cartesian = cylindrical blast
    # (reading c16): R = xi0 (E t^2/rho)^(1/4), |R - R_th| <= 2 dx at N = 128
    N = 128
    g = oracle.Grid(N=(N, N))
    I, log = run_fresh(g, inp.sedov(g.N), t_end=0.05)
    rho = I[0, 0]
    dx = 1.0 / N
    xc = (np.arange(N) + 0.5) * dx - 0.5
    r = np.sqrt(xc[None, :] ** 2 + xc[:, None] ** 2)
    b = (r / dx).astype(int)
    mean = np.bincount(b.ravel(), rho.ravel()) / np.bincount(b.ravel())
    Rnum = (np.argmax(mean) + 0.5) * dx
    Rth = sedov.shock_radius(0.05, 2)
    assert abs(Rnum - Rth) <= 2 * dx
    # mass and energy exactly conserved while the blast is inside the box
    assert abs(rho.sum() * dx * dx - 1.0) <= 1e-14
    assert abs(I[4].sum() * dx * dx - inp.sedov(g.N)[4].sum() * dx * dx) <= 1e-14
    assert log.floor_hits == 0


def test_reflect_wall_equals_mirrored_periodic_domain():
    # a reflecting wall at x=0 is the mirror of the doubled domain: run a
    # symmetric state on [-1,1] periodic and compare its right half bitwise
    N = 32
    base = inp.random_field((N, 8), seed=5)
    dbl = np.concatenate([_mirror(base, 0, 2), base], axis=3)
    gd = oracle.Grid(N=(2 * N, 8), xmin=(-1.0, 0.0), xmax=(1.0, 0.25), bc=((P, P), (P, P), (O, O)))
    D, logd = run_fresh(gd, dbl, nsteps=6)
    gr = oracle.Grid(N=(N, 8), xmin=(0.0, 0.0), xmax=(1.0, 0.25), bc=((R, R), (P, P), (O, O)))
    # reflect on both x ends == doubled periodic domain of the mirrored pair
    Rr, logr = run_fresh(gr, base, nsteps=6)
    assert logd.dts == logr.dts
    assert np.array_equal(D[:, :, :, N:], Rr)


def test_oracle_omp_build_is_bitwise_the_plain_build():
    # SURVEY 8(d) "oracle-omp": the same source with -fopenmp over k-planes
    # must give bitwise the single-threaded result (the bench's labelled
    # multi-core CPU baseline relies on it)
    N = (24, 20, 16)
    g = oracle.Grid(N=N, bc=((P, P), (O, R), (O, O)))
    U0 = inp.random_field(N, seed=17)
    runs = []
    for threads in (1, 4):
        assert oracle.use_threads(threads) == threads
        try:
            runs.append(run_fresh(g, U0, nsteps=4))
        finally:
            oracle.use_threads(1)
    (A, la), (B, lb) = runs
    assert la.dts == lb.dts and la.floor_hits == lb.floor_hits
    assert np.array_equal(A, B)
