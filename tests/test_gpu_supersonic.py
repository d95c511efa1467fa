"""The one-sided branches of the Riemann solvers through the fused 3D
kernels (S_L >= 0 -> F_L, S_R <= 0 -> F_R; HLLC reading c20
the same), against the oracle: parity build bitwise (state and dt every
step), production build <= 1e-12 by the c13 metric and dt to 1e-13.

Every case asserts, from the oracle's own states, that faces of both
one-sided kinds occur along every axis (tests/face_branches.py):
supersonic shear flows on periodic boxes at 8^3, 16^3 and 32^3 blocks, the
pressure-floor band in 3D (floored cells have c ~ 0, so their faces are
one-sided), and a 3D Sedov blast run until its shell is resolved (the
post-shock flow is supersonic in the lab frame: u2 = 0.83 D > c2 = 0.44 D).
P:L665-667 (sec 6)."""
import functools

import numpy as np
import pytest

import oracle
import orcha_inputs as inp
from tests import face_branches as fb
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu
O, P, R = 0, 1, 2
HLL, HLLC = 0, 1


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _floor_band(N):
    # a rough 3D field with a band of cells whose total energy is below the
    # kinetic energy: primitive recovery gives p < 0, the floor fires (c10)
    U = inp.random_field(N, seed=31)
    ke = 0.5 * ((U[1] ** 2 + U[2] ** 2) + U[3] ** 2) / U[0]
    U[4][:, :, 60:68] = ke[:, :, 60:68] * (1 - 1e-3)
    return U


PER = ((P, P),) * 3
CASES = {
    "shear_8": dict(nb=(8, 8, 8), nblk=(2, 2, 2), bc=PER, ic=lambda N: inp.supersonic_field(N, seed=41), steps=8),
    "shear_16": dict(nb=(16, 16, 16), nblk=(2, 2, 1), bc=PER, ic=lambda N: inp.supersonic_field(N, seed=42),
                     steps=8),
    "shear_32": dict(nb=(32, 32, 32), nblk=(2, 1, 1), bc=PER, ic=lambda N: inp.supersonic_field(N, seed=43),
                     steps=4),
    "shear_16_outflow": dict(nb=(16, 16, 16), nblk=(2, 1, 1), bc=((O, O), (P, P), (P, P)),
                             ic=lambda N: inp.supersonic_field(N, seed=44), steps=6),
    "floor_16": dict(nb=(16, 16, 16), nblk=(8, 1, 1), bc=((O, O), (P, P), (P, P)), ic=_floor_band, steps=8),
    "sedov_long_16": dict(nb=(16, 16, 16), nblk=(2, 2, 2), bc=None, ic=inp.sedov, steps=100),
    "sedov_long_8": dict(nb=(8, 8, 8), nblk=(4, 4, 4), bc=None, ic=inp.sedov, steps=100),
}


def _N(c):
    return tuple(a * b for a, b in zip(c["nb"], c["nblk"]))


@functools.lru_cache(maxsize=None)
def _oracle(name, riemann):
    c = CASES[name]
    N = _N(c)
    og = oracle.Grid(N=N, bc=c["bc"] or ((O, O),) * 3, riemann=riemann)
    U0 = c["ic"](N)
    U = oracle.padded(og, U0)
    oracle.fill_ghosts(og, U)
    branches = [fb.count(U, 3)]
    log = oracle.run(og, U, nsteps=c["steps"])
    oracle.fill_ghosts(og, U)
    branches.append(fb.count(U, 3))
    return U0, U[og.interior].copy(), log, branches


def _gpu(name, riemann, parity):
    c = CASES[name]
    U0, Oo, olog, _ = _oracle(name, riemann)
    g = H.make_grid(3, c["nb"], c["nblk"], bc=c["bc"], parity=parity, riemann=riemann)
    G, t, log, pk = H.gpu_run(g, U0, nsteps=c["steps"])
    return G, log, pk


@pytest.mark.parametrize("name", list(CASES))
def test_case_reaches_both_one_sided_branches(name):
    _, _, olog, branches = _oracle(name, HLL)
    for d in range(3):
        left = max(b[d][0] for b in branches)
        right = max(b[d][1] for b in branches)
        assert left > 0 and right > 0, (name, d, branches)
    if name == "floor_16":
        assert olog.floor_hits > 0


@pytest.mark.parametrize("riemann", [HLL, HLLC])
@pytest.mark.parametrize("name", list(CASES))
def test_parity_build_bitwise(name, riemann):
    U0, Oo, olog, _ = _oracle(name, riemann)
    G, log, pk = _gpu(name, riemann, parity=True)
    assert [x[0] for x in log] == olog.dts
    assert [x[2] for x in log] == olog.argmax
    assert np.array_equal(G, Oo)


@pytest.mark.parametrize("riemann", [HLL, HLLC])
@pytest.mark.parametrize("name", list(CASES))
def test_production_within_1e12(name, riemann):
    U0, Oo, olog, _ = _oracle(name, riemann)
    G, log, pk = _gpu(name, riemann, parity=False)
    assert H.parity_error(G, Oo) <= 1e-12, H.error_report(G, Oo)
    for (dt, smax, am, tag), odt in zip(log, olog.dts):
        assert abs(dt - odt) <= 1e-13 * odt
