"""Parity at BASELINE.json's full single-GPU size, in the launch configuration
bench.py times (cfg4: one packet of 4096 blocks of 16^3 = 256^3 cells, fused
kernels): one step against the oracle on the whole global array (bitwise in
the parity build, <= 1e-12 by the c13 metric in the production build), and
size-independent properties over 10 steps (octant mirror symmetry, exact
mass conservation while the blast is inside the box, dt bitwise repeatable
and equal between the builds' first step)."""
import numpy as np
import pytest

import oracle
import orcha_inputs as inp
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu
NB, NBLK = (16, 16, 16), (16, 16, 16)
N = (256, 256, 256)


@pytest.fixture(scope="module")
def oracle_one_step():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    og = oracle.Grid(N=N)
    U = oracle.padded(og, inp.sedov(N))
    oracle.fill_ghosts(og, U)
    r = oracle.compute_dt(og, U)
    rc, hits = oracle.step(og, U, r.dt)
    assert rc == 0 and hits == 0
    return r, U[og.interior].copy()


def _gpu(parity, nsteps):
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, NB, NBLK, parity=parity)
    ids = np.arange(g.nblocks)
    pk = hydro.Packet(g, ids)
    pk.pack(inp.sedov_packet(N, NB, ids))
    t, n, log = hydro.run([pk], nsteps=nsteps)
    return g, pk, log


@pytest.mark.parametrize("parity", [True, False])
def test_cfg4_one_step_against_oracle(oracle_one_step, parity):
    r, ref = oracle_one_step
    g, pk, log = _gpu(parity, 1)
    out = H.gather(g, [pk])
    if parity:
        assert log[0][0] == r.dt and log[0][2] == r.argmax
        assert np.array_equal(out, ref)
    else:
        assert abs(log[0][0] - r.dt) <= 1e-13 * r.dt and log[0][2] == r.argmax
        assert H.parity_error(out, ref) <= 1e-12
    assert pk.counters() == (0, -1)


def test_cfg4_ten_steps_properties():
    g, pk, log = _gpu(False, 10)
    out = H.gather(g, [pk])
    rho = out[0]
    # mass is exact while the blast is inside (boundary fluxes are exactly 0)
    assert abs(rho.sum() / rho.size - 1.0) <= 1e-13
    # octant mirror symmetry of the centred blast (FMA build: to round-off)
    for ax, mom in ((3, 1), (2, 2), (1, 3)):
        m = np.flip(out, axis=ax).copy()
        m[mom] = -m[mom]
        for v in range(5):
            scale = np.abs(out[v]).max()
            assert np.abs(out[v] - m[v]).max() <= 1e-13 * scale
    # dt is positive, decreasing as the blast sharpens, and repeatable
    dts = [x[0] for x in log]
    g2, pk2, log2 = _gpu(False, 10)
    assert dts == [x[0] for x in log2]
    assert np.array_equal(H.gather(g2, [pk2]), out)


@pytest.fixture(scope="module")
def oracle_cfg3():
    # BASELINE configs[2]: 3D Sedov, 512 blocks of 16^3 (128^3 cells), one
    # packet; the north_star's bar is "within 1e-12 relative per cell after
    # 10 steps" -- the oracle (plain C) takes ~20 s here
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    og = oracle.Grid(N=(128, 128, 128))
    O_, olog = H.oracle_run(og, inp.sedov((128, 128, 128)), nsteps=10)
    return O_, olog


@pytest.mark.parametrize("parity", [True, False])
def test_cfg3_ten_steps_against_oracle(oracle_cfg3, parity):
    from paper_2507_09337_b200 import hydro
    O_, olog = oracle_cfg3
    g = H.make_grid(3, NB, (8, 8, 8), parity=parity)
    ids = np.arange(g.nblocks)
    pk = hydro.Packet(g, ids)
    pk.pack(inp.sedov_packet((128, 128, 128), NB, ids))
    t, n, log = hydro.run([pk], nsteps=10)
    out = H.gather(g, [pk])
    if parity:
        assert [x[2] for x in log] == olog.argmax   # the argmax decision in the oracle's arithmetic
        assert [x[0] for x in log] == olog.dts
        assert np.array_equal(out, O_)
    else:
        # the production build's rounding breaks the blast's exact symmetric
        # ties differently after step 0, so only the value of the max is
        # compared there (the argmax decision is pinned by the parity build)
        assert log[0][2] == olog.argmax[0]
        for (dt, smax, am, tag), odt in zip(log, olog.dts):
            assert abs(dt - odt) <= 1e-13 * odt
        assert H.parity_error(out, O_) <= 1e-12, H.error_report(out, O_)
    assert pk.counters() == (0, -1)


def test_cfg4_sedov_to_t005_matches_the_similarity_solution():
    # BASELINE configs[3]'s full single-GPU size run to t = 0.05 through the
    # bench's launch configuration (device dt, fused kernels, gather fill):
    # properties that hold at any size (north_star) -- the shock
    # radius within 2 dx of xi0 (E t^2/rho)^(1/5) = 0.3116 (xi0 = 1.032777,
    # tests/exact/sedov.py), mass and energy conserved while the shock is
    # inside the box, octant mirror symmetry to round-off, no floor hits
    from paper_2507_09337_b200 import hydro
    from tests.exact import sedov
    g = H.make_grid(3, NB, NBLK)
    ids = np.arange(g.nblocks)
    pk = hydro.Packet(g, ids)
    U0 = inp.sedov_packet(N, NB, ids)
    pk.pack(U0)
    clock = hydro.DevClock(0.0, 0.05)
    steps = 0
    while True:  # chunks of device-dt steps (no host sync inside a chunk)
        for _ in range(100):
            hydro.orcha_fill_guardcells([pk])
            hydro.orcha_compute_dt_device([pk], clock)
            hydro.orcha_hydro_advance_devdt(pk, clock.dt_tensor)
        steps += 100
        c = clock.read()
        if c.t >= 0.05 or steps > 20000:
            break
    # steps after t_end have dt = 0 and leave the state bitwise unchanged
    assert c.t == 0.05 and c.tag == 1
    out = H.gather(g, [pk])
    dx = 1.0 / N[0]
    rho = out[0]
    xc = (np.arange(N[0]) + 0.5) * dx - 0.5
    r2 = xc[None, None, :] ** 2 + xc[None, :, None] ** 2 + xc[:, None, None] ** 2
    b = (np.sqrt(r2) / dx).astype(int).ravel()
    mean = np.bincount(b, rho.ravel()) / np.bincount(b)
    R = (np.argmax(mean) + 0.5) * dx
    assert abs(R - sedov.shock_radius(0.05, 3)) <= 2 * dx, R
    assert abs(rho.sum() * dx ** 3 - 1.0) <= 1e-12
    E0 = inp.sedov(N)[4].sum()
    assert abs(out[4].sum() - E0) <= 1e-12 * E0
    for d in range(3):
        ax = 3 - d
        M = np.flip(out, axis=ax).copy()
        M[1 + d] = -M[1 + d]
        assert H.parity_error(out, M) <= 1e-12, d
    assert pk.counters() == (0, -1)
