"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
the same seeded/closed-form inputs.  Parity build (liborcha_parity.so,
--fmad=false): bitwise.  Production build (liborcha.so): <= 1e-12 by the
SURVEY 8(c) c13 metric.  Bookkeeping (pack/unpack, guard values, dt argmax)
is bitwise in both."""
import math

import numpy as np
import pytest

import oracle
import orcha_inputs as inp
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu
TOL = 1e-12
O, P, R = 0, 1, 2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_09337_b200 import build
    build.build()


# ----------------------------------------------------------- bookkeeping --

@pytest.mark.parametrize("ndim,nb,nblk", [(1, (16,), (8,)), (2, (8, 8), (4, 4)), (3, (8, 8, 8), (2, 3, 2)),
                                          (3, (16, 16, 16), (2, 2, 2))])
def test_pack_unpack_roundtrip_bitwise(ndim, nb, nblk):
    # unpack(pack(x)) restores x bitwise (random data, shuffled slots)
    g = H.make_grid(ndim, nb, nblk)
    rng = np.random.default_rng(3)
    U = rng.normal(size=(5,) + tuple(reversed([g.N[a] for a in range(3)])))
    pk = H.gpu_setup(g, U, npackets=3, shuffle=True)
    back = H.gather(g, pk)
    assert np.array_equal(back, U)


@pytest.mark.parametrize("bcode", [O, P, R])
@pytest.mark.parametrize("ndim,nb,nblk", [(1, (8,), (4,)), (2, (8, 8), (4, 3)), (3, (8, 8, 8), (3, 2, 2))])
@pytest.mark.parametrize("npk", [1, 3])
def test_guard_fill_equals_global_ghost_fill(bcode, ndim, nb, nblk, npk):
    # every guard cell (faces, edges, corners) equals the
    # oracle's axis-ordered global ghost fill at the same global coordinate
    bc = ((bcode, bcode),) * 3
    g = H.make_grid(ndim, nb, nblk, bc=bc)
    og = H.oracle_grid(g)
    U0 = inp.random_field(g.N[:ndim], seed=9)
    pk = H.gpu_setup(g, U0, npackets=npk, shuffle=True)
    from paper_2507_09337_b200 import abi, hydro
    abi.call(g.lib, "orcha_set_fill_mode", 0)   # FULL: materialise every guard
    try:
        hydro.orcha_fill_guardcells(pk)
    finally:
        abi.call(g.lib, "orcha_set_fill_mode", 1)
    Ug = oracle.padded(og, U0)
    oracle.fill_ghosts(og, Ug)
    ng = 4
    for p in pk:
        S = p.state_view().cpu().numpy()
        for s, b in enumerate(p.block_ids):
            bi = b % g.nblk[0]
            bj = (b // g.nblk[0]) % g.nblk[1]
            bk = b // (g.nblk[0] * g.nblk[1])
            sl = [slice(None)]
            for a, bcoord in ((2, bk), (1, bj), (0, bi)):
                if a < ndim:
                    lo = bcoord * g.nb[a]
                    sl.append(slice(lo, lo + g.nb[a] + 2 * ng))
                else:
                    sl.append(slice(0, 1))
            assert np.array_equal(S[s], Ug[tuple(sl)]), (s, b)


def test_dt_bitwise_and_tiebreak():
    # A4: dt, smax and the lowest-g argmax over Sedov's tied deposit cells
    for parity in (True, False):
        g = H.make_grid(2, (8, 8), (4, 4), parity=parity)
        og = H.oracle_grid(g)
        U0 = inp.sedov(g.N[:2])
        pk = H.gpu_setup(g, U0, npackets=3, shuffle=True)
        from paper_2507_09337_b200 import hydro
        info = hydro.orcha_compute_dt(pk)
        r = oracle.compute_dt(og, oracle.padded(og, U0))
        if parity:
            assert info.dt == r.dt and info.smax == r.smax
        else:
            assert abs(info.dt - r.dt) <= 1e-13 * r.dt
        assert info.argmax == r.argmax and info.tag == oracle.TAG_CFL
        info2 = hydro.orcha_compute_dt(pk, t_remaining=1e-5)
        assert info2.dt == 1e-5 and info2.tag == oracle.TAG_CLAMP


# ------------------------------------------------------ whole-step parity --

CASES = {
    # BASELINE configs[0]: 2D Sedov, 4x4 blocks of 8x8, 10 steps
    "cfg1_sedov2d": dict(ndim=2, nb=(8, 8), nblk=(4, 4), ic=lambda N: inp.sedov(N), steps=10),
    # BASELINE configs[1] (10-step parity): 1D Sod 64 blocks x 16; 2D tube 64x1 blocks of 16^2
    "cfg2_sod1d": dict(ndim=1, nb=(16,), nblk=(64,), ic=lambda N: inp.sod(N), steps=10),
    "cfg2_sod2d_tube": dict(ndim=2, nb=(16, 16), nblk=(64, 1), ic=lambda N: inp.sod(N), steps=10,
                            bc=((O, O), (P, P), (O, O)), xmax=(1.0, 16 / 1024)),
    # small 3D Sedov spanning several blocks with ragged packet split
    "sedov3d_32": dict(ndim=3, nb=(8, 8, 8), nblk=(4, 4, 4), ic=lambda N: inp.sedov(N), steps=10, npk=3),
    # rough random field, periodic / reflecting walls: every limiter and HLL branch
    "random3d_periodic": dict(ndim=3, nb=(8, 8, 8), nblk=(2, 3, 2), ic=lambda N: inp.random_field(N, seed=4),
                              steps=6, bc=((P, P),) * 3, npk=2),
    "random2d_reflect": dict(ndim=2, nb=(8, 8), nblk=(3, 2), ic=lambda N: inp.random_field(N, seed=5),
                             steps=6, bc=((R, R), (R, O), (O, O))),
    "random3d_16_mixed": dict(ndim=3, nb=(16, 16, 16), nblk=(2, 2, 1), ic=lambda N: inp.random_field(N, seed=6),
                              steps=4, bc=((P, P), (R, O), (O, R))),
}


def _run_case(name, parity, variant=None):
    c = CASES[name]
    g = H.make_grid(c["ndim"], c["nb"], c["nblk"], bc=c.get("bc"), xmax=c.get("xmax", (1.0, 1.0, 1.0)),
                    parity=parity)
    from paper_2507_09337_b200 import hydro
    old = g.lib.orcha_get_kernel_variant()
    if variant is not None:
        hydro.set_kernel_variant(g.lib, variant)
    og = H.oracle_grid(g)
    U0 = c["ic"](g.N[:c["ndim"]])
    try:
        Gout, t, log, pk = H.gpu_run(g, U0, nsteps=c["steps"], npackets=c.get("npk", 1), shuffle=True)
    finally:
        hydro.set_kernel_variant(g.lib, old)
    Oout, olog = H.oracle_run(og, U0, nsteps=c["steps"])
    return Gout, Oout, t, log, olog, pk


@pytest.mark.parametrize("name", list(CASES))
def test_parity_build_bitwise(name):
    G, Oo, t, log, olog, pk = _run_case(name, parity=True)
    assert [x[0] for x in log] == olog.dts                      # dt bitwise every step (c14)
    assert [x[2] for x in log] == olog.argmax                   # argmax (lowest g)
    assert np.array_equal(G, Oo)


@pytest.mark.parametrize("name", list(CASES))
def test_production_build_within_1e12(name):
    G, Oo, t, log, olog, pk = _run_case(name, parity=False)
    err = H.parity_error(G, Oo)
    assert err <= TOL, (err, H.error_report(G, Oo))
    for (dt, smax, am, tag), odt in zip(log, olog.dts):
        assert abs(dt - odt) <= 1e-13 * odt
    fh, bad = pk[0].counters()
    assert bad == -1


@pytest.mark.parametrize("name", ["cfg1_sedov2d", "sedov3d_32", "random3d_16_mixed"])
def test_reference_and_fused_variants_bitwise(name):
    A = _run_case(name, parity=True, variant=0)[0]
    B = _run_case(name, parity=True, variant=1)[0]
    assert np.array_equal(A, B)


def test_decomposition_invariance_production():
    # bitwise identical across packet sizes / splits (same per-cell code)
    g = H.make_grid(3, (8, 8, 8), (4, 4, 4))
    U0 = inp.sedov(g.N)
    A = H.gpu_run(g, U0, nsteps=5, npackets=1)[0]
    B = H.gpu_run(g, U0, nsteps=5, npackets=7, shuffle=True)[0]
    assert np.array_equal(A, B)


def test_state_errors():
    from paper_2507_09337_b200 import abi, hydro
    g = H.make_grid(2, (8, 8), (2, 2))
    U0 = inp.sedov(g.N[:2])
    pk = H.gpu_setup(g, U0)
    with pytest.raises(abi.OrchaError) as e:
        hydro.orcha_hydro_advance(pk[0], 1e-4)          # no fill since pack
    assert e.value.status == "ORCHA_E_STATE"
    # a lone packet whose neighbours are not resident and no communicator
    g2 = H.make_grid(2, (8, 8), (2, 2))
    p = hydro.Packet(g2, [0])
    with pytest.raises(abi.OrchaError) as e:
        hydro.orcha_fill_guardcells([p])
    assert e.value.status == "ORCHA_E_RANGE"
    # non-positive density is latched and reported (SPEC NonPositiveState)
    U1 = U0.copy()
    U1[0, 0, 3, 5] = -1.0
    pk = H.gpu_setup(g, U1)
    hydro.orcha_fill_guardcells(pk)
    info = hydro.orcha_compute_dt(pk, check=False)
    assert info.nonphysical == 1
    with pytest.raises(abi.OrchaError) as e:
        pk[0].unpack()
    assert e.value.status == "ORCHA_E_NONPHYSICAL"


def test_sod_to_t02_against_exact_solution():
    # the whole GPU scheme to t = 0.2 against Toro's exact solution (BASELINE configs[1])
    from tests.exact import riemann
    g = H.make_grid(1, (16,), (64,))
    G, t, log, pk = H.gpu_run(g, inp.sod((1024,)), t_end=0.2)
    assert t == 0.2 and log[-1][3] == oracle.TAG_CLAMP
    ex = riemann.cell_averages(1024, 0.2, 0.5, (1, 0, 1), (0.125, 0, 0.1))
    assert np.abs(G[0, 0, 0] - ex[0]).mean() <= 1.5e-3
