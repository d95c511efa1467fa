"""The per-stage variant (guard refill between the RK2
stages) through orcha_hydro_stage / orcha_fill_guardcells_stage, against the
oracle's `refill` mode: bitwise in the parity build, <= 1e-12 (c13) in the
production build; equal to the telescoped step under periodic boundaries
(pinned on the oracle: P:L668-674's trick changes nothing there)."""
import numpy as np
import pytest

import orcha_inputs as inp
from tests import gpu_helpers as H
from tests.test_gpu_parity import CASES

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(name, parity, variant=None, npk=None):
    from paper_2507_09337_b200 import hydro
    c = CASES[name]
    g = H.make_grid(c["ndim"], c["nb"], c["nblk"], bc=c.get("bc"), xmax=c.get("xmax", (1.0, 1.0, 1.0)),
                    parity=parity)
    old = g.lib.orcha_get_kernel_variant()
    if variant is not None:
        hydro.set_kernel_variant(g.lib, variant)
    U0 = c["ic"](g.N[:c["ndim"]])
    try:
        G, t, log, pk = H.gpu_run(g, U0, nsteps=c["steps"], npackets=npk or c.get("npk", 1), shuffle=True,
                                  method="per-stage")
    finally:
        hydro.set_kernel_variant(g.lib, old)
    O, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=c["steps"], mode="refill")
    return G, O, log, olog


@pytest.mark.parametrize("name", list(CASES))
def test_per_stage_parity_build_bitwise(name):
    G, O, log, olog = _run(name, True)
    assert [x[0] for x in log] == olog.dts
    assert np.array_equal(G, O)


@pytest.mark.parametrize("name", list(CASES))
def test_per_stage_production_within_1e12(name):
    G, O, log, olog = _run(name, False)
    assert H.parity_error(G, O) <= 1e-12, H.error_report(G, O)


@pytest.mark.parametrize("name", ["sedov3d_32", "random3d_16_mixed"])
def test_per_stage_reference_and_fused_bitwise(name):
    A = _run(name, True, variant=0)[0]
    B = _run(name, True, variant=1)[0]
    assert np.array_equal(A, B)


def test_per_stage_equals_telescoped_on_periodic_domain():
    g = H.make_grid(3, (16, 16, 16), (2, 2, 2), bc=((1, 1),) * 3)
    U0 = inp.random_field(g.N, seed=12)
    A = H.gpu_run(g, U0, nsteps=4, method="telescoped")[0]
    B = H.gpu_run(g, U0, nsteps=4, method="per-stage")[0]
    assert np.array_equal(A, B)


def test_per_stage_call_order_is_enforced():
    from paper_2507_09337_b200 import abi, hydro
    g = H.make_grid(3, (8, 8, 8), (2, 2, 2))
    pk = H.gpu_setup(g, inp.sedov(g.N))
    hydro.orcha_fill_guardcells(pk)
    hydro.orcha_hydro_stage(pk[0], 1, 1e-5)
    with pytest.raises(abi.OrchaError) as e:
        hydro.orcha_hydro_stage(pk[0], 2, 1e-5)       # U1 guards not refilled
    assert e.value.status == "ORCHA_E_STATE"
    hydro.orcha_fill_guardcells_stage(pk, 1)
    hydro.orcha_hydro_stage(pk[0], 2, 1e-5)
    with pytest.raises(abi.OrchaError):
        hydro.orcha_fill_guardcells_stage(pk, 1)      # no stage 1 pending


@pytest.mark.parametrize("owners", ["brick", "scattered"])
def test_per_stage_virtual_ranks_bitwise_equal_single_domain(owners):
    # one packet per virtual rank: the gather fill mode with remote sources,
    # for the state and the stage-1 buffer (the scattered map needs the
    # complement pass for exchanged rows with resident x-guard sources)
    from paper_2507_09337_b200 import hydro
    nb, nblk = (8, 8, 8), (4, 4, 2)
    bc = ((1, 1), (2, 0), (0, 2))
    g = H.make_grid(3, nb, nblk, bc=bc)
    if owners == "brick":
        owner = hydro.brick_owner(nblk, (2, 2, 2), (2, 2, 1))
    else:
        owner = (np.random.default_rng(6).random(g.nblocks) * 4).astype(np.int32)
        owner[:4] = [0, 1, 2, 3]
    U0 = inp.random_field(g.N, seed=8)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=3, method="per-stage")
    comms = hydro.Comm.create_local(g, 4, owner)
    pks = []
    for r in range(4):
        ids = np.flatnonzero(owner == r)
        p = hydro.Packet(g, ids)
        p.pack(inp.to_blocks(U0, nb, ids))
        pks.append([p])
    allp = [p for pr in pks for p in pr]
    for _ in range(3):
        for r in range(4):
            comms[r].push(pks[r], buffer=0)
        for r in range(4):
            hydro.orcha_fill_guardcells(pks[r], comms[r])
        info = hydro.orcha_compute_dt(allp)
        for p in allp:
            hydro.orcha_hydro_stage(p, 1, info.dt)
        for r in range(4):
            comms[r].push(pks[r], buffer=1)
        for r in range(4):
            hydro.orcha_fill_guardcells_stage(pks[r], 1, comms[r])
        for p in allp:
            hydro.orcha_hydro_stage(p, 2, info.dt)
    B = H.gather(g, allp)
    for c in comms:
        c.destroy()
    assert np.array_equal(A, B)
