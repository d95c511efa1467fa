"""Borrowed-ring telescoped step (orcha_set_ring_mode(1), the default;
include/orcha.h, fused_impl.cuh launch_hybrid_nb) against the oracle's
telescoped step (sec 6: stage 1 on the block plus the inner
2 cells of the halo, no second guard exchange).

A block computes its stage-1 ring only on "self" sides (physical boundary,
or a neighbour on another rank) and borrows it from the owning block on every
other side.  The claim is that this is the telescoped step itself: the parity
build is bitwise the oracle's telescoped mode (state, dt and argmax every
step) for every boundary kind, 8^3 / 16^3 / 32^3 blocks, shuffled slot
orders, one block along an axis, packets with no self side (all periodic) and
with only self sides, the F4 scheme variants, supersonic flow, virtual ranks
(remote sides are self sides), several packets per device and the full fill
mode (sides towards another packet are self sides).  The production build is checked against
the oracle by the c13 metric and against the literal ring (mode 0)."""
import numpy as np
import pytest

import orcha_inputs as inp
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu
O, P, R = 0, 1, 2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ring(lib, m):
    from paper_2507_09337_b200 import abi
    abi.call(lib, "orcha_set_ring_mode", m)


CASES = {
    # (block size, blocks per axis, bc, initial condition, steps)
    "sedov16_4": ((16, 16, 16), (4, 4, 4), ((O, O),) * 3, "sedov", 6),
    "mixed16": ((16, 16, 16), (3, 2, 2), ((R, O), (O, R), (P, P)), "random", 5),
    "mixed8": ((8, 8, 8), (4, 3, 3), ((O, O), (P, P), (R, R)), "random", 6),
    "mixed32": ((32, 32, 32), (2, 2, 1), ((O, R), (P, P), (R, O)), "random", 3),
    "one_along_x": ((16, 16, 16), (1, 3, 2), ((P, P), (R, R), (O, O)), "random", 5),
    "all_periodic": ((16, 16, 16), (2, 2, 2), ((P, P),) * 3, "supersonic", 6),
    "all_self": ((8, 8, 8), (1, 1, 2), ((O, O), (R, R), (O, O)), "random", 6),
    "supersonic_out": ((16, 16, 16), (3, 2, 2), ((O, O), (P, P), (O, R)), "supersonic", 6),
}


def _ic(kind, N, seed):
    if kind == "sedov":
        return inp.sedov(N)
    if kind == "supersonic":
        return inp.supersonic_field(N, seed=seed)
    return inp.random_field(N, seed=seed)


@pytest.mark.parametrize("shuffle", [False, True])
@pytest.mark.parametrize("name", list(CASES))
def test_parity_build_equals_oracle_telescoped(name, shuffle):
    nb, nblk, bc, ic, steps = CASES[name]
    g = H.make_grid(3, nb, nblk, bc=bc, parity=True)
    _ring(g.lib, 1)
    U0 = _ic(ic, g.N, seed=61)
    G, t, log, pk = H.gpu_run(g, U0, nsteps=steps, shuffle=shuffle)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=steps)
    assert [x[0] for x in log] == olog.dts
    assert [x[2] for x in log] == olog.argmax
    assert np.array_equal(G, Oo)


@pytest.mark.parametrize("nb,nblk", [((16, 16, 16), (3, 2, 2)), ((8, 8, 8), (4, 3, 2)), ((32, 32, 32), (2, 1, 2))])
@pytest.mark.parametrize("variant", [dict(riemann=1), dict(limiter=1), dict(eos=1, eos_work=1, arad=1e-3)])
def test_parity_build_scheme_variants(variant, nb, nblk):
    g = H.make_grid(3, nb, nblk, bc=((O, R), (P, P), (R, O)), parity=True, **variant)
    _ring(g.lib, 1)
    U0 = inp.supersonic_field(g.N, seed=62)
    G, t, log, pk = H.gpu_run(g, U0, nsteps=4)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4)
    assert [x[0] for x in log] == olog.dts
    assert np.array_equal(G, Oo)


@pytest.mark.parametrize("name", ["sedov16_4", "mixed8", "supersonic_out", "mixed32"])
def test_production_against_oracle_and_literal_ring(name):
    nb, nblk, bc, ic, steps = CASES[name]
    g = H.make_grid(3, nb, nblk, bc=bc)
    U0 = _ic(ic, g.N, seed=63)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=steps)
    try:
        _ring(g.lib, 0)
        B, _, logB, _ = H.gpu_run(g, U0, nsteps=steps)
        _ring(g.lib, 1)
        A, _, logA, _ = H.gpu_run(g, U0, nsteps=steps)
    finally:
        _ring(g.lib, 1)
    assert H.parity_error(A, Oo) <= 1e-12, H.error_report(A, Oo)
    assert H.parity_error(A, B) <= 1e-12, H.error_report(A, B)
    for (dt, smax, am, tag), odt, oam in zip(logA, olog.dts, olog.argmax):
        assert abs(dt - odt) <= 1e-13 * odt
        assert am == oam


def test_launches_per_advance():
    # a packet with both kinds of blocks: box stage 1 (self sides), interior
    # stage 1, stage 2 -- three launches; the literal ring: two
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, (8, 8, 8), (4, 4, 4), bc=((O, O),) * 3)
    pk = H.gpu_setup(g, inp.sedov(g.N))
    counts = {}
    try:
        for m in (1, 0, 1):
            _ring(g.lib, m)
            hydro.orcha_fill_guardcells(pk)
            info = hydro.orcha_compute_dt(pk)
            n0 = g.lib.orcha_launch_count()
            hydro.orcha_hydro_advance(pk[0], info.dt)
            counts.setdefault(m, []).append(g.lib.orcha_launch_count() - n0)
    finally:
        _ring(g.lib, 1)
    assert counts == {1: [3, 3], 0: [2]}


def test_ring_mode_argument_checked():
    from paper_2507_09337_b200 import abi
    g = H.make_grid(3, (8, 8, 8), (1, 1, 1))
    with pytest.raises(abi.OrchaError) as e:
        abi.call(g.lib, "orcha_set_ring_mode", 2)
    assert e.value.status == "ORCHA_E_ARG"
    assert g.lib.orcha_get_ring_mode() == 1


def test_virtual_ranks_parity_build_equals_oracle():
    # one packet per virtual rank (gather mode with remote sides: those are
    # self sides, computed from the exchanged guards -- no second exchange)
    from paper_2507_09337_b200 import hydro
    from tests.test_gpu_multirank import _run_virtual
    nblk = (4, 4, 2)
    g = H.make_grid(3, (8, 8, 8), nblk, bc=((P, P), (R, O), (O, R)), parity=True)
    _ring(g.lib, 1)
    owner = hydro.brick_owner(nblk, (2, 2, 2), (2, 2, 1))
    U0 = inp.random_field(g.N, seed=64)
    B, logB = _run_virtual(g, U0, owner, 4, packets_per_rank=1)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4)
    assert [x[0] for x in logB] == olog.dts
    assert np.array_equal(B, Oo)


@pytest.mark.parametrize("npackets,shuffle", [(2, False), (3, True), (5, True)])
@pytest.mark.parametrize("name", ["mixed16", "mixed8", "mixed32", "sedov16_4", "all_periodic"])
def test_multi_packet_parity_build_equals_oracle(name, npackets, shuffle):
    # several packets per device (full fill mode): a side towards another
    # packet is a self side (that packet's stage 1 is another launch)
    nb, nblk, bc, ic, steps = CASES[name]
    g = H.make_grid(3, nb, nblk, bc=bc, parity=True)
    U0 = _ic(ic, g.N, seed=65)
    G, t, log, pk = H.gpu_run(g, U0, nsteps=steps, npackets=npackets, shuffle=shuffle)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=steps)
    assert [x[0] for x in log] == olog.dts
    assert np.array_equal(G, Oo)


@pytest.mark.parametrize("name", ["mixed16", "mixed32"])
def test_full_fill_one_packet_parity_build_equals_oracle(name):
    # the borrowed ring over the packet's materialised guards (no gather)
    from paper_2507_09337_b200 import abi
    nb, nblk, bc, ic, steps = CASES[name]
    g = H.make_grid(3, nb, nblk, bc=bc, parity=True)
    abi.call(g.lib, "orcha_set_fill_mode", 0)
    U0 = _ic(ic, g.N, seed=66)
    G, t, log, pk = H.gpu_run(g, U0, nsteps=steps)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=steps)
    assert [x[0] for x in log] == olog.dts
    assert np.array_equal(G, Oo)


def test_multi_packet_production_against_literal_ring():
    nb, nblk, bc, ic, steps = CASES["sedov16_4"]
    g = H.make_grid(3, nb, nblk, bc=bc)
    U0 = _ic(ic, g.N, seed=67)
    try:
        _ring(g.lib, 0)
        B, _, logB, _ = H.gpu_run(g, U0, nsteps=steps, npackets=4)
        _ring(g.lib, 1)
        A, _, logA, _ = H.gpu_run(g, U0, nsteps=steps, npackets=4)
    finally:
        _ring(g.lib, 1)
    assert H.parity_error(A, B) <= 1e-12, H.error_report(A, B)
    for a, b in zip(logA, logB):
        assert abs(a[0] - b[0]) <= 1e-13 * b[0] and a[2] == b[2]


@pytest.mark.parametrize("name,npackets", [("mixed16", 1), ("mixed8", 1), ("sedov16_4", 3), ("one_along_x", 1)])
def test_every_u1_cell_stage2_reads_is_written_each_step(name, npackets):
    # the U1 cubes are poisoned (NaN bytes) before every advance: a stage-2
    # read of a ring cell that no stage-1 launch of this step wrote (neither
    # the block on a self side nor the owner's push) would spread NaN
    import math
    import torch
    from paper_2507_09337_b200 import hydro
    nb, nblk, bc, ic, steps = CASES[name]
    g = H.make_grid(3, nb, nblk, bc=bc, parity=True)
    U0 = _ic(ic, g.N, seed=68)
    pk = H.gpu_setup(g, U0, npackets, shuffle=True)
    u1_cube = ((nb[0] + 4) ** 3 * 8 + 255) // 256 * 256
    dts = []
    for _ in range(4):
        hydro.orcha_fill_guardcells(pk)
        info = hydro.orcha_compute_dt(pk, math.inf)
        for p in pk:
            p.scratch[: len(p.block_ids) * 5 * u1_cube].fill_(0xFF)
        for p in pk:
            hydro.orcha_hydro_advance(p, info.dt)
        dts.append(info.dt)
    torch.cuda.synchronize()
    G = H.gather(g, pk)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4)
    assert dts == olog.dts
    assert np.array_equal(G, Oo)


def test_production_run_is_deterministic():
    # each U1 cell has one writer per step (the block, or the owner's push;
    # the two stage-1 launches run concurrently on two streams): two runs agree
    # (cfg3: 512 blocks, 216 interior -- large enough for the two-stream launch)
    g = H.make_grid(3, (16, 16, 16), (8, 8, 8), bc=((O, O),) * 3)
    U0 = inp.sedov(g.N)
    A = H.gpu_run(g, U0, nsteps=8)[0]
    B = H.gpu_run(g, U0, nsteps=8)[0]
    assert np.array_equal(A, B)
