"""BASELINE.json configs[4] as a parity case: the same global 3D Sedov grid
decomposed into 8^3, 16^3 or 32^3 blocks and split into packets of 8 ... all
blocks (sec 4.3: "n is provided by the users at runtime") gives
the oracle's global result bitwise (parity build) for every block size and
packet size, and bitwise-identical results across packet sizes in the
production build (determinism across packet sizes)."""
import numpy as np
import pytest

import orcha_inputs as inp
from tests import gpu_helpers as H

O, P, R = 0, 1, 2

pytestmark = pytest.mark.gpu
N = (64, 64, 64)
STEPS = 4


@pytest.fixture(scope="module")
def oracle_ref():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g = H.make_grid(3, (16, 16, 16), (4, 4, 4))
    return H.oracle_run(H.oracle_grid(g), inp.sedov(N), nsteps=STEPS)


def _run(nb, packet_size, parity):
    from paper_2507_09337_b200 import hydro
    nblk = tuple(n // nb for n in N)
    g = H.make_grid(3, (nb,) * 3, nblk, parity=parity)
    ids = np.random.default_rng(nb + packet_size).permutation(g.nblocks)
    parts = [ids[i:i + packet_size] for i in range(0, len(ids), packet_size)]
    pk = [hydro.Packet(g, p) for p in parts]
    for p in pk:
        p.pack(inp.sedov_packet(N, (nb,) * 3, p.block_ids))
    t, n, log = hydro.run(pk, nsteps=STEPS)
    return H.gather(g, pk), log


@pytest.mark.parametrize("nb,packet_size", [(8, 8), (8, 64), (8, 512), (16, 8), (16, 64), (32, 8)])
def test_packet_sweep_parity_build_bitwise(oracle_ref, nb, packet_size):
    O, olog = oracle_ref
    G, log = _run(nb, packet_size, True)
    assert [x[0] for x in log] == olog.dts
    assert np.array_equal(G, O)


@pytest.mark.parametrize("nb", [8, 16, 32])
def test_packet_sizes_bitwise_identical_production(oracle_ref, nb):
    O, _ = oracle_ref
    nblocks = (64 // nb) ** 3
    ref, _ = _run(nb, nblocks, False)
    assert H.parity_error(ref, O) <= 1e-12
    for ps in (8, max(8, nblocks // 3)):
        if ps >= nblocks:
            continue
        G, _ = _run(nb, ps, False)
        assert np.array_equal(G, ref)


def test_many_packets_one_launch_fill_and_dt():
    # >= 128 packets: the fill runs as one launch over every slot of the set
    # and dt as one reduction over every packet's records -- bitwise the same
    # as one packet, and the launch count shows the batching
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, (8, 8, 8), (8, 8, 4), bc=((R, O), (P, P), (O, R)))
    U0 = inp.random_field(g.N, seed=44)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=3)
    pk = H.gpu_setup(g, U0, npackets=128, shuffle=True)
    n0 = g.lib.orcha_launch_count()
    hydro.orcha_fill_guardcells(pk)
    assert g.lib.orcha_launch_count() - n0 == 1
    t, n, log = hydro.run(pk, nsteps=3)
    assert [x[0] for x in log] == [x[0] for x in logA]
    assert np.array_equal(H.gather(g, pk), A)


@pytest.mark.parametrize("parity", [False, True])
@pytest.mark.parametrize("pipelined", [False, True])
def test_streamed_host_mesh_equals_resident_run(pipelined, parity):
    # SURVEY 8(f) F3 / bench.py's e2e: the mesh lives in pinned host memory as
    # K packets shipped in (H2D streams), advanced, and shipped out with
    # orcha_packet_unpack_async (D2H streams) every step, the next step reading
    # the host mesh -- bitwise the device-resident run.  pipelined: each slab's
    # dt records right after its pack and its guard fill right after the next
    # slab's pack (orcha_packet_dt_records / orcha_fill_guardcells_packet;
    # z is not periodic, so a slab's guards read only its neighbour slabs),
    # packets alternating over two copy streams each way.  Parity build: also
    # bitwise the oracle (state and every dt).
    import math
    import torch
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, (8, 8, 8), (4, 4, 4), bc=((R, O), (P, P), (O, R)), parity=parity)
    U0 = inp.random_field(g.N, seed=51)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=4)
    slabs = [a for a in np.array_split(np.arange(g.nblocks), 4)]
    pks = [hydro.Packet(g, a) for a in slabs]
    mesh = [torch.from_numpy(inp.to_blocks(U0, g.nb, a)).pin_memory() for a in slabs]
    comp = torch.cuda.current_stream()
    ns = 2 if pipelined else 1
    h2ds = [torch.cuda.Stream() for _ in range(ns)]
    d2hs = [torch.cuda.Stream() for _ in range(ns)]
    done = [None] * len(pks)
    dts = []
    for _ in range(4):
        ev = []
        for i, p in enumerate(pks):
            h2d = h2ds[i % ns]
            if done[i] is not None:
                h2d.wait_event(done[i])
            p.pack(mesh[i], h2d)
            e = torch.cuda.Event()
            e.record(h2d)
            ev.append(e)
            if pipelined:
                comp.wait_event(e)
                hydro.orcha_packet_dt_records(p, comp)
                if i >= 1:
                    hydro.orcha_fill_guardcells_packet(pks, i - 1, comp)
        if pipelined:
            hydro.orcha_fill_guardcells_packet(pks, len(pks) - 1, comp)
        else:
            for e in ev:
                comp.wait_event(e)
            hydro.orcha_fill_guardcells(pks, None, comp)
        n0 = g.lib.orcha_launch_count()
        info = hydro.orcha_compute_dt(pks, math.inf, None, comp)
        if pipelined:  # the records were computed per packet: only the reduction runs
            assert g.lib.orcha_launch_count() - n0 == 1
        dts.append(info.dt)
        for i, p in enumerate(pks):
            hydro.orcha_hydro_advance(p, info.dt, comp)
            e = torch.cuda.Event()
            e.record(comp)
            d2h = d2hs[i % ns]
            d2h.wait_event(e)
            p.unpack(mesh[i], d2h, sync=False)
            e2 = torch.cuda.Event()
            e2.record(d2h)
            done[i] = e2
    torch.cuda.synchronize()
    out = None
    for a, m in zip(slabs, mesh):
        out = inp.from_blocks(m.numpy(), g.N, g.nb, a, out)
    assert dts == [x[0] for x in logA]
    assert np.array_equal(out, A)
    if parity:
        Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4)
        assert dts == olog.dts
        assert np.array_equal(out, Oo)


def test_per_packet_fill_arguments():
    from paper_2507_09337_b200 import abi, hydro
    g = H.make_grid(3, (8, 8, 8), (2, 2, 2))
    pks = [hydro.Packet(g, [b]) for b in range(g.nblocks)]
    for bad in (-1, len(pks)):
        with pytest.raises(abi.OrchaError, match="ORCHA_E_ARG"):
            hydro.orcha_fill_guardcells_packet(pks, bad)


@pytest.mark.parametrize("parity", [False, True])
def test_bench_streamed_loop_equals_resident_run_and_oracle(parity):
    # bench.py's own e2e loop (streamed_loop: the lagged pipeline -- each
    # slab's fill after the next slab's pack, its advance + unpack after the
    # following fill, the step's dt reduced at the end of the previous step
    # from the stage-2 records) on a 16^3-block grid of 4 z-slabs: the host
    # mesh after 4 steps is bitwise the device-resident run (and, parity
    # build, the oracle), with the same dt every step
    import math
    import sys
    import torch
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, (16, 16, 16), (2, 2, 4), parity=parity)
    N = g.N
    ids = np.arange(g.nblocks)
    U0 = inp.sedov(N)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=4)
    s = torch.cuda.current_stream()
    pks, mesh, one, done = bench.streamed_loop(g, ids, N, 1, 1, 1, None, s, 4, copy_priority=-1, copy_streams=2)
    one.prime()
    torch.cuda.synchronize()
    for _ in range(4):
        one()
    torch.cuda.synchronize()
    out = None
    for p, m in zip(pks, mesh):
        out = inp.from_blocks(m.numpy(), N, g.nb, p.block_ids, out)
    assert np.array_equal(out, A)
    if parity:
        Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4)
        assert np.array_equal(out, Oo)
