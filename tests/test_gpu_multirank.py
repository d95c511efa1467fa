"""Multi-rank path on one GPU: R virtual ranks (LOCAL transport: the NCCL
path's plan, pack and unpack kernels with device copies instead of
ncclSend/Recv) must give results bitwise identical to the single-domain run
(production build) and to the oracle (parity build).  SURVEY 8(e): "Results
must be bitwise identical across 1/2/4/8 GPUs on the same global grid"."""
import ctypes
import math

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


def _run_virtual(g, U0, owner, nsteps, packets_per_rank=2, dt_mode="host"):
    """R virtual ranks stepping together.  Per step: every rank pushes its
    guard sources, every rank fills; every rank publishes its dt record
    (orcha_comm_push_dt, the LOCAL allgather); then EACH rank computes the
    global dt through its own communicator -- the per-rank record reduction
    the NCCL path runs after its ncclAllGather -- and advances its packets.
    dt_mode "device": orcha_compute_dt_device into a per-rank device clock.
    Returns (state, [(dt, smax, argmax, tag) per step]); asserts every rank
    got the same record."""
    from paper_2507_09337_b200 import hydro
    nd = g.ndim
    n = int(owner.max()) + 1
    comms = hydro.Comm.create_local(g, n, owner)
    pks = []
    for r in range(n):
        ids = np.flatnonzero(owner == r)
        parts = [a for a in np.array_split(ids, packets_per_rank) if len(a)]
        pr = [hydro.Packet(g, p) for p in parts]
        for p in pr:
            p.pack(inp.to_blocks(U0, g.nb[:nd], p.block_ids))
        pks.append(pr)
    allp = [p for pr in pks for p in pr]
    clocks = [hydro.DevClock() for _ in range(n)] if dt_mode == "device" else None
    log = []
    for _ in range(nsteps):
        for r in range(n):
            comms[r].push(pks[r])
        for r in range(n):
            hydro.orcha_fill_guardcells(pks[r], comms[r])
        for r in range(n):
            comms[r].push_dt(pks[r])
        recs = []
        for r in range(n):
            if dt_mode == "device":
                hydro.orcha_compute_dt_device(pks[r], clocks[r], comms[r])
                for p in pks[r]:
                    hydro.orcha_hydro_advance_devdt(p, clocks[r].dt_tensor)
            else:
                info = hydro.orcha_compute_dt(pks[r], math.inf, comms[r])
                recs.append((info.dt, info.smax, info.argmax, info.tag))
                for p in pks[r]:
                    hydro.orcha_hydro_advance(p, info.dt)
        if dt_mode == "device":
            recs = [(c.dt, c.smax, c.argmax, c.tag) for c in (k.read() for k in clocks)]
        assert all(x == recs[0] for x in recs), recs
        log.append(recs[0])
    out = H.gather(g, allp)
    for c in comms:
        c.destroy()
    return out, log


CASES = [
    (3, (8, 8, 8), (4, 2, 2), ((O, O),) * 3, (2, 1, 1), (2, 2, 2)),
    (3, (8, 8, 8), (4, 4, 2), ((P, P), (R, O), (O, R)), (2, 2, 1), (2, 2, 2)),
    (3, (16, 16, 16), (2, 2, 2), ((O, O),) * 3, (2, 2, 2), (1, 1, 1)),
]


@pytest.mark.parametrize("case", CASES)
def test_virtual_ranks_bitwise_equal_single_domain(case):
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = case
    g = H.make_grid(ndim, nb, nblk, bc=bc)
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.sedov(g.N[:ndim]) if bc[0][0] == O else inp.random_field(g.N[:ndim], seed=3)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=5)
    B, logB = _run_virtual(g, U0, owner, 5)
    assert logB == [tuple(x) for x in logA]       # dt, smax, argmax (ties across ranks), tag
    assert np.array_equal(A, B)
    C, logC = _run_virtual(g, U0, owner, 5, dt_mode="device")
    assert logC == logB
    assert np.array_equal(A, C)


@pytest.mark.parametrize("case", CASES)
def test_virtual_ranks_gather_mode_one_packet_per_rank(case):
    # one packet per rank: the gather fill mode runs with remote sources (the
    # exchange writes them into the packet's own guards, stage 1 stages the
    # rest from the resident owners); bitwise the single-domain full fill
    from paper_2507_09337_b200 import abi, hydro
    ndim, nb, nblk, bc, gg, brick = case
    g = H.make_grid(ndim, nb, nblk, bc=bc)
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.random_field(g.N[:ndim], seed=8)
    abi.call(g.lib, "orcha_set_fill_mode", 0)
    try:
        A, _, logA, _ = H.gpu_run(g, U0, nsteps=4)
    finally:
        abi.call(g.lib, "orcha_set_fill_mode", 1)
    B, logB = _run_virtual(g, U0, owner, 4, packets_per_rank=1)
    assert [x[0] for x in logB] == [x[0] for x in logA]
    assert np.array_equal(A, B)


def test_virtual_ranks_gather_mode_scattered_owners():
    # a non-brick owner map: some y/z-guard rows have a remote source while
    # their x-guard parts are resident (the fill's complement pass writes those)
    from paper_2507_09337_b200 import abi
    g = H.make_grid(3, (8, 8, 8), (4, 3, 2), bc=((R, O), (P, P), (O, R)))
    owner = (np.random.default_rng(4).random(g.nblocks) * 3).astype(np.int32)
    owner[:3] = [0, 1, 2]
    U0 = inp.random_field(g.N, seed=9)
    abi.call(g.lib, "orcha_set_fill_mode", 0)
    try:
        A, _, logA, _ = H.gpu_run(g, U0, nsteps=4)
    finally:
        abi.call(g.lib, "orcha_set_fill_mode", 1)
    B, logB = _run_virtual(g, U0, owner, 4, packets_per_rank=1)
    assert [x[0] for x in logB] == [x[0] for x in logA]
    assert np.array_equal(A, B)


def test_virtual_ranks_parity_build_equals_oracle():
    # cfg4's decomposition in miniature: 8 bricks (one Sedov octant each)
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = CASES[2]
    g = H.make_grid(ndim, nb, nblk, bc=bc, parity=True)
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.sedov(g.N)
    B, logB = _run_virtual(g, U0, owner, 4)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4)
    assert [x[0] for x in logB] == olog.dts
    assert [x[2] for x in logB] == olog.argmax   # the 8 octants tie; lowest g wins across ranks
    assert np.array_equal(B, Oo)


def test_virtual_ranks_argmax_tie_across_ranks():
    # 8-octant Sedov, one octant per virtual rank: the maximal signal speed is
    # reached in all 8 octants (bitwise, by symmetry) at step 0, so every rank's
    # record ties on s and the global argmax must be the lowest g, i.e. rank 0's
    # -- through the per-rank record reduction, host and device dt alike
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = CASES[2]
    g = H.make_grid(ndim, nb, nblk, bc=bc, parity=True)
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.sedov(g.N)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=2)
    import oracle
    og = H.oracle_grid(g)
    U = oracle.padded(og, U0)
    oracle.fill_ghosts(og, U)
    r0 = oracle.compute_dt(og, U)
    # the argmax cell is in rank 0's octant and its 7 mirror images tie
    Nx = g.N[0]
    i, j, k = r0.argmax % Nx, (r0.argmax // Nx) % g.N[1], r0.argmax // (Nx * g.N[1])
    assert i < Nx // 2 and j < g.N[1] // 2 and k < g.N[2] // 2
    for mode in ("host", "device"):
        B, logB = _run_virtual(g, U0, owner, 2, dt_mode=mode)
        assert logB[0][2] == r0.argmax and logB[0][0] == r0.dt
        assert [x[2] for x in logB] == olog.argmax


def test_local_comm_destroyed_peer_is_an_error():
    # members are indexed by rank; a push towards a destroyed virtual rank fails
    # instead of writing into another rank's buffer
    from paper_2507_09337_b200 import abi, hydro
    g = H.make_grid(3, (8, 8, 8), (2, 1, 1))
    owner = np.array([0, 1], dtype=np.int32)
    comms = hydro.Comm.create_local(g, 2, owner)
    pk = [hydro.Packet(g, [r]) for r in range(2)]
    U0 = inp.sedov(g.N)
    for r in range(2):
        pk[r].pack(inp.to_blocks(U0, g.nb, [r]))
    comms[1].destroy()
    with pytest.raises(abi.OrchaError, match="destroyed"):
        comms[0].push([pk[0]])
    comms[0].destroy()


def test_nccl_single_rank_communicator():
    # the NCCL code path (dlopen, unique id, init) on one rank: no peers, the
    # fill and dt go through the communicator and match the comm-less run
    from paper_2507_09337_b200 import abi, hydro
    g = H.make_grid(3, (8, 8, 8), (2, 2, 2))
    owner = np.zeros(g.nblocks, dtype=np.int32)
    uid = (ctypes.c_uint8 * 128)()
    abi.call(g.lib, "orcha_comm_unique_id", uid)
    h = ctypes.c_void_p()
    abi.call(g.lib, "orcha_comm_create", g.handle, uid, 1, 0, owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
             ctypes.byref(h))
    comm = hydro.Comm(g, h, 1, 0, owner)
    U0 = inp.sedov(g.N)
    pk = H.gpu_setup(g, U0, npackets=2)
    t, n, log = hydro.run(pk, nsteps=3, comm=comm)
    A = H.gather(g, pk)
    B, _, logB, _ = H.gpu_run(g, U0, nsteps=3)
    assert [x[0] for x in log] == [x[0] for x in logB]
    assert np.array_equal(A, B)
    comm.destroy()


def _run_overlap(g, U0, owner, nsteps):
    """Virtual ranks stepping with orcha_hydro_step_overlap (interior-first slots)."""
    from paper_2507_09337_b200 import hydro
    nd = g.ndim
    n = int(owner.max()) + 1
    comms = hydro.Comm.create_local(g, n, owner)
    pks = []
    for r in range(n):
        ids = hydro.interior_first(g.nblk, [tuple(g.desc.bc[a]) for a in range(3)], owner, r, nd)
        p = hydro.Packet(g, ids)
        p.pack(inp.to_blocks(U0, g.nb[:nd], p.block_ids))
        pks.append(p)
    clocks = [hydro.DevClock() for _ in range(n)]
    log = []
    for _ in range(nsteps):
        for r in range(n):
            comms[r].push([pks[r]])
        for r in range(n):
            comms[r].push_dt([pks[r]])
        for r in range(n):
            hydro.orcha_hydro_step_overlap(pks[r], comms[r], clocks[r])
        recs = [(c.dt, c.smax, c.argmax, c.tag) for c in (k.read() for k in clocks)]
        assert all(x == recs[0] for x in recs), recs
        log.append(recs[0])
    out = H.gather(g, pks)
    for c in comms:
        c.destroy()
    return out, log


@pytest.mark.parametrize("case", CASES)
def test_overlap_step_bitwise_equal_single_domain(case):
    # SURVEY 8(e) "Overlap": stage 1 of the interior blocks runs while the
    # halo is in flight; bitwise the sequential step
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = case
    g = H.make_grid(ndim, nb, nblk, bc=bc)
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.sedov(g.N[:ndim]) if bc[0][0] == O else inp.random_field(g.N[:ndim], seed=33)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=5)
    B, logB = _run_overlap(g, U0, owner, 5)
    assert logB == [tuple(x) for x in logA]
    assert np.array_equal(A, B)


def test_overlap_step_parity_build_equals_oracle():
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = CASES[1]
    g = H.make_grid(ndim, nb, nblk, bc=bc, parity=True)
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.random_field(g.N, seed=34)
    B, logB = _run_overlap(g, U0, owner, 4)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4)
    assert [x[0] for x in logB] == olog.dts
    assert np.array_equal(B, Oo)


def test_overlap_step_scattered_owners_falls_back_bitwise():
    # a non-brick owner map needs the gather fill's complement pass: the call
    # runs the plain sequence, with the same results
    g = H.make_grid(3, (8, 8, 8), (4, 3, 2), bc=((R, O), (P, P), (O, R)))
    owner = (np.random.default_rng(4).random(g.nblocks) * 3).astype(np.int32)
    owner[:3] = [0, 1, 2]
    U0 = inp.random_field(g.N, seed=35)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=3)
    B, logB = _run_overlap(g, U0, owner, 3)
    assert [x[0] for x in logB] == [x[0] for x in logA]
    assert np.array_equal(A, B)
