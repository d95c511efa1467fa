"""F2 peer mode (the guard fill reads peer ranks' packets
directly over NVLink instead of exchanging them; dt by a one-shot peer write),
exercised on one GPU with virtual ranks whose packets are separate
allocations ("same-device peers"), each rank on its own CUDA stream so the
device-side barriers between ranks really synchronise concurrent work.
Bitwise equal to the single-domain run and (parity build) to the oracle; no
exchange kernel runs; a rank that never arrives times out into an error
instead of hanging.  P:L663-664, P:L694-695 (sec 6, 6.1)."""
import math
import threading

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


def _setup(g, U0, owner):
    import torch
    from paper_2507_09337_b200 import hydro
    n = int(owner.max()) + 1
    comms = hydro.Comm.create_local(g, n, owner)
    streams = [torch.cuda.Stream() for _ in range(n)]
    pks = []
    for r in range(n):
        p = hydro.Packet(g, np.flatnonzero(owner == r))
        p.pack(inp.to_blocks(U0, g.nb[:g.ndim], p.block_ids), streams[r])
        comms[r].peer_register(p)
        pks.append(p)
    # the fill plans (device tables) before any rank's first barrier: an
    # allocation between two ranks' launches would serialise their streams
    for r in range(n):
        hydro.orcha_fill_prepare([pks[r]], comms[r])
    torch.cuda.synchronize()
    return comms, streams, pks


def _run_peer(g, U0, owner, nsteps, method="telescoped"):
    """Device-dt loop, ranks interleaved on their own streams."""
    import torch
    from paper_2507_09337_b200 import hydro
    comms, streams, pks = _setup(g, U0, owner)
    n = len(pks)
    clocks = [hydro.DevClock() for _ in range(n)]
    log = []
    launches = []
    for _ in range(nsteps):
        c0 = g.lib.orcha_launch_count()
        if method == "per-stage":
            # F1 in peer mode: the U1 "refill" is the barrier between the stages
            for r in range(n):
                hydro.orcha_fill_guardcells_stage([pks[r]], 0, comms[r], streams[r])
            for r in range(n):
                hydro.orcha_compute_dt_device([pks[r]], clocks[r], comms[r], streams[r])
            for r in range(n):
                hydro.orcha_hydro_stage_devdt(pks[r], 1, clocks[r].dt_tensor, streams[r])
            for r in range(n):
                hydro.orcha_fill_guardcells_stage([pks[r]], 1, comms[r], streams[r])
            for r in range(n):
                hydro.orcha_hydro_stage_devdt(pks[r], 2, clocks[r].dt_tensor, streams[r])
        else:
            for r in range(n):
                hydro.orcha_fill_guardcells([pks[r]], comms[r], streams[r])
            for r in range(n):
                hydro.orcha_compute_dt_device([pks[r]], clocks[r], comms[r], streams[r])
            for r in range(n):
                hydro.orcha_hydro_advance_devdt(pks[r], clocks[r].dt_tensor, streams[r])
        torch.cuda.synchronize()
        launches.append(g.lib.orcha_launch_count() - c0)
        recs = [(c.dt, c.smax, c.argmax, c.tag) for c in (k.read() for k in clocks)]
        assert all(x == recs[0] for x in recs), recs
        log.append(recs[0])
    for c in comms:
        c.check()
    out = H.gather(g, pks)
    for c in comms:
        c.destroy()
    return out, log, launches


CASES = [
    (3, (8, 8, 8), (4, 2, 2), ((O, O),) * 3, (2, 1, 1), (2, 2, 2)),
    (3, (8, 8, 8), (4, 4, 2), ((P, P), (R, O), (O, R)), (2, 2, 1), (2, 2, 2)),
    (3, (16, 16, 16), (2, 2, 2), ((O, O),) * 3, (2, 2, 2), (1, 1, 1)),
    (3, (32, 32, 32), (2, 1, 1), ((P, P), (O, O), (O, O)), (2, 1, 1), (1, 1, 1)),
]


@pytest.mark.parametrize("case", CASES)
def test_peer_mode_bitwise_equal_single_domain(case):
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = case
    g = H.make_grid(ndim, nb, nblk, bc=bc)
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.sedov(g.N) if bc[0][0] == O else inp.random_field(g.N, seed=71)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=5)
    B, logB, launches = _run_peer(g, U0, owner, 5)
    assert logB == [tuple(x) for x in logA]
    assert np.array_equal(A, B)
    # steady state per rank and step: dt reduce + record + barrier + finish,
    # stage 1 + barrier + stage 2 -- no fill, pack, exchange or unpack kernel
    n = int(owner.max()) + 1
    assert launches[-1] == 7 * n, launches


@pytest.mark.parametrize("scheme", [(1, 0), (1, 1)])
def test_peer_mode_with_scheme_variants(scheme):
    # the F4 variants (HLLC, MC: the scheme-1 instantiations) through peer mode
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = CASES[1]
    g = H.make_grid(ndim, nb, nblk, bc=bc, riemann=scheme[0], limiter=scheme[1])
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.supersonic_field(g.N, seed=73)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=4)
    B, logB, _ = _run_peer(g, U0, owner, 4)
    assert logB == [tuple(x) for x in logA]
    assert np.array_equal(A, B)


@pytest.mark.parametrize("case", [CASES[1], CASES[2]])
def test_peer_mode_per_stage_variant(case):
    # F1 + F2: the per-stage step in peer mode (U1 rows staged from other
    # ranks' stage-1 buffers, a barrier as the U1 refill) == the single-domain
    # per-stage step; parity build == the oracle's refill mode
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = case
    for parity in (False, True):
        g = H.make_grid(ndim, nb, nblk, bc=bc, parity=parity)
        owner = hydro.brick_owner(nblk, brick, gg)
        U0 = inp.random_field(g.N, seed=74)
        A, _, logA, _ = H.gpu_run(g, U0, nsteps=4, method="per-stage")
        B, logB, launches = _run_peer(g, U0, owner, 4, method="per-stage")
        assert logB == [tuple(x) for x in logA]
        assert np.array_equal(A, B)
        if parity:
            Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4, mode="refill")
            assert np.array_equal(B, Oo)


def test_peer_mode_scattered_owner_map():
    from paper_2507_09337_b200 import hydro  # noqa: F401
    g = H.make_grid(3, (8, 8, 8), (4, 3, 2), bc=((R, O), (P, P), (O, R)))
    owner = (np.random.default_rng(4).random(g.nblocks) * 3).astype(np.int32)
    owner[:3] = [0, 1, 2]
    U0 = inp.random_field(g.N, seed=72)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=4)
    B, logB, _ = _run_peer(g, U0, owner, 4)
    assert [x[0] for x in logB] == [x[0] for x in logA]
    assert np.array_equal(A, B)


def test_peer_mode_parity_build_equals_oracle():
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = CASES[2]
    g = H.make_grid(ndim, nb, nblk, bc=bc, parity=True)
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.sedov(g.N)
    B, logB, _ = _run_peer(g, U0, owner, 4)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4)
    assert [x[0] for x in logB] == olog.dts
    assert [x[2] for x in logB] == olog.argmax
    assert np.array_equal(B, Oo)


def test_peer_mode_host_dt_with_a_thread_per_rank():
    # the host-dt path (orcha_compute_dt synchronizes) with one host thread
    # per rank, as separate processes would drive their GPUs
    import torch
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = CASES[0]
    g = H.make_grid(ndim, nb, nblk, bc=bc)
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.sedov(g.N)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=3)
    comms, streams, pks = _setup(g, U0, owner)
    logs = [[] for _ in pks]
    errs = []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            for _ in range(3):
                hydro.orcha_fill_guardcells([pks[r]], comms[r], streams[r])
                info = hydro.orcha_compute_dt([pks[r]], math.inf, comms[r], streams[r])
                logs[r].append(info.dt)
                hydro.orcha_hydro_advance(pks[r], info.dt, streams[r])
            streams[r].synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=rank, args=(r,)) for r in range(len(pks))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for c in comms:
        c.check()
    assert all(lg == [x[0] for x in logA] for lg in logs)
    assert np.array_equal(H.gather(g, pks), A)
    for c in comms:
        c.destroy()


def test_peer_barrier_timeout_is_an_error_not_a_hang(monkeypatch):
    # only rank 0 steps: its first barrier never completes; with a 300 ms
    # timeout the kernel gives up, sets the flag, and orcha_comm_check reports it
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, '.')
import orcha_inputs as inp
from paper_2507_09337_b200 import hydro, abi
g = hydro.Grid(3, (8, 8, 8), (2, 1, 1))
owner = np.array([0, 1], dtype=np.int32)
comms = hydro.Comm.create_local(g, 2, owner)
pks = [hydro.Packet(g, [r]) for r in range(2)]
U0 = inp.sedov(g.N)
for r in range(2):
    pks[r].pack(inp.to_blocks(U0, g.nb, [r]))
    comms[r].peer_register(pks[r])
hydro.orcha_fill_guardcells([pks[0]], comms[0])
torch.cuda.synchronize()
try:
    comms[0].check()
    print("NO-ERROR")
except abi.OrchaError as e:
    print("TIMEOUT-ERROR", e)
"""
    env = dict(__import__("os").environ, ORCHA_PEER_TIMEOUT_MS="300")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=240)
    assert "TIMEOUT-ERROR" in r.stdout, (r.stdout, r.stderr[-2000:])
