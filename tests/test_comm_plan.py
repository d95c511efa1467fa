"""Multi-GPU host logic on CPU: the guard-exchange plan (orcha_comm_plan, a
pure function of the grid and the block->rank map) and a real two-process
exchange over torch.distributed/gloo that moves the halo values the plan
names and checks them against the oracle's global ghost fill."""
import os
import socket

import numpy as np
import pytest

import oracle
import orcha_inputs as inp

O, P, R = 0, 1, 2


def _grid(ndim, nb, nblk, bc):
    from paper_2507_09337_b200 import hydro
    return hydro.Grid(ndim, nb, nblk, bc=bc)


CONFIGS = [
    # (ndim, nb, nblk, bc, gpu_grid, brick)
    (3, (8, 8, 8), (4, 2, 2), ((O, O),) * 3, (2, 1, 1), (2, 2, 2)),
    (3, (8, 8, 8), (4, 4, 2), ((P, P), (R, O), (O, R)), (2, 2, 1), (2, 2, 2)),
    (3, (8, 8, 8), (2, 2, 2), ((P, P),) * 3, (2, 2, 2), (1, 1, 1)),
    (2, (8, 8), (4, 4), ((P, P), (O, O), (O, O)), (2, 2, 1), (2, 2, 1)),
]


def _owner(nblk, brick, gg):
    from paper_2507_09337_b200 import hydro
    return hydro.brick_owner(nblk, brick, gg)


@pytest.mark.parametrize("cfg", CONFIGS)
def test_plan_is_symmetric(cfg):
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = cfg
    g = _grid(ndim, nb, nblk, bc)
    owner = _owner(nblk, brick, gg)
    n = int(owner.max()) + 1
    total = 0
    for r in range(n):
        for q in range(n):
            if q == r:
                continue
            send = hydro.comm_plan(g, n, r, owner, q, 0)
            recv_on_q = hydro.comm_plan(g, n, q, owner, r, 1)
            assert np.array_equal(send, recv_on_q)          # both sides agree on order without negotiating
            assert np.all(np.diff(send) > 0)                 # sorted, unique
            dst = hydro.comm_plan(g, n, r, owner, q, 2)
            idx = hydro.comm_plan(g, n, r, owner, q, 3)
            recv = hydro.comm_plan(g, n, r, owner, q, 1)
            assert len(np.unique(dst)) == len(dst)
            assert len(idx) == len(dst) and (len(idx) == 0 or (idx.min() >= 0 and idx.max() < len(recv)))
            total += len(send)
    assert total > 0


def _guard_global_value(Ug, g, dst, ng=4):
    """Value of the oracle's ghost-filled global array at guard `dst` (block*P^3 + padded cell)."""
    nd = g.ndim
    Px = [g.nb[a] + 2 * ng if a < nd else 1 for a in range(3)]
    P3 = Px[0] * Px[1] * Px[2]
    b, c = dst // P3, dst % P3
    pi, pj, pk = c % Px[0], (c // Px[0]) % Px[1], c // (Px[0] * Px[1])
    bi, bj, bk = b % g.nblk[0], (b // g.nblk[0]) % g.nblk[1], b // (g.nblk[0] * g.nblk[1])
    # padded global index = block offset + padded local (both arrays carry ng ghosts)
    X = bi * g.nb[0] + pi
    Y = bj * g.nb[1] + pj if nd > 1 else np.zeros_like(pj)
    Z = bk * g.nb[2] + pk if nd > 2 else np.zeros_like(pk)
    return Ug[:, Z, Y, X]


@pytest.mark.parametrize("cfg", CONFIGS)
def test_plan_values_equal_oracle_ghost_fill(cfg):
    # moving the values the plan names reproduces the global ghost fill
    from paper_2507_09337_b200 import hydro
    ndim, nb, nblk, bc, gg, brick = cfg
    g = _grid(ndim, nb, nblk, bc)
    owner = _owner(nblk, brick, gg)
    n = int(owner.max()) + 1
    N = tuple(g.N[:ndim])
    U = inp.random_field(N, seed=21)
    og = oracle.Grid(N=N, bc=tuple(bc[a] for a in range(3)))
    Ug = oracle.padded(og, U)
    oracle.fill_ghosts(og, Ug)
    flat = U.reshape(5, -1)
    for r in range(n):
        for q in range(n):
            if q == r:
                continue
            recv = hydro.comm_plan(g, n, r, owner, q, 1)
            dst = hydro.comm_plan(g, n, r, owner, q, 2)
            idx = hydro.comm_plan(g, n, r, owner, q, 3)
            flip = hydro.comm_plan(g, n, r, owner, q, 4)
            if len(dst) == 0:
                continue
            vals = flat[:, recv][:, idx]
            sign = np.ones((5, len(dst)))
            for v in range(5):
                sign[v, (flip >> v) & 1 == 1] = -1.0
            assert np.array_equal(vals * sign, _guard_global_value(Ug, g, dst))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2507_09337_b200 import hydro
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ndim, nb, nblk, bc, gg, brick = CONFIGS[0]
        g = _grid(ndim, nb, nblk, bc)
        owner = _owner(nblk, brick, gg)
        N = tuple(g.N[:ndim])
        U = inp.random_field(N, seed=33)         # every rank builds the same synthetic field ...
        mine = owner.reshape(nblk[2], nblk[1], nblk[0])
        cell_owner = np.repeat(np.repeat(np.repeat(mine, nb[2], 0), nb[1], 1), nb[0], 2).reshape(-1)
        flat = U.reshape(5, -1).copy()
        flat[:, cell_owner != rank] = np.nan     # ... but may only read the cells it owns
        peer = 1 - rank
        send = hydro.comm_plan(g, world, rank, owner, peer, 0)
        out = torch.from_numpy(np.ascontiguousarray(flat[:, send]))
        assert not torch.isnan(out).any()
        inbuf = torch.empty(5, len(hydro.comm_plan(g, world, rank, owner, peer, 1)), dtype=torch.float64)
        reqs = [dist.isend(out, peer), dist.irecv(inbuf, peer)]
        for rq in reqs:
            rq.wait()
        dst = hydro.comm_plan(g, world, rank, owner, peer, 2)
        idx = hydro.comm_plan(g, world, rank, owner, peer, 3)
        vals = inbuf.numpy()[:, idx]
        og = oracle.Grid(N=N, bc=tuple(bc[a] for a in range(3)))
        Ug = oracle.padded(og, U)
        oracle.fill_ghosts(og, Ug)
        ok = np.array_equal(vals, _guard_global_value(Ug, g, dst)) and len(dst) > 0
        q.put((rank, bool(ok), len(dst)))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_halo_exchange():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert sorted(r for r, _, _ in res) == [0, 1]
    assert all(ok for _, ok, _ in res), res


def test_interior_first_ordering():
    # hydro.interior_first: a rank's blocks whose 26 neighbours it owns come
    # first; for cfg4's (2,2,2) bricks of 16^3 blocks with outflow walls that
    # is the 15^3 blocks away from the three internal faces
    from paper_2507_09337_b200 import hydro
    nblk, brick, gg = (32, 32, 32), (16, 16, 16), (2, 2, 2)
    owner = hydro.brick_owner(nblk, brick, gg)
    bc = ((0, 0),) * 3
    ids = hydro.interior_first(nblk, bc, owner, 0)
    assert sorted(ids.tolist()) == np.flatnonzero(owner == 0).tolist()
    inner = 15 ** 3
    bi, bj, bk = ids % 32, (ids // 32) % 32, ids // 1024
    assert np.all((bi[:inner] < 15) & (bj[:inner] < 15) & (bk[:inner] < 15))
    assert not np.any((bi[inner:] < 15) & (bj[inner:] < 15) & (bk[inner:] < 15))
    # periodic x: the wrap neighbour belongs to the other x-brick, so the x = 0 face is boundary too
    ids_p = hydro.interior_first(nblk, ((1, 1), (0, 0), (0, 0)), owner, 0)
    assert np.all((ids_p[:14 * 15 * 15] % 32 >= 1))
