"""Guard push (push.cuh): after an advance the fused kernels have scattered the
new interior into the guards; those guard values must be bitwise the
oracle's axis-ordered ghost fill of the new state, and runs
with the push on and off must be bitwise identical (telescoped and
per-stage, several packets, every boundary kind)."""
import numpy as np
import pytest

import oracle
import orcha_inputs as inp
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu
O, P, R = 0, 1, 2
CASES = [
    ((8, 8, 8), (3, 2, 2), ((O, O), (P, P), (R, R))),
    ((16, 16, 16), (2, 2, 2), ((R, O), (O, R), (P, P))),
    ((16, 16, 16), (1, 2, 1), ((P, P), (P, P), (O, O))),   # periodic with one block: self-targets
    ((32, 32, 32), (2, 1, 1), ((O, R), (O, O), (O, O))),
]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _set_push(lib, on):
    from paper_2507_09337_b200 import abi
    abi.call(lib, "orcha_set_guard_push", 1 if on else 0)


@pytest.mark.parametrize("nb,nblk,bc", CASES)
@pytest.mark.parametrize("method", ["telescoped", "per-stage"])
def test_pushed_guards_equal_ghost_fill(nb, nblk, bc, method):
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, nb, nblk, bc=bc)
    _set_push(g.lib, True)
    U0 = inp.random_field(g.N, seed=17)
    npk = 1 if method == "telescoped" else 2
    pk = H.gpu_setup(g, U0, npackets=npk, shuffle=True)
    hydro.run(pk, nsteps=2, method=method)   # the second step's fill found the guards pushed
    if npk > 1:
        # same-packet guards were pushed; the fill gathers only the cross-packet directions
        hydro.orcha_fill_guardcells(pk)
    interior = H.gather(g, pk)
    og = H.oracle_grid(g)
    Ug = oracle.padded(og, interior)
    oracle.fill_ghosts(og, Ug)
    ng = 4
    for p in pk:
        S = p.state_view().cpu().numpy()
        for s, b in enumerate(p.block_ids):
            bi, bj, bk = b % g.nblk[0], (b // g.nblk[0]) % g.nblk[1], b // (g.nblk[0] * g.nblk[1])
            sl = (slice(None), slice(bk * nb[2], bk * nb[2] + nb[2] + 2 * ng),
                  slice(bj * nb[1], bj * nb[1] + nb[1] + 2 * ng), slice(bi * nb[0], bi * nb[0] + nb[0] + 2 * ng))
            assert np.array_equal(S[s], Ug[sl]), (s, b)


@pytest.mark.parametrize("nb,nblk,bc", CASES)
@pytest.mark.parametrize("method", ["telescoped", "per-stage"])
def test_push_on_off_bitwise(nb, nblk, bc, method):
    g = H.make_grid(3, nb, nblk, bc=bc)
    U0 = inp.random_field(g.N, seed=19)
    try:
        _set_push(g.lib, True)
        A = H.gpu_run(g, U0, nsteps=4, npackets=3, shuffle=True, method=method)[0]
        _set_push(g.lib, False)
        B = H.gpu_run(g, U0, nsteps=4, npackets=3, shuffle=True, method=method)[0]
    finally:
        _set_push(g.lib, True)
    assert np.array_equal(A, B)
