"""Gather fill mode (orcha_set_fill_mode(1), the default): one packet, only
the x-guards filled, stage 1 staging its y/z guard rows from the owning blocks
(sign flips for mirrored rows) -- bitwise identical to the FULL fill mode and
to the oracle (parity build), for every boundary kind, block size and both
step methods."""
import numpy as np
import pytest

import orcha_inputs as inp
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu
O, P, R = 0, 1, 2
CASES = [
    ((8, 8, 8), (3, 2, 2), ((O, O), (P, P), (R, R))),
    ((16, 16, 16), (2, 2, 2), ((R, O), (O, R), (P, P))),
    ((16, 16, 16), (1, 2, 1), ((P, P), (R, R), (O, O))),   # one block along x and z
    ((32, 32, 32), (2, 1, 1), ((O, R), (R, O), (P, P))),
]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _mode(lib, m):
    from paper_2507_09337_b200 import abi
    abi.call(lib, "orcha_set_fill_mode", m)


@pytest.mark.parametrize("nb,nblk,bc", CASES)
@pytest.mark.parametrize("method", ["telescoped", "per-stage"])
def test_gather_mode_equals_full_mode(nb, nblk, bc, method):
    g = H.make_grid(3, nb, nblk, bc=bc)
    U0 = inp.random_field(g.N, seed=29)
    try:
        _mode(g.lib, 1)
        A = H.gpu_run(g, U0, nsteps=4, method=method)[0]
        _mode(g.lib, 0)
        B = H.gpu_run(g, U0, nsteps=4, method=method)[0]
    finally:
        _mode(g.lib, 1)
    assert np.array_equal(A, B)


@pytest.mark.parametrize("nb,nblk,bc", CASES[:2])
def test_gather_mode_parity_build_equals_oracle(nb, nblk, bc):
    g = H.make_grid(3, nb, nblk, bc=bc, parity=True)
    _mode(g.lib, 1)
    U0 = inp.random_field(g.N, seed=31)
    G, t, log, pk = H.gpu_run(g, U0, nsteps=4)
    O_, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4)
    assert [x[0] for x in log] == olog.dts
    assert np.array_equal(G, O_)


def test_variant_switch_after_gather_fill_is_refused():
    from paper_2507_09337_b200 import abi, hydro
    g = H.make_grid(3, (8, 8, 8), (2, 2, 2))
    _mode(g.lib, 1)
    pk = H.gpu_setup(g, inp.sedov(g.N))
    hydro.orcha_fill_guardcells(pk)
    hydro.set_kernel_variant(g.lib, 0)
    try:
        with pytest.raises(abi.OrchaError) as e:
            hydro.orcha_hydro_advance(pk[0], 1e-5)
        assert e.value.status == "ORCHA_E_STATE"
        hydro.orcha_fill_guardcells(pk)      # refill under the reference variant: full fill
        hydro.orcha_hydro_advance(pk[0], 1e-5)
    finally:
        hydro.set_kernel_variant(g.lib, 1)


def test_gather_mode_steady_state_fill_launches_nothing():
    # after the first advance, stage 2 has scattered U^{n+1} into the x-guards
    # (push_cell_x), so the next gather-mode fill is a no-op on the device
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, (16, 16, 16), (2, 2, 2), bc=((R, O), (P, P), (O, R)))
    _mode(g.lib, 1)
    pk = H.gpu_setup(g, inp.random_field(g.N, seed=3))
    hydro.orcha_fill_guardcells(pk)
    n0 = g.lib.orcha_launch_count()
    hydro.orcha_fill_guardcells(pk)          # refill of unchanged guards (not pushed yet): one fill_x
    assert g.lib.orcha_launch_count() - n0 == 1
    hydro.orcha_hydro_advance(pk[0], 1e-5)
    n1 = g.lib.orcha_launch_count()
    hydro.orcha_fill_guardcells(pk)
    assert g.lib.orcha_launch_count() == n1
