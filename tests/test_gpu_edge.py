"""Degenerate and edge cases of the method on the GPU, against the oracle:
the pressure floor (a strong double rarefaction towards vacuum, reading c10),
a state at rest with no gradients (bitwise unchanged), a ragged packet split
with a single-block packet, and the t_end clamp on the last step."""
import math

import numpy as np
import pytest

import oracle
import orcha_inputs as inp
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _negative_internal_energy(N):
    # a rough field with a band of cells whose total energy is below the kinetic
    # energy: primitive recovery gives p < 0 there and the floor (c10) fires
    U = inp.random_field(N, seed=3)
    ke = 0.5 * (U[1] ** 2 + U[2] ** 2) / U[0]
    U[4][:, :, 60:68] = ke[:, :, 60:68] * (1 - 1e-3)
    return U


@pytest.mark.parametrize("parity", [True, False])
def test_pressure_floor_case(parity):
    from paper_2507_09337_b200 import hydro
    g2 = hydro.Grid(2, (16, 16), (8, 1), bc=((0, 0), (1, 1), (0, 0)), xmax=(1.0, 16 / 128), parity=parity)
    og = oracle.Grid(N=(128, 16), xmax=(1.0, 16 / 128), bc=((0, 0), (1, 1), (0, 0)))
    U0 = _negative_internal_energy((128, 16))
    G, t, log, pk = H.gpu_run(g2, U0, nsteps=8)
    Oarr = oracle.padded(og, U0)
    olog = oracle.run(og, Oarr, nsteps=8)
    O = Oarr[og.interior]
    assert olog.floor_hits > 0                      # the floor path is exercised
    fh, bad = pk[0].counters()
    assert fh > 0 and bad == -1
    if parity:
        assert [x[0] for x in log] == olog.dts
        assert np.array_equal(G, O)
    else:
        assert H.parity_error(G, O) <= 1e-12, H.error_report(G, O)


def test_state_at_rest_is_bitwise_unchanged():
    g = H.make_grid(3, (16, 16, 16), (2, 2, 1))
    U0 = inp.uniform(g.N, 0.7, (0.0, 0.0, 0.0), 2.5)
    G, t, log, pk = H.gpu_run(g, U0, nsteps=3)
    assert np.array_equal(G, U0)


def test_ragged_packets_and_tend_clamp():
    # 27 blocks split 13 / 13 / 1, run to a t_end that the CFL dt does not divide
    g = H.make_grid(3, (8, 8, 8), (3, 3, 3), xmax=(1.0, 1.0, 1.0), parity=True)
    og = H.oracle_grid(g)
    U0 = inp.random_field(g.N, seed=23)
    from paper_2507_09337_b200 import hydro
    ids = np.random.default_rng(2).permutation(27)
    pk = [hydro.Packet(g, ids[:13]), hydro.Packet(g, ids[13:26]), hydro.Packet(g, ids[26:])]
    for p in pk:
        p.pack(inp.to_blocks(U0, g.nb, p.block_ids))
    t_end = 0.0123
    t, n, log = hydro.run(pk, t_end=t_end)
    O, olog = H.oracle_run(og, U0, t_end=t_end)
    assert t == olog.t and abs(t - t_end) <= 1e-15 and n == olog.steps
    assert log[-1][3] == oracle.TAG_CLAMP and olog.tags[-1] == oracle.TAG_CLAMP
    assert np.array_equal(H.gather(g, pk), O)
