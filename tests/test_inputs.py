"""The shared input module: the packet-order Sedov generator equals the
global one re-blocked (so a rank can build only its brick), block reshapes
round-trip, and the closed-form IC invariants hold."""
import numpy as np
import pytest

import orcha_inputs as inp


@pytest.mark.parametrize("N,nb", [((32, 32), (8, 8)), ((64, 64, 64), (16, 16, 16)), ((32, 48, 64), (8, 16, 16)),
                                  ((64,), (16,))])
def test_sedov_packet_equals_reblocked_global(N, nb):
    nblocks = int(np.prod([n // b for n, b in zip(N, nb)]))
    ids = np.random.default_rng(1).permutation(nblocks)
    A = inp.sedov_packet(N, nb, ids)
    B = inp.to_blocks(inp.sedov(N), nb, ids)
    assert np.array_equal(A, B)
    assert (A[:, 4] > 1e-3).sum() == inp.sedov_deposit_count(len(N))


def test_blocks_roundtrip():
    U = inp.random_field((16, 24, 8), seed=2)
    ids = np.random.default_rng(0).permutation(2 * 3 * 1)
    B = inp.to_blocks(U, (8, 8, 8), ids)
    assert np.array_equal(inp.from_blocks(B, (16, 24, 8), (8, 8, 8), ids), U)


def test_random_field_positive_and_seeded():
    a = inp.random_field((8, 8, 8), seed=5)
    b = inp.random_field((8, 8, 8), seed=5)
    assert np.array_equal(a, b) and (a[0] > 0).all()
