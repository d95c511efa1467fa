"""CPU check that the supersonic GPU cases reach the one-sided Riemann
branches (the GPU file asserts the same on its own oracle runs); the cheap
cases only, so the CPU suite stays fast."""
import pytest

import oracle
import orcha_inputs as inp
from tests import face_branches as fb

P = oracle.PERIODIC


@pytest.mark.parametrize("N", [(16, 16, 16), (64, 32, 32)])
def test_supersonic_field_has_one_sided_faces_on_every_axis(N):
    g = oracle.Grid(N=N, bc=((P, P),) * 3)
    U = oracle.padded(g, inp.supersonic_field(N))
    oracle.fill_ghosts(g, U)
    c = fb.count(U, 3)
    for d in range(3):
        left, right, n = c[d]
        assert left > n // 4 and right > n // 4, c


def test_subsonic_random_field_has_none():
    # the counter itself: a rough subsonic field (|v| <= 0.9 < c) takes only
    # the subsonic branch
    N = (16, 16, 16)
    g = oracle.Grid(N=N, bc=((P, P),) * 3)
    U = oracle.padded(g, inp.random_field(N))
    oracle.fill_ghosts(g, U)
    c = fb.count(U, 3)
    assert all(c[d][0] == 0 and c[d][1] == 0 for d in range(3)), c
