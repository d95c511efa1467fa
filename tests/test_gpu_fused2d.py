"""The 2D one-kernel step (csrc/kernels_fused2d.cu: both RK2 stages of a
2D block in one CTA, U1 kept in shared memory) against the oracle and the
reference kernels: parity build bitwise (state, dt and argmax every step),
production build within the c13 metric; every boundary condition, 8^2 and
16^2 blocks, several packets, the F4 variants; one advance launch per step."""
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


CASES = {
    "sedov_cfg1": dict(nb=(8, 8), nblk=(4, 4), bc=None, ic=lambda N: inp.sedov(N), steps=10),
    "sedov_16": dict(nb=(16, 16), nblk=(4, 4), bc=None, ic=lambda N: inp.sedov(N), steps=12),
    "random_mixed_16": dict(nb=(16, 16), nblk=(3, 2), bc=((O, R), (R, O), (O, O)),
                            ic=lambda N: inp.random_field(N, seed=81), steps=6, npk=2),
    "random_periodic_8": dict(nb=(8, 8), nblk=(4, 3), bc=((P, P), (P, P), (O, O)),
                              ic=lambda N: inp.random_field(N, seed=82), steps=6, npk=3),
    "supersonic_16": dict(nb=(16, 16), nblk=(2, 2), bc=((P, P), (P, P), (O, O)),
                          ic=lambda N: inp.supersonic_field(N, seed=83), steps=6),
    "sod_tube_16": dict(nb=(16, 16), nblk=(16, 1), bc=((O, O), (P, P), (O, O)), xmax=(1.0, 16 / 256),
                        ic=lambda N: inp.sod(N), steps=20),
}


def _run(name, parity, variant=None, scheme=(0, 0)):
    from paper_2507_09337_b200 import hydro
    c = CASES[name]
    g = H.make_grid(2, c["nb"], c["nblk"], bc=c["bc"], xmax=c.get("xmax", (1.0, 1.0, 1.0)), parity=parity,
                    riemann=scheme[0], limiter=scheme[1])
    U0 = c["ic"](g.N[:2])
    old = g.lib.orcha_get_kernel_variant()
    if variant is not None:
        hydro.set_kernel_variant(g.lib, variant)
    try:
        G, t, log, pk = H.gpu_run(g, U0, nsteps=c["steps"], npackets=c.get("npk", 1))
    finally:
        hydro.set_kernel_variant(g.lib, old)
    return g, U0, G, log


@pytest.mark.parametrize("name", list(CASES))
def test_fused2d_parity_build_bitwise(name):
    g, U0, G, log = _run(name, True)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=CASES[name]["steps"])
    assert [x[0] for x in log] == olog.dts
    assert [x[2] for x in log] == olog.argmax
    assert np.array_equal(G, Oo)


@pytest.mark.parametrize("name", list(CASES))
def test_fused2d_production_within_c13(name):
    g, U0, G, log = _run(name, False)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=CASES[name]["steps"])
    assert H.parity_error(G, Oo) <= 1e-12, H.error_report(G, Oo)
    for (dt, smax, am, tag), odt in zip(log, olog.dts):
        assert abs(dt - odt) <= 1e-13 * odt


@pytest.mark.parametrize("scheme", [(1, 0), (0, 1), (1, 1)])
def test_fused2d_equals_reference_kernels_with_variants(scheme):
    A = _run("random_mixed_16", True, variant=1, scheme=scheme)[2]
    B = _run("random_mixed_16", True, variant=0, scheme=scheme)[2]
    assert np.array_equal(A, B)


def test_fused2d_is_one_launch_per_advance():
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(2, (16, 16), (4, 4))
    pk = H.gpu_setup(g, inp.sedov(g.N[:2]), 1)
    hydro.orcha_fill_guardcells(pk)
    info = hydro.orcha_compute_dt(pk)
    n0 = g.lib.orcha_launch_count()
    hydro.orcha_hydro_advance(pk[0], info.dt)
    assert g.lib.orcha_launch_count() - n0 == 1
