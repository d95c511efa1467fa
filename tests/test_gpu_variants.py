"""SURVEY 8(f) F4 scheme variants on the GPU (HLLC Riemann solver, MC
limiter; grid flags riemann / limiter): the CUDA path against the oracle with
the same flags -- parity build bitwise, production build <= 1e-12 by the
c13 metric -- through the fused kernels (their scheme-1 instantiations: 8^3,
16^3 and 32^3 blocks, gather and full fill, telescoped and per-stage) and the
reference kernels (1D / 2D grids)."""
import numpy as np
import pytest

import orcha_inputs as inp
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu
O, P, R = 0, 1, 2
HLL, HLLC, MINMOD, MC = 0, 1, 0, 1
SCHEMES = [(HLLC, MINMOD), (HLL, MC), (HLLC, MC)]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CASES = {
    "sedov3d_16": dict(ndim=3, nb=(16, 16, 16), nblk=(2, 2, 2), ic=lambda N: inp.sedov(N), steps=6),
    "random3d_8_mixed": dict(ndim=3, nb=(8, 8, 8), nblk=(3, 2, 2), ic=lambda N: inp.random_field(N, seed=21),
                             steps=5, bc=((P, P), (R, O), (O, R)), npk=2),
    "random3d_32": dict(ndim=3, nb=(32, 32, 32), nblk=(2, 1, 1), ic=lambda N: inp.random_field(N, seed=22),
                        steps=3, bc=((R, O), (P, P), (O, O))),
    "sod1d": dict(ndim=1, nb=(16,), nblk=(32,), ic=lambda N: inp.sod(N), steps=10),
    "random2d_reflect": dict(ndim=2, nb=(8, 8), nblk=(3, 2), ic=lambda N: inp.random_field(N, seed=23), steps=6,
                             bc=((R, R), (R, O), (O, O))),
}


def _run(name, scheme, parity, method="telescoped", variant=None):
    c = CASES[name]
    g = H.make_grid(c["ndim"], c["nb"], c["nblk"], bc=c.get("bc"), parity=parity, riemann=scheme[0],
                    limiter=scheme[1])
    from paper_2507_09337_b200 import hydro
    old = g.lib.orcha_get_kernel_variant()
    if variant is not None:
        hydro.set_kernel_variant(g.lib, variant)
    U0 = c["ic"](g.N[:c["ndim"]])
    try:
        G, t, log, pk = H.gpu_run(g, U0, nsteps=c["steps"], npackets=c.get("npk", 1), method=method)
    finally:
        hydro.set_kernel_variant(g.lib, old)
    mode = "refill" if method == "per-stage" else "telescoped"
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=c["steps"], mode=mode)
    return G, Oo, log, olog, pk


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("name", list(CASES))
def test_variant_parity_build_bitwise(name, scheme):
    G, Oo, log, olog, pk = _run(name, scheme, parity=True)
    assert [x[0] for x in log] == olog.dts
    assert np.array_equal(G, Oo)


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("name", list(CASES))
def test_variant_production_within_1e12(name, scheme):
    G, Oo, log, olog, pk = _run(name, scheme, parity=False)
    assert H.parity_error(G, Oo) <= 1e-12, H.error_report(G, Oo)
    for (dt, smax, am, tag), odt in zip(log, olog.dts):
        assert abs(dt - odt) <= 1e-13 * odt


@pytest.mark.parametrize("scheme", SCHEMES)
def test_variant_per_stage_parity(scheme):
    G, Oo, log, olog, pk = _run("random3d_8_mixed", scheme, parity=True, method="per-stage")
    assert np.array_equal(G, Oo)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_variant_reference_kernels_equal_fused(scheme):
    A = _run("sedov3d_16", scheme, parity=True, variant=0)[0]
    B = _run("sedov3d_16", scheme, parity=True, variant=1)[0]
    assert np.array_equal(A, B)


def test_hllc_keeps_a_stationary_contact_on_the_gpu():
    # a density jump at rest in pressure equilibrium: HLLC holds it (to
    # round-off), HLL diffuses it -- the property the variant exists for
    from paper_2507_09337_b200 import hydro
    out = {}
    for rs in (HLL, HLLC):
        g = H.make_grid(3, (16, 16, 16), (2, 1, 1), bc=((O, O), (P, P), (P, P)), riemann=rs)
        U0 = np.zeros((5,) + tuple(reversed(g.N)))
        U0[0] = 1.0
        U0[0, :, :, g.N[0] // 2:] = 0.125
        U0[4] = 1.0 / 0.4
        G = H.gpu_run(g, U0, nsteps=20)[0]
        out[rs] = np.abs(G[0] - U0[0]).max()
    assert out[HLLC] <= 1e-13 and out[HLL] > 1e-3
