"""SURVEY 8(f) F4 expensive-EOS surrogate on the GPU (grid eos = gas +
radiation, Newton temperature solves, work multiplier; DESIGN.md reading
c22): the CUDA path against the oracle with the same EOS -- parity build
bitwise, production build <= 1e-12 -- through the fused kernels (scheme-1
instantiations), the reference kernels and the per-stage variant."""
import numpy as np
import pytest

import orcha_inputs as inp
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu
O, P, R = 0, 1, 2
RAD = 1


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CASES = {
    "random3d_16": dict(ndim=3, nb=(16, 16, 16), nblk=(2, 2, 1), ic=lambda N: inp.random_field(N, seed=61), steps=4,
                        bc=((P, P), (R, O), (O, R)), arad=0.5, w=1),
    "random3d_8_work3": dict(ndim=3, nb=(8, 8, 8), nblk=(2, 2, 2), ic=lambda N: inp.random_field(N, seed=62),
                             steps=4, bc=((R, R), (P, P), (O, O)), arad=2.0, w=3, npk=2),
    "sedov3d_16": dict(ndim=3, nb=(16, 16, 16), nblk=(2, 2, 2), ic=lambda N: inp.sedov(N), steps=5, arad=1e-3, w=1),
    "sod1d": dict(ndim=1, nb=(16,), nblk=(16,), ic=lambda N: inp.sod(N), steps=8, arad=0.2, w=1),
}


def _run(name, parity, riemann=0, limiter=0, method="telescoped", variant=None):
    c = CASES[name]
    g = H.make_grid(c["ndim"], c["nb"], c["nblk"], bc=c.get("bc"), parity=parity, riemann=riemann, limiter=limiter,
                    eos=RAD, eos_work=c["w"], arad=c["arad"])
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
    return G, Oo, log, olog


@pytest.mark.parametrize("name", list(CASES))
def test_eos_parity_build_bitwise(name):
    G, Oo, log, olog = _run(name, parity=True)
    assert [x[0] for x in log] == olog.dts
    assert np.array_equal(G, Oo)


@pytest.mark.parametrize("name", list(CASES))
def test_eos_production_within_1e12(name):
    G, Oo, log, olog = _run(name, parity=False)
    assert H.parity_error(G, Oo) <= 1e-12, H.error_report(G, Oo)
    for (dt, smax, am, tag), odt in zip(log, olog.dts):
        assert abs(dt - odt) <= 1e-12 * odt


def test_eos_with_hllc_and_mc_parity():
    G, Oo, log, olog = _run("random3d_16", parity=True, riemann=1, limiter=1)
    assert np.array_equal(G, Oo)


def test_eos_per_stage_and_reference_kernels_parity():
    G, Oo, _, _ = _run("random3d_8_work3", parity=True, method="per-stage")
    assert np.array_equal(G, Oo)
    A = _run("random3d_16", parity=True, variant=0)[0]
    B = _run("random3d_16", parity=True, variant=1)[0]
    assert np.array_equal(A, B)
