"""Per-phase instrumentation (orcha_set_phase_timing / orcha_phase_times,
SURVEY 8(d) timing protocol) and the fp64 probe: every phase of a step is
recorded once per step, the stage times add up to the advance measured
around it, and timing off records nothing."""
import math

import pytest

import orcha_inputs as inp
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_phase_times_cover_each_step():
    import torch
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, (16, 16, 16), (4, 4, 4))
    pk = H.gpu_setup(g, inp.sedov(g.N), 1)
    clock = hydro.DevClock(0.0, math.inf)
    s = torch.cuda.current_stream()
    hydro.orcha_set_phase_timing(g.lib, True)
    hydro.orcha_phase_times(g.lib)
    adv = 0.0
    try:
        for _ in range(4):
            hydro.orcha_fill_guardcells(pk, None, s)
            hydro.orcha_compute_dt_device(pk, clock, None, s)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            hydro.orcha_hydro_advance_devdt(pk[0], clock.dt_tensor, s)
            b.record(s)
            torch.cuda.synchronize()
            adv += a.elapsed_time(b)
        pt = hydro.orcha_phase_times(g.lib)
    finally:
        hydro.orcha_set_phase_timing(g.lib, False)
    for k in ("fill", "dt", "stage1", "stage2"):
        assert pt[k][1] == 4, (k, pt)
    assert pt["exchange"][1] == 0 and pt["dt_allgather"][1] == 0
    st = pt["stage1"][0] + pt["stage2"][0]
    assert 0.0 < st <= adv * 1.05 + 0.05 and st >= 0.8 * adv, (st, adv)
    # off: nothing recorded
    hydro.orcha_fill_guardcells(pk, None, s)
    hydro.orcha_compute_dt_device(pk, clock, None, s)
    hydro.orcha_hydro_advance_devdt(pk[0], clock.dt_tensor, s)
    assert all(v[1] == 0 for v in hydro.orcha_phase_times(g.lib).values())


def test_fp64_probe_is_plausible():
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, (8, 8, 8), (1, 1, 1))
    t, ms = hydro.orcha_probe_fp64(g.lib, 2000)
    # 148 SMs x 64 fp64 lanes x <= 2.1 GHz = 19.9 T DFMA/s at most
    assert 1.0 < t < 20.5 and ms > 0.0
