"""Device-resident dt (orcha_compute_dt_device -> orcha_hydro_advance_devdt,
no host synchronization per step): the same records, cross-rank rule and IEEE
operations as orcha_compute_dt, so the time loop is bitwise the host-dt loop
-- dt, s_max, argmax and tag every step, the t_end clamp, and the state
(the dt reduction is one of the step's "1 or 2
MPI operations")."""
import ctypes
import math

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


def _both(g, U0, nsteps, npackets=1, t_end=math.inf, comm=None, method="telescoped"):
    from paper_2507_09337_b200 import hydro
    pa = H.gpu_setup(g, U0, npackets)
    ta, na, loga = hydro.run(pa, nsteps=nsteps, t_end=t_end, comm=comm, method=method)
    pb = H.gpu_setup(g, U0, npackets)
    clock, logb = hydro.run_device(pb, nsteps, t_end=t_end, comm=comm, method=method)
    return (H.gather(g, pa), ta, loga), (H.gather(g, pb), clock.read(), logb)


@pytest.mark.parametrize("parity", [False, True])
@pytest.mark.parametrize("npackets", [1, 3])
@pytest.mark.parametrize("method", ["telescoped", "per-stage"])
def test_device_dt_loop_equals_host_loop(parity, npackets, method):
    g = H.make_grid(3, (16, 16, 16), (2, 2, 2), bc=((R, O), (P, P), (O, R)), parity=parity)
    U0 = inp.random_field(g.N, seed=61)
    (A, ta, loga), (B, c, logb) = _both(g, U0, 5, npackets, method=method)
    assert logb == [tuple(x) for x in loga]
    assert c.t == ta and c.steps == 5 and c.nonphysical == 0
    assert np.array_equal(A, B)


def test_device_dt_clamp_at_t_end():
    from paper_2507_09337_b200 import abi
    g = H.make_grid(3, (8, 8, 8), (2, 2, 2))
    U0 = inp.sedov(g.N)
    _, _, log, _ = H.gpu_run(g, U0, nsteps=3)
    t_end = (log[0][0] + log[1][0]) + 0.5 * log[2][0]
    (A, ta, loga), (B, c, logb) = _both(g, U0, 3, t_end=t_end)
    assert len(loga) == 3 and loga[2][3] == abi.DT_CLAMP
    assert logb == [tuple(x) for x in loga]
    assert c.t == ta and c.tag == abi.DT_CLAMP
    assert np.array_equal(A, B)


def test_device_dt_through_nccl_single_rank():
    # the allgather path on the device (one rank)
    from paper_2507_09337_b200 import abi, hydro
    g = H.make_grid(3, (8, 8, 8), (2, 2, 2))
    owner = np.zeros(g.nblocks, dtype=np.int32)
    uid = (ctypes.c_uint8 * 128)()
    abi.call(g.lib, "orcha_comm_unique_id", uid)
    h = ctypes.c_void_p()
    abi.call(g.lib, "orcha_comm_create", g.handle, uid, 1, 0, owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
             ctypes.byref(h))
    comm = hydro.Comm(g, h, 1, 0, owner)
    try:
        (A, ta, loga), (B, c, logb) = _both(g, inp.sedov(g.N), 3, npackets=2, comm=comm)
        assert logb == [tuple(x) for x in loga]
        assert np.array_equal(A, B)
    finally:
        comm.destroy()


def test_push_dt_refuses_nccl_communicator():
    # orcha_comm_push_dt is the LOCAL transport's allgather; an NCCL
    # communicator allgathers inside orcha_compute_dt(_device) instead
    import ctypes
    from paper_2507_09337_b200 import abi, hydro
    g = H.make_grid(3, (8, 8, 8), (2, 1, 1))
    owner = np.zeros(g.nblocks, dtype=np.int32)
    uid = (ctypes.c_uint8 * 128)()
    abi.call(g.lib, "orcha_comm_unique_id", uid)
    h = ctypes.c_void_p()
    abi.call(g.lib, "orcha_comm_create", g.handle, uid, 1, 0, owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
             ctypes.byref(h))
    comm = hydro.Comm(g, h, 1, 0, owner)
    pk = H.gpu_setup(g, inp.sedov(g.N), 1)
    with pytest.raises(abi.OrchaError, match="ORCHA_E_ARG"):
        comm.push_dt(pk)
    comm.destroy()


def test_device_dt_reports_nonphysical_state():
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, (8, 8, 8), (1, 1, 1))
    U0 = inp.sedov(g.N)
    U0[0, 3, 4, 5] = -1.0
    pk = H.gpu_setup(g, U0, 1)
    clock = hydro.DevClock()
    hydro.orcha_fill_guardcells(pk)
    hydro.orcha_compute_dt_device(pk, clock)
    assert clock.read().nonphysical == 1


@pytest.mark.parametrize("npackets", [1, 2])
def test_cuda_graph_of_device_dt_steps_equals_plain_loop(npackets):
    # the steady-state step (the gather-mode fill launches nothing, dt and the
    # advance read / write device memory only) captured once in a CUDA graph
    # and replayed: bitwise the plain device-dt loop, clock included
    import torch
    from paper_2507_09337_b200 import hydro
    g = H.make_grid(3, (16, 16, 16), (2, 2, 2), bc=((R, O), (P, P), (O, R)))
    U0 = inp.random_field(g.N, seed=67)
    pa = H.gpu_setup(g, U0, npackets)
    ca, loga = hydro.run_device(pa, 8)
    pb = H.gpu_setup(g, U0, npackets)
    clock = hydro.DevClock()
    for _ in range(2):  # steady state first (records from the fused epilogue; not captured)
        hydro.orcha_fill_guardcells(pb)
        hydro.orcha_compute_dt_device(pb, clock)
        hydro.step_devdt(pb, clock.dt_tensor)
    graph = hydro.capture_steps(pb, clock, 2)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert np.array_equal(H.gather(g, pb), H.gather(g, pa))
    cb = clock.read()
    assert (cb.t, cb.dt, cb.argmax, cb.steps) == (ca.read().t, ca.read().dt, ca.read().argmax, 8)


@pytest.mark.parametrize("scheme", [dict(riemann=1), dict(limiter=1), dict(eos=1, arad=1e-4)])
def test_device_dt_loop_with_scheme_variants(scheme):
    # the device clock with the F4 variants (HLLC, MC, the gas + radiation EOS,
    # whose dt uses Gamma_1): bitwise the host-dt loop, parity build against
    # the oracle as well
    g = H.make_grid(3, (8, 8, 8), (2, 2, 2), bc=((O, O), (P, P), (R, O)), parity=True, **scheme)
    U0 = inp.sedov(g.N)
    (A, ta, loga), (B, c, logb) = _both(g, U0, 3)
    assert logb == [tuple(x) for x in loga]
    assert np.array_equal(A, B)
    O_, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=3)
    assert [x[0] for x in logb] == olog.dts
    assert np.array_equal(B, O_)
