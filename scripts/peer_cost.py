"""Cost of the cross-rank part of a step, exchange path vs F2 peer mode,
measured with R virtual ranks on ONE B200, each owning cfg4's brick of
16x16x16 blocks of 16^3 (gpu grids (2,1,1), (2,2,1), (2,2,2)), one packet per
rank, gather fill mode, device-resident dt.

* exchange: the NCCL path's plan, pack, copy and unpack kernels (LOCAL
  transport: a device copy stands in for ncclSend/Recv) and the dt records
  pushed to every rank, all ranks on one stream;
* overlap: the same exchange with stage 1 of each rank's interior blocks
  (interior-first slot order) running while its halo is unpacked on a side
  stream (orcha_hydro_step_overlap);
* peer (F2): every rank on its own stream, stage 1 staging other ranks' rows
  directly, stage 2 pushing x-guards into them, device barriers between the
  stage kernels and before the dt reduction -- no pack / copy / unpack.

Both are compared with one rank stepping the same brick alone.  Per-rank
step time = the whole R-rank step on the GPU / R (the ranks share one GPU).
Prints one JSON object."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import orcha_inputs as inp  # noqa: E402
from paper_2507_09337_b200 import abi, hydro  # noqa: E402


def setup(grid, interior_first=False):
    px, py, pz = grid
    R = px * py * pz
    BB, NB = bench.BRICK_BLOCKS, bench.NB
    nblk = (BB[0] * px, BB[1] * py, BB[2] * pz)
    N = tuple(nblk[a] * NB[a] for a in range(3))
    g = hydro.Grid(3, NB, nblk, xmin=(0.0, 0.0, 0.0), xmax=(float(px), float(py), float(pz)))
    owner = hydro.brick_owner(nblk, BB, grid)
    comms = hydro.Comm.create_local(g, R, owner)
    pks = []
    for r in range(R):
        ids = hydro.interior_first(nblk, ((0, 0),) * 3, owner, r) if interior_first else np.flatnonzero(owner == r)
        p = hydro.Packet(g, ids)
        p.pack(inp.sedov_packet(N, NB, ids, xmax=(float(px), float(py), float(pz))))
        pks.append(p)
    return g, comms, pks


def timed(step, streams, steps, warmup):
    cur = torch.cuda.current_stream()
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    for s in streams:
        s.wait_event(a)
    for _ in range(steps):
        step()
    for s in streams:
        e = torch.cuda.Event()
        e.record(s)
        cur.wait_event(e)
    b.record(cur)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def measure(grid, steps=10, warmup=3):
    R = grid[0] * grid[1] * grid[2]
    out = {"gpu_grid": list(grid), "ranks": R}
    # exchange path, one stream
    g, comms, pks = setup(grid)
    s = torch.cuda.current_stream()
    clocks = [hydro.DevClock() for _ in range(R)]

    def step_x():
        for r in range(R):
            comms[r].push([pks[r]], s)
        for r in range(R):
            hydro.orcha_fill_guardcells([pks[r]], comms[r], s)
        for r in range(R):
            comms[r].push_dt([pks[r]], s)
        for r in range(R):
            hydro.orcha_compute_dt_device([pks[r]], clocks[r], comms[r], s)
            hydro.orcha_hydro_advance_devdt(pks[r], clocks[r].dt_tensor, s)
    out["exchange_ms_per_rank_step"] = timed(step_x, [s], steps, warmup) / R
    for c in comms:
        c.destroy()
    del pks
    # exchange path with the interior/boundary overlap (orcha_hydro_step_overlap)
    g, comms, pks = setup(grid, interior_first=True)
    clocks = [hydro.DevClock() for _ in range(R)]

    def step_o():
        for r in range(R):
            comms[r].push([pks[r]], s)
        for r in range(R):
            comms[r].push_dt([pks[r]], s)
        for r in range(R):
            hydro.orcha_hydro_step_overlap(pks[r], comms[r], clocks[r], s)
    out["overlap_ms_per_rank_step"] = timed(step_o, [s], steps, warmup) / R
    for c in comms:
        c.destroy()
    del pks
    # F2 peer mode, a stream per rank
    g, comms, pks = setup(grid)
    streams = [torch.cuda.Stream() for _ in range(R)]
    for r in range(R):
        comms[r].peer_register(pks[r])
    for r in range(R):
        hydro.orcha_fill_prepare([pks[r]], comms[r])
    clocks = [hydro.DevClock() for _ in range(R)]

    def step_p():
        for r in range(R):
            hydro.orcha_fill_guardcells([pks[r]], comms[r], streams[r])
        for r in range(R):
            hydro.orcha_compute_dt_device([pks[r]], clocks[r], comms[r], streams[r])
        for r in range(R):
            hydro.orcha_hydro_advance_devdt(pks[r], clocks[r].dt_tensor, streams[r])
    out["peer_ms_per_rank_step"] = timed(step_p, streams, steps, warmup) / R
    for c in comms:
        c.check()
        c.destroy()
    del pks
    # F1 + F2: the per-stage step in peer mode (U1 rows read from the other
    # ranks' stage-1 buffers; the U1 refill is a barrier)
    g, comms, pks = setup(grid)
    for r in range(R):
        comms[r].peer_register(pks[r])
    for r in range(R):
        hydro.orcha_fill_prepare([pks[r]], comms[r])
    clocks = [hydro.DevClock() for _ in range(R)]

    def step_ps():
        for r in range(R):
            hydro.orcha_fill_guardcells_stage([pks[r]], 0, comms[r], streams[r])
        for r in range(R):
            hydro.orcha_compute_dt_device([pks[r]], clocks[r], comms[r], streams[r])
        for r in range(R):
            hydro.orcha_hydro_stage_devdt(pks[r], 1, clocks[r].dt_tensor, streams[r])
        for r in range(R):
            hydro.orcha_fill_guardcells_stage([pks[r]], 1, comms[r], streams[r])
        for r in range(R):
            hydro.orcha_hydro_stage_devdt(pks[r], 2, clocks[r].dt_tensor, streams[r])
    out["peer_per_stage_ms_per_rank_step"] = timed(step_ps, streams, steps, warmup) / R
    for c in comms:
        c.check()
        c.destroy()
    del pks
    return out


def single(steps=10, warmup=3, method="telescoped"):
    g, comms, pks = setup((1, 1, 1))
    for c in comms:
        c.destroy()
    s = torch.cuda.current_stream()
    clock = hydro.DevClock()

    def step():
        if method == "per-stage":
            hydro.orcha_fill_guardcells_stage(pks, 0, None, s)
        else:
            hydro.orcha_fill_guardcells(pks, None, s)
        hydro.orcha_compute_dt_device(pks, clock, None, s)
        hydro.step_devdt(pks, clock.dt_tensor, None, s, method)
    return timed(step, [s], steps, warmup)


def main():
    torch.cuda.set_device(0)
    lib = abi.load(False)
    abi.call(lib, "orcha_set_fill_mode", 1)
    one = single()
    one_ps = single(method="per-stage")
    rows = [measure(gr) for gr in ((2, 1, 1), (2, 2, 1), (2, 2, 2))]
    for r in rows:
        r["peer_per_stage_vs_single_telescoped"] = r["peer_per_stage_ms_per_rank_step"] / one - 1.0
        r["exchange_overhead_vs_single"] = r["exchange_ms_per_rank_step"] / one - 1.0
        r["peer_overhead_vs_single"] = r["peer_ms_per_rank_step"] / one - 1.0
        r["overlap_overhead_vs_single"] = r["overlap_ms_per_rank_step"] / one - 1.0
    print(json.dumps({"single_rank_ms_per_step": one, "single_rank_per_stage_ms_per_step": one_ps, "rows": rows, "gpu": torch.cuda.get_device_name(0),
                      "note": "virtual ranks on one GPU, each with cfg4's 4096-block brick; per-rank step = "
                              "the R-rank step / R; no NVLink wire time is included in either path"}))


if __name__ == "__main__":
    main()
