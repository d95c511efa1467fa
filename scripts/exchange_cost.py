"""On-GPU cost of the multi-GPU exchange step measured
with R virtual ranks on ONE B200 (LOCAL transport: the NCCL path's plan, the
halo pack kernel, a device copy standing in for ncclSend/Recv, the unpack
kernel), each rank owning cfg4's 16x16x16-block brick (gpu grids (2,1,1),
(2,2,1), (2,2,2)), one packet per rank in gather mode.

Per rank and step it reports the exchange bytes the plan moves (unique remote
cells x 40 B, both directions), the measured time of push + fill (pack, copy,
unpack, the local x-guard part) against the advance, and the wire time those
bytes would take at a stated NVLink rate (a projection: nothing here crosses
NVLink).  Prints one JSON object."""
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

NVLINK_GBS = 900.0  # B200 NVLink 5, per direction (nominal)


def measure(grid, steps=5, warmup=2):
    px, py, pz = grid
    R = px * py * pz
    BB = bench.BRICK_BLOCKS
    nblk = (BB[0] * px, BB[1] * py, BB[2] * pz)
    NB = bench.NB
    N = tuple(nblk[a] * NB[a] for a in range(3))
    g = hydro.Grid(3, NB, nblk, xmin=(0.0, 0.0, 0.0), xmax=(float(px), float(py), float(pz)))
    owner = hydro.brick_owner(nblk, BB, grid)
    comms = hydro.Comm.create_local(g, R, owner)
    pks = []
    for r in range(R):
        ids = np.flatnonzero(owner == r)
        p = hydro.Packet(g, ids)
        p.pack(inp.sedov_packet(N, NB, ids, xmax=(float(px), float(py), float(pz))))
        pks.append(p)
    s = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(rec=None):
        a, b, c = ev(), ev(), ev()
        a.record(s)
        for r in range(R):
            comms[r].push([pks[r]], s)
        for r in range(R):
            hydro.orcha_fill_guardcells([pks[r]], comms[r], s)
        b.record(s)
        info = hydro.orcha_compute_dt(pks, math.inf, None, s)
        c.record(s)
        for p in pks:
            hydro.orcha_hydro_advance(p, info.dt, s)
        d = ev()
        d.record(s)
        if rec is not None:
            rec.append((a, b, c, d))

    for _ in range(warmup):
        step()
    rec = []
    for _ in range(steps):
        step(rec)
    torch.cuda.synchronize()
    exch = sum(a.elapsed_time(b) for a, b, _, _ in rec) / steps / R
    adv = sum(c.elapsed_time(d) for _, _, c, d in rec) / steps / R
    # bytes: the plan of rank 0 (unique remote cells it receives; it sends as many by symmetry of the bricks)
    cells = sum(len(hydro.comm_plan(g, R, 0, owner, q, 1)) for q in range(1, R))
    plan_bytes = int(cells) * 40
    for c in comms:
        c.destroy()
    out = {"gpu_grid": list(grid), "ranks": R, "exchange_ms_per_rank": exch, "advance_ms_per_rank": adv,
           "exchange_share": exch / (exch + adv)}
    out["recv_bytes_rank0"] = plan_bytes
    out["projected_wire_ms_at_%d_GBs" % int(NVLINK_GBS)] = plan_bytes / (NVLINK_GBS * 1e9) * 1e3
    return out


def main():
    torch.cuda.set_device(0)
    lib = abi.load(False)
    abi.call(lib, "orcha_set_fill_mode", 1)
    rows = [measure(gr) for gr in ((2, 1, 1), (2, 2, 1), (2, 2, 2))]
    print(json.dumps({"exchange_cost": rows, "gpu": torch.cuda.get_device_name(0),
                      "note": "virtual ranks on one GPU: pack + device copy + unpack measured; the NVLink wire "
                              "time is a projection at the nominal per-direction rate"}))


if __name__ == "__main__":
    main()
