"""Timeline of the streamed e2e step (bench.py streamed_e2e) from the CUDA
activity trace of torch.profiler (CUPTI): per step, every memcpy and kernel
with its start / end relative to the step's first H2D.  Diagnostic only."""
import json
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import orcha_inputs as inp  # noqa: E402
from paper_2507_09337_b200 import abi, hydro  # noqa: E402


def main(K=8, nsteps=3, prio=-1):
    torch.cuda.set_device(0)
    lib = abi.load(False)
    abi.call(lib, "orcha_set_fill_mode", 1)
    nblk = bench.BRICK_BLOCKS
    NB = bench.NB
    N = tuple(nblk[a] * NB[a] for a in range(3))
    g = hydro.Grid(3, NB, nblk, xmin=(0.0, 0.0, 0.0), xmax=(1.0, 1.0, 1.0))
    ids = np.arange(nblk[0] * nblk[1] * nblk[2])
    slabs = [a for a in np.array_split(ids, K) if len(a)]
    pks = [hydro.Packet(g, a) for a in slabs]
    mesh = [torch.from_numpy(inp.sedov_packet(N, NB, a, xmax=(1.0, 1.0, 1.0))).pin_memory() for a in slabs]
    stream = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(priority=prio), torch.cuda.Stream(priority=prio)
    done = [None] * len(pks)

    def one():
        ev_in = []
        for i, p in enumerate(pks):
            if done[i] is not None:
                h2d.wait_event(done[i])
            p.pack(mesh[i], h2d)
            e = torch.cuda.Event()
            e.record(h2d)
            ev_in.append(e)
        for e in ev_in:
            stream.wait_event(e)
        hydro.orcha_fill_guardcells(pks, None, stream)
        info = hydro.orcha_compute_dt(pks, math.inf, None, stream)
        for i, p in enumerate(pks):
            hydro.orcha_hydro_advance(p, info.dt, stream)
            e = torch.cuda.Event()
            e.record(stream)
            d2h.wait_event(e)
            p.unpack(mesh[i], d2h, sync=False)
            e2 = torch.cuda.Event()
            e2.record(d2h)
            done[i] = e2

    one()
    one()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(nsteps):
            one()
        torch.cuda.synchronize()
    ev = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        ev.append((e.time_range.start, e.time_range.end, e.name[:48]))
    ev.sort()
    t0 = ev[0][0]
    out = [(round((s - t0) / 1e3, 3), round((e - t0) / 1e3, 3), n) for s, e, n in ev]
    for s, e, n in out:
        print(f"{s:9.3f} {e:9.3f} {e - s:7.3f}  {n}")
    json.dump(out, open("gpurun_out/e2e_timeline.json", "w"))


if __name__ == "__main__":
    main(K=int(sys.argv[1]) if len(sys.argv) > 1 else 8)
