"""Packet-size sweep (BASELINE.json configs[4]; the B200 analogue of the
paper's Fig. sedov3d-perf: time vs blocks per DataPacket).

Per GPU 16.8 M cells = 32768 x 8^3, 4096 x 16^3 or 512 x 32^3 blocks of a 3D
Sedov grid; the blocks are split into packets of P blocks; one step = fill
(all packets) -> dt (all packets) -> advance every packet, through the C ABI.
With S streams the packets' advances are dealt round-robin over S CUDA
streams after the fill (packets in flight concurrently, the paper's
multi-stream ORCHA runtime; the advances of different packets are
independent once the fill is done).  Prints one JSON object (cell-updates/s
per (block size, P, S))."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import orcha_inputs as inp  # noqa: E402
from paper_2507_09337_b200 import hydro  # noqa: E402


def measure(nb, P, S=1, steps=6, warmup=3):
    N = (256, 256, 256)
    nblk = tuple(n // nb for n in N)
    g = hydro.Grid(3, (nb,) * 3, nblk)
    ids = np.arange(g.nblocks)
    t0 = time.perf_counter()
    pk = [hydro.Packet(g, ids[i:i + P]) for i in range(0, len(ids), P)]
    for p in pk:
        p.pack(inp.sedov_packet(N, (nb,) * 3, p.block_ids))
    setup = time.perf_counter() - t0
    s = torch.cuda.current_stream()
    side = [torch.cuda.Stream() for _ in range(S)] if S > 1 else [s]

    def step():
        hydro.orcha_fill_guardcells(pk, None, s)
        info = hydro.orcha_compute_dt(pk, math.inf, None, s)   # synchronizes the host
        if S > 1:
            ev = torch.cuda.Event()
            ev.record(s)
            for st in side:
                st.wait_event(ev)
        for i, p in enumerate(pk):
            hydro.orcha_hydro_advance(p, info.dt, side[i % S])
        if S > 1:
            for st in side:
                e2 = torch.cuda.Event()
                e2.record(st)
                s.wait_event(e2)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(steps):
        step()
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    del pk
    torch.cuda.empty_cache()
    return {"nb": nb, "blocks_per_packet": P, "streams": S, "packets": math.ceil(len(ids) / P), "ms_per_step": ms,
            "cell_updates_per_s": 256 ** 3 / (ms / 1e3), "setup_s": setup}


def main():
    torch.cuda.set_device(0)
    rows = []
    plan = {8: [16, 64, 256, 1024, 4096, 32768], 16: [8, 32, 128, 512, 2048, 4096], 32: [8, 32, 128, 512]}
    for nb, Ps in plan.items():
        for P in Ps:
            for S in ((1, 4, 16) if P * 4 <= 32768 // (nb // 8) ** 3 else (1,)):
                r = measure(nb, P, S)
                rows.append(r)
                print(json.dumps(r), flush=True)
    print(json.dumps({"packet_sweep": rows, "grid": [256, 256, 256], "gpu": torch.cuda.get_device_name(0)}))


if __name__ == "__main__":
    main()
