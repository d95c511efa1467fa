"""F4 "second workload": the cost of the EOS (the paper: the Helmholtz EOS
"makes GPU more favorable").  cfg4's 3D Sedov (4096 blocks of
16^3, one packet, telescoped step) with the gamma law and with the gas +
radiation surrogate at several work multipliers w (temperature solves per
EOS evaluation): GPU cell-updates/s, and the CPU oracle's (1 thread, a 48^3
sub-box of the same setup) for the same EOS -- the GPU/CPU ratio as the EOS
gets more expensive.  Prints one JSON object."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (the CPU baseline leg only)
import orcha_inputs as inp  # noqa: E402
from paper_2507_09337_b200 import hydro  # noqa: E402

ARAD = 1e-4


def gpu(eos, w, steps=8, warmup=3):
    N = (256, 256, 256)
    g = hydro.Grid(3, (16, 16, 16), (16, 16, 16), eos=eos, eos_work=w, arad=ARAD)
    ids = np.arange(g.nblocks)
    pk = hydro.Packet(g, ids)
    pk.pack(inp.sedov_packet(N, (16, 16, 16), ids))
    s = torch.cuda.current_stream()

    def step():
        hydro.orcha_fill_guardcells([pk], None, s)
        info = hydro.orcha_compute_dt([pk], math.inf, None, s)
        hydro.orcha_hydro_advance(pk, info.dt, s)

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
    return 256 ** 3 / (ms / 1e3), ms


def cpu(eos, w, n=48, steps=2):
    kw = dict(eos=eos, eos_work=w, arad=ARAD) if eos else {}
    g = oracle.Grid(N=(n, n, n), **kw)
    U = oracle.padded(g, inp.sedov((n, n, n)))
    t0 = time.perf_counter()
    oracle.run(g, U, nsteps=steps)
    dt = time.perf_counter() - t0
    return n ** 3 * steps / dt, dt


def main():
    torch.cuda.set_device(0)
    rows = []
    for eos, w in ((0, 1), (1, 1), (1, 4), (1, 16)):
        gv, gms = gpu(eos, w)
        cv, cs = cpu(eos, w)
        r = {"eos": "gamma-law" if eos == 0 else "gas+radiation", "work": w, "gpu_cell_updates_per_s": gv,
             "gpu_ms_per_step": gms, "cpu_oracle_cell_updates_per_s": cv, "cpu_seconds": cs,
             "gpu_over_cpu": gv / cv}
        rows.append(r)
        print(json.dumps(r), flush=True)
    print(json.dumps({"eos_sweep": rows, "grid": [256, 256, 256], "arad": ARAD,
                      "cpu": "oracle, 1 thread, 48^3 Sedov sub-box, 2 steps", "gpu": torch.cuda.get_device_name(0)}))


if __name__ == "__main__":
    main()
