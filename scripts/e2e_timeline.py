"""Timeline of bench.py's streamed e2e step (bench.streamed_loop, the exact
loop `e2e` times) from the CUDA activity trace of torch.profiler (CUPTI):
every memcpy and kernel with its start / end, plus per-step link idle time.
Diagnostic only.  Usage: python scripts/e2e_timeline.py [packets] [copy_streams]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2507_09337_b200 import abi, hydro  # noqa: E402


def main(K=16, cs=2, nsteps=3):
    torch.cuda.set_device(0)
    lib = abi.load(False)
    abi.call(lib, "orcha_set_fill_mode", 1)
    nblk = bench.BRICK_BLOCKS
    N = tuple(nblk[a] * bench.NB[a] for a in range(3))
    g = hydro.Grid(3, bench.NB, nblk, xmin=(0.0, 0.0, 0.0), xmax=(1.0, 1.0, 1.0))
    ids = np.arange(nblk[0] * nblk[1] * nblk[2])
    stream = torch.cuda.current_stream()
    pks, mesh, one, done = bench.streamed_loop(g, ids, N, 1, 1, 1, None, stream, K, -1, cs)
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
    # per direction: busy time (union of copy intervals) over the whole trace
    span = out[-1][1] - out[0][0]
    for tag in ("HtoD", "DtoH"):
        iv = sorted((s, e) for s, e, n in out if tag in n and "Pinned" in n)
        busy, cur = 0.0, None
        for s, e in iv:
            if cur is None or s > cur[1]:
                if cur:
                    busy += cur[1] - cur[0]
                cur = [s, e]
            else:
                cur[1] = max(cur[1], e)
        if cur:
            busy += cur[1] - cur[0]
        print(f"# {tag}: busy {busy:.2f} of {span:.2f} ms ({100 * busy / span:.0f} %)")
    json.dump(out, open("gpurun_out/e2e_timeline.json", "w"))


if __name__ == "__main__":
    main(K=int(sys.argv[1]) if len(sys.argv) > 1 else 16, cs=int(sys.argv[2]) if len(sys.argv) > 2 else 2)
