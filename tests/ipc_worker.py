"""Worker of tests/test_gpu_ipc.py: one rank of the F2 peer mode across
PROCESSES (CUDA IPC), launched by torch.distributed.run with every rank on
GPU 0; gloo carries only the IPC blobs and the results.

  python -m torch.distributed.run --nproc-per-node R tests/ipc_worker.py OUT parity|production STEPS CASE [METHOD]
"""
import os
import pickle
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import orcha_inputs as inp  # noqa: E402
from paper_2507_09337_b200 import hydro  # noqa: E402

# (nb, nblk, bc, gpu grid, brick, initial condition)
CASES = {
    "sedov8": ((8, 8, 8), (4, 2, 2), ((0, 0),) * 3, (2, 1, 1), (2, 2, 2), "sedov"),
    "random16": ((16, 16, 16), (2, 2, 1), ((1, 1), (0, 2), (1, 1)), (2, 2, 1), (1, 1, 1), "random"),
}


def main():
    out, mode, steps, case = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    method = sys.argv[5] if len(sys.argv) > 5 else "telescoped"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    nb, nblk, bc, gg, brick, ic = CASES[case]
    g = hydro.Grid(3, nb, nblk, bc=bc, parity=(mode == "parity"))
    owner = hydro.brick_owner(nblk, brick, gg)
    U0 = inp.sedov(g.N) if ic == "sedov" else inp.random_field(g.N, seed=91)
    ids = np.flatnonzero(owner == rank)
    pk = hydro.Packet(g, ids)
    pk.pack(inp.to_blocks(U0, g.nb, ids))
    comm = hydro.Comm.create_ipc(g, world, rank, owner)
    blobs = [None] * world
    dist.all_gather_object(blobs, comm.ipc_export(pk))
    comm.ipc_attach(blobs)
    hydro.orcha_fill_prepare([pk], comm)
    torch.cuda.synchronize()
    dist.barrier()
    clock = hydro.DevClock()
    s = torch.cuda.current_stream()
    log = []
    for _ in range(steps):
        if method == "per-stage":
            hydro.orcha_fill_guardcells_stage([pk], 0, comm, s)
            hydro.orcha_compute_dt_device([pk], clock, comm, s)
            hydro.orcha_hydro_stage_devdt(pk, 1, clock.dt_tensor, s)
            hydro.orcha_fill_guardcells_stage([pk], 1, comm, s)
            hydro.orcha_hydro_stage_devdt(pk, 2, clock.dt_tensor, s)
        else:
            hydro.orcha_fill_guardcells([pk], comm, s)
            hydro.orcha_compute_dt_device([pk], clock, comm, s)
            hydro.orcha_hydro_advance_devdt(pk, clock.dt_tensor, s)
        s.synchronize()
        c = clock.read()
        log.append((c.dt, c.smax, c.argmax, c.tag))
    comm.check()
    res = pk.unpack()
    allr = [None] * world
    dist.all_gather_object(allr, (ids.tolist(), res, log))
    if rank == 0:
        with open(out, "wb") as f:
            pickle.dump(allr, f)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
