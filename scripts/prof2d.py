"""Profiling driver for the one-kernel 2D step: 2D Sedov 2048^2 (128 x 128 blocks of 16^2), 6 device-dt steps (ncu target)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import orcha_inputs as inp
from paper_2507_09337_b200 import hydro
g = hydro.Grid(2, (16, 16), (128, 128))
pk = hydro.Packet(g, np.arange(g.nblocks))
pk.pack(inp.to_blocks(inp.sedov(g.N[:2]), (16, 16), pk.block_ids))
clock = hydro.DevClock()
for _ in range(6):
    hydro.orcha_fill_guardcells([pk])
    hydro.orcha_compute_dt_device([pk], clock)
    hydro.orcha_hydro_advance_devdt(pk, clock.dt_tensor)
torch.cuda.synchronize()
