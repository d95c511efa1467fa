"""The README's Python example, as a script (python scripts/readme_example.py)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, orcha_inputs as inp
from paper_2507_09337_b200 import hydro
g = hydro.Grid(3, (16, 16, 16), (8, 8, 8))            # 128^3 cells, 4 guards, outflow, gamma 1.4
pk = hydro.Packet(g, np.arange(g.nblocks))             # one packet of 512 blocks
pk.pack(inp.to_blocks(inp.sedov(g.N), g.nb, pk.block_ids))
t, nsteps, log = hydro.run([pk], t_end=0.01)           # fill -> dt -> telescoped RK2 step, until t_end
state = pk.unpack()                                    # (blocks, 5, 16, 16, 16) interiors
print(t, nsteps, state.shape)
print(hydro.mesh_checksums([pk]))                      # FNV-1a per variable
