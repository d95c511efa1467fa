"""One or two packet-sweep points (scripts/packet_sweep.measure) for profiling."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts import packet_sweep as ps  # noqa: E402

pts = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or [(16, 2048, 1), (16, 4096, 1)]
for nb, P, S in pts:
    print(json.dumps(ps.measure(nb, P, S)), flush=True)
