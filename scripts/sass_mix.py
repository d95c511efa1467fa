"""Opcode mix (warp-level executed instructions) per kernel from an ncu report's SASS source page."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0   # divide counts by this (e.g. cell-updates/32)
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = txt.split('"Kernel Name",')
for b in blocks[1:]:
    lines = b.splitlines()
    name = lines[0][:80]
    rd = csv.reader(io.StringIO("\n".join(lines[1:])))
    hdr = next(rd)
    ai, si, ei = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    wi = hdr.index("Warp Stall Sampling (All Samples)")
    mix = collections.Counter()
    stall = collections.Counter()
    tot = 0
    for row in rd:
        if len(row) <= ei:
            continue
        op = row[si].strip().split(" ")[0]
        if op.startswith("@"):
            op = row[si].strip().split(" ")[1]
        base = op.split(".")[0]
        n = float(row[ei] or 0)
        mix[base] += n
        stall[base] += float(row[wi] or 0)
        tot += n
    print("===", name, f"total {tot/norm:.1f}")
    for op, n in mix.most_common(28):
        print(f"  {op:12s} {n/norm:10.1f}  {100*n/tot:5.1f}%  stall-samples {stall[op]:.0f}")
