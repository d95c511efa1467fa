"""Per-barrier-interval sampling profile of one kernel in an ncu report:
where the warps are (samples) between consecutive BAR.SYNCs, and which
barrier they wait at.  usage: sass_phases.py REPORT KERNEL_REGEX"""
import csv
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for ln in out.splitlines():
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
blk = [b for b in blocks if re.search(kre, b[0])][0]
print(blk[0][:120])
rows = list(csv.reader(blk[1:]))
h = rows[0]
S = h.index("Source")
W = h.index("Warp Stall Sampling (All Samples)")
E = h.index("Instructions Executed")
B = h.index("stall_barrier")
tot = sum(int(r[W] or 0) for r in rows[1:])
seg, segi, segs = 0, 0, []
start = 0
for n, r in enumerate(rows[1:]):
    seg += int(r[W] or 0)
    segi += int(r[E] or 0)
    if "BAR.SYNC" in r[S] or "BAR.RED" in r[S]:
        segs.append((start, n, seg, segi, r[S].strip(), int(r[B] or 0)))
        seg, segi, start = 0, 0, n + 1
segs.append((start, len(rows) - 2, seg, segi, "(end)", 0))
print(f"total samples {tot}")
for a, b, sm, ie, src, bs in segs:
    print(f"[{a:5d},{b:5d}] samples {sm:7d} ({sm / tot:5.1%})  warp-inst {ie:11d}  ends at {src[:30]:30s} barrier-stall {bs}")
if len(sys.argv) > 3:
    a, b = map(int, sys.argv[3].split(":"))
    top = sorted(((int(r[W] or 0), n, r[S].strip()) for n, r in enumerate(rows[1:]) if a <= n <= b), reverse=True)[:25]
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    for sm, n, src in top:
        r = rows[1 + n]
        st = sorted(((int(r[h.index(c)] or 0), c[6:]) for c in cols), reverse=True)[:3]
        print(f"{n:5d} {sm:6d} {src[:60]:60s} {st}")
