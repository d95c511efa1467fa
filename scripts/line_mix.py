"""Executed instructions per SOURCE LINE / enclosing function of one kernel:
joins an ncu report's SASS page (per-address "Instructions Executed") with
the line table nvdisasm prints for the same cubin (-lineinfo build).

usage: line_mix.py REPORT KERNEL_REGEX CUBIN MANGLED_SUBSTR NORM
  NORM: divide warp-instruction counts by this (e.g. cell-updates / 32).
The library profiled must be the one the cubin came from (cuobjdump -xelf)."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre, cubin, mangled, norm = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], float(sys.argv[5])

# address -> (file, line) from nvdisasm's line table
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
addr_line = {}
inside, cur = False, None
for ln in dis.splitlines():
    if ln.startswith(".text.") and ln.rstrip(":").endswith(mangled) is False and mangled in ln:
        inside = True
        continue
    if inside and ln.startswith("//----") and mangled not in ln:
        break
    if not inside:
        continue
    m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        addr_line[int(m.group(1), 16)] = cur

# address -> executed (warp-level) from the ncu SASS page
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = txt.split('"Kernel Name",')
blk = [b for b in blocks[1:] if re.search(kre, b.splitlines()[0])][0]
lines = blk.splitlines()
rd = csv.reader(io.StringIO("\n".join(lines[1:])))
hdr = next(rd)
ai, ei = hdr.index("Address"), hdr.index("Instructions Executed")
per_line = collections.Counter()
tot = 0.0
base = None
for row in rd:
    if len(row) <= ei:
        continue
    a = int(row[ai], 16)
    if base is None:
        base = a
    n = float(row[ei] or 0)
    tot += n
    per_line[addr_line.get(a - base, ("?", 0))] += n


def enclosing(path_name, line, _cache={}):
    """Name of the function whose definition precedes `line` in the source."""
    if path_name not in _cache:
        import glob
        srcs = glob.glob(f"/root/repo/paper_2507_09337_b200/csrc/{path_name}")
        defs = []
        if srcs:
            for i, s in enumerate(open(srcs[0]).read().splitlines(), 1):
                m = re.match(r"(?:__device__|__global__|template|static|\s*auto)\s.*?(\w+)\s*(?:=\s*\[&\])?\(", s)
                if m and ("__device__" in s or "__global__" in s or "auto " in s):
                    defs.append((i, m.group(1)))
        _cache[path_name] = defs
    name = "?"
    for i, n in _cache[path_name]:
        if i <= line:
            name = n
    return name


per_fn = collections.Counter()
for (f, l), n in per_line.items():
    per_fn[(f, enclosing(f, l))] += n
print(f"{blk.splitlines()[0][:100]}\n  total {tot / norm:.1f} per unit ({len(addr_line)} mapped addresses)")
print("  by function:")
for (f, fn), n in per_fn.most_common(25):
    print(f"    {f:18s} {fn:24s} {n / norm:8.1f}  {100 * n / tot:5.1f}%")
print("  top lines:")
for (f, l), n in per_line.most_common(30):
    print(f"    {f}:{l:<5d} {n / norm:8.1f}  {100 * n / tot:5.1f}%")
