"""Per-kernel mean duration and share of an ncu launch-list CSV."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, mi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
per = {}
for r in rows[1:]:
    per.setdefault((r[ii], r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
tot = {}
for (i, k), m in per.items():
    n = k.split("(")[0][:70]
    t = tot.setdefault(n, [0, 0.0, m.get("launch__grid_size", 0), m.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0)])
    t[0] += 1
    t[1] += m["gpu__time_duration.sum"]
T = sum(v[1] for v in tot.values())
for n, (c, s, gsz, occ) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{n:70s} n={c:3d} mean={s / c / 1e3:8.1f} us share={s / T:.3f} grid={gsz:.0f} warps%={occ:.0f}")
