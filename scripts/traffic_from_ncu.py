"""Write profiles/traffic.json: DRAM bytes (read + write) per advance (every
stage_fused_kernel<16,1,...> launch of one step -- the borrowed ring's box /
18 x 18 and interior kernels -- plus <16,2>) from an ncu --set full report
holding one step's launches."""
import csv
import json
import subprocess
import sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units = r[0], r[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
per = {}
for row in r[2:]:
    name = row[h.index("Kernel Name")].replace("(int)", "").replace("(bool)", "")
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        b += float(row[i]) * scale[units[i]]
    key = "stage1" if "16, 1" in name else "stage2" if "16, 2" in name else name[:40]
    per[key] = per.get(key, 0.0) + b
tot = per.get("stage1", 0.0) + per.get("stage2", 0.0)
src = sys.argv[3] if len(sys.argv) > 3 else rep
json.dump({"advance_bytes_per_launch": tot, "per_kernel_bytes": per, "source": src,
           "bytes_per_cell_update": tot / (4096 * 16 ** 3)}, open(out, "w"), indent=1)
print(open(out).read())
