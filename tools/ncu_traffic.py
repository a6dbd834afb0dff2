"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and duration of
the projection kernel from an `ncu --set full` report and record it in profiles/ncu_traffic.json
(bench.py reports it as roofline.traffic).

    python tools/ncu_traffic.py report.ncu-rep workload [kernel-regex]
"""
import csv
import json
import os
import re
import subprocess
import sys

rep, workload = sys.argv[1], sys.argv[2]
pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else "project_kernel")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def val(r, name):
    i = h.index(name)
    return float(r[i].replace(",", "")) * scale.get(units[i], 1)
recs = []
for r in rows[2:]:
    if pat.search(r[h.index("Kernel Name")]):
        recs.append({"kernel": r[h.index("Kernel Name")][:80],
                     "dram_read": val(r, "dram__bytes_read.sum"), "dram_write": val(r, "dram__bytes_write.sum"),
                     "grid": r[h.index("Grid Size")] if "Grid Size" in h else None})
assert recs, "kernel not found"
r0 = recs[0]
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[workload] = {"project_kernel_bytes_per_launch": r0["dram_read"] + r0["dram_write"], "dram_read": r0["dram_read"],
               "dram_write": r0["dram_write"], "source": os.path.basename(rep), "kernel": r0["kernel"]}
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(d[workload], indent=1))
