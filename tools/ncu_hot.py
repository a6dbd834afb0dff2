"""Hottest SASS instructions (warp-stall samples) per kernel of an ncu report.

    python tools/ncu_hot.py report.ncu-rep [n] [kernel-regex]
"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        sections.append(cur)
    elif r and r[0] == "Address":
        cur["h"] = r
    elif cur is not None and "h" in cur:
        cur["rows"].append(r)
for sec in sections:
    if pat and not pat.search(sec["name"]):
        continue
    h = sec["h"]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    stall = [i for i, x in enumerate(h) if x.startswith("stall_")]
    data = [r for r in sec["rows"] if len(r) > i_s and r[i_s].strip() not in ("", "0")]
    tot = sum(float(r[i_s]) for r in data)
    data.sort(key=lambda r: -float(r[i_s]))
    print(f"== {sec['name'][:100]}  samples {tot:.0f}")
    for r in data[:n]:
        top = sorted(((float(r[i] or 0), h[i]) for i in stall), reverse=True)[:2]
        print(f"{float(r[i_s]) / tot * 100:5.1f}%  {r[0][-5:]} {r[1][:58]:58s} " +
              " ".join(f"{k[6:]}={v:.0f}" for v, k in top if v))
