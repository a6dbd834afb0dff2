"""Print the hottest SASS instructions (warp-stall samples) of an ncu report: python tools/ncu_hot.py rep [n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
i_s = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_")]
data = [r for r in rows[2:] if len(r) > i_s and r[i_s].strip() not in ("", "0")]
tot = sum(float(r[i_s]) for r in data)
data.sort(key=lambda r: -float(r[i_s]))
print(f"total samples {tot:.0f}")
for r in data[:n]:
    top = sorted(((float(r[i] or 0), h[i]) for i in stall_cols), reverse=True)[:2]
    print(f"{float(r[i_s]) / tot * 100:5.1f}%  {r[1][:60]:60s} " + " ".join(f"{k[6:]}={v:.0f}" for v, k in top if v))
