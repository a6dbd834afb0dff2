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

if len(sys.argv) > 3 and sys.argv[3] == "conflicts":
    ic = h.index("L1 Conflicts Shared N-Way") if "L1 Conflicts Shared N-Way" in h else None
    iw = h.index("L1 Wavefronts Shared Excessive")
    allrows = [r for r in rows[2:] if len(r) > iw]
    allrows.sort(key=lambda r: -float(r[iw] or 0))
    print("--- top shared-memory excessive wavefronts")
    for r in allrows[:12]:
        print(r[iw], r[ic] if ic else "", r[0][-6:], r[1][:80])
if len(sys.argv) > 3 and sys.argv[3] == "ctx":
    addr = sys.argv[4]
    for k, r in enumerate(rows):
        if len(r) > 1 and r[0].endswith(addr):
            for rr in rows[max(2, k - 12):k + 4]:
                print(rr[0][-5:], rr[1][:90], rr[i_s] if len(rr) > i_s else "")
