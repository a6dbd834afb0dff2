"""Warp-stall samples per CUDA source line (ncu --page source --print-source cuda,sass; the build
uses -lineinfo), hottest first, with the two dominant stall reasons of each line.

    python tools/ncu_lines.py report.ncu-rep [n] [kernel-regex]
"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, path, h, agg = None, None, None, {}
sections = []


def flush():
    if fn is not None and agg:
        sections.append((fn, agg))


for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r[0] == "Function Name":
        flush()
        fn, agg = r[1], {}
    elif r[0] == "Line No":
        h = r
    elif h is not None and r[0].isdigit() and len(r) == len(h):
        i_s = h.index("Warp Stall Sampling (All Samples)")
        try:
            s = float(r[i_s])
        except ValueError:
            continue
        if s <= 0:
            continue
        key = (path, int(r[0]))
        e = agg.setdefault(key, {"s": 0.0, "src": r[1].strip()[:70], "st": {}})
        e["s"] += s
        for i, x in enumerate(h):
            if x.startswith("stall_"):
                try:
                    e["st"][x[6:]] = e["st"].get(x[6:], 0.0) + float(r[i] or 0)
                except ValueError:
                    pass
flush()
for name, a in sections:
    if pat and not pat.search(name):
        continue
    tot = sum(e["s"] for e in a.values())
    print(f"== {name[:100]}  samples {tot:.0f}")
    for (f, ln), e in sorted(a.items(), key=lambda kv: -kv[1]["s"])[:n]:
        top = sorted(((v, k) for k, v in e["st"].items()), reverse=True)[:2]
        print(f"{e['s'] / tot * 100:5.1f}%  {f}:{ln:<5d} {e['src']:70s} " + " ".join(f"{k}={v:.0f}" for v, k in top if v))
