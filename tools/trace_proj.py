"""Timeline of CTA 0 of the projection kernel (trace build: WDD_NVCC_EXTRA=-DWDD_TRACE)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
NAMES = {2: "prod issue TMA", 3: "conv raw landed", 4: "conv A full", 5: "mma1 A ready",
         6: "mma1 acc free", 8: "epi acc1 full", 10: "epi A2 written", 11: "epi a2_full", 12: "mma2 start",
         13: "conv A slot free", 14: "epi s2 done", 15: "epi C stored"}


def main():
    import torch
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "medium"]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    lib = wdd.load_library()
    lib.wdd_trace_dump.restype = ctypes.c_int
    rng = np.random.default_rng(0)
    fr = rng.poisson(2.0, size=(n, cfg.Q, cfg.Q)).astype(np.uint16)
    dev = torch.from_numpy(fr).cuda()
    plan = wdd.Plan.from_config(cfg, ingest_overlap=True)
    out = torch.empty((n, cfg.K), device="cuda")
    for _ in range(2):
        buf = (ctypes.c_ulonglong * 65536)()
        lib.wdd_trace_dump(buf, 65536)
        plan.project(dev, out)
        torch.cuda.synchronize()
        k = lib.wdd_trace_dump(buf, 65536)
    ev = sorted((v >> 16, (v >> 8) & 0xff, v & 0xff) for v in buf[:k] if v)
    t0 = ev[0][0]
    w0 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    for t, c, j in ev[w0:w0 + 100000]:
        print(f"{(t - t0) / 1000:9.3f} us  {NAMES.get(c, c):18s} {j}")
    for c in sorted(NAMES):
        ts = [t for t, cc, _ in ev if cc == c]
        if len(ts) > 2:
            print(f"{NAMES[c]:18s} n={len(ts)} mean gap {(ts[-1] - ts[0]) / (len(ts) - 1) / 1000:.3f} us")


if __name__ == "__main__":
    main()
