"""Timeline of CTA 0 of the pipelined GEMM flush (trace build: WDD_NVCC_EXTRA=-DWDD_TRACE):
per k-tile c the times of producer issue, converter start / done, MMA start / commit, epilogue
start / done, relative to the producer issue of the same tile."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
NAMES = {0: "prod", 1: "conv0", 2: "conv1", 3: "mma0", 4: "mma1", 5: "epi0", 6: "epi1"}


def main():
    import torch
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS
    from synth.sparse import dense_frames_torch, sparse_events
    cfg = CONFIGS["live"]
    lib = wdd.load_library()
    lib.wdd_trace_dump.restype = ctypes.c_int
    plan = wdd.Plan.from_config(cfg, accumulator=sys.argv[1] if len(sys.argv) > 1 else "G")
    pool = torch.cat([dense_frames_torch(*sparse_events(7, np.arange(a, a + 4096), cfg.Q), cfg.Q, "cuda")
                      for a in range(0, 8192, 4096)])
    out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda")
    buf = (ctypes.c_ulonglong * 65536)()
    for rep in range(2):
        plan.reset()
        for blk in range(2):
            for a in range(blk * 32768, (blk + 1) * 32768, 1024):
                plan.ingest(pool[(a % 8192):(a % 8192) + 1024], np.arange(a, a + 1024, dtype=np.int32))
            torch.cuda.synchronize()
            lib.wdd_trace_dump(buf, 65536)
            plan.readout(out)
            torch.cuda.synchronize()
            k = lib.wdd_trace_dump(buf, 65536)
    ev = [(v >> 16, (v >> 8) & 0xff, v & 0xff) for v in buf[:k] if v]
    by = {}
    for t, code, j in ev:
        by.setdefault(code, []).append(t)
    for code in by:
        by[code].sort()
    n = min(len(v) for v in by.values())
    t0 = by[0][0]
    print("tile  " + " ".join(f"{NAMES[c]:>8s}" for c in sorted(by)))
    for i in list(range(0, min(n, 24))) + list(range(max(24, n - 8), n)):
        print(f"{i:4d}  " + " ".join(f"{(by[c][i] - t0) / 1000:8.2f}" for c in sorted(by)))
    for c in sorted(by):
        ts = by[c]
        print(f"{NAMES[c]:6s} n={len(ts)} mean gap {(ts[-1] - ts[0]) / max(1, len(ts) - 1) / 1000:.3f} us")


if __name__ == "__main__":
    main()
