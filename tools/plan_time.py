#!/usr/bin/env python
"""Plan-creation wall time per config (host active set + device bank build + uploads), median
of 3 creations after one warm-up.  Prints one JSON line per config."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS
    names = sys.argv[1:] or ["tiny", "medium", "large", "live", "box"]
    for name in names:
        cfg = CONFIGS[name]
        wdd.Plan.from_config(cfg).close()
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            p = wdd.Plan.from_config(cfg)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            info = p.info()
            p.close()
        ts.sort()
        print(json.dumps({"config": name, "plan_create_s": ts[1], "n_act": info["n_act"], "K": cfg.K}), flush=True)


if __name__ == "__main__":
    main()
