#!/usr/bin/env python
"""Profiling driver: a device-resident pool of seeded sparse frames (synth/sparse.py) cycled over
the first `--rows` scan rows of a config, ingested in the config's batches, then one readout;
`--reps` times.  Meant to be run under ncu with -k <kernel> -s <skip> -c <count>.

    python tools/prof_cfg.py --config live --rows 64 --reps 2 [--accumulator spectrum]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="live")
    ap.add_argument("--rows", type=int, default=64)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--pool", type=int, default=4096)
    ap.add_argument("--accumulator", default="G")
    ap.add_argument("--readout-rows", type=int, default=0, help="also read out every N rows")
    args = ap.parse_args()
    import torch
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS
    from synth.sparse import dense_frames_torch, sparse_events
    cfg = CONFIGS[args.config]
    batch = args.batch or cfg.batch or 16384
    n = min(cfg.S, args.rows * cfg.Sx)
    pool_n = min(n, max(args.pool, batch))
    pool = torch.cat([dense_frames_torch(*sparse_events(7, np.arange(a, min(pool_n, a + 4096)), cfg.Q), cfg.Q, "cuda")
                      for a in range(0, pool_n, 4096)])
    plan = wdd.Plan.from_config(cfg, accumulator=args.accumulator, ingest_overlap=True)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda")
    for _ in range(args.reps):
        plan.reset()
        for a in range(0, n, batch):
            b = min(n, a + batch)
            p0 = a % pool_n
            fr = pool[p0:p0 + (b - a)] if p0 + (b - a) <= pool_n else pool[:b - a]
            plan.ingest(fr, np.arange(a, b, dtype=np.int32), st)
            if args.readout_rows and (b // cfg.Sx) % args.readout_rows == 0 and b < n and b % cfg.Sx == 0:
                plan.readout(out)
        plan.readout(out)
        torch.cuda.synchronize()
    print("ok", cfg.name, n, "frames")


if __name__ == "__main__":
    main()
