#!/usr/bin/env python
"""Per-rank readout cost of a coefficient-sharded group, measured on one GPU.

For n = 1, 2, 4, 8: n linked plans of the config (k_shards = n) on one device, one whole
acquisition ingested with rows split across the plans (each plan's projection writes every
shard's coefficients), then the readout of ONE plan -- the flush of its K/n coefficients over the
whole scan and its partial Wiener readout, what each rank of an n-GPU group runs before the o
allreduce -- timed with CUDA events (median of --reps).  The projection time per rank is the
single-GPU stage time / n (HBM-bound, independent per GPU).  Prints one JSON line.

    python tools/shard_readout.py [--config box] [--reps 5]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="box")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--shards", default="1,2,4,8")
    args = ap.parse_args()
    import torch
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS
    from synth.gpu import GpuAcquisition
    cfg = CONFIGS[args.config]
    fb = cfg.Q * cfg.Q * 2
    pool_n = min(cfg.S, (1 << 30) // fb)
    pool = torch.cat([GpuAcquisition(cfg).frames(np.arange(a, min(pool_n, a + 4096))) for a in range(0, pool_n, 4096)])
    batch = min(pool_n, 8192)
    res = {}
    for n in [int(x) for x in args.shards.split(",")]:
        plans = [wdd.Plan.from_config(cfg, k_shards=n if n > 1 else 0, k_rank=r, ingest_overlap=True) for r in range(n)]
        if n > 1:
            wdd.link_shards(plans)
        blocks = np.array_split(np.arange(cfg.Sy), n)
        out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda")
        times = []
        for rep in range(args.reps + 1):
            for p in plans:
                p.reset()
            for r, rows in enumerate(blocks):
                idx = (rows[:, None] * cfg.Sx + np.arange(cfg.Sx)[None, :]).reshape(-1).astype(np.int32)
                for a in range(0, len(idx), batch):
                    s = idx[a:a + batch]
                    for q, p in enumerate(plans):
                        if q == r:
                            p.ingest(pool[(a % pool_n):(a % pool_n) + len(s)], s)
                        else:
                            p.ingest_remote(s)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plans[0].readout_spectrum(out, combine=False)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1))
            for p in plans[1:]:                       # (the other shards' flushes, untimed)
                p.readout_spectrum(out, combine=False)
            torch.cuda.synchronize()
        res[n] = {"readout_ms_median": float(np.median(times)), "k_count": plans[0].k_count}
        for p in plans:
            p.close()
        torch.cuda.empty_cache()
    base = res[min(res)]["readout_ms_median"]
    print(json.dumps({"config": cfg.name, "per_rank_readout": res,
                      "ratio_to_n1": {n: base / v["readout_ms_median"] for n, v in res.items()},
                      "how": "one plan's flush + partial readout of its K/n coefficients over the whole scan, "
                             "CUDA events, median of %d" % args.reps}), flush=True)


if __name__ == "__main__":
    main()
