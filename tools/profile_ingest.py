"""Profiling driver (no parity checks): eager ingest of `--batches` batches of a config with
per-kernel CUDA-event timing; meant to be run plain, then under ncu with -k <kernel>.

    python tools/profile_ingest.py --config medium --batches 8
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="medium")
    ap.add_argument("--batches", type=int, default=8)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--synthetic-counts", action="store_true",
                    help="Poisson(0.05) counts instead of the forward model (same bytes, fast startup)")
    args = ap.parse_args()
    import torch
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS, Acquisition
    cfg = CONFIGS[args.config]
    batch = args.batch or cfg.batch or 4096
    n = min(cfg.S, batch * args.batches)
    idx = np.arange(n, dtype=np.int32)
    if args.synthetic_counts:
        rng = np.random.default_rng(0)
        fr = rng.poisson(0.05 * 65536 / (cfg.Q * cfg.Q) * 10, size=(n, cfg.Q, cfg.Q)).astype(
            np.uint16 if cfg.dtype == "u16" else np.float32)
    else:
        fr = Acquisition(cfg).frames_parallel(idx)
    dev = torch.from_numpy(fr).cuda()
    plan = wdd.Plan.from_config(cfg, ingest_overlap=True)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    for rep in range(args.reps):
        plan.reset()
        plan.profile_enable(True)
        for a in range(0, n, batch):
            plan.ingest(dev[a:a + batch], idx[a:a + batch], s)
        out = plan.readout()
        torch.cuda.synchronize()
        line = []
        for k in ("project", "rowdft", "flush", "readout", "finalize"):
            ms, c = plan.profile_read(k)
            line.append(f"{k}: {1e3 * ms / max(c, 1):.2f} us x{c}")
        print(f"rep {rep}: " + ", ".join(line), flush=True)
    plan.profile_enable(False)
    print("ok", float(out.abs().mean()))


if __name__ == "__main__":
    main()
