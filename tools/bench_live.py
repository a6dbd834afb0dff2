#!/usr/bin/env python
"""Live / offline workload timings beyond bench.py's headline line:
per-batch ingest latency (p50 / p99 / max) and readout latency for the Live config (1024-frame
batches in scan order, readout every 64 rows), sustained frames/s of whole scans for Live, Large
and Box, from a device-resident frame pool of >= 1 GiB cycled over the scan positions.

    python tools/bench_live.py [--config live|large|box] [--pool-frames N] [--reps R]

Frames are the seeded sparse counting frames of synth/sparse.py materialised on the device (the
projection's cost does not depend on content).  Every timing is CUDA events on the ingest stream.
Prints one JSON line."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="live")
    ap.add_argument("--pool-frames", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--accumulator", default="G", choices=["G", "spectrum"])
    args = ap.parse_args()
    import torch
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS
    from synth.sparse import dense_frames_torch, sparse_events

    cfg = CONFIGS[args.config]
    batch = args.batch or cfg.batch or 16384
    pool_n = max(batch, args.pool_frames)
    pix, cnt = sparse_events(7, np.arange(pool_n), cfg.Q)
    pool = torch.cat([dense_frames_torch(pix[a:a + 4096], cnt[a:a + 4096], cfg.Q, "cuda")
                      for a in range(0, pool_n, 4096)])
    frame_bytes = cfg.Q * cfg.Q * 2
    plan = wdd.Plan.from_config(cfg, accumulator=args.accumulator, ingest_overlap=True)
    info = plan.info()
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    out = torch.empty((cfg.Sy, cfg.Sx), dtype=torch.complex64, device="cuda")
    rows_per_readout = cfg.readout_rows or cfg.Sy
    n_batches = (cfg.S + batch - 1) // batch

    import time
    host_us = []

    def scan(record):
        plan.reset()
        lat, rdl = [], []
        rows_done = 0
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        for b in range(n_batches):
            a0, a1 = b * batch, min(cfg.S, (b + 1) * batch)
            p0 = a0 % pool_n
            frames = pool[p0:p0 + (a1 - a0)] if p0 + (a1 - a0) <= pool_n else pool[:a1 - a0]
            idx_b = np.arange(a0, a1, dtype=np.int32)
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
            h0 = time.perf_counter()
            plan.ingest(frames, idx_b, st)
            host_us.append((time.perf_counter() - h0) * 1e6)
            if record:
                e1.record(st)
                lat.append((e0, e1))
            rows = a1 // cfg.Sx
            if rows - rows_done >= rows_per_readout or a1 == cfg.S:
                rows_done = rows
                if record:
                    r0 = torch.cuda.Event(enable_timing=True)
                    r1 = torch.cuda.Event(enable_timing=True)
                    r0.record(st)
                plan.readout(out)
                if record:
                    r1.record(st)
                    rdl.append((r0, r1))
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(st)
        torch.cuda.synchronize()
        return (t0.elapsed_time(t1), [a.elapsed_time(b) for a, b in lat], [a.elapsed_time(b) for a, b in rdl])

    scan(False)                                          # warm-up
    # sustained throughput: no events between the batches (an event record between two
    # PDL-chained launches would serialise them); latencies from separate scans with events
    res = [scan(False) for _ in range(args.reps)]
    total_ms = float(np.median([r[0] for r in res]))
    res_l = [scan(True) for _ in range(max(1, args.reps // 2))]
    lat = np.concatenate([r[1] for r in res_l]) * 1e3
    rdl = np.concatenate([r[2] for r in res_l]) * 1e3
    n_readouts = len(res_l[0][2])
    fps = cfg.S / (total_ms / 1e3)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    # algorithmic bytes of a whole scan: frames + C write/read + R write/read + per flush the G
    # read-modify-write (write only on the first flush) and the bank read of the fused readout
    # (spectrum-only accumulator: no G traffic, only the bank read per flush)
    g_passes = (3 * n_readouts - 1) if args.accumulator == "G" else n_readouts
    b_scan = cfg.S * (frame_bytes + 8 * cfg.K + 16 * info["n_vx"] * cfg.K / cfg.Sx) + \
        info["n_act"] * cfg.K * 8 * g_passes
    line = {
        "config": cfg.name, "accumulator": args.accumulator, "scan": [cfg.Sy, cfg.Sx], "detector": [cfg.Q, cfg.Q], "K": cfg.K, "batch": batch,
        "readouts_per_scan": n_readouts, "scan_ms": total_ms, "frames_per_s": fps,
        "step_roofline_frames_per_s": peaks["hbm_gbs"] * 1e9 / (b_scan / cfg.S),
        "frac": fps / (peaks["hbm_gbs"] * 1e9 / (b_scan / cfg.S)),
        "ingest_latency_us": {"p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)),
                              "max": float(lat.max()), "n": int(len(lat))},
        "readout_latency_us": {"p50": float(np.percentile(rdl, 50)), "max": float(rdl.max()), "n": int(len(rdl))},
        "host_us_per_ingest_call": {"p50": float(np.percentile(host_us, 50)), "max": float(np.max(host_us))},
        "pool_frames": pool_n, "pool_bytes": pool_n * frame_bytes,
        "timing": "CUDA events on the ingest stream, eager calls; frames/s: median of %d scans without per-batch events; latencies: separate scans with events around every call" % args.reps,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
