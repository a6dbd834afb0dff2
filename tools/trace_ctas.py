"""Per-CTA timeline of the projection kernel over one chained acquisition (trace build).

    WDD_NVCC_EXTRA=-DWDD_TRACE WDD_LIB_OUT=/tmp/libwdd_trace.so python -m paper_2212_01309_b200.build
    WDD_LIB=/tmp/libwdd_trace.so python tools/trace_ctas.py [config] [batch]
Reports the CTA durations split into setup (entry -> first TMA issue), streaming (first issue ->
last raw landing) and drain (last landing -> exit), the idle gaps between consecutive CTAs on
each SM, and the busy fraction of the SMs over the projection span."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "medium"]
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else (cfg.batch or 512)
    n = min(cfg.S, int(sys.argv[3]) if len(sys.argv) > 3 else 16384)
    lib = wdd.load_library()
    lib.wdd_trace_ctas.restype = ctypes.c_int
    rng = np.random.default_rng(0)
    fr = rng.poisson(0.2, size=(min(n, 16384), cfg.Q, cfg.Q)).astype(np.uint16)
    if n > len(fr):
        fr = np.concatenate([fr] * (n // len(fr)))
    dev = torch.from_numpy(fr).cuda()
    idx = np.arange(n, dtype=np.int32)
    spread = os.environ.get("TRACE_SPREAD", "0") == "1"     # the latency grid (opts.ingest_spread)
    plan = wdd.Plan.from_config(cfg, ingest_overlap=True, ingest_spread=spread)
    s = torch.cuda.Stream()
    buf = (ctypes.c_ulonglong * (8192 * 5))()
    torch.cuda.set_stream(s)
    plan.capture_begin(s)                        # graph-replayed, as bench.py times it
    plan.reset()
    for a in range(0, n, batch):
        plan.ingest(dev[a:a + batch], idx[a:a + batch], s)
    h = plan.capture_end()
    for rep in range(3):
        lib.wdd_trace_ctas(buf)
        plan.graph_launch(h, s)
        torch.cuda.synchronize()
        m = lib.wdd_trace_ctas(buf)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 5)[:m].astype(np.float64)
    t0 = t[:, 0].min()
    ent, iss, land, ext, sm = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, (t[:, 3] - t0) / 1e3, t[:, 4]
    span = ext.max()
    print(f"{cfg.name} batch {batch}: {m} CTAs, span {span:.1f} us, frames {n}")
    print(f"  CTA duration mean {np.mean(ext - ent):.2f} us; setup (entry->1st issue) {np.mean(iss - ent):.2f}; "
          f"stream (1st issue->last landing) {np.mean(land - iss):.2f}; drain (last landing->exit) {np.mean(ext - land):.2f}")
    gaps = []
    for k in np.unique(sm):
        o = np.argsort(ent[sm == k])
        e, x = ent[sm == k][o], ext[sm == k][o]
        gaps += list(e[1:] - x[:-1])
    gaps = np.array(gaps)
    if len(gaps):
        print(f"  SMs used {len(np.unique(sm))}; idle gap between CTAs on an SM: mean {gaps.mean():.2f} us, "
              f"p90 {np.percentile(gaps, 90):.2f}, total {gaps.sum():.1f} SM-us")
    else:
        print(f"  SMs used {len(np.unique(sm))}; one CTA per SM")
    print(f"  per-CTA setup p50 / max {np.median(iss - ent):.2f} / {np.max(iss - ent):.2f} us; first landing "
          f"-> exit p50 {np.median(ext - land):.2f}; entry spread {ent.max() - ent.min():.2f} us; exit spread "
          f"{ext.max() - ext.min():.2f} us")
    busy = np.sum(ext - ent)
    print(f"  SM busy fraction over the span: {busy / (148 * span):.3f}; first entry->all SMs busy, "
          f"last-CTA start {ent.max():.1f} us, first exit {ext.min():.1f} us")
    # busy SM count over time
    ts = np.linspace(0, span, 21)
    print("  busy SMs at t = " + " ".join(f"{int(np.sum((ent <= x) & (ext > x)))}" for x in ts))


if __name__ == "__main__":
    main()
