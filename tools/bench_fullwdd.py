"""Conventional (full) WDD on the GPU (wdd_full_wdd) vs the reduced path on the same frames:
one whole-scan reconstruction, CUDA-event timed after a warm-up.  Prints one JSON line."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2212_01309_b200 as wdd
    from synth import CONFIGS
    from synth.sparse import dense_frames_torch, sparse_events
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "medium"]
    fr = torch.cat([dense_frames_torch(*sparse_events(9, np.arange(a, min(cfg.S, a + 4096)), cfg.Q), cfg.Q, "cuda")
                    for a in range(0, cfg.S, 4096)])
    plan = wdd.Plan.from_config(cfg)
    out = plan.full_wdd(fr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.full_wdd(fr, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    idx = np.arange(cfg.S, dtype=np.int32)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    plan.reset()
    plan.ingest(fr, idx)
    plan.readout()
    torch.cuda.synchronize()
    r0.record()
    plan.reset()
    plan.ingest(fr, idx)
    plan.readout()
    r1.record()
    torch.cuda.synchronize()
    print(json.dumps({"config": cfg.name, "full_wdd_ms": ms, "full_wdd_frames_per_s": cfg.S / (ms / 1e3),
                      "reduced_ms": r0.elapsed_time(r1), "scratch_GB": (cfg.S * 4 + cfg.Sy * (cfg.Sx // 2 + 1) * 8 + plan.n_act * 8) * cfg.Q * cfg.Q / 1e9}))


if __name__ == "__main__":
    main()
