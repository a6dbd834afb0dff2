"""GPU forward simulator throughput (synth/gpu.py): frames/s for one config, CUDA-event timed
over a batch after a warm-up.  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from synth import CONFIGS
    from synth import gpu as sim
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "live"]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    t0 = time.perf_counter()
    g = sim.GpuAcquisition(cfg)
    setup = time.perf_counter() - t0
    idx = np.arange(n) % cfg.S
    g.frames(idx[:256])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.frames(idx)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"config": cfg.name, "detector": cfg.Q, "frames": n, "ms": ms,
                      "frames_per_s": n / (ms / 1e3), "host_setup_s": setup}))


if __name__ == "__main__":
    main()
