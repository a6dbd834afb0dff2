"""Occupancy / lean-variant probe of the projection for every (Q, L): prints the resident CTAs per
SM the runtime reports and the kernel's shared memory (run with a build made with
WDD_NVCC_EXTRA=-DWDD_LEAN_SMEM=<bytes> to try other budgets)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01309_b200 as wdd
from synth import CONFIGS
for name in ("medium", "large", "live", "box"):
    cfg = CONFIGS[name].with_(Sy=16, Sx=16)
    p = wdd.Plan.from_config(cfg)
    print(name, cfg.Q, cfg.L, "ctas/SM", p.info()["proj_ctas_per_sm"])
    p.close()
