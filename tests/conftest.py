import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running oracle test")


@pytest.fixture(scope="session")
def tiny_data():
    """Tiny config: noise-free and noisy frames for the whole scan, plus the phase."""
    import numpy as np
    from synth import CONFIGS, Acquisition
    cfg = CONFIGS["tiny"]
    idx = np.arange(cfg.S)
    clean = Acquisition(cfg, noise=False)
    noisy = Acquisition(cfg, noise=True)
    return dict(cfg=cfg, idx=idx, clean=clean.frames(idx), noisy=noisy.frames(idx),
                phi=clean.phase())
