"""GPU conventional (full) WDD (wdd_full_wdd) against the float64 F-oracle
(oracle.full_wdd: eq:deconv_mat P:90-95 + eq:extract P:97-106, explicit FFTs, no reduction) on the
same seeded frames.  Tolerance: relative L2 <= 1e-4 on the complex image and on the spectrum."""
import numpy as np
import pytest

import oracle as O
from synth import CONFIGS, Acquisition

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    from paper_2212_01309_b200 import build
    build.build()
    import paper_2212_01309_b200 as w
    return torch, w


@pytest.mark.parametrize("name,kw", [("tiny", {}), ("medium", dict(Sy=32, Sx=32, Q=64)),
                                     ("tiny", dict(Sy=24, Sx=40)), ("medium", dict(Sy=16, Sx=16, normalize=True)),
                                     ("tiny", dict(Sy=9, Sx=15))])   # (odd axes: the half-plane mirror indexing)
def test_full_wdd_matches_f_oracle(env, name, kw):
    torch, wdd = env
    kw = dict(kw)
    normalize = kw.pop("normalize", False)
    cfg = CONFIGS[name].with_(**kw)
    idx = np.arange(cfg.S)
    fr = Acquisition(cfg, noise=True).frames_parallel(idx)
    ref, x_ref = O.full_wdd(fr.reshape(cfg.Sy, cfg.Sx, cfg.Q, cfg.Q).astype(np.float64), O.geometry(cfg), cfg.eps,
                            normalize=normalize, return_spectrum=True)
    plan = wdd.Plan.from_config(cfg, normalize=normalize)
    out = plan.full_wdd(torch.from_numpy(np.ascontiguousarray(fr)).cuda())
    torch.cuda.synchronize()
    img = out.cpu().numpy()
    assert rel(img, ref) < 1e-4
    x = np.fft.fft2(np.conj(img.astype(np.complex128)), norm="ortho")
    if not normalize:
        assert rel(x, x_ref) < 1e-4
