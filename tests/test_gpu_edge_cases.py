"""GPU parity on the degenerate and boundary cases of the method (float64 oracle, same tolerance
as the main parity tests: relative L2 <= 1e-4; the active set bit-exact):
  * the smallest scan the plan accepts (2 x 2) and a 2 x 64 strip (one flush row at a time);
  * the basis size limit: L = Q rejected by the Gram check (R1), the largest accepted L run;
  * a readout after a single frame, and after frames that touch only one scan column;
  * frames of all zeros (the image is exactly zero) and one very bright pixel (counts >= 2^10
    take the second count plane of the exact u16 split);
  * ragged batch sizes (1, 7, 129 frames) on a u16 config."""
import numpy as np
import pytest

import oracle as O
from synth import CONFIGS, Acquisition

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel(a, b):
    nb = np.linalg.norm(np.asarray(b))
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    return torch


@pytest.fixture(scope="module")
def wdd():
    from paper_2212_01309_b200 import build
    build.build()
    import paper_2212_01309_b200 as w
    return w


def _oracle(cfg, fr, idx):
    return O.reduced_wdd(fr, idx, O.geometry(cfg), cfg.Sy, cfg.Sx, cfg.L, cfg.eps, return_all=True)


def _run(wdd, torch, cfg, fr, idx, batch):
    plan = wdd.Plan.from_config(cfg)
    dev = torch.from_numpy(np.ascontiguousarray(fr)).cuda()
    for a in range(0, len(idx), batch):
        plan.ingest(dev[a:a + batch], idx[a:a + batch])
    G, act = plan.get_accumulator()
    out = plan.readout()
    torch.cuda.synchronize()
    return plan, G.cpu().numpy(), act, out.cpu().numpy()


@pytest.mark.parametrize("Sy,Sx", [(2, 2), (2, 64), (64, 2)])
def test_tiny_scan_shapes(wdd, torch_cuda, Sy, Sx):
    cfg = CONFIGS["tiny"].with_(Sy=Sy, Sx=Sx)
    idx = np.arange(cfg.S)
    fr = Acquisition(cfg, noise=True).frames_parallel(idx)
    ref = _oracle(cfg, fr, idx)
    plan, G, act, img = _run(wdd, torch_cuda, cfg, fr, idx, 5)
    assert np.array_equal(np.sort(act), O.active_set(O.geometry(cfg), cfg.Sy, cfg.Sx))
    assert rel(G, ref["G"][act]) < TOL
    assert rel(img, ref["O"]) < TOL


def test_largest_basis_and_gram_rejection(wdd, torch_cuda):
    # L = Q would keep every detector degree of freedom, but the sampled Hermite-Gauss functions
    # of the self-reciprocal width (R1) are not orthonormal on so few pixels: the plan rejects
    # it (WDD_E_ARG, Gram check 1e-10).  The largest accepted basis at Q = 64 (L = 24) runs.
    cfg = CONFIGS["tiny"].with_(L=32, Sy=16, Sx=16)
    with pytest.raises(wdd.WddError):
        wdd.Plan.from_config(cfg)
    cfg = CONFIGS["tiny"].with_(Q=64, L=24, Sy=16, Sx=16)
    idx = np.arange(cfg.S)
    fr = Acquisition(cfg, noise=True).frames_parallel(idx)
    ref = _oracle(cfg, fr, idx)
    plan, G, act, img = _run(wdd, torch_cuda, cfg, fr, idx, 64)
    assert rel(G, ref["G"][act]) < TOL
    assert rel(img, ref["O"]) < TOL


def test_single_frame_and_single_column(wdd, torch_cuda):
    torch = torch_cuda
    cfg = CONFIGS["tiny"]
    one = np.array([cfg.Sx * 5 + 7])
    fr = Acquisition(cfg, noise=True).frames_parallel(one)
    ref = _oracle(cfg, fr, one)
    _, G, act, img = _run(wdd, torch, cfg, fr, one, 1)
    assert rel(G, ref["G"][act]) < TOL
    assert rel(img, ref["O"]) < TOL
    col = np.arange(3, cfg.S, cfg.Sx)                      # scan column sx = 3, every row
    fr = Acquisition(cfg, noise=True).frames_parallel(col)
    ref = _oracle(cfg, fr, col)
    _, G, act, img = _run(wdd, torch, cfg, fr, col, 8)
    assert rel(G, ref["G"][act]) < TOL
    assert rel(img, ref["O"]) < TOL


def test_zero_frames_give_zero_image(wdd, torch_cuda):
    torch = torch_cuda
    cfg = CONFIGS["medium"].with_(Sy=16, Sx=16)
    idx = np.arange(cfg.S)
    fr = np.zeros((cfg.S, cfg.Q, cfg.Q), dtype=np.uint16)
    _, G, act, img = _run(wdd, torch, cfg, fr, idx, 64)
    assert np.all(G == 0) and np.all(img == 0)


def test_bright_pixel_and_ragged_batches(wdd, torch_cuda):
    torch = torch_cuda
    cfg = CONFIGS["medium"].with_(Sy=16, Sx=16)
    idx = np.arange(cfg.S)
    fr = Acquisition(cfg, noise=True).frames_parallel(idx)
    fr[17, cfg.Q // 2, cfg.Q // 2 + 3] = 60000              # second count plane (>= 1024)
    fr[200, 5, 9] = 4097
    ref = _oracle(cfg, fr, idx)
    plan = wdd.Plan.from_config(cfg)
    dev = torch.from_numpy(fr).cuda()
    cuts = [0, 1, 8, 137, 138, cfg.S]                      # batches of 1, 7, 129, 1, 118 frames
    for a, b in zip(cuts, cuts[1:]):
        plan.ingest(dev[a:b], idx[a:b])
    G, act = plan.get_accumulator()
    out = plan.readout()
    torch.cuda.synchronize()
    assert rel(G.cpu().numpy(), ref["G"][act]) < TOL
    assert rel(out.cpu().numpy(), ref["O"]) < TOL
